"""Model geometry for the TP-reconfiguration data path.

The reference's only model geometry is ``PerfProfile`` (pkg/src/tpsim/profile.py:21-45):
``total_kv_heads``, ``kv_bytes_per_token_per_head``, ``weight_full_copy_gb``,
``gpu_memory_gb``, ``tp_levels``, with the check that every TP level divides the
KV-head count (profile.py:41-45). Here the byte figures are derived from the
architecture they summarise (layers x K/V x head_dim x dtype), because the
data path needs the layout, not just the product.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .migration import MigrationError

MAX_TP = 8  # weights are stored in 1/MAX_TP slices of their split dimension


@dataclass(frozen=True)
class KvGeometry:
    """Paged KV pool geometry.

    One pool unit ("page") holds one KV head x ``block_tokens`` tokens x all
    layers x {K, V}, laid out [layer][K|V][token][head_dim]. A page's plane of
    one (layer, K|V) is ``block_tokens * head_dim * dtype_bytes`` contiguous
    bytes, which is what an attention kernel reads per layer.
    """

    layers: int
    head_dim: int
    total_heads: int
    dtype_bytes: int = 2
    block_tokens: int = 16

    @property
    def kv_bytes_per_token_per_head(self) -> int:
        """``PerfProfile.kv_bytes_per_token_per_head`` (profile.py:33)."""
        return self.layers * 2 * self.head_dim * self.dtype_bytes

    @property
    def tok_bytes(self) -> int:
        return self.head_dim * self.dtype_bytes

    @property
    def plane_bytes(self) -> int:
        return self.block_tokens * self.tok_bytes

    @property
    def unit_bytes(self) -> int:
        return self.block_tokens * self.kv_bytes_per_token_per_head

    def blocks(self, context_len: int) -> int:
        return -(-int(context_len) // self.block_tokens)


@dataclass(frozen=True)
class MatrixSpec:
    """One weight matrix of the model and how TP splits it.

    split: "col"  column-parallel (QKV, gate/up, vocab-parallel embedding and
                  lm_head): each rank holds a contiguous range of ROWS
                  (output features / vocab entries);
           "row"  row-parallel (O, down): each rank holds a contiguous range
                  of COLUMNS (input features);
           "rep"  replicated (norms).
    """

    name: str
    layer: int
    rows: int
    cols: int
    split: str
    key: int  # pattern key of the synthetic full matrix

    @property
    def split_len(self) -> int:
        return self.rows if self.split == "col" else self.cols


@dataclass(frozen=True)
class ModelGeometry:
    name: str
    layers: int
    hidden: int
    intermediate: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    dtype_bytes: int = 2
    gpu_memory_gb: float = 180.0
    tp_levels: tuple[int, ...] = (1, 2, 4, 8)
    matrices: tuple[MatrixSpec, ...] = field(default=(), compare=False, repr=False)

    def __post_init__(self):
        for tp in self.tp_levels:
            if self.n_kv_heads % tp:
                raise MigrationError(
                    f"total_kv_heads={self.n_kv_heads} not divisible by tp={tp}")
        if not self.matrices:
            object.__setattr__(self, "matrices", tuple(_catalog(self)))
        for m in self.matrices:
            if m.split != "rep" and m.split_len % MAX_TP:
                raise MigrationError(f"{m.name}: split dim {m.split_len} not divisible by {MAX_TP}")

    # -- PerfProfile-compatible geometry (profile.py:21-45) -------------------
    @property
    def total_kv_heads(self) -> int:
        return self.n_kv_heads

    @property
    def kv_bytes_per_token_per_head(self) -> int:
        return self.kv.kv_bytes_per_token_per_head

    @property
    def weight_full_copy_gb(self) -> float:
        return self.weight_bytes / 1e9

    @property
    def kv(self) -> KvGeometry:
        return KvGeometry(layers=self.layers, head_dim=self.head_dim,
                          total_heads=self.n_kv_heads, dtype_bytes=self.dtype_bytes)

    @property
    def weight_bytes(self) -> int:
        return sum(m.rows * m.cols for m in self.matrices) * self.dtype_bytes

    @property
    def params(self) -> int:
        return sum(m.rows * m.cols for m in self.matrices)


def _key(name: str, layer: int) -> int:
    h = 0xCBF29CE484222325
    for ch in f"{name}/{layer}".encode():
        h = ((h ^ ch) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _catalog(g: ModelGeometry) -> list[MatrixSpec]:
    """Llama-style decoder weights with Megatron/SGLang TP conventions."""
    q = g.n_heads * g.head_dim
    kv = g.n_kv_heads * g.head_dim
    h, f = g.hidden, g.intermediate
    out = [MatrixSpec("embed_tokens", -1, g.vocab, h, "col", _key("embed_tokens", -1))]
    for layer in range(g.layers):
        for name, rows, cols, split in (
            ("input_layernorm", 1, h, "rep"),
            ("q_proj", q, h, "col"),
            ("k_proj", kv, h, "col"),
            ("v_proj", kv, h, "col"),
            ("o_proj", h, q, "row"),
            ("post_attention_layernorm", 1, h, "rep"),
            ("gate_proj", f, h, "col"),
            ("up_proj", f, h, "col"),
            ("down_proj", h, f, "row"),
        ):
            out.append(MatrixSpec(name, layer, rows, cols, split, _key(name, layer)))
    out.append(MatrixSpec("norm", -1, 1, h, "rep", _key("norm", -1)))
    out.append(MatrixSpec("lm_head", -1, g.vocab, h, "col", _key("lm_head", -1)))
    return out


LLAMA_3_1_8B = ModelGeometry(
    name="Llama-3.1-8B", layers=32, hidden=4096, intermediate=14336, n_heads=32,
    n_kv_heads=8, head_dim=128, vocab=128256,
)
LLAMA_3_1_70B = ModelGeometry(
    name="Llama-3.1-70B", layers=80, hidden=8192, intermediate=28672, n_heads=64,
    n_kv_heads=8, head_dim=128, vocab=128256,
)


def tiny_geometry(layers: int = 2, hidden: int = 256, intermediate: int = 512, n_heads: int = 8,
                  n_kv_heads: int = 8, head_dim: int = 32, vocab: int = 1024) -> ModelGeometry:
    """A small Llama-shaped model for parity tests at oracle-friendly sizes."""
    return ModelGeometry(name=f"tiny-{layers}x{hidden}", layers=layers, hidden=hidden,
                         intermediate=intermediate, n_heads=n_heads, n_kv_heads=n_kv_heads,
                         head_dim=head_dim, vocab=vocab)


MODELS = {m.name: m for m in (LLAMA_3_1_8B, LLAMA_3_1_70B)}
