"""Sharded weight store and TP-aware weight reshard (K2).

The reference models weights only as GB per GPU (``weight_memory``,
migration.py:295-306: full copy, per-TP copies, or ``full/tp`` when sharded)
and as a fixed ``reload_ms`` on a naive switch (migration.py:85, 288-289).
The paper keeps one full copy per GPU and selects the TP shard at execution
time. This store realises both regimes on B200:

* every non-replicated matrix is cut into MAX_TP=8 equal slices of its split
  dimension: ROWS for column-parallel matrices (q/k/v, gate/up, vocab-parallel
  embedding and lm_head), COLUMNS for row-parallel ones (o, down). Rank r of a
  TP-N group uses slices [r*8/N, (r+1)*8/N) -- the same contiguous 1/N that
  Megatron/SGLang give rank r, and for k/v the rows of exactly the KV heads
  that ``KvLayout`` puts on that rank (migration.py:27);
* a GPU holds one *resident* slice range [a, b) of every matrix in one arena,
  laid out matrix by matrix: column-parallel slices as contiguous rows,
  row-parallel slices as a [rows, (b-a)*cols/8] block;
* a reshard reuses resident slices in place -- if the new shard lies inside
  the resident range the new shard is just a view (zero bytes moved) -- and
  otherwise builds a new arena from local slices plus slices fetched from
  peers that hold them (egress balanced across holders). That copy list is
  executed by K2 (``tpr_weight_reshard``) as one batched 2-D strided copy.

``mode="full_copy_per_gpu"`` makes every GPU resident on all 8 slices: every
switch is then views only (the paper's zero-overhead weight switching).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native
from .geometry import MAX_TP, ModelGeometry
from .migration import MigrationError

CHUNK_BYTES = int(os.environ.get("TPR_K2_CHUNK", 32 * 1024))  # K2 work-item size (bytes)


@dataclass
class ReshardStats:
    local_bytes: int = 0    # bytes copied from the GPU's own old arena
    remote_bytes: int = 0   # bytes fetched from peers (NVLink in multi-GPU mode)
    segments: int = 0
    views: int = 0          # GPUs whose new shard is a view of resident slices
    egress: dict = field(default_factory=dict)   # gpu -> bytes sent to peers
    ingress: dict = field(default_factory=dict)  # gpu -> bytes fetched

    @property
    def bytes(self) -> int:
        return self.local_bytes + self.remote_bytes


def groups_ranges(groups: Sequence[Sequence[int]]) -> dict[int, tuple[int, int]]:
    """Active slice range of every GPU for a set of TP groups."""
    out = {}
    for grp in groups:
        n = len(grp)
        if n < 1 or MAX_TP % n:
            raise MigrationError(f"tp={n} must divide {MAX_TP}")
        per = MAX_TP // n
        for r, g in enumerate(grp):
            if g in out:
                raise MigrationError(f"gpu {g} appears in two groups")
            out[g] = (r * per, (r + 1) * per)
    return out


class ShardedWeightStore:
    def __init__(self, model: ModelGeometry, gpu_ids: Sequence[int],
                 device: str | torch.device = "cuda", devices: dict | None = None,
                 mode: str = "sharded"):
        if mode not in ("sharded", "full_copy_per_gpu"):
            raise MigrationError(f"unknown weight storage mode {mode!r}")
        _native.load()
        self.model = model
        self.mode = mode
        self.gpu_ids = tuple(gpu_ids)
        default = torch.device(device)
        self.device_of = {g: torch.device(devices[g]) if devices else default for g in self.gpu_ids}
        es = model.dtype_bytes
        self.split = [m for m in model.matrices if m.split != "rep"]
        self.replicated = [m for m in model.matrices if m.split == "rep"]
        # per-matrix bytes of ONE slice and its offset inside a one-slice arena
        self.slice_bytes = np.array(
            [(m.rows // MAX_TP) * m.cols * es if m.split == "col" else m.rows * (m.cols // MAX_TP) * es
             for m in self.split], dtype=np.int64)
        self.slice_off = np.concatenate([[0], np.cumsum(self.slice_bytes)[:-1]]).astype(np.int64)
        self.bytes_per_slice = int(self.slice_bytes.sum())
        self.is_col = np.array([m.split == "col" for m in self.split])
        self._step = np.where(self.is_col, self.slice_bytes,
                              np.array([m.cols // MAX_TP for m in self.split], np.int64) * es)
        self._seg_rows = np.where(self.is_col, 1, np.array([m.rows for m in self.split], np.int64))
        self.rows = np.array([m.rows for m in self.split], dtype=np.int64)
        self.cols = np.array([m.cols for m in self.split], dtype=np.int64)
        self.index = {(m.name, m.layer): i for i, m in enumerate(self.split)}
        self.rep_index = {(m.name, m.layer): i for i, m in enumerate(self.replicated)}
        self.resident: dict[int, tuple[int, int]] = {}
        self.active: dict[int, tuple[int, int]] = {}
        self.arena: dict[int, torch.Tensor] = {}
        self.rep_arena: dict[int, torch.Tensor] = {}
        self._segs_dev = {}  # device -> (pinned staging, device scratch) for K2 segments

    # ----------------------------------------------------------------- load
    def load(self, groups: Sequence[Sequence[int]], stream: torch.cuda.Stream | None = None) -> None:
        """Materialise the initial shards (synthetic weights) for ``groups``."""
        act = groups_ranges(groups)
        if set(act) != set(self.gpu_ids):
            raise MigrationError("groups must cover exactly the store's GPUs")
        self.arena.clear()
        for g in self.gpu_ids:
            res = (0, MAX_TP) if self.mode == "full_copy_per_gpu" else act[g]
            dev = self.device_of[g]
            st = stream or torch.cuda.current_stream(dev)
            self.arena[g] = torch.empty((res[1] - res[0]) * self.bytes_per_slice, dtype=torch.uint8,
                                        device=dev)
            self.resident[g] = res
            self.active[g] = act[g]
            rep_bytes = sum(m.rows * m.cols for m in self.replicated) * self.model.dtype_bytes
            self.rep_arena[g] = torch.empty(max(rep_bytes, 16), dtype=torch.uint8, device=dev)
            with torch.cuda.device(dev):
                self._fill(g, st)

    def _fill(self, g: int, st: torch.cuda.Stream) -> None:
        a, b = self.resident[g]
        s = b - a
        es = self.model.dtype_bytes
        base = self.arena[g].data_ptr()
        for i, m in enumerate(self.split):
            ptr = base + s * int(self.slice_off[i])
            if m.split == "col":
                rows = s * (m.rows // MAX_TP)
                args = (ptr, rows, m.cols, m.cols, a * (m.rows // MAX_TP), 0)
            else:
                cols = s * (m.cols // MAX_TP)
                args = (ptr, m.rows, cols, cols, 0, a * (m.cols // MAX_TP))
            _native.call("tpr_matrix_fill", *args, m.cols, m.key, es, st.cuda_stream)
        off = 0
        rbase = self.rep_arena[g].data_ptr()
        for m in self.replicated:
            _native.call("tpr_matrix_fill", rbase + off, m.rows, m.cols, m.cols, 0, 0, m.cols, m.key,
                         es, st.cuda_stream)
            off += m.rows * m.cols * es

    # ---------------------------------------------------------------- views
    def shard(self, gpu: int, name: str, layer: int = -1) -> torch.Tensor:
        """The TP shard GPU ``gpu`` computes with (a view; never a copy)."""
        es = self.model.dtype_bytes
        dtype = {1: torch.uint8, 2: torch.bfloat16, 4: torch.float32}[es]
        if (name, layer) in self.rep_index:
            off = 0
            for m in self.replicated[: self.rep_index[(name, layer)]]:
                off += m.rows * m.cols * es
            m = self.replicated[self.rep_index[(name, layer)]]
            return self.rep_arena[gpu][off: off + m.rows * m.cols * es].view(dtype).view(m.rows, m.cols)
        i = self.index[(name, layer)]
        m = self.split[i]
        a, b = self.resident[gpu]
        x, y = self.active[gpu]
        s = b - a
        lo = s * int(self.slice_off[i])
        mat = self.arena[gpu][lo: lo + s * int(self.slice_bytes[i])].view(dtype)
        if m.split == "col":
            rps = m.rows // MAX_TP
            return mat.view(s * rps, m.cols)[(x - a) * rps:(y - a) * rps]
        cps = m.cols // MAX_TP
        return mat.view(m.rows, s * cps)[:, (x - a) * cps:(y - a) * cps]

    def memory_bytes(self, gpu: int) -> int:
        a, b = self.resident[gpu]
        return (b - a) * self.bytes_per_slice + self.rep_arena[gpu].numel()

    # -------------------------------------------------------------- reshard
    def plan(self, new_groups: Sequence[Sequence[int]], parked: Sequence[int] = (),
             trim: bool = False):
        """Host reshard planner: new resident ranges, sources of missing slices.

        ``parked`` GPUs leave service (scale-in): they keep their resident
        slices, which stay available as sources. ``trim`` shrinks a GPU whose
        resident range is larger than its new shard to exactly that shard (a
        local compaction copy that frees the extra slices, e.g. for KV pages);
        without it the shard is a view and the extra slices stay resident for
        reuse by a later switch. Returns (new_active,
        new_resident, moves) where moves[g] is a list of (src_gpu, slice_lo,
        slice_hi) runs building g's new arena (empty when the new shard is a
        view of resident slices).
        """
        act = groups_ranges(new_groups)
        if set(act) | set(parked) != set(self.gpu_ids) or set(act) & set(parked):
            raise MigrationError("groups + parked GPUs must cover exactly the store's GPUs")
        egress = {g: 0 for g in self.gpu_ids}
        new_res, moves = {}, {}
        for g in self.gpu_ids:
            if g in parked:
                new_res[g] = self.resident[g]
                moves[g] = []
                continue
            x, y = act[g]
            a, b = self.resident[g]
            if a <= x and y <= b and not (trim and (a, b) != (x, y)):
                new_res[g] = (a, b)
                moves[g] = []
                continue
            new_res[g] = (x, y)
            runs = []
            for sl in range(x, y):
                if a <= sl < b:
                    src = g
                else:
                    holders = [h for h in self.gpu_ids
                               if h != g and self.resident[h][0] <= sl < self.resident[h][1]]
                    if not holders:
                        raise MigrationError(f"weight slice {sl} is resident nowhere")
                    src = min(holders, key=lambda h: (egress[h], self.gpu_ids.index(h)))
                    egress[src] += self.bytes_per_slice
                if runs and runs[-1][0] == src and runs[-1][2] == sl:
                    runs[-1][2] = sl + 1
                else:
                    runs.append([src, sl, sl + 1])
            moves[g] = [tuple(r) for r in runs]
        return act, new_res, moves

    def _segments(self, g: int, new_res, moves, new_arena: torch.Tensor) -> np.ndarray:
        """Copy segments (uint64/int64 x 8 per row, tpr_copy_seg_t layout)."""
        x, y = new_res[g]
        s_new = y - x
        dbase = new_arena.data_ptr()
        # Within a matrix region of an arena holding s slices, slice k starts at
        # k * step: whole rows for column-parallel matrices (step = one slice,
        # contiguous), a column block for row-parallel ones (step = cols/8
        # elements, rows strided by s * step).
        step = self._step
        runs = moves[g]
        seg = np.zeros((len(runs), len(self.split), 8), dtype=np.int64)
        for i, (src, lo, hi) in enumerate(runs):
            ha, hb = self.resident[src]
            s_src = hb - ha
            row_bytes = (hi - lo) * step
            seg[i, :, 0] = self.arena[src].data_ptr() + s_src * self.slice_off + (lo - ha) * step
            seg[i, :, 1] = dbase + s_new * self.slice_off + (lo - x) * step
            seg[i, :, 2] = self._seg_rows
            seg[i, :, 3] = row_bytes
            seg[i, :, 4] = np.where(self.is_col, row_bytes, s_src * step)
            seg[i, :, 5] = np.where(self.is_col, row_bytes, s_new * step)
        return seg.reshape(-1, 8)

    def reshard(self, new_groups: Sequence[Sequence[int]], stream: torch.cuda.Stream | None = None,
                events: tuple | None = None, parked: Sequence[int] = (),
                trim: bool = False) -> ReshardStats:
        """Move to ``new_groups``: K2 copies for every GPU whose new shard is not
        resident; views for the rest. Stream-ordered, no host sync: new arenas
        are allocated and old ones released on ``stream`` (the caching
        allocator reuses a block on the same stream only after the K2 that
        last touched it), so the host may run ahead without holding memory."""
        act, new_res, moves = self.plan(new_groups, parked, trim)
        for g in parked:
            act[g] = new_res[g]
        stats = ReshardStats(egress={g: 0 for g in self.gpu_ids}, ingress={g: 0 for g in self.gpu_ids})
        devs = {self.device_of[g] for g in self.gpu_ids}
        if len(devs) != 1:
            raise MigrationError("multi-device weight reshard goes through the distributed executor")
        dev = next(iter(devs))
        stream = stream or torch.cuda.current_stream(dev)
        new_arena, segs = {}, []
        for g in self.gpu_ids:
            if not moves[g]:
                stats.views += 1
                continue
            x, y = new_res[g]
            with torch.cuda.stream(stream):
                new_arena[g] = torch.empty((y - x) * self.bytes_per_slice, dtype=torch.uint8,
                                           device=dev)
            segs.append(self._segments(g, new_res, moves, new_arena[g]))
            for src, lo, hi in moves[g]:
                nb = (hi - lo) * self.bytes_per_slice
                if src == g:
                    stats.local_bytes += nb
                else:
                    stats.remote_bytes += nb
                    stats.egress[src] += nb
                    stats.ingress[g] += nb
        if events:
            events[0].record(stream)
        if segs:
            seg = np.ascontiguousarray(np.concatenate(segs))
            stats.segments = len(seg)
            self._launch(seg, dev, stream)
        if events:
            events[1].record(stream)
        for g, t in new_arena.items():
            if self.arena[g].device == dev:
                self.arena[g].record_stream(stream)
            self.arena[g] = t
        self.resident = new_res
        self.active = act
        self._stream = stream
        return stats

    def _launch(self, seg: np.ndarray, dev: torch.device, stream: torch.cuda.Stream) -> None:
        """Normalise segments (host), upload segments + item prefix through
        pinned staging, launch K2."""
        from .kvcache import _PinnedStaging, _Scratch

        n = len(seg)
        # segments | prefix[n + 1] | dynamic-claim counter (uploaded as 0)
        buf = np.empty(seg.size + n + 2, dtype=np.int64)
        buf[: seg.size] = seg.reshape(-1)
        buf[-1] = 0
        n_items = ctypes.c_int64(0)
        _native.call("tpr_copy_prepare", buf.ctypes.data, n, CHUNK_BYTES,
                     buf.ctypes.data + seg.nbytes, ctypes.byref(n_items))
        if dev not in self._segs_dev:
            self._segs_dev[dev] = (_PinnedStaging(), _Scratch(torch.int64, dev))
        staging, scratch = self._segs_dev[dev]
        d = scratch.get(buf.size, stream)
        with torch.cuda.device(dev):
            staging.upload(buf, d, stream)
            _native.call("tpr_weight_reshard", d.data_ptr(), d.data_ptr() + seg.nbytes, n,
                         n_items.value, CHUNK_BYTES, d.data_ptr() + 8 * (buf.size - 1),
                         stream.cuda_stream)

    def finish(self) -> None:
        """Wait for the last reshard's copies."""
        if getattr(self, "_stream", None) is not None:
            self._stream.synchronize()

    # ------------------------------------------------------------- checking
    def verify(self, stream: torch.cuda.Stream | None = None) -> int:
        """Pattern check of every GPU's active shards (host sync). Returns the
        number of mismatching elements (0 = bit-exact)."""
        es = self.model.dtype_bytes
        total = 0
        for g in self.gpu_ids:
            dev = self.device_of[g]
            st = stream or torch.cuda.current_stream(dev)
            bad = torch.zeros(1, dtype=torch.int64, device=dev)
            x, y = self.active[g]
            for m in self.split:
                v = self.shard(g, m.name, m.layer)
                if m.split == "col":
                    r0, c0 = x * (m.rows // MAX_TP), 0
                else:
                    r0, c0 = 0, x * (m.cols // MAX_TP)
                with torch.cuda.device(dev):
                    _native.call("tpr_matrix_verify", v.data_ptr(), v.shape[0], v.shape[1],
                                 v.stride(0), r0, c0, m.cols, m.key, es, bad.data_ptr(),
                                 st.cuda_stream)
            for m in self.replicated:
                v = self.shard(g, m.name, m.layer)
                with torch.cuda.device(dev):
                    _native.call("tpr_matrix_verify", v.data_ptr(), m.rows, m.cols, m.cols, 0, 0,
                                 m.cols, m.key, es, bad.data_ptr(), st.cuda_stream)
            total += int(bad.item())
        return total
