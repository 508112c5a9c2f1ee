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
* a GPU's arena is slice-addressed: it holds one aligned *window* of
  ``max_slices`` slices of every matrix, laid out matrix by matrix
  (column-parallel: [window * rows/8, cols] rows; row-parallel: a
  [rows, window * cols/8] block), and slice k sits at position k - base
  whether or not the GPU holds it. A shard [x, y) inside the window is a
  contiguous row range / a strided column block: a view the GEMMs read;
* a reshard reuses resident slices in place: a shard that is resident is a
  view (zero bytes); a shard that grows inside the window keeps its resident
  slices where they are and K2 fetches only the missing slices into their
  positions, from peers that hold them (egress balanced across holders). That
  copy list is executed by K2 (``tpr_weight_reshard_host``) as one batched 2-D
  strided copy. Only a shard that outgrows its window needs a new arena and a
  local relayout copy (``ReshardStats.local_bytes``).

``mode="full_copy_per_gpu"`` makes every GPU resident on all 8 slices: every
switch is then views only (the paper's zero-overhead weight switching).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _native
from .geometry import MAX_TP, ModelGeometry
from .migration import MigrationError

CHUNK_BYTES = 32 * 1024  # K2 work-item size (bytes): one ring stage


@dataclass
class ReshardStats:
    local_bytes: int = 0    # relayout copies inside a GPU (only when a shard outgrows its window)
    remote_bytes: int = 0   # missing slices fetched from peers (NVLink in multi-GPU mode)
    segments: int = 0
    views: int = 0          # GPUs whose new shard is a view of resident slices
    in_place: int = 0       # GPUs that grew their shard in place (fetches only)
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


def window_for(x: int, y: int, m: int) -> tuple[int, int]:
    """The m-slice window (base, m) holding shard [x, y): shards are aligned to
    their size (rank r of TP-N holds [r*8/N, (r+1)*8/N)), so with m a power of
    two >= y - x the aligned window floor(x / m) * m contains the shard, and
    two shards either share a window or are disjoint."""
    m = max(m, y - x)
    return (x // m) * m, m


@dataclass
class ReshardPlan:
    """Host reshard plan (``ShardedWeightStore.plan``).

    active[g] / have[g] / window[g]: the new shard, resident slices and arena
    window of every GPU; fetch[g]: runs (src gpu, lo, hi) of missing slices;
    relayout[g]: g needs a new arena (its shard left its window), and then
    local[g] lists the resident slices copied into it."""

    active: dict
    have: dict
    window: dict
    fetch: dict
    relayout: dict
    local: dict


class ShardedWeightStore:
    def __init__(self, model: ModelGeometry, gpu_ids: Sequence[int],
                 device: str | torch.device = "cuda", devices: dict | None = None,
                 mode: str = "sharded", max_slices=MAX_TP):
        """``max_slices``: the window of every GPU's arena, in slices (an int for
        all or {gpu: int}; a power of two dividing 8). An arena holds one window
        of every matrix, slice-addressed, so a shard that grows inside its
        window keeps its resident slices in place and only the missing slices
        are fetched. Default: the whole matrix (never a relayout copy)."""
        if mode not in ("sharded", "full_copy_per_gpu"):
            raise MigrationError(f"unknown weight storage mode {mode!r}")
        _native.load()
        self.model = model
        self.mode = mode
        self.gpu_ids = tuple(gpu_ids)
        default = torch.device(device)
        self.device_of = {g: torch.device(devices[g]) if devices else default for g in self.gpu_ids}
        ms = max_slices if isinstance(max_slices, dict) else {g: max_slices for g in self.gpu_ids}
        self.max_slices = {g: MAX_TP if mode == "full_copy_per_gpu" else int(ms[g])
                           for g in self.gpu_ids}
        for g, m in self.max_slices.items():
            if m < 1 or MAX_TP % m:
                raise MigrationError(f"gpu {g}: max_slices={m} must divide {MAX_TP}")
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
        # slice k of a matrix region starts at k * step: whole rows for a
        # column-parallel matrix (contiguous), a column block for a row-parallel
        # one (rows strided by window * step)
        self._step = np.where(self.is_col, self.slice_bytes,
                              np.array([m.cols // MAX_TP for m in self.split], np.int64) * es)
        self._seg_rows = np.where(self.is_col, 1, np.array([m.rows for m in self.split], np.int64))
        self.rows = np.array([m.rows for m in self.split], dtype=np.int64)
        self.cols = np.array([m.cols for m in self.split], dtype=np.int64)
        self.index = {(m.name, m.layer): i for i, m in enumerate(self.split)}
        self.rep_index = {(m.name, m.layer): i for i, m in enumerate(self.replicated)}
        self.have: dict[int, frozenset] = {}
        self.window: dict[int, tuple[int, int]] = {}
        self.active: dict[int, tuple[int, int]] = {}
        self.arena: dict[int, torch.Tensor] = {}
        self.rep_arena: dict[int, torch.Tensor] = {}
        self._segs_dev = {}  # device -> (pinned staging, device scratch) for K2 segments

    @property
    def resident(self) -> dict[int, tuple[int, int]]:
        """[lo, hi) hull of every GPU's resident slices."""
        return {g: (min(h), max(h) + 1) for g, h in self.have.items()}

    # ----------------------------------------------------------------- load
    def load(self, groups: Sequence[Sequence[int]], stream: torch.cuda.Stream | None = None) -> None:
        """Materialise the initial shards (synthetic weights) for ``groups``."""
        act = groups_ranges(groups)
        if set(act) != set(self.gpu_ids):
            raise MigrationError("groups must cover exactly the store's GPUs")
        self.arena.clear()
        for g in self.gpu_ids:
            res = (0, MAX_TP) if self.mode == "full_copy_per_gpu" else act[g]
            self.window[g] = window_for(*res, self.max_slices[g])
            self.have[g] = frozenset(range(*res))
            self.active[g] = act[g]
            dev = self.device_of[g]
            st = stream or torch.cuda.current_stream(dev)
            self.arena[g] = torch.empty(self.window[g][1] * self.bytes_per_slice, dtype=torch.uint8,
                                        device=dev)
            rep_bytes = sum(m.rows * m.cols for m in self.replicated) * self.model.dtype_bytes
            self.rep_arena[g] = torch.empty(max(rep_bytes, 16), dtype=torch.uint8, device=dev)
            with torch.cuda.device(dev):
                self._fill(g, st, *res)

    def _fill(self, g: int, st: torch.cuda.Stream, a: int, b: int) -> None:
        """Synthetic content of slices [a, b) at their window positions."""
        w0, m_ = self.window[g]
        es = self.model.dtype_bytes
        base = self.arena[g].data_ptr()
        for i, m in enumerate(self.split):
            ptr = base + m_ * int(self.slice_off[i]) + (a - w0) * int(self._step[i])
            if m.split == "col":
                rows = (b - a) * (m.rows // MAX_TP)
                args = (ptr, rows, m.cols, m.cols, a * (m.rows // MAX_TP), 0)
            else:
                cps = m.cols // MAX_TP
                args = (ptr, m.rows, (b - a) * cps, m_ * cps, 0, a * cps)
            _native.call("tpr_matrix_fill", *args, m.cols, m.key, es, st.cuda_stream)
        off = 0
        rbase = self.rep_arena[g].data_ptr()
        for m in self.replicated:
            _native.call("tpr_matrix_fill", rbase + off, m.rows, m.cols, m.cols, 0, 0, m.cols, m.key,
                         es, st.cuda_stream)
            off += m.rows * m.cols * es

    # ---------------------------------------------------------------- views
    def slices(self, gpu: int, name: str, layer: int, x: int, y: int) -> torch.Tensor:
        """View of slices [x, y) of one matrix on ``gpu`` (all resident)."""
        es = self.model.dtype_bytes
        dtype = {1: torch.uint8, 2: torch.bfloat16, 4: torch.float32}[es]
        i = self.index[(name, layer)]
        m = self.split[i]
        w0, m_ = self.window[gpu]
        if not all(s in self.have[gpu] for s in range(x, y)):
            raise MigrationError(f"gpu {gpu}: slices [{x}, {y}) of {name} are not resident")
        lo = m_ * int(self.slice_off[i])
        mat = self.arena[gpu][lo: lo + m_ * int(self.slice_bytes[i])].view(dtype)
        if m.split == "col":
            rps = m.rows // MAX_TP
            return mat.view(m_ * rps, m.cols)[(x - w0) * rps:(y - w0) * rps]
        cps = m.cols // MAX_TP
        return mat.view(m.rows, m_ * cps)[:, (x - w0) * cps:(y - w0) * cps]

    def shard(self, gpu: int, name: str, layer: int = -1) -> torch.Tensor:
        """The TP shard GPU ``gpu`` computes with (a view; never a copy). A
        row-parallel shard is a strided view (row pitch = the window)."""
        es = self.model.dtype_bytes
        dtype = {1: torch.uint8, 2: torch.bfloat16, 4: torch.float32}[es]
        if (name, layer) in self.rep_index:
            off = 0
            for m in self.replicated[: self.rep_index[(name, layer)]]:
                off += m.rows * m.cols * es
            m = self.replicated[self.rep_index[(name, layer)]]
            return self.rep_arena[gpu][off: off + m.rows * m.cols * es].view(dtype).view(m.rows, m.cols)
        return self.slices(gpu, name, layer, *self.active[gpu])

    def memory_bytes(self, gpu: int) -> int:
        return self.window[gpu][1] * self.bytes_per_slice + self.rep_arena[gpu].numel()

    # -------------------------------------------------------------- reshard
    def plan(self, new_groups: Sequence[Sequence[int]], parked: Sequence[int] = (),
             trim: bool = False) -> ReshardPlan:
        """Host reshard planner.

        A GPU whose new shard is resident is a view (0 bytes). A shard that
        grows inside its arena window keeps every resident slice in place and
        fetches only the missing slices (weight_memory("sharded"),
        migration.py:295-306: the new shard is full/tp, and what is already
        there is not moved), from peers that hold them, balancing egress. A
        shard that leaves its window (or outgrows it) gets a new arena: by the
        alignment of shards it shares no slice with the old window unless it
        outgrew it, and only then are resident slices copied (``local``).

        ``parked`` GPUs leave service (scale-in) and keep their slices as
        sources. ``trim`` drops every resident slice outside the new shard
        (bookkeeping only: the arena keeps its window), so a later switch
        fetches them again."""
        act = groups_ranges(new_groups)
        if set(act) | set(parked) != set(self.gpu_ids) or set(act) & set(parked):
            raise MigrationError("groups + parked GPUs must cover exactly the store's GPUs")
        egress = {g: 0 for g in self.gpu_ids}
        out = ReshardPlan(dict(act), {}, {}, {}, {}, {})
        for g in self.gpu_ids:
            have, win = self.have[g], self.window[g]
            out.fetch[g], out.local[g], out.relayout[g] = [], [], False
            if g in parked:
                out.active[g] = self.active[g]
                out.have[g], out.window[g] = have, win
                continue
            x, y = act[g]
            shard = frozenset(range(x, y))
            w0, m_ = win
            if w0 <= x and y <= w0 + m_:
                out.window[g] = win
                out.have[g] = shard if trim else have | shard
                missing = [s for s in range(x, y) if s not in have]
            else:
                out.window[g] = window_for(x, y, m_)
                out.relayout[g] = True
                out.have[g] = shard
                out.local[g] = [s for s in range(x, y) if s in have]
                missing = [s for s in range(x, y) if s not in have]
            runs = []
            for sl in missing:
                holders = [h for h in self.gpu_ids if h != g and sl in self.have[h]]
                if not holders:
                    raise MigrationError(f"weight slice {sl} is resident nowhere")
                src = min(holders, key=lambda h: (egress[h], self.gpu_ids.index(h)))
                egress[src] += self.bytes_per_slice
                if runs and runs[-1][0] == src and runs[-1][2] == sl:
                    runs[-1][2] = sl + 1
                else:
                    runs.append([src, sl, sl + 1])
            out.fetch[g] = [tuple(r) for r in runs]
        return out

    def _segments(self, g: int, plan: ReshardPlan, dst_arena, src_arena=None) -> np.ndarray:
        """Copy segments into g's arena (uint64/int64 x 8 per row,
        tpr_copy_seg_t layout): the fetched runs, plus the local relayout
        copies from g's old arena."""
        dw0, dm = plan.window[g]
        dbase = dst_arena.data_ptr()
        step = self._step
        runs = list(plan.fetch[g])
        runs += [(g, s, s + 1) for s in plan.local[g]]
        seg = np.zeros((len(runs), len(self.split), 8), dtype=np.int64)
        for i, (src, lo, hi) in enumerate(runs):
            sw0, sm = self.window[src]
            sbase = (src_arena if (src == g and src_arena is not None) else self.arena[src]).data_ptr()
            row_bytes = (hi - lo) * step
            seg[i, :, 0] = sbase + sm * self.slice_off + (lo - sw0) * step
            seg[i, :, 1] = dbase + dm * self.slice_off + (lo - dw0) * step
            seg[i, :, 2] = self._seg_rows
            seg[i, :, 3] = row_bytes
            seg[i, :, 4] = np.where(self.is_col, row_bytes, sm * step)
            seg[i, :, 5] = np.where(self.is_col, row_bytes, dm * step)
        return seg.reshape(-1, 8)

    def _stats(self, plan: ReshardPlan) -> ReshardStats:
        stats = ReshardStats(egress={g: 0 for g in self.gpu_ids},
                             ingress={g: 0 for g in self.gpu_ids})
        for g in self.gpu_ids:
            if not plan.fetch[g] and not plan.relayout[g]:
                stats.views += 1
                continue
            if not plan.relayout[g]:
                stats.in_place += 1
            stats.local_bytes += len(plan.local[g]) * self.bytes_per_slice
            for src, lo, hi in plan.fetch[g]:
                nb = (hi - lo) * self.bytes_per_slice
                stats.remote_bytes += nb
                stats.egress[src] += nb
                stats.ingress[g] += nb
        return stats

    def reshard(self, new_groups: Sequence[Sequence[int]], stream: torch.cuda.Stream | None = None,
                events: tuple | None = None, parked: Sequence[int] = (),
                trim: bool = False) -> ReshardStats:
        """Move to ``new_groups``: K2 fetches every GPU's missing slices into
        their window positions (in place), views for the rest. Stream-ordered,
        no host sync: a relayout arena is allocated and the old one released on
        ``stream`` (the caching allocator reuses a block on the same stream only
        after the K2 that last touched it), so the host may run ahead."""
        plan = self.plan(new_groups, parked, trim)
        stats = self._stats(plan)
        devs = {self.device_of[g] for g in self.gpu_ids}
        if len(devs) != 1:
            raise MigrationError("multi-device weight reshard goes through the distributed executor")
        dev = next(iter(devs))
        stream = stream or torch.cuda.current_stream(dev)
        new_arena, segs = {}, []
        for g in self.gpu_ids:
            if not plan.fetch[g] and not plan.relayout[g]:
                continue
            dst = self.arena[g]
            if plan.relayout[g]:
                with torch.cuda.stream(stream):
                    dst = new_arena[g] = torch.empty(plan.window[g][1] * self.bytes_per_slice,
                                                     dtype=torch.uint8, device=dev)
            segs.append(self._segments(g, plan, dst))
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
        self.have, self.window, self.active = plan.have, plan.window, plan.active
        self._stream = stream
        return stats

    def _launch(self, seg: np.ndarray, dev: torch.device, stream: torch.cuda.Stream) -> None:
        """Normalise segments (host), upload segments + item prefix through
        pinned staging, launch K2."""
        from .kvcache import _PinnedStaging, _Scratch

        n = len(seg)
        # segments | prefix[n + 1] | dynamic-claim counter, built in pinned
        # memory; libtpr normalises them, uploads and launches K2 in one call
        # (the copy engine follows the segment addresses: TMA on local HBM,
        # 16-byte loads/stores when a slice comes from another GPU)
        nbytes = int(_native.load().tpr_reshard_buffer_bytes(n))
        if dev not in self._segs_dev:
            self._segs_dev[dev] = (_PinnedStaging(), _Scratch(torch.int64, dev))
        staging, scratch = self._segs_dev[dev]
        h_ptr, raw = staging.acquire(nbytes)
        raw.view(np.int64)[: seg.size] = seg.reshape(-1)
        d = scratch.get(nbytes // 8, stream)
        with torch.cuda.device(dev):
            _native.call("tpr_weight_reshard_host", h_ptr, n, CHUNK_BYTES, d.data_ptr(),
                         d.numel() * 8, None, stream.cuda_stream)
        staging.fence(stream)

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
