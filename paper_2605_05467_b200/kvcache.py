"""Paged KV block manager + migration engine on B200.

The reference has no KV memory at all: a TP switch is priced, not executed
(pkg/src/tpsim/engine.py:567-597 builds per-request ``KvLayout``s, calls
``head_transfers`` and charges ``switch_cost``). This module is the executed
counterpart. Its placement semantics are the reference's: after ``migrate``
every (request, KV head) sits on ``layout_placement(new)`` (migration.py:210-218),
and it moves exactly ``plan.total_bytes`` bytes (migration.py:128-130).

Memory model (per GPU slot):

* pool         uint8  [units, unit_bytes]; a unit is one KV head x one page
                      of ``block_tokens`` tokens x all layers x {K, V}. The pool
                      shape does not depend on the TP degree.
* block table  int32  [max_requests, H, max_blocks]; entry = unit id or -1.
                      Indexed by the GLOBAL head id, so a TP-N rank r reads rows
                      [r*H/N, (r+1)*H/N) -- shard selection at execution time.
* free ring    int32  [units] + host-owned monotonic (head, tail) counters.
                      Allocation pops at head, release pushes at tail.

A migration is two device steps behind ONE native call (``tpr_kv_switch``):
K3 allocates destination units and rewrites both block tables in the plan's
sequential order, then K1 copies the valid tokens. The host side is kept to
table lookups so that small switches are not host-bound. All GPU slots may
live on one device ("logical ranks", one B200) or on their own devices.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native
from .geometry import KvGeometry
from .migration import (BYTES, DST, HI, LO, REQ, SRC, KvLayout, MigrationError, MigrationPlan,
                        head_transfers_array, pack_layouts, plan_repartition)

_LUT_MAX = 1 << 24  # ids below this use dense lookup tables, others a dict


@dataclass
class MigrationStats:
    transfers: int
    units: int
    bytes: int            # plan.total_bytes: valid KV bytes moved
    in_units: dict        # gpu id -> units allocated there
    out_units: dict       # gpu id -> units released there


class _PinnedStaging:
    """Double-buffered pinned host staging for H2D metadata.

    ``stage`` copies an int32 array into the next pinned buffer (waiting for
    the copy that used it two calls ago) and returns its address; the caller
    launches the H2D copy and then calls ``fence(stream)``."""

    def __init__(self, nbytes: int = 1 << 16):
        self._bufs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self._views = [b.numpy() for b in self._bufs]
        self._events = [torch.cuda.Event(), torch.cuda.Event()]
        self._armed = [False, False]
        self._i = 0

    def stage(self, arr: np.ndarray) -> int:
        raw = np.ascontiguousarray(arr).reshape(-1).view(np.uint8)
        i = self._i
        if self._armed[i]:
            self._events[i].synchronize()
            self._armed[i] = False
        if self._bufs[i].numel() < raw.nbytes:
            self._bufs[i] = torch.empty(max(raw.nbytes, 2 * self._bufs[i].numel()),
                                        dtype=torch.uint8, pin_memory=True)
            self._views[i] = self._bufs[i].numpy()
        self._views[i][: raw.nbytes] = raw
        return self._bufs[i].data_ptr()

    def acquire(self, nbytes: int) -> tuple[int, np.ndarray]:
        """The next pinned buffer (address, uint8 view of ``nbytes``) to be
        written in place; ``fence`` after the H2D copy that reads it."""
        i = self._i
        if self._armed[i]:
            self._events[i].synchronize()
            self._armed[i] = False
        if self._bufs[i].numel() < nbytes:
            self._bufs[i] = torch.empty(max(nbytes, 2 * self._bufs[i].numel()),
                                        dtype=torch.uint8, pin_memory=True)
            self._views[i] = self._bufs[i].numpy()
        return self._bufs[i].data_ptr(), self._views[i][:nbytes]

    def fence(self, stream: torch.cuda.Stream) -> None:
        self._events[self._i].record(stream)
        self._armed[self._i] = True
        self._i ^= 1

    def upload(self, arr: np.ndarray, dst: torch.Tensor, stream: torch.cuda.Stream) -> int:
        """Stage ``arr`` and copy it into ``dst`` on ``stream``."""
        ptr = self.stage(arr)
        n = arr.nbytes
        _native.call("tpr_memcpy_h2d", dst.data_ptr(), ptr, n, stream.cuda_stream)
        self.fence(stream)
        return n


class _Scratch:
    """Grow-only device buffer used on one stream (zeroed when it grows: the
    work-list scratch holds K31's epoch-tagged reader counters)."""

    def __init__(self, dtype, device):
        self.t = torch.zeros(0, dtype=dtype, device=device)
        self.n = 0
        self.version = 0  # bumped on every reallocation

    def get(self, n: int, stream: torch.cuda.Stream) -> torch.Tensor:
        if self.n < n:
            with torch.cuda.stream(stream):
                self.t = torch.zeros(max(n, 2 * self.n, 1024), dtype=self.t.dtype,
                                     device=self.t.device)
            self.n = self.t.numel()
            self.version += 1
        return self.t


class PagedKvCluster:
    """KV pools, block tables and free rings of a set of GPUs."""

    def __init__(self, kv: KvGeometry, gpu_ids: Sequence[int], units_per_gpu,
                 max_requests: int, max_blocks: int, device: str | torch.device = "cuda",
                 devices: dict | None = None, fragmented: bool = False, seed: int = 0):
        if not 1 <= len(gpu_ids) <= _native.TPR_MAX_GPUS:
            raise MigrationError(f"1..{_native.TPR_MAX_GPUS} GPUs per cluster")
        if len(set(gpu_ids)) != len(gpu_ids):
            raise MigrationError("duplicate gpu ids")
        _native.load()
        self.kv = kv
        self.gpu_ids = tuple(gpu_ids)
        self.slot_of = {g: i for i, g in enumerate(self.gpu_ids)}
        # pool capacity per GPU: one int for all, or {gpu id: units}
        if isinstance(units_per_gpu, dict):
            self.units = [int(units_per_gpu[g]) for g in self.gpu_ids]
        else:
            self.units = [int(units_per_gpu)] * len(self.gpu_ids)
        self.n_units = max(self.units)
        self.max_requests = int(max_requests)
        self.max_blocks = int(max_blocks)
        default = torch.device(device)
        if default.type == "cuda" and default.index is None:
            default = torch.device("cuda", torch.cuda.current_device())
        self.devices = [torch.device(devices[g]) if devices else default for g in self.gpu_ids]
        self.home = self.devices[0]
        self._single_device = len(set(self.devices)) == 1
        H = kv.total_heads
        self.pools, self.block_tables, self.rings = [], [], []
        gen = np.random.default_rng(seed)
        for dev, units in zip(self.devices, self.units):
            self.pools.append(torch.empty(units * kv.unit_bytes, dtype=torch.uint8, device=dev))
            self.block_tables.append(torch.full((self.max_requests, H, self.max_blocks), -1,
                                                dtype=torch.int32, device=dev))
            order = gen.permutation(units) if fragmented else np.arange(units)
            self.rings.append(torch.from_numpy(order.astype(np.int32)).to(dev))
        # request bookkeeping (host is authoritative; device copies for checks)
        self.req_slot: dict[int, int] = {}
        self.ctx_of: dict[int, int] = {}
        self._free_req_slots = list(range(self.max_requests - 1, -1, -1))
        self.owner = np.full((self.max_requests, H), -1, dtype=np.int32)  # gpu slot per head
        self.slot_ctx = np.full(self.max_requests, -1, dtype=np.int32)
        # id -> slot lookup tables
        ids = np.asarray(self.gpu_ids, dtype=np.int64)
        self._gpu_lut = None
        if ids.min() >= 0 and ids.max() < _LUT_MAX:
            self._gpu_lut = np.full(int(ids.max()) + 1, -1, dtype=np.int64)
            self._gpu_lut[ids] = np.arange(len(ids))
        self._req_lut = np.full(1024, -1, dtype=np.int64)
        # device scratch + the cached C view of the cluster
        self._staging = _PinnedStaging()
        self._xf = _Scratch(torch.int32, self.home)
        self._meta = _Scratch(torch.int64, self.home)
        self._work = _Scratch(torch.int32, self.home)
        self._work_ext = _Scratch(torch.int32, self.home)
        self._totals = torch.zeros(_native.TPR_TOTALS_LEN, dtype=torch.int64, device=self.home)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.home)
        # pinned host mirror of the status word, kept current by the one-call
        # switch on its stream (no separate read-back for a synchronous caller)
        # [status word, completion ticket] (tpr_switch_tables_t.h_status / .ticket)
        self.status_host = torch.zeros(2, dtype=torch.int32, pin_memory=True)
        self.status_mirrored = False  # the last switch_layouts refreshed status_host
        self._swt = self._swt_lut = None  # the cached tpr_switch_tables_t (_switch_tables)
        self.last_ticket = 0  # nonzero: the last switch_layouts' kernel writes it to status_host[1]
        self._geo = _native.KvGeometryC(kv.layers, kv.head_dim, kv.dtype_bytes, kv.block_tokens,
                                        H, self.max_blocks, self.max_requests, self.n_units)
        # the C view of the cluster; its ring counters (monotonic head/tail per
        # slot) are the host's authoritative copy, advanced in place by the
        # one-call switch
        self._cl = _native.KvClusterC()
        self._cl.n_gpus = self.n_gpus
        for s in range(self.n_gpus):
            self._cl.pool[s] = self.pools[s].data_ptr()
            self._cl.block_table[s] = self.block_tables[s].data_ptr()
            self._cl.free_ring[s] = self.rings[s].data_ptr()
            self._cl.units[s] = self.units[s]
            self._cl.ring_head[s] = 0
            self._cl.ring_tail[s] = self.units[s]
        self._last_in = self._last_out = np.zeros(self.n_gpus, np.int64)
        self._gpu_ids_arr = np.asarray(self.gpu_ids, dtype=np.int64)
        self._n_units_c = ctypes.c_int64(0)
        self.pattern_seed = 0
        self._default_stream = torch.cuda.current_stream(self.home)

    # ------------------------------------------------------------------ utils
    @property
    def n_gpus(self) -> int:
        return len(self.gpu_ids)

    @property
    def ring_head(self) -> list:
        """Units ever allocated per slot (monotonic free-ring head), a copy."""
        return self._cl.ring_head[: self.n_gpus]

    @property
    def ring_tail(self) -> list:
        """Units ever released per slot + capacity (monotonic free-ring tail), a copy."""
        return self._cl.ring_tail[: self.n_gpus]

    def free_units(self, gpu: int) -> int:
        s = self.slot_of[gpu]
        return self._cl.ring_tail[s] - self._cl.ring_head[s]

    def _cluster_c(self) -> _native.KvClusterC:
        return self._cl

    def _units_per_record(self, xf: np.ndarray) -> np.ndarray:
        B = self.kv.block_tokens
        nblk = (xf[:, 5].astype(np.int64) + B - 1) // B
        return (xf[:, 4] - xf[:, 3]).astype(np.int64) * nblk

    def _gpu_slots(self, ids: np.ndarray) -> np.ndarray:
        lut = self._gpu_lut
        if lut is not None and len(ids) and ids.min() >= 0 and ids.max() < len(lut):
            s = lut[ids]
            if (s >= 0).all():
                return s
        try:
            return np.fromiter((self.slot_of[g] for g in ids.tolist()), np.int64, len(ids))
        except KeyError as exc:
            raise MigrationError(f"gpu {exc.args[0]} is not part of this cluster") from None

    def _req_slots(self, ids: np.ndarray) -> np.ndarray:
        lut = self._req_lut
        if len(ids) and ids.min() >= 0 and ids.max() < len(lut):
            s = lut[ids]
            if (s >= 0).all():
                return s
        try:
            return np.fromiter((self.req_slot[r] for r in ids.tolist()), np.int64, len(ids))
        except KeyError as exc:
            raise MigrationError(f"request {exc.args[0]} is not resident") from None

    def _set_req(self, rid: int, slot: int) -> None:
        if 0 <= rid < _LUT_MAX:
            if rid >= len(self._req_lut):
                grown = np.full(max(rid + 1, 2 * len(self._req_lut)), -1, dtype=np.int64)
                grown[: len(self._req_lut)] = self._req_lut
                self._req_lut = grown
                self._rec_tables = None
            self._req_lut[rid] = slot

    def _deltas(self, xf: np.ndarray, units: np.ndarray):
        if len(xf) <= 64:  # small plans: plain loops beat numpy call overhead
            in_u = [0] * self.n_gpus
            out_u = [0] * self.n_gpus
            for (s, d), u in zip(xf[:, :2].tolist(), units.tolist()):
                if d >= 0:
                    in_u[d] += u
                if s >= 0:
                    out_u[s] += u
            return np.asarray(in_u, np.int64), np.asarray(out_u, np.int64)
        has_dst = xf[:, 1] >= 0
        has_src = xf[:, 0] >= 0
        in_u = np.bincount(xf[has_dst, 1], weights=units[has_dst], minlength=self.n_gpus)
        out_u = np.bincount(xf[has_src, 0], weights=units[has_src], minlength=self.n_gpus)
        return in_u.astype(np.int64), out_u.astype(np.int64)

    def _reserve(self, xf: np.ndarray):
        """Capacity check + ring bookkeeping for records; returns (#units, in, out)."""
        if len(xf) <= 64:
            B = self.kv.block_tokens
            in_u = [0] * self.n_gpus
            out_u = [0] * self.n_gpus
            total = 0
            for s, d, _, lo, hi, ctx in xf.tolist():
                u = (hi - lo) * (-(-ctx // B))
                total += u
                if d >= 0:
                    in_u[d] += u
                if s >= 0:
                    out_u[s] += u
        else:
            units = self._units_per_record(xf)
            total = int(units.sum())
            in_u, out_u = self._deltas(xf, units)
        self._check_capacity(in_u)
        self._last_in, self._last_out = in_u, out_u
        return total, in_u, out_u

    def _check_capacity(self, in_u) -> None:
        head, tail = self._cl.ring_head, self._cl.ring_tail
        for s in range(self.n_gpus):
            free = tail[s] - head[s]
            if in_u[s] > free:
                raise MigrationError(
                    f"gpu {self.gpu_ids[s]}: {in_u[s]} KV units needed, {free} free")

    def _commit(self, in_u, out_u):
        head, tail = self._cl.ring_head, self._cl.ring_tail
        for s in range(self.n_gpus):
            head[s] += int(in_u[s])
            tail[s] += int(out_u[s])

    # -------------------------------------------------------------- K3 driver
    def _remap(self, xf: np.ndarray, stream: torch.cuda.Stream, want_ext: bool) -> int:
        """Upload records, run K3 only (admission / release); returns #units."""
        total, in_u, out_u = self._reserve(xf)
        if total == 0:  # e.g. zero-length contexts: nothing to allocate or move
            return 0
        n = len(xf)
        d_xf = self._xf.get(n * 6, stream)
        self._staging.upload(xf.astype(np.int32), d_xf, stream)
        d_work = self._work.get((total + 1) * 4, stream)  # + K1 claim slot
        d_ext = self._work_ext.get(total * 4, stream) if want_ext else None
        cl = self._cluster_c()
        _native.call(
            "tpr_kv_remap", ctypes.byref(self._geo), ctypes.byref(cl), d_xf.data_ptr(), n, -1,
            self._meta.get(n * 4, stream).data_ptr(), self._totals.data_ptr(), total,
            d_work.data_ptr(), d_ext.data_ptr() if want_ext else None, self.status.data_ptr(),
            stream.cuda_stream,
        )
        self._commit(in_u, out_u)
        return total

    # -------------------------------------------------------------- admission
    def admit(self, layouts: Iterable[KvLayout], seed: int = 1,
              stream: torch.cuda.Stream | None = None) -> int:
        """Allocate pages for new requests in their canonical layout and fill
        them with the placement-invariant synthetic pattern. Returns #units."""
        stream = stream or self._default_stream
        H = self.kv.total_heads
        recs, new = [], []  # new: (rid, slot, ctx, [(gpu slot, lo, hi)])
        free = list(self._free_req_slots)
        seen = set()
        for lay in layouts:
            if lay.total_heads != H:
                raise MigrationError("all layouts must share total_heads")
            hpr = lay.heads_per_rank
            slots = [self.slot_of[g] for g in lay.group]
            for rid, ctx in lay.requests:
                if rid in self.req_slot or rid in seen:
                    raise MigrationError(f"request {rid} already resident")
                if self.kv.blocks(ctx) > self.max_blocks:
                    raise MigrationError(f"request {rid}: {ctx} tokens exceed max_blocks")
                if not free:
                    raise MigrationError("no free request slots")
                seen.add(rid)
                rs = free.pop()
                runs = [(s, r * hpr, (r + 1) * hpr) for r, s in enumerate(slots)]
                new.append((rid, rs, int(ctx), runs))
                recs.extend((-1, s, rs, lo, hi, int(ctx)) for s, lo, hi in runs)
        if not recs:
            return 0
        xf = np.asarray(recs, dtype=np.int64)
        total = self._remap(xf, stream, want_ext=True)  # raises before any state change
        # commit host bookkeeping only once the device work is enqueued
        self._free_req_slots = free
        for rid, rs, ctx, runs in new:
            self.req_slot[rid] = rs
            self._set_req(rid, rs)
            self.ctx_of[rid] = ctx
            self.slot_ctx[rs] = ctx
            for s, lo, hi in runs:
                self.owner[rs, lo:hi] = s
        if total:
            cl = self._cluster_c()
            with torch.cuda.device(self.home):
                _native.call("tpr_kv_fill", ctypes.byref(self._geo), ctypes.byref(cl),
                             self._work.t.data_ptr(), self._work_ext.t.data_ptr(), total, seed,
                             stream.cuda_stream)
        self.pattern_seed = seed
        return total

    def release(self, request_ids: Iterable[int], stream: torch.cuda.Stream | None = None) -> int:
        """Free every page of finished / evicted requests (K3 with dst = -1:
        block-table entries cleared, units pushed back on their owners' free
        rings in (request, head, page) order). Returns #units released."""
        stream = stream or self._default_stream
        request_ids = list(request_ids)
        recs = []
        for rid in request_ids:
            rs = self.req_slot.get(rid)
            if rs is None:
                raise MigrationError(f"request {rid} is not resident")
            own = self.owner[rs]
            h = 0
            while h < len(own):  # one record per run of heads on the same GPU
                e = h
                while e < len(own) and own[e] == own[h]:
                    e += 1
                recs.append((int(own[h]), -1, rs, h, e, int(self.slot_ctx[rs])))
                h = e
        if not recs:
            return 0
        total = self._remap(np.asarray(recs, np.int64), stream, want_ext=False)
        self._forget(request_ids)
        return total

    def fill_garbage(self, seed: int = 99, stream: torch.cuda.Stream | None = None) -> None:
        """Fill whole pools with per-unit garbage (so stale bytes are visible)."""
        stream = stream or self._default_stream
        for s in range(self.n_gpus):
            geo = _native.KvGeometryC(*[getattr(self._geo, f) for f, _ in self._geo._fields_])
            geo.n_units = self.units[s]
            _native.call("tpr_pool_fill", ctypes.byref(geo), self.pools[s].data_ptr(), s,
                         seed, stream.cuda_stream)

    # -------------------------------------------------------------- migration
    def _native_records(self, arr: np.ndarray, validate: bool, out: np.ndarray):
        """``tpr_kv_records``: plan rows -> int32 records in ``out`` + unit
        deltas, with the reference checks. None when an id is outside the
        lookup tables (the Python path resolves it or raises its error)."""
        if self._gpu_lut is None:
            return None
        tables = self.__dict__.get("_rec_tables")
        if tables is None:  # the cluster's table pointers (rebuilt when _req_lut grows)
            tables = self._rec_tables = (
                self._gpu_lut.ctypes.data, len(self._gpu_lut), self._gpu_ids_arr.ctypes.data,
                self.n_gpus, self._req_lut.ctypes.data, len(self._req_lut),
                self.slot_ctx.ctypes.data, self.owner.ctypes.data, self.max_requests,
                self.kv.total_heads, self.kv.block_tokens, self.kv.kv_bytes_per_token_per_head)
        deltas = np.empty((2, self.n_gpus), np.int64)
        dp = deltas.ctypes.data
        lib = _native.load()
        rc = lib.tpr_kv_records(arr.ctypes.data, len(arr), *tables, int(validate),
                                out.ctypes.data, dp, dp + 8 * self.n_gpus,
                                ctypes.byref(self._n_units_c))
        if rc == _native.TPR_ENOTFOUND:
            return None
        if rc != 0:
            raise MigrationError(lib.tpr_last_error().decode(errors="replace"))
        return self._n_units_c.value, deltas[0], deltas[1]

    def records(self, plan: MigrationPlan, validate: bool = True) -> np.ndarray:
        """Plan -> int64 [n, 6] device records (slots), with reference checks."""
        arr = plan.as_array()
        n = len(arr)
        if n == 0:
            return np.zeros((0, 6), dtype=np.int64)
        rec = np.empty((n, 6), dtype=np.int32)
        if self._native_records(arr, validate, rec) is not None:
            return rec.astype(np.int64)
        return self._records_py(arr, validate)

    def _records_py(self, arr: np.ndarray, validate: bool) -> np.ndarray:
        """records() for ids outside the lookup tables (dict maps)."""
        n = len(arr)
        if n <= 32 and not validate:  # small plans: dict lookups beat numpy call overhead
            H = self.kv.total_heads
            out = []
            for s, d, r, lo, hi, _ in arr.tolist():
                ss, ds, rs = self.slot_of.get(s), self.slot_of.get(d), self.req_slot.get(r)
                if ss is None or ds is None:
                    raise MigrationError(f"gpu {s if ss is None else d} is not part of this cluster")
                if rs is None:
                    raise MigrationError(f"request {r} is not resident")
                if not 0 <= lo < hi <= H:
                    raise MigrationError("head range outside [0, total_heads)")
                out.append((ss, ds, rs, lo, hi, self.ctx_of[r]))
            return np.array(out, dtype=np.int64)
        src = self._gpu_slots(arr[:, SRC])
        dst = self._gpu_slots(arr[:, DST])
        req = self._req_slots(arr[:, REQ])
        ctx = self.slot_ctx[req].astype(np.int64)
        lo, hi = arr[:, LO], arr[:, HI]
        if ((lo < 0) | (hi > self.kv.total_heads) | (lo >= hi)).any():
            raise MigrationError("head range outside [0, total_heads)")
        if validate:
            if (arr[:, BYTES] != (hi - lo) * ctx * self.kv.kv_bytes_per_token_per_head).any():
                raise MigrationError(
                    "transfer bytes disagree with (head_hi-head_lo)*context_len*kv_bytes_per_token_per_head")
            heads = np.arange(self.kv.total_heads)
            mask = (heads >= lo[:, None]) & (heads < hi[:, None])
            # each (request, head) may move once per plan
            cover = np.zeros_like(self.owner, dtype=np.int32)
            np.add.at(cover, (np.repeat(req, self.kv.total_heads)[mask.ravel()],
                              np.tile(heads, n)[mask.ravel()]), 1)
            if (cover > 1).any():
                raise MigrationError("a (request, head) is moved twice in one plan")
            wrong = mask & (self.owner[req] != src[:, None])
            if wrong.any():
                t, h = map(int, np.argwhere(wrong)[0])
                rid = int(arr[t, REQ])
                here = self.owner[req[t], h]
                raise MigrationError(
                    f"transfer of request {rid} head {h} from gpu {int(arr[t, SRC])}, "
                    f"but it is on {self.gpu_ids[here] if here >= 0 else None}")
        return np.stack([src, dst, req, lo, hi, ctx], axis=1)

    def migrate(self, plan: MigrationPlan, stream: torch.cuda.Stream | None = None,
                validate: bool = True, k1_events: tuple | None = None) -> MigrationStats:
        """Execute ``plan``: K3 remap + K1 page copy, stream-ordered, no host sync.

        ``k1_events`` = (start, end) CUDA events recorded around K1 (this
        splits the fused call in two so the events can sit between them).
        """
        stream = stream or self._default_stream
        self.status_mirrored = False  # this path leaves status_host stale
        arr = plan.as_array()
        n = len(arr)
        if n == 0:
            return MigrationStats(0, 0, 0, {}, {})
        if not self._single_device:
            raise MigrationError("multi-device clusters migrate through distributed.py")
        # records go straight into the pinned staging buffer the H2D reads
        h_ptr, raw = self._staging.acquire(n * 6 * 4)
        xf32 = raw.view(np.int32).reshape(n, 6)
        fast = self._native_records(arr, validate, xf32)
        if fast is None:
            xf = self._records_py(arr, validate)
            total, in_u, out_u = self._reserve(xf)
            xf32[:] = xf
        else:
            total, in_u, out_u = fast
            self._check_capacity(in_u)
        cl = self._cluster_c()
        d_xf = self._xf.get(n * 6, stream)
        d_meta = self._meta.get(n * 4, stream)
        d_work = self._work.get((total + 1) * 4, stream)  # + K1 claim slot
        if k1_events:
            _native.call("tpr_kv_switch", ctypes.byref(self._geo), ctypes.byref(cl), h_ptr,
                         d_xf.data_ptr(), n, -1, d_meta.data_ptr(), self._totals.data_ptr(), 0,
                         d_work.data_ptr(), self.status.data_ptr(), stream.cuda_stream)
            if total:
                _native.call("tpr_kv_remap", ctypes.byref(self._geo), ctypes.byref(cl),
                             d_xf.data_ptr(), n, -1, d_meta.data_ptr(), self._totals.data_ptr(),
                             total, d_work.data_ptr(), None, self.status.data_ptr(),
                             stream.cuda_stream)
            k1_events[0].record(stream)
            full = not (xf32[:, 5] % self.kv.block_tokens).any()
            _native.call("tpr_kv_migrate_ex", ctypes.byref(self._geo), ctypes.byref(cl),
                         d_work.data_ptr(), total,
                         _native.TPR_MIGRATE_FULL_PAGES if full else 0, stream.cuda_stream)
            k1_events[1].record(stream)
        else:
            _native.call("tpr_kv_switch", ctypes.byref(self._geo), ctypes.byref(cl), h_ptr,
                         d_xf.data_ptr(), n, -1, d_meta.data_ptr(), self._totals.data_ptr(), total,
                         d_work.data_ptr(), self.status.data_ptr(), stream.cuda_stream)
        self._staging.fence(stream)
        self._commit(in_u, out_u)
        # host placement bookkeeping (apply_plan semantics)
        _native.call("tpr_kv_apply_owner", xf32.ctypes.data, n, self.owner.ctypes.data,
                     self.kv.total_heads)
        return MigrationStats(
            transfers=n, units=total, bytes=plan.total_bytes,
            in_units={self.gpu_ids[s]: int(v) for s, v in enumerate(in_u) if v},
            out_units={self.gpu_ids[s]: int(v) for s, v in enumerate(out_u) if v},
        )

    def _switch_tables(self, validate: bool) -> _native.SwitchTablesC:
        """The cached tpr_switch_tables_t of this cluster (lookup tables, host
        outputs, device scratch); pointers refreshed when a table grows."""
        t = self._swt
        if t is None or self._swt_lut is not self._req_lut:
            t = self._swt = _native.SwitchTablesC()
            self._swt_lut = self._req_lut
            t.gpu_lut = self._gpu_lut.ctypes.data
            t.gpu_lut_len = len(self._gpu_lut)
            t.gpu_ids = self._gpu_ids_arr.ctypes.data
            t.req_lut = self._req_lut.ctypes.data
            t.req_lut_len = len(self._req_lut)
            t.slot_ctx = self.slot_ctx.ctypes.data
            t.owner = self.owner.ctypes.data
            t.kvb = self.kv.kv_bytes_per_token_per_head
            t.d_totals = self._totals.data_ptr()
            t.d_status = self.status.data_ptr()
            t.h_status = self.status_host.data_ptr()
            base = ctypes.addressof(self._cl)
            t.ring_head_io = base + _native.KvClusterC.ring_head.offset
            t.ring_tail_io = base + _native.KvClusterC.ring_tail.offset
            self._swt_plan = np.empty((0, 6), np.int64)
            self._swt_bufs = None
            self._swt_records = None
        t.validate = int(validate)
        return t

    def _switch_buffers(self, t, stream) -> None:
        """Point the tables at plan/records/device scratch sized for the
        current plan capacity (grow-only; set again only when one grew)."""
        rows = self._swt_plan
        held = self._swt_bufs
        xf, meta, work = self._xf, self._meta, self._work
        if (held is not None and held[0] is rows and held[1] == xf.version
                and held[2] == meta.version and held[3] == work.version):
            return
        cap = max(len(rows), 1)
        xf.get(cap * 6, stream)
        meta.get(cap * 4, stream)
        t.plan, t.plan_cap = rows.ctypes.data, len(rows)
        t.d_xfers, t.d_meta, t.xfers_cap = xf.t.data_ptr(), meta.t.data_ptr(), len(rows)
        t.d_work, t.work_cap = work.t.data_ptr(), work.n // 4
        self._swt_bufs = (rows, xf.version, meta.version, work.version)

    def switch_layouts(self, old_layouts, new_layouts, stream: torch.cuda.Stream | None = None,
                       validate: bool = True, handshake_ms: float = 0.0,
                       planner: str = "repartition", k1_events: tuple | None = None,
                       release=(), start_event: int | None = None, want_ticket: bool = False):
        """``plan_repartition(old, new)`` + ``migrate(plan)`` in one native call
        (``tpr_kv_switch_layouts``): plan, records, capacity check, K3 + K1 and
        the placement update. Returns (MigrationPlan, MigrationStats) equal to
        the two-step path's. Anything the reference reports as an error, a
        repeated old request id or an id outside the lookup tables goes through
        the two-step path, which raises the reference's error.

        ``planner="head_transfers"``: one old and one new layout planned with
        ``head_transfers`` (any GPU sets: the prefill->decode handoff).
        ``k1_events``: (start, end) CUDA events recorded around K1.
        ``release``: resident request ids (in neither layout list) whose pages
        the same native call frees -- the destination's KV-capacity evictions
        (engine.py:630-645); their records follow the plan's.
        ``start_event``: a CUDA event handle recorded on ``stream`` right
        before the switch's first launch (on every path).
        ``want_ticket``: ask the one-launch kernel for a completion ticket
        (``last_ticket``, written to ``status_host[1]`` when the switch is
        done) for a caller that spins on it; it delays the kernel's exit by
        the ticket's host write, so asynchronous callers leave it off."""
        stream = stream or self._default_stream
        self.status_mirrored = False
        self.last_ticket = 0
        if planner not in ("repartition", "head_transfers"):
            raise MigrationError(f"unknown planner {planner!r}")
        heads = planner == "head_transfers"
        if heads:
            old_layouts, new_layouts = [old_layouts], [new_layouts]
        release = [int(r) for r in release]
        if release:
            carried = {r for lay in (*old_layouts, *new_layouts) for r, _ in lay.requests}
            for rid in release:
                if rid not in self.req_slot:
                    raise MigrationError(f"request {rid} is not resident")
                if rid in carried:
                    raise MigrationError(f"request {rid} is both released and carried")
        if self._gpu_lut is None or not self._single_device:
            if start_event:
                _native.call("tpr_event_record", start_event, stream.cuda_stream)
            return self._switch_general(old_layouts, new_layouts, stream, validate, handshake_ms,
                                        heads, release=release)
        blob = pack_layouts(old_layouts, new_layouts, release)
        t = self._switch_tables(validate)
        t.mode = _native.TPR_SWITCH_HEAD_TRANSFERS if heads else _native.TPR_SWITCH_REPARTITION
        if k1_events:
            for e in k1_events:  # torch creates the event on its first record; libtpr
                e.record(stream)  # then re-records it around K1 on the same stream
            t.k1_events[0], t.k1_events[1] = k1_events[0].cuda_event, k1_events[1].cuda_event
        elif t.k1_events[0]:
            t.k1_events[0] = t.k1_events[1] = None
        if start_event != t.start_event:
            t.start_event = start_event
        t.ticket = 1 if want_ticket else 0
        lib = _native.load()
        addr = blob.buffer_info()[0]
        for _ in range(3):  # grow-and-retry when a buffer is too small
            rows = self._swt_plan
            h_ptr, _raw = self._staging.acquire(max(len(rows), 1) * 24)
            if h_ptr != self._swt_records:
                t.records = self._swt_records = h_ptr
            self._switch_buffers(t, stream)
            rc = lib.tpr_kv_switch_layouts(ctypes.byref(self._geo), ctypes.byref(self._cl), addr,
                                           len(blob), ctypes.byref(t), stream.cuda_stream)
            if rc != _native.TPR_ECAPACITY:
                break
            t.ticket = 1 if want_ticket else 0
            if t.n_plan > len(rows):
                self._swt_plan = np.empty((max(t.n_plan, 2 * len(rows)), 6), np.int64)
            if t.total_units + 1 > t.work_cap:
                self._work.get((t.total_units + 1) * 4, stream)
        if rc == _native.TPR_ENOTFOUND:  # nothing was enqueued
            if start_event:
                _native.call("tpr_event_record", start_event, stream.cuda_stream)
            return self._switch_general(old_layouts, new_layouts, stream, validate, handshake_ms,
                                        heads, k1_events, release)
        if rc != 0:
            raise MigrationError(lib.tpr_last_error().decode(errors="replace"))
        n = t.n_plan
        self.status_mirrored = True
        self.last_ticket = t.ticket
        plan = MigrationPlan.from_rows(self._swt_plan[:n].copy(), handshake_ms)
        if release:
            self._forget(release)
        if t.n_records == 0:
            return plan, MigrationStats(0, 0, 0, {}, {})
        if t.records_async:  # the device still reads the pinned records
            self._staging.fence(stream)
        # the native call advanced the ring counters (t.ring_head_io / ring_tail_io)
        ng = self.n_gpus
        ids = self.gpu_ids
        in_d = {ids[s_]: a for s_, a in enumerate(t.in_units[:ng]) if a}
        out_d = {ids[s_]: b for s_, b in enumerate(t.out_units[:ng]) if b}
        return plan, MigrationStats(transfers=n, units=t.total_units, bytes=t.plan_bytes,
                                    in_units=in_d, out_units=out_d)

    def _switch_general(self, old_layouts, new_layouts, stream, validate, handshake_ms,
                        heads: bool = False, k1_events=None, release=()):
        kvb = self.kv.kv_bytes_per_token_per_head
        if heads:
            plan = head_transfers_array(old_layouts[0], new_layouts[0], kvb)
        else:
            plan = plan_repartition(old_layouts, new_layouts, kvb, handshake_ms=handshake_ms)
        stats = self.migrate(plan, stream=stream, validate=validate, k1_events=k1_events)
        if release:
            self.release(release, stream=stream)
        return plan, stats

    def _forget(self, request_ids) -> None:
        """Host bookkeeping of requests whose pages a switch released."""
        for rid in request_ids:
            rs = self.req_slot.pop(rid)
            if 0 <= rid < len(self._req_lut):
                self._req_lut[rid] = -1
            self.ctx_of.pop(rid, None)
            self.owner[rs] = -1
            self.slot_ctx[rs] = -1
            self._free_req_slots.append(rs)

    # ------------------------------------------------------------ inspection
    def placement(self) -> dict:
        """{(request, head): gpu} as recorded by the host (layout_placement form)."""
        out = {}
        for rid, rs in self.req_slot.items():
            for h in range(self.kv.total_heads):
                out[(rid, h)] = self.gpu_ids[self.owner[rs, h]]
        return out

    def verify(self, seed: int | None = None, stream: torch.cuda.Stream | None = None) -> dict:
        """Full-size device check: block tables realise the host placement and
        every owned page carries its pattern. Returns counts (host sync)."""
        seed = self.pattern_seed if seed is None else seed
        out = {"placement_errors": 0, "word_mismatches": 0, "pages_checked": 0}
        for s in range(self.n_gpus):
            dev = self.devices[s]
            st = stream or torch.cuda.current_stream(dev)
            ctx = torch.from_numpy(self.slot_ctx).to(dev)
            owner = torch.from_numpy(self.owner).to(dev)
            counts = torch.zeros(3, dtype=torch.int64, device=dev)
            geo = _native.KvGeometryC(*[getattr(self._geo, f) for f, _ in self._geo._fields_])
            geo.n_units = self.units[s]
            with torch.cuda.device(dev):
                _native.call("tpr_kv_verify", ctypes.byref(geo), self.pools[s].data_ptr(),
                             self.block_tables[s].data_ptr(), ctx.data_ptr(), owner.data_ptr(), s,
                             seed, counts.data_ptr(), st.cuda_stream)
            c = counts.cpu().tolist()
            out["placement_errors"] += c[0]
            out["word_mismatches"] += c[1]
            out["pages_checked"] += c[2]
        out["status"] = int(self.status.item())
        return out

    def tables_snapshot(self) -> dict:
        """Host copies of block tables, rings and ring counters (no pools): the
        K3 state at any size."""
        torch.cuda.synchronize()
        return {
            "block_tables": [b.cpu().numpy() for b in self.block_tables],
            "rings": [r.cpu().numpy() for r in self.rings],
            "ring_head": list(self.ring_head),
            "ring_tail": list(self.ring_tail),
        }

    def snapshot(self) -> dict:
        """Host copies of pools, block tables, rings and ring counters."""
        torch.cuda.synchronize()
        return {
            "pools": [p.cpu().numpy() for p in self.pools],
            "block_tables": [b.cpu().numpy() for b in self.block_tables],
            "rings": [r.cpu().numpy() for r in self.rings],
            "ring_head": list(self.ring_head),
            "ring_tail": list(self.ring_tail),
        }
