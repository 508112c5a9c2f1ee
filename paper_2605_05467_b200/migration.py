"""Drop-in replacement for ``tpsim.migration`` (reference pkg/src/tpsim/migration.py).

Same names, fields, argument meaning, return values and error messages as the
reference API, so the reference's scheduler / controller / CLI / tests can
import this module instead. Differences are underneath:

* head-range planning runs in the native planner of libtpr (``tpr_plan_heads``)
  and a plan keeps its transfers as an int64 SoA array, materialising
  ``Transfer`` objects only when ``plan.transfers`` is read; the execution path
  (``paper_2605_05467_b200.kvcache``) consumes the array directly;
* a plan can be executed on B200 pools (see ``kvcache.PagedKvCluster.migrate``).

The cost models are restated formula-for-formula (migration.py:221-292) so the
reference's exact-equality event-oracle test holds bit for bit.
"""

from __future__ import annotations

import math
import threading
from array import array as _array
from dataclasses import dataclass, field

import numpy as np

from . import _native

WARM = "warm"
NAIVE_RELOAD = "naive_reload"
NAIVE_KERNEL_INIT = "naive_kernel_init"

# columns of the transfer SoA array
SRC, DST, REQ, LO, HI, BYTES = range(6)


class MigrationError(ValueError):
    """Invalid layout / plan / parameter (reference: migration.py:21-22)."""


@dataclass(frozen=True)
class KvLayout:
    """KV placement of one TP group (reference: migration.py:25-47).

    Rank r of ``group`` owns KV heads [r*H/N, (r+1)*H/N) of every request in
    ``requests`` (tuples of (request id, context length in tokens)).
    """

    group: tuple[int, ...]
    tp: int
    total_heads: int
    requests: tuple[tuple[int, int], ...]

    def __post_init__(self):
        if self.tp != len(self.group):
            raise MigrationError("group size must equal tp")
        if self.total_heads % self.tp:
            raise MigrationError(
                f"total_heads={self.total_heads} not divisible by tp={self.tp}"
            )

    @property
    def heads_per_rank(self) -> int:
        return self.total_heads // self.tp

    def gpu_for_head(self, head: int) -> int:
        return self.group[head // self.heads_per_rank]

    def owners(self) -> tuple[int, ...]:
        """GPU id owning each head 0..H-1."""
        per = self.heads_per_rank
        return tuple(g for g in self.group for _ in range(per))

    def request_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """(request ids, context lengths) as int64 arrays, cached when immutable.

        The planner's vectorised path reads these instead of walking the
        tuples; a layout built with a list of requests is re-read every call.
        """
        cached = self.__dict__.get("_req_arrays")
        if cached is not None:
            return cached
        if self.requests:
            arr = np.asarray(self.requests, dtype=np.int64).reshape(-1, 2)
            out = (np.ascontiguousarray(arr[:, 0]), np.ascontiguousarray(arr[:, 1]))
        else:
            out = (np.zeros(0, np.int64), np.zeros(0, np.int64))
        if isinstance(self.requests, tuple):
            self.__dict__["_req_arrays"] = out  # frozen: bypass __setattr__
        return out

    def packed(self) -> tuple[int, ...]:
        """(total_heads, tp, *group, count, id0, ctx0, id1, ctx1, ...): this
        layout as ``tpr_switch_prepare`` reads it, cached when immutable."""
        cached = self.__dict__.get("_packed")
        if cached is not None:
            return cached
        flat = [self.total_heads, self.tp, *self.group, len(self.requests)]
        for rid, ctx in self.requests:
            flat.append(rid)
            flat.append(ctx)
        out = tuple(map(int, flat))
        if isinstance(self.requests, tuple):
            self.__dict__["_packed"] = out
        return out


@dataclass(frozen=True)
class Transfer:
    """One coalesced head-range move (reference: migration.py:50-57)."""

    src_gpu: int
    dst_gpu: int
    request_id: int
    head_lo: int
    head_hi: int  # exclusive
    bytes: int


@dataclass
class MigrationPlan:
    """Transfer list + handshake + predicted latencies (migration.py:60-74).

    A dataclass with the reference's fields, so ``dataclasses.fields`` /
    ``asdict`` / ``replace`` and equality behave the same. Plans built by the
    native planner hold an int64 [n, 6] array (src, dst, request, head_lo,
    head_hi, bytes) and build ``Transfer`` objects lazily (``transfers`` is a
    property over that storage), so the execution path never pays for Python
    objects.
    """

    transfers: list[Transfer]
    handshake_ms: float = 0.0
    predicted_latency_ms: dict = field(default_factory=dict)

    @classmethod
    def from_array(cls, arr: np.ndarray, handshake_ms: float = 0.0) -> "MigrationPlan":
        plan = cls.__new__(cls)
        plan._list = None
        plan._arr = np.ascontiguousarray(arr, dtype=np.int64).reshape(-1, 6)
        plan.handshake_ms = handshake_ms
        plan.predicted_latency_ms = {}
        return plan

    @classmethod
    def from_rows(cls, arr: np.ndarray, handshake_ms: float = 0.0) -> "MigrationPlan":
        """from_array for an array that is already C-contiguous int64 [n, 6]
        and owned by the plan (the one-call switch's copy of its plan rows)."""
        plan = cls.__new__(cls)
        plan._list = None
        plan._arr = arr
        plan.handshake_ms = handshake_ms
        plan.predicted_latency_ms = {}
        return plan

    def _get_transfers(self) -> list[Transfer]:
        if self._list is None:
            self._list = [Transfer(*map(int, row)) for row in self._arr]
        # the caller may mutate the list; the array view is rebuilt on demand
        self._arr = None
        return self._list

    def _set_transfers(self, value) -> None:
        self._list = list(value)
        self._arr = None

    def as_array(self) -> np.ndarray:
        """Transfers as int64 [n, 6] (src, dst, request, head_lo, head_hi, bytes)."""
        if self._arr is None:
            rows = [(t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes)
                    for t in self._list]
            self._arr = np.asarray(rows, dtype=np.int64).reshape(-1, 6)
        return self._arr

    @property
    def n_transfers(self) -> int:
        """len(plan.transfers) without building Transfer objects. (The reference
        dataclass defines no __len__, so neither does this one: an empty plan
        stays truthy, as there.)"""
        return len(self._list) if self._list is not None else len(self._arr)

    @property
    def total_bytes(self) -> int:
        if self._list is not None:
            return sum(t.bytes for t in self._list)
        return int(self._arr[:, BYTES].sum())

    def bytes_by_source(self) -> dict[int, int]:
        out: dict[int, int] = {}
        if self._list is not None:
            for t in self._list:
                out[t.src_gpu] = out.get(t.src_gpu, 0) + t.bytes
            return out
        arr = self._arr
        for src in dict.fromkeys(arr[:, SRC].tolist()):  # first-appearance order
            out[int(src)] = int(arr[arr[:, SRC] == src, BYTES].sum())
        return out

    def __repr__(self):
        return (f"MigrationPlan(transfers=<{self.n_transfers} transfers>, handshake_ms={self.handshake_ms}, "
                f"predicted_latency_ms={self.predicted_latency_ms})")


# the dataclass __init__ assigns `transfers` through this property
MigrationPlan.transfers = property(MigrationPlan._get_transfers, MigrationPlan._set_transfers)


@dataclass(frozen=True)
class CostModelParams:
    """Latency-model constants (reference: migration.py:77-98)."""

    copy_bw_gbps: float = 900.0
    link_bw_gbps: float = 200.0
    per_transfer_overhead_us: float = 100.0
    page_bytes: int = 65536
    chunk_bytes: int = 128 * 1024 * 1024
    handshake_ms: float = 0.5
    reload_ms: float = 30000.0
    kernel_init_ms: float = 10000.0

    def __post_init__(self):
        for name in ("copy_bw_gbps", "link_bw_gbps", "per_transfer_overhead_us",
                     "page_bytes", "chunk_bytes", "handshake_ms"):
            if not getattr(self, name) > 0:
                raise MigrationError(f"{name} must be positive")


# ---------------------------------------------------------------------------
# planning (native)
# ---------------------------------------------------------------------------

class _GroupTable:
    """Concatenated GPU-id groups for the native planner."""

    def __init__(self):
        self.ids: list[int] = []
        self._off: dict[tuple[int, ...], int] = {}

    def offset(self, group: tuple[int, ...]) -> int:
        off = self._off.get(group)
        if off is None:
            off = self._off[group] = len(self.ids)
            self.ids.extend(group)
        return off


_scratch = threading.local()


def _out_buffer(rows: int) -> np.ndarray:
    buf = getattr(_scratch, "out", None)
    if buf is None or len(buf) < rows:
        buf = _scratch.out = np.empty((max(rows, 4096), 6), dtype=np.int64)
    return buf


def _plan_native(rows: list[tuple[int, int, tuple, int, tuple, int]], total_heads: int,
                 kvb: int) -> np.ndarray:
    """rows: (request id, ctx, old group, old tp, new group, new tp) in plan order."""
    n = len(rows)
    if n == 0:
        return np.zeros((0, 6), dtype=np.int64)
    table = _GroupTable()
    cols = np.array([(r, c, table.offset(og), otp, table.offset(ng), ntp)
                     for r, c, og, otp, ng, ntp in rows], dtype=np.int64)
    meta = np.ascontiguousarray(cols[:, 2:6].T, dtype=np.int32)  # old_off, old_tp, new_off, new_tp
    return _call_planner(np.ascontiguousarray(cols[:, 0]), np.ascontiguousarray(cols[:, 1]), meta,
                         np.asarray(table.ids, dtype=np.int64), total_heads, kvb)


def _layout_table(layouts) -> tuple[np.ndarray, np.ndarray, _GroupTable]:
    """Per-layout (group offset, tp) into one shared group table."""
    table = _GroupTable()
    off = np.array([table.offset(lay.group) for lay in layouts], dtype=np.int32)
    tp = np.array([lay.tp for lay in layouts], dtype=np.int32)
    return off, tp, table


# below this many requests the row walk's lower fixed cost wins (measured on
# this host: 36 vs 60 us at 1 request, 98 vs 66 us at 32, 277 vs 85 us at 128)
_NATIVE_MIN_REQUESTS = 24


def _plan_layouts(old_layouts, new_layouts, total_heads: int, kvb: int):
    """plan_repartition's matching, checks and planning in libtpr
    (``tpr_plan_repartition``) over the layouts' cached request arrays.

    Same checks, order and messages as the row-by-row path below; returns None
    (use that path) when an old request id repeats, where the reference's
    last-one-wins dict semantics apply (migration.py:160-163).
    """
    o = [lay.request_arrays() for lay in old_layouts]
    nw = [lay.request_arrays() for lay in new_layouts]
    off, tp, table = _layout_table([*old_layouts, *new_layouts])
    n_old = len(old_layouts)
    cnt = np.array([len(a) for a, _ in o] + [len(a) for a, _ in nw], dtype=np.int64)
    cat = (lambda parts: np.concatenate(parts) if len(parts) > 1 else parts[0]) if o and nw else None
    if cat is None:
        return None
    old_req, old_ctx = cat([a for a, _ in o]), cat([c for _, c in o])
    new_req, new_ctx = cat([a for a, _ in nw]), cat([c for _, c in nw])
    ids = np.asarray(table.ids, dtype=np.int64)
    cap = max(len(new_req), 1) * total_heads
    out = _out_buffer(cap)
    n_out = _native.c_int64(0)
    lib = _native.load()
    cp, op, tpp = cnt.ctypes.data, off.ctypes.data, tp.ctypes.data
    rc = lib.tpr_plan_repartition(
        n_old, cp, op, tpp, old_req.ctypes.data, old_ctx.ctypes.data,
        len(new_layouts), cp + 8 * n_old, op + 4 * n_old, tpp + 4 * n_old,
        new_req.ctypes.data, new_ctx.ctypes.data, ids.ctypes.data, total_heads, int(kvb), cap,
        out.ctypes.data, _native.ctypes.byref(n_out))
    if rc == _native.TPR_ENOTFOUND:
        return None
    if rc != 0:
        raise MigrationError(lib.tpr_last_error().decode(errors="replace"))
    return out[: n_out.value].copy()


def _call_planner(req: np.ndarray, ctx: np.ndarray, meta: np.ndarray, ids: np.ndarray,
                  total_heads: int, kvb: int) -> np.ndarray:
    """tpr_plan_heads over int64 req/ctx and int32 meta [4][n]."""
    n = len(req)
    cap = n * total_heads
    out = _out_buffer(cap)
    n_out = _native.c_int64(0)
    base = meta.ctypes.data
    _native.call(
        "tpr_plan_heads", n, req.ctypes.data, ctx.ctypes.data, base, base + 4 * n, base + 8 * n,
        base + 12 * n, ids.ctypes.data, total_heads, int(kvb), cap, out.ctypes.data,
        _native.ctypes.byref(n_out),
    )
    return out[: n_out.value].copy()


def head_transfers(old: KvLayout, new: KvLayout, kv_bytes_per_token_per_head: int) -> list[Transfer]:
    """Coalesced head-range moves taking ``old``'s requests to ``new``'s placement.

    Reference: migration.py:101-134 (GPU sets are not checked, so the engine
    may use it for disjoint groups, engine.py:571-589).
    """
    return head_transfers_array(old, new, kv_bytes_per_token_per_head).transfers


def head_transfers_array(old: KvLayout, new: KvLayout, kvb: int) -> MigrationPlan:
    if old.total_heads != new.total_heads:
        raise MigrationError("head counts differ between layouts")
    req, ctx = old.request_arrays()
    if len(req) == 0:
        return MigrationPlan.from_array(np.zeros((0, 6), dtype=np.int64))
    off, tp, table = _layout_table([old, new])
    meta = np.empty((4, len(req)), dtype=np.int32)
    meta[0], meta[1], meta[2], meta[3] = off[0], tp[0], off[1], tp[1]
    return MigrationPlan.from_array(_call_planner(
        req, ctx, meta, np.asarray(table.ids, dtype=np.int64), old.total_heads, kvb))


_PACKED: list = []  # the last few (layout objects, blob): a controller alternates a few layout lists


def pack_layouts(old_layouts, new_layouts, release=()):
    """Old and new layouts as one int64 array for ``tpr_switch_prepare``
    (include/tpr.h): n_old, n_new, then every layout's ``packed()``, then --
    when ``release`` is not empty -- the ids of requests freed by the switch.
    Blobs of immutable layouts are remembered (looked up by equality)."""
    if isinstance(new_layouts, KvLayout):
        new_layouts = [new_layouts]
    if not release:
        key = (*old_layouts, None, *new_layouts)
        for k, blob in _PACKED:
            # tuple equality: identical layouts short-circuit in C; equal ones
            # (frozen dataclasses) pack to the same blob anyway
            if k == key:
                return blob
        if all(isinstance(lay.requests, tuple) for lay in key if lay is not None):
            blob = _pack(old_layouts, new_layouts, ())
            _PACKED.insert(0, (key, blob))
            del _PACKED[8:]
            return blob
    return _pack(old_layouts, new_layouts, release)


def _pack(old_layouts, new_layouts, release):
    flat = [len(old_layouts), len(new_layouts)]
    for lay in old_layouts:
        flat.extend(lay.packed())
    for lay in new_layouts:
        flat.extend(lay.packed())
    if release:
        flat.append(len(release))
        flat.extend(int(r) for r in release)
    return _array("q", flat)


def plan_repartition(old_layouts: list[KvLayout], new_layouts, kv_bytes_per_token_per_head: int,
                     handshake_ms: float = 0.0) -> MigrationPlan:
    """Transfers converting old TP groups into the new layout(s) (migration.py:137-189).

    Validation and transfer order follow the reference: new layouts in list
    order, each layout's requests in order, head runs ascending.
    """
    if isinstance(new_layouts, KvLayout):
        new_layouts = [new_layouts]
    old_gpus = {g for lay in old_layouts for g in lay.group}
    new_gpus = {g for lay in new_layouts for g in lay.group}
    if old_gpus != new_gpus:
        raise MigrationError(f"GPU sets differ: old={sorted(old_gpus)} new={sorted(new_gpus)}")
    if len({lay.total_heads for lay in [*old_layouts, *new_layouts]}) != 1:
        raise MigrationError("all layouts must share total_heads")
    total_heads = new_layouts[0].total_heads if new_layouts else (
        old_layouts[0].total_heads if old_layouts else 1)
    fast = None
    if sum(len(lay.requests) for lay in new_layouts) >= _NATIVE_MIN_REQUESTS:
        fast = _plan_layouts(old_layouts, new_layouts, total_heads, kv_bytes_per_token_per_head)
    if fast is not None:
        return MigrationPlan.from_array(fast, handshake_ms=handshake_ms)
    source: dict[int, tuple[KvLayout, int]] = {}
    for lay in old_layouts:
        for rid, ctx in lay.requests:
            source[rid] = (lay, ctx)  # a duplicated request: the last one wins
    carried = [rid for lay in new_layouts for rid, _ in lay.requests]
    if sorted(carried) != sorted(source):
        raise MigrationError("new layouts must carry exactly the old requests")
    rows = []
    for lay in new_layouts:
        for rid, ctx in lay.requests:
            old, old_ctx = source[rid]
            if old_ctx != ctx:
                raise MigrationError(f"request {rid}: context length changed")
            rows.append((rid, ctx, old.group, old.tp, lay.group, lay.tp))
    arr = _plan_native(rows, total_heads, kv_bytes_per_token_per_head)
    return MigrationPlan.from_array(arr, handshake_ms=handshake_ms)


def layout_placement(layouts) -> dict:
    """{(request, head): gpu} of canonical layouts (migration.py:210-218)."""
    if isinstance(layouts, KvLayout):
        layouts = [layouts]
    placement = {}
    for lay in layouts:
        owners = lay.owners()
        for rid, _ in lay.requests:
            for h, g in enumerate(owners):
                placement[(rid, h)] = g
    return placement


def apply_plan(old_layouts: list[KvLayout], plan: MigrationPlan) -> dict:
    """Replay ``plan`` on the old placement (migration.py:192-207)."""
    placement = layout_placement(list(old_layouts))
    for src, dst, rid, lo, hi, _ in plan.as_array().tolist():
        for h in range(lo, hi):
            here = placement.get((rid, h))
            if here != src:
                raise MigrationError(
                    f"transfer of request {rid} head {h} from gpu {src}, but it is on {here}"
                )
            placement[(rid, h)] = dst
    return placement


# ---------------------------------------------------------------------------
# cost models (migration.py:221-292), kept operation-for-operation
# ---------------------------------------------------------------------------

def _send_ms(nbytes: float, params: CostModelParams) -> float:
    return params.per_transfer_overhead_us / 1000.0 + nbytes / (params.link_bw_gbps * 1e9) * 1000.0


def _copy_ms(nbytes: float, params: CostModelParams) -> float:
    return nbytes / (params.copy_bw_gbps * 1e9) * 1000.0


def latency_per_page(plan: MigrationPlan, params: CostModelParams) -> float:
    """Page-at-a-time sends, serial per source, parallel across sources."""
    page_ms = _send_ms(params.page_bytes, params)
    per_source: dict[int, float] = {}
    for src, _dst, _r, _lo, _hi, nbytes in _rows(plan):
        per_source[src] = per_source.get(src, 0.0) + math.ceil(nbytes / params.page_bytes) * page_ms
    ms = max(per_source.values(), default=0.0)
    plan.predicted_latency_ms["per_page"] = ms
    return ms


def latency_aggregate(plan: MigrationPlan, params: CostModelParams) -> float:
    """Pack each source's fragments into one buffer, then one send."""
    ms = 0.0
    for nbytes in plan.bytes_by_source().values():
        ms = max(ms, _copy_ms(nbytes, params) + _send_ms(nbytes, params))
    plan.predicted_latency_ms["aggregate"] = ms
    return ms


def _pipelined_source_ms(total_bytes: int, params: CostModelParams) -> float:
    """Two-buffer schedule walked chunk by chunk (migration.py:252-272).

    copy i starts after copy i-1 and after send i-2 freed its buffer; send i
    starts after copy i and send i-1.
    """
    chunk = params.chunk_bytes
    n = math.ceil(total_bytes / chunk)
    copy_done = 0.0
    send_done = 0.0        # send i-1
    send_done_prev = 0.0   # send i-2
    for i in range(n):
        size = min(chunk, total_bytes - i * chunk)
        start = copy_done if i >= 1 else 0.0
        if i >= 2:
            start = max(start, send_done_prev)
        copy_done = start + _copy_ms(size, params)
        go = copy_done
        if i >= 1:
            go = max(go, send_done)
        send_done_prev, send_done = send_done, go + _send_ms(size, params)
    return send_done if n else 0.0


def latency_pipelined(plan: MigrationPlan, params: CostModelParams) -> float:
    ms = max((_pipelined_source_ms(b, params) for b in plan.bytes_by_source().values()),
             default=0.0)
    plan.predicted_latency_ms["pipelined"] = ms
    return ms


def switch_cost(mode: str, plan: MigrationPlan, params: CostModelParams) -> float:
    """Pause of a TP switch under a weight-handling regime (migration.py:284-292)."""
    if mode == WARM:
        return params.handshake_ms + latency_pipelined(plan, params)
    if mode == NAIVE_RELOAD:
        return params.reload_ms + latency_per_page(plan, params)
    if mode == NAIVE_KERNEL_INIT:
        return params.kernel_init_ms + latency_per_page(plan, params)
    raise MigrationError(f"unknown switch mode {mode!r}")


def weight_memory(mode: str, profile, tp: int | None = None) -> float:
    """GB of weights per GPU under a storage scheme (migration.py:295-306)."""
    full = profile.weight_full_copy_gb
    if mode == "full_copy_per_gpu":
        return full
    if mode == "per_tp_copies":
        return sum(full / level for level in profile.tp_levels)
    if mode == "sharded":
        if tp is None:
            raise MigrationError("sharded mode needs a tp level")
        return full / tp
    raise MigrationError(f"unknown weight memory mode {mode!r}")


def _rows(plan: MigrationPlan):
    if plan._list is not None:
        for t in plan._list:
            yield t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes
    else:
        yield from plan._arr.tolist()
