"""One process per GPU: push-model KV migration over CUDA-IPC peer pools.

Each rank owns the pool, block table and free ring of one GPU slot. The
buffers come from ``tpr_device_alloc`` (whole cudaMalloc allocations). Their
IPC handles are exchanged once with ``all_gather_object``, and every rank maps
its peers' buffers (``tpr_ipc_open``). A switch then runs like this:

1. handshake (modeled as ``handshake_ms``, migration.py:84): an
   all-gather of the plan digest and the ring counters, which every rank also
   tracks itself. It proves all ranks execute the same plan from the same
   state. It is the only exchange step.
2. K3 with ``filter_src = my slot``: allocation offsets follow the WHOLE plan,
   so a source rank computes the destination pages by itself, reading the
   peer's free ring and writing the peer's block table remotely.
3. K1 pushes the pages straight into peer pools (NVLink stores between GPUs).
4. stream sync + barrier: after it, every destination sees complete pages.

No data-path collective is involved; transfers leaving different ranks are
independent (migration.py:275-281 takes the max over sources).
The same code runs several ranks on ONE GPU (IPC between processes on one
device), which is how it is tested here.
"""

from __future__ import annotations

import ctypes
import hashlib
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .geometry import MAX_TP, KvGeometry, ModelGeometry
from .kvcache import MigrationStats, _PinnedStaging
from .migration import (BYTES, KvLayout, MigrationError, MigrationPlan, pack_layouts,
                        plan_repartition)
from .weights import ReshardStats, ShardedWeightStore, groups_ranges, window_for


class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (zero copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class DeviceBuffer:
    """A whole cudaMalloc allocation, viewed as a uint8 torch tensor."""

    def __init__(self, nbytes: int, device: torch.device):
        self.nbytes = int(nbytes)
        ptr = ctypes.c_uint64()
        with torch.cuda.device(device):
            _native.call("tpr_device_alloc", self.nbytes, ctypes.byref(ptr))
        self.ptr = ptr.value
        self.device = device
        self.tensor = torch.as_tensor(_CudaArray(self.ptr, self.nbytes), device=device)

    def handle(self) -> bytes:
        buf = (ctypes.c_uint8 * 64)()
        _native.call("tpr_ipc_get_handle", self.ptr, buf)
        return bytes(buf)

    def free(self):
        if self.ptr:
            self.tensor = None
            _native.call("tpr_device_free", self.ptr)
            self.ptr = 0


def open_peer(handle: bytes) -> int:
    buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    ptr = ctypes.c_uint64()
    _native.call("tpr_ipc_open", buf, ctypes.byref(ptr))
    return ptr.value


# ---------------------------------------------------------------------------
# host logic (CPU-testable)
# ---------------------------------------------------------------------------

def units_per_record(rec: np.ndarray, block_tokens: int) -> np.ndarray:
    nblk = (rec[:, 5].astype(np.int64) + block_tokens - 1) // block_tokens
    return (rec[:, 4] - rec[:, 3]).astype(np.int64) * nblk


def ring_deltas(rec: np.ndarray, n_slots: int, block_tokens: int):
    """Units allocated on / released by every slot for a record list."""
    u = units_per_record(rec, block_tokens)
    in_u = np.bincount(rec[:, 1], weights=u, minlength=n_slots).astype(np.int64)
    src = rec[:, 0] >= 0
    out_u = np.bincount(rec[src, 0], weights=u[src], minlength=n_slots).astype(np.int64)
    return in_u, out_u


def my_units(rec: np.ndarray, slot: int, block_tokens: int) -> int:
    """Pages the rank owning ``slot`` pushes (transfers leaving it)."""
    return int(units_per_record(rec[rec[:, 0] == slot], block_tokens).sum())


def plan_digest(rec: np.ndarray) -> int:
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(rec, np.int64).tobytes(),
                                          digest_size=8).digest(), "little", signed=True)


@dataclass
class HandshakeResult:
    digest: int
    heads: np.ndarray
    tails: np.ndarray


def handshake(rec: np.ndarray, heads, tails, group=None) -> HandshakeResult:
    """All-gather of (plan digest, ring counters); raises if ranks disagree."""
    mine = np.concatenate([[plan_digest(rec)], np.asarray(heads, np.int64),
                           np.asarray(tails, np.int64)]).astype(np.int64)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(mine).to(dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    rows = np.stack([o.cpu().numpy() for o in out])
    if not (rows == rows[0]).all():
        raise MigrationError("handshake: ranks disagree on the plan or on ring state")
    n = len(heads)
    return HandshakeResult(int(rows[0, 0]), rows[0, 1:1 + n], rows[0, 1 + n:])


# ---------------------------------------------------------------------------
# the per-rank cluster
# ---------------------------------------------------------------------------

class DistributedKvCluster:
    """The KV pool of ONE GPU slot (this rank) plus IPC views of its peers."""

    def __init__(self, kv: KvGeometry, gpu_ids, units_per_gpu: int, max_requests: int,
                 max_blocks: int, device: torch.device, group=None, fragmented: bool = False,
                 seed: int = 0):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if len(gpu_ids) != self.world:
            raise MigrationError("one GPU slot per rank")
        _native.load()
        self.kv = kv
        self.gpu_ids = tuple(gpu_ids)
        self.slot_of = {g: i for i, g in enumerate(self.gpu_ids)}
        self.slot = self.rank
        self.n_units = int(units_per_gpu)
        self.max_requests = int(max_requests)
        self.max_blocks = int(max_blocks)
        self.device = torch.device(device)
        H = kv.total_heads
        self.pool = DeviceBuffer(self.n_units * kv.unit_bytes, self.device)
        self.bt = DeviceBuffer(self.max_requests * H * self.max_blocks * 4, self.device)
        self.ring = DeviceBuffer(self.n_units * 4, self.device)
        self.bt.tensor.view(torch.int32).fill_(-1)
        order = (np.random.default_rng(seed + self.slot).permutation(self.n_units) if fragmented
                 else np.arange(self.n_units))
        self.ring.tensor.view(torch.int32).copy_(torch.from_numpy(order.astype(np.int32)))
        torch.cuda.synchronize(self.device)
        handles = (self.pool.handle(), self.bt.handle(), self.ring.handle())
        allh = [None] * self.world
        dist.all_gather_object(allh, handles, group=group)
        self.peer_ptrs = []
        for r, hs in enumerate(allh):
            if r == self.rank:
                self.peer_ptrs.append((self.pool.ptr, self.bt.ptr, self.ring.ptr))
            else:
                self.peer_ptrs.append(tuple(open_peer(h) for h in hs))
        self.ring_head = [0] * self.world
        self.ring_tail = [self.n_units] * self.world
        self.req_slot: dict[int, int] = {}
        self.slot_ctx = np.full(self.max_requests, -1, np.int32)
        self.owner = np.full((self.max_requests, H), -1, np.int32)
        self._free_req_slots = list(range(self.max_requests - 1, -1, -1))
        self._geo = _native.KvGeometryC(kv.layers, kv.head_dim, kv.dtype_bytes, kv.block_tokens,
                                        H, self.max_blocks, self.max_requests, self.n_units)
        self._staging = _PinnedStaging()
        # id -> slot lookup tables for the native switch bookkeeping
        ids = np.asarray(self.gpu_ids, dtype=np.int64)
        self._gpu_ids_arr = ids
        self._gpu_lut = None
        if ids.min() >= 0 and ids.max() < (1 << 24):
            self._gpu_lut = np.full(int(ids.max()) + 1, -1, dtype=np.int64)
            self._gpu_lut[ids] = np.arange(len(ids))
        self._req_lut = np.full(1024, -1, dtype=np.int64)
        self._swt = None
        self._plan_rows = np.empty((0, 6), np.int64)
        self._xf = torch.empty(0, dtype=torch.int32, device=self.device)
        self._meta = torch.empty(0, dtype=torch.int64, device=self.device)
        self._totals = torch.zeros(_native.TPR_TOTALS_LEN, dtype=torch.int64, device=self.device)
        self._work = torch.empty(0, dtype=torch.int32, device=self.device)
        self._work_ext = torch.empty(0, dtype=torch.int32, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.stream = torch.cuda.Stream(device=self.device)
        dist.barrier(group=group)

    def _cluster_c(self) -> _native.KvClusterC:
        c = _native.KvClusterC()
        c.n_gpus = self.world
        for s, (pool, bt, ring) in enumerate(self.peer_ptrs):
            c.pool[s], c.block_table[s], c.free_ring[s] = pool, bt, ring
            c.ring_head[s] = self.ring_head[s]
            c.ring_tail[s] = self.ring_tail[s]
        return c

    def _run_k3(self, rec: np.ndarray, filter_src: int, n_mine: int, want_ext: bool):
        st = self.stream
        grow = lambda t, n: t if t.numel() >= n else torch.zeros(max(n, 2 * t.numel()), dtype=t.dtype,
                                                                 device=self.device)
        with torch.cuda.stream(st):
            self._xf = grow(self._xf, len(rec) * 6)
            self._meta = grow(self._meta, len(rec) * 4)
            self._work = grow(self._work, (n_mine + 1) * 4)  # + K1 claim slot
            if want_ext:
                self._work_ext = grow(self._work_ext, max(n_mine, 1) * 4)
            self._staging.upload(rec.astype(np.int32), self._xf, st)
        cl = self._cluster_c()
        with torch.cuda.device(self.device):
            _native.call("tpr_kv_remap", ctypes.byref(self._geo), ctypes.byref(cl), self._xf.data_ptr(),
                         len(rec), filter_src, self._meta.data_ptr(), self._totals.data_ptr(), n_mine,
                         self._work.data_ptr(), self._work_ext.data_ptr() if want_ext else None,
                         self.status.data_ptr(), st.cuda_stream)
        return cl

    def _advance(self, rec: np.ndarray):
        in_u, out_u = ring_deltas(rec, self.world, self.kv.block_tokens)
        for s in range(self.world):
            free = self.ring_tail[s] - self.ring_head[s]
            if in_u[s] > free:
                raise MigrationError(f"gpu {self.gpu_ids[s]}: {in_u[s]} KV units needed, {free} free")
        return in_u, out_u

    def _commit(self, in_u, out_u):
        for s in range(self.world):
            self.ring_head[s] += int(in_u[s])
            self.ring_tail[s] += int(out_u[s])

    def admit(self, layouts, seed: int = 1) -> int:
        """Every rank calls with the same layouts; each allocates + fills its pages."""
        recs, new = [], []
        free = list(self._free_req_slots)
        seen = set()
        H = self.kv.total_heads
        for lay in layouts:
            # the checks of PagedKvCluster.admit: K3 indexes block-table rows by
            # (request slot, head, page), and these tables are mapped by peers
            if lay.total_heads != H:
                raise MigrationError("all layouts must share total_heads")
            hpr = lay.heads_per_rank
            for rid, ctx in lay.requests:
                if rid in self.req_slot or rid in seen:
                    raise MigrationError(f"request {rid} already resident")
                if self.kv.blocks(ctx) > self.max_blocks:
                    raise MigrationError(f"request {rid}: {ctx} tokens exceed max_blocks")
                if not free:
                    raise MigrationError("no free request slots")
                seen.add(rid)
                rs = free.pop()
                runs = [(self.slot_of[g], r * hpr, (r + 1) * hpr) for r, g in enumerate(lay.group)]
                new.append((rid, rs, int(ctx), runs))
                recs.extend((-1, s, rs, lo, hi, int(ctx)) for s, lo, hi in runs)
        rec = np.asarray(recs, np.int64).reshape(-1, 6)
        in_u, out_u = self._advance(rec)  # capacity check before any state change
        self._free_req_slots = free
        for rid, rs, ctx, runs in new:
            self.req_slot[rid] = rs
            self._set_req_lut(rid, rs)
            self.slot_ctx[rs] = ctx
            for s, lo, hi in runs:
                self.owner[rs, lo:hi] = s
        mine = rec[rec[:, 1] == self.slot]
        n = int(units_per_record(mine, self.kv.block_tokens).sum())
        if n:
            cl = self._run_k3(mine, -1, n, want_ext=True)
            with torch.cuda.device(self.device):
                _native.call("tpr_kv_fill", ctypes.byref(self._geo), ctypes.byref(cl),
                             self._work.data_ptr(), self._work_ext.data_ptr(), n, seed,
                             self.stream.cuda_stream)
        self._commit(in_u, out_u)
        self.pattern_seed = seed
        self.stream.synchronize()
        dist.barrier(group=self.group)
        return n

    def _set_req_lut(self, rid: int, slot: int) -> None:
        if 0 <= rid < (1 << 24):
            if rid >= len(self._req_lut):
                grown = np.full(max(rid + 1, 2 * len(self._req_lut)), -1, dtype=np.int64)
                grown[: len(self._req_lut)] = self._req_lut
                self._req_lut = grown
                self._swt = None
            self._req_lut[rid] = slot

    def _prepare(self, old_layouts, new_layouts):
        """The host half of the switch in libtpr (``tpr_switch_prepare``: plan,
        records, capacity check), identical on every rank. None when the
        switch needs the Python path (every error the reference reports)."""
        if self._gpu_lut is None:
            return None
        t = self._swt
        if t is None:
            t = self._swt = _native.SwitchTablesC()
            t.gpu_lut, t.gpu_lut_len = self._gpu_lut.ctypes.data, len(self._gpu_lut)
            t.gpu_ids = self._gpu_ids_arr.ctypes.data
            t.req_lut, t.req_lut_len = self._req_lut.ctypes.data, len(self._req_lut)
            t.slot_ctx, t.owner = self.slot_ctx.ctypes.data, self.owner.ctypes.data
            t.kvb = self.kv.kv_bytes_per_token_per_head
            t.validate, t.mode = 1, _native.TPR_SWITCH_REPARTITION
        blob = pack_layouts(old_layouts, new_layouts)
        cl = self._cluster_c()
        lib = _native.load()
        for _ in range(2):
            rows = self._plan_rows
            h_ptr, raw = self._staging.acquire(max(len(rows), 1) * 24)
            t.plan, t.plan_cap, t.records = rows.ctypes.data, len(rows), h_ptr
            rc = lib.tpr_switch_prepare(ctypes.byref(self._geo), ctypes.byref(cl),
                                        blob.buffer_info()[0], len(blob), ctypes.byref(t))
            if rc != _native.TPR_ECAPACITY:
                break
            self._plan_rows = np.empty((max(t.n_plan, 2 * len(rows)), 6), np.int64)
        if rc == _native.TPR_ENOTFOUND:
            return None
        if rc != 0:
            raise MigrationError(lib.tpr_last_error().decode(errors="replace"))
        n = t.n_plan
        rec32 = raw.view(np.int32)[: n * 6].reshape(n, 6)
        plan = MigrationPlan.from_array(self._plan_rows[:n].copy())
        in_u = np.array(t.in_units[: self.world], np.int64)
        out_u = np.array(t.out_units[: self.world], np.int64)
        return plan, h_ptr, rec32.astype(np.int64), in_u, out_u

    def launch_layouts(self, old_layouts, new_layouts, k1_events=None,
                       host_handshake: bool = True):
        """``plan_repartition`` + ``launch`` with the host half in libtpr; the
        pushes of this rank go out through ``tpr_kv_switch`` (records read
        zero-copy, K3 with filter_src = this slot, K1). Returns (plan, pending)."""
        prep = self._prepare(old_layouts, new_layouts)
        if prep is None:
            plan = plan_repartition(old_layouts, new_layouts, self.kv.kv_bytes_per_token_per_head)
            return plan, self.launch(plan, k1_events, host_handshake)
        plan, h_ptr, rec, in_u, out_u = prep
        if host_handshake:
            handshake(rec, self.ring_head, self.ring_tail, self.group)  # also the start barrier
        n = int(out_u[self.slot])  # units this slot pushes
        if n and k1_events:  # K1 alone between events: the split path
            self._staging.fence(self.stream)
            cl = self._run_k3(rec, self.slot, n, want_ext=False)
            k1_events[0].record(self.stream)
            self._k1(cl, n, rec)
            k1_events[1].record(self.stream)
        elif n:
            st = self.stream
            grow = lambda t_, k: t_ if t_.numel() >= k else torch.zeros(  # noqa: E731
                max(k, 2 * t_.numel()), dtype=t_.dtype, device=self.device)
            with torch.cuda.stream(st):
                self._xf = grow(self._xf, len(rec) * 6)
                self._meta = grow(self._meta, len(rec) * 4)
                self._work = grow(self._work, (n + 1) * 4)  # + K1 claim slot
            cl = self._cluster_c()
            with torch.cuda.device(self.device):
                _native.call("tpr_kv_switch", ctypes.byref(self._geo), ctypes.byref(cl), h_ptr,
                             self._xf.data_ptr(), len(rec), self.slot, self._meta.data_ptr(),
                             self._totals.data_ptr(), n, self._work.data_ptr(),
                             self.status.data_ptr(), st.cuda_stream)
            self._staging.fence(st)
        else:
            self._staging.fence(self.stream)
        return plan, (rec, in_u, out_u, n)

    def _k1(self, cl, n: int, rec: np.ndarray) -> None:
        full = not (rec[:, 5] % self.kv.block_tokens).any()
        with torch.cuda.device(self.device):
            _native.call("tpr_kv_migrate_ex", ctypes.byref(self._geo), ctypes.byref(cl),
                         self._work.data_ptr(), n, _native.TPR_MIGRATE_FULL_PAGES if full else 0,
                         self.stream.cuda_stream)

    def migrate_layouts(self, old_layouts, new_layouts) -> tuple:
        """Collective ``launch_layouts`` + barrier + ``finish``: (plan, stats)."""
        plan, pending = self.launch_layouts(old_layouts, new_layouts)
        self.stream.synchronize()
        dist.barrier(group=self.group)
        return plan, self.finish(plan, pending)

    def records(self, plan: MigrationPlan) -> np.ndarray:
        arr = plan.as_array()
        if len(arr) == 0:
            return np.zeros((0, 6), np.int64)
        src = np.array([self.slot_of[g] for g in arr[:, 0].tolist()], np.int64)
        dst = np.array([self.slot_of[g] for g in arr[:, 1].tolist()], np.int64)
        req = np.array([self.req_slot[r] for r in arr[:, 2].tolist()], np.int64)
        ctx = self.slot_ctx[req].astype(np.int64)
        if (arr[:, BYTES] != (arr[:, 4] - arr[:, 3]) * ctx * self.kv.kv_bytes_per_token_per_head).any():
            raise MigrationError("transfer bytes disagree with context length")
        return np.stack([src, dst, req, arr[:, 3], arr[:, 4], ctx], axis=1)

    def migrate(self, plan: MigrationPlan, k1_events=None) -> MigrationStats:
        """Collective over the group: every rank passes the same plan."""
        pending = self.launch(plan, k1_events)
        self.stream.synchronize()
        dist.barrier(group=self.group)  # every page has landed everywhere
        return self.finish(plan, pending)

    def launch(self, plan: MigrationPlan, k1_events=None, host_handshake: bool = True):
        """Handshake, then enqueue this rank's K3 + K1 on ``self.stream``.

        With ``host_handshake=False`` the caller provides the start barrier on
        the stream (DeviceBarrier) and no host collective runs."""
        rec = self.records(plan)
        in_u, out_u = self._advance(rec)
        if host_handshake:
            handshake(rec, self.ring_head, self.ring_tail, self.group)  # also the start barrier
        n = my_units(rec, self.slot, self.kv.block_tokens)
        if n:
            cl = self._run_k3(rec, self.slot, n, want_ext=False)
            if k1_events:
                k1_events[0].record(self.stream)
            self._k1(cl, n, rec)
            if k1_events:
                k1_events[1].record(self.stream)
        return rec, in_u, out_u, n

    def finish(self, plan: MigrationPlan, pending) -> MigrationStats:
        """Host bookkeeping once every rank's pages have landed (after the barrier)."""
        rec, in_u, out_u, n = pending
        self._commit(in_u, out_u)
        heads = np.arange(self.kv.total_heads)
        mask = (heads >= rec[:, 3:4]) & (heads < rec[:, 4:5])
        rows = np.broadcast_to(rec[:, 2:3], mask.shape)
        self.owner[rows[mask], np.broadcast_to(heads, mask.shape)[mask]] = \
            np.broadcast_to(rec[:, 1:2], mask.shape)[mask]
        return MigrationStats(len(rec), n, int(plan.as_array()[:, BYTES].sum()) if len(rec) else 0,
                              {self.gpu_ids[s]: int(v) for s, v in enumerate(in_u) if v},
                              {self.gpu_ids[s]: int(v) for s, v in enumerate(out_u) if v})

    def verify(self) -> dict:
        ctx = torch.from_numpy(self.slot_ctx).to(self.device)
        owner = torch.from_numpy(self.owner).to(self.device)
        counts = torch.zeros(3, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            _native.call("tpr_kv_verify", ctypes.byref(self._geo), self.pool.ptr, self.bt.ptr,
                         ctx.data_ptr(), owner.data_ptr(), self.slot, self.pattern_seed,
                         counts.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
        c = counts.cpu().tolist()
        return {"placement_errors": c[0], "word_mismatches": c[1], "pages_checked": c[2],
                "status": int(self.status.item())}

    def tables_snapshot(self) -> dict:
        """This slot's block table and free ring + all ring counters (no pool)."""
        torch.cuda.synchronize(self.device)
        return {"block_tables": [self.bt.tensor.view(torch.int32).cpu().numpy()],
                "rings": [self.ring.tensor.view(torch.int32).cpu().numpy()],
                "ring_head": list(self.ring_head), "ring_tail": list(self.ring_tail)}

    def snapshot(self) -> dict:
        torch.cuda.synchronize(self.device)
        return {"pool": self.pool.tensor.cpu().numpy(),
                "block_table": self.bt.tensor.view(torch.int32).cpu().numpy(),
                "ring": self.ring.tensor.view(torch.int32).cpu().numpy(),
                "ring_head": list(self.ring_head), "ring_tail": list(self.ring_tail)}

    def close(self):
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for r, ptrs in enumerate(self.peer_ptrs):
            if r != self.rank:
                for p in ptrs:
                    _native.call("tpr_ipc_close", p)
        dist.barrier(group=self.group)
        for b in (self.pool, self.bt, self.ring):
            b.free()


# ---------------------------------------------------------------------------
# weights: K2 pulls missing slices from peers' arenas over IPC
# ---------------------------------------------------------------------------

class _PeerPtr:
    """A peer's arena as seen through its IPC mapping (only .data_ptr())."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def data_ptr(self) -> int:
        return self.ptr


class DistributedWeightStore(ShardedWeightStore):
    """The sharded weights of ONE GPU (this rank) + IPC views of its peers.

    Each rank owns two slice-addressed arenas (double buffer) of ``max_slices``
    slices (its window). Both are registered with every peer once. A reshard
    uses the same planner as the single-process store, so every rank computes
    the same plan, source choice and egress balance. A shard that grows inside
    its window pulls only the missing slices from the peers' current arenas
    straight into their positions of its CURRENT arena (remote loads over
    NVLink; the resident slices are not touched, and peers may read them
    meanwhile). A shard that leaves its window is rebuilt into the idle arena,
    and the rank flips to it after the end barrier; the old one stays readable
    until the next reshard, which starts after a barrier."""

    def __init__(self, model: ModelGeometry, gpu_ids, device: torch.device, group=None,
                 max_slices: int = MAX_TP, mode: str = "sharded"):
        super().__init__(model, gpu_ids, device=device, mode=mode, max_slices=max_slices)
        self.group = group
        self.rank = dist.get_rank(group)
        if len(self.gpu_ids) != dist.get_world_size(group):
            raise MigrationError("one GPU per rank")
        self.me = self.gpu_ids[self.rank]
        self.device = torch.device(device)
        cap = max(self.max_slices[self.me] * self.bytes_per_slice, 16)
        self.bufs = [DeviceBuffer(cap, self.device), DeviceBuffer(cap, self.device)]
        handles = [b.handle() for b in self.bufs]
        allh = [None] * len(self.gpu_ids)
        dist.all_gather_object(allh, handles, group=group)
        self.peer_bufs = {}
        for r, g in enumerate(self.gpu_ids):
            self.peer_bufs[g] = ([b.ptr for b in self.bufs] if g == self.me
                                 else [open_peer(h) for h in allh[r]])
        self.cur = {g: 0 for g in self.gpu_ids}
        self.stream = torch.cuda.Stream(device=self.device)

    def _views(self):
        arena = {}
        for g in self.gpu_ids:
            if g == self.me:
                arena[g] = self.bufs[self.cur[g]].tensor[: self.window[g][1] * self.bytes_per_slice]
            else:
                arena[g] = _PeerPtr(self.peer_bufs[g][self.cur[g]])
        self.arena = arena

    def _check_windows(self, windows) -> None:
        for g, (_, m) in windows.items():
            if m > self.max_slices[g]:
                raise MigrationError(f"gpu {g}: shard exceeds max_slices={self.max_slices[g]}")

    def load(self, groups, stream=None) -> None:
        act = groups_ranges(groups)
        if set(act) != set(self.gpu_ids):
            raise MigrationError("groups must cover exactly the store's GPUs")
        for g in self.gpu_ids:
            res = (0, MAX_TP) if self.mode == "full_copy_per_gpu" else act[g]
            self.window[g] = window_for(*res, self.max_slices[g])
            self.have[g] = frozenset(range(*res))
            self.active[g] = act[g]
        self._check_windows(self.window)
        self._views()
        rep_bytes = sum(m.rows * m.cols for m in self.replicated) * self.model.dtype_bytes
        self.rep_arena = {self.me: torch.empty(max(rep_bytes, 16), dtype=torch.uint8, device=self.device)}
        st = stream or self.stream
        with torch.cuda.device(self.device):
            self._fill(self.me, st, *((0, MAX_TP) if self.mode == "full_copy_per_gpu"
                                      else act[self.me]))
        st.synchronize()
        dist.barrier(group=self.group)

    def launch(self, new_groups, parked=(), events=None):
        """Plan (same on every rank) and enqueue this rank's K2 pull."""
        plan = self.plan(new_groups, parked)
        self._check_windows(plan.window)
        stats = self._stats(plan)
        if events:
            events[0].record(self.stream)
        me = self.me
        if plan.fetch[me] or plan.relayout[me]:
            # in place: the current arena; a new window: the idle one
            target = self.bufs[self.cur[me] ^ int(plan.relayout[me])].tensor
            seg = np.ascontiguousarray(self._segments(me, plan, target))
            stats.segments = len(seg)
            self._launch(seg, self.device, self.stream)
        if events:
            events[1].record(self.stream)
        return plan, stats

    def finish(self, pending) -> ReshardStats:
        """After the barrier: flip GPUs that moved to a new window."""
        plan, stats = pending
        for g in self.gpu_ids:
            if plan.relayout[g]:
                self.cur[g] ^= 1
        self.have, self.window, self.active = plan.have, plan.window, plan.active
        self._views()
        return stats

    def reshard(self, new_groups, stream=None, events=None, parked=()) -> ReshardStats:
        pending = self.launch(new_groups, parked, events)
        self.stream.synchronize()
        dist.barrier(group=self.group)
        return self.finish(pending)

    def verify(self, stream=None) -> int:
        saved = self.gpu_ids
        try:
            self.gpu_ids = (self.me,)
            return super().verify(stream)
        finally:
            self.gpu_ids = saved

    def close(self):
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for g, ptrs in self.peer_bufs.items():
            if g != self.me:
                for p in ptrs:
                    _native.call("tpr_ipc_close", p)
        dist.barrier(group=self.group)
        self.arena = {}
        for b in self.bufs:
            b.free()


class DeviceBarrier:
    """Stream-ordered barrier across the group through IPC-mapped flags
    (``tpr_device_barrier``): no host collective on the switch path."""

    def __init__(self, device: torch.device, group=None, timeout_s: float = 30.0):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.timeout_ns = int(timeout_s * 1e9)
        self.status = torch.zeros(1, dtype=torch.int32, device=torch.device(device))
        self.flags = DeviceBuffer(8 * self.world, torch.device(device))
        self.flags.tensor.zero_()
        torch.cuda.synchronize(device)
        allh = [None] * self.world
        dist.all_gather_object(allh, self.flags.handle(), group=group)
        ptrs = [self.flags.ptr if r == self.rank else open_peer(h) for r, h in enumerate(allh)]
        self._peers = ptrs
        self.ptrs = (ctypes.c_uint64 * self.world)(*ptrs)
        self.epoch = 0
        dist.barrier(group=group)

    def __call__(self, stream: torch.cuda.Stream, status: torch.Tensor | None = None) -> None:
        """Enqueue the barrier. A timeout ORs TPR_STATUS_BARRIER_TIMEOUT into
        ``status`` (default: this barrier's own word). Passing the KV cluster's
        status word makes the K3 that follows abort (no table, ring or pool is
        touched, K1 skips every item) instead of writing into peers that never
        arrived."""
        self.epoch += 1
        st = self.status if status is None else status
        _native.call("tpr_device_barrier", self.ptrs, self.rank, self.world, self.epoch,
                     self.timeout_ns, st.data_ptr(), stream.cuda_stream)

    def check(self, *extra: torch.Tensor) -> None:
        """Raise if a barrier gave up waiting (host sync on the status words)."""
        for st in (self.status, *extra):
            if int(st.item()) & _native.TPR_STATUS_BARRIER_TIMEOUT:
                raise MigrationError("device barrier timed out: a peer rank never arrived")

    def close(self):
        dist.barrier(group=self.group)
        for r, p in enumerate(self._peers):
            if r != self.rank:
                _native.call("tpr_ipc_close", p)
        dist.barrier(group=self.group)
        self.flags.free()


class DistributedExecutor:
    """One-process-per-GPU TP switch: start barrier, this rank's K3 + K1 push
    on one stream and its K2 pull on another, end barrier, commit.

    ``device_barrier=True`` (default) runs both barriers as tiny kernels over
    IPC-mapped flags, so a switch costs no host collective; the metadata
    handshake (plan digest + ring counters, an all-gather) is then optional
    (``check_every`` switches, 0 = never)."""

    def __init__(self, kv: DistributedKvCluster, weights: DistributedWeightStore | None = None,
                 device_barrier: bool = True, check_every: int = 0,
                 barrier_timeout_s: float = 30.0):
        self.kv = kv
        self.weights = weights
        self.barrier = (DeviceBarrier(kv.device, kv.group, timeout_s=barrier_timeout_s)
                        if device_barrier else None)
        self.check_every = check_every
        self.n = 0
        self.broken = False

    def switch(self, old_layouts, new_layouts, new_weight_groups=None, parked=(),
               k1_events=None, k2_events=None):
        import time
        if self.broken:
            raise MigrationError("a device barrier timed out earlier: the barrier epochs and "
                                 "ring counters of the ranks may disagree; rebuild the executor")
        t0 = time.perf_counter()
        self.n += 1
        kst = self.kv.stream
        wst = self.weights.stream if self.weights is not None else None
        start = None
        if self.barrier is None:  # host handshake = the start barrier
            plan, kv_pending = self.kv.launch_layouts(old_layouts, new_layouts, k1_events)
        else:
            # every rank is here: peers' pools / tables / rings are quiescent. A
            # timeout lands in the KV status word, so this rank's K3 + K1 abort
            self.barrier(kst, self.kv.status)
            start = torch.cuda.Event()
            start.record(kst)
            check = bool(self.check_every and self.n % self.check_every == 0)
            plan, kv_pending = self.kv.launch_layouts(old_layouts, new_layouts, k1_events,
                                                      host_handshake=check)
        w_pending = None
        if self.weights is not None and new_weight_groups is not None:
            # K2 pulls only need the start barrier: it runs alongside K3 + K1
            # (KV pushes use egress links, weight pulls ingress)
            if start is not None:
                wst.wait_event(start)
            w_pending = self.weights.launch(new_weight_groups, parked, k2_events)
        if self.barrier is None:
            kst.synchronize()
            if wst is not None:
                wst.synchronize()
            dist.barrier(group=self.kv.group)
        else:
            if wst is not None:
                kst.wait_stream(wst)
            self.barrier(kst)  # every rank's pushes and pulls have completed
            kst.synchronize()
            try:
                self.barrier.check(self.kv.status)
            except MigrationError:
                self.broken = True
                raise
        kv_stats = self.kv.finish(plan, kv_pending)
        w_stats = self.weights.finish(w_pending) if w_pending is not None else None
        return plan, kv_stats, w_stats, (time.perf_counter() - t0) * 1e3

    def close(self):
        if self.barrier is not None:
            self.barrier.close()


__all__ = ["DistributedKvCluster", "DistributedWeightStore", "DistributedExecutor", "DeviceBuffer",
           "handshake", "ring_deltas", "my_units", "plan_digest", "units_per_record", "KvLayout"]
