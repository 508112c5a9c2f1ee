"""Reconfiguration controller execution hook.

In the reference the controller's hook ``Simulator._apply_config``
(pkg/src/tpsim/engine.py:500-621) builds per-request ``KvLayout``s
(engine.py:571-582), calls ``head_transfers`` (engine.py:583-589), prices the
resulting ``MigrationPlan`` with ``switch_cost`` (+ ``planning_delay_ms``,
engine.py:590-597) and pauses the destination groups for that long
(engine.py:607-609). ``ReconfigurationExecutor.switch`` is the executed form
of steps d-g: handshake, plan, K3 block-table remap, K1 KV migration on one
stream in parallel with K2 weight reshard on another, barrier, resume. It
returns the measured pause, which replaces ``switch_cost`` in the engine
(see INTEGRATION.md).
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass, field

import torch

from . import _native
from .kvcache import MigrationStats, PagedKvCluster
from .migration import KvLayout, MigrationPlan, plan_repartition
from .placement import Arrival, KvBudget, enforce_kv_capacity, kv_capacity_decisions, reuse_layouts
from .tracing import nvtx
from .weights import ReshardStats, ShardedWeightStore


@dataclass
class SwitchResult:
    plan: MigrationPlan
    kv: MigrationStats
    weights: ReshardStats | None
    host_ms: float = 0.0        # pause -> resume wall time (only when synced)
    status: int = 0             # K3 status bits (0 = every head was where the plan said)
    events: dict = field(default_factory=dict)
    new_layouts: list | None = None  # the layouts the switch realised (reuse_order may reorder ranks)
    evicted: list = field(default_factory=list)  # arrivals the destination could not hold (released)
    _device_ms: float | None = field(default=None, repr=False)
    _timed: bool = field(default=False, repr=False)

    @property
    def bytes(self) -> int:
        return self.kv.bytes + (self.weights.bytes if self.weights else 0)

    @property
    def device_ms(self) -> float:
        """CUDA-event time of the switch on the device, from its first launch
        to the end of its last kernel (only when synced; 0.0 otherwise). Read
        from the switch's events on first access: cudaEventElapsedTime costs
        ~6 us of host time, which a synchronous switch does not pay."""
        if self._device_ms is None:
            if self._timed:
                self.events["end"].synchronize()  # a ticket-waited switch may still be retiring
                self._device_ms = self.events["start"].elapsed_time(self.events["end"])
            else:
                self._device_ms = 0.0
        return self._device_ms

    @device_ms.setter
    def device_ms(self, value: float) -> None:
        self._device_ms = float(value)


_SYNC_EVENT_PAIRS = 64  # event pairs an executor cycles through for synchronous switches


class ReconfigurationExecutor:
    """Executes TP switches on a PagedKvCluster (+ optional ShardedWeightStore)."""

    def __init__(self, kv: PagedKvCluster, weights: ShardedWeightStore | None = None,
                 handshake=None, time_kernels: bool = False, overlap: bool | None = None):
        self.kv = kv
        self.weights = weights
        self.handshake = handshake  # callable(plan) for multi-process metadata exchange
        dev = kv.home
        self.device = dev
        self.kv_stream = torch.cuda.Stream(device=dev)
        # K1 || K2 on two streams pays off when they use different links (KV
        # pushes egress, weight pulls ingress). With every slot in one HBM both
        # are bound by the same bandwidth, so by default they run back to back
        # on one stream and each kernel streams at full rate.
        if overlap is None:
            overlap = not kv._single_device
        self.overlap = overlap
        self.w_stream = torch.cuda.Stream(device=dev) if overlap else self.kv_stream
        self.time_kernels = time_kernels
        self._status_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        # numpy views of the pinned status words (indexing a tensor costs
        # microseconds on the small-switch path)
        self._status_np = self._status_host.numpy()
        self._kv_status_np = kv.status_host.numpy()
        self.main_stream = torch.cuda.current_stream(dev)
        # synchronous switches cycle through a ring of event pairs; a result
        # reads its device time lazily, and a pair is re-used only after the
        # result that last held it (if still alive and unread) has read it
        self._ev_ring = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                         for _ in range(_SYNC_EVENT_PAIRS)]
        for pair in self._ev_ring:  # create the CUDA events now; libtpr records them by handle
            for e in pair:
                e.record(self.main_stream)
        self._ev_handles = [(e0.cuda_event, e1.cuda_event) for e0, e1 in self._ev_ring]
        self._ev_users = [None] * _SYNC_EVENT_PAIRS
        self._ev_next = 0
        self._record = _native.load().tpr_event_record

    @property
    def _ev_sync(self):
        """The event pair the next synchronous switch records (tools use it)."""
        return self._ev_ring[self._ev_next]

    def _take_sync_events(self):
        i = self._ev_next
        self._ev_next = (i + 1) % _SYNC_EVENT_PAIRS
        prev = self._ev_users[i]
        if prev is not None:
            r = prev()
            if r is not None and r._device_ms is None:
                r.device_ms  # noqa: B018 -- read before the pair is re-recorded
            self._ev_users[i] = None
        return i, self._ev_ring[i]

    def _finish(self, res: SwitchResult, main: torch.cuda.Stream, t0: float,
                slot: int | None = None) -> SwitchResult:
        """Synchronous tail: the end event is recorded, the host waits -- on the
        one-launch kernel's completion ticket in pinned memory when it has one
        (no weight copy followed), else on the end event -- and reads the
        status word, which the one-call switch mirrors into pinned memory on
        the stream (other paths: a 4-byte D2H here)."""
        mirrored = self.kv.status_mirrored
        if not mirrored:
            _native.call("tpr_memcpy_d2h", self._status_host.data_ptr(), self.kv.status.data_ptr(),
                         4, main.cuda_stream)
        end = res.events["end"]
        if slot is not None:
            if self._record(self._ev_handles[slot][1], main.cuda_stream):
                raise _native.NativeError(_native.load().tpr_last_error().decode(errors="replace"))
        else:
            end.record(main)
        no_k2 = res.weights is None or res.weights.segments == 0
        ticket = self.kv.last_ticket if mirrored and no_k2 else 0
        if ticket:
            # the one-launch switch writes its ticket into pinned memory once
            # every copy and table write is done: spin on it instead of
            # waiting for the end event (which completes a few us later)
            word = self._kv_status_np
            spins = 0
            while word[1] != ticket:
                spins += 1
                if not spins & 0xfff and end.query() and word[1] != ticket:
                    raise _native.NativeError("switch kernel finished without its ticket")
        else:
            end.synchronize()
        res.status = int((self._kv_status_np if mirrored else self._status_np)[0])
        res.host_ms = (time.perf_counter() - t0) * 1e3
        res._timed = True  # device_ms: read on first access
        if slot is not None:
            self._ev_users[slot] = weakref.ref(res)
        return res

    def switch(self, old_layouts: list[KvLayout], new_layouts: list[KvLayout],
               new_weight_groups=None, parked=(), sync: bool = True,
               validate: bool = True, stream: torch.cuda.Stream | None = None,
               trim: bool = False, reuse_order: bool = False,
               arrivals=None, kv_budget: KvBudget | None = None) -> SwitchResult:
        """Stop-and-migrate TP switch. With ``sync`` the call returns after the
        switch completed on the device and reports measured latencies; without
        it, work is only enqueued and ``stream`` (default: the device's default
        stream) waits for it. ``trim`` compacts GPUs whose resident weight
        slices exceed their new shard (ShardedWeightStore.reshard).
        ``reuse_order`` re-ranks every new group to keep the most KV in place
        (placement.reuse_layouts); the realised layouts are in
        ``SwitchResult.new_layouts``. It changes the plan the reference would
        produce, so it is off by default. Weight groups follow the new ranks.

        ``arrivals`` (placement.Arrival per migrating request): destination
        KV-capacity admission inside the switch, as the reference's hook does
        with ``kv_accounting`` (engine.py:600-601, 623-645). For every new
        layout, its arrivals are decided against ``kv_budget`` bytes
        ((gpu_memory_gb - weight_full_copy_gb) * 1e9 * tp, with the group's
        other requests as ``used``) -- or, without a budget, against the
        destination GPUs' free pages. Evicted requests leave both layout lists
        and their pages are freed by the same native call; they are listed in
        ``SwitchResult.evicted`` for the caller to re-queue."""
        t0 = time.perf_counter()
        if isinstance(new_layouts, KvLayout):
            new_layouts = [new_layouts]
        evicted = []
        if arrivals is not None:
            old_layouts, new_layouts, evicted = self._admit(old_layouts, new_layouts, arrivals,
                                                            kv_budget)
        if reuse_order:
            new_layouts = reuse_layouts(old_layouts, new_layouts,
                                        self.kv.kv.kv_bytes_per_token_per_head)
            if new_weight_groups is not None:  # a weight group follows its KV group's ranks
                ranked = {frozenset(lay.group): lay.group for lay in new_layouts}
                new_weight_groups = [ranked.get(frozenset(g), tuple(g)) for g in new_weight_groups]
        main = stream or self.main_stream
        ev = {}
        slot = None
        # one stream unless K1 and K2 overlap: no cross-stream event waits on
        # the (latency-bound) small-switch path
        ks = self.kv_stream if self.overlap else main
        one_call = self.handshake is None
        start_handle = None
        if sync:
            slot, (e0, e1) = self._take_sync_events()
            ev = {"start": e0, "end": e1}
            if one_call and ks is main:  # recorded by libtpr right before the first launch
                start_handle = self._ev_handles[slot][0]
            else:
                e0.record(main)
        if self.time_kernels:
            for k in ("k1_start", "k1_end", "k2_start", "k2_end"):
                ev[k] = torch.cuda.Event(enable_timing=True)
        if ks is not main:
            ks.wait_stream(main)
        if one_call:
            # plan + records + K3 + K1 in one native call (K1 bracketed by events
            # when the kernels are timed)
            with nvtx("plan+kv K3+K1"):
                plan, kv_stats = self.kv.switch_layouts(
                    old_layouts, new_layouts, stream=ks, validate=validate,
                    k1_events=(ev["k1_start"], ev["k1_end"]) if self.time_kernels else None,
                    release=evicted, start_event=start_handle,
                    want_ticket=sync and (self.weights is None or new_weight_groups is None))
        else:
            with nvtx("plan"):
                plan = plan_repartition(old_layouts, new_layouts,
                                        self.kv.kv.kv_bytes_per_token_per_head)
            if self.handshake is not None:
                with nvtx("handshake"):
                    self.handshake(plan)
            with nvtx("kv K3+K1"):
                kv_stats = self.kv.migrate(
                    plan, stream=ks, validate=validate,
                    k1_events=(ev["k1_start"], ev["k1_end"]) if self.time_kernels else None)
                if evicted:
                    self.kv.release(evicted, stream=ks)
        w_stats = None
        if self.weights is not None and new_weight_groups is not None:
            ws = self.w_stream if self.overlap else main
            if ws is not main:
                ws.wait_stream(main)
            with nvtx("weights K2"):
                w_stats = self.weights.reshard(
                    new_weight_groups, stream=ws, parked=parked, trim=trim,
                    events=(ev["k2_start"], ev["k2_end"]) if self.time_kernels else None)
            if ws is not main:
                main.wait_stream(ws)
        if ks is not main:
            main.wait_stream(ks)
        res = SwitchResult(plan=plan, kv=kv_stats, weights=w_stats, events=ev,
                           new_layouts=list(new_layouts), evicted=evicted)
        return self._finish(res, main, t0, slot) if sync else res

    def _admit(self, old_layouts, new_layouts, arrivals, kv_budget):
        """(old, new, evicted): the layouts without the arrivals each new
        group cannot hold (placement.kv_capacity_decisions per group)."""
        kv = self.kv.kv
        per_token = kv.kv_bytes_per_token_per_head * kv.total_heads
        by_id = {a.request_id: a for a in arrivals}
        gone, out_new = [], []
        for lay in new_layouts:
            ctx = dict(lay.requests)
            arr = [Arrival(r, ctx[r], by_id[r].label, by_id[r].arrival_time)
                   for r, _ in lay.requests if r in by_id]
            if not arr:
                out_new.append(lay)
                continue
            if kv_budget is not None:
                used = sum(c for r, c in lay.requests if r not in by_id) * per_token
                _, ev = kv_capacity_decisions(arr, kv_budget.bytes(lay.tp), used, per_token)
            else:
                _, ev = enforce_kv_capacity(self.kv, lay, arr)
            drop = {a.request_id for a in ev}
            gone.extend(a.request_id for a in ev)
            out_new.append(KvLayout(lay.group, lay.tp, lay.total_heads,
                                    tuple(rc for rc in lay.requests if rc[0] not in drop)))
        if not gone:
            return old_layouts, out_new, []
        drop = set(gone)
        out_old = [KvLayout(lay.group, lay.tp, lay.total_heads,
                            tuple(rc for rc in lay.requests if rc[0] not in drop))
                   for lay in old_layouts]
        return out_old, out_new, gone

    def handoff(self, prefill: KvLayout, decode: KvLayout, sync: bool = True) -> SwitchResult:
        """Prefill->decode KV handoff between disjoint groups.

        The reference prices it as ``_pipelined_source_ms(_kv_bytes)`` when a
        prefill completes (engine.py:340-354). The engine path plans with
        ``head_transfers`` on arbitrary groups (engine.py:571-589); that is
        exactly what runs here, through K3 + K1."""
        t0 = time.perf_counter()
        main = torch.cuda.current_stream(self.device)
        slot = None
        if sync:
            slot, (e0, e1) = self._take_sync_events()
            ev = {"start": e0, "end": e1}
        else:
            ev = {k: torch.cuda.Event(enable_timing=True) for k in ("start", "end")}
        ev["start"].record(main)
        ks = self.kv_stream if self.overlap else main
        if ks is not main:
            ks.wait_event(ev["start"])
        # head_transfers + records + K3 + K1 in one native call
        plan, stats = self.kv.switch_layouts(prefill, decode, stream=ks, planner="head_transfers",
                                             want_ticket=sync)
        if ks is not main:
            main.wait_stream(ks)
        res = SwitchResult(plan=plan, kv=stats, weights=None, events=ev)
        if sync:
            return self._finish(res, main, t0, slot)
        ev["end"].record(main)
        return res


def measured_switch_cost(executor: ReconfigurationExecutor):
    """Adapter with the signature of ``migration.switch_cost(mode, plan, params)``
    that executes ``plan`` (already in this cluster's placement) and returns the
    pause in ms, for wiring into the reference engine.

    The modes keep the reference's meaning (migration.py:284-292): ``warm`` is
    the measured switch plus the metadata handshake ``params.handshake_ms``
    (the reference's warm cost is handshake + the pipelined copy model);
    ``naive_reload`` / ``naive_kernel_init`` add ``params.reload_ms`` /
    ``params.kernel_init_ms`` to the measured KV move, since a naive switch
    also reloads weights / re-initialises kernels, which this data path does
    not execute. Any other mode raises the reference's MigrationError."""
    from .migration import NAIVE_KERNEL_INIT, NAIVE_RELOAD, WARM, MigrationError

    def cost(mode, plan: MigrationPlan, params) -> float:
        if mode not in (WARM, NAIVE_RELOAD, NAIVE_KERNEL_INIT):
            raise MigrationError(f"unknown switch mode {mode!r}")
        t0 = time.perf_counter()
        executor.kv.migrate(plan, stream=executor.kv_stream)
        executor.kv_stream.synchronize()
        measured = (time.perf_counter() - t0) * 1e3
        if mode == WARM:
            return params.handshake_ms + measured
        if mode == NAIVE_RELOAD:
            return params.reload_ms + measured
        return params.kernel_init_ms + measured

    return cost


def host_to_device_bytes(plan: MigrationPlan, w: ReshardStats | None) -> int:
    """Bytes a switch uploads: transfer records + weight copy segments/prefix."""
    n = plan.n_transfers
    segs = w.segments if w else 0
    return n * 6 * 4 + (segs * 64 + (segs + 1) * 8 if segs else 0)


__all__ = ["ReconfigurationExecutor", "SwitchResult", "measured_switch_cost",
           "host_to_device_bytes"]
