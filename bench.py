"""TP-switch benchmark (BASELINE.json metric: TP-switch latency (ms) and
KV+weight reshard GB/s vs the NVLink/HBM roofline).

One step = one complete stop-and-migrate TP switch of the workload: plan
(native planner), K3 block-table remap, K1 paged-KV migration on one stream in
parallel with K2 weight reshard on another, joined. Steps alternate A->B and
B->A so every step is a real switch of the same workload (the reverse moves
the same KV bytes, test_migration.py:146-155).

Default workload (N=1): BASELINE configs[1], Llama-3.1-8B TP2<->TP4, 64 seqs x
4096 tokens of bf16 KV + sharded weights, on 4 logical GPUs whose pools all
live in one B200's HBM (the 1-GPU mode: every byte is an HBM read + write).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N>1) there is one process per GPU slot and the switch is real
and cross-GPU: TP(N/2) <-> TP(N) over the N GPUs (16 seqs x 4096 per GPU, so
per-GPU work is fixed: weak scaling). KV pages are pushed and weight slices
pulled through CUDA-IPC peer mappings, with device-side barriers over IPC
flags. Rank 0 prints value = bytes moved by all ranks / max-over-ranks device
time. (On a box with fewer GPUs than ranks, ranks share devices.)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TP-switch latency (ms) and KV+weight reshard GB/s vs NVLink/HBM roofline"


def _engine_name() -> str:
    from paper_2605_05467_b200 import _native
    return _native.copy_engine()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def copy_peak_in_run(device, gib: int = 2, reps: int = 5) -> float:
    """The MEASURED_PEAKS.json method repeated inside this run on this box:
    ``b.copy_(a)`` over ``gib`` GiB, read + write bytes, best of ``reps``
    (CUDA events). Context for a K1 fraction at or above 1.0: the peak file
    was written on another box/run, and TMA bulk copies can edge past the copy
    kernel the peak was taken with."""
    import torch
    a = torch.empty(gib << 30, dtype=torch.uint8, device=device)
    b = torch.empty_like(a)
    best = 0.0
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * a.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del a, b
    torch.cuda.empty_cache()
    return best


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = 10):
        self.index = index
        self.interval_ms = interval_ms
        self.proc = None
        self.samples: list[tuple[float, str]] = []
        self.t0 = self.t1 = None

    def _reader(self):
        for line in self.proc.stdout:
            if line.strip():
                self.samples.append((time.time(), line))

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self.thread = threading.Thread(target=self._reader, daemon=True)
            self.thread.start()
            deadline = time.time() + 3.0
            while not self.samples and time.time() < deadline:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = self.t0 or 0.0, self.t1 or float("inf")
        window = [l for t, l in self.samples if t0 <= t <= t1]
        if not window and self.samples:  # region shorter than one interval
            mid = (t0 + t1) / 2
            window = [min(self.samples, key=lambda s: abs(s[0] - mid))[1]]
        for line in window:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# setup
# ---------------------------------------------------------------------------

def build_workload(cfg: int, seqs: int | None):
    from paper_2605_05467_b200 import workloads
    kw = {}
    if seqs:
        kw["seqs"] = seqs
    return workloads.config(cfg, **kw)


def capacity_units(w, kv) -> dict:
    """Pool units per GPU at the peak of either switch direction: pages
    resident before the switch + pages received (sources release only after
    the copy)."""
    from paper_2605_05467_b200 import migration as M
    ctx = dict(w.requests)
    peak = {g: 0 for g in w.gpus}
    for a, b in ((w.old, w.new), (w.new, w.old)):
        need = {g: 0 for g in w.gpus}
        for lay in a:
            for rid, c in lay.requests:
                for g in lay.owners():
                    need[g] += kv.blocks(c)
        arr = M.plan_repartition(a, b, kv.kv_bytes_per_token_per_head).as_array()
        for src, dst, rid, lo, hi, _ in arr.tolist():
            need[dst] += (hi - lo) * kv.blocks(ctx[rid])
        for g in w.gpus:
            peak[g] = max(peak[g], need[g])
    return {g: n + 64 for g, n in peak.items()}


def setup_ours(w, device, overlap=None, weights_mode="sharded", fragmented=True):
    import torch
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    from paper_2605_05467_b200.kvcache import PagedKvCluster
    from paper_2605_05467_b200.weights import ShardedWeightStore

    kv = w.model.kv
    max_ctx = max(c for _, c in w.requests)
    cluster = PagedKvCluster(kv, w.gpus, units_per_gpu=capacity_units(w, kv),
                             max_requests=len(w.requests), max_blocks=kv.blocks(max_ctx),
                             device=device, fragmented=fragmented, seed=0)
    cluster.admit(w.old, seed=1234)
    store = None
    if w.old_weight_groups is not None:
        # every GPU's arena window holds its largest shard of the workload, so
        # growing shards fetch only their missing slices, in place
        store = ShardedWeightStore(w.model, w.gpus, device=device, mode=weights_mode,
                                   max_slices=cpu_windows(w))
        store.load(w.old_weight_groups)
    torch.cuda.synchronize()
    return ReconfigurationExecutor(cluster, store, time_kernels=True, overlap=overlap)


def k1_kernel_name(w) -> str:
    """The K1 kernel this workload launches: the TMA bulk kernel (partial pages
    as tensor boxes), or the vector engine's when that is selected."""
    from paper_2605_05467_b200 import _native
    if _native.copy_engine() != "bulk":
        return "tpr_k1_kv_migrate<8> (vector engine)"
    B = w.model.kv.block_tokens
    full = all(c % B == 0 for _, c in w.requests)
    return "tpr_k1_kv_migrate_bulk" + ("" if full else " (tensor boxes for partial pages)")


def weights_note(w, w_bytes) -> str:
    if w.old_weight_groups is None:
        if w.model.name.endswith("70B"):
            return ("KV only at N=1: 8 logical slots of 70B shards (2 full copies at TP4) exceed one "
                    "180 GB HBM; K2 on the 70B matrix shapes: tools/weight_sweep.py --model 70b")
        return "KV only (the BASELINE config names no weight reshard)"
    if w_bytes == 0:
        return ("weight reshard runs, but after the first switch every new shard lies inside a "
                "resident slice range (reuse): steady-state switches are views, 0 bytes")
    if w.trim_on_reverse:
        return ("sharded weights: the consolidation gathers 7/8 of the model onto GPU0 (K2), the "
                "reverse switch compacts GPU0 back to its TP8 slice (trim)")
    return "sharded weights: missing slices rebuilt by K2 every switch"


def one_switch(ex, w, forward: bool, sync: bool):
    if forward:
        return ex.switch(w.old, w.new, new_weight_groups=w.new_weight_groups,
                         parked=w.parked, sync=sync, validate=False)
    return ex.switch(w.new, w.old, new_weight_groups=w.old_weight_groups, parked=(),
                     sync=sync, validate=False, trim=w.trim_on_reverse)


# ---------------------------------------------------------------------------
# CPU reference path (oracle restatement; test infrastructure)
# ---------------------------------------------------------------------------

def reference_planner():
    """The reference's own ``tpsim.migration`` from ``baseline/_ref`` (the
    unmodified reference, installed by build() from /root/reference), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "tpsim" / "migration.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import tpsim.migration as RM  # noqa: N813
    return RM


class CpuReference:
    """The reference's CPU path for one switch of the workload, on host memory:

    * the plan from the reference's OWN planner, ``tpsim.migration.
      plan_repartition`` of the unmodified reference (baseline/_ref; the
      restatement oracle/plan_oracle.py only when it is absent), timed apart
      as ``planner_ms``;
    * page movement and weight slicing: the reference has no KV or weight bytes,
      so these run as the C restatement (oracle/kvmove.c), all host threads.

    ``sample_seqs`` < all runs a bounded sample (the same share of every weight
    slice) when the full workload does not fit the host's free memory."""

    def __init__(self, w, sample_seqs: int, threads: int):
        from oracle import kvmove, plan_oracle
        self.kvmove, self.po = kvmove, plan_oracle
        kvmove.build()
        self.RM = reference_planner()
        self.threads = threads
        reqs = w.requests[:sample_seqs]
        groups_old = [lay.group for lay in w.old]
        groups_new = [lay.group for lay in w.new]
        H = w.model.n_kv_heads
        self.H = H
        self.old = [(g, H, r) for g, r in zip(groups_old, _split(w.old, reqs))]
        self.new = [(g, H, r) for g, r in zip(groups_new, _split(w.new, reqs))]
        if self.RM is not None:
            mk = lambda lays: [self.RM.KvLayout(tuple(g), len(g), H, tuple(r)) for g, _, r in lays]
            self.ref_old, self.ref_new = mk(self.old), mk(self.new)
        kv = w.model.kv
        self.kv = kv
        self.kvb = kv.kv_bytes_per_token_per_head
        self.slot = {g: i for i, g in enumerate(w.gpus)}
        self.rslot = {rid: i for i, (rid, _) in enumerate(reqs)}
        self.ctx = dict(reqs)
        max_blocks = max(kv.blocks(c) for _, c in reqs)
        units = cpu_units(w, reqs)
        self.geo = dict(layers=kv.layers, head_dim=kv.head_dim, dtype_bytes=kv.dtype_bytes,
                        block_tokens=kv.block_tokens, total_heads=H, max_blocks=max_blocks,
                        n_req_slots=len(reqs), n_units=max(units))
        n = len(w.gpus)
        self.pools = [kvmove.filled(u * kv.unit_bytes, 1, threads) for u in units]
        self.tables = [np.full(len(reqs) * H * max_blocks, -1, np.int32) for _ in range(n)]
        rng = np.random.default_rng(0)
        self.rings = [rng.permutation(u).astype(np.int32) for u in units]
        self.head = [0] * n
        self.tail = list(units)
        adm = []
        for grp, _, rr in self.old:
            per = H // len(grp)
            for rid, c in rr:
                for r, g in enumerate(grp):
                    adm.append((-1, self.slot[g], self.rslot[rid], r * per, (r + 1) * per, c))
        self._exec(np.asarray(adm, np.int64))
        # weights: every GPU holds whole slices (one host buffer per slice, the
        # `frac` share of its bytes); a switch fetches exactly the slices the
        # GPU arm's K2 fetches (cpu_weight_moves), copied from a holder
        self.frac = sample_seqs / len(w.requests)
        self.wbytes_slice = None
        if w.old_weight_groups is not None:
            from paper_2605_05467_b200.weights import groups_ranges
            self.wbytes_slice = cpu_slice_bytes(w, self.frac)
            self.ranges = {True: groups_ranges(w.new_weight_groups),
                           False: groups_ranges(w.old_weight_groups)}
            self.trim = {True: False, False: w.trim_on_reverse}
            self.parked = {True: set(w.parked), False: set()}
            m = cpu_windows(w)
            old = self.ranges[False]
            self.win = {g: _window(*old[g], m[g]) for g in w.gpus}
            self.held = {g: {sl: kvmove.filled(self.wbytes_slice, 1, threads)
                             for sl in range(*old[g])} for g in w.gpus}
        self.fwd = True
        self.planner_s = 0.0

    def _exec(self, rec):
        n, status, self.head, self.tail = self.kvmove.kv_migrate(
            self.geo, self.pools, self.tables, self.rings, self.head, self.tail, rec, self.threads)
        assert status == 0
        return n

    def plan(self):
        """(src, dst, request, lo, hi, bytes) rows of this step's switch, from the
        reference's plan_repartition (timed)."""
        t0 = time.perf_counter()
        if self.RM is not None:
            src, dst = (self.ref_old, self.ref_new) if self.fwd else (self.ref_new, self.ref_old)
            plan = self.RM.plan_repartition(src, dst, self.kvb)
            moves = [(t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes)
                     for t in plan.transfers]
        else:
            src, dst = (self.old, self.new) if self.fwd else (self.new, self.old)
            moves = self.po.plan(src, dst, self.kvb)
        self.planner_s += time.perf_counter() - t0
        return moves

    def step(self) -> int:
        """One switch of the sample; returns bytes moved."""
        moves = self.plan()
        rec = np.array([(self.slot[s], self.slot[d], self.rslot[r], lo, hi, self.ctx[r])
                        for s, d, r, lo, hi, _ in moves], np.int64).reshape(-1, 6)
        self._exec(rec)
        moved = sum(m[5] for m in moves)
        if self.wbytes_slice:
            moved += self._weights(self.fwd)
        self.fwd = not self.fwd
        return moved

    def _weights(self, fwd: bool) -> int:
        moves, self.win, keep = cpu_weight_step(self.held, self.win, self.ranges[fwd],
                                                self.parked[fwd], self.trim[fwd])
        blocks, new = [], {}
        for g, sl, h in moves:
            buf = np.empty(self.wbytes_slice, np.uint8)
            new.setdefault(g, {})[sl] = buf
            blocks.append((buf, 0, self.held[h][sl], 0, 1, self.wbytes_slice, self.wbytes_slice,
                           self.wbytes_slice))
        if blocks:
            self.kvmove.copy_blocks(blocks, self.threads)
        for g in self.held:
            self.held[g] = {sl: b for sl, b in self.held[g].items() if sl in keep[g]}
            self.held[g].update(new.get(g, {}))
        return len(moves) * self.wbytes_slice


def cpu_windows(w) -> dict:
    """Arena window (slices) of every GPU: the largest shard it takes in the
    workload (the bench's max_slices for the GPU arm)."""
    from paper_2605_05467_b200.weights import groups_ranges
    out = {g: 1 for g in w.gpus}
    for groups in (w.old_weight_groups, w.new_weight_groups):
        for g, (a, b) in groups_ranges(groups).items():
            out[g] = max(out[g], b - a)
    return out


def _window(x: int, y: int, m: int):
    m = max(m, y - x)
    return (x // m) * m, m


def cpu_weight_step(held: dict, win: dict, act: dict, parked: set, trim: bool):
    """The slice-level rules of ShardedWeightStore.plan restated on host slice
    buffers: a shard inside its GPU's window keeps every held slice (only the
    shard's with ``trim``), one that leaves it starts a new window; every
    missing slice of the new shard is fetched from the least-loaded holder.
    Returns (moves [(gpu, slice, holder)], new windows, kept slices)."""
    order = list(held)
    egress = {g: 0 for g in order}
    moves, keep, new_win = [], {}, dict(win)
    for g in order:
        if g in parked or g not in act:
            keep[g] = set(held[g])
            continue
        x, y = act[g]
        w0, m = win[g]
        if w0 <= x and y <= w0 + m:
            keep[g] = (set(range(x, y)) & set(held[g])) if trim else set(held[g])
        else:
            new_win[g] = _window(x, y, m)
            keep[g] = set(range(x, y)) & set(held[g])
        for sl in range(x, y):
            if sl in held[g]:
                continue
            h = min((k for k in order if k != g and sl in held[k]),
                    key=lambda k: (egress[k], order.index(k)))
            egress[h] += 1
            moves.append((g, sl, h))
    return moves, new_win, keep


def cpu_slice_bytes(w, frac: float) -> int:
    split = [m for m in w.model.matrices if m.split != "rep"]
    per_slice = sum((m.rows * m.cols) // 8 for m in split) * w.model.dtype_bytes
    return max(int(per_slice * frac) // 64 * 64, 64)


def cpu_units(w, reqs) -> list:
    """Pool units per slot for the CPU sample: resident + incoming at the peak
    of either switch direction (bench.capacity_units on the sample)."""
    H = w.model.n_kv_heads
    kv = w.model.kv
    rid = {r for r, _ in reqs}
    from paper_2605_05467_b200.migration import KvLayout
    sub = lambda lays: [KvLayout(l.group, l.tp, H, tuple(r for r in l.requests if r[0] in rid))
                        for l in lays]
    ws = type(w)(w.name, w.model, w.gpus, sub(w.old), sub(w.new), None, None)
    cap = capacity_units(ws, kv)
    return [cap[g] for g in w.gpus]


def _split(layouts, reqs):
    """The sample's requests, grouped like ``layouts``."""
    rid = {r for r, _ in reqs}
    return [[r for r in lay.requests if r[0] in rid] for lay in layouts]


def _rr(groups, reqs):
    per = [[] for _ in groups]
    for i, r in enumerate(reqs):
        per[i % len(groups)].append(r)
    return per


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_host_bytes(w, n_seqs: int) -> int:
    """Host bytes the CPU arm holds for ``n_seqs`` of the workload: KV pools at
    their peak plus the weight slices at their peak over a few alternating
    switches (held + fetched before the replaced ones are freed)."""
    reqs = w.requests[:n_seqs]
    kv = sum(cpu_units(w, reqs)) * w.model.kv.unit_bytes
    if w.old_weight_groups is None:
        return kv
    from paper_2605_05467_b200.weights import groups_ranges
    m = cpu_windows(w)
    ranges = {True: groups_ranges(w.new_weight_groups), False: groups_ranges(w.old_weight_groups)}
    held = {g: dict.fromkeys(range(*ranges[False][g])) for g in w.gpus}
    win = {g: _window(*ranges[False][g], m[g]) for g in w.gpus}
    peak = sum(len(h) for h in held.values())
    fwd = True
    for _ in range(4):
        moves, win, keep = cpu_weight_step(held, win, ranges[fwd], set(w.parked) if fwd else set(),
                                           w.trim_on_reverse and not fwd)
        peak = max(peak, sum(len(h) for h in held.values()) + len(moves))
        for g in held:
            held[g] = {sl: None for sl in held[g] if sl in keep[g]}
        for g, sl, _ in moves:
            held[g][sl] = None
        fwd = not fwd
    return kv + peak * cpu_slice_bytes(w, n_seqs / len(w.requests))


def cpu_sample_seqs(w, requested: int | None, budget_frac: float = 0.6) -> int:
    """The whole workload (``requested`` None) when it fits ``budget_frac`` of
    the host's available memory, else the largest sample that does."""
    import psutil
    n = len(w.requests) if not requested else min(requested, len(w.requests))
    budget = psutil.virtual_memory().available * budget_frac
    while n > 1 and cpu_host_bytes(w, n) > budget:
        n = max(1, int(n * budget / cpu_host_bytes(w, n)) if n > 8 else n - 1)
    return n


def run_cpu_reference(w, steps: int, warmup: int, sample_seqs: int | None = None,
                      min_seconds: float = 0.0):
    """Time the reference's CPU path: `steps` switches of the workload (or of a
    sample when the host cannot hold it), continuing until at least
    `min_seconds` of CPU work have been timed."""
    sample_seqs = cpu_sample_seqs(w, sample_seqs)
    threads = cpu_threads()
    ref = CpuReference(w, sample_seqs, threads)
    for _ in range(warmup):
        ref.step()
    ref.planner_s = 0.0
    t0 = time.perf_counter()
    moved = done = 0
    while done < steps or time.perf_counter() - t0 < min_seconds:
        moved += ref.step()
        done += 1
    dt = time.perf_counter() - t0
    full = sample_seqs == len(w.requests)
    what = "the whole workload" if full else (
        f"{sample_seqs} of {len(w.requests)} seqs (+ the same share of every weight slice)")
    planner = ("reference tpsim.migration.plan_repartition (baseline/_ref, unmodified)"
               if ref.RM is not None else "restatement oracle/plan_oracle.py")
    return {"value": moved / dt / 1e9, "ms_per_step": dt / done * 1e3, "bytes": moved,
            "threads": threads, "seconds": dt, "same_config": full,
            "planner": planner, "planner_ms": ref.planner_s / done * 1e3,
            "sample": f"{what}, {done} alternating switches, {dt:.1f} s timed; plan: {planner}, "
                      "pages + weight slices: oracle/kvmove.c on all host threads"}


# ---------------------------------------------------------------------------
# N > 1: one process per GPU, real cross-GPU switch (push KV, pull weights)
# ---------------------------------------------------------------------------

def distributed_workload(world: int, seqs: int | None):
    """Weak scaling: TP(N/2) <-> TP(N) over N GPUs, 16 seqs x 4096 per GPU,
    Llama-3.1-8B KV + sharded weights (N=4 is BASELINE configs[1])."""
    from paper_2605_05467_b200 import workloads
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    return workloads.transition(LLAMA_3_1_8B, world, max(world // 2, 1), world,
                                seqs or 16 * world, 4096, weights=True,
                                name=f"Llama-3.1-8B TP{max(world // 2, 1)}<->TP{world} "
                                     f"{seqs or 16 * world}x4096 KV+weights, {world} GPUs")


# NVLink roofline denominator: the measured peer copy per direction per GPU
# (B200_PROFILING.md; 900 GB/s nominal NVLink 5, for context)
NVLINK_GBS = 770.0


def link_roofline(own_gpus: bool, egress: dict, ingress: dict, total_bytes: int, ms: float,
                  hbm: float, hbm_src: str, k1_ms: float) -> dict:
    """Roofline of a multi-process switch. With a GPU per rank the bound is the
    busiest NVLink direction: t_roof = max_g max(E_g, I_g) / 770 GB/s, the
    measured peer copy (SURVEY §8d with B200_PROFILING.md's denominator);
    ``achieved`` is that GPU's bytes over the measured time. With ranks sharing
    one device every byte is an HBM read + write."""
    if own_gpus:
        busiest = max(max(egress.values()), max(ingress.values()))
        achieved = busiest / (ms * 1e-3) / 1e9
        return {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_GBS, "unit": "GB/s",
                "frac": achieved / NVLINK_GBS, "traffic": None, "kernel": "tpr_k1_kv_migrate",
                "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 nominal)",
                "busiest_gpu_bytes": busiest, "k1_ms_rank0": k1_ms}
    achieved = 2 * total_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "kernel": "tpr_k1_kv_migrate",
            "peak_source": hbm_src, "k1_ms_rank0": k1_ms}


def run_distributed(args, w, rank: int, world: int, local: int):
    import datetime

    import torch
    import torch.distributed as dist

    from paper_2605_05467_b200.distributed import (DistributedExecutor, DistributedKvCluster,
                                                   DistributedWeightStore)

    n_dev = torch.cuda.device_count()
    device = torch.device("cuda", local % n_dev)
    torch.cuda.set_device(device)
    # NCCL carries the control plane (IPC-handle exchange, optional handshake)
    # when every rank has its own GPU; ranks that share a device use gloo
    backend = "nccl" if n_dev >= world else "gloo"
    # libtpr picks the copy engine per pointer: peer pools / arenas on other
    # GPUs take the 16-byte vector engine (the TMA engine is validated on local
    # HBM only), so no override is needed here
    dist.init_process_group(backend, timeout=datetime.timedelta(minutes=10),
                            **({"device_id": device} if backend == "nccl" else {}))
    kv = w.model.kv
    units = capacity_units(w, kv)
    max_ctx = max(c for _, c in w.requests)
    cl = DistributedKvCluster(kv, w.gpus, units_per_gpu=max(units.values()),
                              max_requests=len(w.requests), max_blocks=kv.blocks(max_ctx),
                              device=device, fragmented=True, seed=rank)
    cl.admit(w.old, seed=1234)
    ws = DistributedWeightStore(w.model, w.gpus, device=device, max_slices=cpu_windows(w))
    ws.load(w.old_weight_groups)
    # ranks sharing one device are time-sliced, so a spinning device barrier
    # would wait for a context switch; use the host barrier there
    ex = DistributedExecutor(cl, ws, device_barrier=n_dev >= world)

    def step(fwd):
        if fwd:
            return ex.switch(w.old, w.new, new_weight_groups=w.new_weight_groups)
        return ex.switch(w.new, w.old, new_weight_groups=w.old_weight_groups)

    fwd = True
    for _ in range(max(args.warmup, 1)):
        step(fwd)
        fwd = not fwd
    from paper_2605_05467_b200 import _native
    dev_ms, wall_ms, kv_bytes, w_bytes, k1, h2d = 0.0, [], 0, 0, [], 0
    # per-GPU link bytes over the timed steps (whole job; every rank plans the same)
    egress = {g: 0 for g in w.gpus}
    ingress = {g: 0 for g in w.gpus}
    launches = 0
    with ClockSampler(device.index) as clk:
        dist.barrier()
        clk.start()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(cl.stream)
            plan, ks, wst, ms = ex.switch(*((w.old, w.new) if fwd else (w.new, w.old)),
                                          new_weight_groups=w.new_weight_groups if fwd else w.old_weight_groups,
                                          k1_events=(e[2], e[3]))
            e[1].record(cl.stream)
            fwd = not fwd
            torch.cuda.synchronize(device)
            # the switch's device span on this rank: KV stream start -> end (K2 ran alongside)
            dev_ms += e[0].elapsed_time(e[1])
            k1.append(e[2].elapsed_time(e[3]))
            wall_ms.append(ms)
            kv_bytes += ks.bytes
            w_bytes += wst.bytes if wst else 0
            arr = plan.as_array()
            for src, dst, nb in zip(arr[:, 0].tolist(), arr[:, 1].tolist(), arr[:, 5].tolist()):
                egress[src] += nb
                ingress[dst] += nb
            if wst:
                for g in w.gpus:
                    egress[g] += wst.egress.get(g, 0)
                    ingress[g] += wst.ingress.get(g, 0)
            # this rank's kernels: 2 device barriers, K3 (+ K1) over its pushes, K2 pull
            launches += (2 if ex.barrier is not None else 0) + _native.kv_switch_launches(ks.units, ks.transfers) \
                + (1 if wst and wst.segments else 0)
            h2d += plan.n_transfers * 24 + (wst.segments * 72 + 8 if wst and wst.segments else 0)
        wall = time.perf_counter() - t0
        clk.stop()
        dist.barrier()
    cdev = device if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([dev_ms, wall], dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, wall = float(t[0]), float(t[1])
    nl = torch.tensor([launches], dtype=torch.int64, device=cdev)
    dist.all_reduce(nl, op=dist.ReduceOp.SUM)
    launches = int(nl.item())
    v1 = cl.verify()
    v2 = ws.verify()
    ok = torch.tensor([int(v1["placement_errors"] == 0 and v1["word_mismatches"] == 0 and v2 == 0)],
                      device=cdev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    ex.close()
    ws.close()
    cl.close()
    dist.destroy_process_group()
    if rank != 0:
        return
    total = kv_bytes + w_bytes
    hbm, src = peaks()
    line = {
        "metric": METRIC, "value": total / (dev_ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": w.name, "model": w.model.name, "seqs": len(w.requests),
                   "ctx": w.requests[0][1], "parallelism": f"{world} processes, one GPU slot each, "
                   "KV pushed / weights pulled through CUDA-IPC peer mappings",
                   "devices_used": n_dev, "kv_bytes_per_step": kv_bytes / args.steps,
                   "weight_bytes_per_step": w_bytes / args.steps,
                   "l2": "inputs larger than L2"},
        "roofline": link_roofline(n_dev >= world, egress, ingress, kv_bytes + w_bytes, dev_ms,
                                  hbm, src, float(np.mean(k1))),
        "clocks": clk.summary(),
        "e2e": {"value": total / wall / 1e9, "unit": "GB/s", "ms_per_step": wall / args.steps * 1e3,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": 0},
        "gpu_launches": launches,
        "bit_exact_property": bool(ok.item()),
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def measure_single(args, w, device, with_cpu: bool, e2e_on: bool = True) -> dict:
    """One GPU, logical ranks: the device-timed switches, the end-to-end public
    call, the full-size correctness property and (``cpu``) the reference's CPU
    path on the same workload (``with_cpu``). Returns the JSON fields."""
    import torch
    from paper_2605_05467_b200 import _native
    from paper_2605_05467_b200.controller import host_to_device_bytes

    ex = setup_ours(w, device, overlap={"auto": None, "on": True, "off": False}[args.overlap],
                    weights_mode=args.weights_mode, fragmented=args.pool_layout == "fragmented")
    fwd = True
    for _ in range(max(args.warmup, 1)):
        one_switch(ex, w, fwd, sync=True)
        fwd = not fwd

    # ---- device-timed region: K switches enqueued back to back --------------
    main_stream = torch.cuda.current_stream(device)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    results = []
    with ClockSampler(device.index if device.index is not None else 0) as clk:
        torch.cuda.synchronize()
        clk.start()
        start.record(main_stream)
        for _ in range(args.steps):
            results.append(one_switch(ex, w, fwd, sync=False))
            fwd = not fwd
        end.record(main_stream)
        torch.cuda.synchronize()
        clk.stop()
    ms = start.elapsed_time(end)
    kv_bytes = sum(r.kv.bytes for r in results)
    w_bytes = sum(r.weights.bytes for r in results if r.weights)
    w_local = sum(r.weights.local_bytes for r in results if r.weights)
    total_bytes = kv_bytes + w_bytes
    k1_ms = [r.events["k1_start"].elapsed_time(r.events["k1_end"]) for r in results]
    k2_ms = [r.events["k2_start"].elapsed_time(r.events["k2_end"]) for r in results
             if r.weights is not None and r.weights.segments]
    launches = sum(_native.kv_switch_launches(r.kv.units, r.kv.transfers)
                   + (1 if r.weights is not None and r.weights.segments else 0) for r in results)
    status = int(ex.kv.status.item())

    # ---- end to end through the public API (host layouts -> device -> status) --
    e2e = None
    if e2e_on:
        torch.cuda.synchronize()
        ex.time_kernels = False  # the production call: plan + K3 + K1 in one native call
        t0 = time.perf_counter()
        eb, h2d = 0, 0
        for _ in range(args.steps):
            r = one_switch(ex, w, fwd, sync=True)
            fwd = not fwd
            eb += r.bytes
            h2d += host_to_device_bytes(r.plan, r.weights)
            status |= r.status
        e2e_s = time.perf_counter() - t0
        e2e = {"value": eb / e2e_s / 1e9, "unit": "GB/s", "ms_per_step": e2e_s / args.steps * 1e3,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": 4}

    # ---- after the timed regions: full-size correctness of the final state ----
    # every owned page carries its placement-invariant pattern, every block-table
    # entry realises the host placement, every weight shard equals its slice
    vkv = ex.kv.verify()
    vw = ex.weights.verify() if ex.weights is not None else 0
    bit_exact = (vkv["placement_errors"] == 0 and vkv["word_mismatches"] == 0
                 and vkv["status"] == 0 and vw == 0 and status == 0)
    overlap = ex.overlap
    del ex, results
    import gc
    gc.collect()
    torch.cuda.empty_cache()

    hbm, hbm_src = peaks()
    k1_avg = float(np.mean(k1_ms))
    kv_per_step = kv_bytes / args.steps
    achieved = 2 * kv_per_step / (k1_avg * 1e-3) / 1e9  # HBM read + write GB/s
    # DRAM bytes of one K1 launch of this workload from this round's ncu --set
    # full capture (tools/ncu_traffic.py writes the file from the raw CSV)
    traffic = None
    prof = ROOT / "profiles" / "k1_traffic.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            if tj.get("workload") == w.name:
                traffic = tj.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    cpu = None
    if with_cpu:
        r = run_cpu_reference(w, 2, 1, args.cpu_sample_seqs, min_seconds=args.cpu_seconds)
        cpu = {"value": r["value"], "unit": "GB/s", "cores": r["threads"], "kind": "port",
               "sample": r["sample"], "cpu": cpu_model(), "ms_per_step": r["ms_per_step"],
               "same_config": r["same_config"], "planner": r["planner"],
               "planner_ms": r["planner_ms"]}
    return {
        "ms": ms, "value": total_bytes / (ms * 1e-3) / 1e9, "kv_per_step": kv_per_step,
        "w_per_step": w_bytes / args.steps, "w_local_per_step": w_local / args.steps,
        "w_bytes": w_bytes, "overlap": overlap,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "kernel": k1_kernel_name(w),
                     "k1_ms": k1_avg, "k2_ms": float(np.mean(k2_ms)) if k2_ms else None,
                     "peak_source": hbm_src,
                     # the whole switch (K3 + K1 + K2 + gaps): all bytes read + written
                     "step_achieved": 2 * total_bytes / args.steps / (ms / args.steps * 1e-3) / 1e9,
                     "step_frac": 2 * total_bytes / (ms * 1e-3) / 1e9 / hbm},
        "cpu_baseline": cpu, "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches,
        "status": status, "bit_exact_property": bit_exact, "pages_verified": vkv["pages_checked"],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=1, help="BASELINE configs[] index (0-based)")
    ap.add_argument("--seqs", type=int, default=None)
    ap.add_argument("--cpu-sample-seqs", type=int, default=None,
                    help="sequences of the CPU arm (default: the whole workload if the host "
                         "memory holds it)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="minimum timed CPU work of the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-headline", action="store_true",
                    help="skip the north-star headline (Llama-3.1-8B 8 x 32768 TP2<->TP4)")
    ap.add_argument("--engine", choices=("vector", "bulk"), default=None,
                    help="K1/K2 copy engine (default: the library default)")
    ap.add_argument("--overlap", choices=("auto", "on", "off"), default="auto",
                    help="K1 || K2 on two streams (auto: only across devices)")
    ap.add_argument("--pool-layout", choices=("fragmented", "contiguous"), default="fragmented",
                    help="free-ring order of the KV pools: a random permutation (PAPER.md:342) "
                         "or ascending")
    ap.add_argument("--weights-mode", choices=("sharded", "full_copy_per_gpu"), default="sharded",
                    help="weight storage (weight_memory modes): sharded moves missing slices, "
                         "full_copy_per_gpu (the paper's design) switches by views only")
    args = ap.parse_args()
    if args.engine and args.impl == "ours":
        from paper_2605_05467_b200 import _native
        _native.set_copy_engine(args.engine)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = build_workload(args.config, args.seqs) if world == 1 else distributed_workload(world, args.seqs)

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_cpu_reference(w, args.steps, args.warmup, args.cpu_sample_seqs)
        line = {
            "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": w.name, "cpu_sample": r["sample"],
                       "same_config": r["same_config"]},
            "cpu_baseline": {"value": r["value"], "unit": "GB/s", "cores": r["threads"],
                             "kind": "port", "sample": r["sample"], "cpu": cpu_model(),
                             "planner": r["planner"], "planner_ms": r["planner_ms"]},
            "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    import torch

    if world > 1:
        run_distributed(args, w, rank, world, local)
        return
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    m = measure_single(args, w, device, with_cpu=not args.no_cpu, e2e_on=not args.no_e2e)
    copy_peak = copy_peak_in_run(device)
    m["roofline"]["copy_peak_in_run"] = copy_peak
    m["roofline"]["frac_vs_copy_in_run"] = m["roofline"]["achieved"] / copy_peak
    headline = None
    if not args.no_headline and args.config != 4 and args.seqs is None:
        # the north star's headline in the same run: Llama-3.1-8B at 32k context
        wh = build_workload(4, None)
        h = measure_single(args, wh, device, with_cpu=not args.no_cpu, e2e_on=True)
        headline = {
            "workload": wh.name, "ms_per_switch": h["ms"] / args.steps,
            "e2e_ms_per_switch": h["e2e"]["ms_per_step"], "gbs": h["value"],
            "e2e_gbs": h["e2e"]["value"], "kv_bytes_per_step": h["kv_per_step"],
            "weight_bytes_per_step": h["w_per_step"], "k1_ms": h["roofline"]["k1_ms"],
            "k1_frac": h["roofline"]["frac"], "step_frac": h["roofline"]["step_frac"],
            "bit_exact_property": h["bit_exact_property"],
            "cpu_ms_per_switch": h["cpu_baseline"]["ms_per_step"] if h["cpu_baseline"] else None,
            "cpu_gbs": h["cpu_baseline"]["value"] if h["cpu_baseline"] else None,
            "cpu_same_config": h["cpu_baseline"]["same_config"] if h["cpu_baseline"] else None,
            "cpu_planner_ms": h["cpu_baseline"]["planner_ms"] if h["cpu_baseline"] else None,
            "cpu_cores": h["cpu_baseline"]["cores"] if h["cpu_baseline"] else None,
        }
    line = {
        "metric": METRIC, "value": m["value"], "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {
            "workload": w.name, "model": w.model.name, "logical_gpus_per_device": len(w.gpus),
            "seqs": len(w.requests), "ctx": w.requests[0][1],
            "switch": "alternating forward/reverse, full stop-and-migrate (plan+K3+K1+K2)",
            "k1_k2_overlap": m["overlap"], "copy_engine": _engine_name(),
            "weights_mode": args.weights_mode, "pool_layout": args.pool_layout,
            "kv_bytes_per_step": m["kv_per_step"], "weight_bytes_per_step": m["w_per_step"],
            "weight_relayout_bytes_per_step": m["w_local_per_step"],
            "weights_note": weights_note(w, m["w_bytes"]),
            "l2": "inputs larger than L2 (>= 24 GiB moved per step)",
            "parallelism": "1 GPU, logical ranks",
        },
        "roofline": m["roofline"], "cpu_baseline": m["cpu_baseline"], "clocks": m["clocks"],
        "e2e": m["e2e"], "gpu_launches": m["gpu_launches"], "status": m["status"],
        "bit_exact_property": m["bit_exact_property"], "pages_verified": m["pages_verified"],
        "headline": headline,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
