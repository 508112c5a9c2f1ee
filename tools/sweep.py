"""BASELINE config 5: trace-driven switch sweep.

All 12 ordered TP transitions among {1,2,4,8} on 8 GPU slots, 1..128 sequences,
with contexts fixed at 4096 tokens or taken from the reference's bursty trace
(scenarios.py:58-85, seed 11; committed as tests/golden: context = prompt +
output/2, i.e. mid-decode). Llama-3.1-8B KV geometry.

On one B200 the 8 slots are logical (all pools in one HBM). So each switch is
bounded by HBM: t_roof = 2 * bytes / measured copy peak. Every point reports:

* the measured switch latency (device events and host wall, synchronous), the
  device work alone (stream held while the host enqueues), and the public
  synchronous call ``ReconfigurationExecutor.switch`` end to end;
* GB/s and the fraction of that roofline;
* the reference cost model's prediction for the same plan (default
  CostModelParams, migration.py:77-98);
* the CPU restatement's time for the small points.

    python tools/sweep.py --out profiles/r01_sweep.jsonl
"""

from __future__ import annotations

import argparse
import gzip
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2605_05467_b200 import migration as M, workloads
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "sweep.jsonl"))
    ap.add_argument("--max-seqs", type=int, default=128,
                    help="largest sequence count with fixed 4096-token contexts")
    ap.add_argument("--trace-max-seqs", type=int, default=256,
                    help="largest sequence count with bursty-trace contexts")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--cpu-max-seqs", type=int, default=8)
    ap.add_argument("--modes", default="fixed4096,trace")
    ap.add_argument("--only", default="", help="comma list of tp_old:tp_new:seqs points")
    ap.add_argument("--k1-reps", type=int, default=2,
                    help="extra switches timed with events around K1 alone (k1_ms)")
    args = ap.parse_args()

    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    kv = LLAMA_3_1_8B.kv
    gpus = tuple(range(8))
    trace = json.load(gzip.open(ROOT / "tests" / "golden" / "reference_golden.json.gz", "rt"))["bursty_trace"]
    trace_ctx = [p + o // 2 for p, o in trace]
    params = M.CostModelParams()
    only = {tuple(int(v) for v in x.split(":")) for x in args.only.split(",") if x}
    out = open(args.out, "w")
    stream = torch.cuda.current_stream()

    def slot_units(layouts):
        """Pool units each slot holds for ``layouts`` (one page per head-block)."""
        need = [0] * len(gpus)
        for lay in layouts:
            for _, c in lay.requests:
                for g in lay.owners():
                    need[g] += kv.blocks(c)
        return need

    def points(mode):
        top = args.max_seqs if mode == "fixed4096" else args.trace_max_seqs
        for a in (1, 2, 4, 8):
            for b in (1, 2, 4, 8):
                if a == b:
                    continue
                for n in (1, 2, 4, 8, 16, 32, 64, 128, 256):
                    if n > top or (only and (a, b, n) not in only):
                        continue
                    ctxs = [4096] * n if mode == "fixed4096" else trace_ctx[:n]
                    reqs = [(i, c) for i, c in enumerate(ctxs)]
                    la = workloads.round_robin(workloads.tp_groups(gpus, a), reqs, 8)
                    lb = workloads.round_robin(workloads.tp_groups(gpus, b), reqs, 8)
                    yield a, b, n, ctxs, reqs, la, lb

    for mode in args.modes.split(","):
        # one cluster per mode, sized for its largest point: old and new pages
        # coexist while a switch runs (sources are released after the copy)
        units, max_ctx, max_n = 0, 0, 0
        for a, b, n, ctxs, reqs, la, lb in points(mode):
            units = max(units, max(x + y for x, y in zip(slot_units(la), slot_units(lb))))
            max_ctx, max_n = max(max_ctx, max(ctxs)), max(max_n, n)
        cluster = PagedKvCluster(kv, gpus, units_per_gpu=units + 256, max_requests=max_n,
                                 max_blocks=kv.blocks(max_ctx), fragmented=True, seed=0)
        ex = ReconfigurationExecutor(cluster)
        # touch every pool page once: first writes to fresh cudaMalloc memory
        # are slower, and which points would pay for them depends on the order
        cluster.fill_garbage(seed=1)
        for a, b, n, ctxs, reqs, la, lb in points(mode):
            cluster.admit(la, seed=n)
            fwd = M.plan_repartition(la, lb, kv.kv_bytes_per_token_per_head)
            back = M.plan_repartition(lb, la, kv.kv_bytes_per_token_per_head)
            for x, y in ((la, lb), (lb, la)):  # warm-up, leaves the cluster in layout A
                cluster.switch_layouts(x, y, stream=stream, validate=False)
            torch.cuda.synchronize()
            dev_ms, host_ms, exec_ms, plan_ms = [], [], [], []
            # short switches are host/latency-bound and jittery: more repetitions
            reps = args.reps if fwd.total_bytes >= (256 << 20) else max(args.reps, 24)
            for r in range(reps):
                a_b = (la, lb) if r % 2 == 0 else (lb, la)
                t0 = time.perf_counter()  # the planner alone (host), for the split
                M.plan_repartition(*a_b, kv.kv_bytes_per_token_per_head)
                plan_ms.append((time.perf_counter() - t0) * 1e3)
                # the switch as the executor runs it: one native call (plan,
                # records, K3, K1); e0 -> e1 includes the host's planning
                # time, during which the GPU idles
                e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                t0 = time.perf_counter()
                e0.record(stream)
                cluster.switch_layouts(*a_b, stream=stream, validate=False)
                e1.record(stream)
                e1.synchronize()
                host_ms.append((time.perf_counter() - t0) * 1e3)
                dev_ms.append(e0.elapsed_time(e1))
            for r in range(reps, 2 * reps):  # device work alone: stream held
                a_b = (la, lb) if r % 2 == 0 else (lb, la)  # while the host enqueues
                e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                torch.cuda._sleep(400_000)
                e0.record(stream)
                cluster.switch_layouts(*a_b, stream=stream, validate=False)
                e1.record(stream)
                e1.synchronize()
                exec_ms.append(e0.elapsed_time(e1))
            e2e_ms = []  # the public synchronous call (ReconfigurationExecutor.switch)
            for r in range(2 * reps):  # fwd/back pairs: ends in layout A
                res = ex.switch(*((la, lb) if r % 2 == 0 else (lb, la)), validate=False)
                if r % 2 == 0:
                    e2e_ms.append(res.host_ms)
            k1_ms = []
            for r in range(2 * args.k1_reps):  # fwd/back pairs: ends in layout A
                k0, k1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                cluster.migrate(fwd if r % 2 == 0 else back, validate=False,
                                k1_events=(k0, k1))
                k1.synchronize()
                if r % 2 == 0:
                    k1_ms.append(k0.elapsed_time(k1))
            v = cluster.verify(seed=n)
            ok = v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
            cluster.release([r for r, _ in reqs])
            nbytes = fwd.total_bytes
            d = float(np.median(dev_ms))
            x = float(np.median(exec_ms))
            cpu_ms = cpu_point(la, lb, reqs, gpus, kv) if n <= args.cpu_max_seqs else None
            row = {
                "mode": mode, "tp_old": a, "tp_new": b, "seqs": n,
                "ctx_total": int(sum(ctxs)), "transfers": fwd.n_transfers, "bytes": nbytes,
                "device_ms": d, "host_ms": float(np.median(host_ms)),
                "gbs": nbytes / (d * 1e-3) / 1e9 if d > 0 else None,
                "hbm_frac": (2 * nbytes / (peak * 1e9)) / (d * 1e-3) if d > 0 else None,
                # the planner alone on the host; the switch's device work alone
                "plan_host_ms": float(np.median(plan_ms)), "exec_device_ms": x,
                "exec_hbm_frac": (2 * nbytes / (peak * 1e9)) / (x * 1e-3) if x > 0 else None,
                # end to end through the public synchronous call (host wall time)
                "e2e_ms": float(np.median(e2e_ms)),
                "e2e_hbm_frac": (2 * nbytes / (peak * 1e9)) / (float(np.median(e2e_ms)) * 1e-3),
                "k1_ms": float(np.median(k1_ms)) if k1_ms else None,
                "k1_hbm_frac": (2 * nbytes / (peak * 1e9)) / (float(np.median(k1_ms)) * 1e-3)
                if k1_ms else None,
                "predicted_ms_ref_model": M.switch_cost(M.WARM, fwd, params),
                "cpu_restatement_ms": cpu_ms, "bit_exact_property": ok,
            }
            out.write(json.dumps(row) + "\n")
            out.flush()
            print(json.dumps(row))
        del cluster
        torch.cuda.empty_cache()
    out.close()


def cpu_point(la, lb, reqs, gpus, kv):
    """Time the CPU restatement (planner + threaded page copies) on host pools."""
    import os
    from oracle import kvmove, plan_oracle as PO
    H = kv.total_heads
    old = [(l.group, H, list(l.requests)) for l in la]
    new = [(l.group, H, list(l.requests)) for l in lb]
    rslot = {r: i for i, (r, _) in enumerate(reqs)}
    ctx = dict(reqs)
    mb = max(kv.blocks(c) for _, c in reqs)
    units = 2 * sum(kv.blocks(c) for _, c in reqs) + 16
    geo = dict(layers=kv.layers, head_dim=kv.head_dim, dtype_bytes=kv.dtype_bytes,
               block_tokens=kv.block_tokens, total_heads=H, max_blocks=mb, n_req_slots=len(reqs),
               n_units=units)
    pools = [np.ones(units * kv.unit_bytes, np.uint8) for _ in gpus]
    tables = [np.full(len(reqs) * H * mb, -1, np.int32) for _ in gpus]
    rings = [np.arange(units, dtype=np.int32) for _ in gpus]
    heads, tails = [0] * len(gpus), [units] * len(gpus)
    adm = [(-1, g, rslot[r], i * (H // len(grp)), (i + 1) * (H // len(grp)), c)
           for grp, _, rr in old for r, c in rr for i, g in enumerate(grp)]
    _, _, heads, tails = kvmove.kv_migrate(geo, pools, tables, rings, heads, tails,
                                           np.array(adm, np.int64))
    threads = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    moves = PO.plan(old, new, kv.kv_bytes_per_token_per_head)
    rec = np.array([(s, d, rslot[r], lo, hi, ctx[r]) for s, d, r, lo, hi, _ in moves],
                   np.int64).reshape(-1, 6)
    kvmove.kv_migrate(geo, pools, tables, rings, heads, tails, rec, threads)
    return (time.perf_counter() - t0) * 1e3


if __name__ == "__main__":
    main()
