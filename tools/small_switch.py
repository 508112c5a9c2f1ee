"""Fixed cost of small TP switches (the latency-bound end of BASELINE config 5).

For a few small plans (Llama-3.1-8B KV, 8 GPU slots in one HBM) this reports
per switch, median over --reps:

* ``sync_us``: the public call ``ReconfigurationExecutor.switch(sync=True)``,
  host wall time (plan + enqueue + device + status read back);
* ``enqueue_us``: host time to plan and enqueue (``sync=False``);
* ``device_us``: device span of the enqueued work alone (the stream is held
  by a spin kernel while the host enqueues, so host stalls are excluded);
* ``k1_roof_us``: 2 x bytes / measured copy peak.

Run it with TPR_K31=0 and/or TPR_K3_FUSE_UNITS=0 to compare the launch
variants (one JSON line per case, tagged with the environment).

    python tools/small_switch.py --out profiles/small_switch.jsonl
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

CASES = (  # (name, slots, tp_old, tp_new, seqs, ctx)
    ("cfg1 4x512 TP1->TP2", 2, 1, 2, 4, 512),
    ("1 seq x 463 TP1->TP2", 8, 1, 2, 1, 463),
    ("1 seq x 4096 TP8->TP1", 8, 8, 1, 1, 4096),
    ("1 seq x 4096 TP1->TP2", 8, 1, 2, 1, 4096),
    ("4 seqs x 4096 TP1->TP2", 8, 1, 2, 4, 4096),
    ("8 seqs x 4096 TP2->TP4", 8, 2, 4, 8, 4096),
    ("16 seqs x 4096 TP4->TP8", 8, 4, 8, 16, 4096),
    ("64 seqs x 4096 TP4->TP8", 8, 4, 8, 64, 4096),
)


def main():
    import torch

    from paper_2605_05467_b200 import _native, migration as M, workloads
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--cases", type=int, default=len(CASES), help="run the first N switch cases")
    ap.add_argument("--no-handoff", action="store_true")
    args = ap.parse_args()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    env = {k: os.environ.get(k, "") for k in ("TPR_K3_FUSE_UNITS", "TPR_K31", "TPR_BULK_K31",
                                              "TPR_TENSOR_PARTIAL")}
    kv = LLAMA_3_1_8B.kv
    out = open(args.out, "a") if args.out else None
    torch.cuda.set_device(0)
    main_stream = torch.cuda.current_stream()
    for name, slots, a, b, n, ctx in CASES[:args.cases]:
        gpus = tuple(range(slots))
        reqs = [(i, ctx) for i in range(n)]
        la = workloads.round_robin(workloads.tp_groups(gpus, a), reqs, kv.total_heads)
        lb = workloads.round_robin(workloads.tp_groups(gpus, b), reqs, kv.total_heads)
        def need(tp):  # pool units one slot holds in a TP-tp layout (round robin)
            return -(-n * tp // slots) * (kv.total_heads // tp) * kv.blocks(ctx)
        units = need(a) + need(b) + 64  # old and new pages coexist during a switch
        cl = PagedKvCluster(kv, gpus, units_per_gpu=units, max_requests=n,
                            max_blocks=kv.blocks(ctx), fragmented=True, seed=0)
        cl.admit(la, seed=5)
        ex = ReconfigurationExecutor(cl)
        for i in range(20):
            ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False)
        torch.cuda.synchronize()
        sync_us, enq_us, dev_us = [], [], []
        nbytes = 0
        for i in range(args.reps):
            r = ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False)
            sync_us.append(r.host_ms * 1e3)
            nbytes = max(nbytes, r.kv.bytes)
        torch.cuda.synchronize()
        for i in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200_000)  # hold the stream while the host enqueues
            e0.record(main_stream)
            t0 = time.perf_counter()
            ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False, sync=False)
            enq_us.append((time.perf_counter() - t0) * 1e6)
            e1.record(main_stream)
            e1.synchronize()
            dev_us.append(e0.elapsed_time(e1) * 1e3)
        v = cl.verify(seed=5)
        ok = v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
        roof = 2 * nbytes / (peak * 1e9) * 1e6
        row = {"case": name, "env": env, "bytes": nbytes,
               "launches": _native.kv_switch_launches(r.kv.units, r.kv.transfers), "units": r.kv.units,
               "sync_us": float(np.median(sync_us)), "enqueue_us": float(np.median(enq_us)),
               "device_us": float(np.median(dev_us)), "k1_roof_us": roof,
               "sync_hbm_frac": roof / float(np.median(sync_us)),
               "device_hbm_frac": roof / float(np.median(dev_us)), "bit_exact_property": ok}
        print(json.dumps(row), flush=True)
        if out:
            out.write(json.dumps(row) + "\n")
        del ex, cl
        torch.cuda.empty_cache()
    # prefill -> decode handoffs (disjoint groups, head_transfers): the most
    # frequent small transfer of a disaggregated deployment
    handoffs = (("handoff 1 seq x 463 TP2(0,1)->TP4(2..5)", (0, 1), (2, 3, 4, 5), 463),
                ("handoff 1 seq x 4096 TP1(0)->TP1(1)", (0,), (1,), 4096))
    for name, src, dst, ctx in () if args.no_handoff else handoffs:
        gpus = tuple(range(6))
        pre = M.KvLayout(src, len(src), kv.total_heads, ((0, ctx),))
        dec = M.KvLayout(dst, len(dst), kv.total_heads, ((0, ctx),))
        cl = PagedKvCluster(kv, gpus, units_per_gpu=2 * kv.total_heads * kv.blocks(ctx) + 64,
                            max_requests=1, max_blocks=kv.blocks(ctx), fragmented=True, seed=0)
        cl.admit([pre], seed=5)
        ex = ReconfigurationExecutor(cl)
        sync_us, nbytes = [], 0
        for i in range(args.reps + 20):
            r = ex.handoff(*((pre, dec) if i % 2 == 0 else (dec, pre)))
            if i >= 20:
                sync_us.append(r.host_ms * 1e3)
            nbytes = r.kv.bytes
        v = cl.verify(seed=5)
        roof = 2 * nbytes / (peak * 1e9) * 1e6
        row = {"case": name, "env": env, "bytes": nbytes, "sync_us": float(np.median(sync_us)),
               "k1_roof_us": roof, "sync_hbm_frac": roof / float(np.median(sync_us)),
               "bit_exact_property": v["placement_errors"] == 0 and v["word_mismatches"] == 0}
        print(json.dumps(row), flush=True)
        if out:
            out.write(json.dumps(row) + "\n")
        del ex, cl
        torch.cuda.empty_cache()
    if out:
        out.close()


if __name__ == "__main__":
    main()
