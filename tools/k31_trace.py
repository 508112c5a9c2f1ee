"""Where the time of a small switch goes inside K31 (knob "k31_trace"): every
CTA stamps %globaltimer at its entry, after its page decisions (the copies
start), after its copies (warp 0) and after its bookkeeping (warp 1). Prints, per phase, the
min / median / max over CTAs relative to the first CTA's entry (ns), plus the
spread of CTA entry times (launch ramp).

    python tools/k31_trace.py [--case 1seq|cfg1|1seq4096] [--engine bulk]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

# stamps of the item-share schedule and of the dynamic one (TPR_K31: 1 = by
# plan size, dynamic from 512 pages; 2 = dynamic; 3 = item shares)
NAMES_ITEM = ("entry", "decide", "copies", "books")
NAMES_DYN = ("entry", "decide", "barrier", "copies")

CASES = {"1seq": (8, 1, 2, 1, 463), "cfg1": (2, 1, 2, 4, 512), "1seq4096": (8, 8, 1, 1, 4096)}


def main():
    import torch

    from paper_2605_05467_b200 import _native, workloads
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="1seq", choices=sorted(CASES))
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    slots, a, b, n, ctx = CASES[args.case]
    kv = LLAMA_3_1_8B.kv
    gpus = tuple(range(slots))
    reqs = [(i, ctx) for i in range(n)]
    la = workloads.round_robin(workloads.tp_groups(gpus, a), reqs, kv.total_heads)
    lb = workloads.round_robin(workloads.tp_groups(gpus, b), reqs, kv.total_heads)
    units = 2 * n * kv.total_heads * kv.blocks(ctx) + 64
    cl = PagedKvCluster(kv, gpus, units_per_gpu=units, max_requests=n, max_blocks=kv.blocks(ctx),
                        fragmented=True, seed=0)
    cl.admit(la, seed=5)
    ex = ReconfigurationExecutor(cl)
    buf = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
    _native.set_tuning("k31_trace", buf.data_ptr())
    knob = os.environ.get("TPR_K31", "1") or "1"
    rows = []
    dyn = False
    try:
        for i in range(args.reps):
            buf.zero_()
            torch.cuda._sleep(200_000)  # the launch waits on the stream, not the host
            r = ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False)
            dyn = knob == "2" or (knob == "1" and r.kv.units >= 512)
            t = buf.view(-1, 8).cpu().numpy()
            grid = int(t[0, 7])
            if grid <= 0:
                raise SystemExit("no K31 launch (plan outside the fused path?)")
            t = t[:grid]
            base = t[:, 0].min()
            rows.append({k: (t[:, j] - base) for j, k in enumerate(NAMES_DYN if dyn else NAMES_ITEM)})
    finally:
        _native.set_tuning("k31_trace", 0)
    last = rows[len(rows) // 2:]
    NAMES = NAMES_DYN if dyn else NAMES_ITEM
    out = {"case": args.case, "variant": "dynamic" if dyn else "item-share", "grid": grid}
    if not dyn:
        out["items_per_cta"] = [int(x) for x in np.unique(t[:, 6])]
    for k in NAMES:
        v = np.concatenate([r[k] for r in last])
        out[k] = {"min": int(v.min()), "median": int(np.median(v)), "max": int(v.max())}
    out["copy_phase_median_ns"] = int(np.median(np.concatenate(
        [r["copies"] - r["barrier" if dyn else "decide"] for r in last])))
    out["kernel_span_median_ns"] = int(np.median([max(r[k].max() for k in NAMES[1:])
                                                   for r in last]))
    print(json.dumps(out))
    if args.out:
        with open(args.out, "a") as f:
            f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
