"""Migration-minimising rank order on all 12 TP transitions.

For 64 sequences x 4096 tokens of Llama-3.1-8B on 8 GPU slots (requests
round-robin over the old groups, tests/test_migration.py:131-135), every new
group's rank order is either the canonical one (the reference's plan) or
``placement.reuse_rank_order`` (the linear assignment that keeps the most
resident KV in place). Reports the KV fraction each plan moves and, with
--measure on a GPU, the measured switch time of both plans (bit-exactness
property checked after each).

    python tools/reuse_order.py [--measure] [--out profiles/r01_reuse_order.jsonl]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def reuse_layouts(old, new, kvb):
    from paper_2605_05467_b200 import migration as M, placement
    out = []
    for lay in new:
        rid = {r for r, _ in lay.requests}
        sub = [M.KvLayout(o.group, o.tp, o.total_heads,
                          tuple((r, c) for r, c in o.requests if r in rid)) for o in old]
        order = placement.reuse_rank_order(sub, lay.group, kvb)
        out.append(M.KvLayout(tuple(order), lay.tp, lay.total_heads, lay.requests))
    return out


def main():
    from paper_2605_05467_b200 import migration as M, workloads
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B

    ap = argparse.ArgumentParser()
    ap.add_argument("--measure", action="store_true")
    ap.add_argument("--seqs", type=int, default=64)
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    kv = LLAMA_3_1_8B.kv
    kvb = kv.kv_bytes_per_token_per_head
    gpus = tuple(range(8))
    reqs = [(i, 4096) for i in range(args.seqs)]
    total = sum(c for _, c in reqs) * kv.total_heads * kvb
    out = open(args.out, "w") if args.out else None
    for a in (1, 2, 4, 8):
        for b in (1, 2, 4, 8):
            if a == b:
                continue
            la = workloads.round_robin(workloads.tp_groups(gpus, a), reqs, kv.total_heads)
            lb = workloads.round_robin(workloads.tp_groups(gpus, b), reqs, kv.total_heads)
            lr = reuse_layouts(la, lb, kvb)
            row = {"tp_old": a, "tp_new": b, "seqs": args.seqs,
                   "moved_canonical": M.plan_repartition(la, lb, kvb).total_bytes / total,
                   "moved_reuse_order": M.plan_repartition(la, lr, kvb).total_bytes / total}
            if args.measure:
                row.update(measure(la, lb, lr, kv, gpus))
            print(json.dumps(row), flush=True)
            if out:
                out.write(json.dumps(row) + "\n")
    if out:
        out.close()


def measure(la, lb, lr, kv, gpus) -> dict:
    import torch

    from paper_2605_05467_b200.kvcache import PagedKvCluster

    res = {}
    for tag, new in (("canonical", lb), ("reuse_order", lr)):
        n = sum(len(x.requests) for x in la)
        units = 2 * n * kv.blocks(4096) * kv.total_heads // len(gpus) + 256
        c = PagedKvCluster(kv, gpus, units_per_gpu=units, max_requests=n,
                           max_blocks=kv.blocks(4096), fragmented=True, seed=0)
        c.fill_garbage(seed=1)
        c.admit(la, seed=7)
        st = torch.cuda.current_stream()
        times = []
        for r in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a, b = (la, new) if r % 2 == 0 else (new, la)
            e0.record(st)
            c.switch_layouts(a, b, stream=st, validate=False)
            e1.record(st)
            e1.synchronize()
            if r >= 2 and r % 2 == 0:
                times.append(e0.elapsed_time(e1))
        v = c.verify(seed=7)
        res[f"{tag}_ms"] = float(np.median(times))
        res[f"{tag}_bit_exact_property"] = v["placement_errors"] == 0 and v["word_mismatches"] == 0
        del c
        torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    main()
