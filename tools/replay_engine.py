"""Replay the reference controller's reconfiguration decisions on a B200.

tests/golden/engine_trace.json.gz holds every KV-migration plan the
reference simulator's hook made on its demo experiment (captured by
tests/golden/gen_engine_trace.py). Each plan is one destination group's
``head_transfers`` calls (engine.py:571-589) and its modeled
``switch_cost(WARM)`` (engine.py:590-597). Here every plan runs for real:

1. its requests are admitted on their source groups with their context at
   that moment (untimed);
2. the plan executes through PagedKvCluster.migrate (K3 + K1, timed with CUDA
   events and host wall clock);
3. the result is verified at full size, and the requests are released.

Geometry: the reference profile (32 KV heads, 4096 B/token/head) as 8 layers x
128 dim x bf16, 8 GPU slots in one B200.

    python tools/replay_engine.py --out profiles/r01_engine_replay.jsonl
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
TRACE = ROOT / "tests" / "golden" / "engine_trace.json.gz"


def load_trace() -> dict:
    with gzip.open(TRACE, "rt") as f:
        return json.load(f)


def plan_for(event, kvb, H):
    """The destination group's plan, built like engine.py:571-590."""
    from paper_2605_05467_b200 import migration as M
    arrs = []
    for og, ng, rid, ctx in event["calls"]:
        old = M.KvLayout(tuple(og), len(og), H, ((rid, ctx),))
        new = M.KvLayout(tuple(ng), len(ng), H, ((rid, ctx),))
        arrs.append(M.head_transfers_array(old, new, kvb).as_array())
    return M.MigrationPlan.from_array(np.concatenate(arrs) if arrs else np.zeros((0, 6), np.int64))


def replay(events, kv, gpus, verify=True, reps=3):
    import torch

    from paper_2605_05467_b200 import migration as M
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    H = kv.total_heads
    need = max(sum(H * kv.blocks(c[3]) for c in e["calls"]) for e in events)
    c = PagedKvCluster(kv, gpus, units_per_gpu=need + 64, max_requests=64,
                       max_blocks=max(kv.blocks(x[3]) for e in events for x in e["calls"]),
                       fragmented=True, seed=3)
    st = torch.cuda.current_stream()
    rows = []
    for i, e in enumerate(events):
        plan = plan_for(e, kv.kv_bytes_per_token_per_head, H)
        back = M.MigrationPlan.from_array(
            plan.as_array()[:, [1, 0, 2, 3, 4, 5]])  # the same moves in reverse
        srcs = [M.KvLayout(tuple(og), len(og), H, ((rid, ctx),)) for og, _, rid, ctx in e["calls"]]
        c.admit(srcs, seed=11)
        dev, host = [], []
        for r in range(2 * reps):  # forward, back, forward, ...: every repetition is real
            p = plan if r % 2 == 0 else back
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record(st)
            c.migrate(p, validate=(r == 0))
            e1.record(st)
            e1.synchronize()
            host.append((time.perf_counter() - t0) * 1e3)
            if r % 2 == 0:
                dev.append(e0.elapsed_time(e1))
        c.migrate(plan, validate=False)
        ok = True
        if verify:
            v = c.verify(seed=11)
            ok = v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
            want = M.layout_placement([M.KvLayout(tuple(ng), len(ng), H, ((rid, ctx),))
                                       for _, ng, rid, ctx in e["calls"]])
            ok = ok and c.placement() == want
        c.release([rid for _, _, rid, _ in e["calls"]])
        rows.append({"event": i, "t_sim_s": e["t"], "calls": len(e["calls"]),
                     "transfers": plan.n_transfers, "bytes": plan.total_bytes,
                     "reference_plan_bytes": e["total_bytes"],
                     "reference_plan_transfers": e["transfers"],
                     "modeled_switch_cost_ms": e["modeled_switch_cost_ms"],
                     "measured_device_ms": float(np.median(dev)),
                     "measured_host_ms": float(np.median(host[0::2])),
                     "bit_exact_property": ok})
    return rows


def main():
    from paper_2605_05467_b200.geometry import KvGeometry

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "engine_replay.jsonl"))
    args = ap.parse_args()
    doc = load_trace()
    prof = doc["profile"]
    kvb, H = prof["kv_bytes_per_token_per_head"], prof["total_kv_heads"]
    kv = KvGeometry(layers=kvb // (2 * 128 * 2), head_dim=128, total_heads=H)
    assert kv.kv_bytes_per_token_per_head == kvb
    rows = replay(doc["events"], kv, tuple(range(prof["pool_size"])))
    with open(args.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
            print(json.dumps(r))
    tot_m = sum(r["modeled_switch_cost_ms"] for r in rows)
    tot_d = sum(r["measured_device_ms"] for r in rows)
    print(json.dumps({"plans": len(rows), "modeled_ms_total": tot_m, "measured_ms_total": tot_d,
                      "all_bit_exact": all(r["bit_exact_property"] for r in rows)}))


if __name__ == "__main__":
    main()
