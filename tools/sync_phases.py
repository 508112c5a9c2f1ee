"""Where the host time of a synchronous one-sequence switch goes: the steps
of ``ReconfigurationExecutor.switch(sync=True)`` replayed with a timestamp
after each (median of --n, microseconds), plus the same switch waited for by
polling the end event instead of ``synchronize``.

    python tools/sync_phases.py [--n 2000]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2605_05467_b200 import workloads
    from paper_2605_05467_b200.controller import ReconfigurationExecutor, SwitchResult
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    kv = LLAMA_3_1_8B.kv
    gpus, ctx = tuple(range(8)), 463
    reqs = [(0, ctx)]
    la = workloads.round_robin(workloads.tp_groups(gpus, 1), reqs, kv.total_heads)
    lb = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, kv.total_heads)
    cl = PagedKvCluster(kv, gpus, units_per_gpu=2 * kv.total_heads * kv.blocks(ctx) + 64,
                        max_requests=1, max_blocks=kv.blocks(ctx), fragmented=True, seed=0)
    cl.admit(la, seed=5)
    ex = ReconfigurationExecutor(cl)
    main_st = ex.main_stream
    for i in range(200):
        ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False)
    names = ("start_event", "switch_layouts", "result", "end_event", "synchronize", "status",
             "elapsed_time")
    t = {k: [] for k in names}
    total, poll_total = [], []
    e0, e1 = ex._ev_sync
    for i in range(args.n):
        a, b = (la, lb) if i % 2 == 0 else (lb, la)
        ts = [time.perf_counter()]
        e0.record(main_st)
        ts.append(time.perf_counter())
        plan, st = cl.switch_layouts(a, b, stream=main_st, validate=False)
        ts.append(time.perf_counter())
        res = SwitchResult(plan=plan, kv=st, weights=None, events={"start": e0, "end": e1},
                           new_layouts=list(b), evicted=[])
        ts.append(time.perf_counter())
        e1.record(main_st)
        ts.append(time.perf_counter())
        e1.synchronize()
        ts.append(time.perf_counter())
        res.status = int(ex._kv_status_np[0])
        ts.append(time.perf_counter())
        res.device_ms = e0.elapsed_time(e1)
        ts.append(time.perf_counter())
        for k, x, y in zip(names, ts, ts[1:]):
            t[k].append((y - x) * 1e6)
        total.append((ts[-1] - ts[0]) * 1e6)
    for i in range(args.n):  # the public call, waited for by polling the end event
        a, b = (la, lb) if i % 2 == 0 else (lb, la)
        t0 = time.perf_counter()
        r = ex.switch(a, b, validate=False, sync=False)
        e1.record(main_st)
        while not e1.query():
            pass
        poll_total.append((time.perf_counter() - t0) * 1e6)
        assert r.kv.units > 0
    out = {k: float(np.median(v)) for k, v in t.items()}
    out["total"] = float(np.median(total))
    out["public_sync_poll_total"] = float(np.median(poll_total))
    print(json.dumps(out))
    if args.out:
        Path(args.out).write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
