"""Host-side cost of one small TP switch (cfg1 shape), profiled.

    python tools/host_overhead.py [--n 300]
"""

from __future__ import annotations

import argparse
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2605_05467_b200 import workloads
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--config", type=int, default=0)
    args = ap.parse_args()
    import bench

    w = workloads.config(args.config, weights=False) if args.config else workloads.config(0)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=bench.capacity_units(w, kv),
                       max_requests=len(w.requests),
                       max_blocks=kv.blocks(max(x for _, x in w.requests)))
    c.admit(w.old)
    ex = ReconfigurationExecutor(c)
    for _ in range(10):
        ex.switch(w.old, w.new, validate=False)
        ex.switch(w.new, w.old, validate=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.n):
        a, b = (w.old, w.new) if i % 2 == 0 else (w.new, w.old)
        ex.switch(a, b, validate=False, sync=False)
    enq = (time.perf_counter() - t0) / args.n * 1e6
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.n):
        a, b = (w.old, w.new) if i % 2 == 0 else (w.new, w.old)
        r = ex.switch(a, b, validate=False, sync=True)
    e2e = (time.perf_counter() - t0) / args.n * 1e6
    print(f"enqueue-only {enq:.1f} us/switch; synchronous e2e {e2e:.1f} us/switch; "
          f"device {r.device_ms * 1e3:.1f} us")
    pr = cProfile.Profile()
    pr.enable()
    for i in range(args.n):
        a, b = (w.old, w.new) if i % 2 == 0 else (w.new, w.old)
        ex.switch(a, b, validate=False, sync=False)
    pr.disable()
    torch.cuda.synchronize()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(s.getvalue())


if __name__ == "__main__":
    main()
