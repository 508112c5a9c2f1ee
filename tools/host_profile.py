"""cProfile of the public small-switch call (ReconfigurationExecutor.switch,
1 seq x 463 tokens TP1->TP2, enqueue only): where the host microseconds go.

    python tools/host_profile.py [--n 3000]
"""

from __future__ import annotations

import argparse
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2605_05467_b200 import workloads
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3000)
    args = ap.parse_args()
    kv = LLAMA_3_1_8B.kv
    gpus, ctx = (0, 1), 463
    reqs = [(0, ctx)]
    la = workloads.round_robin(workloads.tp_groups(gpus, 1), reqs, kv.total_heads)
    lb = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, kv.total_heads)
    cl = PagedKvCluster(kv, gpus, units_per_gpu=2 * kv.total_heads * kv.blocks(ctx) + 64,
                        max_requests=1, max_blocks=kv.blocks(ctx), fragmented=True, seed=0)
    cl.admit(la, seed=5)
    ex = ReconfigurationExecutor(cl)

    def run(n, sync):
        for i in range(n):
            ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False, sync=sync)
            if not sync and i % 16 == 15:
                torch.cuda.synchronize()
        torch.cuda.synchronize()

    run(200, False)
    for sync in (False, True):
        t = []
        for i in range(args.n):
            t0 = time.perf_counter()
            ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False, sync=sync)
            t.append(time.perf_counter() - t0)
            if not sync and i % 16 == 15:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        print(f"switch(sync={sync}) median {np.median(t) * 1e6:.1f} us", flush=True)
    # the native call alone, and its host half (plan + records, no launch)
    from paper_2605_05467_b200 import _native
    lib = _native.load()
    real = lib.tpr_kv_switch_layouts
    prep = lib.tpr_switch_prepare
    t_nat, t_prep = [], []

    class Timed:
        def __call__(self, geo, cl_, addr, n, t, stream):
            t0 = time.perf_counter()
            prep(geo, cl_, addr, n, t)
            t1 = time.perf_counter()
            rc = real(geo, cl_, addr, n, t, stream)
            t_nat.append(time.perf_counter() - t1)
            t_prep.append(t1 - t0)
            return rc

    lib.tpr_kv_switch_layouts = Timed()
    try:
        t = []
        for i in range(args.n):
            t0 = time.perf_counter()
            ex.switch(*((la, lb) if i % 2 == 0 else (lb, la)), validate=False, sync=False)
            t.append(time.perf_counter() - t0)
            if i % 16 == 15:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
    finally:
        lib.tpr_kv_switch_layouts = real
    nat, pre, tot = (np.median(x) * 1e6 for x in (t_nat, t_prep, t))
    print(f"split: native call {nat:.1f} us (of which plan+records {pre:.1f}, launch path "
          f"{nat - pre:.1f}); Python around it {tot - nat - pre:.1f} us", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    run(args.n, False)
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(30)
    print(s.getvalue())


if __name__ == "__main__":
    main()
