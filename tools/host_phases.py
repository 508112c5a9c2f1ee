"""Per-phase host cost of a small switch (cfg1 shape), median over N."""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main(n=400):
    import ctypes

    import torch

    import bench
    from paper_2605_05467_b200 import _native, migration as M, workloads
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    w = workloads.config(0)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=bench.capacity_units(w, kv),
                       max_requests=len(w.requests), max_blocks=kv.blocks(512))
    c.admit(w.old)
    st = torch.cuda.Stream()
    t = {k: [] for k in ("plan", "records", "reserve", "stage", "native", "owner", "total")}
    for i in range(n):
        a, b = (w.old, w.new) if i % 2 == 0 else (w.new, w.old)
        t0 = time.perf_counter()
        plan = M.plan_repartition(a, b, kv.kv_bytes_per_token_per_head)
        t1 = time.perf_counter()
        xf = c.records(plan, validate=False)
        t2 = time.perf_counter()
        total, in_u, out_u = c._reserve(xf)
        t3 = time.perf_counter()
        cl = c._cluster_c()
        d_xf = c._xf.get(len(xf) * 6, st)
        d_meta = c._meta.get(len(xf) * 4, st)
        d_work = c._work.get(total * 4, st)
        h = c._staging.stage(xf.astype(np.int32))
        t4 = time.perf_counter()
        _native.call("tpr_kv_switch", ctypes.byref(c._geo), ctypes.byref(cl), h, d_xf.data_ptr(),
                     len(xf), -1, d_meta.data_ptr(), c._totals.data_ptr(), total, d_work.data_ptr(),
                     c.status.data_ptr(), st.cuda_stream)
        c._staging.fence(st)
        t5 = time.perf_counter()
        c._commit(in_u, out_u)
        for s, d, r, lo, hi, _ in xf.tolist():
            c.owner[r, lo:hi] = d
        t6 = time.perf_counter()
        for k, (x, y) in zip(t, ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t4, t5), (t5, t6), (t0, t6))):
            t[k].append((y - x) * 1e6)
        if i % 16 == 15:
            st.synchronize()
    st.synchronize()
    print({k: round(float(np.median(v)), 1) for k, v in t.items()}, "us (median)")


if __name__ == "__main__":
    main()
