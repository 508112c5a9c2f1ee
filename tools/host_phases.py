"""Per-phase host cost of a small switch through the one-call path
(PagedKvCluster.switch_layouts), median over N. The switch is enqueued only
(no sync inside the timed phases); every 16 switches the stream is drained.

    python tools/host_phases.py [--config 0] [--n 400]
"""

from __future__ import annotations

import argparse
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from paper_2605_05467_b200 import _native, migration as M, workloads
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--n", type=int, default=400)
    args = ap.parse_args()
    w = workloads.config(args.config, weights=False) if args.config else workloads.config(0)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=bench.capacity_units(w, kv),
                       max_requests=len(w.requests),
                       max_blocks=kv.blocks(max(x for _, x in w.requests)))
    c.admit(w.old)
    st = torch.cuda.current_stream()
    for i in range(20):
        c.switch_layouts(*((w.old, w.new) if i % 2 == 0 else (w.new, w.old)), stream=st)
    st.synchronize()
    lib = _native.load()
    t = {k: [] for k in ("pack", "tables+staging", "native", "post", "total", "switch_layouts")}
    for i in range(args.n):
        a, b = (w.old, w.new) if i % 2 == 0 else (w.new, w.old)
        t0 = time.perf_counter()
        blob = M.pack_layouts(a, b)
        t1 = time.perf_counter()
        tab = c._switch_tables(False)
        tab.mode = _native.TPR_SWITCH_REPARTITION
        rows = c._swt_plan
        h_ptr, _ = c._staging.acquire(max(len(rows), 1) * 24)
        tab.plan, tab.plan_cap, tab.records = rows.ctypes.data, len(rows), h_ptr
        tab.d_xfers = c._xf.get(max(len(rows), 1) * 6, st).data_ptr()
        tab.d_meta = c._meta.get(max(len(rows), 1) * 4, st).data_ptr()
        tab.xfers_cap = len(rows)
        work = c._work.t
        tab.d_work, tab.work_cap = work.data_ptr(), work.numel() // 4
        cl = c._cluster_c()
        t2 = time.perf_counter()
        rc = lib.tpr_kv_switch_layouts(ctypes.byref(c._geo), ctypes.byref(cl),
                                       blob.buffer_info()[0], len(blob), ctypes.byref(tab),
                                       st.cuda_stream)
        t3 = time.perf_counter()
        assert rc == 0, rc
        n = tab.n_plan
        plan = M.MigrationPlan.from_array(rows[:n].copy())
        c._staging.fence(st)
        for s_ in range(c.n_gpus):
            c.ring_head[s_] += tab.in_units[s_]
            c.ring_tail[s_] += tab.out_units[s_]
        _ = plan.total_bytes
        t4 = time.perf_counter()
        for k, (x, y) in zip(t, ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t0, t4))):
            t[k].append((y - x) * 1e6)
        if i % 16 == 15:
            st.synchronize()
    st.synchronize()
    for i in range(args.n):  # the public call, for comparison
        a, b = (w.old, w.new) if i % 2 == 0 else (w.new, w.old)
        t0 = time.perf_counter()
        c.switch_layouts(a, b, stream=st, validate=False)
        t["switch_layouts"].append((time.perf_counter() - t0) * 1e6)
        if i % 16 == 15:
            st.synchronize()
    st.synchronize()
    print({k: round(float(np.median(v)), 1) for k, v in t.items()}, "us (median)")


if __name__ == "__main__":
    main()
