"""A/B of the executor's two host paths on one workload (sync switches):
two-step (plan_repartition + migrate, K1 events) vs one native call.

    python tools/e2e_paths.py [--config 1] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    w = bench.build_workload(args.config, None)
    device = torch.device("cuda", 0)
    ex = bench.setup_ours(w, device)
    fwd = True
    for _ in range(4):
        bench.one_switch(ex, w, fwd, sync=True)
        fwd = not fwd
    for mode in ("two_step", "one_call", "two_step", "one_call"):
        ex.time_kernels = mode == "two_step"
        host, dev = [], []
        for _ in range(args.reps):
            r = bench.one_switch(ex, w, fwd, sync=True)
            fwd = not fwd
            host.append(r.host_ms)
            dev.append(r.device_ms)
            assert r.status == 0
        print(json.dumps({"mode": mode, "host_ms": float(np.median(host)),
                          "device_ms": float(np.median(dev)), "host_ms_mean": float(np.mean(host))}))


if __name__ == "__main__":
    main()
