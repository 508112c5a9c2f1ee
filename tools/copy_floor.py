"""The copy floor of one B200 at small sizes: how long the device itself
takes to move N bytes (read + write) when nothing else is in the way.

For each size this times, on the device clock (CUDA events around ONE
operation, median of --reps, the stream held by a sleep kernel while the host
enqueues so launch latency on the host side is excluded):

* ``torch``: ``dst.copy_(src)`` of one contiguous buffer (the copy kernel the
  measured HBM peak in MEASURED_PEAKS.json comes from);
* ``memcpy``: ``cudaMemcpyAsync`` device-to-device (the copy engines).

It bounds what a TP switch of the same byte count can reach: K1/K31 move
scattered 256 KiB pages, so they cannot beat a contiguous copy.

    python tools/copy_floor.py --out profiles/r02_copy_floor.jsonl
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SIZES_MIB = (4, 8, 16, 29, 64, 128, 256, 448, 1024, 3584)


def main():
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=100)
    args = ap.parse_args()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    big = max(SIZES_MIB) << 20
    src = torch.empty(big, dtype=torch.uint8, device="cuda")
    dst = torch.empty(big, dtype=torch.uint8, device="cuda")
    src.fill_(1)
    dst.fill_(2)
    import ctypes

    from paper_2605_05467_b200 import _native
    out = open(args.out, "w") if args.out else None
    for mib in SIZES_MIB:
        n = mib << 20
        srcp = (ctypes.c_uint64 * 1)(src.data_ptr())
        dstp = (ctypes.c_uint64 * 1)(dst.data_ptr())
        nbytes = (ctypes.c_uint64 * 1)(n)
        row = {"mib": mib, "bytes": n, "roof_us": 2 * n / (peak * 1e9) * 1e6}
        for how in ("torch", "memcpy"):
            ts = []
            for i in range(args.reps + 5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(100_000)
                e0.record(st)
                if how == "torch":
                    dst[:n].copy_(src[:n])
                else:  # one cudaMemcpyAsync through libtpr's baseline entry
                    _native.call("tpr_baseline_copy_pages", srcp, dstp, nbytes, 1, 0,
                                 st.cuda_stream)
                e1.record(st)
                e1.synchronize()
                if i >= 5:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            us = float(np.median(ts))
            row[f"{how}_us"] = us
            row[f"{how}_frac"] = row["roof_us"] / us
        print(json.dumps(row), flush=True)
        if out:
            out.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
