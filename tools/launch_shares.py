"""Per-kernel launch counts, device time and share of the step from an ncu
launch list (``ncu --metrics gpu__time_duration.sum --csv``). The list is
cold-cache and serialised: compare shares, not absolute times.

    python tools/launch_shares.py profiles/r02_launches_cfg2.csv [--json out.json]
"""

from __future__ import annotations

import argparse
import csv
import json
from collections import defaultdict

UNIT_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def shares(path: str) -> dict:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui, mi = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].strip()
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * UNIT_US[r[ui]]
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": n, "total_us": t, "avg_us": t / n, "share": t / tot}
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    out = shares(args.csv)
    for k, v in out.items():
        print(f"{k:40s} n={v['launches']:4d} avg={v['avg_us']:10.1f} us  share={v['share']:.3f}")
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
