"""profiles/k1_traffic.json from an ncu --set full raw CSV of the bench's K1.

``bench.py`` reports ``roofline.traffic`` = dram__bytes_read.sum +
dram__bytes_write.sum of one K1 launch of the workload (B200_PROFILING.md):
this script reads those two counters (and the duration) from the raw page of
an ``ncu --set full`` capture and writes them next to the algorithmic bytes.

    ncu -i cap.ncu-rep --page raw --csv > profiles/rNN_k1_full_raw.csv
    python tools/ncu_traffic.py profiles/rNN_k1_full_raw.csv --workload "<bench workload name>" \\
        --algorithmic 51539607552
"""

from __future__ import annotations

import argparse
import csv
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TIME = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def read(path: str, kernel_substr: str):
    rows = list(csv.reader(open(path)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[head.index("Kernel Name")]
        if kernel_substr not in name:
            continue

        def val(metric, scale):
            i = head.index(metric)
            return float(r[i].replace(",", "")) * scale[units[i]]

        out.append({"kernel": name,
                    "dram_bytes": val("dram__bytes_read.sum", SCALE) + val("dram__bytes_write.sum", SCALE),
                    "duration_ms": val("gpu__time_duration.sum", TIME)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--algorithmic", type=int, required=True, help="read + write bytes of one K1")
    ap.add_argument("--kernel", default="tpr_k1_kv_migrate")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "k1_traffic.json"))
    args = ap.parse_args()
    launches = read(args.csv, args.kernel)
    if not launches:
        raise SystemExit(f"no {args.kernel} launch in {args.csv}")
    k = launches[0]
    doc = {"kernel": k["kernel"].split("(")[0], "workload": args.workload,
           "source": f"{args.csv} (ncu --set full)",
           "algorithmic_bytes_per_launch": args.algorithmic,
           "dram_bytes_per_launch": int(k["dram_bytes"]), "duration_ms_ncu": k["duration_ms"],
           "dram_over_algorithmic": k["dram_bytes"] / args.algorithmic}
    Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
