"""Weight-reshard sweep: every TP transition of Llama-3.1-8B sharded weights,
{1,2,4} on 4 GPU slots and {2,4,8} on 8 slots (TP1 on 8 slots would hold 8 full
copies). All slots are logical, in one B200. For each transition: bytes
rebuilt (local + fetched), K2 time (CUDA events on its stream), GB/s and the
HBM-roofline fraction, and a pattern check of every resulting shard.

    python tools/weight_sweep.py --out profiles/r01_weight_sweep.jsonl
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2605_05467_b200 import workloads
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.weights import ShardedWeightStore

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "weight_sweep.jsonl"))
    args = ap.parse_args()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    out = open(args.out, "w")
    for n, levels in ((4, (1, 2, 4)), (8, (2, 4, 8))):
        gpus = tuple(range(n))
        for a in levels:
            for b in levels:
                if a == b:
                    continue
                # untimed pass first: the first touch of freshly cudaMalloc'd
                # arenas costs ~0.1 ms/GB once per process; serving reuses them
                warm = ShardedWeightStore(LLAMA_3_1_8B, gpus)
                warm.load(workloads.tp_groups(gpus, a))
                warm.reshard(workloads.tp_groups(gpus, b))
                torch.cuda.synchronize()
                del warm
                store = ShardedWeightStore(LLAMA_3_1_8B, gpus)
                store.load(workloads.tp_groups(gpus, a))
                torch.cuda.synchronize()
                st = torch.cuda.current_stream()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s = store.reshard(workloads.tp_groups(gpus, b), stream=st, events=(e0, e1))
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                bad = store.verify()
                row = {"gpus": n, "tp_old": a, "tp_new": b, "views": s.views,
                       "local_bytes": s.local_bytes, "remote_bytes": s.remote_bytes,
                       "segments": s.segments, "k2_ms": ms,
                       "gbs": s.bytes / (ms * 1e-3) / 1e9 if s.bytes else None,
                       "hbm_frac": (2 * s.bytes / (peak * 1e9)) / (ms * 1e-3) if s.bytes else None,
                       "max_ingress": max(s.ingress.values()), "max_egress": max(s.egress.values()),
                       "bit_exact_property": bad == 0}
                print(json.dumps(row))
                out.write(json.dumps(row) + "\n")
                out.flush()
                del store
                torch.cuda.empty_cache()
    out.close()


if __name__ == "__main__":
    main()
