"""Weight-reshard sweep: every TP transition of Llama-3.1-8B sharded weights,
{1,2,4} on 4 GPU slots and {2,4,8} on 8 slots (TP1 on 8 slots would hold 8 full
copies). All slots are logical, in one B200. For each transition: bytes
rebuilt (local + fetched), K2 time (CUDA events on its stream), GB/s and the
HBM-roofline fraction, and a pattern check of every resulting shard.

    python tools/weight_sweep.py --out profiles/r01_weight_sweep.jsonl

Llama-3.1-70B: its full sharded copy is 141 GB, so 8 logical slots of it
cannot sit in one 180 GB HBM. ``--model 70b --layers 20`` keeps every 70B
matrix shape (and the embedding / lm_head) with 20 of the 80 decoder layers:
K2's per-byte behaviour (row lengths, segment mix) is that of the full model
and bytes scale linearly with the layer count.

    python tools/weight_sweep.py --model 70b --layers 20 --sets 8:4,8 --sets 4:2,4
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
    import dataclasses

    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B, LLAMA_3_1_70B, MAX_TP
    from paper_2605_05467_b200.weights import ShardedWeightStore

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "weight_sweep.jsonl"))
    ap.add_argument("--reps", type=int, default=5, help="timed a->b reshards (median)")
    ap.add_argument("--engine", choices=["bulk", "vector"], default="bulk")
    ap.add_argument("--only", default="", help="comma list of slots:a:b, e.g. 8:2:4")
    ap.add_argument("--model", choices=["8b", "70b"], default="8b")
    ap.add_argument("--layers", type=int, default=None, help="decoder layers kept (default: all)")
    ap.add_argument("--sets", action="append", default=None,
                    help="slots:levels, e.g. 8:2,4,8 (repeatable)")
    args = ap.parse_args()
    model = LLAMA_3_1_8B if args.model == "8b" else LLAMA_3_1_70B
    if args.layers is not None and args.layers != model.layers:
        model = dataclasses.replace(model, name=f"{model.name} ({args.layers} of {model.layers} layers)",
                                    layers=args.layers, matrices=())
    sets = [(4, (1, 2, 4)), (8, (2, 4, 8))] if not args.sets else [
        (int(x.split(":")[0]), tuple(int(v) for v in x.split(":")[1].split(","))) for x in args.sets]
    from paper_2605_05467_b200 import _native
    _native.set_copy_engine(args.engine)
    only = {tuple(int(v) for v in x.split(":")) for x in args.only.split(",") if x}
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    out = open(args.out, "w")
    for n, levels in sets:
        gpus = tuple(range(n))
        for a in levels:
            for b in levels:
                if a == b or (only and (n, a, b) not in only):
                    continue
                # a->b timed, b->a untimed, repeated; the first pair is warm-up
                # (the first touch of freshly cudaMalloc'd arenas costs ~0.1
                # ms/GB once per process; the caching allocator reuses them)
                # arena window: the larger of the two shards (slices), the least
                # HBM that still lets a growing shard stay in place
                store = ShardedWeightStore(model, gpus, max_slices=max(MAX_TP // a, MAX_TP // b))
                store.load(workloads.tp_groups(gpus, a))
                torch.cuda.synchronize()
                st = torch.cuda.current_stream()
                times = []
                for r in range(args.reps + 1):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s = store.reshard(workloads.tp_groups(gpus, b), stream=st, events=(e0, e1))
                    torch.cuda.synchronize()
                    if r:
                        times.append(e0.elapsed_time(e1))
                    if r < args.reps:
                        # back to exactly TP-a residency (trim drops slices a
                        # TP-b shard kept for reuse), so every timed a->b
                        # reshard rebuilds what a fresh TP-a deployment would
                        store.reshard(workloads.tp_groups(gpus, a), stream=st, trim=True)
                ms = sorted(times)[len(times) // 2]
                bad = store.verify()
                row = {"model": model.name, "gpus": n, "tp_old": a, "tp_new": b, "views": s.views,
                       "local_bytes": s.local_bytes, "remote_bytes": s.remote_bytes,
                       "segments": s.segments, "k2_ms": ms, "k2_ms_min": min(times),
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
