"""``migrate-plan`` with the reference's JSON contract (cli.py:196-253), plus
optional execution on a B200.

    python -m paper_2605_05467_b200.cli migrate-plan --layout L.json --new-tp N
        [--out plan.json] [--execute] [--model Llama-3.1-8B] [--fragmented]

Input schema (reference cli.py:197-209): {total_heads, kv_bytes_per_token_per_head
(default 4096), groups: [{gpus: [...], requests: [{id, context_len}]}]}. The
old groups merge into one TP group of all their GPUs (``new_tp`` must equal
its size, else exit 2). Output: {transfers: [...], total_bytes, handshake_ms,
latency_ms: {per_page_ms, aggregate_ms, pipelined_ms}} -- identical to the
reference -- and, with --execute, a "measured" object for the plan executed
on the current CUDA device (all GPUs of the layout as logical slots).
"""

from __future__ import annotations

import argparse
import json
import sys
import time

from . import migration as M

EXIT_VALIDATION = 2


def _plan(doc: dict, new_tp: int):
    kvb = int(doc.get("kv_bytes_per_token_per_head", 4096))
    H = int(doc["total_heads"])
    old = [M.KvLayout(group=tuple(g["gpus"]), tp=len(g["gpus"]), total_heads=H,
                      requests=tuple((int(r["id"]), int(r["context_len"])) for r in g["requests"]))
           for g in doc["groups"]]
    gpus = tuple(g for lay in old for g in lay.group)
    if new_tp != len(gpus):
        raise ValueError(f"new_tp: target tp {new_tp} must equal the merged group size {len(gpus)}")
    new = M.KvLayout(group=gpus, tp=new_tp, total_heads=H,
                     requests=tuple(r for lay in old for r in lay.requests))
    params = M.CostModelParams()
    plan = M.plan_repartition(old, new, kvb, handshake_ms=params.handshake_ms)
    return old, new, kvb, plan, params


def _execute(old, new, kvb, model_name: str, fragmented: bool) -> dict:
    import torch

    from .geometry import MODELS, KvGeometry
    from .kvcache import PagedKvCluster

    if model_name not in MODELS:
        raise ValueError(f"unknown model {model_name!r}; choose from {sorted(MODELS)}")
    geo = MODELS[model_name].kv
    H = old[0].total_heads
    if geo.kv_bytes_per_token_per_head != kvb or geo.total_heads != H:
        # keep the model's layer/dim split but honour the layout's head count and kvb
        if kvb % (2 * geo.dtype_bytes * geo.head_dim):
            raise ValueError(f"kv_bytes_per_token_per_head={kvb} does not fit head_dim {geo.head_dim}")
        geo = KvGeometry(layers=kvb // (2 * geo.dtype_bytes * geo.head_dim), head_dim=geo.head_dim,
                         total_heads=H, dtype_bytes=geo.dtype_bytes, block_tokens=geo.block_tokens)
    if not torch.cuda.is_available():
        raise ValueError("--execute needs a CUDA device")
    reqs = [r for lay in old for r in lay.requests]
    pages = {g: 0 for g in new.group}
    for lay in (*old, new):
        for _, c in lay.requests:
            for g in lay.owners():
                pages[g] += geo.blocks(c)
    cluster = PagedKvCluster(geo, new.group, units_per_gpu={g: n + 16 for g, n in pages.items()},
                             max_requests=len(reqs), max_blocks=max(1, max(geo.blocks(c) for _, c in reqs)),
                             fragmented=fragmented)
    cluster.admit(old, seed=7)
    plan = M.plan_repartition(old, new, kvb)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    start.record()
    stats = cluster.migrate(plan)
    end.record()
    end.synchronize()
    host_ms = (time.perf_counter() - t0) * 1e3
    dev_ms = start.elapsed_time(end)
    check = cluster.verify()
    return {
        "device": torch.cuda.get_device_name(),
        "device_ms": dev_ms, "host_ms": host_ms,
        "gbs": stats.bytes / (dev_ms * 1e-3) / 1e9 if dev_ms > 0 else None,
        "pages": stats.units, "bytes": stats.bytes,
        "bit_exact_property": check["placement_errors"] == 0 and check["word_mismatches"] == 0
        and check["status"] == 0,
        "placement_matches_reference": cluster.placement() == M.layout_placement(new),
        "geometry": {"layers": geo.layers, "head_dim": geo.head_dim, "block_tokens": geo.block_tokens},
    }


def cmd_migrate_plan(args) -> int:
    with open(args.layout) as f:
        doc = json.load(f)
    old, new, kvb, plan, params = _plan(doc, args.new_tp)
    table = {
        "per_page_ms": M.latency_per_page(plan, params),
        "aggregate_ms": M.latency_aggregate(plan, params),
        "pipelined_ms": M.latency_pipelined(plan, params),
    }
    out = {
        "transfers": [dict(zip(("src_gpu", "dst_gpu", "request_id", "head_lo", "head_hi", "bytes"), row))
                      for row in plan.as_array().tolist()],
        "total_bytes": plan.total_bytes,
        "handshake_ms": plan.handshake_ms,
        "latency_ms": table,
    }
    if args.execute:
        out["measured"] = _execute(old, new, kvb, args.model, args.fragmented)
    text = json.dumps(out, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    print(text)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2605_05467_b200")
    sub = p.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("migrate-plan", help="plan a TP transition, cost it, optionally execute it")
    sp.add_argument("--layout", required=True, help="JSON old-layout file")
    sp.add_argument("--new-tp", dest="new_tp", type=int, required=True)
    sp.add_argument("--out")
    sp.add_argument("--execute", action="store_true", help="run the plan on the current B200")
    sp.add_argument("--model", default="Llama-3.1-8B")
    sp.add_argument("--fragmented", action="store_true", help="fragmented free lists")
    sp.set_defaults(func=cmd_migrate_plan)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (FileNotFoundError, ValueError, KeyError) as e:  # MigrationError is a ValueError
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VALIDATION


if __name__ == "__main__":
    sys.exit(main())
