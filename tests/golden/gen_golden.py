"""Generate golden vectors by running the UNMODIFIED reference (tpsim) here.

Run in the build container (where /root/reference exists):

    python tests/golden/gen_golden.py

Writes tests/golden/reference_golden.json.gz. The GPU box never needs the
reference: tests read only the committed fixture. Contents:

* ac1      -- the reference's exhaustive AC-1 sweep inputs (45 (H, TP_old,
              TP_new) combos x seeds, rng 2024, 20 requests,
              pkg/tests/test_migration.py:110-143) with every plan's full
              transfer list;
* figures  -- the paper-figure cases (test_migration.py:42-79);
* configs  -- the BASELINE configs' plans (cfg1..cfg4 + the TP1->TP8 256-seq
              sweep extreme) as transfer arrays + total bytes;
* engine   -- head_transfers on disjoint groups (engine path, engine.py:571-589);
* costs    -- latency_per_page / aggregate / pipelined / switch_cost on 500
              random plans (rng 7, test_migration.py:263-305) and default params;
* weights  -- weight_memory for the three modes;
* cli      -- `tpsim migrate-plan` JSON for the test_cli.py layout.
"""

from __future__ import annotations

import gzip
import io
import json
import sys
from contextlib import redirect_stdout
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "reference_golden.json.gz"


def main():
    sys.path.insert(0, str(REF))
    import tpsim
    from tpsim import migration as M
    from tpsim.cli import main as cli_main

    def rows(plan):
        return [[t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes]
                for t in plan.transfers]

    def lay(group, H, reqs):
        return M.KvLayout(group=tuple(group), tp=len(group), total_heads=H, requests=tuple(reqs))

    doc = {"reference": "tpsim " + getattr(tpsim, "__version__", "?"), "kvb": 4096}

    # -- AC-1 sweep -----------------------------------------------------------
    rng = np.random.default_rng(2024)
    ac1 = []
    for h in (2, 4, 8, 16):
        for a in (1, 2, 4, 8):
            for b in (1, 2, 4, 8):
                if h % a or h % b:
                    continue
                n = max(a, b)
                gpus = list(range(1, n + 1))
                for _ in range(50 if (h, a, b) != (2, 1, 1) else 5):
                    ctxs = [int(c) for c in rng.integers(1, 5000, size=20)]
                    og = [gpus[i:i + a] for i in range(0, n, a)]
                    ng = [gpus[i:i + b] for i in range(0, n, b)]
                    orq = [[] for _ in og]
                    nrq = [[] for _ in ng]
                    for rid, c in enumerate(ctxs):
                        orq[rid % len(og)].append((rid, c))
                        nrq[rid % len(ng)].append((rid, c))
                    old = [lay(g, h, r) for g, r in zip(og, orq)]
                    new = [lay(g, h, r) for g, r in zip(ng, nrq)]
                    plan = M.plan_repartition(old, new, 4096)
                    assert M.apply_plan(old, plan) == M.layout_placement(new)
                    ac1.append({"H": h, "tp_old": a, "tp_new": b, "ctxs": ctxs,
                                "old": [[g, r] for g, r in zip(og, orq)],
                                "new": [[g, r] for g, r in zip(ng, nrq)],
                                "transfers": rows(plan)})
    doc["ac1"] = ac1

    # -- paper figure cases ----------------------------------------------------
    figs = {}
    figs["tp1_tp2"] = rows(M.plan_repartition(
        [lay([1], 8, [(0, 100)]), lay([2], 8, [(1, 100)])], lay([1, 2], 8, [(0, 100), (1, 100)]), 4096))
    figs["tp2_tp4"] = rows(M.plan_repartition(
        [lay([1, 2], 8, [(0, 10)]), lay([3, 4], 8, [(1, 10)])],
        lay([1, 2, 3, 4], 8, [(0, 10), (1, 10)]), 4096))
    figs["identity"] = rows(M.plan_repartition([lay([1, 2], 8, [(0, 50)])], lay([1, 2], 8, [(0, 50)]), 4096))
    figs["tp4_tp2"] = rows(M.plan_repartition(
        [lay([0, 1, 2, 3], 8, [(0, 7)])], [lay([0, 1], 8, [(0, 7)]), lay([2, 3], 8, [])], 16384))
    figs["reversed_group"] = rows(M.plan_repartition([lay([0, 1], 8, [(0, 3)])], lay([1, 0], 8, [(0, 3)]), 16))
    figs["zero_ctx"] = rows(M.plan_repartition([lay([0], 8, [(5, 0)]), lay([1], 8, [])],
                                               lay([0, 1], 8, [(5, 0)]), 4096))
    figs["order"] = rows(M.plan_repartition([lay([0], 8, [(5, 10), (3, 20)]), lay([1], 8, [(9, 30)])],
                                            lay([0, 1], 8, [(9, 30), (3, 20), (5, 10)]), 4096))
    doc["figures"] = figs

    # -- BASELINE configs (8 KV heads, Llama-3.1 kvb) ----------------------------
    def rr(groups, reqs, H):
        per = [[] for _ in groups]
        for i, r in enumerate(reqs):
            per[i % len(groups)].append(r)
        return [lay(g, H, p) for g, p in zip(groups, per)]

    def grp(n, tp):
        return [list(range(i, i + tp)) for i in range(0, n, tp)]

    cfgs = {}
    cfgs["cfg1"] = (rr(grp(2, 1), [(i, 512) for i in range(4)], 8),
                    rr(grp(2, 2), [(i, 512) for i in range(4)], 8), 16384)
    cfgs["cfg2"] = (rr(grp(4, 2), [(i, 4096) for i in range(64)], 8),
                    rr(grp(4, 4), [(i, 4096) for i in range(64)], 8), 16384)
    reqs = [(i, 4096) for i in range(64)]
    cfgs["cfg3"] = ([lay(list(range(8)), 8, reqs)],
                    [lay([0], 8, reqs)] + [lay([g], 8, []) for g in range(1, 8)], 16384)
    cfgs["cfg4"] = (rr(grp(8, 4), [(i, 32768) for i in range(8)], 8),
                    rr(grp(8, 8), [(i, 32768) for i in range(8)], 8), 40960)
    cfgs["sweep_tp1_tp8_256"] = (rr(grp(8, 1), [(i, 4096) for i in range(256)], 8),
                                 rr(grp(8, 8), [(i, 4096) for i in range(256)], 8), 16384)
    doc["configs"] = {}
    for name, (old, new, kvb) in cfgs.items():
        plan = M.plan_repartition(old, new, kvb)
        doc["configs"][name] = {
            "old": [[list(l.group), [list(r) for r in l.requests]] for l in old],
            "new": [[list(l.group), [list(r) for r in l.requests]] for l in new],
            "kvb": kvb, "transfers": rows(plan), "total_bytes": plan.total_bytes,
            "bytes_by_source": {str(k): v for k, v in plan.bytes_by_source().items()},
        }

    # -- engine path: disjoint groups through head_transfers -------------------
    eng = []
    for og, ng, rq in (([0, 1], [4, 5, 6, 7], [(0, 33)]), ([0], [1], [(3, 17), (4, 1)]),
                       ([0, 1, 2, 3], [4, 5], [(7, 100)]), ([2, 3], [3, 2], [(1, 5)])):
        eng.append({"old": og, "new": ng, "requests": rq,
                    "transfers": [[t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes]
                                  for t in M.head_transfers(lay(og, 8, rq), lay(ng, 8, rq), 4096)]})
    doc["engine"] = eng

    # -- cost models -------------------------------------------------------------
    rng = np.random.default_rng(7)
    costs = []
    for _ in range(500):
        page = int(2 ** rng.integers(12, 18))
        chunk = int(2 ** rng.integers(24, 29))
        link = float(rng.uniform(10, 300))
        copy = link * float(rng.uniform(1.5, 10.0))
        lo = 10.0 * page / (copy * 1e9) * 1e6
        hi = 0.5 * chunk / (copy * 1e9) * 1e6
        overhead = float(np.exp(rng.uniform(np.log(lo), np.log(hi))))
        params = M.CostModelParams(copy_bw_gbps=copy, link_bw_gbps=link,
                                   per_transfer_overhead_us=overhead, page_bytes=page,
                                   chunk_bytes=chunk)
        transfers = []
        for src in range(int(rng.integers(1, 5))):
            remaining = int(rng.integers(chunk, 2_000_000_000))
            for dst in range(int(rng.integers(1, 4))):
                part = max(1, remaining // int(rng.integers(1, 4)))
                transfers.append([src, 100 + dst, dst, 0, 1, part])
                remaining -= part
                if remaining <= 0:
                    break
        plan = M.MigrationPlan(transfers=[M.Transfer(*t) for t in transfers])
        costs.append({
            "params": {k: getattr(params, k) for k in ("copy_bw_gbps", "link_bw_gbps",
                                                       "per_transfer_overhead_us", "page_bytes",
                                                       "chunk_bytes", "handshake_ms", "reload_ms",
                                                       "kernel_init_ms")},
            "transfers": transfers,
            "per_page": repr(M.latency_per_page(plan, params)),
            "aggregate": repr(M.latency_aggregate(plan, params)),
            "pipelined": repr(M.latency_pipelined(plan, params)),
            "warm": repr(M.switch_cost(M.WARM, plan, params)),
            "naive_reload": repr(M.switch_cost(M.NAIVE_RELOAD, plan, params)),
        })
    doc["costs"] = costs
    defaults = M.CostModelParams()
    doc["default_costs"] = {}
    for gb in (0.5, 1.0, 2.0, 5.0):
        plan = M.MigrationPlan(transfers=[M.Transfer(1, 2, 0, 0, 1, int(gb * 1e9))])
        doc["default_costs"][str(gb)] = [repr(M.latency_per_page(plan, defaults)),
                                         repr(M.latency_aggregate(plan, defaults)),
                                         repr(M.latency_pipelined(plan, defaults))]

    # -- weight memory -------------------------------------------------------------
    class P:
        weight_full_copy_gb = 26.0
        tp_levels = (1, 2, 4, 8)

    doc["weights"] = {"full_copy_per_gpu": M.weight_memory("full_copy_per_gpu", P),
                      "per_tp_copies": M.weight_memory("per_tp_copies", P),
                      **{f"sharded_{t}": M.weight_memory("sharded", P, tp=t) for t in (1, 2, 4, 8)}}

    # -- trace for the switch sweep (BASELINE config 5): the reference's bursty
    # workload (scenarios.py:58-85, seed 11) -> (prompt_len, output_len) pairs ----
    from tpsim.scenarios import bursty_spec
    from tpsim.trace import generate_trace
    trace = generate_trace(bursty_spec())
    doc["bursty_trace"] = [[r.prompt_len, r.output_len] for r in trace[:1024]]

    # -- CLI migrate-plan ----------------------------------------------------------
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "layout.json"
        path.write_text(json.dumps({
            "total_heads": 8, "kv_bytes_per_token_per_head": 4096,
            "groups": [{"gpus": [1], "requests": [{"id": 0, "context_len": 100}]},
                       {"gpus": [2], "requests": [{"id": 1, "context_len": 100}]}]}))
        buf = io.StringIO()
        with redirect_stdout(buf):
            rc = cli_main(["migrate-plan", "--layout", str(path), "--new-tp", "2"])
        doc["cli"] = {"rc": rc, "layout": json.loads(path.read_text()), "stdout": json.loads(buf.getvalue())}

    with gzip.open(OUT, "wt") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(OUT, OUT.stat().st_size, "bytes;", len(ac1), "AC-1 plans")


if __name__ == "__main__":
    main()
