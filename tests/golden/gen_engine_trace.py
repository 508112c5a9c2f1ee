"""Capture the reference simulator's own reconfiguration decisions.

Runs the UNMODIFIED reference (tpsim) on its demo experiment
(pkg/configs/demo.yaml: two-phase workload, 8 GPUs, dynamic policy, warm
switches) and records every KV migration its controller hook plans:
``Simulator._apply_config`` (engine.py:500-621) calls ``head_transfers`` once
per migrating request (engine.py:571-589) and prices each destination group's
plan with ``switch_cost`` (engine.py:590-597). The wrappers below only observe
those calls. tools/replay_engine.py executes the same plans on a B200 and
compares measured pauses with the modeled ones.

    python tests/golden/gen_engine_trace.py   # needs /root/reference
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "engine_trace.json.gz"


def main():
    sys.path.insert(0, str(REF / "src"))
    import tpsim.engine as E
    from tpsim.cli import _run_one
    from tpsim.config import load_config

    events, pending, clock = [], [], {"now": 0.0, "window": -1}
    real_ht, real_cost, real_apply = E.head_transfers, E.switch_cost, E.Simulator._apply_config

    def head_transfers(old, new, kvb):
        (rid, ctx), = old.requests
        pending.append([list(old.group), list(new.group), rid, ctx])
        return real_ht(old, new, kvb)

    def switch_cost(mode, plan, params):
        cost = real_cost(mode, plan, params)
        events.append({"t": clock["now"], "mode": mode, "calls": list(pending),
                       "total_bytes": plan.total_bytes, "transfers": len(plan.transfers),
                       "modeled_switch_cost_ms": cost})
        pending.clear()
        return cost

    def apply_config(self, new):
        clock["now"] = self.now
        return real_apply(self, new)

    E.head_transfers, E.switch_cost = head_transfers, switch_cost
    E.Simulator._apply_config = apply_config
    cfg = load_config(str(REF / "configs" / "demo.yaml"))
    result, report = _run_one(cfg, "dynamic")
    prof = cfg.profile
    doc = {
        "source": "tpsim demo.yaml, dynamic policy, warm switches",
        "profile": {"total_kv_heads": prof.total_kv_heads,
                    "kv_bytes_per_token_per_head": prof.kv_bytes_per_token_per_head,
                    "weight_full_copy_gb": prof.weight_full_copy_gb, "pool_size": cfg.pool_size},
        "planning_delay_ms": cfg.engine.planning_delay_ms,
        "migration_count": result.migration_count, "total_pause_ms": result.total_pause_ms,
        "events": [e for e in events if e["calls"]],
    }
    with gzip.open(OUT, "wt") as f:
        json.dump(doc, f)
    n_calls = sum(len(e["calls"]) for e in doc["events"])
    print(OUT, len(doc["events"]), "plans,", n_calls, "head_transfers calls,",
          "migration_count", result.migration_count)


if __name__ == "__main__":
    main()
