"""Capture the reference's KV-capacity admission / eviction decisions.

``Simulator._enforce_kv_capacity`` (pkg/src/tpsim/engine.py:623-645) runs inside
the controller hook when ``kv_accounting`` is on (engine.py:600-601): the
destination group's budget is ``(gpu_memory_gb - weight_full_copy_gb) * 1e9 *
tp`` bytes, ``used`` counts its running requests, arrivals are taken feasible
first then by arrival time, and a best-effort arrival that does not fit is
evicted (re-queued) while a feasible one is always kept.

Two sources of decisions, both from the UNMODIFIED reference:

* the demo experiment (pkg/configs/demo.yaml, dynamic policy) with
  ``kv_accounting`` on and the bundled profile's ``gpu_memory_gb`` lowered to
  26.2 GB (0.2 GB of KV per GPU above the 26 GB of weights), so its own
  migrations hit the budget; the wrapper below only observes each call;
* 300 random calls of the same method on reference ``_ReqState`` objects
  (random labels, arrival times, contexts, running sets, TP degrees and
  budgets; numpy seed 2026), so ties and boundary cases are pinned too.

    python tests/golden/gen_kv_capacity.py   # needs /root/reference
"""

from __future__ import annotations

import collections
import dataclasses
import gzip
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "kv_capacity.json.gz"


def _record(sim, state, arrivals, kept, pending_before):
    evicted = [rs.req.id for rs in list(sim.pending)[pending_before:]]
    return {
        "tp": state.group.tp,
        "gpu_memory_gb": sim.profile.gpu_memory_gb,
        "weight_full_copy_gb": sim.profile.weight_full_copy_gb,
        "kv_bytes_per_token": sim.profile.total_kv_heads * sim.profile.kv_bytes_per_token_per_head,
        "running": [rs.context_len for rs in state.running],
        "arrivals": [[rs.req.id, rs.context_len, rs.label, rs.req.arrival_time]
                     for _, rs in arrivals],
        "kept": [rs.req.id for _, rs in kept],
        "evicted": evicted,
    }


def demo_calls():
    import tpsim.engine as E
    from tpsim.cli import _run_one
    from tpsim.config import load_config

    out = []
    real = E.Simulator._enforce_kv_capacity

    def wrap(self, state, arrivals):
        snap = [(p, p[1].context_len) for p in arrivals]  # before eviction resets `generated`
        n0 = len(self.pending)
        kept = real(self, state, arrivals)
        rec = _record(self, state, arrivals, kept, n0)
        rec["arrivals"] = [[p[1].req.id, ctx, p[1].label, p[1].req.arrival_time] for p, ctx in snap]
        out.append(rec)
        return kept

    E.Simulator._enforce_kv_capacity = wrap
    try:
        cfg = load_config(str(REF / "configs" / "demo.yaml"))
        prof = dataclasses.replace(cfg.profile, gpu_memory_gb=26.2)
        cfg = dataclasses.replace(cfg, profile=prof,
                                  engine=dataclasses.replace(cfg.engine, kv_accounting=True))
        _run_one(cfg, "dynamic")
    finally:
        E.Simulator._enforce_kv_capacity = real
    return [c for c in out if c["arrivals"]]


def random_calls(n=300, seed=2026):
    import tpsim.engine as E
    from tpsim.trace import Request

    rng = np.random.default_rng(seed)
    out = []
    rid = 0
    for _ in range(n):
        tp = int(rng.choice([1, 2, 4, 8]))
        heads, kvb = 32, 4096
        prof = SimpleNamespace(gpu_memory_gb=float(rng.uniform(26.0, 27.0)), weight_full_copy_gb=26.0,
                               total_kv_heads=heads, kv_bytes_per_token_per_head=kvb)

        def req_state(label):
            nonlocal rid
            rid += 1
            prompt = int(rng.integers(1, 3000))
            rq = Request(id=rid, tier_id=int(label == E.BEST_EFFORT),
                         arrival_time=float(rng.choice([rng.uniform(0, 40), 5.0])),
                         prompt_len=prompt, output_len=int(rng.integers(1, 300)))
            rs = E._ReqState(req=rq, label=label)
            rs.generated = int(rng.integers(0, rq.output_len))
            return rs

        labels = [E.FEASIBLE, E.BEST_EFFORT]
        running = [req_state(labels[int(rng.integers(2))]) for _ in range(int(rng.integers(0, 6)))]
        arrivals = [(None, req_state(labels[int(rng.integers(2))]))
                    for _ in range(int(rng.integers(1, 12)))]
        sim = SimpleNamespace(profile=prof, pending=collections.deque(), preemptions=0)
        sim._kv_bytes = lambda rs, _s=sim: E.Simulator._kv_bytes(_s, rs)
        state = SimpleNamespace(running=running, group=SimpleNamespace(tp=tp))
        snap = [(p, p[1].context_len) for p in arrivals]
        kept = E.Simulator._enforce_kv_capacity(sim, state, arrivals)
        rec = _record(sim, state, arrivals, kept, 0)
        rec["arrivals"] = [[p[1].req.id, ctx, p[1].label, p[1].req.arrival_time] for p, ctx in snap]
        out.append(rec)
    return out


def main():
    sys.path.insert(0, str(REF / "src"))
    doc = {"source": "tpsim Simulator._enforce_kv_capacity (engine.py:623-645)",
           "demo": demo_calls(), "random": random_calls()}
    with gzip.open(OUT, "wt") as f:
        json.dump(doc, f)
    ev = sum(len(c["evicted"]) for c in doc["demo"] + doc["random"])
    print(OUT, len(doc["demo"]), "demo calls,", len(doc["random"]), "random calls,", ev, "evictions")


if __name__ == "__main__":
    main()
