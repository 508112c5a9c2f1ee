"""Reuse-aware rank order and KV-capacity admission (§8f.2)."""

import itertools

import numpy as np
import pytest

from paper_2605_05467_b200 import migration as M
from paper_2605_05467_b200.placement import (BEST_EFFORT, FEASIBLE, Arrival, enforce_kv_capacity,
                                             reuse_rank_order)


def lay(group, reqs, H=8):
    return M.KvLayout(tuple(group), len(group), H, tuple(reqs))


def test_reuse_order_is_optimal_over_all_permutations():
    rng = np.random.default_rng(3)
    for _ in range(20):
        reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 500, size=6))]
        old = [lay([3, 1], reqs[:2]), lay([0], reqs[2:4]), lay([2], reqs[4:])]
        gpus = (0, 1, 2, 3)
        order = reuse_rank_order(old, gpus, 4096)
        best = M.plan_repartition(old, lay(order, reqs), 4096).total_bytes
        brute = min(M.plan_repartition(old, lay(p, reqs), 4096).total_bytes
                    for p in itertools.permutations(gpus))
        assert best == brute
        assert best <= M.plan_repartition(old, lay(gpus, reqs), 4096).total_bytes


def test_reuse_order_keeps_canonical_when_already_optimal():
    reqs = [(0, 10), (1, 10)]
    old = [lay([0], reqs[:1]), lay([1], reqs[1:])]
    assert reuse_rank_order(old, (0, 1), 4096) == (0, 1)


def test_reuse_order_cuts_tp2_to_tp4_traffic():
    # canonical TP2 (0,1),(2,3) -> TP4 (0,1,2,3) moves 3/4 of the KV; interleaving
    # the two old groups' rank-0 GPUs first keeps half of it in place
    reqs = [(i, 4096) for i in range(8)]
    old = [lay([0, 1], reqs[0::2]), lay([2, 3], reqs[1::2])]
    canonical = M.plan_repartition(old, lay([0, 1, 2, 3], reqs), 16384).total_bytes
    order = reuse_rank_order(old, (0, 1, 2, 3), 16384)
    assert order == (0, 2, 1, 3)
    reuse = M.plan_repartition(old, lay(order, reqs), 16384).total_bytes
    total = 8 * 8 * 4096 * 16384
    assert canonical == total * 3 // 4 and reuse == total // 2


def test_reversed_group_avoids_full_swap():
    # old group (0,1) -> caller proposes (1,0): every head would move; reuse keeps (0,1)
    old = [lay([0, 1], [(0, 100)])]
    assert M.plan_repartition(old, lay([1, 0], [(0, 100)]), 16).total_bytes > 0
    order = reuse_rank_order(old, (1, 0), 16)
    assert order == (0, 1)
    assert M.plan_repartition(old, lay(order, [(0, 100)]), 16).total_bytes == 0


class _FakeCluster:
    class kv:
        @staticmethod
        def blocks(c):
            return -(-c // 16)

    def __init__(self, free):
        self._free = free

    def free_units(self, g):
        return self._free[g]


def test_capacity_orders_feasible_first_then_oldest():
    c = _FakeCluster({0: 40, 1: 40})
    layout = lay([0, 1], [])
    arr = [Arrival(1, 160, BEST_EFFORT, 0.5),   # 10 pages x 4 heads = 40 per gpu
           Arrival(2, 80, FEASIBLE, 2.0),       # 20 per gpu
           Arrival(3, 16, BEST_EFFORT, 0.1),    # 4 per gpu
           Arrival(4, 400, FEASIBLE, 3.0)]      # never evicted even though it overflows
    kept, evicted = enforce_kv_capacity(c, layout, arr)
    assert [a.request_id for a in kept] == [2, 4, 3] or [a.request_id for a in kept] == [2, 4]
    assert 1 in [a.request_id for a in evicted]
    assert all(a.label == BEST_EFFORT for a in evicted)


def test_capacity_keeps_everything_that_fits():
    c = _FakeCluster({0: 1000})
    kept, evicted = enforce_kv_capacity(c, lay([0], []), [Arrival(i, 100) for i in range(5)])
    assert len(kept) == 5 and not evicted


def test_kv_capacity_decisions_match_the_reference_engine():
    # every _enforce_kv_capacity call of the unmodified reference
    # (tests/golden/gen_kv_capacity.py): its demo run with kv_accounting on,
    # plus 300 random calls; same kept order, same evictions
    import gzip
    import json

    from conftest import ROOT
    from paper_2605_05467_b200.placement import KvBudget, kv_capacity_decisions
    with gzip.open(ROOT / "tests" / "golden" / "kv_capacity.json.gz", "rt") as f:
        doc = json.load(f)
    n_ev = 0
    for c in doc["demo"] + doc["random"]:
        arr = [Arrival(r, ctx, label, t) for r, ctx, label, t in c["arrivals"]]
        budget = KvBudget(c["gpu_memory_gb"], c["weight_full_copy_gb"]).bytes(c["tp"])
        used = sum(c["running"]) * c["kv_bytes_per_token"]
        kept, ev = kv_capacity_decisions(arr, budget, used, c["kv_bytes_per_token"])
        assert [a.request_id for a in kept] == c["kept"]
        assert [a.request_id for a in ev] == c["evicted"]
        n_ev += len(ev)
    assert len(doc["demo"]) >= 10 and n_ev > 100
