"""Host reshard planner (no device): reuse of resident slices, sources for
missing ones, and ``trim`` (PAPER.md:307 shard selection; weight_memory
volumes, migration.py:295-306)."""

import pytest

from paper_2605_05467_b200 import workloads
from paper_2605_05467_b200.geometry import MAX_TP, tiny_geometry
from paper_2605_05467_b200.migration import MigrationError
from paper_2605_05467_b200.weights import ShardedWeightStore, groups_ranges


def store_at(gpus, tp):
    s = ShardedWeightStore(tiny_geometry(), gpus, device="cpu")
    s.resident = groups_ranges(workloads.tp_groups(gpus, tp))
    s.active = dict(s.resident)
    return s


def test_scale_out_is_views_and_scale_in_fetches():
    gpus = (0, 1, 2, 3)
    s = store_at(gpus, 1)  # every GPU holds all 8 slices
    act, res, moves = s.plan(workloads.tp_groups(gpus, 4))
    assert all(m == [] for m in moves.values())  # TP1 -> TP4: views only
    assert res == {g: (0, MAX_TP) for g in gpus}
    s = store_at(gpus, 4)
    act, res, moves = s.plan(workloads.tp_groups(gpus, 1))
    for g in gpus:
        assert res[g] == (0, MAX_TP)
        got = sorted((lo, hi) for _, lo, hi in moves[g])
        assert got[0][0] == 0 and got[-1][1] == MAX_TP
        assert sum(hi - lo for _, lo, hi in moves[g] if _ != g) == 6  # 6/8 fetched
        assert all(src != g or (2 * g <= lo and hi <= 2 * g + 2) for src, lo, hi in moves[g])


def test_trim_compacts_to_the_active_shard():
    gpus = (0, 1, 2, 3)
    s = store_at(gpus, 1)
    _, res, moves = s.plan(workloads.tp_groups(gpus, 2), trim=True)
    assert res == groups_ranges(workloads.tp_groups(gpus, 2))
    for g in gpus:  # everything is local: a compaction copy, no fetch
        assert moves[g] and all(src == g for src, _, _ in moves[g])
    # an exact match is still a view with trim
    s = store_at(gpus, 2)
    _, _, moves = s.plan(workloads.tp_groups(gpus, 2), trim=True)
    assert all(m == [] for m in moves.values())


def test_groups_must_cover_store():
    s = store_at((0, 1), 2)
    with pytest.raises(MigrationError):
        s.plan([(0,)])
