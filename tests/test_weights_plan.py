"""Host reshard planner (no device): reuse of resident slices in place,
sources for missing ones, windows, and ``trim`` (PAPER.md:307 shard
selection; weight_memory volumes, migration.py:295-306)."""

import pytest

from paper_2605_05467_b200 import workloads
from paper_2605_05467_b200.geometry import MAX_TP, tiny_geometry
from paper_2605_05467_b200.migration import MigrationError
from paper_2605_05467_b200.weights import ShardedWeightStore, groups_ranges, window_for


def store_at(gpus, tp, max_slices=MAX_TP):
    s = ShardedWeightStore(tiny_geometry(), gpus, device="cpu", max_slices=max_slices)
    act = groups_ranges(workloads.tp_groups(gpus, tp))
    s.have = {g: frozenset(range(*r)) for g, r in act.items()}
    s.window = {g: window_for(*r, s.max_slices[g]) for g, r in act.items()}
    s.active = dict(act)
    return s


def test_scale_out_is_views_and_scale_in_fetches_only_missing_slices():
    gpus = (0, 1, 2, 3)
    s = store_at(gpus, 1)  # every GPU holds all 8 slices
    p = s.plan(workloads.tp_groups(gpus, 4))
    assert all(m == [] for m in p.fetch.values()) and not any(p.relayout.values())
    assert p.have == {g: frozenset(range(MAX_TP)) for g in gpus}
    s = store_at(gpus, 4)
    p = s.plan(workloads.tp_groups(gpus, 1))
    for g in gpus:
        assert p.have[g] == frozenset(range(MAX_TP)) and not p.relayout[g] and p.local[g] == []
        fetched = sorted(x for _, lo, hi in p.fetch[g] for x in range(lo, hi))
        # exactly the 6 slices g did not hold, none from itself
        assert fetched == [x for x in range(MAX_TP) if not 2 * g <= x < 2 * g + 2]
        assert all(src != g for src, _, _ in p.fetch[g])


def test_trim_drops_slices_without_moving_bytes():
    gpus = (0, 1, 2, 3)
    s = store_at(gpus, 1)
    p = s.plan(workloads.tp_groups(gpus, 2), trim=True)
    assert p.have == {g: frozenset(range(*r)) for g, r in groups_ranges(workloads.tp_groups(gpus, 2)).items()}
    assert all(m == [] for m in p.fetch.values()) and not any(p.local.values())


def test_windows_are_aligned_and_disjoint_or_shared():
    for m in (1, 2, 4, 8):
        for n in (1, 2, 4, 8):
            per = MAX_TP // n
            for r in range(n):
                w0, mm = window_for(r * per, (r + 1) * per, m)
                assert w0 <= r * per and (r + 1) * per <= w0 + mm and w0 % mm == 0


def test_leaving_the_window_relayouts_without_local_copies():
    gpus = (0, 1, 2, 3)
    s = store_at(gpus, 2, max_slices=4)  # GPU1 holds [4, 8) in window (4, 4)
    p = s.plan(workloads.tp_groups(gpus, 4))  # GPU1 -> [2, 4): another window, disjoint
    assert p.relayout[1] and p.window[1] == (0, 4) and p.local[1] == []
    assert sorted(x for _, lo, hi in p.fetch[1] for x in range(lo, hi)) == [2, 3]
    assert not p.relayout[0] and p.fetch[0] == []  # GPU0 [0, 4) -> [0, 2): a view


def test_groups_must_cover_store():
    s = store_at((0, 1), 2)
    with pytest.raises(MigrationError):
        s.plan([(0,)])
