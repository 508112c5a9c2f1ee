"""Drop-in API parity: paper_2605_05467_b200.migration vs the reference's
tpsim.migration, through the golden vectors the reference produced
(tests/golden/gen_golden.py) and the reference tests' own known answers
(pkg/tests/test_migration.py)."""

import math

import numpy as np
import pytest

from paper_2605_05467_b200 import migration as M


def lay(group, H, reqs):
    return M.KvLayout(group=tuple(group), tp=len(group), total_heads=H,
                      requests=tuple(tuple(r) for r in reqs))


def as_rows(plan):
    return [[t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes]
            for t in plan.transfers]


# -- known answers (test_migration.py:42-107) ---------------------------------

def test_merge_two_tp1_into_tp2():
    plan = M.plan_repartition([lay([1], 8, [(0, 100)]), lay([2], 8, [(1, 100)])],
                              lay([1, 2], 8, [(0, 100), (1, 100)]), 4096)
    moves = {(t.request_id, t.src_gpu, t.dst_gpu, t.head_lo, t.head_hi) for t in plan.transfers}
    assert moves == {(0, 1, 2, 4, 8), (1, 2, 1, 0, 4)}
    assert all(t.bytes == 4 * 100 * 4096 for t in plan.transfers)


def test_merge_two_tp2_into_tp4():
    plan = M.plan_repartition([lay([1, 2], 8, [(0, 10)]), lay([3, 4], 8, [(1, 10)])],
                              lay([1, 2, 3, 4], 8, [(0, 10), (1, 10)]), 4096)
    moves = {(t.request_id, t.src_gpu, t.dst_gpu, t.head_lo, t.head_hi) for t in plan.transfers}
    assert moves == {(0, 1, 2, 2, 4), (0, 2, 3, 4, 6), (0, 2, 4, 6, 8),
                     (1, 3, 1, 0, 2), (1, 3, 2, 2, 4), (1, 4, 3, 4, 6)}


def test_identity_is_empty():
    old = lay([1, 2], 8, [(0, 50)])
    assert M.plan_repartition([old], old, 4096).transfers == []


@pytest.mark.parametrize("call,match", [
    (lambda: M.plan_repartition([lay([1], 8, [(0, 10)])], lay([2], 8, [(0, 10)]), 4096),
     "GPU sets differ"),
    (lambda: M.plan_repartition([lay([1, 2], 8, [(0, 10)])], lay([1, 2], 8, [(0, 20)]), 4096),
     "context length"),
    (lambda: M.KvLayout(group=(1, 2, 3), tp=3, total_heads=8, requests=()), "divisible"),
    (lambda: M.KvLayout(group=(1, 2), tp=3, total_heads=6, requests=()), "group size must equal tp"),
    (lambda: M.plan_repartition([lay([1], 8, [(0, 10)])], lay([1], 4, [(0, 10)]), 4096),
     "share total_heads"),
    (lambda: M.plan_repartition([lay([1], 8, [(0, 10)])], lay([1], 8, [(1, 10)]), 4096),
     "exactly the old requests"),
    (lambda: M.head_transfers(lay([1], 8, []), lay([1], 4, []), 4096), "head counts differ"),
])
def test_error_messages(call, match):
    with pytest.raises(M.MigrationError, match=match):
        call()


def test_apply_plan_detects_wrong_source():
    bad = M.MigrationPlan(transfers=[M.Transfer(9, 1, 0, 0, 4, 1)])
    with pytest.raises(M.MigrationError, match="on 1"):
        M.apply_plan([lay([1], 8, [(0, 10)])], bad)


def test_migration_error_is_value_error():
    assert issubclass(M.MigrationError, ValueError)


# -- golden vectors from the reference -------------------------------------------

def test_ac1_sweep_transfer_lists_identical(ref_golden):
    kvb = ref_golden["kvb"]
    for case in ref_golden["ac1"]:
        H = case["H"]
        old = [lay(g, H, r) for g, r in case["old"]]
        new = [lay(g, H, r) for g, r in case["new"]]
        plan = M.plan_repartition(old, new, kvb)
        assert plan.as_array().tolist() == case["transfers"], (H, case["tp_old"], case["tp_new"])
        assert M.apply_plan(old, plan) == M.layout_placement(new)
    assert len(ref_golden["ac1"]) >= 2000


def test_ac1_lazy_transfers_match_array(ref_golden):
    case = ref_golden["ac1"][123]
    old = [lay(g, case["H"], r) for g, r in case["old"]]
    new = [lay(g, case["H"], r) for g, r in case["new"]]
    plan = M.plan_repartition(old, new, 4096)
    assert as_rows(plan) == case["transfers"]
    assert plan.total_bytes == sum(t[5] for t in case["transfers"])


def test_figures(ref_golden):
    f = ref_golden["figures"]
    assert as_rows(M.plan_repartition([lay([1], 8, [(0, 100)]), lay([2], 8, [(1, 100)])],
                                      lay([1, 2], 8, [(0, 100), (1, 100)]), 4096)) == f["tp1_tp2"]
    assert as_rows(M.plan_repartition([lay([1, 2], 8, [(0, 10)]), lay([3, 4], 8, [(1, 10)])],
                                      lay([1, 2, 3, 4], 8, [(0, 10), (1, 10)]), 4096)) == f["tp2_tp4"]
    assert as_rows(M.plan_repartition([lay([0, 1, 2, 3], 8, [(0, 7)])],
                                      [lay([0, 1], 8, [(0, 7)]), lay([2, 3], 8, [])], 16384)) == f["tp4_tp2"]
    assert as_rows(M.plan_repartition([lay([0, 1], 8, [(0, 3)])], lay([1, 0], 8, [(0, 3)]), 16)) \
        == f["reversed_group"]
    assert as_rows(M.plan_repartition([lay([0], 8, [(5, 0)]), lay([1], 8, [])],
                                      lay([0, 1], 8, [(5, 0)]), 4096)) == f["zero_ctx"]
    assert as_rows(M.plan_repartition([lay([0], 8, [(5, 10), (3, 20)]), lay([1], 8, [(9, 30)])],
                                      lay([0, 1], 8, [(9, 30), (3, 20), (5, 10)]), 4096)) == f["order"]


def test_baseline_config_plans(ref_golden):
    for name, c in ref_golden["configs"].items():
        old = [lay(g, 8, r) for g, r in c["old"]]
        new = [lay(g, 8, r) for g, r in c["new"]]
        plan = M.plan_repartition(old, new, c["kvb"])
        assert plan.as_array().tolist() == c["transfers"], name
        assert plan.total_bytes == c["total_bytes"]
        assert {str(k): v for k, v in plan.bytes_by_source().items()} == c["bytes_by_source"]


def test_engine_disjoint_groups(ref_golden):
    for e in ref_golden["engine"]:
        got = M.head_transfers(lay(e["old"], 8, e["requests"]), lay(e["new"], 8, e["requests"]), 4096)
        assert [[t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes] for t in got] \
            == e["transfers"]


def _params(d):
    return M.CostModelParams(**d)


def test_cost_models_bit_identical(ref_golden):
    for c in ref_golden["costs"]:
        p = _params(c["params"])
        plan = M.MigrationPlan(transfers=[M.Transfer(*t) for t in c["transfers"]])
        assert repr(M.latency_per_page(plan, p)) == c["per_page"]
        assert repr(M.latency_aggregate(plan, p)) == c["aggregate"]
        assert repr(M.latency_pipelined(plan, p)) == c["pipelined"]
        assert repr(M.switch_cost(M.WARM, plan, p)) == c["warm"]
        assert repr(M.switch_cost(M.NAIVE_RELOAD, plan, p)) == c["naive_reload"]
        assert set(plan.predicted_latency_ms) == {"per_page", "aggregate", "pipelined"}


def test_cost_models_on_array_plans(ref_golden):
    # same numbers when the plan holds an SoA array instead of Transfer objects
    for c in ref_golden["costs"][:50]:
        p = _params(c["params"])
        plan = M.MigrationPlan.from_array(np.array(c["transfers"], dtype=np.int64))
        assert repr(M.latency_per_page(plan, p)) == c["per_page"]
        assert repr(M.latency_pipelined(plan, p)) == c["pipelined"]


def test_default_params_calibration(ref_golden):
    d = M.CostModelParams()
    for gb, want in ref_golden["default_costs"].items():
        plan = M.MigrationPlan(transfers=[M.Transfer(1, 2, 0, 0, 1, int(float(gb) * 1e9))])
        got = [M.latency_per_page(plan, d), M.latency_aggregate(plan, d), M.latency_pipelined(plan, d)]
        assert [repr(x) for x in got] == want
        assert 0.4e3 <= got[0] <= 12e3 and 1.8 <= got[2] <= 50.0 and got[0] / got[2] >= 100


def test_pipelined_hand_schedule():
    chunk = 128 * 1024 * 1024
    bw = chunk / 0.002 / 1e9
    p = M.CostModelParams(copy_bw_gbps=bw, link_bw_gbps=bw, per_transfer_overhead_us=1000.0,
                          chunk_bytes=chunk)
    plan = M.MigrationPlan(transfers=[M.Transfer(1, 2, 0, 0, 1, 4 * chunk)])
    assert M.latency_pipelined(plan, p) == pytest.approx(14.0)


def test_switch_modes_and_validation():
    p = M.CostModelParams()
    empty = M.MigrationPlan(transfers=[], handshake_ms=p.handshake_ms)
    assert M.switch_cost(M.WARM, empty, p) == pytest.approx(p.handshake_ms)
    one = M.MigrationPlan(transfers=[M.Transfer(1, 2, 0, 0, 1, int(1e9))])
    assert M.switch_cost(M.NAIVE_RELOAD, one, p) >= 30_000
    assert M.switch_cost(M.NAIVE_KERNEL_INIT, one, p) >= 10_000
    with pytest.raises(M.MigrationError, match="unknown switch mode"):
        M.switch_cost("cold", one, p)
    with pytest.raises(M.MigrationError, match="must be positive"):
        M.CostModelParams(copy_bw_gbps=0.0)
    with pytest.raises(M.MigrationError):
        M.CostModelParams(page_bytes=0)


def test_weight_memory(ref_golden):
    class P:
        weight_full_copy_gb = 26.0
        tp_levels = (1, 2, 4, 8)

    w = ref_golden["weights"]
    assert M.weight_memory("full_copy_per_gpu", P) == w["full_copy_per_gpu"]
    assert M.weight_memory("per_tp_copies", P) == w["per_tp_copies"]
    for t in (1, 2, 4, 8):
        assert M.weight_memory("sharded", P, tp=t) == w[f"sharded_{t}"]
    with pytest.raises(M.MigrationError):
        M.weight_memory("sharded", P)
    with pytest.raises(M.MigrationError):
        M.weight_memory("quantized", P)


def test_reversibility_same_bytes():
    rng = np.random.default_rng(5)
    for _ in range(20):
        ctxs = [(i, int(rng.integers(1, 2000))) for i in range(8)]
        a = [lay([1, 2], 8, ctxs[:4]), lay([3, 4], 8, ctxs[4:])]
        b = lay([1, 2, 3, 4], 8, ctxs)
        assert M.plan_repartition(a, b, 4096).total_bytes == M.plan_repartition([b], a, 4096).total_bytes


def test_plan_is_a_dataclass_like_the_reference():
    import dataclasses
    plan = M.plan_repartition([lay([1], 8, [(0, 10)]), lay([2], 8, [(1, 10)])],
                              lay([1, 2], 8, [(0, 10), (1, 10)]), 4096, handshake_ms=0.5)
    assert [f.name for f in dataclasses.fields(plan)] == ["transfers", "handshake_ms",
                                                          "predicted_latency_ms"]
    d = dataclasses.asdict(plan)
    assert d["handshake_ms"] == 0.5 and len(d["transfers"]) == 2
    q = dataclasses.replace(plan, handshake_ms=1.0)
    assert q.transfers == plan.transfers and q.handshake_ms == 1.0
    assert plan == M.MigrationPlan(list(plan.transfers), 0.5, {})
    for cls in (M.KvLayout, M.Transfer, M.CostModelParams):
        assert dataclasses.is_dataclass(cls)
    # like the reference dataclass: `transfers` is required, an empty plan is truthy
    with pytest.raises(TypeError):
        M.MigrationPlan()
    empty = M.plan_repartition([lay([1], 8, [(0, 10)])], [lay([1], 8, [(0, 10)])], 4096)
    assert empty and empty.n_transfers == 0 and not hasattr(M.MigrationPlan, "__len__")


def test_plan_mutation_keeps_array_in_sync():
    plan = M.plan_repartition([lay([1], 8, [(0, 10)]), lay([2], 8, [(1, 10)])],
                              lay([1, 2], 8, [(0, 10), (1, 10)]), 4096)
    plan.transfers.append(M.Transfer(1, 2, 7, 0, 1, 5))
    assert plan.as_array()[-1].tolist() == [1, 2, 7, 0, 1, 5]
    assert plan.total_bytes == 2 * 4 * 10 * 4096 + 5
    assert math.isclose(M.latency_aggregate(plan, M.CostModelParams()),
                        plan.predicted_latency_ms["aggregate"])
