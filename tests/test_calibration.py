"""B200 cost-model calibration: the fit recovers known parameters, the
ingress term catches incast (which the reference model ignores,
migration.py:275-281), and the reference switch_cost with calibrated params
reproduces the calibrated prediction."""

import pytest

from paper_2605_05467_b200 import migration as M
from paper_2605_05467_b200.calibration import B200CostModel, fit, from_sweep


def test_fit_recovers_line():
    xs = [1e6, 1e8, 1e9, 4e9, 1.6e10]
    ys = [0.05 + x / 3.2e12 * 1e3 for x in xs]
    a, gbs = fit(xs, ys)
    assert a == pytest.approx(0.05, rel=1e-6) and gbs == pytest.approx(3200, rel=1e-6)


def test_ingress_term_prices_incast():
    # TP8 -> 8xTP1 consolidation onto GPU 0: every source sends 1/8, GPU 0 ingests 7/8
    reqs = tuple((i, 4096) for i in range(64))
    old = [M.KvLayout(tuple(range(8)), 8, 8, reqs)]
    new = [M.KvLayout((0,), 1, 8, reqs)] + [M.KvLayout((g,), 1, 8, ()) for g in range(1, 8)]
    plan = M.plan_repartition(old, new, 16384)
    model = B200CostModel(fixed_ms=0.0, hbm_moved_gbs=3000, link_gbs=770)
    ours = model.predict(plan, "nvlink")
    ref = M.latency_pipelined(plan, M.CostModelParams(copy_bw_gbps=1e12, link_bw_gbps=770,
                                                      per_transfer_overhead_us=1e-6,
                                                      chunk_bytes=1 << 50))
    assert ours == pytest.approx(plan.total_bytes / 770e9 * 1e3)   # 28 GiB into GPU 0
    assert ours == pytest.approx(7 * ref, rel=1e-6)                  # the source-only model is 7x low


def test_reference_switch_cost_reproduces_calibration():
    reqs = tuple((i, 4096) for i in range(16))
    old = [M.KvLayout((0, 1), 2, 8, reqs[::2]), M.KvLayout((2, 3), 2, 8, reqs[1::2])]
    new = M.KvLayout((0, 1, 2, 3), 4, 8, reqs)
    plan = M.plan_repartition(old, new, 16384)
    model = B200CostModel(fixed_ms=0.12, hbm_moved_gbs=3100)
    p = model.cost_params("logical")
    # reference formula with one source = its bytes; logical mode is whole-plan bound,
    # so compare against a single-source view of the same bytes
    single = M.MigrationPlan(transfers=[M.Transfer(0, 1, 0, 0, 1, plan.total_bytes)])
    assert M.switch_cost(M.WARM, single, p) == pytest.approx(model.predict(plan, "logical"), rel=1e-6)


def test_from_sweep_rows():
    rows = [{"mode": "fixed4096", "bytes": b, "device_ms": 0.2 + b / 3.1e12 * 1e3}
            for b in (2**28, 2**30, 2**33, 2**35)]
    m = from_sweep(rows)
    assert m.fixed_ms == pytest.approx(0.2, rel=1e-6) and m.hbm_moved_gbs == pytest.approx(3100, rel=1e-6)
