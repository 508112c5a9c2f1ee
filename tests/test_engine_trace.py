"""The reference controller's own decisions (captured from its demo run,
tests/golden/engine_trace.json.gz): our planner reproduces each plan's
transfer count and bytes exactly (CPU), and the B200 executes every plan with
the resulting placement verified (GPU)."""

import sys

import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT / "tools"))
import replay_engine as R  # noqa: E402


def test_plans_match_reference_engine():
    doc = R.load_trace()
    prof = doc["profile"]
    assert len(doc["events"]) >= 10
    n_calls = 0
    for e in doc["events"]:
        plan = R.plan_for(e, prof["kv_bytes_per_token_per_head"], prof["total_kv_heads"])
        assert plan.total_bytes == e["total_bytes"]
        assert plan.n_transfers == e["transfers"]
        n_calls += len(e["calls"])
    assert n_calls == 75  # 75 head_transfers calls on demo.yaml


@pytest.mark.gpu
def test_replay_engine_decisions_on_b200():
    from paper_2605_05467_b200.geometry import KvGeometry
    doc = R.load_trace()
    prof = doc["profile"]
    kv = KvGeometry(layers=8, head_dim=128, total_heads=prof["total_kv_heads"])
    rows = R.replay(doc["events"], kv, tuple(range(prof["pool_size"])), reps=1)
    assert all(r["bit_exact_property"] for r in rows)
    assert all(r["bytes"] == r["reference_plan_bytes"] for r in rows)
