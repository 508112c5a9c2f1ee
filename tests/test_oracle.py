"""Pin the oracle before trusting it: plan_oracle against the reference's
golden vectors, the C plan-execution restatement against the pure-Python one,
and the numpy pattern mirror against itself (the device fill kernels are
pinned to it in the GPU tests)."""

import numpy as np
import pytest

from oracle import kvmove, plan_oracle as PO
from oracle import weights as W
from paper_2605_05467_b200 import pattern
from paper_2605_05467_b200.geometry import KvGeometry


def test_plan_oracle_matches_reference_ac1(ref_golden):
    for case in ref_golden["ac1"][::7]:
        H = case["H"]
        old = [(tuple(g), H, [tuple(x) for x in r]) for g, r in case["old"]]
        new = [(tuple(g), H, [tuple(x) for x in r]) for g, r in case["new"]]
        moves = PO.plan(old, new, ref_golden["kvb"])
        assert [list(m) for m in moves] == case["transfers"]
        assert PO.replay(old, moves) == PO.placement(new)


def test_plan_oracle_matches_reference_configs(ref_golden):
    for name, c in ref_golden["configs"].items():
        old = [(tuple(g), 8, [tuple(x) for x in r]) for g, r in c["old"]]
        new = [(tuple(g), 8, [tuple(x) for x in r]) for g, r in c["new"]]
        assert [list(m) for m in PO.plan(old, new, c["kvb"])] == c["transfers"], name


def test_cost_oracle_matches_reference(ref_golden):
    for c in ref_golden["costs"][::5]:
        p = c["params"]
        moves = [tuple(t) for t in c["transfers"]]
        assert repr(PO.per_page_ms(moves, p)) == c["per_page"]
        assert repr(PO.aggregate_ms(moves, p)) == c["aggregate"]
        assert repr(PO.pipelined_ms(moves, p)) == c["pipelined"]


def test_weight_gb_oracle(ref_golden):
    w = ref_golden["weights"]
    assert PO.weight_gb("per_tp_copies", 26.0, (1, 2, 4, 8)) == w["per_tp_copies"]
    assert PO.weight_gb("sharded", 26.0, (1, 2, 4, 8), tp=4) == w["sharded_4"]


def _random_cluster(rng, n_gpus, geo, units, n_req):
    pools = [rng.integers(0, 256, units * geo["block_tokens"] * geo["layers"] * 2 * geo["head_dim"]
                          * geo["dtype_bytes"], dtype=np.uint8) for _ in range(n_gpus)]
    H, MB = geo["total_heads"], geo["max_blocks"]
    tables = [np.full(n_req * H * MB, -1, np.int32) for _ in range(n_gpus)]
    rings = [rng.permutation(units).astype(np.int32) for _ in range(n_gpus)]
    return pools, tables, rings, [0] * n_gpus, [units] * n_gpus


@pytest.mark.parametrize("seed", range(4))
def test_c_restatement_matches_python(seed):
    rng = np.random.default_rng(seed)
    geo = dict(layers=2, head_dim=16, dtype_bytes=2, block_tokens=4, total_heads=4, max_blocks=8,
               n_req_slots=6, n_units=96)
    n_gpus = 4
    state = _random_cluster(rng, n_gpus, geo, geo["n_units"], geo["n_req_slots"])
    # admission on TP1 groups, then a TP1 -> TP4 repartition
    ctx = rng.integers(0, 30, size=6)
    adm = [(-1, r % n_gpus, r, 0, 4, int(ctx[r])) for r in range(6)]
    plans = [np.array(adm, np.int64)]
    moves = PO.plan([((g,), 4, [(r, int(ctx[r])) for r in range(6) if r % 4 == g]) for g in range(4)],
                    [((0, 1, 2, 3), 4, [(r, int(ctx[r])) for r in range(6)])], 1)
    plans.append(np.array([(s, d, r, lo, hi, int(ctx[r])) for s, d, r, lo, hi, _ in moves],
                          np.int64).reshape(-1, 6))
    a = ([p.copy() for p in state[0]], [t.copy() for t in state[1]], [r.copy() for r in state[2]],
         list(state[3]), list(state[4]))
    b = ([p.copy() for p in state[0]], [t.copy() for t in state[1]], [r.copy() for r in state[2]],
         list(state[3]), list(state[4]))
    for rec in plans:
        na, sa, ha, ta = kvmove.kv_migrate(geo, a[0], a[1], a[2], a[3], a[4], rec, 2)
        nb, sb, hb, tb = kvmove.kv_migrate_py(geo, b[0], b[1], b[2], b[3], b[4], rec)
        a = (a[0], a[1], a[2], ha, ta)
        b = (b[0], b[1], b[2], hb, tb)
        assert (na, sa, ha, ta) == (nb, sb, hb, tb)
        assert sa == 0
    for x, y in zip(a[0] + a[1] + a[2], b[0] + b[1] + b[2]):
        assert np.array_equal(x, y)


def test_oracle_flags_wrong_source():
    geo = dict(layers=1, head_dim=8, dtype_bytes=2, block_tokens=2, total_heads=2, max_blocks=2,
               n_req_slots=1, n_units=8)
    rng = np.random.default_rng(0)
    pools, tables, rings, h, t = _random_cluster(rng, 2, geo, 8, 1)
    rec = np.array([[1, 0, 0, 0, 1, 3]], np.int64)  # nothing was admitted on gpu 1
    _, status, _, _ = kvmove.kv_migrate(geo, pools, tables, rings, h, t, rec)
    assert status & 1


def test_copy_blocks_strided():
    src = np.arange(4096, dtype=np.uint8)
    dst = np.zeros(4096, np.uint8)
    kvmove.copy_blocks([(dst, 16, src, 32, 10, 48, 128, 64)], 3)
    want = np.zeros(4096, np.uint8)
    for r in range(10):
        want[16 + r * 64: 16 + r * 64 + 48] = src[32 + r * 128: 32 + r * 128 + 48]
    assert np.array_equal(dst, want)


def test_pattern_is_placement_invariant_and_keyed():
    kv = KvGeometry(layers=2, head_dim=32, total_heads=8)
    a = pattern.page_bytes(7, 3, 2, 5, kv, 16)
    b = pattern.page_bytes(7, 3, 2, 5, kv, 16)
    c = pattern.page_bytes(7, 3, 3, 5, kv, 16)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    part = pattern.page_bytes(7, 3, 2, 5, kv, 5)
    assert np.array_equal(part, a[:, : 5 * kv.tok_bytes])


def test_weight_oracle_shards():
    full = np.arange(64, dtype=np.uint16).reshape(8, 8)
    assert np.array_equal(W.expected_shard(full, "col", 4, 1), full[2:4])
    assert np.array_equal(W.expected_shard(full, "row", 2, 1), full[:, 4:])
    f, seen = W.assemble_full([(0, 0, full[:4]), (4, 0, full[4:])], 8, 8)
    assert seen.all() and np.array_equal(f, full)
    with pytest.raises(ValueError):
        W.assemble_full([(0, 0, full[:4]), (2, 0, full[:4])], 8, 8)


@pytest.mark.parametrize("seed", range(6))
def test_c_and_python_oracles_agree_on_error_rules(seed):
    # the K3 error rules (tpr_kernels.cu k3_page): a page with a missing source,
    # an occupied destination, an index outside the table or a poisoned ring slot
    # is not touched, and the ring positions are still consumed
    rng = np.random.default_rng(100 + seed)
    geo = dict(layers=1, head_dim=8, dtype_bytes=2, block_tokens=4, total_heads=4, max_blocks=3,
               n_req_slots=3, n_units=24)
    state = _random_cluster(rng, 3, geo, 24, 3)
    a = [[x.copy() for x in part] if isinstance(part, list) and hasattr(part[0], "copy") else list(part)
         for part in state]
    b = [[x.copy() for x in part] if isinstance(part, list) and hasattr(part[0], "copy") else list(part)
         for part in state]
    statuses = set()
    for _ in range(8):
        n = int(rng.integers(1, 6))
        rec = np.stack([rng.integers(-1, 3, n), rng.integers(-1, 3, n), rng.integers(0, 4, n),
                        rng.integers(0, 3, n), rng.integers(3, 5, n), rng.integers(0, 16, n)], 1)
        rec = rec.astype(np.int64)
        ra = kvmove.kv_migrate(geo, a[0], a[1], a[2], a[3], a[4], rec, 1)
        rb = kvmove.kv_migrate_py(geo, b[0], b[1], b[2], b[3], b[4], rec)
        assert ra == rb
        a[3], a[4] = ra[2], ra[3]
        b[3], b[4] = rb[2], rb[3]
        statuses.add(ra[1])
        for x, y in zip(a[0] + a[1] + a[2], b[0] + b[1] + b[2]):
            assert np.array_equal(x, y)
    assert any(s & 1 for s in statuses) and any(s & 8 for s in statuses)


def test_tables_only_replay_matches_full_replay():
    rng = np.random.default_rng(7)
    geo = dict(layers=1, head_dim=8, dtype_bytes=2, block_tokens=4, total_heads=4, max_blocks=8,
               n_req_slots=4, n_units=64)
    pools, tables, rings, h, t = _random_cluster(rng, 2, geo, 64, 4)
    adm = np.array([(-1, r % 2, r, 0, 4, 5 + 7 * r) for r in range(4)], np.int64)
    mv = np.array([(r % 2, 1 - r % 2, r, 0, 4, 5 + 7 * r) for r in range(4)], np.int64)
    full = kvmove.kv_migrate(geo, pools, tables, rings, h, t, adm)
    t2 = [x.copy() for x in tables]
    r2 = [x.copy() for x in rings]
    want = kvmove.kv_migrate(geo, pools, tables, rings, full[2], full[3], mv)
    got = kvmove.kv_migrate(geo, None, t2, r2, full[2], full[3], mv)
    assert got == want
    for x, y in zip(tables + rings, t2 + r2):
        assert np.array_equal(x, y)
