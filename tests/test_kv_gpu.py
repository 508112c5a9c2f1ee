"""K3 + K1 on B200 vs the oracle (oracle/kvmove.c): pools, block tables and
free rings must be bit-exact after every migration, at oracle-friendly sizes;
at BASELINE sizes through the size-independent property check (every owned
page still carries its placement-invariant pattern, block tables realise
layout_placement)."""

import numpy as np
import pytest
import torch

from oracle import check
from paper_2605_05467_b200 import geometry, migration as M, pattern, workloads
from paper_2605_05467_b200.kvcache import PagedKvCluster

pytestmark = pytest.mark.gpu

TINY = geometry.KvGeometry(layers=2, head_dim=32, total_heads=8)


def make(kv, gpus, units=512, reqs=8, blocks=16, fragmented=True, seed=0):
    c = PagedKvCluster(kv, gpus, units_per_gpu=units, max_requests=reqs, max_blocks=blocks,
                       fragmented=fragmented, seed=seed)
    c.fill_garbage(seed=seed + 100)
    return c


def migrate_and_compare(cluster, plan):
    before = cluster.snapshot()
    rec = cluster.records(plan, validate=False)
    stats = cluster.migrate(plan)
    after = cluster.snapshot()
    want = check.expected_after(cluster, before, rec)
    diff = check.compare(after, want)
    assert want["status"] == 0
    assert int(cluster.status.item()) == 0
    assert not any(diff.values()), diff
    assert stats.units == want["pages"]
    return stats


@pytest.mark.parametrize("tp_old,tp_new", [(a, b) for a in (1, 2, 4, 8) for b in (1, 2, 4, 8) if a != b])
@pytest.mark.parametrize("fragmented", [False, True])
def test_all_transitions_bit_exact(tp_old, tp_new, fragmented):
    gpus = tuple(range(8))
    rng = np.random.default_rng(tp_old * 10 + tp_new)
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 200, size=12))]
    old = workloads.round_robin(workloads.tp_groups(gpus, tp_old), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, tp_new), reqs, 8)
    c = make(TINY, gpus, units=1024, reqs=16, blocks=16, fragmented=fragmented, seed=tp_new)
    c.admit(old, seed=5)
    plan = M.plan_repartition(old, new, TINY.kv_bytes_per_token_per_head)
    stats = migrate_and_compare(c, plan)
    assert stats.bytes == plan.total_bytes
    assert c.placement() == M.layout_placement(new)
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


@pytest.mark.parametrize("H,tp_old,tp_new", [(2, 1, 2), (2, 2, 1), (4, 4, 1), (4, 1, 4), (4, 2, 4),
                                             (16, 8, 2), (16, 1, 8), (16, 4, 8), (16, 8, 1)])
def test_head_counts_bit_exact(H, tp_old, tp_new):
    # the AC-1 head counts (test_migration.py:115-121) beyond Llama's 8
    kv = geometry.KvGeometry(layers=1, head_dim=16, total_heads=H)
    n = max(tp_old, tp_new)
    gpus = tuple(range(10, 10 + n))  # non-zero gpu ids exercise the id -> slot tables
    rng = np.random.default_rng(H * 100 + tp_old * 10 + tp_new)
    reqs = [(int(r), int(c)) for r, c in zip(rng.permutation(1000)[:9], rng.integers(1, 90, size=9))]
    old = workloads.round_robin(workloads.tp_groups(gpus, tp_old), reqs, H)
    new = workloads.round_robin(workloads.tp_groups(gpus, tp_new), reqs, H)
    c = make(kv, gpus, units=1024, reqs=12, blocks=8)
    c.admit(old, seed=6)
    plan = M.plan_repartition(old, new, kv.kv_bytes_per_token_per_head)
    migrate_and_compare(c, plan)
    assert c.placement() == M.layout_placement(new)
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


def test_chain_of_switches_and_back():
    gpus = (0, 1, 2, 3)
    reqs = [(i, 1 + 37 * i) for i in range(10)]  # ragged, incl. 1-token request
    c = make(TINY, gpus, units=512, reqs=16, blocks=32)
    layouts = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 4)}
    c.admit(layouts[1], seed=9)
    seq = [1, 2, 4, 2, 1, 4, 1]
    for a, b in zip(seq, seq[1:]):
        plan = M.plan_repartition(layouts[a], layouts[b], TINY.kv_bytes_per_token_per_head)
        migrate_and_compare(c, plan)
    v = c.verify(seed=9)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    assert v["pages_checked"] == sum(8 * TINY.blocks(ctx) for _, ctx in reqs)


LAUNCH_PATHS = {  # tpr_kv_switch launch variants: all must give the same bytes
    "k31_one_launch": dict(k31=1, k3_fuse_units=1 << 30),
    "k31_dynamic": dict(k31=2, k3_fuse_units=1 << 30),
    "k31_item_share": dict(k31=3, k3_fuse_units=1 << 30),
    "k31_dynamic_rows_for_partial_pages": dict(k31=2, k3_fuse_units=1 << 30, tensor_partial=0),
    "k31_rows_for_partial_pages": dict(k31=1, k3_fuse_units=1 << 30, tensor_partial=0),
    "k31_vector_engine_fallback": dict(k31=1, k3_fuse_units=1 << 30, engine="vector"),
    "fused_k3_tensor": dict(k31=0, k3_fuse_units=1 << 30, tensor_partial=1),
    "fused_k3_rows": dict(k31=0, k3_fuse_units=1 << 30, tensor_partial=0),
    "split_k3_tensor": dict(k3_fuse_units=0, tensor_partial=1),
    "split_k3_rows": dict(k3_fuse_units=0, tensor_partial=0),
}


@pytest.fixture
def launch_path(request):
    from paper_2605_05467_b200 import _native
    saved = {k: _native.get_tuning(k) for k in _native.TUNING_KEYS}
    engine = _native.copy_engine()
    for k, v in LAUNCH_PATHS[request.param].items():
        if k == "engine":
            _native.set_copy_engine(v)
        else:
            _native.set_tuning(k, v)
    yield request.param
    for k, v in saved.items():
        _native.set_tuning(k, v)
    _native.set_copy_engine(engine)


@pytest.mark.parametrize("launch_path", sorted(LAUNCH_PATHS), indirect=True)
def test_launch_paths_bit_exact(launch_path):
    # fused single-CTA K3 vs scan + remap, with and without programmatic
    # dependent launch and zero-copy records: identical pools, tables, rings
    gpus = tuple(range(8))
    rng = np.random.default_rng(77)
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 300, size=40))]
    lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 4, 8)}
    c = make(TINY, gpus, units=4096, reqs=48, blocks=24, fragmented=True, seed=3)
    c.admit(lay[2], seed=8)
    for a, b in ((2, 8), (8, 1), (1, 4), (4, 2)):
        plan = M.plan_repartition(lay[a], lay[b], TINY.kv_bytes_per_token_per_head)
        migrate_and_compare(c, plan)
    v = c.verify(seed=8)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


def test_large_plan_takes_split_k3_and_matches_oracle():
    # > k3_fuse_units units with the default knobs: scan + remap launches
    from paper_2605_05467_b200 import _native
    gpus = (0, 1, 2, 3)
    reqs = [(i, 16 * 40) for i in range(40)]  # 40 blocks x 8 heads x 40 reqs = 12800 units
    lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 4)}
    c = make(TINY, gpus, units=8192, reqs=40, blocks=40, fragmented=True, seed=5)
    c.admit(lay[1], seed=3)
    plan = M.plan_repartition(lay[1], lay[4], TINY.kv_bytes_per_token_per_head)
    stats = migrate_and_compare(c, plan)
    assert stats.units > _native.k3_fuse_units()
    assert _native.kv_switch_launches(stats.units) == 3


@pytest.mark.parametrize("n_reqs", [1, 31, 96, 97, 512, 513, 900])
def test_fused_k3_record_counts_bit_exact(n_reqs):
    # fused K3 (<= k3_fuse_units pages) keeps up to 512 records in shared
    # memory and reads larger plans from global: both sides of the boundary,
    # one-warp blocks included, through the one-call and the two-step path
    from paper_2605_05467_b200 import _native
    gpus = (0, 1)
    reqs = [(i, 16) for i in range(n_reqs)]  # one page per head: TP1 -> TP2 = 1 transfer, 4 pages
    lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2)}
    c = make(TINY, gpus, units=8 * n_reqs + 64, reqs=n_reqs, blocks=1, seed=n_reqs)
    c.admit(lay[1], seed=4)
    plan = M.plan_repartition(lay[1], lay[2], TINY.kv_bytes_per_token_per_head)
    stats = migrate_and_compare(c, plan)
    assert stats.transfers == n_reqs and stats.units <= _native.k3_fuse_units()
    assert _native.kv_switch_launches(stats.units, stats.transfers) == (1 if n_reqs <= 96 else 2)
    before = c.snapshot()
    plan_b, st = c.switch_layouts(lay[2], lay[1])
    want = check.expected_after(c, before, c.records(plan_b, validate=False))
    assert not any(check.compare(c.snapshot(), want).values())
    assert c.placement() == M.layout_placement(lay[1]) and int(c.status.item()) == 0


@pytest.mark.parametrize("tp_old,tp_new", [(16, 1), (1, 16), (4, 16), (16, 2)])
def test_sixteen_slots_bit_exact(tp_old, tp_new):
    # TPR_MAX_GPUS = 16 slots (16 KV heads so TP16 is a valid KvLayout)
    kv = geometry.KvGeometry(layers=1, head_dim=32, total_heads=16)
    gpus = tuple(range(100, 116))
    rng = np.random.default_rng(tp_old * 100 + tp_new)
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 70, size=16))]
    old = workloads.round_robin(workloads.tp_groups(gpus, tp_old), reqs, 16)
    new = workloads.round_robin(workloads.tp_groups(gpus, tp_new), reqs, 16)
    c = make(kv, gpus, units=256, reqs=16, blocks=8, seed=1)
    c.admit(old, seed=2)
    plan, stats = c.switch_layouts(old, new)
    assert np.array_equal(plan.as_array(), M.plan_repartition(old, new, kv.kv_bytes_per_token_per_head).as_array())
    assert c.placement() == M.layout_placement(new)
    v = c.verify(seed=2)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0


def test_one_call_switch_matches_two_step_path():
    # PagedKvCluster.switch_layouts (tpr_kv_switch_layouts) vs plan_repartition
    # + migrate on twin clusters: same plan, same pools / tables / rings
    gpus = tuple(range(8))
    rng = np.random.default_rng(5)
    reqs = [(int(r), int(c)) for r, c in zip(rng.permutation(700)[:30], rng.integers(1, 260, 30))]
    lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 4, 8)}
    a = make(TINY, gpus, units=2048, reqs=32, blocks=20, seed=9)
    b = make(TINY, gpus, units=2048, reqs=32, blocks=20, seed=9)
    a.admit(lay[4], seed=3)
    b.admit(lay[4], seed=3)
    for x, y in ((4, 1), (1, 8), (8, 2), (2, 4)):
        before = a.snapshot()
        plan_a, st_a = a.switch_layouts(lay[x], lay[y])
        plan_b = M.plan_repartition(lay[x], lay[y], TINY.kv_bytes_per_token_per_head)
        st_b = b.migrate(plan_b)
        assert np.array_equal(plan_a.as_array(), plan_b.as_array())
        assert (st_a.units, st_a.bytes, st_a.in_units, st_a.out_units) == \
            (st_b.units, st_b.bytes, st_b.in_units, st_b.out_units)
        sa, sb = a.snapshot(), b.snapshot()
        for k in ("pools", "block_tables", "rings"):
            assert all(np.array_equal(u, v) for u, v in zip(sa[k], sb[k])), k
        assert (sa["ring_head"], sa["ring_tail"]) == (sb["ring_head"], sb["ring_tail"])
        rec = b.records(plan_b, validate=False)
        want = check.expected_after(a, before, rec)
        assert not any(check.compare(sa, want).values())
        assert np.array_equal(a.owner, b.owner)
    assert int(a.status.item()) == 0


def test_one_call_switch_edge_cases():
    gpus = (0, 1, 2, 3)
    reqs = ((1, 0), (2, 16), (3, 5))  # zero-context, one full page, one partial page
    tp2 = workloads.round_robin(workloads.tp_groups(gpus, 2), list(reqs), 8)
    tp4 = workloads.round_robin(workloads.tp_groups(gpus, 4), list(reqs), 8)
    c = make(TINY, gpus, units=64, reqs=4, blocks=4)
    c.admit(tp2, seed=1)
    plan, st = c.switch_layouts(tp2, tp2)  # identity: empty plan, nothing launched
    assert plan.n_transfers == 0 and st.units == 0
    plan, st = c.switch_layouts(tp2, tp4)
    assert plan.total_bytes == M.plan_repartition(tp2, tp4, TINY.kv_bytes_per_token_per_head).total_bytes
    assert c.placement() == M.layout_placement(tp4)
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0


def test_one_call_switch_raises_reference_errors():
    gpus = (0, 1, 2, 3)
    reqs = [(1, 50), (2, 70)]
    c = make(TINY, gpus, units=64, reqs=4, blocks=8)
    tp2 = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, 8)
    c.admit(tp2, seed=1)
    snap = c.snapshot()
    with pytest.raises(M.MigrationError, match="GPU sets differ"):
        c.switch_layouts(tp2, [M.KvLayout((0, 1), 2, 8, tuple(reqs))])
    with pytest.raises(M.MigrationError, match="context length changed"):
        c.switch_layouts(tp2, [M.KvLayout(gpus, 4, 8, ((1, 50), (2, 71)))])
    onto0 = [M.KvLayout((0,), 1, 8, tuple(reqs))] + [M.KvLayout((g,), 1, 8, ()) for g in gpus[1:]]
    with pytest.raises(M.MigrationError, match="KV units needed"):
        c.switch_layouts(tp2, onto0)  # GPU0 needs 56 units, 48 are free
    after = c.snapshot()
    for k in ("pools", "block_tables", "rings"):  # failed switches changed nothing
        assert all(np.array_equal(u, v) for u, v in zip(snap[k], after[k])), k
    assert (snap["ring_head"], snap["ring_tail"]) == (after["ring_head"], after["ring_tail"])


def test_engine_path_disjoint_groups():
    # prefill->decode handoff style: head_transfers between disjoint groups
    gpus = (0, 1, 2, 3, 4, 5)
    c = make(TINY, gpus)
    old = M.KvLayout((0, 1), 2, 8, ((3, 70), (4, 16)))
    c.admit([old], seed=2)
    new = M.KvLayout((2, 3, 4, 5), 4, 8, ((3, 70), (4, 16)))
    plan = M.head_transfers_array(old, new, TINY.kv_bytes_per_token_per_head)
    migrate_and_compare(c, plan)
    assert c.placement() == M.layout_placement(new)


def test_release_then_readmit_bit_exact():
    gpus = (0, 1, 2, 3)
    reqs = [(i, 3 + 41 * i) for i in range(8)]
    c = make(TINY, gpus, units=256, reqs=8, blocks=32)
    tp2 = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, 8)
    c.admit(tp2, seed=4)
    free0 = [c.free_units(g) for g in gpus]
    before = c.snapshot()
    gone = [1, 4, 6]
    rec = np.array([(int(c.owner[c.req_slot[r], h0]), -1, c.req_slot[r], h0, h0 + 4,
                     c.ctx_of[r]) for r in gone for h0 in (0, 4)], np.int64)
    n = c.release(gone)
    want = check.expected_after(c, before, rec)
    diff = check.compare(c.snapshot(), want)
    assert not any(diff.values()), diff
    assert n == sum(8 * TINY.blocks(ctx) for r, ctx in reqs if r in gone)
    assert sum(c.free_units(g) for g in gpus) == sum(free0) + n
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    # the freed pages are reused by a new request
    c.admit([M.KvLayout((0, 1, 2, 3), 4, 8, ((100, 300),))], seed=4)
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


def test_c_oracle_matches_python_oracle():
    gpus = (0, 1)
    c = make(TINY, gpus, units=128, reqs=4, blocks=8)
    old = workloads.round_robin([(0,), (1,)], [(0, 33), (1, 17), (2, 64)], 8)
    new = workloads.round_robin([(0, 1)], [(0, 33), (1, 17), (2, 64)], 8)
    c.admit(old, seed=1)
    before = c.snapshot()
    rec = c.records(M.plan_repartition(old, new, TINY.kv_bytes_per_token_per_head))
    a = check.expected_after(c, before, rec, impl="c")
    b = check.expected_after(c, before, rec, impl="py")
    assert not any(check.compare(a, b).values())


def test_device_fill_matches_numpy_pattern():
    c = make(TINY, (0, 1), units=64, reqs=4, blocks=8)
    c.admit([M.KvLayout((0, 1), 2, 8, ((0, 37),))], seed=21)
    snap = c.snapshot()
    pools = snap["pools"]
    bts = [b.reshape(4, 8, 8) for b in snap["block_tables"]]
    rs = c.req_slot[0]
    for h in range(8):
        g = 0 if h < 4 else 1
        for b in range(TINY.blocks(37)):
            unit = int(bts[g][rs, h, b])
            ntok = min(16, 37 - 16 * b)
            page = pools[g][unit * TINY.unit_bytes:(unit + 1) * TINY.unit_bytes]
            page = page.reshape(2 * TINY.layers, TINY.plane_bytes)[:, : ntok * TINY.tok_bytes]
            assert np.array_equal(page, pattern.page_bytes(21, rs, h, b, TINY, ntok))
    # garbage fill of a free unit is keyed by (slot, unit)
    free_unit = int(snap["rings"][1][snap["ring_head"][1] % c.n_units])
    got = pools[1][free_unit * TINY.unit_bytes:(free_unit + 1) * TINY.unit_bytes]
    assert np.array_equal(got, pattern.unit_garbage(100, 1, free_unit, TINY.unit_bytes))


def test_wrong_source_rejected_on_host():
    c = make(TINY, (0, 1))
    c.admit([M.KvLayout((0,), 1, 8, ((0, 10),))], seed=1)
    bad = M.MigrationPlan(transfers=[M.Transfer(1, 0, 0, 0, 4, 4 * 10 * TINY.kv_bytes_per_token_per_head)])
    with pytest.raises(M.MigrationError, match="but it is on 0"):
        c.migrate(bad)


def test_wrong_source_flagged_on_device_without_host_validation():
    c = make(TINY, (0, 1))
    c.admit([M.KvLayout((0,), 1, 8, ((0, 10),))], seed=1)
    bad = M.MigrationPlan(transfers=[M.Transfer(1, 0, 0, 0, 4, 4 * 10 * TINY.kv_bytes_per_token_per_head)])
    c.migrate(bad, validate=False)
    torch.cuda.synchronize()
    assert int(c.status.item()) & 1


def test_status_mirror_reports_device_errors():
    # the one-call switch mirrors K3's status word into pinned host memory; a
    # synchronous executor reads it from there (fused K3 store or D2H)
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    for fuse in (1 << 30, 0):
        from paper_2605_05467_b200 import _native
        saved = _native.get_tuning("k3_fuse_units")
        _native.set_tuning("k3_fuse_units", fuse)
        try:
            c = make(TINY, (0, 1))
            c.admit([M.KvLayout((0,), 1, 8, ((0, 10),))], seed=1)
            ex = ReconfigurationExecutor(c)
            ok = ex.switch([M.KvLayout((0,), 1, 8, ((0, 10),)), M.KvLayout((1,), 1, 8, ())],
                           [M.KvLayout((0, 1), 2, 8, ((0, 10),))], validate=False)
            assert ok.status == 0 and c.status_mirrored
            # claim every head sits on GPU 1 (heads 0-3 are on GPU 0): K3 flags the
            # missing sources and the occupied destinations on the device
            lie = [M.KvLayout((1,), 1, 8, ((0, 10),)), M.KvLayout((0,), 1, 8, ())]
            bad = ex.switch(lie, [M.KvLayout((0, 1), 2, 8, ((0, 10),))], validate=False)
            assert c.status_mirrored
            assert bad.status & _native.TPR_STATUS_WRONG_SOURCE, bad.status
            assert bad.status & _native.TPR_STATUS_DST_OCCUPIED, bad.status
        finally:
            _native.set_tuning("k3_fuse_units", saved)


def test_capacity_error():
    c = make(TINY, (0, 1), units=16, reqs=4, blocks=8)
    c.admit([M.KvLayout((0,), 1, 8, ((0, 16),))], seed=1)  # 8 units on gpu 0
    c.admit([M.KvLayout((1,), 1, 8, ((1, 16),))], seed=1)  # 8 units on gpu 1
    with pytest.raises(M.MigrationError, match="units needed"):
        c.admit([M.KvLayout((1,), 1, 8, ((2, 64),))], seed=1)  # 32 more units


def test_empty_plan_is_a_noop():
    c = make(TINY, (0, 1))
    lay = M.KvLayout((0, 1), 2, 8, ((0, 5),))
    c.admit([lay], seed=1)
    s = c.migrate(M.plan_repartition([lay], lay, TINY.kv_bytes_per_token_per_head))
    assert s.units == 0 and s.bytes == 0


def test_zero_context_request_moves_nothing():
    c = make(TINY, (0, 1))
    old = [M.KvLayout((0,), 1, 8, ((5, 0),)), M.KvLayout((1,), 1, 8, ())]
    new = M.KvLayout((0, 1), 2, 8, ((5, 0),))
    c.admit(old, seed=1)
    plan = M.plan_repartition(old, new, TINY.kv_bytes_per_token_per_head)
    assert plan.n_transfers == 1 and plan.total_bytes == 0
    migrate_and_compare(c, plan)


@pytest.mark.slow
def test_cfg1_full_size_bit_exact():
    w = workloads.config(0)
    kv = w.model.kv
    c = make(kv, w.gpus, units=1024, reqs=4, blocks=32)
    c.admit(w.old, seed=3)
    plan = M.plan_repartition(w.old, w.new, kv.kv_bytes_per_token_per_head)
    assert plan.total_bytes == 128 * 2**20
    migrate_and_compare(c, plan)
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


@pytest.mark.parametrize("model", ["8b", "70b"])
@pytest.mark.parametrize("tensor_partial", [0, 1])
def test_llama_geometry_ragged_bit_exact(model, tensor_partial):
    # real page geometry (8B: 64 planes = one 16 KiB tensor box per token;
    # 70B: 160 planes = two 20 KiB boxes per token) with partial last pages,
    # tensor boxes vs row copies, against the C oracle
    from paper_2605_05467_b200 import _native
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B, LLAMA_3_1_70B
    kv = (LLAMA_3_1_8B if model == "8b" else LLAMA_3_1_70B).kv
    saved = _native.get_tuning("tensor_partial")
    _native.set_tuning("tensor_partial", tensor_partial)
    try:
        gpus = (0, 1, 2, 3)
        reqs = [(0, 1), (1, 17), (2, 47), (3, 64), (4, 95)]  # 1 token .. 15 valid tokens
        lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 4)}
        c = make(kv, gpus, units=96, reqs=6, blocks=6, fragmented=True, seed=4)
        c.admit(lay[1], seed=6)
        for a, b in ((1, 4), (4, 2), (2, 1)):
            plan = M.plan_repartition(lay[a], lay[b], kv.kv_bytes_per_token_per_head)
            migrate_and_compare(c, plan)
        v = c.verify(seed=6)
        assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    finally:
        _native.set_tuning("tensor_partial", saved)


@pytest.mark.slow
def test_cfg4_70b_32k_full_size_property():
    # BASELINE configs[3]: Llama-3.1-70B TP4 <-> TP8, 8 x 32768 tokens, 640 KiB pages;
    # the largest single-B200 case (70 GiB moved per direction)
    import bench
    w = workloads.config(3)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=bench.capacity_units(w, kv), max_requests=8,
                       max_blocks=kv.blocks(32768), fragmented=True, seed=2)
    c.admit(w.old, seed=8)
    for a, b in ((w.old, w.new), (w.new, w.old)):
        plan = M.plan_repartition(a, b, kv.kv_bytes_per_token_per_head)
        assert plan.total_bytes == 70 * 2**30
        c.migrate(plan)
        v = c.verify()
        assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
        assert v["pages_checked"] == 8 * 8 * 2048
        assert c.placement() == M.layout_placement(b)


@pytest.mark.slow
def test_cfg2_full_size_property():
    w = workloads.config(1, weights=False)
    kv = w.model.kv
    # GPU1 keeps 4 heads x 32 requests and receives heads 2-3 of all 64 before
    # releasing: 2 x 32768 pages at peak
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=65536 + 64, max_requests=64, max_blocks=256,
                       fragmented=True, seed=1)
    c.admit(w.old, seed=4)
    plan = M.plan_repartition(w.old, w.new, kv.kv_bytes_per_token_per_head)
    assert plan.total_bytes == 24 * 2**30
    s = c.migrate(plan)
    assert s.bytes == plan.total_bytes
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
    assert v["pages_checked"] == 64 * 8 * 256
    assert c.placement() == M.layout_placement(w.new)


@pytest.fixture(params=[3, 2], ids=["item_share", "dynamic"])
def k31_variant(request):
    from paper_2605_05467_b200 import _native
    saved = _native.get_tuning("k31")
    _native.set_tuning("k31", request.param)
    yield request.param
    _native.set_tuning("k31", saved)


@pytest.mark.parametrize("model", ["tiny", "8b", "70b"])
@pytest.mark.parametrize("tp_old,tp_new", [(1, 2), (2, 1), (1, 8), (8, 1), (4, 8), (8, 2)])
def test_k31_single_launch_bit_exact(model, tp_old, tp_new, k31_variant):
    # small plans (<= 96 transfers, <= k3_fuse_units pages): the whole switch is
    # one launch (K31), with ragged contexts (partial pages as TMA tensor boxes:
    # 64 planes per box on 8B pages, 80 on 70B pages) and 8 slots, against the
    # oracle
    from paper_2605_05467_b200 import _native
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B, LLAMA_3_1_70B
    kv = {"tiny": TINY, "8b": LLAMA_3_1_8B.kv, "70b": LLAMA_3_1_70B.kv}[model]
    gpus = tuple(range(8))
    rng = np.random.default_rng(tp_old * 31 + tp_new)
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 300, size=6))]
    old = workloads.round_robin(workloads.tp_groups(gpus, tp_old), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, tp_new), reqs, 8)
    units = 400 if model == "70b" else 1024  # 640 KiB pages: keep the host snapshots small
    c = make(kv, gpus, units=units, reqs=8, blocks=20, fragmented=True, seed=tp_new)
    c.admit(old, seed=5)
    for a, b in ((old, new), (new, old)):
        before = c.snapshot()
        plan = M.plan_repartition(a, b, kv.kv_bytes_per_token_per_head)
        rec = c.records(plan, validate=False)
        got, st = c.switch_layouts(a, b)
        assert _native.kv_switch_launches(st.units, st.transfers) == 1
        want = check.expected_after(c, before, rec)
        diff = check.compare(c.snapshot(), want)
        assert not any(diff.values()), diff
        assert int(c.status.item()) == 0 and c.status_host[0] == 0
    v = c.verify(seed=5)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


def test_k31_reports_errors_per_call(k31_variant):
    # K31's status word is this call's bits only, also in the pinned mirror
    from paper_2605_05467_b200.controller import ReconfigurationExecutor
    c = make(TINY, (0, 1))
    c.admit([M.KvLayout((0,), 1, 8, ((0, 10),))], seed=1)
    # request 7 is admitted first: the bad switch below "releases" units GPU1
    # never held, and the poisoned ring slots it pushes then land on positions
    # request 7's pages were already popped from (a full ring would have them
    # overwrite free slots -- a corrupted state that later pops report)
    c.admit([M.KvLayout((0, 1), 2, 8, ((7, 33),))], seed=1)
    ex = ReconfigurationExecutor(c)
    lie = [M.KvLayout((1,), 1, 8, ((0, 10),)), M.KvLayout((0,), 1, 8, ())]
    bad = ex.switch(lie, [M.KvLayout((0, 1), 2, 8, ((0, 10),))], validate=False)
    assert bad.status & 1 and bad.status & 2
    # a correct switch of the other request reports a clean word
    ok = ex.switch([M.KvLayout((0, 1), 2, 8, ((7, 33),))],
                   [M.KvLayout((1, 0), 2, 8, ((7, 33),))], validate=False)
    assert ok.status == 0 and int(c.status.item()) == 0


def test_host_record_offsets_equal_the_device_scan():
    # K31 takes K3's keyed scans from the host (tpr_record_offsets); the split
    # K3 writes the same rows to d_meta on the device: they must agree
    import ctypes
    from paper_2605_05467_b200 import _native
    gpus = tuple(range(8))
    rng = np.random.default_rng(5)
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 400, size=40))]
    old = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, 8), reqs, 8)
    c = make(TINY, gpus, units=4096, reqs=48, blocks=32, fragmented=True, seed=2)
    c.admit(old, seed=3)
    plan = M.plan_repartition(old, new, TINY.kv_bytes_per_token_per_head)
    rec = c.records(plan, validate=False).astype(np.int32)
    saved = {k: _native.get_tuning(k) for k in ("k31", "k3_fuse_units")}
    try:
        _native.set_tuning("k31", 0)
        _native.set_tuning("k3_fuse_units", 0)
        c.migrate(plan)
        torch.cuda.synchronize()
    finally:
        for k, v in saved.items():
            _native.set_tuning(k, v)
    n = len(rec)
    dev = c._meta.t[: n * 4].cpu().numpy().reshape(n, 4)
    host = np.zeros((n, 4), np.int64)
    _native.call("tpr_record_offsets", rec.ctypes.data, n, -1, TINY.block_tokens,
                 host.ctypes.data, None)
    assert np.array_equal(dev, host)


@pytest.mark.parametrize("pages", [504, 508, 512, 516])
def test_k31_schedule_boundary_bit_exact(pages):
    # the auto K31 schedule switches from item shares to the dynamic one at
    # 512 pages: plans on both sides, ragged contexts, the one-call path
    from paper_2605_05467_b200 import _native
    assert _native.get_tuning("k31") == 1
    gpus = (0, 1)
    # TP1 -> TP2 moves 4 heads of every request: pages = 4 * sum(blocks)
    blocks = pages // 4
    ctxs = [16 * 9] * (blocks // 9) + ([16 * (blocks % 9) - 3] if blocks % 9 else [])
    reqs = [(i, c) for i, c in enumerate(ctxs)]
    lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2)}
    c = make(TINY, gpus, units=16 * pages, reqs=len(reqs), blocks=16, seed=pages)
    c.admit(lay[1], seed=6)
    for a, b in ((1, 2), (2, 1)):
        before = c.snapshot()
        plan = M.plan_repartition(lay[a], lay[b], TINY.kv_bytes_per_token_per_head)
        rec = c.records(plan, validate=False)
        got, st = c.switch_layouts(lay[a], lay[b])
        assert st.units == pages and _native.kv_switch_launches(st.units, st.transfers) == 1
        want = check.expected_after(c, before, rec)
        assert not any(check.compare(c.snapshot(), want).values())
    v = c.verify(seed=6)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
