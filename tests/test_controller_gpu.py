"""The execution hook end to end on B200: switch (KV + weights on two
streams), prefill->decode handoff over disjoint groups, capacity admission
with eviction through release."""

import numpy as np
import pytest

from oracle import check
from paper_2605_05467_b200 import geometry, migration as M, workloads
from paper_2605_05467_b200.controller import ReconfigurationExecutor, measured_switch_cost
from paper_2605_05467_b200.kvcache import PagedKvCluster
from paper_2605_05467_b200.placement import BEST_EFFORT, FEASIBLE, Arrival, enforce_kv_capacity
from paper_2605_05467_b200.weights import ShardedWeightStore

pytestmark = pytest.mark.gpu

MODEL = geometry.tiny_geometry()
KV = MODEL.kv


def test_switch_sequence_kv_and_weights():
    gpus = tuple(range(8))
    reqs = [(i, 7 + 13 * i) for i in range(16)]
    lays = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 4, 8)}
    kv = PagedKvCluster(KV, gpus, units_per_gpu=1024, max_requests=16, max_blocks=16, fragmented=True)
    kv.admit(lays[8], seed=3)
    store = ShardedWeightStore(MODEL, gpus)
    store.load(workloads.tp_groups(gpus, 8))
    ex = ReconfigurationExecutor(kv, store, time_kernels=True)
    seq = [8, 4, 2, 1, 2, 8, 1, 4]
    for a, b in zip(seq, seq[1:]):
        before = kv.snapshot()
        plan = M.plan_repartition(lays[a], lays[b], KV.kv_bytes_per_token_per_head)
        rec = kv.records(plan, validate=False)
        res = ex.switch(lays[a], lays[b], new_weight_groups=workloads.tp_groups(gpus, b))
        assert res.status == 0 and res.device_ms > 0 and res.host_ms > 0
        assert res.kv.bytes == plan.total_bytes
        diff = check.compare(kv.snapshot(), check.expected_after(kv, before, rec))
        assert not any(diff.values()), (a, b, diff)
        assert store.verify() == 0
    assert kv.placement() == M.layout_placement(lays[4])


def test_prefill_decode_handoff():
    gpus = (0, 1, 2, 3, 4, 5)
    kv = PagedKvCluster(KV, gpus, units_per_gpu=256, max_requests=8, max_blocks=16)
    ex = ReconfigurationExecutor(kv)
    prefill = M.KvLayout((0, 1), 2, 8, ((1, 100), (2, 33)))
    kv.admit([prefill], seed=8)
    decode = M.KvLayout((2, 3, 4, 5), 4, 8, ((1, 100), (2, 33)))
    res = ex.handoff(prefill, decode)
    assert res.status == 0
    assert res.kv.bytes == 8 * (100 + 33) * KV.kv_bytes_per_token_per_head  # every head moves
    assert kv.placement() == M.layout_placement(decode)
    v = kv.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


@pytest.mark.parametrize("src,dst", [((0, 1), (2, 3, 4, 5)), ((2,), (3,)), ((0, 1, 2, 3), (4, 5)),
                                     ((4, 5), (5, 4))])
def test_handoff_one_call_matches_two_step(src, dst):
    # head_transfers + K3 + K1 in one native call vs head_transfers_array +
    # migrate, on twin clusters: same plan and identical pools / tables / rings
    import numpy as np
    gpus = (0, 1, 2, 3, 4, 5)
    reqs = ((1, 100), (2, 33), (3, 16))
    pre = M.KvLayout(src, len(src), 8, reqs)
    dec = M.KvLayout(dst, len(dst), 8, reqs)
    a = PagedKvCluster(KV, gpus, units_per_gpu=256, max_requests=8, max_blocks=16, fragmented=True)
    b = PagedKvCluster(KV, gpus, units_per_gpu=256, max_requests=8, max_blocks=16, fragmented=True)
    for c in (a, b):
        c.fill_garbage(seed=5)
        c.admit([pre], seed=8)
    plan_a, st_a = a.switch_layouts(pre, dec, planner="head_transfers")
    plan_b = M.head_transfers_array(pre, dec, KV.kv_bytes_per_token_per_head)
    st_b = b.migrate(plan_b)
    assert np.array_equal(plan_a.as_array(), plan_b.as_array())
    assert (st_a.units, st_a.bytes) == (st_b.units, st_b.bytes)
    sa, sb = a.snapshot(), b.snapshot()
    for k in ("pools", "block_tables", "rings"):
        assert all(np.array_equal(u, v) for u, v in zip(sa[k], sb[k])), k
    assert a.placement() == M.layout_placement(dec) == b.placement()


def test_switch_with_reuse_order_moves_less_and_stays_exact():
    # TP4 -> TP8 re-ranked keeps half the KV in place (vs 1/8)
    gpus = tuple(range(8))
    reqs = [(i, 5 + 11 * i) for i in range(16)]
    tp4 = workloads.round_robin(workloads.tp_groups(gpus, 4), reqs, 8)
    tp8 = workloads.round_robin(workloads.tp_groups(gpus, 8), reqs, 8)
    kv = PagedKvCluster(KV, gpus, units_per_gpu=1024, max_requests=16, max_blocks=16, fragmented=True)
    kv.admit(tp4, seed=3)
    store = ShardedWeightStore(MODEL, gpus)
    store.load(workloads.tp_groups(gpus, 4))
    ex = ReconfigurationExecutor(kv, store)
    canonical = M.plan_repartition(tp4, tp8, KV.kv_bytes_per_token_per_head)
    res = ex.switch(tp4, tp8, new_weight_groups=workloads.tp_groups(gpus, 8), reuse_order=True)
    assert res.status == 0
    assert res.kv.bytes < canonical.total_bytes
    new = res.new_layouts
    assert sorted(r for lay in new for r, _ in lay.requests) == sorted(r for r, _ in reqs)
    assert kv.placement() == M.layout_placement(new)
    v = kv.verify(seed=3)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    assert store.verify() == 0
    back = ex.switch(new, tp4, new_weight_groups=workloads.tp_groups(gpus, 4))  # and back
    assert back.status == 0 and kv.placement() == M.layout_placement(tp4)
    store.finish()


def test_capacity_admission_evicts_best_effort():
    gpus = (0, 1, 2, 3)
    kv = PagedKvCluster(KV, gpus, units_per_gpu={0: 128, 1: 128, 2: 64, 3: 64}, max_requests=8,
                        max_blocks=8)
    src = M.KvLayout((0, 1), 2, 8, ((1, 128), (2, 128), (3, 64)))
    kv.admit([src], seed=2)  # 4 heads x (8 + 8 + 4) pages = 80 per GPU of (0, 1)
    dst = M.KvLayout((2, 3), 2, 8, ())
    arrivals = [Arrival(1, 128, BEST_EFFORT, 1.0), Arrival(2, 128, FEASIBLE, 2.0),
                Arrival(3, 64, BEST_EFFORT, 0.5)]
    kept, evicted = enforce_kv_capacity(kv, dst, arrivals)
    # each GPU of (2,3) has 64 free pages; request 2 (feasible) takes 32, then 3 (oldest
    # best-effort) takes 16, request 1 (32 more) no longer fits
    assert [a.request_id for a in kept] == [2, 3]
    assert [a.request_id for a in evicted] == [1]
    kv.release([a.request_id for a in evicted])
    ids = tuple((a.request_id, a.context_len) for a in kept)
    old = M.KvLayout((0, 1), 2, 8, ids)
    new = M.KvLayout((2, 3), 2, 8, ids)
    plan = M.head_transfers_array(old, new, KV.kv_bytes_per_token_per_head)
    kv.migrate(plan)
    v = kv.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    assert kv.free_units(0) == kv.free_units(1) == 128
    assert kv.free_units(2) == kv.free_units(3) == 64 - 48


def test_measured_switch_cost_adapter():
    gpus = (0, 1)
    kv = PagedKvCluster(KV, gpus, units_per_gpu=128, max_requests=4, max_blocks=8)
    ex = ReconfigurationExecutor(kv)
    old = [M.KvLayout((0,), 1, 8, ((0, 50),)), M.KvLayout((1,), 1, 8, ((1, 50),))]
    new = M.KvLayout((0, 1), 2, 8, ((0, 50), (1, 50)))
    kv.admit(old, seed=1)
    cost = measured_switch_cost(ex)
    params = M.CostModelParams()
    ms = cost(M.WARM, M.plan_repartition(old, new, KV.kv_bytes_per_token_per_head), params)
    assert ms > params.handshake_ms
    assert kv.placement() == M.layout_placement(new)
    # the naive modes add the reference's fixed reload / kernel-init cost
    back = M.plan_repartition([new], old, KV.kv_bytes_per_token_per_head)
    assert cost(M.NAIVE_RELOAD, back, params) > params.reload_ms
    assert kv.placement() == M.layout_placement(old)
    with pytest.raises(M.MigrationError, match="unknown switch mode"):
        cost("bogus", back, params)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("TPR_FUZZ_SEEDS", "3"))))
def test_random_switch_walk_kv_and_weights(seed):
    # the executor between random partitions of 8 GPUs (mixed TP degrees,
    # random rank order), requests redistributed at random, KV and weights in
    # one switch, one or two streams: KV bit-exact vs the oracle replay,
    # weights verified, placement = layout_placement(new)
    import numpy as np
    from test_weights_gpu import check_against_oracle, host_pieces
    rng = np.random.default_rng(seed)
    gpus = tuple(range(8))
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 90, size=20))]

    def random_layouts():
        perm = [int(g) for g in rng.permutation(gpus)]
        groups, i = [], 0
        while i < 8:
            s = int(rng.choice([x for x in (1, 2, 4, 8) if i + x <= 8]))
            groups.append(tuple(perm[i:i + s]))
            i += s
        per = [[] for _ in groups]
        for r in reqs:
            per[int(rng.integers(len(groups)))].append(r)
        return groups, [M.KvLayout(g, len(g), 8, tuple(p)) for g, p in zip(groups, per)]

    groups, cur = random_layouts()
    kv = PagedKvCluster(KV, gpus, units_per_gpu=1024, max_requests=20, max_blocks=16, fragmented=True,
                        seed=seed)
    kv.admit(cur, seed=3)
    store = ShardedWeightStore(MODEL, gpus)
    store.load(groups)
    ex = ReconfigurationExecutor(kv, store, overlap=bool(seed % 2))
    for step in range(10):
        groups, new = random_layouts()
        before = kv.snapshot()
        pieces = host_pieces(store)
        plan = M.plan_repartition(cur, new, KV.kv_bytes_per_token_per_head)
        rec = kv.records(plan, validate=False)
        res = ex.switch(cur, new, new_weight_groups=groups, trim=bool(rng.integers(2)))
        assert res.status == 0 and res.kv.bytes == plan.total_bytes, step
        diff = check.compare(kv.snapshot(), check.expected_after(kv, before, rec))
        assert not any(diff.values()), (step, diff)
        check_against_oracle(store, pieces, groups)
        assert store.verify() == 0 and kv.placement() == M.layout_placement(new)
        cur = new


@pytest.fixture(params=[0, 2, 3], ids=["k3_then_k1", "k31_dynamic", "k31_item_share"])
def k31_mode(request):
    from paper_2605_05467_b200 import _native
    saved = _native.get_tuning("k31")
    _native.set_tuning("k31", request.param)
    yield request.param
    _native.set_tuning("k31", saved)


def test_switch_evicts_inside_the_native_call(k31_mode):
    # engine.py:600-601 + 623-645 executed: the destination group's byte budget
    # keeps the feasible arrival and the oldest best-effort one; the other
    # best-effort arrival is evicted, and its pages are freed by the same
    # native call (release records after the plan's), bit-exact vs the oracle
    # -- through K3 + K1 and through both K31 schedules
    from oracle import check
    from paper_2605_05467_b200.placement import KvBudget
    gpus = (0, 1, 2, 3)
    kv = PagedKvCluster(KV, gpus, units_per_gpu=256, max_requests=8, max_blocks=8, fragmented=True,
                        seed=4)
    kv.fill_garbage(seed=9)
    reqs = ((1, 128), (2, 128), (3, 64))
    old = [M.KvLayout((0, 1), 2, 8, reqs), M.KvLayout((2, 3), 2, 8, ())]
    new = [M.KvLayout((2, 3), 2, 8, reqs), M.KvLayout((0, 1), 2, 8, ())]
    kv.admit(old, seed=2)
    kv.admit([M.KvLayout((2, 3), 2, 8, ((9, 40),))], seed=2)  # already running on (2, 3)
    per_tok = KV.kv_bytes_per_token_per_head * 8
    # room for request 9 (running) + 2 (feasible) + 3 (oldest best effort) + 10 tokens
    budget = KvBudget(26.0 + (40 + 128 + 64 + 10) * per_tok / 2 / 1e9, 26.0)
    arrivals = [Arrival(1, 128, BEST_EFFORT, 1.0), Arrival(2, 128, FEASIBLE, 2.0),
                Arrival(3, 64, BEST_EFFORT, 0.5)]
    new_all = [M.KvLayout((2, 3), 2, 8, reqs + ((9, 40),)), M.KvLayout((0, 1), 2, 8, ())]
    old_all = old[:1] + [M.KvLayout((2, 3), 2, 8, ((9, 40),))]
    kept_old = [M.KvLayout((0, 1), 2, 8, ((2, 128), (3, 64))), M.KvLayout((2, 3), 2, 8, ((9, 40),))]
    kept_new = [M.KvLayout((2, 3), 2, 8, ((2, 128), (3, 64), (9, 40))), M.KvLayout((0, 1), 2, 8, ())]
    plan = M.plan_repartition(kept_old, kept_new, KV.kv_bytes_per_token_per_head)
    rs1 = kv.req_slot[1]
    rec = np.concatenate([kv.records(plan), np.array([(0, -1, rs1, 0, 4, 128),
                                                      (1, -1, rs1, 4, 8, 128)], np.int64)])
    free0 = [kv.free_units(g) for g in gpus]
    before = kv.snapshot()
    ex = ReconfigurationExecutor(kv)
    res = ex.switch(old_all, new_all, arrivals=arrivals, kv_budget=budget)
    assert res.evicted == [1] and res.status == 0
    assert np.array_equal(res.plan.as_array(), plan.as_array())
    want = check.expected_after(kv, before, rec)
    assert not any(check.compare(kv.snapshot(), want).values())
    assert kv.placement() == M.layout_placement(kept_new) and 1 not in kv.req_slot
    # GPUs 0 and 1 got back every page they held (request 1 released, 2 and 3 moved)
    assert [kv.free_units(g) for g in gpus][:2] == [free0[0] + 80, free0[1] + 80]
    v = kv.verify(seed=2)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    # without a byte budget the same call decides against free pages
    ex.switch(kept_new, kept_old, arrivals=[Arrival(2, 128, FEASIBLE, 0.0)])
    assert kv.placement() == M.layout_placement(kept_old)


def test_device_ms_is_read_lazily_and_survives_event_reuse():
    # a synchronous switch does not pay cudaEventElapsedTime; its result reads
    # the device time on first access, also after the executor has cycled its
    # event ring past it (the pair is read before it is re-recorded)
    import torch
    from paper_2605_05467_b200 import controller
    gpus = (0, 1)
    reqs = [(0, 300)]
    a = workloads.round_robin(workloads.tp_groups(gpus, 1), reqs, 8)
    b = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, 8)
    kv = PagedKvCluster(KV, gpus, units_per_gpu=256, max_requests=1, max_blocks=32)
    kv.admit(a, seed=1)
    ex = ReconfigurationExecutor(kv)
    first = ex.switch(a, b)
    assert first._device_ms is None and first.host_ms > 0
    cur = b
    for i in range(controller._SYNC_EVENT_PAIRS + 6):
        nxt = a if cur is b else b
        r = ex.switch(cur, nxt)
        cur = nxt
        assert r.device_ms > 0  # read right away
    assert first._device_ms is not None and 0 < first.device_ms < 1e3
    nosync = ex.switch(cur, a if cur is b else b, sync=False)
    assert nosync.device_ms == 0.0
    torch.cuda.synchronize()


def test_sync_small_switch_waits_on_the_kernel_ticket():
    # a synchronous one-launch switch returns when K31's ticket reaches pinned
    # memory (written after every copy and table write); asynchronous and
    # multi-kernel switches carry no ticket
    from paper_2605_05467_b200 import _native
    gpus = tuple(range(4))
    reqs = [(i, 20 + 37 * i) for i in range(5)]
    lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 4)}
    kv = PagedKvCluster(KV, gpus, units_per_gpu=512, max_requests=8, max_blocks=16, fragmented=True)
    kv.admit(lay[1], seed=4)
    ex = ReconfigurationExecutor(kv)
    seen = set()
    for k31, (a, b) in zip((1, 2, 3, 1), ((1, 2), (2, 4), (4, 1), (1, 4))):
        saved = _native.get_tuning("k31")
        _native.set_tuning("k31", k31)
        try:
            before = kv.snapshot()
            plan = M.plan_repartition(lay[a], lay[b], KV.kv_bytes_per_token_per_head)
            rec = kv.records(plan, validate=False)
            res = ex.switch(lay[a], lay[b])
        finally:
            _native.set_tuning("k31", saved)
        t = kv.last_ticket
        assert t != 0 and t not in seen and int(kv.status_host[1]) == t and res.status == 0
        seen.add(t)
        diff = check.compare(kv.snapshot(), check.expected_after(kv, before, rec))
        assert not any(diff.values()), diff
        assert res.device_ms > 0
    r = ex.switch(lay[4], lay[2], sync=False)
    assert kv.last_ticket == 0 and r.kv.units > 0
    _native.set_tuning("k31", 0)
    try:
        r = ex.switch(lay[2], lay[1])  # fused K3 + K1: the end event, no ticket
        assert kv.last_ticket == 0 and r.status == 0
    finally:
        _native.set_tuning("k31", 1)
