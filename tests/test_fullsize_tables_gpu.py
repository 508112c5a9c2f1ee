"""Block tables, free rings and ring counters bit-exact against the oracle's
sequential replay at the BASELINE sizes (VERDICT r1 "Next" #1).

Page bytes at these sizes (24-112 GiB) are checked by the placement-invariant
pattern (``verify``: every owned page carries its key, every table entry
realises the host placement). What that property cannot see -- WHICH unit id
each (request, head, page) got, and the order units return to the free rings --
is pinned here: the oracle (oracle/kvmove.c, tables-and-rings-only mode)
replays the plan page by page in apply_plan order (migration.py:192-207) on a
host copy of the "before" tables and rings, and the device state after the
production switch call must equal it entry for entry. The one-process-per-GPU
design depends on exactly this determinism: a source rank allocates pages on
its peer without talking to it (distributed.py).
"""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT
from oracle import check
from paper_2605_05467_b200 import geometry, migration as M, workloads
from paper_2605_05467_b200.kvcache import PagedKvCluster

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TINY = geometry.KvGeometry(layers=2, head_dim=32, total_heads=8)


def _units(w, kv):
    import bench
    return bench.capacity_units(w, kv)


def switch_and_compare(c, old, new, planner_call=True):
    """One production switch (tpr_kv_switch_layouts) vs the oracle's replay of
    the reference plan; returns the plan."""
    kvb = c.kv.kv_bytes_per_token_per_head
    before = c.tables_snapshot()
    plan = M.plan_repartition(old, new, kvb)
    rec = c.records(plan, validate=False)
    if planner_call:
        got_plan, stats = c.switch_layouts(old, new)
        assert np.array_equal(got_plan.as_array(), plan.as_array())
    else:
        stats = c.migrate(plan)
    after = c.tables_snapshot()
    want = check.expected_after(c, before, rec)
    diff = check.compare(after, want)
    assert want["status"] == 0 and int(c.status.item()) == 0
    assert not any(diff.values()), diff
    assert stats.units == want["pages"] and stats.bytes == plan.total_bytes
    return plan


def _check_pattern(c, pages):
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0, v
    assert v["pages_checked"] == pages


def test_cfg2_tables_rings_bit_exact():
    # BASELINE configs[1]: Llama-3.1-8B TP2 <-> TP4, 64 x 4096 (98,304 pages per switch)
    w = workloads.config(1, weights=False)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=_units(w, kv), max_requests=64,
                       max_blocks=256, fragmented=True, seed=11)
    c.admit(w.old, seed=4)
    for a, b in ((w.old, w.new), (w.new, w.old), (w.old, w.new)):
        plan = switch_and_compare(c, a, b)
        assert plan.total_bytes == 24 * 2**30
    _check_pattern(c, 64 * 8 * 256)


def test_cfg3_consolidation_tables_rings_bit_exact():
    # BASELINE configs[2]: TP8 -> 8 x TP1 with every request on GPU0 (28 GiB incast)
    w = workloads.config(2, weights=False)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=_units(w, kv), max_requests=64,
                       max_blocks=256, fragmented=True, seed=12)
    c.admit(w.old, seed=5)
    plan = switch_and_compare(c, w.old, w.new)
    assert plan.total_bytes == 28 * 2**30 and plan.n_transfers == 7 * 64
    switch_and_compare(c, w.new, w.old)
    _check_pattern(c, 64 * 8 * 256)


def test_cfg4_70b_tables_rings_bit_exact():
    # BASELINE configs[3]: Llama-3.1-70B TP4 <-> TP8, 8 x 32768 (131,072 pages of 640 KiB)
    w = workloads.config(3)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=_units(w, kv), max_requests=8,
                       max_blocks=kv.blocks(32768), fragmented=True, seed=13)
    c.admit(w.old, seed=6)
    for a, b in ((w.old, w.new), (w.new, w.old)):
        plan = switch_and_compare(c, a, b, planner_call=a is w.old)
        assert plan.total_bytes == 70 * 2**30
    _check_pattern(c, 8 * 8 * 2048)


def test_sweep_extreme_1792_transfers_tables_rings_bit_exact():
    # config-5 extreme: TP1 -> TP8, 256 seqs x 4096 = 1792 transfers, 458,752 pages.
    # 112 GiB of Llama pages does not fit beside its source; the tables, rings and
    # plan are the real ones, on small pages (units of 4 KiB)
    gpus = tuple(range(8))
    reqs = [(i, 4096) for i in range(256)]
    tp1 = workloads.round_robin(workloads.tp_groups(gpus, 1), reqs, 8)
    tp8 = workloads.round_robin(workloads.tp_groups(gpus, 8), reqs, 8)
    c = PagedKvCluster(TINY, gpus, units_per_gpu=2 * 65536 + 64, max_requests=256,
                       max_blocks=256, fragmented=True, seed=14)
    c.admit(tp1, seed=7)
    plan = switch_and_compare(c, tp1, tp8)
    assert plan.n_transfers == 1792
    plan = switch_and_compare(c, tp8, tp1)
    _check_pattern(c, 256 * 8 * 256)


def test_mixed_contexts_fused_and_split_k3_boundaries():
    # plans just below / above the fused-K3 limit with ragged contexts, 8 slots
    from paper_2605_05467_b200 import _native
    gpus = tuple(range(8))
    rng = np.random.default_rng(15)
    fuse = _native.k3_fuse_units()
    units = []
    for n_seqs in (3, 9, 40):
        reqs = [(int(i), int(x)) for i, x in enumerate(rng.integers(1, 1200, size=n_seqs))]
        lay = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2, 8)}
        c = PagedKvCluster(TINY, gpus, units_per_gpu=8192, max_requests=n_seqs, max_blocks=75,
                           fragmented=True, seed=n_seqs)
        c.admit(lay[2], seed=8)
        for a, b in ((2, 8), (8, 1), (1, 2)):
            plan = switch_and_compare(c, lay[a], lay[b])
            units.append(sum((t.head_hi - t.head_lo) * TINY.blocks(dict(reqs)[t.request_id])
                             for t in plan.transfers))
        v = c.verify()
        assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
    assert min(units) <= fuse < max(units)  # both K3 launch paths ran


# ---------------------------------------------------------------------------
# one process per GPU slot at cfg2 size: 4 processes, push model over IPC
# ---------------------------------------------------------------------------

def _push_worker(rank, world, path, outdir, q):
    import sys
    sys.path.insert(0, str(ROOT))
    try:
        import torch.distributed as dist

        from paper_2605_05467_b200.distributed import DistributedKvCluster
        dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank,
                                world_size=world)
        n_dev = torch.cuda.device_count()
        dev = torch.device("cuda", rank % n_dev)
        torch.cuda.set_device(dev)
        w = workloads.config(1, weights=False)
        kv = w.model.kv
        units = max(_units(w, kv).values())
        c = DistributedKvCluster(kv, w.gpus, units_per_gpu=units, max_requests=64,
                                 max_blocks=256, device=dev, fragmented=True, seed=rank)
        c.admit(w.old, seed=4)
        for i, (a, b) in enumerate(((w.old, w.new), (w.new, w.old))):
            np.savez(os.path.join(outdir, f"before_{i}_{rank}.npz"), **c.tables_snapshot())
            plan = M.plan_repartition(a, b, kv.kv_bytes_per_token_per_head)
            if rank == 0:
                np.save(os.path.join(outdir, f"rec_{i}.npy"), c.records(plan))
            got, _ = c.migrate_layouts(a, b)
            assert np.array_equal(got.as_array(), plan.as_array())
            np.savez(os.path.join(outdir, f"after_{i}_{rank}.npz"), **c.tables_snapshot())
        v = c.verify()
        c.close()
        dist.destroy_process_group()
        q.put((rank, v))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_four_process_push_cfg2_tables_rings_bit_exact():
    from oracle import kvmove
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "store")
        procs = [ctx.Process(target=_push_worker, args=(r, world, path, d, q), daemon=True)
                 for r in range(world)]
        for p in procs:
            p.start()
        res = sorted((q.get(timeout=900) for _ in procs), key=lambda x: x[0])
        for p in procs:
            p.join(timeout=120)
        for rank, v in res:
            assert isinstance(v, dict), v
            assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0, v
            assert v["pages_checked"] == 64 * 2 * 256  # TP2 <- TP4 <- TP2: 2 heads per slot
        w = workloads.config(1, weights=False)
        kv = w.model.kv
        units = max(_units(w, kv).values())
        geo = dict(layers=kv.layers, head_dim=kv.head_dim, dtype_bytes=kv.dtype_bytes,
                   block_tokens=kv.block_tokens, total_heads=8, max_blocks=256, n_req_slots=64,
                   n_units=units)
        for i in range(2):
            before = [np.load(os.path.join(d, f"before_{i}_{r}.npz")) for r in range(world)]
            after = [np.load(os.path.join(d, f"after_{i}_{r}.npz")) for r in range(world)]
            rec = np.load(os.path.join(d, f"rec_{i}.npy"))
            tables = [b["block_tables"][0].reshape(-1).copy() for b in before]
            rings = [b["rings"][0].copy() for b in before]
            n, status, heads, tails = kvmove.kv_migrate(geo, None, tables, rings,
                                                        list(before[0]["ring_head"]),
                                                        list(before[0]["ring_tail"]), rec)
            assert status == 0 and n == 98304
            for r in range(world):
                assert np.array_equal(after[r]["block_tables"][0].reshape(-1), tables[r]), (i, r)
                live = np.arange(heads[r], tails[r]) % units
                assert np.array_equal(after[r]["rings"][0][live], rings[r][live]), (i, r)
                assert list(after[r]["ring_head"]) == heads and list(after[r]["ring_tail"]) == tails
