"""One process per GPU slot. CPU: the handshake and plan partition logic over
gloo with world_size 2. GPU: the full push-model migration with 2 and 4
processes through CUDA IPC; pools, block tables and rings of all ranks
together must equal the oracle's replay bit for bit. Each rank takes GPU
``rank % device_count``: one GPU per rank on a multi-GPU node (peer pools over
NVLink, the copy engine libtpr picks for peer mappings), all ranks on one
device otherwise (the gpurun boxes)."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _init(rank, world, path):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)


def _device(rank):
    """This rank's GPU: its own when the node has one per rank, else shared."""
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    return dev


def _handshake_worker(rank, world, path, q):
    import sys
    sys.path.insert(0, str(ROOT))
    from paper_2605_05467_b200 import distributed as D
    from paper_2605_05467_b200.migration import MigrationError
    _init(rank, world, path)
    rec = np.array([[0, 1, 3, 4, 8, 33], [1, 0, 5, 0, 4, 17]], np.int64)
    res = D.handshake(rec, [0, 0], [64, 64])
    ok1 = res.digest == D.plan_digest(rec) and list(res.tails) == [64, 64]
    # a rank with a different plan makes every rank fail
    bad = rec.copy()
    if rank == 1:
        bad[0, 5] = 34
    try:
        D.handshake(bad, [0, 0], [64, 64])
        ok2 = False
    except MigrationError:
        ok2 = True
    q.put((rank, ok1, ok2))
    dist.destroy_process_group()


def test_handshake_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "store")
        procs = [ctx.Process(target=_handshake_worker, args=(r, 2, path, q)) for r in range(2)]
        for p in procs:
            p.start()
        out = sorted(q.get(timeout=120) for _ in procs)
        for p in procs:
            p.join(timeout=60)
    assert out == [(0, True, True), (1, True, True)]


def test_partition_counts():
    from paper_2605_05467_b200 import distributed as D
    rec = np.array([[0, 1, 0, 4, 8, 33], [1, 0, 1, 0, 4, 17], [-1, 1, 2, 0, 8, 16]], np.int64)
    in_u, out_u = D.ring_deltas(rec, 2, 16)
    assert in_u.tolist() == [4 * 2, 4 * 3 + 8 * 1] and out_u.tolist() == [4 * 3, 4 * 2]
    assert D.my_units(rec, 0, 16) == 12 and D.my_units(rec, 1, 16) == 8


# ---------------------------------------------------------------------------
# GPU: several processes on one device, IPC-mapped peer pools
# ---------------------------------------------------------------------------

def _gpu_worker(rank, world, path, outdir, q):
    import sys
    sys.path.insert(0, str(ROOT))
    try:
        from paper_2605_05467_b200 import geometry, migration as M, workloads
        from paper_2605_05467_b200.distributed import DistributedKvCluster
        _init(rank, world, path)
        dev = _device(rank)
        kv = geometry.KvGeometry(layers=2, head_dim=32, total_heads=8)
        gpus = tuple(range(world))
        reqs = [(i, 5 + 29 * i) for i in range(7)]
        lays = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8)
                for tp in (1, 2, 4) if tp <= world}
        c = DistributedKvCluster(kv, gpus, units_per_gpu=512, max_requests=8, max_blocks=16,
                                 device=dev, fragmented=True, seed=rank)
        c.admit(lays[1], seed=17)
        seq = [1, world, 1] if world == 2 else [1, 2, 4, 2]
        for i, (a, b) in enumerate(zip(seq, seq[1:])):
            np.savez(os.path.join(outdir, f"before_{i}_{rank}.npz"), **c.snapshot())
            plan = M.plan_repartition(lays[a], lays[b], kv.kv_bytes_per_token_per_head)
            np.save(os.path.join(outdir, f"rec_{i}.npy"), c.records(plan))
            if i % 2:  # the native host half (tpr_switch_prepare) + zero-copy tpr_kv_switch
                got, _ = c.migrate_layouts(lays[a], lays[b])
                assert np.array_equal(got.as_array(), plan.as_array())
            else:
                c.migrate(plan)
            np.savez(os.path.join(outdir, f"after_{i}_{rank}.npz"), **c.snapshot())
        v = c.verify()
        from paper_2605_05467_b200 import _native
        k1_engine, _ = _native.last_engines()
        # peer pools on another GPU never take the TMA engine
        if torch.cuda.device_count() >= world:
            assert k1_engine == "vector", k1_engine
        c.close()
        dist.destroy_process_group()
        q.put((rank, v, len(seq) - 1))
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc(), -1))


def _exec_worker(rank, world, path, q, device_barrier=True):
    import sys
    sys.path.insert(0, str(ROOT))
    try:
        from paper_2605_05467_b200 import geometry, migration as M, workloads
        from paper_2605_05467_b200.distributed import (DistributedExecutor, DistributedKvCluster,
                                                       DistributedWeightStore)
        _init(rank, world, path)
        dev = _device(rank)
        model = geometry.tiny_geometry()
        gpus = tuple(range(world))
        reqs = [(i, 9 + 17 * i) for i in range(6)]
        tps = [t for t in (1, 2, 4) if t <= world]
        lays = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in tps}
        kv = DistributedKvCluster(model.kv, gpus, units_per_gpu=512, max_requests=8, max_blocks=16,
                                  device=dev, fragmented=True, seed=rank)
        kv.admit(lays[1], seed=5)
        ws = DistributedWeightStore(model, gpus, device=dev)
        ws.load(workloads.tp_groups(gpus, 1))
        ex = DistributedExecutor(kv, ws, device_barrier=device_barrier, check_every=2)
        seq = [1, 2, 1] if world == 2 else [1, 2, 4, 2, 4, 1]
        results = []
        for a, b in zip(seq, seq[1:]):
            plan, ks, wst, ms = ex.switch(lays[a], lays[b], new_weight_groups=workloads.tp_groups(gpus, b))
            results.append((a, b, ks.bytes, wst.local_bytes, wst.remote_bytes, wst.views))
            assert ws.verify() == 0, (a, b)
        v = kv.verify()
        bad_w = ws.verify()
        ex.close()
        ws.close()
        kv.close()
        dist.destroy_process_group()
        q.put((rank, v, bad_w, results))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc(), -1, None))


def _barrier_timeout_worker(rank, world, path, q):
    import sys
    sys.path.insert(0, str(ROOT))
    try:
        from paper_2605_05467_b200.distributed import DeviceBarrier
        from paper_2605_05467_b200.migration import MigrationError
        _init(rank, world, path)
        bar = DeviceBarrier(_device(rank), timeout_s=0.5)
        st = torch.cuda.Stream()
        bar(st)                      # both ranks arrive: passes
        st.synchronize()
        bar.check()
        raised = None
        if rank == 0:                # rank 1 "crashes": rank 0 must time out, not hang
            bar(st)
            st.synchronize()
            try:
                bar.check()
                raised = False
            except MigrationError:
                raised = True
        dist.barrier()
        q.put((rank, raised))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
def test_device_barrier_times_out_instead_of_hanging():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "store")
        procs = [ctx.Process(target=_barrier_timeout_worker, args=(r, 2, path, q), daemon=True)
                 for r in range(2)]
        for p in procs:
            p.start()
        res = sorted(q.get(timeout=120) for _ in procs)
        for p in procs:
            p.join(timeout=60)
    assert res == [(0, True), (1, None)], res


@pytest.mark.gpu
@pytest.mark.parametrize("world,device_barrier", [(2, True), (4, True), (2, False)])
def test_distributed_executor_kv_and_weights(world, device_barrier):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "store")
        procs = [ctx.Process(target=_exec_worker, args=(r, world, path, q, device_barrier),
                             daemon=True) for r in range(world)]
        for p in procs:
            p.start()
        res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
        for p in procs:
            p.join(timeout=60)
    for rank, v, bad_w, results in res:
        assert results is not None, v
        assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0, v
        assert bad_w == 0
    # every rank computed the same global stats for every switch
    assert all(r[3] == res[0][3] for r in res)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_multiprocess_push_migration_bit_exact(world):
    from oracle import kvmove
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "store")
        procs = [ctx.Process(target=_gpu_worker, args=(r, world, path, d, q), daemon=True)
                 for r in range(world)]
        for p in procs:
            p.start()
        res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
        for p in procs:
            p.join(timeout=60)
        for rank, v, n in res:
            assert n > 0, v
            assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0, v
        geo = dict(layers=2, head_dim=32, dtype_bytes=2, block_tokens=16, total_heads=8,
                   max_blocks=16, n_req_slots=8, n_units=512)
        for i in range(res[0][2]):
            before = [np.load(os.path.join(d, f"before_{i}_{r}.npz")) for r in range(world)]
            after = [np.load(os.path.join(d, f"after_{i}_{r}.npz")) for r in range(world)]
            rec = np.load(os.path.join(d, f"rec_{i}.npy"))
            pools = [b["pool"].copy() for b in before]
            tables = [b["block_table"].copy() for b in before]
            rings = [b["ring"].copy() for b in before]
            _, status, heads, tails = kvmove.kv_migrate(geo, pools, tables, rings,
                                                        list(before[0]["ring_head"]),
                                                        list(before[0]["ring_tail"]), rec)
            assert status == 0
            for r in range(world):
                assert np.array_equal(after[r]["pool"], pools[r]), (i, r)
                assert np.array_equal(after[r]["block_table"], tables[r]), (i, r)
                live = np.arange(heads[r], tails[r]) % 512
                assert np.array_equal(after[r]["ring"][live], rings[r][live]), (i, r)
                assert list(after[r]["ring_head"]) == heads and list(after[r]["ring_tail"]) == tails


def _abort_worker(rank, world, path, q):
    import sys
    sys.path.insert(0, str(ROOT))
    try:
        from paper_2605_05467_b200 import geometry, workloads
        from paper_2605_05467_b200.distributed import DistributedExecutor, DistributedKvCluster
        from paper_2605_05467_b200.migration import MigrationError
        _init(rank, world, path)
        dev = _device(rank)
        kv = geometry.KvGeometry(layers=2, head_dim=32, total_heads=8)
        gpus = (0, 1)
        reqs = [(i, 20 + 9 * i) for i in range(4)]
        lays = {tp: workloads.round_robin(workloads.tp_groups(gpus, tp), reqs, 8) for tp in (1, 2)}
        c = DistributedKvCluster(kv, gpus, units_per_gpu=256, max_requests=4, max_blocks=8,
                                 device=dev, fragmented=True, seed=rank)
        c.admit(lays[1], seed=3)
        ex = DistributedExecutor(c, device_barrier=True, barrier_timeout_s=0.5)
        before = c.snapshot()
        raised = None
        if rank == 0:  # rank 1 never arrives: the start barrier times out, K3 + K1 abort
            try:
                ex.switch(lays[1], lays[2])
                raised = False
            except MigrationError:
                raised = True
            try:  # and the executor refuses further switches
                ex.switch(lays[1], lays[2])
                raised = False
            except MigrationError as exc:
                raised = raised and "rebuild" in str(exc)
        dist.barrier()
        after = c.snapshot()
        same = all(np.array_equal(before[k], after[k]) for k in ("pool", "block_table", "ring"))
        q.put((rank, raised, same))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None))


@pytest.mark.gpu
def test_start_barrier_timeout_aborts_the_switch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "store")
        procs = [ctx.Process(target=_abort_worker, args=(r, 2, path, q), daemon=True)
                 for r in range(2)]
        for p in procs:
            p.start()
        res = sorted((q.get(timeout=180) for _ in procs), key=lambda x: x[0])
        for p in procs:
            p.join(timeout=60)
    # no table, ring or pool byte changed on either rank
    assert res == [(0, True, True), (1, None, True)], res
