"""Both copy engines -- the TMA bulk engine (cp.async.bulk through shared
memory, the default) and the 16-B vector engine -- must give the same bytes as
the oracle, for K1 (pages, incl. partial last pages) and K2 (contiguous and
strided weight segments)."""

import numpy as np
import pytest
import torch

from oracle import check
from paper_2605_05467_b200 import _native, geometry, migration as M, workloads
from paper_2605_05467_b200.kvcache import PagedKvCluster
from paper_2605_05467_b200.weights import ShardedWeightStore

pytestmark = pytest.mark.gpu

DEFAULT = "bulk"


@pytest.fixture(params=["bulk", "vector"])
def engine(request):
    _native.set_copy_engine(request.param)
    yield request.param
    _native.set_copy_engine(DEFAULT)


def test_engine_switch_roundtrip():
    assert _native.copy_engine() == DEFAULT
    _native.set_copy_engine("vector")
    assert _native.copy_engine() == "vector"
    _native.set_copy_engine(DEFAULT)
    with pytest.raises(ValueError):
        _native.set_copy_engine("dma")


@pytest.mark.parametrize("tp_old,tp_new", [(1, 8), (8, 2), (2, 4), (4, 1)])
def test_kv_bit_exact(engine, tp_old, tp_new):
    kv = geometry.KvGeometry(layers=3, head_dim=64, total_heads=8)  # 24 KiB pages: >1 piece each
    gpus = tuple(range(8))
    rng = np.random.default_rng(tp_old + 10 * tp_new)
    reqs = [(i, int(c)) for i, c in enumerate(rng.integers(1, 120, size=10))]
    old = workloads.round_robin(workloads.tp_groups(gpus, tp_old), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, tp_new), reqs, 8)
    c = PagedKvCluster(kv, gpus, units_per_gpu=512, max_requests=16, max_blocks=8, fragmented=True)
    c.fill_garbage(seed=3)
    c.admit(old, seed=4)
    before = c.snapshot()
    plan = M.plan_repartition(old, new, kv.kv_bytes_per_token_per_head)
    rec = c.records(plan)
    c.migrate(plan)
    diff = check.compare(c.snapshot(), check.expected_after(c, before, rec))
    assert not any(diff.values()), diff
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0


def test_large_pages_cross_piece_boundaries(engine):
    # 70B-shaped pages (640 KiB = 20 x 32 KiB pieces) with ragged last pages
    kv = geometry.LLAMA_3_1_70B.kv
    gpus = (0, 1)
    reqs = [(0, 33), (1, 16), (2, 1), (3, 47)]
    c = PagedKvCluster(kv, gpus, units_per_gpu=64, max_requests=4, max_blocks=4, fragmented=True)
    c.fill_garbage(seed=5)
    old = workloads.round_robin([(0,), (1,)], reqs, 8)
    new = workloads.round_robin([(0, 1)], reqs, 8)
    c.admit(old, seed=6)
    before = c.snapshot()
    plan = M.plan_repartition(old, new, kv.kv_bytes_per_token_per_head)
    rec = c.records(plan)
    c.migrate(plan)
    diff = check.compare(c.snapshot(), check.expected_after(c, before, rec))
    assert not any(diff.values()), diff


@pytest.mark.parametrize("tp_old,tp_new", [(8, 1), (2, 4), (4, 2)])
def test_weights_bit_exact(engine, tp_old, tp_new):
    model = geometry.tiny_geometry(hidden=512, intermediate=1024, vocab=2048)
    gpus = tuple(range(8))
    store = ShardedWeightStore(model, gpus)
    store.load(workloads.tp_groups(gpus, tp_old))
    store.reshard(workloads.tp_groups(gpus, tp_new))
    torch.cuda.synchronize()
    assert store.verify() == 0


@pytest.mark.slow
def test_cfg2_full_size_property(engine):
    w = workloads.config(1, weights=False)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=65536 + 64, max_requests=64, max_blocks=256,
                       fragmented=True, seed=1)
    c.admit(w.old, seed=4)
    c.migrate(M.plan_repartition(w.old, w.new, kv.kv_bytes_per_token_per_head))
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
