"""The TMA bulk-copy engine (cp.async.bulk through shared memory) must give
the same bytes as the oracle, for K1 (pages, incl. partial last pages) and
K2 (contiguous and strided weight segments)."""

import numpy as np
import pytest
import torch

from oracle import check
from paper_2605_05467_b200 import _native, geometry, migration as M, workloads
from paper_2605_05467_b200.kvcache import PagedKvCluster
from paper_2605_05467_b200.weights import ShardedWeightStore

pytestmark = pytest.mark.gpu


@pytest.fixture
def bulk():
    _native.set_copy_engine("bulk")
    yield
    _native.set_copy_engine("vector")


def test_engine_switch_roundtrip():
    assert _native.copy_engine() == "vector"
    _native.set_copy_engine("bulk")
    assert _native.copy_engine() == "bulk"
    _native.set_copy_engine("vector")
    with pytest.raises(ValueError):
        _native.set_copy_engine("dma")


@pytest.mark.parametrize("tp_old,tp_new", [(1, 8), (8, 2), (2, 4), (4, 1)])
def test_bulk_kv_bit_exact(bulk, tp_old, tp_new):
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


@pytest.mark.parametrize("tp_old,tp_new", [(8, 1), (2, 4), (4, 2)])
def test_bulk_weights_bit_exact(bulk, tp_old, tp_new):
    model = geometry.tiny_geometry(hidden=512, intermediate=1024, vocab=2048)
    gpus = tuple(range(8))
    store = ShardedWeightStore(model, gpus)
    store.load(workloads.tp_groups(gpus, tp_old))
    store.reshard(workloads.tp_groups(gpus, tp_new))
    torch.cuda.synchronize()
    assert store.verify() == 0


@pytest.mark.slow
def test_bulk_cfg2_full_size_property(bulk):
    w = workloads.config(1, weights=False)
    kv = w.model.kv
    c = PagedKvCluster(kv, w.gpus, units_per_gpu=65536 + 64, max_requests=64, max_blocks=256,
                       fragmented=True, seed=1)
    c.admit(w.old, seed=4)
    c.migrate(M.plan_repartition(w.old, w.new, kv.kv_bytes_per_token_per_head))
    v = c.verify()
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
