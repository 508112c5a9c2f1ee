"""Many switches in a row (KV + weights, async enqueue like a serving loop):
device memory stays flat after warm-up and the final state is exact."""

import pytest
import torch

from paper_2605_05467_b200 import geometry, migration as M, workloads
from paper_2605_05467_b200.controller import ReconfigurationExecutor
from paper_2605_05467_b200.kvcache import PagedKvCluster
from paper_2605_05467_b200.weights import ShardedWeightStore

pytestmark = pytest.mark.gpu


def test_soak_400_switches():
    model = geometry.tiny_geometry()
    gpus = tuple(range(8))
    reqs = [(i, 5 + 11 * i) for i in range(24)]
    tps = (1, 2, 4, 8)
    lays = {t: workloads.round_robin(workloads.tp_groups(gpus, t), reqs, 8) for t in tps}
    kv = PagedKvCluster(model.kv, gpus, units_per_gpu=2048, max_requests=32, max_blocks=32,
                        fragmented=True, seed=5)
    kv.admit(lays[1], seed=3)
    store = ShardedWeightStore(model, gpus)
    store.load(workloads.tp_groups(gpus, 1))
    ex = ReconfigurationExecutor(kv, store)
    seq = [1, 2, 4, 8, 4, 2, 8, 1, 4, 1, 2, 1]
    cur, mem = 1, []
    for i in range(400):
        nxt = seq[i % len(seq)]
        if nxt == cur:
            nxt = seq[(i + 1) % len(seq)]
        ex.switch(lays[cur], lays[nxt], new_weight_groups=workloads.tp_groups(gpus, nxt),
                  sync=(i % 50 == 49), validate=False)
        cur = nxt
        if i % 50 == 49:
            torch.cuda.synchronize()
            mem.append(torch.cuda.memory_allocated())
    torch.cuda.synchronize()
    assert max(mem[2:]) <= mem[1] * 1.01, mem  # flat after warm-up
    v = kv.verify(seed=3)
    assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0
    assert kv.placement() == M.layout_placement(lays[cur])
    assert store.verify() == 0
    assert sum(kv.free_units(g) for g in gpus) == 8 * 2048 - sum(8 * model.kv.blocks(c) for _, c in reqs)
