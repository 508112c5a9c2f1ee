"""Random walks over the block manager on B200, every step checked against
the oracle replay: admissions, releases, and TP switches between random
partitions of 8 GPU slots (mixed TP levels in one config), with pools small
enough that capacity errors happen. A rejected operation must leave device
state untouched."""

import os

import numpy as np
import pytest

from oracle import check
from paper_2605_05467_b200 import geometry, migration as M
from paper_2605_05467_b200.kvcache import PagedKvCluster

pytestmark = pytest.mark.gpu

# TPR_FUZZ_GEOMETRY=8b|70b runs the walks on Llama-3.1 pages (8B: 256 KiB, 64
# planes; 70B: 640 KiB, 160 planes; partial pages as TMA tensor boxes) instead
# of the tiny default
KV = {"8b": geometry.LLAMA_3_1_8B.kv, "70b": geometry.LLAMA_3_1_70B.kv}.get(
    os.environ.get("TPR_FUZZ_GEOMETRY", ""),
    geometry.KvGeometry(layers=1, head_dim=16, total_heads=8, block_tokens=4))
GPUS = tuple(range(8))


def random_groups(rng):
    gpus = list(rng.permutation(GPUS))
    out, i = [], 0
    while i < len(gpus):
        s = int(rng.choice([x for x in (1, 2, 4, 8) if i + x <= len(gpus)]))
        out.append(tuple(int(g) for g in gpus[i:i + s]))
        i += s
    return out


def layouts(groups, reqs, rng):
    per = [[] for _ in groups]
    for r in reqs:
        per[int(rng.integers(len(groups)))].append(r)
    return [M.KvLayout(g, len(g), 8, tuple(p)) for g, p in zip(groups, per)]


def same_state(a, b):
    return (all(np.array_equal(x, y) for x, y in zip(a["block_tables"], b["block_tables"]))
            and all(np.array_equal(x, y) for x, y in zip(a["rings"], b["rings"]))
            and a["ring_head"] == b["ring_head"] and a["ring_tail"] == b["ring_tail"])


# TPR_FUZZ_SEEDS=n widens the campaign to n seeds (alternating launch paths)
_N = int(os.environ.get("TPR_FUZZ_SEEDS", "5"))
SEEDS = [(0, False), (1, False), (2, False), (3, True), (4, True)] + \
    [(s, s % 2 == 1) for s in range(5, _N)]


@pytest.mark.parametrize("seed,one_call", SEEDS)
def test_random_walk(seed, one_call):
    rng = np.random.default_rng(seed)
    c = PagedKvCluster(KV, GPUS, units_per_gpu=128, max_requests=24, max_blocks=32,
                       fragmented=True, seed=seed)
    c.fill_garbage(seed=seed)
    groups = random_groups(rng)
    cur = [M.KvLayout(g, len(g), 8, ()) for g in groups]
    next_id = 0
    stats = {"admit": 0, "release": 0, "switch": 0, "rejected": 0}
    for step in range(60):
        op = rng.choice(["admit", "release", "switch"], p=[0.35, 0.2, 0.45])
        before = c.snapshot()
        try:
            if op == "admit":
                n = int(rng.integers(1, 4))
                new_reqs = [(next_id + i, int(rng.integers(1, 60))) for i in range(n)]
                g = cur[int(rng.integers(len(cur)))]
                lay = M.KvLayout(g.group, g.tp, 8, tuple(new_reqs))
                c.admit([lay], seed=7)
                next_id += n
                cur = [M.KvLayout(x.group, x.tp, 8, x.requests + (tuple(new_reqs) if x is g else ()))
                       for x in cur]
            elif op == "release":
                resident = [r for lay in cur for r in lay.requests]
                if not resident:
                    continue
                k = int(rng.integers(1, len(resident) + 1))
                gone = [resident[i][0] for i in rng.choice(len(resident), size=k, replace=False)]
                rec = []
                for rid in gone:
                    rs = c.req_slot[rid]
                    own = c.owner[rs]
                    h = 0
                    while h < 8:
                        e = h
                        while e < 8 and own[e] == own[h]:
                            e += 1
                        rec.append((int(own[h]), -1, rs, h, e, c.ctx_of[rid]))
                        h = e
                c.release(gone)
                want = check.expected_after(c, before, np.array(rec, np.int64))
                assert not any(check.compare(c.snapshot(), want).values())
                cur = [M.KvLayout(x.group, x.tp, 8, tuple(r for r in x.requests if r[0] not in gone))
                       for x in cur]
            else:
                resident = [r for lay in cur for r in lay.requests]
                new = layouts(random_groups(rng), resident, rng)
                plan = M.plan_repartition(cur, new, KV.kv_bytes_per_token_per_head)
                rec = c.records(plan)
                if one_call:  # tpr_kv_switch_layouts (general path on any reference error)
                    got, _ = c.switch_layouts(cur, new)
                    assert np.array_equal(got.as_array(), plan.as_array())
                else:
                    c.migrate(plan)
                want = check.expected_after(c, before, rec)
                diff = check.compare(c.snapshot(), want)
                assert not any(diff.values()), (step, diff)
                cur = new
            stats[op] += 1
        except M.MigrationError as exc:
            assert "units needed" in str(exc) or "request slots" in str(exc), exc
            assert same_state(c.snapshot(), before), f"step {step}: rejected {op} changed state"
            stats["rejected"] += 1
        v = c.verify(seed=7)
        assert v["placement_errors"] == 0 and v["word_mismatches"] == 0 and v["status"] == 0, (step, v)
        assert c.placement() == M.layout_placement(cur)
    if seed < 5:  # the fixed seeds are chosen to cover every operation; a wider
        # campaign (TPR_FUZZ_SEEDS) checks correctness only: some walks mostly hit capacity
        assert stats["switch"] >= 5 and stats["admit"] >= 3, stats
