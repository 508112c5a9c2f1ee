"""K2 weight reshard on B200 vs the narrow/concatenate oracle (oracle/weights.py).

Every TP shard a GPU computes with after a reshard must equal the matching
rows/columns of the full matrix reassembled from the OLD shards on the host,
bit for bit; and the fetched volume must equal what weight_memory("sharded")
implies."""

import numpy as np
import pytest
import torch

from oracle import weights as W
from paper_2605_05467_b200 import geometry, migration as M, workloads
from paper_2605_05467_b200.weights import ShardedWeightStore, groups_ranges

pytestmark = pytest.mark.gpu

MODEL = geometry.tiny_geometry()


def host_pieces(store):
    """{matrix index: [(row0, col0, ndarray)]} from every GPU's resident slices."""
    out = {}
    for g in store.gpu_ids:
        for a in sorted(store.have[g]):
            for i, m in enumerate(store.split):
                v = store.slices(g, m.name, m.layer, a, a + 1)
                v = v.cpu().view(torch.int16).numpy().view(np.uint16)
                r0 = a * (m.rows // 8) if m.split == "col" else 0
                c0 = a * (m.cols // 8) if m.split == "row" else 0
                out.setdefault(i, []).append((r0, c0, v.copy()))
    return out


def check_against_oracle(store, pieces, groups):
    for grp in groups:
        tp = len(grp)
        for rank, g in enumerate(grp):
            for i, m in enumerate(store.split):
                full, seen = W.assemble_full(pieces[i], m.rows, m.cols)
                want = W.expected_shard(full, m.split, tp, rank)
                (r0, r1), (c0, c1) = W.shard_bounds(m.split, m.rows, m.cols, tp, rank)
                assert seen[r0:r1, c0:c1].all()
                got = store.shard(g, m.name, m.layer).cpu().view(torch.int16).numpy().view(np.uint16)
                assert np.array_equal(got, want), (m.name, m.layer, g)


@pytest.mark.parametrize("tp_old,tp_new", [(a, b) for a in (1, 2, 4, 8) for b in (1, 2, 4, 8) if a != b])
def test_all_transitions_bit_exact(tp_old, tp_new):
    gpus = tuple(range(8))
    store = ShardedWeightStore(MODEL, gpus)
    store.load(workloads.tp_groups(gpus, tp_old))
    pieces = host_pieces(store)
    new_groups = workloads.tp_groups(gpus, tp_new)
    stats = store.reshard(new_groups)
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, new_groups)
    assert store.verify() == 0
    local, remote, views = expected_volume(workloads.tp_groups(gpus, tp_old), new_groups,
                                           store.bytes_per_slice)
    assert (stats.local_bytes, stats.remote_bytes, stats.views) == (local, remote, views)
    # what a GPU fetches is its new shard, weight_memory("sharded", tp_new) of
    # the split matrices (replicated norms never move), minus what it held
    rep = sum(m.rows * m.cols for m in store.replicated) * MODEL.dtype_bytes
    per_gpu = M.weight_memory("sharded", MODEL, tp=tp_new) * 1e9 - rep / tp_new
    old, new = groups_ranges(workloads.tp_groups(gpus, tp_old)), groups_ranges(new_groups)
    held = sum(max(0, min(old[g][1], y) - max(old[g][0], x)) for g, (x, y) in new.items()
               if not (old[g][0] <= x and y <= old[g][1]))
    assert stats.local_bytes == 0
    assert stats.remote_bytes == pytest.approx((8 - views) * per_gpu - held * store.bytes_per_slice)
    store.finish()


def expected_volume(old_groups, new_groups, per_slice):
    """Independent count: a GPU whose new slice range lies inside its old one
    is a view; otherwise its resident slices stay in place (slice-addressed
    arena) and exactly the missing ones are fetched -- no local copy."""
    old, new = groups_ranges(old_groups), groups_ranges(new_groups)
    remote = views = 0
    for g, (x, y) in new.items():
        a, b = old[g]
        if a <= x and y <= b:
            views += 1
            continue
        inter = max(0, min(b, y) - max(a, x))
        remote += (y - x) - inter
    return 0, remote * per_slice, views


def test_sequence_reuses_resident_slices():
    gpus = (0, 1, 2, 3)
    store = ShardedWeightStore(MODEL, gpus)
    store.load(workloads.tp_groups(gpus, 2))
    fwd = store.reshard(workloads.tp_groups(gpus, 4))   # GPU1, GPU2 fetch a quarter each
    assert fwd.remote_bytes == 2 * store.bytes_per_slice * 2 and fwd.local_bytes == 0
    assert fwd.views == 2
    pieces = host_pieces(store)
    # every GPU still holds its TP2 half: GPU0 / GPU3 kept theirs, GPU1 / GPU2
    # grew in place (their halves stayed at their window positions)
    back = store.reshard(workloads.tp_groups(gpus, 2))
    assert back.views == 4 and back.bytes == 0
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, workloads.tp_groups(gpus, 2))
    assert store.verify() == 0
    store.finish()


def test_trim_drops_slices_and_regrowth_fetches_them_in_place():
    gpus = (0, 1, 2, 3)
    store = ShardedWeightStore(MODEL, gpus)
    store.load(workloads.tp_groups(gpus, 4))
    grow = store.reshard(workloads.tp_groups(gpus, 1))   # every GPU gathers all 8 slices
    assert grow.local_bytes == 0 and grow.remote_bytes == 4 * 6 * store.bytes_per_slice
    assert grow.in_place == 4
    pieces = host_pieces(store)
    kept = store.reshard(workloads.tp_groups(gpus, 2))   # views: the full copy stays resident
    assert kept.views == 4 and kept.bytes == 0
    trimmed = store.reshard(workloads.tp_groups(gpus, 2), trim=True)  # drop to TP2 halves
    assert trimmed.bytes == 0 and trimmed.views == 4
    assert store.resident == groups_ranges(workloads.tp_groups(gpus, 2))
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, workloads.tp_groups(gpus, 2))
    assert store.verify() == 0
    regrow = store.reshard(workloads.tp_groups(gpus, 1))  # the dropped halves come back
    assert regrow.local_bytes == 0 and regrow.remote_bytes == 4 * 4 * store.bytes_per_slice
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, workloads.tp_groups(gpus, 1))
    store.finish()


def test_window_change_and_overflow():
    # windows of 2 slices: TP4 -> TP4 in another rank order leaves the window
    # (a new arena, everything fetched); TP4 -> TP2 outgrows it (the one case
    # with a local relayout copy)
    gpus = (0, 1, 2, 3)
    store = ShardedWeightStore(MODEL, gpus, max_slices=2)
    store.load(workloads.tp_groups(gpus, 4))
    pieces = host_pieces(store)
    s = store.reshard([(3, 2, 1, 0)])
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, [(3, 2, 1, 0)])
    assert s.local_bytes == 0 and s.remote_bytes == 4 * 2 * store.bytes_per_slice
    assert store.window == {3: (0, 2), 2: (2, 2), 1: (4, 2), 0: (6, 2)}
    s = store.reshard([(3, 2), (1, 0)])
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, [(3, 2), (1, 0)])
    # GPU3 and GPU0 keep 2 of their 4 new slices (copied into the larger
    # arena), GPU2 and GPU1 hold none of theirs: 4 local + 12 fetched slices
    assert s.local_bytes == 4 * store.bytes_per_slice and s.remote_bytes == 12 * store.bytes_per_slice
    assert store.verify() == 0
    store.finish()


def test_k2_mixed_segments_bit_exact():
    # TP2 -> TP8 (views + in-place fetches) and TP8 -> TP4 (in-place growth
    # of every GPU): column- and row-parallel slices through one K2 launch
    gpus = tuple(range(8))
    for a, b in ((2, 8), (8, 4)):
        store = ShardedWeightStore(MODEL, gpus)
        store.load(workloads.tp_groups(gpus, a))
        pieces = host_pieces(store)
        store.reshard(workloads.tp_groups(gpus, b))
        torch.cuda.synchronize()
        check_against_oracle(store, pieces, workloads.tp_groups(gpus, b))
        assert store.verify() == 0
        store.finish()


def test_device_matrix_fill_matches_numpy_pattern():
    from paper_2605_05467_b200 import pattern
    store = ShardedWeightStore(MODEL, (0, 1))
    store.load([(0, 1)])
    for name, layer in (("q_proj", 0), ("o_proj", 1), ("lm_head", -1), ("input_layernorm", 0)):
        m = next(x for x in MODEL.matrices if (x.name, x.layer) == (name, layer))
        got = store.shard(1, name, layer).cpu().view(torch.int16).numpy().view(np.uint16)
        if m.split == "col":
            want = pattern.matrix(m.key, m.rows // 2, m.cols, m.rows // 2, 0, m.cols)
        elif m.split == "row":
            want = pattern.matrix(m.key, m.rows, m.cols // 2, 0, m.cols // 2, m.cols)
        else:
            want = pattern.matrix(m.key, m.rows, m.cols, 0, 0, m.cols)
        assert np.array_equal(got, want), name


def test_full_copy_mode_moves_nothing():
    gpus = (0, 1, 2, 3)
    store = ShardedWeightStore(MODEL, gpus, mode="full_copy_per_gpu")
    store.load(workloads.tp_groups(gpus, 4))
    for tp in (1, 2, 4, 2, 1):
        s = store.reshard(workloads.tp_groups(gpus, tp))
        assert s.bytes == 0 and s.views == 4
        assert store.verify() == 0


def test_scale_in_parks_gpus():
    gpus = tuple(range(8))
    store = ShardedWeightStore(MODEL, gpus)
    store.load([gpus])
    s = store.reshard([(0,)], parked=gpus[1:])
    torch.cuda.synchronize()
    split_bytes = sum(m.rows * m.cols for m in store.split) * MODEL.dtype_bytes
    assert s.remote_bytes == 7 * split_bytes // 8 and s.local_bytes == 0
    assert store.verify() == 0
    # egress balanced: every parked GPU serves exactly its own slice
    assert sorted(v for g, v in s.egress.items() if g) == [split_bytes // 8] * 7


@pytest.mark.slow
def test_llama8b_tp2_tp4_full_size():
    gpus = (0, 1, 2, 3)
    store = ShardedWeightStore(geometry.LLAMA_3_1_8B, gpus)
    store.load(workloads.tp_groups(gpus, 2))
    s = store.reshard(workloads.tp_groups(gpus, 4))
    torch.cuda.synchronize()
    split = sum(m.rows * m.cols for m in store.split) * 2
    assert s.remote_bytes == 2 * split // 4 and s.views == 2
    assert store.verify() == 0
    store.finish()


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("TPR_FUZZ_SEEDS", "4"))))
def test_random_reshard_walk(seed):
    # random partitions of 8 GPUs into groups of mixed TP degree, in random
    # rank order, with and without trim: after every reshard each GPU's shard
    # equals the oracle's slice of the matrix reassembled from the old shards
    rng = np.random.default_rng(seed)
    gpus = tuple(range(8))

    def random_groups():
        perm = [int(g) for g in rng.permutation(gpus)]
        out, i = [], 0
        while i < 8:
            s = int(rng.choice([x for x in (1, 2, 4, 8) if i + x <= 8]))
            out.append(tuple(perm[i:i + s]))
            i += s
        return out

    store = ShardedWeightStore(MODEL, gpus)
    store.load(random_groups())
    for step in range(8):
        pieces = host_pieces(store)
        groups = random_groups()
        store.reshard(groups, trim=bool(rng.integers(2)))
        torch.cuda.synchronize()
        check_against_oracle(store, pieces, groups)
        assert store.verify() == 0, step


def _real_shape_layer(base):
    """One decoder layer with the model's real matrix shapes (q/k/v, o,
    gate/up, down), vocab cut to 1024 so the host oracle stays small."""
    import dataclasses
    return dataclasses.replace(base, name=f"{base.name} (1 layer, vocab 1024)", layers=1, vocab=1024,
                               matrices=())


@pytest.mark.slow
@pytest.mark.parametrize("base,tp_old,tp_new", [
    ("8b", 8, 1), ("8b", 1, 2), ("8b", 2, 8), ("8b", 4, 2), ("8b", 8, 4), ("8b", 2, 4),
    ("70b", 8, 1), ("70b", 8, 4), ("70b", 4, 8), ("70b", 4, 2)])
def test_real_matrix_shapes_bit_exact(base, tp_old, tp_new):
    # the Llama-3.1-8B / 70B matrix shapes (row-parallel rows of 1-7 KiB,
    # 14336 / 28672-wide gate/up/down) through K2, against the narrow/concat
    # oracle, with the arena window of the larger shard
    model = _real_shape_layer(geometry.LLAMA_3_1_8B if base == "8b" else geometry.LLAMA_3_1_70B)
    gpus = tuple(range(8))
    store = ShardedWeightStore(model, gpus, max_slices=max(8 // tp_old, 8 // tp_new))
    store.load(workloads.tp_groups(gpus, tp_old))
    pieces = host_pieces(store)
    new_groups = workloads.tp_groups(gpus, tp_new)
    stats = store.reshard(new_groups)
    torch.cuda.synchronize()
    check_against_oracle(store, pieces, new_groups)
    assert store.verify() == 0
    assert (stats.local_bytes, stats.remote_bytes) == expected_volume(
        workloads.tp_groups(gpus, tp_old), new_groups, store.bytes_per_slice)[:2]
    store.finish()
