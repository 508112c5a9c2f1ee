"""Property tests (hypothesis) for the native planner against the oracle
restatement: random GPU ids, mixed TP levels across groups, random request
order, disjoint groups through head_transfers (engine path)."""

from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import plan_oracle as PO
from paper_2605_05467_b200 import migration as M

HEADS = st.sampled_from([1, 2, 4, 8, 16])


@st.composite
def partitions(draw, gpus, H):
    """Split `gpus` into consecutive groups whose sizes divide H."""
    out, i = [], 0
    while i < len(gpus):
        sizes = [s for s in (1, 2, 4, 8) if H % s == 0 and i + s <= len(gpus)]
        s = draw(st.sampled_from(sizes))
        out.append(tuple(gpus[i:i + s]))
        i += s
    return out


@st.composite
def transitions(draw):
    H = draw(HEADS)
    n = draw(st.integers(1, 8))
    gpus = draw(st.lists(st.integers(0, 1000), min_size=n, max_size=n, unique=True))
    old_groups = draw(partitions(gpus, H))
    new_groups = draw(partitions(draw(st.permutations(gpus)), H))
    n_req = draw(st.integers(0, 12))
    ids = draw(st.lists(st.integers(0, 10**6), min_size=n_req, max_size=n_req, unique=True))
    ctxs = draw(st.lists(st.integers(0, 5000), min_size=n_req, max_size=n_req))
    reqs = list(zip(ids, ctxs))
    old_assign = draw(st.lists(st.integers(0, len(old_groups) - 1), min_size=n_req, max_size=n_req))
    new_assign = draw(st.lists(st.integers(0, len(new_groups) - 1), min_size=n_req, max_size=n_req))
    order = draw(st.permutations(range(n_req)))
    old = [[] for _ in old_groups]
    new = [[] for _ in new_groups]
    for i, r in enumerate(reqs):
        old[old_assign[i]].append(r)
    for i in order:
        new[new_assign[i]].append(reqs[i])
    kvb = draw(st.sampled_from([1, 16, 4096, 16384, 40960]))
    return H, old_groups, old, new_groups, new, kvb


@settings(max_examples=300, deadline=None)
@given(transitions())
def test_plan_matches_oracle(t):
    H, og, old, ng, new, kvb = t
    lo = [M.KvLayout(g, len(g), H, tuple(r)) for g, r in zip(og, old)]
    ln = [M.KvLayout(g, len(g), H, tuple(r)) for g, r in zip(ng, new)]
    plan = M.plan_repartition(lo, ln, kvb)
    want = PO.plan([(g, H, r) for g, r in zip(og, old)], [(g, H, r) for g, r in zip(ng, new)], kvb)
    assert plan.as_array().tolist() == [list(m) for m in want]
    assert M.apply_plan(lo, plan) == M.layout_placement(ln)
    for s, d, rid, a, b, nb in plan.as_array().tolist():
        assert s != d and a < b


@settings(max_examples=200, deadline=None)
@given(st.data())
def test_head_transfers_disjoint_groups(data):
    H = data.draw(HEADS)
    sizes = [s for s in (1, 2, 4, 8) if H % s == 0]
    a = data.draw(st.sampled_from(sizes))
    b = data.draw(st.sampled_from(sizes))
    ids = data.draw(st.lists(st.integers(0, 64), min_size=a + b, max_size=a + b, unique=True))
    reqs = [(i, data.draw(st.integers(1, 999))) for i in range(data.draw(st.integers(0, 5)))]
    old = M.KvLayout(tuple(ids[:a]), a, H, tuple(reqs))
    new = M.KvLayout(tuple(ids[a:]), b, H, tuple(reqs))
    got = [[t.src_gpu, t.dst_gpu, t.request_id, t.head_lo, t.head_hi, t.bytes]
           for t in M.head_transfers(old, new, 4096)]
    want = [list(m) for r, c in reqs for m in PO.request_moves(old.group, new.group, H, r, c, 4096)]
    assert got == want
    # disjoint groups: every head of every request moves
    assert sum(t[4] - t[3] for t in got) == H * len(reqs)


def _both_paths(lo, ln, kvb):
    """plan_repartition through the row walk and through libtpr's
    tpr_plan_repartition (the default path)."""
    out = []
    saved = M._NATIVE_MIN_REQUESTS
    for threshold in (10**9, 0):
        M._NATIVE_MIN_REQUESTS = threshold
        try:
            out.append(("ok", M.plan_repartition(lo, ln, kvb).as_array().tolist()))
        except M.MigrationError as exc:
            out.append(("err", str(exc)))
        finally:
            M._NATIVE_MIN_REQUESTS = saved
    return out


@settings(max_examples=300, deadline=None)
@given(transitions(), st.sampled_from(["none", "drop", "ctx", "dup_old", "dup_new"]), st.data())
def test_native_repartition_matches_row_walk(t, corrupt, data):
    """Plans and error messages agree between the two planning paths,
    including invalid inputs (missing / duplicated requests, changed context)."""
    H, og, old, ng, new, kvb = t
    old = [list(r) for r in old]
    new = [list(r) for r in new]
    flat_new = [(i, j) for i, rs in enumerate(new) for j in range(len(rs))]
    if corrupt != "none" and flat_new:
        i, j = data.draw(st.sampled_from(flat_new))
        rid, ctx = new[i][j]
        if corrupt == "drop":
            del new[i][j]
        elif corrupt == "ctx":
            new[i][j] = (rid, ctx + 1)
        elif corrupt == "dup_old":
            old[0].append((rid, ctx))
        else:
            new[i].append((rid, ctx))
    lo = [M.KvLayout(g, len(g), H, tuple(r)) for g, r in zip(og, old)]
    ln = [M.KvLayout(g, len(g), H, tuple(r)) for g, r in zip(ng, new)]
    rows, vec = _both_paths(lo, ln, kvb)
    assert rows == vec
