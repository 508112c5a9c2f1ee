"""The native switch bookkeeping (``tpr_kv_records`` / ``tpr_kv_apply_owner``,
host code in libtpr) against the Python restatement it replaces
(``PagedKvCluster._records_py`` + ``_reserve``): same records, unit deltas,
placement update and MigrationError text, on valid and corrupted plans.
CPU only: the cluster is built without device buffers."""

import ctypes

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2605_05467_b200 import _native, migration as M
from paper_2605_05467_b200.geometry import KvGeometry
from paper_2605_05467_b200.kvcache import PagedKvCluster


def host_cluster(gpu_ids, H, max_requests, reqs):
    """A PagedKvCluster holding only the host bookkeeping, requests placed in
    the canonical layouts of ``reqs`` = [(rid, ctx, group)]."""
    c = PagedKvCluster.__new__(PagedKvCluster)
    c.kv = KvGeometry(layers=2, head_dim=64, total_heads=H)
    c.gpu_ids = tuple(gpu_ids)
    c.slot_of = {g: i for i, g in enumerate(c.gpu_ids)}
    c.max_requests = max_requests
    c.owner = np.full((max_requests, H), -1, dtype=np.int32)
    c.slot_ctx = np.full(max_requests, -1, dtype=np.int32)
    c.req_slot, c.ctx_of = {}, {}
    ids = np.asarray(c.gpu_ids, dtype=np.int64)
    c._gpu_lut = np.full(int(ids.max()) + 1, -1, dtype=np.int64)
    c._gpu_lut[ids] = np.arange(len(ids))
    c._gpu_ids_arr = ids
    c._req_lut = np.full(16, -1, dtype=np.int64)
    c._n_units_c = ctypes.c_int64(0)
    c._cl = _native.KvClusterC()  # ring counters live in the C view of the cluster
    c._cl.n_gpus = len(gpu_ids)
    for s in range(len(gpu_ids)):
        c._cl.ring_head[s], c._cl.ring_tail[s] = 0, 10**9
    for rs, (rid, ctx, group) in enumerate(reqs):
        c.req_slot[rid] = rs
        c._set_req(rid, rs)
        c.ctx_of[rid] = ctx
        c.slot_ctx[rs] = ctx
        per = H // len(group)
        for r, g in enumerate(group):
            c.owner[rs, r * per:(r + 1) * per] = c.slot_of[g]
    return c


def run_both(c, plan, validate):
    arr = plan.as_array()
    out = {}
    try:
        rec = np.empty((len(arr), 6), dtype=np.int32)
        r = c._native_records(arr, validate, rec)
        out["native"] = ("fallback",) if r is None else (
            "ok", rec.tolist(), r[0], r[1].tolist(), r[2].tolist())
    except M.MigrationError as exc:
        out["native"] = ("err", str(exc))
    try:
        xf = c._records_py(arr, validate)
        total, in_u, out_u = c._reserve(xf)
        out["py"] = ("ok", xf.tolist(), total, list(map(int, in_u)), list(map(int, out_u)))
    except M.MigrationError as exc:
        out["py"] = ("err", str(exc))
    return out


@st.composite
def cases(draw):
    H = draw(st.sampled_from([1, 2, 4, 8]))
    n = draw(st.integers(1, 8))
    gpus = draw(st.lists(st.integers(0, 40), min_size=n, max_size=n, unique=True))
    sizes = [s for s in (1, 2, 4, 8) if H % s == 0 and s <= n]
    a = draw(st.sampled_from(sizes))
    b = draw(st.sampled_from(sizes))
    n_req = draw(st.integers(1, 10))
    rids = draw(st.lists(st.integers(0, 60), min_size=n_req, max_size=n_req, unique=True))
    ctxs = draw(st.lists(st.integers(0, 200), min_size=n_req, max_size=n_req))
    old_g = [tuple(gpus[i:i + a]) for i in range(0, n - a + 1, a)]
    new_g = [tuple(gpus[i:i + b]) for i in range(0, n - b + 1, b)]
    perm = draw(st.permutations(gpus))
    new_g = [tuple(perm[i:i + b]) for i in range(0, n - b + 1, b)] if draw(st.booleans()) else new_g
    reqs = [(r, c, draw(st.sampled_from(old_g))) for r, c in zip(rids, ctxs)]
    new_of = {r: draw(st.sampled_from(new_g)) for r in rids}
    return H, gpus, reqs, new_of, draw(st.sampled_from(["none", "bytes", "twice", "src", "gpu", "req",
                                                          "range", "bigid"])), draw(st.booleans())


@settings(max_examples=400, deadline=None)
@given(cases())
def test_native_records_match_python(case):
    H, gpus, reqs, new_of, corrupt, validate = case
    c = host_cluster(gpus, H, 16, reqs)
    rows = []
    for rid, ctx, og in reqs:
        old = M.KvLayout(og, len(og), H, ((rid, ctx),))
        ng = new_of[rid]
        new = M.KvLayout(ng, len(ng), H, ((rid, ctx),))
        rows.extend(M.head_transfers_array(old, new, c.kv.kv_bytes_per_token_per_head).as_array().tolist())
    if not rows:
        return
    if corrupt == "bytes":
        rows[0][5] += 1
    elif corrupt == "twice":
        rows.append(list(rows[-1]))
    elif corrupt == "src":
        rows[0][0] = rows[0][1]
    elif corrupt == "gpu":
        rows[-1][1] = 999
    elif corrupt == "req":
        rows[0][2] = 61
    elif corrupt == "range":
        rows[-1][4] = H + 1
    elif corrupt == "bigid":  # a request id beyond the lookup table: dict path
        rid = rows[0][2]
        rs = c.req_slot.pop(rid)
        c._req_lut[rid] = -1
        c.req_slot[10**12] = rs
        c.ctx_of[10**12] = c.ctx_of.pop(rid)
        for r in rows:
            if r[2] == rid:
                r[2] = 10**12
    plan = M.MigrationPlan.from_array(np.asarray(rows, dtype=np.int64))
    got = run_both(c, plan, validate)
    if got["native"] == ("fallback",):
        assert corrupt in ("gpu", "req", "bigid")
        return
    assert got["native"] == got["py"]


def test_apply_owner_matches_numpy():
    rng = np.random.default_rng(0)
    H, R = 8, 12
    owner = rng.integers(0, 4, size=(R, H)).astype(np.int32)
    want = owner.copy()
    recs = []
    for r in range(R):
        lo = int(rng.integers(0, H))
        hi = int(rng.integers(lo + 1, H + 1))
        d = int(rng.integers(0, 4))
        recs.append((0, d, r, lo, hi, 5))
        want[r, lo:hi] = d
    rec = np.asarray(recs, dtype=np.int32)
    _native.call("tpr_kv_apply_owner", rec.ctypes.data, len(rec), owner.ctypes.data, H)
    assert (owner == want).all()


def test_records_errors_are_reference_text():
    c = host_cluster((3, 5), 4, 4, [(7, 40, (3,))])
    plan = M.MigrationPlan.from_array(np.array([[5, 3, 7, 0, 4, 4 * 40 * c.kv.kv_bytes_per_token_per_head]]))
    with pytest.raises(M.MigrationError, match="transfer of request 7 head 0 from gpu 5, but it is on 3"):
        c.records(plan)
