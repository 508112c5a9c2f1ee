"""tpr_switch_prepare (the host half of the one-call switch) against the
two-step path: plan_repartition (migration.py:137-189) + the K3 records of
tpr_kv_records. CPU only: no device call."""

import ctypes

import numpy as np
import pytest

from paper_2605_05467_b200 import _native, migration as M, workloads
from paper_2605_05467_b200.geometry import KvGeometry

KV = KvGeometry(layers=2, head_dim=32, total_heads=8)
KVB = KV.kv_bytes_per_token_per_head


class Tables:
    """Host tables of a cluster whose requests sit in ``layouts``."""

    def __init__(self, gpus, layouts, units=10_000, max_req=64):
        self.gpus = tuple(gpus)
        self.gpu_lut = np.full(max(self.gpus) + 1, -1, np.int64)
        self.gpu_lut[list(self.gpus)] = np.arange(len(self.gpus))
        self.ids = np.asarray(self.gpus, np.int64)
        self.req_lut = np.full(1024, -1, np.int64)
        self.slot_ctx = np.full(max_req, -1, np.int32)
        self.owner = np.full((max_req, KV.total_heads), -1, np.int32)
        slot = 0
        for lay in layouts:
            for rid, ctx in lay.requests:
                self.req_lut[rid] = slot
                self.slot_ctx[slot] = ctx
                for h, g in enumerate(lay.owners()):
                    self.owner[slot, h] = self.gpu_lut[g]
                slot += 1
        self.geo = _native.KvGeometryC(KV.layers, KV.head_dim, KV.dtype_bytes, KV.block_tokens,
                                       KV.total_heads, 64, max_req, units)
        self.cl = _native.KvClusterC()
        self.cl.n_gpus = len(self.gpus)
        for s in range(len(self.gpus)):
            self.cl.ring_head[s], self.cl.ring_tail[s], self.cl.units[s] = 0, units, units
        self.plan = np.zeros((max_req * KV.total_heads, 6), np.int64)
        self.rec = np.zeros((max_req * KV.total_heads, 6), np.int32)

    def prepare(self, old, new, validate=True, mode=0):
        t = _native.SwitchTablesC()
        t.mode = mode
        t.gpu_lut, t.gpu_lut_len = self.gpu_lut.ctypes.data, len(self.gpu_lut)
        t.gpu_ids = self.ids.ctypes.data
        t.req_lut, t.req_lut_len = self.req_lut.ctypes.data, len(self.req_lut)
        t.slot_ctx, t.owner, t.kvb, t.validate = (self.slot_ctx.ctypes.data, self.owner.ctypes.data,
                                                  KVB, int(validate))
        t.plan, t.plan_cap, t.records = self.plan.ctypes.data, len(self.plan), self.rec.ctypes.data
        blob = M.pack_layouts(old, new)
        rc = _native.load().tpr_switch_prepare(ctypes.byref(self.geo), ctypes.byref(self.cl),
                                               blob.buffer_info()[0], len(blob), ctypes.byref(t))
        return rc, t


def expected_records(tab, arr):
    rows = []
    for s, d, r, lo, hi, _ in arr.tolist():
        rs = tab.req_lut[r]
        rows.append((tab.gpu_lut[s], tab.gpu_lut[d], rs, lo, hi, tab.slot_ctx[rs]))
    return np.asarray(rows, np.int32).reshape(-1, 6)


@pytest.mark.parametrize("a,b", [(a, b) for a in (1, 2, 4, 8) for b in (1, 2, 4, 8) if a != b])
def test_prepare_matches_two_step_path(a, b):
    gpus = tuple(range(3, 11))  # non-zero ids exercise the lookup tables
    rng = np.random.default_rng(a * 10 + b)
    reqs = [(int(r), int(c)) for r, c in zip(rng.permutation(900)[:21], rng.integers(1, 300, 21))]
    old = workloads.round_robin(workloads.tp_groups(gpus, a), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, b), reqs, 8)
    tab = Tables(gpus, old)
    rc, t = tab.prepare(old, new)
    assert rc == 0, _native.load().tpr_last_error()
    want = M.plan_repartition(old, new, KVB).as_array()
    assert t.n_plan == len(want)
    assert np.array_equal(tab.plan[: t.n_plan], want)
    assert np.array_equal(tab.rec[: t.n_plan], expected_records(tab, want))
    assert t.plan_bytes == int(want[:, 5].sum())
    units = [(hi - lo) * KV.blocks(c) for _, _, _, lo, hi, c in expected_records(tab, want).tolist()]
    assert t.total_units == sum(units)
    for s, g in enumerate(gpus):
        assert t.in_units[s] == sum(u for (x, u) in zip(want.tolist(), units) if x[1] == g)
        assert t.out_units[s] == sum(u for (x, u) in zip(want.tolist(), units) if x[0] == g)


def test_reference_errors_and_duplicates_take_the_general_path():
    gpus = (0, 1, 2, 3)
    reqs = [(1, 50), (2, 70), (3, 9)]
    old = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, 4), reqs, 8)
    tab = Tables(gpus, old)
    nf = _native.TPR_ENOTFOUND
    # GPU sets differ (migration.py:150-155)
    assert tab.prepare(old, [M.KvLayout((0, 1), 2, 8, tuple(reqs))])[0] == nf
    # context length changed (:172-173)
    assert tab.prepare(old, [M.KvLayout(gpus, 4, 8, ((1, 50), (2, 71), (3, 9)))])[0] == nf
    # new layouts must carry exactly the old requests (:160-166)
    assert tab.prepare(old, [M.KvLayout(gpus, 4, 8, ((1, 50), (2, 70)))])[0] == nf
    # an old request id that repeats: last-one-wins semantics stay in Python
    dup = [M.KvLayout((0, 1), 2, 8, ((1, 50),)), M.KvLayout((2, 3), 2, 8, ((1, 50), (2, 70), (3, 9)))]
    assert tab.prepare(dup, new)[0] == nf
    # a head that is not on its source (validate), and a request unknown to the tables
    moved = [M.KvLayout((2, 3), 2, 8, ((1, 50),)), M.KvLayout((0, 1), 2, 8, ((2, 70), (3, 9)))]
    assert tab.prepare(moved, new)[0] == nf
    assert tab.prepare(moved, new, validate=False)[0] == 0
    stranger = [M.KvLayout(gpus, 4, 8, ((99, 5),))]
    assert tab.prepare(stranger, stranger)[0] == 0  # identity: empty plan, nothing to look up
    assert tab.prepare(stranger, [M.KvLayout((1, 0, 2, 3), 4, 8, ((99, 5),))])[0] == nf
    # out of KV units on a destination
    tab.cl.ring_tail[1] = 3
    assert tab.prepare(old, new)[0] == nf


def test_plan_capacity_is_reported():
    gpus = (0, 1)
    reqs = [(i, 40) for i in range(5)]
    old = workloads.round_robin(workloads.tp_groups(gpus, 1), reqs, 8)
    new = workloads.round_robin(workloads.tp_groups(gpus, 2), reqs, 8)
    tab = Tables(gpus, old)
    tab.plan = np.zeros((2, 6), np.int64)
    rc, t = tab.prepare(old, new)
    assert rc == _native.TPR_ECAPACITY and t.n_plan == len(reqs) * 8


def test_struct_size_matches_header():
    # tpr_switch_tables_t (include/tpr.h), 496 bytes: 28 pointer/int64 fields, four
    # int32 and two [TPR_MAX_GPUS] int64 arrays
    assert ctypes.sizeof(_native.SwitchTablesC) == 28 * 8 + 4 * 4 + 2 * 8 * _native.TPR_MAX_GPUS


def test_packed_layout_is_cached_and_exact():
    lay = M.KvLayout((4, 5), 2, 8, ((7, 100), (9, 3)))
    assert lay.packed() == (8, 2, 4, 5, 2, 7, 100, 9, 3)
    assert lay.packed() is lay.packed()
    blob = M.pack_layouts([lay], lay)
    assert list(blob) == [1, 1, *lay.packed(), *lay.packed()]
    blob = M.pack_layouts([lay], lay, release=[11, 12])  # + the release section
    assert list(blob) == [1, 1, *lay.packed(), *lay.packed(), 2, 11, 12]


@pytest.mark.parametrize("src,dst", [((0, 1), (4, 5, 6, 7)), ((2,), (3,)), ((0, 1, 2, 3), (4, 5)),
                                     ((4, 5), (5, 4))])
def test_head_transfers_mode_matches_reference_planner(src, dst):
    # the engine's handoff path: head_transfers between arbitrary groups
    # (engine.py:571-589, migration.py:101-134), incl. disjoint GPU sets
    gpus = tuple(range(8))
    reqs = ((11, 70), (12, 16), (13, 1))
    old = M.KvLayout(src, len(src), 8, reqs)
    new = M.KvLayout(dst, len(dst), 8, reqs)
    tab = Tables(gpus, [old])
    rc, t = tab.prepare([old], [new], mode=_native.TPR_SWITCH_HEAD_TRANSFERS)
    assert rc == 0, _native.load().tpr_last_error()
    want = M.head_transfers_array(old, new, KVB).as_array()
    assert t.n_plan == len(want) and np.array_equal(tab.plan[: t.n_plan], want)
    assert np.array_equal(tab.rec[: t.n_plan], expected_records(tab, want))


def test_head_transfers_mode_takes_one_layout_each():
    gpus = (0, 1)
    a = M.KvLayout((0,), 1, 8, ((1, 5),))
    b = M.KvLayout((1,), 1, 8, ((1, 5),))
    tab = Tables(gpus, [a])
    rc, _ = tab.prepare([a, b], [b], mode=_native.TPR_SWITCH_HEAD_TRANSFERS)
    assert rc == -1


def _offsets_restated(rec: np.ndarray, filt: int, B: int) -> np.ndarray:
    """K3's three keyed exclusive scans (tpr_kernels.cu k3_scan_body) as plain
    loops: per record, units before it this caller moves, units before it its
    destination ring hands out, units before it its source ring takes back,
    and its own units this caller moves."""
    out = np.zeros((len(rec), 4), np.int64)
    mine, into, outof = 0, {}, {}
    for t, (s, d, _, lo, hi, ctx) in enumerate(rec.tolist()):
        u = (hi - lo) * (-(-ctx // B) if ctx > 0 else 0)
        m = u if (filt < 0 or s == filt) else 0
        out[t] = (mine, into.get(d, 0) if d >= 0 else 0, outof.get(s, 0) if s >= 0 else 0, m)
        mine += m
        if d >= 0:
            into[d] = into.get(d, 0) + u
        if s >= 0:
            outof[s] = outof.get(s, 0) + u
    return out


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("filt", [-1, 0, 3])
def test_record_offsets_match_the_k3_scan_restated(seed, filt):
    # tpr_record_offsets: the host-side scan K31 carries in its parameters
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 97))
    rec = np.empty((n, 6), np.int32)
    rec[:, 0] = rng.integers(-1, 8, n)
    rec[:, 1] = rng.integers(-1, 8, n)
    rec[:, 2] = rng.integers(0, 50, n)
    rec[:, 3] = rng.integers(0, 4, n)
    rec[:, 4] = rec[:, 3] + rng.integers(1, 5, n)
    rec[:, 5] = rng.integers(0, 3000, n)
    meta = np.full((n, 4), -7, np.int64)
    total = ctypes.c_int64(-1)
    _native.call("tpr_record_offsets", rec.ctypes.data, n, filt, 16, meta.ctypes.data,
                 ctypes.byref(total))
    want = _offsets_restated(rec, filt, 16)
    assert np.array_equal(meta, want)
    assert total.value == int(want[:, 3].sum())
