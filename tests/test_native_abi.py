"""The C-ABI library loads, exports every symbol of include/tpr.h, and its
host-only entry points behave (no device calls here)."""

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2605_05467_b200 import _native


def declared_symbols():
    text = (ROOT / "include" / "tpr.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(tpr_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_symbols()
    assert len(names) >= 15
    assert set(names) == set(_native.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name


def test_tuning_knobs_roundtrip():
    lib = _native.load()
    saved = {k: _native.get_tuning(k) for k in _native.TUNING_KEYS}
    try:
        assert saved["k3_fuse_units"] >= 0 and saved["k31"] in (0, 1, 2, 3)
        _native.set_tuning("k3_fuse_units", 0)
        assert _native.get_tuning("k3_fuse_units") == 0
        _native.set_tuning("tensor_partial", 5)
        assert _native.get_tuning("tensor_partial") == 1
        _native.set_tuning("k31", 9)
        assert _native.get_tuning("k31") == 3
        assert lib.tpr_set_tuning(b"nope", 1) == -1 and b"unknown tuning key" in lib.tpr_last_error()
        assert lib.tpr_set_tuning(b"k31", -1) == -1
        assert lib.tpr_set_tuning(b"pdl", 1) == -1  # retired knobs are unknown keys
        assert lib.tpr_get_tuning(b"nope") == -1
        _native.set_tuning("tensor_partial", 0)
        assert _native.get_tuning("tensor_partial") == 0
    finally:
        for k, v in saved.items():
            _native.set_tuning(k, v)


def test_abi_version():
    assert _native.load().tpr_version() == _native.TPR_ABI_VERSION


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_native.KvGeometryC) == 8 * 4
    assert ctypes.sizeof(_native.KvClusterC) == 8 + 6 * 8 * _native.TPR_MAX_GPUS
    assert ctypes.sizeof(_native.CopySegC) == 64


def test_planner_errors_are_reported():
    lib = _native.load()
    out = np.zeros((8, 6), np.int64)
    n = ctypes.c_int64()
    req = np.array([0], np.int64)
    ctx = np.array([10], np.int64)
    off = np.array([0], np.int32)
    tp3 = np.array([3], np.int32)
    ids = np.array([0, 1, 2], np.int64)
    rc = lib.tpr_plan_heads(1, req.ctypes.data, ctx.ctypes.data, off.ctypes.data, tp3.ctypes.data,
                            off.ctypes.data, tp3.ctypes.data, ids.ctypes.data, 8, 4096, 8,
                            out.ctypes.data, ctypes.byref(n))
    assert rc == -1
    assert b"divisible" in lib.tpr_last_error()


def test_planner_capacity_error():
    lib = _native.load()
    out = np.zeros((1, 6), np.int64)
    n = ctypes.c_int64()
    req = np.array([0], np.int64)
    ctx = np.array([10], np.int64)
    oo, ot = np.array([0], np.int32), np.array([1], np.int32)
    no, nt = np.array([1], np.int32), np.array([2], np.int32)
    ids = np.array([5, 6, 7], np.int64)  # old (5) -> new (6, 7): two runs
    rc = lib.tpr_plan_heads(1, req.ctypes.data, ctx.ctypes.data, oo.ctypes.data, ot.ctypes.data,
                            no.ctypes.data, nt.ctypes.data, ids.ctypes.data, 8, 4096, 1,
                            out.ctypes.data, ctypes.byref(n))
    assert rc == -3


def test_copy_prepare_normalises_and_counts():
    segs = (_native.CopySegC * 3)()
    # contiguous 2-D -> collapsed; 100 KiB at 32 KiB chunks = 4 items
    segs[0].src, segs[0].dst = 0x1000, 0x2000
    segs[0].rows, segs[0].row_bytes, segs[0].src_pitch, segs[0].dst_pitch = 25, 4096, 4096, 4096
    # strided rows of 1 KiB: 32 rows per item -> 10 rows = 1 item
    segs[1].src, segs[1].dst = 0x10000, 0x20000
    segs[1].rows, segs[1].row_bytes, segs[1].src_pitch, segs[1].dst_pitch = 10, 1024, 4096, 2048
    # unaligned
    segs[2].src, segs[2].dst = 0x3001, 0x4000
    segs[2].rows, segs[2].row_bytes, segs[2].src_pitch, segs[2].dst_pitch = 1, 100, 100, 100
    prefix = np.zeros(4, np.int64)
    n = ctypes.c_int64()
    _native.call("tpr_copy_prepare", ctypes.addressof(segs), 3, 32768, prefix.ctypes.data,
                 ctypes.byref(n))
    assert segs[0].rows == 1 and segs[0].row_bytes == 25 * 4096
    assert segs[0].flags == 1 and segs[1].flags == 1 and segs[2].flags == 0
    assert prefix.tolist() == [0, 4, 5, 6] and n.value == 6


def test_copy_prepare_rejects_bad_chunk():
    prefix = np.zeros(1, np.int64)
    n = ctypes.c_int64()
    with pytest.raises(_native.NativeError, match="multiple of 16"):
        _native.call("tpr_copy_prepare", None, 0, 100, prefix.ctypes.data, ctypes.byref(n))


def test_small_switch_entries_check_arguments_without_a_gpu():
    # argument checks that return before any CUDA call: a null event, bad
    # record-offset arguments; and tpr_record_offsets on an empty plan
    import ctypes
    lib = _native.load()
    assert lib.tpr_event_record(None, None) == -1 and b"null event" in lib.tpr_last_error()
    assert lib.tpr_record_offsets(None, 3, -1, 16, None, None) == -1
    assert lib.tpr_record_offsets(None, 0, -1, 0, None, None) == -1  # block_tokens < 1
    total = ctypes.c_int64(7)
    assert lib.tpr_record_offsets(None, 0, -1, 16, None, ctypes.byref(total)) == 0 and total.value == 0
