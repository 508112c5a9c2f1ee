"""ctypes binding of libtpr.so (the C ABI declared in include/tpr.h).

This is the only way the package reaches the device: there is no eager /
PyTorch fallback for the data path. If the library is missing or fails to
load, every device entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, Structure, c_char_p, c_int32, c_int64, c_uint8, c_uint64, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtpr.so"

TPR_ABI_VERSION = 2
TPR_MAX_GPUS = 16
TPR_XFER_FIELDS = 6
TPR_META_FIELDS = 4
TPR_TOTALS_LEN = 12 + 2 * TPR_MAX_GPUS  # + scratch words of the fused small switch
TPR_STATUS_WRONG_SOURCE = 1
TPR_STATUS_DST_OCCUPIED = 2
TPR_STATUS_BARRIER_TIMEOUT = 4
TPR_STATUS_OUT_OF_RANGE = 8
TPR_STATUS_RING_POISONED = 16
TPR_ENOTFOUND = -4  # an id outside the caller's lookup tables (use the Python maps)

# Every exported symbol of include/tpr.h; tests check the library exports all.
EXPORTS = (
    "tpr_set_copy_engine", "tpr_get_copy_engine", "tpr_set_tuning", "tpr_get_tuning",
    "tpr_version", "tpr_last_error", "tpr_device_info", "tpr_plan_heads", "tpr_plan_repartition",
    "tpr_kv_remap", "tpr_kv_migrate", "tpr_kv_migrate_ex", "tpr_kv_records", "tpr_record_offsets",
    "tpr_kv_apply_owner", "tpr_kv_switch",
    "tpr_switch_prepare", "tpr_kv_switch_layouts",
    "tpr_memcpy_h2d", "tpr_memcpy_d2h", "tpr_event_record",
    "tpr_copy_prepare", "tpr_weight_reshard", "tpr_reshard_buffer_bytes", "tpr_weight_reshard_host",
    "tpr_kv_fill", "tpr_pool_fill", "tpr_kv_verify", "tpr_matrix_fill",
    "tpr_matrix_verify", "tpr_baseline_copy_pages", "tpr_device_barrier", "tpr_device_alloc",
    "tpr_device_free",
    "tpr_ipc_get_handle", "tpr_ipc_open", "tpr_ipc_close",
)


class NativeUnavailable(RuntimeError):
    pass


class NativeError(RuntimeError):
    pass


class KvGeometryC(Structure):
    _fields_ = [
        ("layers", c_int32), ("head_dim", c_int32), ("dtype_bytes", c_int32),
        ("block_tokens", c_int32), ("total_heads", c_int32), ("max_blocks", c_int32),
        ("n_req_slots", c_int32), ("n_units", c_int32),
    ]


class KvClusterC(Structure):
    _fields_ = [
        ("n_gpus", c_int32), ("_pad", c_int32),
        ("pool", c_uint64 * TPR_MAX_GPUS),
        ("block_table", c_uint64 * TPR_MAX_GPUS),
        ("free_ring", c_uint64 * TPR_MAX_GPUS),
        ("ring_head", c_int64 * TPR_MAX_GPUS),
        ("ring_tail", c_int64 * TPR_MAX_GPUS),
        ("units", c_int64 * TPR_MAX_GPUS),
    ]


class CopySegC(Structure):
    _fields_ = [
        ("src", c_uint64), ("dst", c_uint64), ("rows", c_int64), ("row_bytes", c_int64),
        ("src_pitch", c_int64), ("dst_pitch", c_int64), ("flags", c_int64), ("_pad", c_int64),
    ]


class SwitchTablesC(Structure):
    _fields_ = [
        ("gpu_lut", c_void_p), ("gpu_lut_len", c_int64), ("gpu_ids", c_void_p),
        ("req_lut", c_void_p), ("req_lut_len", c_int64), ("slot_ctx", c_void_p),
        ("owner", c_void_p), ("kvb", c_int64), ("validate", c_int32), ("mode", c_int32),
        ("plan", c_void_p), ("plan_cap", c_int64), ("records", c_void_p),
        ("in_units", c_int64 * TPR_MAX_GPUS), ("out_units", c_int64 * TPR_MAX_GPUS),
        ("n_plan", c_int64), ("total_units", c_int64),
        ("d_xfers", c_void_p), ("d_meta", c_void_p), ("xfers_cap", c_int64),
        ("d_totals", c_void_p), ("d_work", c_void_p), ("work_cap", c_int64),
        ("d_status", c_void_p), ("plan_bytes", c_int64), ("h_status", c_void_p),
        ("k1_events", c_void_p * 2), ("n_records", c_int64), ("records_async", c_int32),
        ("ticket", c_int32), ("ring_head_io", c_void_p), ("ring_tail_io", c_void_p),
        ("start_event", c_void_p),
    ]


TPR_ECAPACITY = -3
TPR_MIGRATE_FULL_PAGES = 1
TPR_SWITCH_REPARTITION = 0
TPR_SWITCH_HEAD_TRANSFERS = 1

_P64 = POINTER(c_int64)
_P32 = POINTER(c_int32)

_SIGNATURES = {
    "tpr_set_copy_engine": (c_int32, [c_int32]),
    "tpr_get_copy_engine": (c_int32, []),
    "tpr_set_tuning": (c_int32, [c_char_p, c_int64]),
    "tpr_get_tuning": (c_int64, [c_char_p]),
    "tpr_version": (c_int32, []),
    "tpr_last_error": (c_char_p, []),
    "tpr_device_info": (c_int32, [_P32, _P32, _P32]),
    "tpr_plan_heads": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_int32, c_int64, c_int64, c_void_p, _P64]),
    "tpr_plan_repartition": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_int32, c_int64, c_int64, c_void_p, _P64]),
    "tpr_kv_remap": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p, c_int32,
                               c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                               c_void_p, c_void_p]),
    "tpr_kv_migrate": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p, c_int64,
                                 c_void_p]),
    "tpr_kv_migrate_ex": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p, c_int64,
                                    c_int32, c_void_p]),
    "tpr_kv_records": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int32, c_void_p,
                                 c_int64, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int64,
                                 c_int32, c_void_p, c_void_p, c_void_p, _P64]),
    "tpr_kv_apply_owner": (c_int32, [c_void_p, c_int64, c_void_p, c_int32]),
    "tpr_record_offsets": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "tpr_event_record": (c_int32, [c_void_p, c_void_p]),
    "tpr_kv_switch": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p, c_void_p,
                                c_int32, c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                c_void_p]),
    "tpr_switch_prepare": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p, c_int64,
                                     POINTER(SwitchTablesC)]),
    "tpr_kv_switch_layouts": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p,
                                        c_int64, POINTER(SwitchTablesC), c_void_p]),
    "tpr_memcpy_h2d": (c_int32, [c_uint64, c_void_p, c_uint64, c_void_p]),
    "tpr_memcpy_d2h": (c_int32, [c_void_p, c_uint64, c_uint64, c_void_p]),
    "tpr_copy_prepare": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, _P64]),
    "tpr_weight_reshard": (c_int32, [c_void_p, c_void_p, c_int32, c_int64, c_int64, c_void_p,
                                     c_void_p]),
    "tpr_reshard_buffer_bytes": (ctypes.c_size_t, [c_int32]),
    "tpr_weight_reshard_host": (c_int32, [c_void_p, c_int32, c_int64, c_uint64, c_uint64, _P64,
                                          c_void_p]),
    "tpr_kv_fill": (c_int32, [POINTER(KvGeometryC), POINTER(KvClusterC), c_void_p, c_void_p,
                              c_int64, c_uint64, c_void_p]),
    "tpr_pool_fill": (c_int32, [POINTER(KvGeometryC), c_uint64, c_int32, c_uint64, c_void_p]),
    "tpr_kv_verify": (c_int32, [POINTER(KvGeometryC), c_uint64, c_void_p, c_void_p, c_void_p,
                                c_int32, c_uint64, c_void_p, c_void_p]),
    "tpr_matrix_fill": (c_int32, [c_uint64, c_int64, c_int64, c_int64, c_int64, c_int64,
                                  c_int64, c_uint64, c_int32, c_void_p]),
    "tpr_matrix_verify": (c_int32, [c_uint64, c_int64, c_int64, c_int64, c_int64, c_int64,
                                    c_int64, c_uint64, c_int32, c_void_p, c_void_p]),
    "tpr_baseline_copy_pages": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                          c_void_p]),
    "tpr_device_barrier": (c_int32, [c_void_p, c_int32, c_int32, c_uint64, c_uint64, c_void_p,
                                     c_void_p]),
    "tpr_device_alloc": (c_int32, [c_uint64, POINTER(c_uint64)]),
    "tpr_device_free": (c_int32, [c_uint64]),
    "tpr_ipc_get_handle": (c_int32, [c_uint64, POINTER(c_uint8)]),
    "tpr_ipc_open": (c_int32, [POINTER(c_uint8), POINTER(c_uint64)]),
    "tpr_ipc_close": (c_int32, [c_uint64]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libtpr.so once; raise NativeUnavailable when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: run `python -m paper_2605_05467_b200.build` "
            "(there is no CPU fallback for the TP-reconfiguration data path)"
        )
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tpr_version() != TPR_ABI_VERSION:
        raise NativeUnavailable(
            f"libtpr ABI {lib.tpr_version()} != expected {TPR_ABI_VERSION}; rebuild"
        )
    _lib = lib
    return lib


ENGINES = {"vector": 0, "bulk": 1}


def k3_fuse_units() -> int:
    """Plan size (units) up to which K3 runs as one fused CTA."""
    return int(load().tpr_get_tuning(b"k3_fuse_units"))


TUNING_KEYS = ("k3_fuse_units", "tensor_partial", "k31")


def set_tuning(key: str, value: int) -> None:
    """Launch-path knob of tpr_kv_switch (see include/tpr.h)."""
    call("tpr_set_tuning", key.encode(), int(value))


def get_tuning(key: str) -> int:
    return int(load().tpr_get_tuning(key.encode()))


def kv_switch_launches(units: int, n_transfers: int = 0) -> int:
    """Kernels one tpr_kv_switch launches: K31 alone for a small plan (<=
    k3_fuse_units pages, <= 96 transfers, TMA engine), else K3 (fused, or scan +
    remap) + K1."""
    if units <= 0:
        return 0
    if units <= k3_fuse_units():
        if 0 < n_transfers <= 96 and get_tuning("k31") and copy_engine() == "bulk":
            return 1
        return 2
    return 3


def set_copy_engine(name: str) -> None:
    """K1/K2 copy engine: "bulk" (TMA, default) or "vector" (16-B ld/st)."""
    if name not in ENGINES:
        raise ValueError(f"unknown copy engine {name!r}; choose from {sorted(ENGINES)}")
    call("tpr_set_copy_engine", ENGINES[name])


def last_engines() -> tuple[str | None, str | None]:
    """The copy engine the last K1 and K2 launches used (None before the first)."""
    names = {v: k for k, v in ENGINES.items()}
    return tuple(names.get(int(load().tpr_get_tuning(k)))
                 for k in (b"k1_engine_last", b"k2_engine_last"))


def copy_engine() -> str:
    v = load().tpr_get_copy_engine()
    return next(k for k, e in ENGINES.items() if e == v)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().tpr_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
