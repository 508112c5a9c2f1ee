"""ORACLE -- test infrastructure only (tests/, smoke(), bench.py cpu_baseline).

ctypes wrapper of oracle/kvmove.c (C restatement of plan execution on paged
pools) plus a tiny pure-Python restatement used to pin the C one.
"""

from __future__ import annotations

import ctypes
import shutil
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "kvmove.c"
LIB = HERE / "liboracle.so"


class OracleGeo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "layers", "head_dim", "dtype_bytes", "block_tokens", "total_heads", "max_blocks",
        "n_req_slots", "n_units")]


def build(force: bool = False) -> Path:
    if not force and LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("no C compiler for the oracle")
    subprocess.run([cc, "-O3", "-march=native", "-fopenmp", "-shared", "-fPIC", str(SRC),
                    "-o", str(LIB)], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
        _lib.oracle_kv_migrate.restype = ctypes.c_int64
        _lib.oracle_kv_migrate.argtypes = [
            ctypes.POINTER(OracleGeo), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
            ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]
        _lib.oracle_copy_blocks.restype = None
        _lib.oracle_copy_blocks.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 6 + [ctypes.c_int32]
        _lib.oracle_max_threads.restype = ctypes.c_int32
        _lib.oracle_fill.restype = None
        _lib.oracle_fill.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint8, ctypes.c_int32]
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def filled(nbytes: int, value: int = 1, n_threads: int = 0) -> np.ndarray:
    """A uint8 host buffer of ``nbytes``, first-touched by all threads."""
    a = np.empty(nbytes, np.uint8)
    lib().oracle_fill(a.ctypes.data, nbytes, value, n_threads)
    return a


def _ptrs(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def kv_migrate(geo: dict, pools, tables, rings, ring_head, ring_tail, records: np.ndarray,
               n_threads: int = 0):
    """Execute int64 [n, 6] slot records (src, dst, req_slot, lo, hi, ctx) in place.

    Mutates pools/tables/rings (numpy arrays; ``pools=None`` replays block
    tables, free rings and ring counters only) and returns
    (pages moved, status bits, ring_head, ring_tail)."""
    g = OracleGeo(**geo)
    heads = np.asarray(ring_head, dtype=np.int64).copy()
    tails = np.asarray(ring_tail, dtype=np.int64).copy()
    rec = np.ascontiguousarray(records, dtype=np.int64)
    status = ctypes.c_int32(0)
    lens = np.array([len(r) for r in rings], dtype=np.int64)  # a ring's length is its modulus
    n = lib().oracle_kv_migrate(ctypes.byref(g), None if pools is None else _ptrs(pools),
                                _ptrs(tables), _ptrs(rings),
                                lens.ctypes.data, heads.ctypes.data, tails.ctypes.data,
                                rec.ctypes.data, len(rec), n_threads, ctypes.byref(status))
    if n < 0:
        raise MemoryError("oracle allocation failed")
    return int(n), status.value, heads.tolist(), tails.tolist()


def copy_blocks(blocks, n_threads: int = 0) -> None:
    """blocks: list of (dst ndarray, dst byte offset, src ndarray, src byte offset,
    rows, row_bytes, src_pitch, dst_pitch)."""
    n = len(blocks)
    dst = (ctypes.c_void_p * n)(*[b[0].ctypes.data + b[1] for b in blocks])
    src = (ctypes.c_void_p * n)(*[b[2].ctypes.data + b[3] for b in blocks])
    rows = np.array([b[4] for b in blocks], np.int64)
    rb = np.array([b[5] for b in blocks], np.int64)
    sp = np.array([b[6] for b in blocks], np.int64)
    dp = np.array([b[7] for b in blocks], np.int64)
    lib().oracle_copy_blocks(n, dst, src, rows.ctypes.data, rb.ctypes.data, sp.ctypes.data,
                             dp.ctypes.data, n_threads)


def kv_migrate_py(geo: dict, pools, tables, rings, ring_head, ring_tail, records):
    """Pure-Python page-by-page restatement (small cases only)."""
    H, MB, B = geo["total_heads"], geo["max_blocks"], geo["block_tokens"]
    tok = geo["head_dim"] * geo["dtype_bytes"]
    plane = B * tok
    unit = plane * 2 * geo["layers"]
    heads, tails = list(ring_head), list(ring_tail)
    status = 0
    moves = []
    for src, dst, req, lo, hi, ctx in np.asarray(records).tolist():
        pages = -(-ctx // B)
        for h in range(lo, hi):
            for b in range(pages):
                # the rules of tpr_kernels.cu k3_page / kvmove.c
                ok = 0 <= h < H and b < MB and 0 <= req < geo["n_req_slots"]
                status |= 0 if ok else 8
                su = du = -1
                if src >= 0:
                    if ok:
                        tb_s = tables[src].reshape(-1, H, MB)
                        su = int(tb_s[req, h, b])
                        if not 0 <= su < len(rings[src]):
                            status |= 1
                            su = -1
                        tb_s[req, h, b] = -1
                    rings[src][tails[src] % len(rings[src])] = su
                    tails[src] += 1
                if dst >= 0:
                    v = int(rings[dst][heads[dst] % len(rings[dst])])
                    heads[dst] += 1
                    if not 0 <= v < len(rings[dst]):
                        status |= 16
                    elif ok:
                        tb_d = tables[dst].reshape(-1, H, MB)
                        if tb_d[req, h, b] >= 0:
                            status |= 2
                        elif not (src >= 0 and su < 0):
                            tb_d[req, h, b] = v
                            du = v
                ntok = ctx - b * B if b == pages - 1 else B
                moves.append((su, du, src, dst, ntok))
    for su, du, src, dst, ntok in moves:
        if su < 0 or du < 0:
            continue
        for p in range(2 * geo["layers"]):
            s0 = su * unit + p * plane
            d0 = du * unit + p * plane
            pools[dst][d0:d0 + ntok * tok] = pools[src][s0:s0 + ntok * tok]
    return len(moves), status, heads, tails
