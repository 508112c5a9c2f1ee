"""numpy mirror of the synthetic-data pattern in csrc/tpr_common.cuh.

Used by tests to pin the device fill kernels; the data path never calls it.
"""

from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def page_key(seed: int, req_slot: int, head: int, block: int) -> np.uint64:
    ident = (np.uint64(req_slot) << np.uint64(40)) ^ (np.uint64(head) << np.uint64(24)) ^ np.uint64(block)
    return splitmix64(np.uint64(seed) ^ splitmix64(ident))


def unit_key(seed: int, slot: int, unit: int) -> np.uint64:
    ident = (np.uint64(slot) << np.uint64(48)) ^ np.uint64(unit) ^ np.uint64(0x5A5A000000000000)
    return splitmix64(np.uint64(seed) ^ splitmix64(ident))


def words(key, start_word: int, n: int) -> np.ndarray:
    w = np.arange(start_word, start_word + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return (splitmix64(np.uint64(key) + w) >> np.uint64(16)).astype(np.uint32)


def page_bytes(seed, req_slot, head, block, kv, ntok) -> np.ndarray:
    """Expected bytes of a page's valid tokens, as uint8 [rows, ntok*tok_bytes]."""
    key = page_key(seed, req_slot, head, block)
    rows = 2 * kv.layers
    pitch_w = kv.plane_bytes // 4
    nw = ntok * kv.tok_bytes // 4
    out = np.empty((rows, nw), dtype=np.uint32)
    for r in range(rows):
        out[r] = words(key, r * pitch_w, nw)
    return out.view(np.uint8)


def unit_garbage(seed, slot, unit, unit_bytes) -> np.ndarray:
    return words(unit_key(seed, slot, unit), 0, unit_bytes // 4).view(np.uint8)


def matrix(key: int, rows, cols, row0: int, col0: int, full_cols: int, elem_bytes: int = 2):
    r = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    c = np.arange(col0, col0 + cols, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        v = splitmix64(np.uint64(key) + r * np.uint64(full_cols) + c) >> np.uint64(24)
    return v.astype({1: np.uint8, 2: np.uint16, 4: np.uint32}[elem_bytes])
