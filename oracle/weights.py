"""ORACLE -- test infrastructure only.

Restatement of TP weight resharding as plain narrow/concatenate on host
arrays (the Megatron/SGLang convention the paper relies on, PAPER.md:307:
"under TP2, the first GPU ... uses the first half of each weight matrix"):

* column-parallel matrix (q/k/v, gate/up, embedding, lm_head): rank r of TP-N
  holds rows [r*R/N, (r+1)*R/N);
* row-parallel matrix (o, down): columns [r*C/N, (r+1)*C/N);
* replicated (norms): everything.

The reference only accounts this as GB per GPU (migration.py:295-306); the
tests pin the byte volumes to ``weight_memory("sharded", tp)`` and the
contents to this restatement.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(split: str, rows: int, cols: int, tp: int, rank: int):
    if split == "col":
        return (rank * rows // tp, (rank + 1) * rows // tp), (0, cols)
    if split == "row":
        return (0, rows), (rank * cols // tp, (rank + 1) * cols // tp)
    return (0, rows), (0, cols)


def assemble_full(pieces, rows: int, cols: int, dtype=np.uint16):
    """Rebuild a full matrix from (row_lo, col_lo, array) pieces held by the
    old shards; overlapping pieces must agree."""
    full = np.zeros((rows, cols), dtype=dtype)
    seen = np.zeros((rows, cols), dtype=bool)
    for r0, c0, arr in pieces:
        r1, c1 = r0 + arr.shape[0], c0 + arr.shape[1]
        prev = seen[r0:r1, c0:c1]
        if prev.any() and not np.array_equal(full[r0:r1, c0:c1][prev], arr[prev]):
            raise ValueError("old shards disagree on overlapping weights")
        full[r0:r1, c0:c1] = arr
        seen[r0:r1, c0:c1] = True
    return full, seen


def expected_shard(full: np.ndarray, split: str, tp: int, rank: int) -> np.ndarray:
    (r0, r1), (c0, c1) = shard_bounds(split, full.shape[0], full.shape[1], tp, rank)
    return full[r0:r1, c0:c1]
