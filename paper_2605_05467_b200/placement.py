"""Placement decisions around a TP switch.

* ``reuse_rank_order`` -- migration-minimising GPU order for a new TP group.
  The reference keeps identical groups in place (policy.py:285-311,
  ``_match_previous``) but takes new groups' rank order as given, and rank
  order fixes which heads each GPU owns (migration.py:27). A TP-N group has N!
  rank orders. Picking the one that maximises the KV bytes already resident
  on the right GPU is a linear assignment of ranks to GPUs. The gain of
  (rank r, gpu g) is the bytes of heads [r*H/N, (r+1)*H/N) already on g. It is
  opt-in, because it changes the plan the reference would produce.

* ``kv_capacity_decisions`` -- destination admission/eviction exactly as the
  reference's controller hook decides it (``Simulator._enforce_kv_capacity``,
  engine.py:623-645, with ``kv_accounting`` on, engine.py:600-601): the budget
  is ``(gpu_memory_gb - weight_full_copy_gb) * 1e9 * tp`` bytes, ``used``
  counts the requests already running on the group, arrivals are taken
  feasible first, then by arrival time (a stable sort), and a best-effort
  arrival that does not fit is evicted while a feasible one is always kept.
  Pinned to the reference's own decisions (tests/golden/kv_capacity.json.gz).
  ``ReconfigurationExecutor.switch(arrivals=...)`` applies it inside the switch
  and frees the evicted requests' pages in the same native call.

* ``enforce_kv_capacity`` -- the same rule against the destination GPUs'
  actual free pages (the ring counters) instead of the byte budget.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .migration import KvLayout, MigrationError

FEASIBLE = "feasible"        # engine.py:33
BEST_EFFORT = "best_effort"  # engine.py:34


def resident_gain(old_layouts: Sequence[KvLayout], new_gpus: Sequence[int], kvb: int) -> np.ndarray:
    """gain[r, i] = bytes of rank r's heads already on new_gpus[i]."""
    H = old_layouts[0].total_heads if old_layouts else 1
    N = len(new_gpus)
    if H % N:
        raise MigrationError(f"total_heads={H} not divisible by tp={N}")
    per = H // N
    col = {g: i for i, g in enumerate(new_gpus)}
    gain = np.zeros((N, N), dtype=np.float64)
    for lay in old_layouts:
        owners = lay.owners()
        tokens = sum(c for _, c in lay.requests)
        for h, g in enumerate(owners):
            if g in col:
                gain[h // per, col[g]] += tokens * kvb
    return gain


def reuse_rank_order(old_layouts: Sequence[KvLayout], new_gpus: Sequence[int], kvb: int) -> tuple:
    """GPU order for a new group that keeps the most KV bytes in place."""
    from scipy.optimize import linear_sum_assignment

    gain = resident_gain(old_layouts, new_gpus, kvb)
    rows, cols = linear_sum_assignment(-gain)
    order = [None] * len(new_gpus)
    for r, c in zip(rows, cols):
        order[r] = new_gpus[c]
    # ties: keep the caller's order when it is already optimal
    base = np.trace(gain)
    best = gain[rows, cols].sum()
    return tuple(new_gpus) if base >= best else tuple(order)


def reuse_layouts(old_layouts: Sequence[KvLayout], new_layouts: Sequence[KvLayout],
                  kvb: int) -> list[KvLayout]:
    """``new_layouts`` with every group's rank order replaced by
    ``reuse_rank_order`` over the old placement of that group's requests (the
    same GPUs, requests and TP degree; only which rank each GPU is changes)."""
    out = []
    for lay in new_layouts:
        rid = {r for r, _ in lay.requests}
        sub = [KvLayout(o.group, o.tp, o.total_heads,
                        tuple((r, c) for r, c in o.requests if r in rid)) for o in old_layouts]
        order = reuse_rank_order(sub, lay.group, kvb) if lay.requests else tuple(lay.group)
        out.append(KvLayout(tuple(order), lay.tp, lay.total_heads, lay.requests))
    return out


@dataclass
class Arrival:
    request_id: int
    context_len: int
    label: str = FEASIBLE
    arrival_time: float = 0.0


@dataclass(frozen=True)
class KvBudget:
    """The reference's KV budget of a destination group (engine.py:623-628)."""

    gpu_memory_gb: float
    weight_full_copy_gb: float

    def bytes(self, tp: int) -> float:
        return (self.gpu_memory_gb - self.weight_full_copy_gb) * 1e9 * tp


def kv_capacity_decisions(arrivals: Sequence[Arrival], budget_bytes: float, used_bytes: int,
                          kv_bytes_per_token: int):
    """(kept, evicted) of engine.py:629-645: ``need`` = context x total KV heads
    x bytes per token per head (engine.py:246-251); kept in the decision order
    (feasible first, then arrival time), evicted in the order they are
    re-queued."""
    kept, evicted = [], []
    used = used_bytes
    for a in sorted(arrivals, key=lambda a: (a.label == BEST_EFFORT, a.arrival_time)):
        need = a.context_len * kv_bytes_per_token
        if used + need > budget_bytes and a.label == BEST_EFFORT:
            evicted.append(a)
        else:
            used += need
            kept.append(a)
    return kept, evicted


def enforce_kv_capacity(cluster, layout: KvLayout, arrivals: Sequence[Arrival]):
    """Split arrivals into (kept, evicted) against the destination group's
    free pages. Each GPU of ``layout`` receives H/N heads of every kept arrival,
    so the per-GPU need is pages(ctx) * H/N. Order and rule follow
    engine.py:630-645: feasible first, then oldest. Best-effort arrivals that
    do not fit are evicted; feasible arrivals are always kept."""
    per = layout.heads_per_rank
    free = {g: cluster.free_units(g) for g in layout.group}
    kept, evicted = [], []
    for a in sorted(arrivals, key=lambda a: (a.label == BEST_EFFORT, a.arrival_time)):
        need = cluster.kv.blocks(a.context_len) * per
        fits = all(free[g] >= need for g in layout.group)
        if not fits and a.label == BEST_EFFORT:
            evicted.append(a)
            continue
        for g in layout.group:
            free[g] -= need
        kept.append(a)
    return kept, evicted
