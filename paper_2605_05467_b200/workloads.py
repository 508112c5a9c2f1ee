"""The BASELINE.json workloads as old/new KvLayouts + weight groups.

Requests are assigned round-robin over the TP groups, the way the reference's
tests build multi-group layouts (pkg/tests/test_migration.py:131-135).
"""

from __future__ import annotations

from dataclasses import dataclass

from .geometry import LLAMA_3_1_8B, LLAMA_3_1_70B, ModelGeometry
from .migration import KvLayout


def tp_groups(gpus, tp: int) -> list[tuple[int, ...]]:
    gpus = list(gpus)
    return [tuple(gpus[i:i + tp]) for i in range(0, len(gpus), tp)]


def round_robin(groups, requests, total_heads: int) -> list[KvLayout]:
    per = [[] for _ in groups]
    for i, r in enumerate(requests):
        per[i % len(groups)].append(r)
    return [KvLayout(tuple(g), len(g), total_heads, tuple(p)) for g, p in zip(groups, per)]


@dataclass
class Workload:
    name: str
    model: ModelGeometry
    gpus: tuple[int, ...]
    old: list[KvLayout]
    new: list[KvLayout]
    old_weight_groups: list[tuple[int, ...]] | None  # None: KV only
    new_weight_groups: list[tuple[int, ...]] | None
    parked: tuple[int, ...] = ()  # GPUs left idle by the new config (weights untouched)
    # the reverse switch compacts weights to the old shards (frees the slices a
    # consolidation gathered), so every forward switch gathers them again
    trim_on_reverse: bool = False

    @property
    def requests(self):
        return [r for lay in self.old for r in lay.requests]

    def reversed(self) -> "Workload":
        return Workload(self.name + " (reverse)", self.model, self.gpus, self.new, self.old,
                        self.new_weight_groups, self.old_weight_groups, self.parked,
                        self.trim_on_reverse)


def transition(model, n_gpus, tp_old, tp_new, n_seqs, ctx, weights=True, name=None) -> Workload:
    gpus = tuple(range(n_gpus))
    reqs = [(i, ctx) for i in range(n_seqs)]
    og, ng = tp_groups(gpus, tp_old), tp_groups(gpus, tp_new)
    H = model.n_kv_heads
    return Workload(name or f"{model.name} TP{tp_old}->TP{tp_new} {n_seqs}x{ctx}", model, gpus,
                    round_robin(og, reqs, H), round_robin(ng, reqs, H),
                    og if weights else None, ng if weights else None)


def config(idx: int, **kw) -> Workload:
    """BASELINE.json configs[idx] (0-based)."""
    seqs, ctx = kw.get("seqs"), kw.get("ctx")
    if idx == 0:  # 8B TP1->TP2, 4 x 512, KV only
        seqs, ctx = seqs or 4, ctx or 512
        return transition(LLAMA_3_1_8B, 2, 1, 2, seqs, ctx, weights=False,
                          name=f"cfg1 Llama-3.1-8B TP1->TP2 {seqs}x{ctx} KV")
    if idx == 1:  # 8B TP2->TP4, 64 x 4k + weights
        seqs, ctx = seqs or 64, ctx or 4096
        w = kw.get("weights", True)
        return transition(LLAMA_3_1_8B, 4, 2, 4, seqs, ctx, weights=w,
                          name=f"cfg2 Llama-3.1-8B TP2->TP4 {seqs}x{ctx} KV" + ("+weights" if w else ""))
    if idx == 2:  # 8B TP8 -> TP1 on GPU0 (scale-in), 64 x 4k
        m = LLAMA_3_1_8B
        gpus = tuple(range(8))
        seqs, ctx = seqs or 64, ctx or 4096
        reqs = [(i, ctx) for i in range(seqs)]
        old = [KvLayout(gpus, 8, m.n_kv_heads, tuple(reqs))]
        new = [KvLayout((0,), 1, m.n_kv_heads, tuple(reqs))] + [
            KvLayout((g,), 1, m.n_kv_heads, ()) for g in gpus[1:]]
        w = kw.get("weights", True)
        return Workload(f"cfg3 Llama-3.1-8B TP8->TP1 consolidation {seqs}x{ctx}", m, gpus, old, new,
                        [gpus] if w else None, [(0,)] if w else None, parked=gpus[1:],
                        trim_on_reverse=True)
    if idx == 3:  # 70B TP4 <-> TP8, 8 x 32k
        seqs, ctx = seqs or 8, ctx or 32768
        return transition(LLAMA_3_1_70B, 8, 4, 8, seqs, ctx, weights=kw.get("weights", False),
                          name=f"cfg4 Llama-3.1-70B TP4->TP8 {seqs}x{ctx}")
    if idx == 4:  # the north star's headline: Llama-3.1-8B at 32k context, TP2 <-> TP4 + weights
        seqs, ctx = seqs or 8, ctx or 32768
        return transition(LLAMA_3_1_8B, 4, 2, 4, seqs, ctx, weights=kw.get("weights", True),
                          name=f"headline Llama-3.1-8B TP2->TP4 {seqs}x{ctx} KV+weights")
    raise ValueError(idx)
