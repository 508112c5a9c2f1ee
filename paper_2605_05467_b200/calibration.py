"""Cost-model calibration for B200.

The reference prices a switch with ``switch_cost(WARM, plan, params)`` =
handshake + a two-buffer copy/send pipeline per source (migration.py:252-292),
with A100/H100-era constants (copy 900 GB/s, link 200 GB/s, 100 us per
transfer; migration.py:79-84). It also ignores ingress: the maximum is taken over
sources only (migration.py:275-281). On B200 this data path has no pack
stage: K1 writes pages straight into the destination pool. A switch is a fixed
cost plus bytes over the bottleneck bandwidth:

    t = fixed + max_g max(E_g, I_g) / link_bw     (GPUs on NVLink; ingress counted)
    t = fixed + B / hbm_moved_bw                  (one B200, logical GPUs: HBM bound)

``fit`` gets (fixed, bandwidth) from measured (bytes, ms) points by least
squares. ``B200CostModel.predict`` applies the formula.
``B200CostModel.cost_params`` gives reference ``CostModelParams`` that make the
unmodified ``switch_cost(WARM, ...)`` reproduce the calibrated latency. To do
that it sets an unbounded copy stage, one chunk, and the fixed cost as the
per-transfer overhead; the reference model stays source-only.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .migration import CostModelParams, MigrationPlan


def fit(bytes_moved, ms) -> tuple[float, float]:
    """Least-squares fixed cost (ms) and bandwidth (GB/s) for t = a + b * bytes."""
    x = np.asarray(bytes_moved, dtype=np.float64)
    y = np.asarray(ms, dtype=np.float64)
    A = np.stack([np.ones_like(x), x], axis=1)
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    gbs = 1.0 / (b * 1e6) if b > 0 else float("inf")  # ms per byte -> GB/s
    return float(max(a, 0.0)), float(gbs)


@dataclass(frozen=True)
class B200CostModel:
    fixed_ms: float
    hbm_moved_gbs: float      # logical mode: moved bytes per second (HBM r+w bound)
    link_gbs: float = 770.0   # measured peer copy per direction (B200_PROFILING.md)

    def predict(self, plan: MigrationPlan, mode: str = "logical") -> float:
        if mode == "logical":
            return self.fixed_ms + plan.total_bytes / (self.hbm_moved_gbs * 1e9) * 1e3
        if mode != "nvlink":
            raise ValueError(mode)
        arr = plan.as_array()
        if len(arr) == 0:
            return self.fixed_ms
        eg: dict[int, int] = {}
        ing: dict[int, int] = {}
        for s, d, _, _, _, b in arr.tolist():
            eg[s] = eg.get(s, 0) + b
            ing[d] = ing.get(d, 0) + b
        worst = max(max(eg.values()), max(ing.values()))
        return self.fixed_ms + worst / (self.link_gbs * 1e9) * 1e3

    def cost_params(self, mode: str = "logical") -> CostModelParams:
        bw = self.hbm_moved_gbs if mode == "logical" else self.link_gbs
        return CostModelParams(copy_bw_gbps=1e12, link_bw_gbps=bw,
                               per_transfer_overhead_us=max(self.fixed_ms, 1e-6) * 1e3,
                               chunk_bytes=1 << 50, handshake_ms=1e-9)


def from_sweep(rows, mode: str = "fixed4096") -> B200CostModel:
    """Calibrate from tools/sweep.py rows (profiles/r01_sweep.jsonl)."""
    pts = [(r["bytes"], r["device_ms"]) for r in rows if r["mode"] == mode and r["bytes"] > 0]
    a, gbs = fit([p[0] for p in pts], [p[1] for p in pts])
    return B200CostModel(fixed_ms=a, hbm_moved_gbs=gbs)
