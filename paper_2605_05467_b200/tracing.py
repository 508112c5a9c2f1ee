"""NVTX ranges around the phases of a TP switch (plan, K3+K1, K2, barrier).

Off by default (each range costs ~1 us of host time); enable with
``TPR_NVTX=1`` to see the phases in Nsight Systems / ncu's NVTX filter. The
reference has no tracer (only perf_counter around the planner).
"""

from __future__ import annotations

import contextlib
import os

ENABLED = os.environ.get("TPR_NVTX", "0") == "1"
_OFF = contextlib.nullcontext()  # reusable: nothing is allocated per range when off


def nvtx(name: str):
    if not ENABLED:
        return _OFF
    import torch

    return torch.cuda.nvtx.range(f"tpr:{name}")
