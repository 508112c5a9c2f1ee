"""ORACLE -- test infrastructure only.

CPU restatements of the reference's TP-reconfiguration semantics used to check
the CUDA path: ``plan_oracle`` (planner + cost models, pinned to golden vectors
from the reference), ``kvmove`` (C restatement of plan execution on paged
pools) and ``weights`` (narrow/concatenate restatement of TP resharding).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package; the product never does.
"""
