"""B200-native TP-reconfiguration data path (Nitsum, arXiv 2605.05467).

``paper_2605_05467_b200.migration`` is a drop-in for the reference's
``tpsim.migration`` API; ``kvcache``, ``weights`` and ``controller`` execute
plans on B200 through libtpr.so (include/tpr.h): K3 block-table remap, K1
paged-KV head-shard migration, K2 weight reshard.
"""

from .migration import (  # noqa: F401
    NAIVE_KERNEL_INIT,
    NAIVE_RELOAD,
    WARM,
    CostModelParams,
    KvLayout,
    MigrationError,
    MigrationPlan,
    Transfer,
    apply_plan,
    head_transfers,
    latency_aggregate,
    latency_per_page,
    latency_pipelined,
    layout_placement,
    plan_repartition,
    switch_cost,
    weight_memory,
)

__version__ = "0.1.0"
