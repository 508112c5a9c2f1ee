"""ORACLE -- test infrastructure only: GPU-vs-oracle comparison helpers.

Used by tests/ and __graft_entry__.smoke(). Takes host snapshots of a
PagedKvCluster before and after a device migration, replays the same records
with the C restatement (oracle/kvmove.c) on the "before" snapshot and compares
pools, block tables, free rings and ring counters byte for byte (or, for
full-size plans, block tables, free rings and ring counters only).
"""

from __future__ import annotations

import numpy as np

from . import kvmove


def geo_dict(cluster) -> dict:
    kv = cluster.kv
    return dict(layers=kv.layers, head_dim=kv.head_dim, dtype_bytes=kv.dtype_bytes,
                block_tokens=kv.block_tokens, total_heads=kv.total_heads,
                max_blocks=cluster.max_blocks, n_req_slots=cluster.max_requests,
                n_units=cluster.n_units)


def expected_after(cluster, before: dict, records: np.ndarray, impl: str = "c") -> dict:
    """The oracle's state after ``records``. A snapshot without "pools"
    (``tables_snapshot``) replays block tables, free rings and ring counters
    only: the full-size K3 parity check, page bytes being covered there by the
    placement-invariant pattern (``verify``)."""
    if "pools" not in before:
        tables = [t.copy().reshape(-1) for t in before["block_tables"]]
        rings = [r.copy() for r in before["rings"]]
        n, status, heads, tails = kvmove.kv_migrate(geo_dict(cluster), None, tables, rings,
                                                    before["ring_head"], before["ring_tail"],
                                                    records)
        return {"block_tables": tables, "rings": rings, "ring_head": heads, "ring_tail": tails,
                "status": status, "pages": n}
    pools = [p.copy() for p in before["pools"]]
    tables = [t.copy().reshape(-1) for t in before["block_tables"]]
    rings = [r.copy() for r in before["rings"]]
    fn = kvmove.kv_migrate if impl == "c" else kvmove.kv_migrate_py
    n, status, heads, tails = fn(geo_dict(cluster), pools, tables, rings, before["ring_head"],
                                 before["ring_tail"], records)
    return {"pools": pools, "block_tables": tables, "rings": rings, "ring_head": heads,
            "ring_tail": tails, "status": status, "pages": n}


def compare(got: dict, want: dict) -> dict:
    """Counts of differing bytes / entries per component (all zero = bit-exact)."""
    out = {"pool_bytes": 0, "table_entries": 0, "ring_entries": 0, "counters": 0}
    for g, w in zip(got.get("pools", ()), want.get("pools", ())):
        out["pool_bytes"] += int(np.count_nonzero(g != w))
    for g, w in zip(got["block_tables"], want["block_tables"]):
        out["table_entries"] += int(np.count_nonzero(g.reshape(-1) != w.reshape(-1)))
    for g, w, h0, t0 in zip(got["rings"], want["rings"], want["ring_head"], want["ring_tail"]):
        # only the live part of the ring (free units) is defined state
        cap = len(w)
        idx = np.arange(h0, t0) % cap
        out["ring_entries"] += int(np.count_nonzero(g[idx] != w[idx]))
    out["counters"] = int(got["ring_head"] != want["ring_head"]) + int(
        got["ring_tail"] != want["ring_tail"])
    return out
