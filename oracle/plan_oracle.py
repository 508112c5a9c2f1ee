"""ORACLE -- test infrastructure only; never imported by the product path.

Pure-Python restatement of the reference planner and cost models
(pkg/src/tpsim/migration.py). Pinned against golden vectors produced by the
reference itself (tests/golden/gen_golden.py, run in the build container where
/root/reference exists); see tests/test_oracle.py.

Plain tuples, no classes: a layout is (group tuple, total_heads, requests).
"""

from __future__ import annotations

import math


def owner_of(group, total_heads, head):
    """migration.py:42-47 -- rank r owns heads [r*H/N, (r+1)*H/N)."""
    per = total_heads // len(group)
    return group[head // per]


def request_moves(old_group, new_group, total_heads, rid, ctx, kvb):
    """migration.py:101-134 for one request: maximal runs of heads sharing a
    (src, dst) pair with src != dst, in ascending head order."""
    moves = []
    cur = None  # [src, dst, lo]
    for h in range(total_heads):
        s = owner_of(old_group, total_heads, h)
        d = owner_of(new_group, total_heads, h)
        key = (s, d) if s != d else None
        if cur is not None and (key is None or key != (cur[0], cur[1])):
            moves.append((cur[0], cur[1], rid, cur[2], h, (h - cur[2]) * ctx * kvb))
            cur = None
        if key is not None and cur is None:
            cur = [s, d, h]
    if cur is not None:
        moves.append((cur[0], cur[1], rid, cur[2], total_heads,
                       (total_heads - cur[2]) * ctx * kvb))
    return moves


def plan(old_layouts, new_layouts, kvb):
    """migration.py:137-189 ordering: new layouts in order, their requests in
    order. Layouts are (group, total_heads, requests). Validation omitted."""
    src_of = {}
    for group, H, reqs in old_layouts:
        for rid, ctx in reqs:
            src_of[rid] = (group, ctx)
    out = []
    for group, H, reqs in new_layouts:
        for rid, ctx in reqs:
            og, _ = src_of[rid]
            out.extend(request_moves(og, group, H, rid, ctx, kvb))
    return out


def placement(layouts):
    """migration.py:210-218."""
    out = {}
    for group, H, reqs in layouts:
        for rid, _ in reqs:
            for h in range(H):
                out[(rid, h)] = owner_of(group, H, h)
    return out


def replay(old_layouts, moves):
    """migration.py:192-207; returns placement or raises ValueError."""
    where = placement(old_layouts)
    for s, d, rid, lo, hi, _ in moves:
        for h in range(lo, hi):
            if where.get((rid, h)) != s:
                raise ValueError(f"request {rid} head {h} not on {s}")
            where[(rid, h)] = d
    return where


# -- cost models (migration.py:221-292) --------------------------------------

def send_ms(nbytes, p):
    return p["per_transfer_overhead_us"] / 1000.0 + nbytes / (p["link_bw_gbps"] * 1e9) * 1000.0


def copy_ms(nbytes, p):
    return nbytes / (p["copy_bw_gbps"] * 1e9) * 1000.0


def by_source(moves):
    acc = {}
    for m in moves:
        acc[m[0]] = acc.get(m[0], 0) + m[5]
    return acc


def per_page_ms(moves, p):
    page = send_ms(p["page_bytes"], p)
    acc = {}
    for m in moves:
        acc[m[0]] = acc.get(m[0], 0.0) + math.ceil(m[5] / p["page_bytes"]) * page
    return max(acc.values(), default=0.0)


def aggregate_ms(moves, p):
    best = 0.0
    for b in by_source(moves).values():
        best = max(best, copy_ms(b, p) + send_ms(b, p))
    return best


def two_buffer_ms(total, p):
    """Explicit two-buffer schedule: buffer i%2 is reused by chunk i only
    after chunk i-2's send finished."""
    chunk = p["chunk_bytes"]
    n = math.ceil(total / chunk)
    copy_end, send_end = [], []
    for i in range(n):
        size = min(chunk, total - i * chunk)
        start = copy_end[-1] if copy_end else 0.0
        if i >= 2:
            start = max(start, send_end[i - 2])
        copy_end.append(start + copy_ms(size, p))
        go = copy_end[-1]
        if send_end:
            go = max(go, send_end[-1])
        send_end.append(go + send_ms(size, p))
    return send_end[-1] if n else 0.0


def pipelined_ms(moves, p):
    return max((two_buffer_ms(b, p) for b in by_source(moves).values()), default=0.0)


DEFAULT_PARAMS = dict(copy_bw_gbps=900.0, link_bw_gbps=200.0, per_transfer_overhead_us=100.0,
                      page_bytes=65536, chunk_bytes=128 * 1024 * 1024, handshake_ms=0.5,
                      reload_ms=30000.0, kernel_init_ms=10000.0)


def weight_gb(mode, full_gb, tp_levels, tp=None):
    """migration.py:295-306."""
    if mode == "full_copy_per_gpu":
        return full_gb
    if mode == "per_tp_copies":
        return sum(full_gb / t for t in tp_levels)
    if mode == "sharded":
        return full_gb / tp
    raise ValueError(mode)
