// Page bookkeeping shared by K3 (tpr_kernels.cu) and the fused small-switch
// kernel K31 (tpr_bulk.cu).
#pragma once

#include <stdint.h>

#include "tpr.h"
#include "tpr_internal.h"

namespace tpr {

// ---------------------------------------------------------------------------
// Bookkeeping of one page (req, h, b) moving src -> dst (either may be -1):
// push the source unit at release position rel_pos of the source ring, pop the
// destination unit at allocation position alloc_pos of the destination ring,
// rewrite both block-table entries. Returns the work item
// {src_unit, dst_unit, src | dst << 16, ntok}; a page that must not be touched
// comes back with ntok = 0 (and status_bits says why). The ring positions
// the host counts are always written, so ring state stays defined after an
// error: a missing source is pushed as -1 (a poisoned slot that a later pop
// reports instead of using), a destination unit that cannot be placed leaks.
// oracle/kvmove.c restates exactly these rules.
// ---------------------------------------------------------------------------
// The decision half reads (source entry, popped ring slot, destination
// entry) and decides; the write half applies it. K3 runs both per page; K31
// lets every CTA that copies a piece of the page decide (same reads, same
// decision) and lets the last of them write (tpr_bulk.cu).
struct PageOp {
  int4 item;         // the K1 work item
  int bits;          // TPR_STATUS_* of this page
  int64_t bt_idx;    // block-table index, -1 when out of range
  int64_t ring_pos;  // source ring position of the push (src >= 0)
  int32_t src, dst;
  bool place;        // write the destination entry (item.y)
};

__device__ __forceinline__ PageOp k3_page_decide(const KvClusterParams& cl,
                                                 const tpr_kv_geometry_t& geo, int src, int dst,
                                                 int req, int h, int b, int ntok,
                                                 int64_t alloc_pos, int64_t rel_pos) {
  const int H = geo.total_heads, MB = geo.max_blocks;
  const bool in_range = h >= 0 && h < H && b >= 0 && b < MB && req >= 0 && req < geo.n_req_slots;
  PageOp op;
  op.bt_idx = in_range ? ((int64_t)req * H + h) * MB + b : -1;
  op.src = src;
  op.dst = dst;
  op.ring_pos = src >= 0 ? (cl.ring_tail[src] + rel_pos) % cl.units[src] : 0;
  // All loads first: the three reads are independent (an entry moves once per
  // plan, and the released ring positions never overlap the allocated ones),
  // so they cost one memory latency instead of three.
  const int32_t* bts = (src >= 0 && in_range) ? reinterpret_cast<const int32_t*>(cl.block_table[src]) : nullptr;
  const int32_t* btd = (dst >= 0 && in_range) ? reinterpret_cast<const int32_t*>(cl.block_table[dst]) : nullptr;
  int32_t src_unit = bts ? __ldcg(bts + op.bt_idx) : -1;
  const int32_t popped =
      dst >= 0 ? __ldcg(reinterpret_cast<const int32_t*>(cl.free_ring[dst]) +
                        (cl.ring_head[dst] + alloc_pos) % cl.units[dst])
               : -1;
  const int32_t dst_prev = btd ? __ldcg(btd + op.bt_idx) : -1;
  int bits = in_range ? 0 : TPR_STATUS_OUT_OF_RANGE;
  if (src >= 0 && in_range && (src_unit < 0 || src_unit >= cl.units[src])) {
    bits |= TPR_STATUS_WRONG_SOURCE;
    src_unit = -1;
  }
  int32_t dst_unit = -1;
  if (dst >= 0) {
    if (popped < 0 || popped >= cl.units[dst]) bits |= TPR_STATUS_RING_POISONED;
    else if (!in_range) {}  // leaked
    else if (dst_prev >= 0) bits |= TPR_STATUS_DST_OCCUPIED;  // a live entry stays; popped leaks
    else if (src >= 0 && src_unit < 0) {}  // nothing to place
    else dst_unit = popped;
  }
  op.bits = bits;
  op.place = dst_unit >= 0;
  const bool ok = dst_unit >= 0 && (src < 0 || src_unit >= 0);
  op.item = make_int4(src_unit, dst_unit, (src & 0xffff) | ((dst & 0xffff) << 16),
                      ok || (dst < 0 && src_unit >= 0) ? ntok : 0);
  return op;
}

__device__ __forceinline__ void k3_page_write(const KvClusterParams& cl, const PageOp& op) {
  if (op.src >= 0) {
    if (op.bt_idx >= 0) reinterpret_cast<int32_t*>(cl.block_table[op.src])[op.bt_idx] = -1;
    reinterpret_cast<int32_t*>(cl.free_ring[op.src])[op.ring_pos] = op.item.x;  // -1: poisoned
  }
  if (op.place) reinterpret_cast<int32_t*>(cl.block_table[op.dst])[op.bt_idx] = op.item.y;
}

__device__ __forceinline__ int4 k3_page(const KvClusterParams& cl, const tpr_kv_geometry_t& geo,
                                        int src, int dst, int req, int h, int b, int ntok,
                                        int64_t alloc_pos, int64_t rel_pos, int& status_bits) {
  const PageOp op = k3_page_decide(cl, geo, src, dst, req, h, b, ntok, alloc_pos, rel_pos);
  k3_page_write(cl, op);
  status_bits |= op.bits;
  return op.item;
}

}  // namespace tpr
