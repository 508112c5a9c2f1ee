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
__device__ __forceinline__ int4 k3_page(const KvClusterParams& cl, const tpr_kv_geometry_t& geo,
                                        int src, int dst, int req, int h, int b, int ntok,
                                        int64_t alloc_pos, int64_t rel_pos, int& status_bits) {
  const int H = geo.total_heads, MB = geo.max_blocks;
  const bool in_range = h >= 0 && h < H && b >= 0 && b < MB && req >= 0 && req < geo.n_req_slots;
  const int64_t bt_idx = ((int64_t)req * H + h) * MB + b;
  // All loads first, then the stores: the three reads are independent (an
  // entry moves once per plan, and the released ring positions never overlap
  // the allocated ones), so they cost one memory latency instead of three.
  int32_t* bts = (src >= 0 && in_range) ? reinterpret_cast<int32_t*>(cl.block_table[src]) : nullptr;
  int32_t* btd = (dst >= 0 && in_range) ? reinterpret_cast<int32_t*>(cl.block_table[dst]) : nullptr;
  int32_t src_unit = bts ? __ldcg(bts + bt_idx) : -1;
  const int32_t popped =
      dst >= 0 ? __ldcg(reinterpret_cast<const int32_t*>(cl.free_ring[dst]) +
                        (cl.ring_head[dst] + alloc_pos) % cl.units[dst])
               : -1;
  const int32_t dst_prev = btd ? __ldcg(btd + bt_idx) : -1;
  int bits = in_range ? 0 : TPR_STATUS_OUT_OF_RANGE;
  if (src >= 0) {
    if (in_range && (src_unit < 0 || src_unit >= cl.units[src])) {
      bits |= TPR_STATUS_WRONG_SOURCE;
      src_unit = -1;
    }
    if (bts) bts[bt_idx] = -1;
    int32_t* ring_s = reinterpret_cast<int32_t*>(cl.free_ring[src]);
    ring_s[(cl.ring_tail[src] + rel_pos) % cl.units[src]] = src_unit;
  }
  int32_t dst_unit = -1;
  if (dst >= 0) {
    if (popped < 0 || popped >= cl.units[dst]) bits |= TPR_STATUS_RING_POISONED;
    else if (!in_range) {}  // leaked
    else if (dst_prev >= 0) bits |= TPR_STATUS_DST_OCCUPIED;  // a live entry stays; popped leaks
    else if (src >= 0 && src_unit < 0) {}  // nothing to place
    else {
      btd[bt_idx] = popped;
      dst_unit = popped;
    }
  }
  status_bits |= bits;
  const bool ok = dst_unit >= 0 && (src < 0 || src_unit >= 0);
  return make_int4(src_unit, dst_unit, (src & 0xffff) | ((dst & 0xffff) << 16),
                   ok || (dst < 0 && src_unit >= 0) ? ntok : 0);
}

}  // namespace tpr
