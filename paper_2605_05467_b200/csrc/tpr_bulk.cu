// TMA bulk-copy engine for K1 / K2 (sm_100a): global -> shared -> global with
// cp.async.bulk, an mbarrier per shared-memory stage and bulk-group
// completion tracking. One elected thread per CTA issues every copy, so the
// SMs spend almost no instructions on data movement; the copy engine moves the
// bytes. Pieces are <= `piece` bytes, 16-B aligned, multiples of 16 B.
//
// Pipeline per CTA (S stages, lookahead L = S - 2 loads in flight):
//   load piece j+L into stage (j+L)%S once the store that last read that
//   stage (piece j-2) has finished reading shared memory
//   (cp.async.bulk.wait_group.read 1); wait for piece j's load (mbarrier
//   parity); store piece j; commit its bulk group.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "tpr.h"
#include "tpr_common.cuh"
#include "tpr_internal.h"
#include "tpr_k3page.cuh"

namespace tpr {

constexpr int kMaxStages = 8;  // shared-memory ring: stages x piece bytes (runtime)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_smem),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void bulk_store(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(src_smem), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA tensor copies (3-D, no swizzle) through a CUtensorMap kernel parameter.
__device__ __forceinline__ void tensor_load(uint32_t dst_smem, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(dst_smem),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tensor_store(const CUtensorMap* map, int32_t c0, int32_t c1,
                                             int32_t c2, uint32_t src_smem) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(src_smem)
      : "memory");
}

// One copy the pipeline moves through a stage: a linear byte range (map < 0)
// or a TMA tensor box of the source / destination pool maps.
struct Copy {
  const char* src;
  char* dst;
  uint32_t nb;
  int32_t smap, dmap;  // tensor map index (GPU slot) or -1 for a linear copy
  int32_t c1, sc2, dc2;  // tensor coordinates: token, first plane (src / dst)
};

// ---- piece sources ---------------------------------------------------------

// K1: the CTA's work items (grid-stride) -> copies. A full page item is one
// contiguous span cut into `piece`-byte copies. A partial page item is either
// one copy per plane row (ntok valid tokens each) or, with the pools' tensor
// maps, one TMA box per (token, r_box planes): item g of the unit takes tokens
// g, g + items_per_unit, ... (no strided short copies at all).
// K1 items are handed out statically (grid-stride) or, with a claim counter,
// dynamically in batches of `batch` consecutive items (4 by
// default) claimed one batch ahead: CTAs then stay on neighbouring items (a
// small, shared working set of pages) and none drains late. One kernel serves
// every plan: with tm->enabled = 0 (a plan of full pages, or tensor boxes
// switched off) partial pages fall back to row copies.

struct KvPieces {
  const int4* work;
  int64_t n_items;
  KvCopyParams p;
  const KvClusterParams* cl;    // the kernel's __grid_constant__ parameter
  const KvTensorMaps* tm;       // likewise (tm->enabled = 0: row copies)
  uint32_t piece;
  int64_t item;
  unsigned long long* claim = nullptr;  // dynamic schedule (0 at kernel start)
  int64_t batch = 4, item_end = 0, next_batch = 0;
  bool work_l2 = false;  // work items written by this launch: read them from L2
  int64_t stride = -1;  // static schedule step (-1: gridDim.x, grid-stride shares)
  // current item: linear rows ...
  const char* s;
  char* d;
  int64_t rows_left, row_bytes, pitch, off;
  // ... or tensor boxes
  int32_t t_src, t_dst, t_tok, t_ntok, t_step, t_pb, t_sc2, t_dc2;
  bool tensor;
  bool boxes;  // partial pages as tensor boxes (the pools' maps are enabled)

  __device__ void start(int64_t first) {
    rows_left = 0;
    tensor = false;
    boxes = tm != nullptr && tm->enabled;
    if (claim) {
      item = first * batch;
      item_end = min(item + batch, n_items);
      next_batch = (int64_t)gridDim.x + (int64_t)atomicAdd(claim, 1ull);
    } else {
      item = first;
      if (stride < 0) stride = gridDim.x;
    }
  }
  __device__ bool take(int64_t& k) {
    if (!claim) {
      if (item >= n_items) return false;
      k = item;
      item += stride;
      return true;
    }
    if (item >= item_end) {
      item = next_batch * batch;
      if (item >= n_items) return false;
      item_end = min(item + batch, n_items);
      next_batch = (int64_t)gridDim.x + (int64_t)atomicAdd(claim, 1ull);
    }
    k = item++;
    return true;
  }
  __device__ bool load_item() {
    int64_t it;
    while (take(it)) {
      const int64_t u = it / p.items_per_unit;
      const int g = (int)(it - u * p.items_per_unit);
      const int4 w = work_l2 ? __ldcg(work + u) : work[u];
      const int src_slot = w.z & 0xffff, dst_slot = (w.z >> 16) & 0xffff, ntok = w.w;
      if (w.x < 0 || w.y < 0 || ntok <= 0) continue;  // a page K3 refused (status word)
      const int64_t nb = (int64_t)ntok * p.tok_bytes;
      if (boxes && nb != p.pitch) {  // partial page: tensor boxes
        if (g >= ntok) continue;            // no token for this item slot
        tensor = true;
        t_src = src_slot;
        t_dst = dst_slot;
        t_tok = g;
        t_ntok = ntok;
        t_step = p.items_per_unit;
        t_pb = 0;
        t_sc2 = w.x * p.rows;
        t_dc2 = w.y * p.rows;
        return true;
      }
      const int row0 = g * p.rows_per_item;
      const int nr = min(p.rows_per_item, p.rows - row0);
      s = reinterpret_cast<const char*>(cl->pool[src_slot]) + (int64_t)w.x * p.unit_bytes +
          (int64_t)row0 * p.pitch;
      d = reinterpret_cast<char*>(cl->pool[dst_slot]) + (int64_t)w.y * p.unit_bytes +
          (int64_t)row0 * p.pitch;
      if (nb == p.pitch) {  // contiguous planes
        rows_left = 1;
        row_bytes = nb * nr;
      } else {
        rows_left = nr;
        row_bytes = nb;
      }
      pitch = p.pitch;
      off = 0;
      if (row_bytes > 0) return true;
    }
    return false;
  }
  // The next copy: 1 = produced (a linear copy of at most avail_linear bytes,
  // or one tensor box when it fits avail_box), 2 = the next copy is a box
  // that does not fit this stage (nothing consumed), 0 = no work left.
  __device__ int next(Copy& c, uint32_t avail_linear, uint32_t avail_box) {
    if (!tensor && rows_left == 0 && !load_item()) return 0;
    if (tensor) {
      const uint32_t bb = (uint32_t)(tm->r_box * p.tok_bytes);
      if (bb > avail_box) return 2;
      c.smap = t_src;
      c.dmap = t_dst;
      c.c1 = t_tok;
      c.sc2 = t_sc2 + t_pb * tm->r_box;
      c.dc2 = t_dc2 + t_pb * tm->r_box;
      c.nb = bb;
      if (++t_pb == tm->n_pb) {
        t_pb = 0;
        t_tok += t_step;
        if (t_tok >= t_ntok) tensor = false;
      }
      return 1;
    }
    const uint32_t max_bytes = avail_linear;
    const int64_t take = min((int64_t)max_bytes, row_bytes - off);
    c.src = s + off;
    c.dst = d + off;
    c.nb = (uint32_t)take;
    c.smap = c.dmap = -1;
    off += take;
    if (off == row_bytes) {
      off = 0;
      s += pitch;
      d += pitch;
      --rows_left;
    }
    return 1;
  }
};

// K2: the CTA's segment items -> pieces. Items are scheduled either
// statically (grid-stride, claim == nullptr) or dynamically: the CTA owns a
// batch of kClaimBatch consecutive items and claims its next batch from
// *claim (a per-launch counter, 0 at kernel start) one batch ahead, so the
// atomic's latency hides behind the current batch's copies. Dynamic claims
// remove the tail left when CTAs drain at different speeds (ncu: SM-active
// 86-89% of elapsed with the static schedule). Consecutive items mostly hit
// the cached segment, so the prefix binary search runs once per segment.
constexpr int64_t kClaimBatch = 4;

struct SegPieces {
  const tpr_copy_seg_t* segs;
  const int64_t* prefix;
  int64_t* claim;
  uint32_t piece;
  int32_t n_segs;
  int64_t n_items, chunk, item, item_end, next_batch;
  // cached segment
  int32_t cur;
  int64_t cur_lo, cur_hi;
  tpr_copy_seg_t sg;
  const char* s;
  char* d;
  int64_t rows_left, row_bytes, sp, dp, off;
  bool aligned;

  __device__ void start(int64_t first) {
    rows_left = 0;
    cur = -1;
    cur_lo = cur_hi = 0;
    if (claim) {
      item = first * kClaimBatch;
      item_end = min(item + kClaimBatch, n_items);
      next_batch = (int64_t)gridDim.x + (int64_t)atomicAdd((unsigned long long*)claim, 1ull);
    } else {
      item = first;
    }
  }
  // the item to load next (and advance the schedule); false when exhausted
  __device__ bool take(int64_t& k) {
    if (!claim) {
      if (item >= n_items) return false;
      k = item;
      item += gridDim.x;
      return true;
    }
    if (item >= item_end) {
      item = next_batch * kClaimBatch;
      if (item >= n_items) return false;
      item_end = min(item + kClaimBatch, n_items);
      next_batch = (int64_t)gridDim.x + (int64_t)atomicAdd((unsigned long long*)claim, 1ull);
    }
    k = item++;
    return true;
  }
  __device__ void find_segment(int64_t k) {
    if (k >= cur_lo && k < cur_hi) return;
    int lo;
    if (cur >= 0 && k >= cur_hi && cur + 2 <= n_segs && k < prefix[cur + 2]) {
      lo = cur + 1;  // the next segment (a batch crossing a boundary)
    } else {
      lo = 0;
      int hi = n_segs;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (prefix[mid] <= k) lo = mid; else hi = mid;
      }
    }
    cur = lo;
    cur_lo = prefix[lo];
    cur_hi = prefix[lo + 1];
    sg = segs[lo];
  }
  __device__ bool load_item() {
    int64_t k;
    while (take(k)) {
      if (!load_one(k)) continue;
      if (aligned) return true;
      // unaligned segment (never for the Llama geometries): plain byte copy by
      // the issuing thread, then move on
      for (int64_t r = 0; r < rows_left; ++r)
        for (int64_t b = 0; b < row_bytes; ++b) d[r * dp + b] = s[r * sp + b];
      rows_left = 0;
    }
    return false;
  }
  __device__ bool load_one(int64_t item_id) {
    {
      find_segment(item_id);
      const int64_t k = item_id - cur_lo;
      int64_t r0, nr, b0, nb;
      if (sg.row_bytes <= chunk) {
        const int64_t rpi = chunk / sg.row_bytes;
        r0 = k * rpi;
        nr = min(rpi, sg.rows - r0);
        b0 = 0;
        nb = sg.row_bytes;
      } else {
        const int64_t ipr = (sg.row_bytes + chunk - 1) / chunk;
        r0 = k / ipr;
        nr = 1;
        b0 = (k - r0 * ipr) * chunk;
        nb = min(chunk, sg.row_bytes - b0);
      }
      s = reinterpret_cast<const char*>(sg.src) + r0 * sg.src_pitch + b0;
      d = reinterpret_cast<char*>(sg.dst) + r0 * sg.dst_pitch + b0;
      rows_left = nr;
      row_bytes = nb;
      sp = sg.src_pitch;
      dp = sg.dst_pitch;
      off = 0;
      aligned = (sg.flags & TPR_SEG_ALIGNED16) != 0;
      if (nr > 0 && nb > 0) return true;
      rows_left = 0;
    }
    return false;
  }
  __device__ int next(Copy& c, uint32_t max_bytes, uint32_t /*avail_box*/) {
    if (rows_left == 0 && !load_item()) return 0;
    const int64_t take = min((int64_t)max_bytes, row_bytes - off);
    c.src = s + off;
    c.dst = d + off;
    c.nb = (uint32_t)take;
    c.smap = c.dmap = -1;
    off += take;
    if (off == row_bytes) {
      off = 0;
      s += sp;
      d += dp;
      --rows_left;
    }
    return 1;
  }
};

constexpr int kMaxSub = 16;  // copies packed into one shared-memory stage

// The shared-memory ring's per-stage copy descriptors, and the two halves of
// moving one stage: fill() packs copies into stage t and issues their loads,
// store() issues the stage's stores. A stage is `piece` bytes of shared
// memory filled with up to kMaxSub consecutive copies (one 32 KiB page chunk,
// many short rows of row-parallel weight slices, or -- K1, kTensor -- TMA
// tensor boxes of partial pages, 128-byte aligned). The stage's loads all
// complete on one mbarrier; its stores form one bulk group, so small copies
// still keep a full stage of bytes in flight.
//
// The issuing thread is the throughput limit for short copies, so the per-copy
// path stays in registers and each load is issued as soon as its copy is
// produced; the stage's single arrive.expect_tx follows (the tx-count may go
// transiently negative; the phase cannot complete before the arrival). Only
// K2's pipeline (linear copies only, kTensor = false) takes the fast path for
// a full linear stage, expect_tx before the load: that order costs 4-20% when
// tensor-box stages use it or mix with it; with dynamic claims
// K1 runs full pages as fast without it (7.649 vs 7.657 ms on cfg2).
template <bool kTensor>
struct StageRing {
  char* dst[kMaxStages][kMaxSub];
  uint32_t nb[kMaxStages][kMaxSub];
  uint32_t off[kMaxStages][kMaxSub];
  int32_t dmap[kTensor ? kMaxStages : 1][kMaxSub];  // -1: linear store
  int32_t c1[kTensor ? kMaxStages : 1][kMaxSub];
  int32_t dc2[kTensor ? kMaxStages : 1][kMaxSub];
  int cnt[kMaxStages];

  // Stage t from its first copy `c` on; false when the source ran dry.
  template <class Source>
  __device__ __forceinline__ bool fill(Source& src_it, Copy& c, int t, uint32_t sbase,
                                       uint32_t piece, uint64_t* bar, const KvTensorMaps* tm) {
    if (!kTensor && c.nb == piece) {  // fast path: one linear copy fills the stage
      cnt[t] = 1;
      dst[t][0] = c.dst;
      nb[t][0] = piece;
      off[t][0] = 0;
      bulk_load(sbase, c.src, piece, bar);
      return true;
    }
    bool more = true;
    uint32_t used = 0, tx = 0;
    int n = 0;
    while (true) {
      uint32_t o = used;
      if (kTensor && c.smap >= 0) {
        o = (used + 127u) & ~127u;
        tensor_load(sbase + o, &tm->map[c.smap], 0, c.c1, c.sc2, bar);
        dmap[t][n] = c.dmap;
        c1[t][n] = c.c1;
        dc2[t][n] = c.dc2;
      } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sbase + o),
            "l"(c.src), "r"(c.nb), "r"(smem_u32(bar))
            : "memory");
        if (kTensor) dmap[t][n] = -1;
      }
      dst[t][n] = c.dst;
      nb[t][n] = c.nb;
      off[t][n] = o;
      used = o + c.nb;
      tx += c.nb;
      ++n;
      // pack a further copy: a linear one needs >= 1 KiB left, a box its size
      if (n == kMaxSub) break;
      const uint32_t aligned = (used + 127u) & ~127u;
      const uint32_t avail_box = (kTensor && aligned <= piece) ? piece - aligned : 0;
      const uint32_t avail_lin = piece - used >= 1024 ? piece - used : 0;
      if (avail_lin == 0 && avail_box == 0) break;
      const int r = src_it.next(c, avail_lin, avail_box);
      if (r == 0) {
        more = false;
        break;
      }
      if (r == 2 || c.nb == 0) break;  // the next copy needs a fresh stage
    }
    cnt[t] = n;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(tx)
                 : "memory");
    return more;
  }

  __device__ __forceinline__ void store(int t, uint32_t sbase, const KvTensorMaps* tm) {
    for (int i = 0; i < cnt[t]; ++i) {
      if (kTensor && dmap[t][i] >= 0)
        tensor_store(&tm->map[dmap[t][i]], 0, c1[t][i], dc2[t][i], sbase + off[t][i]);
      else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[t][i]),
                     "r"(sbase + off[t][i]), "r"(nb[t][i])
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
};

// One elected thread issues every load and store (lookahead L = S - 2 stages:
// the refilled stage's last store may still be reading shared memory).
template <bool kTensor, class Source>
__device__ __forceinline__ void bulk_pipeline(Source& src_it, int stages,
                                              const KvTensorMaps* tm) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[kMaxStages];
  __shared__ StageRing<kTensor> ring;
  if (threadIdx.x != 0) return;
  const uint32_t piece = src_it.piece;
  const int lookahead = stages - 2;
  for (int s = 0; s < stages; ++s) bar_init(&bar[s]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t base = smem_u32(smem);
  int64_t issued = 0, stored = 0;
  bool more = true;
  auto issue = [&]() {
    const int t = (int)(issued % stages);
    Copy c;
    if (src_it.next(c, piece, piece) != 1) {
      more = false;
      return;
    }
    if (issued >= stages) bulk_wait_read_1();  // stores of stage issued-S done reading
    more = ring.fill(src_it, c, t, base + (uint32_t)t * piece, piece, &bar[t], tm);
    ++issued;
  };
  while (more && issued < lookahead) issue();
  while (stored < issued) {
    if (more) issue();
    const int t = (int)(stored % stages);
    bar_wait(&bar[t], (uint32_t)((stored / stages) & 1));
    ring.store(t, base + (uint32_t)t * piece, tm);
    ++stored;
  }
  bulk_wait_all();
}

// K1: the work list K3 wrote -> page copies (partial pages as TMA tensor
// boxes of the pools' maps when tm.enabled, else as row copies)
__global__ void __launch_bounds__(32)
    tpr_k1_kv_migrate_bulk(const int4* __restrict__ work, int64_t n_units, KvCopyParams p,
                           const __grid_constant__ KvClusterParams cl,
                           const __grid_constant__ KvTensorMaps tm, int32_t stages,
                           uint32_t piece, int32_t dynamic) {
  KvPieces it;
  // the claim counter is the int4 slot after the work list (zeroed by K3);
  // `dynamic` = items per claim, 0 = static grid-stride shares
  if (dynamic > 0) {
    it.claim = reinterpret_cast<unsigned long long*>(const_cast<int4*>(work + n_units));
    it.batch = dynamic;
  }
  it.work = work;
  it.n_items = n_units * p.items_per_unit;
  it.p = p;
  it.cl = &cl;
  it.tm = &tm;
  it.piece = piece;
  if (threadIdx.x != 0) return;  // one issuing thread per CTA
  pdl_wait();  // K3's work list (launched with programmatic serialization)
  it.start(blockIdx.x);
  bulk_pipeline<true>(it, stages, &tm);
}

__global__ void __launch_bounds__(32)
    tpr_k2_copy_segments_bulk(const tpr_copy_seg_t* __restrict__ segs,
                              const int64_t* __restrict__ prefix, int32_t n_segs, int64_t n_items,
                              int64_t chunk, int64_t* claim, int32_t stages, uint32_t piece) {
  SegPieces it;
  it.segs = segs;
  it.prefix = prefix;
  it.claim = claim;
  it.n_segs = n_segs;
  it.n_items = n_items;
  it.chunk = chunk;
  it.piece = piece;
  if (threadIdx.x != 0) return;  // one issuing thread: start() claims its first batch
  it.start(blockIdx.x);
  bulk_pipeline<false>(it, stages, nullptr);
}

// ---------------------------------------------------------------------------
// K31: the whole switch of a small plan in ONE launch (K3 bookkeeping + K1
// copy). The records and their three keyed exclusive scans (units before
// each record that this rank moves / its destination ring hands out / its
// source ring takes back) ride in the kernel parameters: the host builds the
// records, so it does K3's scan in passing, and every CTA starts deciding at
// entry. CTA c copies an equal contiguous share of the ITEMS (32 KiB pieces
// of pages), items [c*N/G, (c+1)*N/G). For each page its items touch, the
// CTA makes the page's bookkeeping decision itself (k3_page_decide: the same
// three reads and the same result in every CTA that shares the page, since
// nothing is written before all of them have read) and counts itself in the
// page's reader counter; the LAST reader applies the writes (source entry
// cleared, source unit pushed, destination entry set). No CTA ever waits for
// another, and the work is balanced to one item.
//
// Two warps per CTA. The copies need only the decisions (unit ids), not the
// bookkeeping writes, and the writes touch tables and rings, never page
// bytes. So once the 64 threads have decided the CTA's pages (one read round
// trip, one thread per page), warp 0's elected thread streams the copies
// while warp 1 does the reader counting, the writes, the status bits and the
// completion counter off the copy's critical path.
//
// Reader counters live in the caller's work-list scratch (d_work, 8 bytes per
// page), tagged with the launch epoch (totals[TPR_TOTALS_K31_EPOCH], advanced
// by the last CTA), so they never need clearing (a freshly allocated d_work
// must be zeroed once). The status word reports this
// call only: CTAs OR their bits into totals[TPR_TOTALS_K31_STATUS]; the last
// count of the completion counter totals[TPR_TOTALS_K31_DONE]
// (k31_item_share_done) publishes them to *status (+ the pinned mirror and
// the caller's ticket) and resets both scratch words. A device-barrier
// timeout already in *status aborts the call (no copy, no write; the bit
// stays).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t k31_cta_of(int64_t item, int64_t n_items, int64_t grid) {
  return ((item + 1) * grid - 1) / n_items;  // the CTA whose share holds `item`
}

// The item-share kernel's completion: each CTA counts itself after its
// bookkeeping and status bits (warp 1) and, when the caller asked for a
// ticket, after its copies too (warp 0); the last count publishes the status
// word (device + pinned mirror), then the ticket into mirror[1] -- a host
// that spins on the ticket knows every copy and every table write of the call
// is done -- and resets the scratch words and advances the epoch (every CTA
// read it at entry).
__device__ __forceinline__ void k31_item_share_done(int64_t* totals, int32_t* status,
                                                    int32_t* status_mirror, int32_t st0,
                                                    uint64_t epoch, bool abort, int64_t n_mine,
                                                    int32_t ticket) {
  __threadfence();
  unsigned long long* done = reinterpret_cast<unsigned long long*>(totals + TPR_TOTALS_K31_DONE);
  const unsigned long long counts = (ticket ? 2ull : 1ull) * gridDim.x;
  if (atomicAdd(done, 1ull) != counts - 1) return;
  __threadfence();
  const int32_t acc = (int32_t)atomicExch(
      reinterpret_cast<unsigned long long*>(totals + TPR_TOTALS_K31_STATUS), 0ull);
  const int32_t out = acc | (st0 & TPR_STATUS_BARRIER_TIMEOUT);
  *status = out;
  if (status_mirror) {
    *reinterpret_cast<volatile int32_t*>(status_mirror) = out;
    if (ticket) {
      __threadfence_system();  // the status word lands first
      *reinterpret_cast<volatile int32_t*>(status_mirror + 1) = ticket;
    }
  }
  totals[TPR_TOTALS_K31_EPOCH] = (int64_t)(epoch + 1);
  *done = 0ull;
  if (!abort) totals[0] = n_mine;
}

constexpr int kK31Threads = 64;
constexpr int64_t kK31DynamicUnits = 512;  // auto schedule: dynamic from here up
static_assert(kK31MaxPages <= kK31Threads, "one deciding thread per page");

// Partial pages move as TMA tensor boxes of the pools' maps when tm.enabled
// (the maps ride in the parameters too: > 4 KiB of parameters, CUDA >= 12.1).
__global__ void __launch_bounds__(kK31Threads)
    tpr_k31_switch(const __grid_constant__ K31Params rp, tpr_kv_geometry_t geo, KvCopyParams p,
                   const __grid_constant__ KvClusterParams cl,
                   const __grid_constant__ KvTensorMaps tm, int64_t* __restrict__ totals,
                   unsigned long long* __restrict__ readers, int32_t* __restrict__ status,
                   int32_t* status_mirror, int32_t stages, uint32_t piece) {
  __shared__ __align__(16) int4 s_work[kK31MaxPages];
  __shared__ PageOp s_op[kK31MaxPages];
  __shared__ int s_bits[2];
  __shared__ int32_t s_st0;
  __shared__ uint64_t s_epoch;
  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  // phase stamps for tools/k31_trace.py: entry, decisions, copies, bookkeeping
  auto stamp = [&](int k) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    rp.trace[blockIdx.x * 8 + k] = t;
  };
  const bool tracing = rp.trace != nullptr;
  if (tracing && tid == 0) stamp(0);
  const int n = rp.n, B = geo.block_tokens;
  if (warp == 1) {  // the call's status and epoch words, tensor maps warmed
    if (lane == 0) {
      s_st0 = __ldcg(status);
      s_epoch = (uint64_t)__ldcg(totals + TPR_TOTALS_K31_EPOCH);
    }
    if (tm.enabled && lane < TPR_MAX_GPUS && cl.pool[lane] != 0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.map[lane]))
                   : "memory");
  }
  const int64_t n_mine = rp.n_mine;
  const int64_t ipu = p.items_per_unit, n_items = n_mine * ipu, grid = gridDim.x;
  // this CTA's share of the items and the pages they belong to
  const int64_t i0 = (int64_t)blockIdx.x * n_items / grid;
  const int64_t i1 = ((int64_t)blockIdx.x + 1) * n_items / grid;
  const int64_t p0 = i0 / ipu;
  const int n_pages = i1 <= i0 ? 0 : (int)((i1 - 1) / ipu - p0 + 1);
  // decisions: one thread per page (reads only)
  int bits = 0;
  if ((int)tid < n_pages) {
    const int64_t pg = p0 + tid;
    int lo = 0, hi = n;  // upper_bound(mine offsets, pg) - 1
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rp.off[0][mid] <= pg) lo = mid; else hi = mid;
    }
    const int32_t* r = rp.rec[lo];
    const int64_t local = pg - rp.off[0][lo];
    const int ctx = r[5], nblk = (ctx + B - 1) / B;
    const int h = r[3] + (int)(local / nblk);
    const int b = (int)(local - (int64_t)(h - r[3]) * nblk);
    const int ntok = (b == nblk - 1) ? ctx - b * B : B;
    const PageOp op = k3_page_decide(cl, geo, r[0], r[1], r[2], h, b, ntok, rp.off[1][lo] + local,
                                     rp.off[2][lo] + local);
    s_work[tid] = op.item;
    s_op[tid] = op;
    bits = op.bits;
  }
  bits = (int)__reduce_or_sync(0xffffffffu, (unsigned)bits);
  if (lane == 0) s_bits[warp] = bits;
  __syncthreads();  // s_work complete: the copies can start
  if (tracing && tid == 0) stamp(1);
  const int32_t st0 = s_st0;
  const bool abort = (st0 & TPR_STATUS_BARRIER_TIMEOUT) != 0;
  if (warp == 0) {
    if (tid == 0 && n_pages > 0 && !abort) {
      KvPieces it;
      it.work = s_work - p0;  // work[u] for the pages p0 .. p0 + n_pages - 1
      it.n_items = i1;
      it.p = p;
      it.cl = &cl;
      it.tm = &tm;
      it.piece = piece;
      it.stride = 1;
      it.start(i0);
      bulk_pipeline<true>(it, stages, &tm);  // waits for its last store
    }
    if (tid == 0) {
      if (tracing) {
        stamp(2);
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        rp.trace[blockIdx.x * 8 + 5] = smid;
        rp.trace[blockIdx.x * 8 + 6] = (uint64_t)(i1 - i0);
        rp.trace[blockIdx.x * 8 + 7] = (uint64_t)gridDim.x;
      }
      if (rp.ticket)  // with a ticket, the copies count too: it is published after them
        k31_item_share_done(totals, status, status_mirror, st0, s_epoch, abort, n_mine, rp.ticket);
    }
    return;
  }
  // warp 1: bookkeeping of the pages this CTA decided (the deciding threads'
  // ops are in shared memory), then the completion counter
  const uint64_t epoch = s_epoch;
  // tags have the high bit set and are never 0xffffffff, so neither a work
  // item K3 left in d_work ({unit >= 0 or -1, ...}) nor zeroed memory reads as
  // a counter of this launch
  const uint32_t tag = 0x80000000u | (uint32_t)((epoch + 1) % 0x7fffffffull);
  __threadfence();  // this CTA's reads of the pages' entries come first
  for (int j = (int)lane; j < (abort ? 0 : n_pages); j += 32) {
    const int64_t pg = p0 + j;
    const uint32_t n_readers =
        (uint32_t)(k31_cta_of((pg + 1) * ipu - 1, n_items, grid) - k31_cta_of(pg * ipu, n_items, grid) + 1);
    unsigned long long old = __ldcg(readers + pg), assumed;
    do {
      assumed = old;
      const uint32_t cnt = (uint32_t)(assumed >> 32) == tag ? (uint32_t)assumed + 1u : 1u;
      old = atomicCAS(readers + pg, assumed, ((unsigned long long)tag << 32) | cnt);
    } while (old != assumed);
    const uint32_t before = (uint32_t)(old >> 32) == tag ? (uint32_t)old : 0u;
    if (before + 1u == n_readers) {
      __threadfence();  // every other reader's reads happened before its count
      k3_page_write(cl, s_op[j]);
    }
  }
  __syncwarp();
  if (lane == 0) {
    const int all_bits = abort ? 0 : (s_bits[0] | s_bits[1]);
    if (all_bits) atomicOr(reinterpret_cast<unsigned long long*>(totals + TPR_TOTALS_K31_STATUS),
                           (unsigned long long)all_bits);
    k31_item_share_done(totals, status, status_mirror, st0, epoch, abort, n_mine, rp.ticket);
    if (tracing) stamp(3);
  }
}

// ---------------------------------------------------------------------------
// K31 dynamic variant (knob k31 = 2): every page is decided exactly once, by
// the CTA whose static share of PAGES holds it, which applies its
// bookkeeping writes at once (no other CTA reads that page's entries) and
// stores its work item. A CTA then counts itself as decided and waits until
// every CTA has (a grid-wide dependency: the kernel is launched cooperatively,
// so all CTAs are resident), and copies items under K1's dynamic claims, so
// CTAs that stream faster take more items and none drains late. The claim,
// decided and status words are double-buffered by launch parity (rp.parity,
// tracked by the host per d_totals): CTA 0 resets the other parity's words,
// which only the previous launch on the stream used.
// ---------------------------------------------------------------------------
// The dynamic kernel's completion: the last CTA to finish its copies writes
// the status (already final: every CTA counted itself decided, bits first,
// before any copy) and then the caller's ticket into the pinned mirror.
__device__ __forceinline__ void k31_dyn_done(unsigned long long* words, int par, int64_t grid,
                                             int32_t* status_mirror, int32_t st0, int32_t ticket) {
  if (!ticket || !status_mirror) return;
  __threadfence();
  if (atomicAdd(&words[6 + par], 1ull) != (unsigned long long)grid - 1) return;
  __threadfence();
  const int32_t out = (int32_t)atomicOr(&words[4 + par], 0ull) | (st0 & TPR_STATUS_BARRIER_TIMEOUT);
  *reinterpret_cast<volatile int32_t*>(status_mirror) = out;
  __threadfence_system();  // the status word lands first
  *reinterpret_cast<volatile int32_t*>(status_mirror + 1) = ticket;
}

__global__ void __launch_bounds__(kK31Threads)
    tpr_k31_switch_dyn(const __grid_constant__ K31Params rp, tpr_kv_geometry_t geo,
                       KvCopyParams p, const __grid_constant__ KvClusterParams cl,
                       const __grid_constant__ KvTensorMaps tm, int64_t* __restrict__ totals,
                       int4* __restrict__ work, int32_t* __restrict__ status,
                       int32_t* status_mirror, int32_t stages, uint32_t piece) {
  __shared__ int s_bits[2];
  const unsigned tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  auto stamp = [&](int k) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    rp.trace[blockIdx.x * 8 + k] = t;
  };
  const bool tracing = rp.trace != nullptr;
  if (tracing && tid == 0) stamp(0);
  const int par = rp.parity & 1;
  unsigned long long* words = reinterpret_cast<unsigned long long*>(totals + TPR_TOTALS_K31_PAR);
  if (blockIdx.x == 0 && tid < 4) words[2 * tid + (par ^ 1)] = 0ull;
  const int n = rp.n, B = geo.block_tokens;
  const int32_t st0 = __ldcg(status);
  const bool abort = (st0 & TPR_STATUS_BARRIER_TIMEOUT) != 0;
  const int64_t n_mine = rp.n_mine, grid = gridDim.x;
  const int64_t pa = (int64_t)blockIdx.x * n_mine / grid;
  const int64_t pb = ((int64_t)blockIdx.x + 1) * n_mine / grid;
  int bits = 0;
  for (int64_t pg = pa + tid; pg < pb; pg += kK31Threads) {
    int lo = 0, hi = n;  // upper_bound(mine offsets, pg) - 1
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rp.off[0][mid] <= pg) lo = mid; else hi = mid;
    }
    const int32_t* r = rp.rec[lo];
    const int64_t local = pg - rp.off[0][lo];
    const int ctx = r[5], nblk = (ctx + B - 1) / B;
    const int h = r[3] + (int)(local / nblk);
    const int b = (int)(local - (int64_t)(h - r[3]) * nblk);
    const int ntok = (b == nblk - 1) ? ctx - b * B : B;
    const PageOp op = k3_page_decide(cl, geo, r[0], r[1], r[2], h, b, ntok, rp.off[1][lo] + local,
                                     rp.off[2][lo] + local);
    if (!abort) {
      k3_page_write(cl, op);
      work[pg] = op.item;
    }
    bits |= op.bits;
  }
  bits = (int)__reduce_or_sync(0xffffffffu, (unsigned)bits);
  if (lane == 0) s_bits[warp] = bits;
  __syncthreads();
  if (tid != 0) return;
  if (tracing) stamp(1);
  const int all_bits = abort ? 0 : (s_bits[0] | s_bits[1]);
  if (all_bits) atomicOr(&words[4 + par], (unsigned long long)all_bits);
  __threadfence();  // this CTA's writes and bits before its count
  if (atomicAdd(&words[2 + par], 1ull) == (unsigned long long)grid - 1) {
    __threadfence();
    const int32_t out = (int32_t)atomicOr(&words[4 + par], 0ull) | (st0 & TPR_STATUS_BARRIER_TIMEOUT);
    *status = out;
    if (status_mirror) *reinterpret_cast<volatile int32_t*>(status_mirror) = out;
    if (!abort) totals[0] = n_mine;
  }
  if (abort) {
    k31_dyn_done(words, par, grid, status_mirror, st0, rp.ticket);
    return;
  }
  // every page decided (and its bookkeeping written) before any copy reads
  // a work item
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&words[2 + par]) : "memory");
    if (v >= (unsigned long long)grid) break;
  }
  if (tracing) stamp(2);
  KvPieces it;
  it.work = work;
  it.work_l2 = true;
  it.n_items = n_mine * p.items_per_unit;
  it.p = p;
  it.cl = &cl;
  it.tm = &tm;
  it.piece = piece;
  if (rp.batch > 0) {
    it.claim = &words[par];
    it.batch = rp.batch;
  }
  it.start(blockIdx.x);
  bulk_pipeline<true>(it, stages, &tm);
  if (tracing) {
    stamp(3);
    rp.trace[blockIdx.x * 8 + 7] = (uint64_t)gridDim.x;
  }
  k31_dyn_done(words, par, grid, status_mirror, st0, rp.ticket);
}

// Ring shape per kernel (shared memory = stages x piece per CTA). Measured on
// B200 (profiles/README.md): K1 streams 32 KiB page items with one CTA per SM
// and a 192 KiB ring; 3 stages of 64 KiB (two items per stage) beat 6 x 32 KiB
// by 0.3% on cfg2 and 0.4% on the 70B switch, even on trace contexts; K2's row-parallel slices are 1-7 KiB rows, so it wants
// more issuing CTAs per SM: 3 x 32 KiB = 96 KiB, 2 CTAs/SM (with dynamic
// claims; 4 x 16 KiB / 3 CTAs/SM is within 1%, >= 128 KiB rings lose 25-45%,
// profiles/README.md). Override with TPR_BULK_K1 / TPR_BULK_K2 =
// "<stages>x<piece bytes>".
struct BulkConfig {
  int stages;
  uint32_t piece;
  int smem() const { return stages * (int)piece; }
};

static BulkConfig parse_bulk(const char* env, BulkConfig c) {
  if (const char* v = getenv(env)) {
    int st = 0;
    unsigned pc = 0;
    if (sscanf(v, "%dx%u", &st, &pc) == 2) {
      c.stages = st;
      c.piece = pc;
    }
  }
  if (c.stages < 3) c.stages = 3;
  if (c.stages > kMaxStages) c.stages = kMaxStages;
  c.piece = (c.piece / 16) * 16;
  if (c.piece < 1024) c.piece = 1024;
  while (c.smem() > 227 * 1024 && c.stages > 3) --c.stages;
  return c;
}

static const BulkConfig& k1_config() {
  static BulkConfig c = parse_bulk("TPR_BULK_K1", BulkConfig{3, 65536});
  return c;
}
// Short K1s (up to 24 items per SM, ~110 MiB) finish sooner with more,
// shallower rings: 3 x 32 KiB (2 CTAs/SM) takes a one-sequence switch from
// 21.5 to 19.4 us of device time, while 6 x 32 KiB stays ahead from cfg1 (4096 items, 27.7 per SM) up
// (profiles/ab/r01_k1small_*).
static const BulkConfig& k1_small_config() {
  static BulkConfig c = parse_bulk("TPR_BULK_K1_SMALL", BulkConfig{3, 32768});
  return c;
}
static int64_t k1_small_items() { return (int64_t)24 * sm_count(); }  // 24 items per SM
static const BulkConfig& k2_config() {
  static BulkConfig c = parse_bulk("TPR_BULK_K2", BulkConfig{3, 32768});
  return c;
}

static int bulk_grid(const void* fn, const BulkConfig& c, int64_t items, int threads) {
  // attribute + occupancy per (kernel, device, ring size) are fixed: set/query
  // once (the occupancy query costs microseconds of host time per small switch)
  struct Entry {
    const void* fn;
    int dev, smem, occ;
  };
  static thread_local Entry done[16];
  static thread_local int n_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = 0;
  for (int i = 0; i < n_done; ++i)
    if (done[i].fn == fn && done[i].dev == dev && done[i].smem == c.smem()) per_sm = done[i].occ;
  if (per_sm == 0) {
    // the attribute is an upper bound: keep the largest ring this kernel uses
    int attr = c.smem();
    for (int i = 0; i < n_done; ++i)
      if (done[i].fn == fn && done[i].dev == dev && done[i].smem > attr) attr = done[i].smem;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, attr);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, c.smem());
    if (per_sm < 1) per_sm = 1;
    if (n_done < 16) done[n_done++] = Entry{fn, dev, c.smem(), per_sm};
  }
  int64_t grid = (int64_t)sm_count() * per_sm;
  if (items < grid) grid = items;
  return grid < 1 ? 1 : (int)grid;
}

// items per dynamic claim for a K1 of `items` items: 4 (profiles/ab/
// r01_claimbatch_*: 2 contends on the counter, 4-6 best), or 0 (static
// grid-stride shares) below 32 items per SM, where a copy is too short to
// drift and every CTA should start at once
static int64_t k1_batch_for(int64_t items) {
  return items >= (int64_t)sm_count() * 32 ? 4 : 0;
}

// schedulable units of a K1 launch: items, or claim batches when dynamic
static int64_t k1_grid_units(int64_t items) {
  const int64_t b = k1_batch_for(items);
  return b > 0 ? (items + b - 1) / b : items;
}

static cudaError_t k1_launch(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                             int64_t n_units, cudaStream_t st, bool pdl, const KvTensorMaps& tm,
                             const BulkConfig& c) {
  const int64_t items = n_units * p.items_per_unit;
  const int grid = bulk_grid(reinterpret_cast<const void*>(&tpr_k1_kv_migrate_bulk), c,
                             k1_grid_units(items), 32);
  return launch_ex(tpr_k1_kv_migrate_bulk, dim3(grid), dim3(32), (size_t)c.smem(), st, pdl, work,
                   n_units, p, cl, tm, (int32_t)c.stages, (uint32_t)c.piece,
                   (int32_t)k1_batch_for(items));
}

cudaError_t launch_k1_bulk(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                           int64_t n_units, cudaStream_t st, bool pdl,
                           const tpr_kv_geometry_t* geo, int n_gpus, bool partial) {
  if (n_units <= 0) return cudaSuccess;

  const BulkConfig& c = n_units * p.items_per_unit <= k1_small_items() ? k1_small_config()
                                                                        : k1_config();
  KvTensorMaps tm;
  tm.enabled = 0;  // a plan of full pages needs no tensor map
  if (geo && partial) kv_tensor_maps(*geo, cl, n_gpus, c.piece, &tm);
  return k1_launch(p, cl, work, n_units, st, pdl, tm, c);
}

// K31 ring: 3 x 32 KiB, two CTAs per SM (a one-sequence switch: 19.5 ->
// 15.4 us of device time against 6 x 32 KiB with one CTA per SM, cfg1 even);
// TPR_BULK_K31 overrides
static const BulkConfig& k31_config() {
  static BulkConfig c = parse_bulk("TPR_BULK_K31", BulkConfig{3, 32768});
  return c;
}

// launch parity per d_totals (the dynamic K31's double-buffered words): the
// parity of a buffer's next launch; advanced only by a launch that succeeded
static std::mutex g_par_mu;
static std::unordered_map<const int64_t*, uint32_t> g_par;

cudaError_t launch_k31(const tpr_kv_geometry_t& geo, const KvCopyParams& p,
                       const KvClusterParams& cl, const int32_t* h_rec, int32_t n, int32_t filter,
                       int64_t n_units, int64_t* totals, int32_t* status, int32_t* status_mirror,
                       cudaStream_t st, int n_gpus, bool partial, int32_t* d_work, int variant,
                       int32_t ticket) {
  if (n < 1 || n > kK31Xfers || n_units < 1 || !d_work) return cudaErrorNotSupported;
  const BulkConfig& c = k31_config();
  KvTensorMaps tm;
  tm.enabled = 0;
  if (partial) kv_tensor_maps(geo, cl, n_gpus, c.piece, &tm);
  // schedule: item shares with redundant decisions for the smallest plans,
  // owner decisions + dynamic claims from 512 pages up (profiles/README.md
  // §4d: 116 pages 15.4 vs 19.5 us, 1024 pages 97.3 vs 93.0 us, 1792 pages
  // 160.8 vs 152.6 us); knob k31 = 2 / 3 forces one
  const bool dyn = variant == 2 || (variant == 1 && n_units >= kK31DynamicUnits);
  const void* fn = dyn ? reinterpret_cast<const void*>(&tpr_k31_switch_dyn)
                       : reinterpret_cast<const void*>(&tpr_k31_switch);
  const int64_t items = n_units * p.items_per_unit;
  const int grid = bulk_grid(fn, c, items, kK31Threads);
  if (!dyn && ((items + grid - 1) / grid + p.items_per_unit - 1) / p.items_per_unit + 1 >
                  kK31MaxPages)  // pages one CTA's share of the items touches
    return cudaErrorNotSupported;
  K31Params rp;
  memcpy(rp.rec, h_rec, sizeof(int32_t) * TPR_XFER_FIELDS * (size_t)n);
  // K3's three keyed exclusive scans (tpr_kernels.cu k3_scan_body), on the
  // host: the per-record offsets K3 would write to d_meta
  int64_t meta[kK31Xfers * TPR_META_FIELDS], mine = 0;
  tpr_record_offsets(h_rec, n, filter, geo.block_tokens, meta, &mine);
  for (int t = 0; t < n; ++t)
    for (int k = 0; k < 3; ++k) rp.off[k][t] = meta[t * TPR_META_FIELDS + k];
  rp.n_mine = mine;
  rp.n = n;
  rp.filter = filter;
  rp.trace = reinterpret_cast<uint64_t*>(k31_trace_buffer());
  rp.parity = 0;
  rp.batch = 0;
  rp.ticket = ticket;
  if (dyn) {
    // one item per claim (cfg1 52.2 us against 54.0 with 2 or 4 per claim)
    rp.batch = items > (int64_t)grid ? 1 : 0;  // 0: one static item each covers it
    std::lock_guard<std::mutex> lk(g_par_mu);
    uint32_t& par = g_par[totals];
    rp.parity = (int32_t)(par & 1u);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kK31Threads);
    cfg.dynamicSmemBytes = (size_t)c.smem();
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the decided wait
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int4* work = reinterpret_cast<int4*>(d_work);
    cudaError_t e = cudaLaunchKernelEx(&cfg, tpr_k31_switch_dyn, rp, geo, p, cl, tm, totals, work,
                                       status, status_mirror, (int32_t)c.stages, (uint32_t)c.piece);
    if (e == cudaSuccess) ++par;
    return e;
  }
  unsigned long long* readers = reinterpret_cast<unsigned long long*>(d_work);
  tpr_k31_switch<<<grid, kK31Threads, (size_t)c.smem(), st>>>(rp, geo, p, cl, tm, totals, readers,
                                                              status, status_mirror, c.stages,
                                                              c.piece);
  return cudaGetLastError();
}

cudaError_t launch_k2_bulk(const tpr_copy_seg_t* segs, const int64_t* prefix, int32_t n_segs,
                           int64_t n_items, int64_t chunk, int64_t* claim, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  const BulkConfig& c = k2_config();
  // dynamic claims hand out kClaimBatch items per CTA and batch
  const int64_t units = claim ? (n_items + kClaimBatch - 1) / kClaimBatch : n_items;
  const int grid = bulk_grid(reinterpret_cast<const void*>(&tpr_k2_copy_segments_bulk), c, units, 32);
  tpr_k2_copy_segments_bulk<<<grid, 32, c.smem(), st>>>(segs, prefix, n_segs, n_items, chunk, claim,
                                                        c.stages, c.piece);
  return cudaGetLastError();
}

}  // namespace tpr
