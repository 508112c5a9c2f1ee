// libtpr device side: the three kernels of the TP-reconfiguration data path
// for sm_100a, plus synthetic-data fill/verify kernels.
//
//   K3  tpr_k3_scan / tpr_k3_remap   block-table remap + free-ring allocation
//   K1  tpr_k1_kv_migrate            paged-KV head-shard movement
//   K2  tpr_k2_copy_segments         weight reshard (batched 2-D strided copy)
//
// All three are HBM/NVLink-bound byte movers; none of this work is GEMM-shaped,
// so there is no tensor-core path. The design rules that matter are 16-byte
// vector accesses, many bytes in flight per SM, and a persistent grid sized to
// the SM count (B200: 148 SMs).
#include <cuda_runtime.h>
#include <stdint.h>

#include "tpr.h"
#include "tpr_common.cuh"
#include "tpr_internal.h"
#include "tpr_k3page.cuh"

namespace tpr {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// 16-byte vector access helpers. Loads of source pages go through the
// non-coherent path without L1 allocation: every byte is read exactly once.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Warp-cooperative copy of a 2-D region: nr rows of nb bytes (nb % 16 == 0,
// all addresses 16-B aligned). The (row, vector) space is flattened so short
// rows still keep all 32 lanes x kUnroll vectors in flight.
template <int kUnroll>
__device__ __forceinline__ void warp_copy2d(const char* __restrict__ src,
                                            char* __restrict__ dst, uint32_t nr,
                                            uint32_t nb, int64_t src_pitch,
                                            int64_t dst_pitch, unsigned lane) {
  const uint32_t vpr = nb >> 4;  // vectors per row
  if (nr == 1 || ((int64_t)nb == src_pitch && (int64_t)nb == dst_pitch)) {
    const uint64_t nvec = (uint64_t)vpr * nr;
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    for (uint64_t base = 0; base < nvec; base += 32u * kUnroll) {
      int4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t k = base + (uint64_t)u * 32u + lane;
        if (k < nvec) v[u] = ld_stream(s + k);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t k = base + (uint64_t)u * 32u + lane;
        if (k < nvec) st_stream(d + k, v[u]);
      }
    }
    return;
  }
  const uint32_t nvec = vpr * nr;
  for (uint32_t base = 0; base < nvec; base += 32u * kUnroll) {
    int4 v[kUnroll];
    uint32_t row[kUnroll], col[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t k = base + (uint32_t)u * 32u + lane;
      row[u] = k / vpr;
      col[u] = k - row[u] * vpr;
      if (k < nvec)
        v[u] = ld_stream(reinterpret_cast<const int4*>(src + row[u] * src_pitch) + col[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t k = base + (uint32_t)u * 32u + lane;
      if (k < nvec)
        st_stream(reinterpret_cast<int4*>(dst + row[u] * dst_pitch) + col[u], v[u]);
    }
  }
}

// Byte-granular fallback for unaligned weight segments (never taken for the
// Llama geometries; kept so arbitrary shapes stay correct).
__device__ __forceinline__ void warp_copy2d_bytes(const char* src, char* dst, uint32_t nr,
                                                  uint32_t nb, int64_t sp, int64_t dp,
                                                  unsigned lane) {
  const uint64_t n = (uint64_t)nr * nb;
  for (uint64_t k = lane; k < n; k += 32) {
    const uint64_t r = k / nb, c = k - r * nb;
    dst[r * dp + c] = src[r * sp + c];
  }
}

// ---------------------------------------------------------------------------
// K3a: per-transfer offsets by block-wide keyed exclusive scans.
//
// For transfer t (plan order) with u_t = (head_hi-head_lo)*ceil(ctx/B) units:
//   mine_off  = sum of u over earlier transfers this caller processes
//   alloc_off = sum of u over earlier transfers with the same dst slot
//   rel_off   = sum of u over earlier transfers with the same src slot
// which is exactly where a sequential replay of the plan (apply_plan,
// migration.py:192-207) would put each head-block in the destination free
// ring and the source release ring. Keyed scans: warp level via
// __match_any_sync + shuffles, block level via a [warp][key] table.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kKeys = TPR_MAX_GPUS + 1;  // key TPR_MAX_GPUS = "no gpu" sink

// Three keyed exclusive scans in one pass (shared barriers; the 3 x kKeys
// column scans over the warp table run in parallel).
constexpr int kScans = 3;
__device__ __forceinline__ void block_keyed_exclusive3(const int (&key)[kScans],
                                                       const int64_t (&val)[kScans],
                                                       int64_t* s_tab,  // [kScans][warps][kKeys]
                                                       int64_t* s_run,  // [kScans][kKeys]
                                                       int64_t (&out)[kScans]) {
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;  // sized to the plan: small plans scan with one warp
  const int plane = nwarps * kKeys;
  for (int i = threadIdx.x; i < kScans * plane; i += blockDim.x) s_tab[i] = 0;
  __syncthreads();
  int64_t in_warp[kScans];
#pragma unroll
  for (int s = 0; s < kScans; ++s) {
    const unsigned peers = __match_any_sync(kFull, key[s]);
    const unsigned lower = peers & ((1u << lane) - 1u);
    int64_t acc = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t vj = __shfl_sync(kFull, val[s], j);
      if ((lower >> j) & 1u) acc += vj;
    }
    in_warp[s] = acc;
    if (lane == 31u - (unsigned)__clz(peers)) s_tab[s * plane + warp * kKeys + key[s]] = acc + val[s];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kScans * kKeys; c += blockDim.x) {  // one-warp blocks loop
    const int s = c / kKeys, k = c - s * kKeys;
    int64_t* col = s_tab + s * plane + k;
    int64_t run = s_run[c];
    for (int w = 0; w < nwarps; ++w) {
      const int64_t t = col[w * kKeys];
      col[w * kKeys] = run;
      run += t;
    }
    s_run[c] = run;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kScans; ++s) out[s] = s_tab[s * plane + warp * kKeys + key[s]] + in_warp[s];
  __syncthreads();
}

// Scan body (one CTA). Records are read from `xf_in`, which may be the
// caller's pinned host buffer (mapped: zero-copy over PCIe, no separate H2D
// copy) and are written to `xf` (device) when the two differ.
__device__ __forceinline__ int64_t k3_scan_body(const int32_t* xf_in,  // may alias xf
                                             int32_t* xf, int32_t n,
                                             int32_t block_tokens, int32_t filter,
                                             int64_t* __restrict__ meta,
                                             int64_t* __restrict__ totals,
                                             int32_t* s_xf = nullptr,    // shared copies
                                             int64_t* s_meta = nullptr)  // (fused K3, small n)
{
  __shared__ int64_t s_tab[kScans * kScanWarps * kKeys];
  __shared__ int64_t s_run[kScans][kKeys];
  for (int i = threadIdx.x; i < kScans * kKeys; i += blockDim.x) (&s_run[0][0])[i] = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int t = base + threadIdx.x;
    int src = TPR_MAX_GPUS, dst = TPR_MAX_GPUS;
    int64_t units = 0, mine = 0;
    if (t < n) {
      int32_t r[TPR_XFER_FIELDS];
      const int32_t* in = xf_in + (int64_t)t * TPR_XFER_FIELDS;
#pragma unroll
      for (int f = 0; f < TPR_XFER_FIELDS; ++f) r[f] = in[f];
      if (xf_in != xf) {
        int32_t* o = xf + (int64_t)t * TPR_XFER_FIELDS;
#pragma unroll
        for (int f = 0; f < TPR_XFER_FIELDS; ++f) o[f] = r[f];
      }
      if (s_xf != nullptr) {
#pragma unroll
        for (int f = 0; f < TPR_XFER_FIELDS; ++f) s_xf[t * TPR_XFER_FIELDS + f] = r[f];
      }
      const int32_t ctx = r[5];
      const int64_t nblk = ctx > 0 ? (ctx + block_tokens - 1) / block_tokens : 0;
      units = (int64_t)(r[4] - r[3]) * nblk;
      src = r[0] >= 0 ? r[0] : TPR_MAX_GPUS;
      dst = r[1] >= 0 ? r[1] : TPR_MAX_GPUS;
      mine = (filter < 0 || r[0] == filter) ? units : 0;
    }
    const int keys[kScans] = {0, dst, src};
    const int64_t vals[kScans] = {mine, dst < TPR_MAX_GPUS ? units : 0,
                                  src < TPR_MAX_GPUS ? units : 0};
    int64_t offs[kScans];
    block_keyed_exclusive3(keys, vals, s_tab, &s_run[0][0], offs);
    const int64_t mine_off = offs[0], alloc_off = offs[1], rel_off = offs[2];
    if (t < n) {
      int64_t* m = meta + (int64_t)t * TPR_META_FIELDS;
      m[0] = mine_off;
      m[1] = alloc_off;
      m[2] = rel_off;
      m[3] = mine;
      if (s_meta != nullptr) {
        int64_t* sm = s_meta + t * TPR_META_FIELDS;
        sm[0] = mine_off;
        sm[1] = alloc_off;
        sm[2] = rel_off;
        sm[3] = mine;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) totals[0] = s_run[0][0];
  if (threadIdx.x < TPR_MAX_GPUS) {
    totals[1 + threadIdx.x] = s_run[1][threadIdx.x];
    totals[1 + TPR_MAX_GPUS + threadIdx.x] = s_run[2][threadIdx.x];
  }
  return s_run[0][0];  // units this filter processes (every thread)
}

__global__ void __launch_bounds__(kScanThreads)
    tpr_k3_scan(const int32_t* xf_in, int32_t* xf, int32_t n,
                int32_t block_tokens, int32_t filter, int64_t* __restrict__ meta,
                int64_t* __restrict__ totals, int32_t* __restrict__ status) {
  pdl_trigger();  // the remap grid may get resident; it waits for this scan
  // the status word reports this K3 call only (the remap grid sets bits after
  // pdl_wait, i.e. after this store) -- unless a device barrier timed out into
  // it: then the bit stays and the remap grid aborts (k3_remap_body)
  if (threadIdx.x == 0 && !(*status & TPR_STATUS_BARRIER_TIMEOUT)) *status = 0;
  k3_scan_body(xf_in, xf, n, block_tokens, filter, meta, totals);
}

// ---------------------------------------------------------------------------
// K3b: expand every processed head-block into a work unit. Thread per unit;
// the owning transfer is found by binary search over mine_off. Order inside a
// transfer is head-major, block-minor (the order a sequential replay walks).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void k3_remap_body(const int32_t* __restrict__ xf, int32_t n,
                                              const int64_t* __restrict__ meta, int64_t n_mine,
                                              const tpr_kv_geometry_t& geo,
                                              const KvClusterParams& cl, int4* __restrict__ work,
                                              int4* __restrict__ work_ext,
                                              int32_t* __restrict__ status, int64_t first,
                                              int64_t stride, bool abort) {
  const int B = geo.block_tokens;
  // the int4 slot after the work list is K1's claim counter: zero it here, in
  // the kernel that K1 waits for
  if (first == 0) work[n_mine] = make_int4(0, 0, 0, 0);
  if (abort) {  // the start barrier timed out (a peer never arrived): touch no
    // table, ring or pool; K1 skips every item
    for (int64_t i = first; i < n_mine; i += stride) work[i] = make_int4(-1, -1, 0, 0);
    return;
  }
  for (int64_t i = first; i < n_mine; i += stride) {
    // upper_bound(mine_off, i) - 1
    int lo = 0, hi = n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (meta[(int64_t)mid * TPR_META_FIELDS] <= i) lo = mid; else hi = mid;
    }
    const int t = lo;
    const int32_t* r = xf + (int64_t)t * TPR_XFER_FIELDS;
    const int src = r[0], dst = r[1], req = r[2], h_lo = r[3], ctx = r[5];
    const int64_t* m = meta + (int64_t)t * TPR_META_FIELDS;
    const int64_t local = i - m[0];
    const int nblk = (ctx + B - 1) / B;
    const int h = h_lo + (int)(local / nblk);
    const int b = (int)(local - (int64_t)(h - h_lo) * nblk);
    const int ntok = (b == nblk - 1) ? ctx - b * B : B;
    int bits = 0;
    work[i] = k3_page(cl, geo, src, dst, req, h, b, ntok, m[1] + local, m[2] + local, bits);
    if (bits) atomicOr(status, bits);
    if (work_ext != nullptr) work_ext[i] = make_int4(req, h, b, t);
  }
}

__global__ void __launch_bounds__(256)
    tpr_k3_remap(const int32_t* __restrict__ xf, int32_t n, const int64_t* __restrict__ meta,
                 const int64_t* __restrict__ totals, tpr_kv_geometry_t geo,
                 KvClusterParams cl, int4* __restrict__ work, int4* __restrict__ work_ext,
                 int32_t* __restrict__ status) {
  pdl_trigger();  // K1 may get resident; it waits for the whole remap grid
  pdl_wait();     // the scan's offsets
  const bool abort = (__ldcg(status) & TPR_STATUS_BARRIER_TIMEOUT) != 0;
  k3_remap_body(xf, n, meta, totals[0], geo, cl, work, work_ext, status,
                (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x,
                abort);
}

constexpr int kFusedSmemXfers = 512;

// K3 fused (small plans): one CTA scans, then the same CTA expands every unit.
// Saves the second launch and its dependency gap; the scan's meta/totals are
// re-read from L2 by the block that wrote them (visible after __syncthreads).
__global__ void __launch_bounds__(kScanThreads)
    tpr_k3_fused(const int32_t* xf_in, int32_t* xf, int32_t n,
                 int32_t filter, int64_t* __restrict__ meta, int64_t* __restrict__ totals,
                 tpr_kv_geometry_t geo, KvClusterParams cl, int4* __restrict__ work,
                 int4* __restrict__ work_ext, int32_t* __restrict__ status,
                 int32_t* status_mirror) {
  // up to kFusedSmemXfers records and their offsets stay in shared memory, so
  // the per-unit binary search and record reads do not go to L2
  __shared__ int32_t s_xf[kFusedSmemXfers * TPR_XFER_FIELDS];
  __shared__ int64_t s_meta[kFusedSmemXfers * TPR_META_FIELDS];
  __shared__ int s_abort;
  const bool in_smem = n <= kFusedSmemXfers;
  pdl_trigger();
  if (threadIdx.x == 0) {  // this call's bits only, unless a device barrier timed out into it
    s_abort = (*status & TPR_STATUS_BARRIER_TIMEOUT) != 0;
    if (!s_abort) *status = 0;
  }
  __syncthreads();
  const int64_t n_mine = k3_scan_body(xf_in, xf, n, geo.block_tokens, filter, meta, totals,
                                      in_smem ? s_xf : nullptr, in_smem ? s_meta : nullptr);
  __syncthreads();
  k3_remap_body(in_smem ? s_xf : xf, n, in_smem ? s_meta : meta, n_mine, geo, cl, work,
                work_ext, status, threadIdx.x, blockDim.x, s_abort != 0);
  if (status_mirror != nullptr) {  // the status word, straight into pinned host memory
    __syncthreads();                // every thread's atomicOr has landed
    if (threadIdx.x == 0) *reinterpret_cast<volatile int32_t*>(status_mirror) = atomicOr(status, 0);
  }
}

// ---------------------------------------------------------------------------
// K1: paged-KV head-shard migration. A work item is `rows_per_item` rows
// ((layer, K|V) planes) of one page; a full page (ntok == B) is one contiguous
// span, a partial last page copies only its ntok valid tokens per plane.
// Persistent grid, warp-independent items, no block-level synchronisation.
// ---------------------------------------------------------------------------
template <int kUnroll>
__device__ __forceinline__ void k1_vector_item(const int4* __restrict__ work, int64_t item,
                                               const KvCopyParams& p, const KvClusterParams& cl,
                                               unsigned lane) {
  const int64_t u = item / p.items_per_unit;
  const int g = (int)(item - u * p.items_per_unit);
  const int4 w = work[u];
  const int src_slot = w.z & 0xffff, dst_slot = (w.z >> 16) & 0xffff, ntok = w.w;
  if (w.x < 0 || w.y < 0 || ntok <= 0) return;  // a page K3 refused (status word)
  const int row0 = g * p.rows_per_item;
  const int nr = min(p.rows_per_item, p.rows - row0);
  const char* s = reinterpret_cast<const char*>(cl.pool[src_slot]) + (int64_t)w.x * p.unit_bytes +
                  (int64_t)row0 * p.pitch;
  char* d = reinterpret_cast<char*>(cl.pool[dst_slot]) + (int64_t)w.y * p.unit_bytes +
            (int64_t)row0 * p.pitch;
  warp_copy2d<kUnroll>(s, d, (uint32_t)nr, (uint32_t)(ntok * p.tok_bytes), p.pitch, p.pitch, lane);
}

// dynamic: warps claim batches of kVecClaimBatch items from the counter after
// the work list (zeroed by K3), so warps stay on neighbouring items
constexpr int64_t kVecClaimBatch = 4;

template <int kUnroll>
__global__ void __launch_bounds__(kCopyThreads)
    tpr_k1_kv_migrate(const int4* __restrict__ work, int64_t n_units, KvCopyParams p,
                      KvClusterParams cl, int32_t dynamic) {
  pdl_wait();  // K3's work list (launched with programmatic serialization)
  const unsigned lane = threadIdx.x & 31u;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_items = n_units * p.items_per_unit;
  if (!dynamic) {
    for (int64_t item = gwarp; item < n_items; item += nwarps)
      k1_vector_item<kUnroll>(work, item, p, cl, lane);
    return;
  }
  unsigned long long* claim =
      reinterpret_cast<unsigned long long*>(const_cast<int4*>(work + n_units));
  for (int64_t batch = gwarp;;) {
    const int64_t first = batch * kVecClaimBatch;
    if (first >= n_items) break;
    unsigned long long nb = 0;  // the next batch, claimed one batch ahead
    if (lane == 0) nb = atomicAdd(claim, 1ull);
    nb = __shfl_sync(kFull, nb, 0);
    const int64_t last = min(first + kVecClaimBatch, n_items);
    for (int64_t item = first; item < last; ++item) k1_vector_item<kUnroll>(work, item, p, cl, lane);
    batch = nwarps + (int64_t)nb;
  }
}

// ---------------------------------------------------------------------------
// K2: weight reshard. Segments come from the host reshard planner (local
// re-layout copies and remote fetches of missing shard slices); an item is at
// most `chunk` bytes of one segment.
// ---------------------------------------------------------------------------
template <int kUnroll>
__global__ void __launch_bounds__(kCopyThreads)
    tpr_k2_copy_segments(const tpr_copy_seg_t* __restrict__ segs,
                         const int64_t* __restrict__ prefix, int32_t n_segs, int64_t n_items,
                         int64_t chunk) {
  const unsigned lane = threadIdx.x & 31u;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // items are dealt round-robin over warps: neighbouring warps stream
  // neighbouring chunks (measured faster than contiguous runs per warp)
  for (int64_t item = gwarp; item < n_items; item += nwarps) {
    int lo = 0, hi = n_segs;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (prefix[mid] <= item) lo = mid; else hi = mid;
    }
    const tpr_copy_seg_t sg = segs[lo];
    const int64_t k = item - prefix[lo];
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
    const char* s = reinterpret_cast<const char*>(sg.src) + r0 * sg.src_pitch + b0;
    char* d = reinterpret_cast<char*>(sg.dst) + r0 * sg.dst_pitch + b0;
    if (sg.flags & TPR_SEG_ALIGNED16)
      warp_copy2d<kUnroll>(s, d, (uint32_t)nr, (uint32_t)nb, sg.src_pitch, sg.dst_pitch, lane);
    else
      warp_copy2d_bytes(s, d, (uint32_t)nr, (uint32_t)nb, sg.src_pitch, sg.dst_pitch, lane);
  }
}

// ---------------------------------------------------------------------------
// Synthetic data: pattern fill of admitted pages, whole-pool garbage fill,
// full-size verification of block tables + page contents, weight slices.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    tpr_kv_fill_kernel(const int4* __restrict__ work, const int4* __restrict__ work_ext,
                       int64_t n_units, KvCopyParams p, KvClusterParams cl, uint64_t seed) {
  const unsigned lane = threadIdx.x & 31u;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_items = n_units * p.rows;
  for (int64_t item = gwarp; item < n_items; item += nwarps) {
    const int64_t u = item / p.rows;
    const int row = (int)(item - u * p.rows);
    const int4 w = work[u];
    if (w.y < 0 || w.w <= 0) continue;  // a page K3 refused
    const int4 e = work_ext[u];
    const uint64_t key = tpr_page_key(seed, (uint32_t)e.x, (uint32_t)e.y, (uint32_t)e.z);
    char* pool = reinterpret_cast<char*>(cl.pool[(w.z >> 16) & 0xffff]);
    uint4* d = reinterpret_cast<uint4*>(pool + (int64_t)w.y * p.unit_bytes + (int64_t)row * p.pitch);
    const uint32_t nvec = (uint32_t)(w.w * p.tok_bytes) >> 4;
    const uint64_t w0 = ((uint64_t)row * p.pitch) >> 2;
    for (uint32_t k = lane; k < nvec; k += 32) {
      const uint64_t wi = w0 + 4ull * k;
      d[k] = make_uint4(tpr_word(key, wi), tpr_word(key, wi + 1), tpr_word(key, wi + 2),
                        tpr_word(key, wi + 3));
    }
  }
}

__global__ void __launch_bounds__(256)
    tpr_pool_fill_kernel(KvCopyParams p, int64_t n_units, char* __restrict__ pool, int32_t slot,
                         uint64_t seed) {
  const int64_t vec_per_unit = p.unit_bytes >> 4;
  const int64_t total = n_units * vec_per_unit;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = k / vec_per_unit;
    const uint64_t wi = (uint64_t)(k - u * vec_per_unit) * 4ull;
    const uint64_t key = tpr_unit_key(seed, (uint32_t)slot, (uint32_t)u);
    reinterpret_cast<uint4*>(pool)[k] =
        make_uint4(tpr_word(key, wi), tpr_word(key, wi + 1), tpr_word(key, wi + 2),
                   tpr_word(key, wi + 3));
  }
}

__global__ void __launch_bounds__(256)
    tpr_kv_verify_kernel(tpr_kv_geometry_t geo, KvCopyParams p, const char* __restrict__ pool,
                         const int32_t* __restrict__ bt, const int32_t* __restrict__ ctx_by_slot,
                         const int32_t* __restrict__ owner, int32_t slot, uint64_t seed,
                         unsigned long long* __restrict__ counts) {
  const unsigned lane = threadIdx.x & 31u;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int H = geo.total_heads, MB = geo.max_blocks, B = geo.block_tokens;
  const int64_t n_entries = (int64_t)geo.n_req_slots * H * MB;
  unsigned long long placement_err = 0, mismatches = 0, checked = 0;
  for (int64_t idx = gwarp; idx < n_entries; idx += nwarps) {
    const int b = (int)(idx % MB);
    const int64_t rh = idx / MB;
    const int h = (int)(rh % H);
    const int req = (int)(rh / H);
    const int ctx = ctx_by_slot[req];
    const int nblk = ctx > 0 ? (ctx + B - 1) / B : 0;
    const bool expected = owner[rh] == slot && b < nblk;
    const int32_t unit = bt[idx];
    const bool present = unit >= 0;
    if (present != expected || (present && unit >= geo.n_units)) {
      if (lane == 0) ++placement_err;
      continue;
    }
    if (!present) continue;
    if (lane == 0) ++checked;
    const int ntok = (b == nblk - 1) ? ctx - b * B : B;
    const uint64_t key = tpr_page_key(seed, (uint32_t)req, (uint32_t)h, (uint32_t)b);
    const uint32_t vpr = (uint32_t)(ntok * p.tok_bytes) >> 4;
    const uint32_t nvec = vpr * (uint32_t)p.rows;
    const char* base = pool + (int64_t)unit * p.unit_bytes;
    for (uint32_t k = lane; k < nvec; k += 32) {
      const uint32_t row = k / vpr, col = k - row * vpr;
      const uint4 v = *reinterpret_cast<const uint4*>(base + (int64_t)row * p.pitch + 16ll * col);
      const uint64_t wi = (((uint64_t)row * p.pitch) >> 2) + 4ull * col;
      mismatches += (v.x != tpr_word(key, wi)) + (v.y != tpr_word(key, wi + 1)) +
                    (v.z != tpr_word(key, wi + 2)) + (v.w != tpr_word(key, wi + 3));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mismatches += __shfl_xor_sync(kFull, mismatches, o);
  if (lane == 0) {
    if (placement_err) atomicAdd(counts + 0, placement_err);
    if (mismatches) atomicAdd(counts + 1, mismatches);
    if (checked) atomicAdd(counts + 2, checked);
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
    tpr_matrix_kernel(char* __restrict__ buf, int64_t rows, int64_t cols, int64_t pitch,
                      int64_t row0, int64_t col0, int64_t full_cols, uint64_t key, bool verify,
                      unsigned long long* __restrict__ mismatch) {
  unsigned long long bad = 0;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    T* row = reinterpret_cast<T*>(buf) + r * pitch;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
         c += (int64_t)gridDim.x * blockDim.x) {
      const T want = (T)tpr_matrix_elem(key, (uint64_t)(row0 + r), (uint64_t)(col0 + c),
                                        (uint64_t)full_cols);
      if (verify) bad += (row[c] != want);
      else row[c] = want;
    }
  }
  if (verify) {
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(kFull, bad, o);
    if ((threadIdx.x & 31u) == 0 && bad) atomicAdd(mismatch, bad);
  }
}

// ---------------------------------------------------------------------------
// Device barrier over IPC-mapped flag arrays: lane r signals rank r, then
// lane r waits for rank r's signal in the local array.
// ---------------------------------------------------------------------------
struct BarrierParams {
  uint64_t flags[TPR_MAX_GPUS];
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void tpr_barrier_kernel(BarrierParams p, int32_t rank, int32_t world, uint64_t epoch,
                                   uint64_t timeout_ns, int32_t* status) {
  const int lane = threadIdx.x;
  // order every store this stream issued before (K1 pushes into peer pools,
  // K3 block-table writes) ahead of the signal, at system scope
  __threadfence_system();
  if (lane < world) {
    unsigned long long* peer = reinterpret_cast<unsigned long long*>(p.flags[lane]) + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer), "l"(epoch) : "memory");
    const unsigned long long* mine =
        reinterpret_cast<const unsigned long long*>(p.flags[rank]) + lane;
    const uint64_t t0 = globaltimer_ns();
    unsigned long long v = 0;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= epoch) break;
      // a peer that never arrives (crashed rank) must not wedge the GPU
      if (globaltimer_ns() - t0 > timeout_ns) {
        if (status) atomicOr(status, TPR_STATUS_BARRIER_TIMEOUT);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncwarp();
}

}  // namespace tpr

// ===========================================================================
// Launchers (called from tpr_api.cpp)
// ===========================================================================
namespace tpr {

static int copy_grid(const void* fn, int threads, int64_t want_warps) {
  int sms = sm_count();
  // occupancy per (kernel, device) is fixed: query once (the query costs
  // microseconds, which matters for small switches)
  static thread_local const void* cached_fn[8] = {nullptr};
  static thread_local int cached_dev[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  static thread_local int cached_occ[8] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = 0;
  for (int i = 0; i < 8; ++i)
    if (cached_fn[i] == fn && cached_dev[i] == dev) per_sm = cached_occ[i];
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
    if (per_sm < 1) per_sm = 1;
    for (int i = 0; i < 8; ++i)
      if (cached_fn[i] == nullptr) {
        cached_fn[i] = fn;
        cached_dev[i] = dev;
        cached_occ[i] = per_sm;
        break;
      }
  }
  const int64_t want_blocks = (want_warps * 32 + threads - 1) / threads;
  int64_t grid = (int64_t)sms * per_sm;
  if (want_blocks < grid) grid = want_blocks;
  return grid < 1 ? 1 : (int)grid;
}

cudaError_t launch_k3(const tpr_kv_geometry_t& geo, const KvClusterParams& cl,
                      const int32_t* xf_in, int32_t* xf, int32_t n, int32_t filter,
                      int64_t* meta, int64_t* totals, int64_t n_hint, int4* work,
                      int4* work_ext, int32_t* status, cudaStream_t st, int32_t* status_mirror,
                      bool* mirrored) {
  if (mirrored) *mirrored = false;
  int threads = ((n + 31) / 32) * 32;
  if (threads > kScanThreads) threads = kScanThreads;
  if (threads < 32) threads = 32;
  if (n_hint <= 0) n_hint = 1;
  if (n_hint <= k3_fuse_units()) {
    // small plan: one CTA scans and expands (one launch instead of two)
    int ft = threads;
    const int64_t want = ((n_hint + 31) / 32) * 32;
    if (want > ft) ft = (int)(want < kScanThreads ? want : kScanThreads);
    tpr_k3_fused<<<1, ft, 0, st>>>(xf_in, xf, n, filter, meta, totals, geo, cl, work, work_ext,
                                   status, status_mirror);
    if (mirrored) *mirrored = status_mirror != nullptr;
    return cudaGetLastError();
  }
  tpr_k3_scan<<<1, threads, 0, st>>>(xf_in, xf, n, geo.block_tokens, filter, meta, totals, status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t blocks = (n_hint + 255) / 256;
  const int64_t max_blocks = (int64_t)sm_count() * 8;
  if (blocks > max_blocks) blocks = max_blocks;
  return launch_ex(tpr_k3_remap, dim3((unsigned)blocks), dim3(256), 0, st, pdl_for(n_hint),
                   (const int32_t*)xf, n, (const int64_t*)meta, (const int64_t*)totals, geo, cl,
                   work, work_ext, status);
}

cudaError_t launch_k1(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                      int64_t n_units, cudaStream_t st, bool pdl) {
  if (n_units <= 0) return cudaSuccess;
  const void* fn = reinterpret_cast<const void*>(&tpr_k1_kv_migrate<kCopyUnroll>);
  const int64_t items = n_units * p.items_per_unit;
  const bool dyn = items >= (int64_t)sm_count() * 32;  // as the bulk K1
  const int grid = copy_grid(fn, kCopyThreads, dyn ? (items + kVecClaimBatch - 1) / kVecClaimBatch : items);
  return launch_ex(tpr_k1_kv_migrate<kCopyUnroll>, dim3(grid), dim3(kCopyThreads), 0, st, pdl,
                   work, n_units, p, cl, (int32_t)dyn);
}

cudaError_t launch_k2(const tpr_copy_seg_t* segs, const int64_t* prefix, int32_t n_segs,
                      int64_t n_items, int64_t chunk, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  const void* fn = reinterpret_cast<const void*>(&tpr_k2_copy_segments<kCopyUnroll>);
  const int grid = copy_grid(fn, kCopyThreads, n_items);
  tpr_k2_copy_segments<kCopyUnroll><<<grid, kCopyThreads, 0, st>>>(segs, prefix, n_segs,
                                                                   n_items, chunk);
  return cudaGetLastError();
}

cudaError_t launch_kv_fill(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                           const int4* work_ext, int64_t n_units, uint64_t seed, cudaStream_t st) {
  if (n_units <= 0) return cudaSuccess;
  const int64_t want = (n_units * p.rows * 32 + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  tpr_kv_fill_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(work, work_ext, n_units,
                                                                          p, cl, seed);
  return cudaGetLastError();
}

cudaError_t launch_pool_fill(const KvCopyParams& p, int64_t n_units, char* pool, int32_t slot,
                             uint64_t seed, cudaStream_t st) {
  tpr_pool_fill_kernel<<<sm_count() * 8, 256, 0, st>>>(p, n_units, pool, slot, seed);
  return cudaGetLastError();
}

cudaError_t launch_kv_verify(const tpr_kv_geometry_t& geo, const KvCopyParams& p,
                             const char* pool, const int32_t* bt, const int32_t* ctx,
                             const int32_t* owner, int32_t slot, uint64_t seed,
                             unsigned long long* counts, cudaStream_t st) {
  tpr_kv_verify_kernel<<<sm_count() * 8, 256, 0, st>>>(geo, p, pool, bt, ctx, owner, slot, seed,
                                                       counts);
  return cudaGetLastError();
}

cudaError_t launch_barrier(const uint64_t* flags, int32_t rank, int32_t world, uint64_t epoch,
                           uint64_t timeout_ns, int32_t* status, cudaStream_t st) {
  BarrierParams p{};
  for (int i = 0; i < world; ++i) p.flags[i] = flags[i];
  tpr_barrier_kernel<<<1, 32, 0, st>>>(p, rank, world, epoch, timeout_ns, status);
  return cudaGetLastError();
}

cudaError_t launch_matrix(char* buf, int64_t rows, int64_t cols, int64_t pitch, int64_t row0,
                          int64_t col0, int64_t full_cols, uint64_t key, int32_t elem_bytes,
                          bool verify, unsigned long long* mismatch, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t gx64 = (cols + 255) / 256;
  const unsigned gx = (unsigned)(gx64 < 64 ? gx64 : 64);
  const unsigned gy = (unsigned)(rows < 16384 ? rows : 16384);
  dim3 grid(gx, gy);
  switch (elem_bytes) {
    case 1:
      tpr_matrix_kernel<uint8_t><<<grid, 256, 0, st>>>(buf, rows, cols, pitch, row0, col0,
                                                       full_cols, key, verify, mismatch);
      break;
    case 2:
      tpr_matrix_kernel<uint16_t><<<grid, 256, 0, st>>>(buf, rows, cols, pitch, row0, col0,
                                                        full_cols, key, verify, mismatch);
      break;
    case 4:
      tpr_matrix_kernel<uint32_t><<<grid, 256, 0, st>>>(buf, rows, cols, pitch, row0, col0,
                                                        full_cols, key, verify, mismatch);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace tpr
