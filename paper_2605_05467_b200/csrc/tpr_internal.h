// Internal interfaces between the C-ABI layer (tpr_api.cpp) and the kernels.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded through cudaGetDriverEntryPoint, no -lcuda)
#include <cuda_runtime.h>
#include <stdint.h>

#include "tpr.h"

namespace tpr {

// Sets tpr_last_error() (printf-style) and returns `code`.
int set_error(int code, const char* fmt, ...);

constexpr int kCopyThreads = 256;  // 8 warps per CTA, warp-independent items
constexpr int kCopyUnroll = 8;     // 8 x 16 B x 32 lanes = 4 KiB in flight per warp
constexpr int kRowsPerItemTarget = 32 * 1024;  // bytes of one K1 work item

// Pointer tables passed by value as kernel parameters (<= 4 KiB).
struct KvClusterParams {
  uint64_t pool[TPR_MAX_GPUS];
  uint64_t block_table[TPR_MAX_GPUS];
  uint64_t free_ring[TPR_MAX_GPUS];
  int64_t ring_head[TPR_MAX_GPUS];
  int64_t ring_tail[TPR_MAX_GPUS];
  int64_t units[TPR_MAX_GPUS];  // ring capacity per slot (resolved, > 0)
};

// Derived page geometry for the copy/fill kernels.
struct KvCopyParams {
  int64_t unit_bytes;     // bytes of one pool unit
  int64_t pitch;          // bytes of one (layer, K|V) plane = block_tokens * tok_bytes
  int32_t tok_bytes;      // head_dim * dtype_bytes
  int32_t rows;           // planes per unit = 2 * layers
  int32_t rows_per_item;  // planes per K1 work item
  int32_t items_per_unit;
};

// TMA tensor maps of the KV pools, one per GPU slot, for the partial pages of
// K1 (bulk engine). A pool is viewed as a 3-D tensor of 8-byte elements
//   d0 = tok_bytes / 8 (one token of one plane), d1 = block_tokens, d2 = planes
// (units x rows), and one box is {one token} x {r_box planes}: the valid
// tokens of a partial page move as ntok x (rows / r_box) tensor copies of
// r_box x tok_bytes bytes instead of `rows` short row copies.
struct KvTensorMaps {
  CUtensorMap map[TPR_MAX_GPUS];  // 64-byte aligned (CUtensorMap is)
  int32_t enabled;                // 0: partial pages use row copies
  int32_t r_box;                  // planes per tensor copy (divides rows)
  int32_t n_pb;                   // rows / r_box
  int32_t _pad;
};

// K31 (fused small switch): the plan's records ride in the kernel parameters.
constexpr int kK31Xfers = 96;      // records per fused launch (2304 B of parameters)
constexpr int kK31MaxPages = 64;   // pages one CTA owns
struct K31Params {
  int32_t rec[kK31Xfers][TPR_XFER_FIELDS];
  // per record: units before it that this rank moves (filter), that its
  // destination ring hands out, that its source ring takes back -- the three
  // keyed exclusive scans K3 does on the device, done on the host (the
  // records are on the host anyway)
  int64_t off[3][kK31Xfers];
  int64_t n_mine;   // units this rank moves
  int32_t n;
  int32_t filter;
  int32_t parity;   // dynamic kernel: which scratch words of d_totals this launch uses
  int32_t batch;    // dynamic kernel: items per claim (0 = static shares)
  int32_t ticket;   // != 0: written to status_mirror[1] once every copy and write is done
  uint64_t* trace;  // nullable: per-CTA globaltimer stamps (knob "k31_trace")
};
int64_t k31_trace_buffer();

// Tensor maps for the pools of `cl` (cached per pool); out->enabled = 0 when
// the geometry does not fit TMA's limits or the driver entry point is missing.
void kv_tensor_maps(const tpr_kv_geometry_t& geo, const KvClusterParams& cl, int n_gpus,
                    uint32_t piece_bytes, KvTensorMaps* out);
void kv_tensor_maps_uncached(const tpr_kv_geometry_t& geo, const KvClusterParams& cl, int n_gpus,
                             uint32_t piece_bytes, KvTensorMaps* out);
bool tensor_partial_enabled();

int sm_count();

// Device index owning a device address (-1: host / unknown), cached per
// allocation range; all_local: every non-null pointer is on the current device.
int ptr_device(uint64_t p);
bool all_local(const uint64_t* ptrs, int n);
void forget_ranges();

// The plan size (units) up to which K3 runs as one fused CTA (or the whole
// switch as K31; TPR_K3_FUSE_UNITS, 0 = never); programmatic dependent launch
// of K3b / K1 behind their producer is used up to the same size.
int64_t k3_fuse_units();
bool pdl_for(int64_t n_units);

// tpr_kv_switch with an optional pinned host mirror of the status word, kept
// current on the stream (fused K3 store, else a 4-byte D2H after K1)
// k1_events (nullable): cudaEvent_t pair recorded on the stream around K1.
// ticket (nullable, out): when the switch ran as K31 with a status mirror, a
// nonzero number the kernel writes to status_mirror[1] once every copy and
// table write is done (the caller may spin on it); 0 otherwise.
int kv_switch_impl(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                   const int32_t* h_xfers, int32_t* d_xfers, int32_t n_xfers, int32_t filter_src,
                   int64_t* d_meta, int64_t* d_totals, int64_t n_units, int32_t* d_work,
                   int32_t* d_status, void* stream, int32_t* status_mirror,
                   void* const* k1_events = nullptr, int32_t* records_async = nullptr,
                   int32_t* ticket = nullptr);

// cudaLaunchKernelEx with the programmatic-serialization attribute when `pdl`.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t st, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? attr : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}

// xf_in: records as the caller holds them (device memory, or mapped pinned
// host memory read zero-copy); xf: the device copy K3b reads (may equal xf_in).
// status_mirror (nullable, pinned host memory): the fused K3 stores the status
// word there at its end; *mirrored tells whether it did (the split K3 does not).
cudaError_t launch_k3(const tpr_kv_geometry_t& geo, const KvClusterParams& cl,
                      const int32_t* xf_in, int32_t* xf, int32_t n, int32_t filter,
                      int64_t* meta, int64_t* totals, int64_t n_hint, int4* work,
                      int4* work_ext, int32_t* status, cudaStream_t st,
                      int32_t* status_mirror = nullptr, bool* mirrored = nullptr);
// pdl: launched right behind K3 on the same stream (waits for it on device)
cudaError_t launch_k1(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                      int64_t n_units, cudaStream_t st, bool pdl);
cudaError_t launch_k2(const tpr_copy_seg_t* segs, const int64_t* prefix, int32_t n_segs,
                      int64_t n_items, int64_t chunk, cudaStream_t st);
// TMA bulk-copy engine variants (tpr_bulk.cu)
cudaError_t launch_k1_bulk(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                           int64_t n_units, cudaStream_t st, bool pdl,
                           const tpr_kv_geometry_t* geo, int n_gpus, bool partial);
// K31: n_units pages, records from host memory (copied into the parameters);
// returns cudaErrorNotSupported when the plan does not fit the fused path.
cudaError_t launch_k31(const tpr_kv_geometry_t& geo, const KvCopyParams& p,
                       const KvClusterParams& cl, const int32_t* h_rec, int32_t n, int32_t filter,
                       int64_t n_units, int64_t* totals, int32_t* status, int32_t* status_mirror,
                       cudaStream_t st, int n_gpus, bool partial, int32_t* d_work,
                       int variant, int32_t ticket = 0);
cudaError_t launch_k2_bulk(const tpr_copy_seg_t* segs, const int64_t* prefix, int32_t n_segs,
                           int64_t n_items, int64_t chunk, int64_t* claim, cudaStream_t st);
cudaError_t launch_kv_fill(const KvCopyParams& p, const KvClusterParams& cl, const int4* work,
                           const int4* work_ext, int64_t n_units, uint64_t seed,
                           cudaStream_t st);
cudaError_t launch_pool_fill(const KvCopyParams& p, int64_t n_units, char* pool, int32_t slot,
                             uint64_t seed, cudaStream_t st);
cudaError_t launch_kv_verify(const tpr_kv_geometry_t& geo, const KvCopyParams& p,
                             const char* pool, const int32_t* bt, const int32_t* ctx,
                             const int32_t* owner, int32_t slot, uint64_t seed,
                             unsigned long long* counts, cudaStream_t st);
cudaError_t launch_barrier(const uint64_t* flags, int32_t rank, int32_t world, uint64_t epoch,
                           uint64_t timeout_ns, int32_t* status, cudaStream_t st);
cudaError_t launch_matrix(char* buf, int64_t rows, int64_t cols, int64_t pitch, int64_t row0,
                          int64_t col0, int64_t full_cols, uint64_t key, int32_t elem_bytes,
                          bool verify, unsigned long long* mismatch, cudaStream_t st);

}  // namespace tpr
