// libtpr C ABI (see include/tpr.h). Host-side validation, the native head
// planner, segment preparation for K2, and thin launch wrappers.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>
#include <string>

#include "tpr.h"
#include "tpr_common.cuh"
#include "tpr_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int vfail(int code, const char* fmt, va_list ap) {
  char buf[512];
  vsnprintf(buf, sizeof(buf), fmt, ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(TPR_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int check_geometry(const tpr_kv_geometry_t* g) {
  if (!g) return fail(TPR_EINVAL, "null geometry");
  if (g->layers <= 0 || g->head_dim <= 0 || g->dtype_bytes <= 0 || g->block_tokens <= 0 ||
      g->total_heads <= 0 || g->max_blocks <= 0 || g->n_req_slots <= 0 || g->n_units <= 0)
    return fail(TPR_EINVAL, "geometry fields must be positive");
  if ((g->head_dim * g->dtype_bytes) % 16 != 0)
    return fail(TPR_EINVAL, "head_dim*dtype_bytes=%d is not a multiple of 16 bytes",
                g->head_dim * g->dtype_bytes);
  return TPR_OK;
}

tpr::KvCopyParams copy_params(const tpr_kv_geometry_t* g) {
  tpr::KvCopyParams p;
  p.tok_bytes = g->head_dim * g->dtype_bytes;
  p.pitch = (int64_t)g->block_tokens * p.tok_bytes;
  p.rows = 2 * g->layers;
  p.unit_bytes = p.pitch * p.rows;
  int64_t rpi = tpr::kRowsPerItemTarget / p.pitch;
  if (rpi < 1) rpi = 1;
  if (rpi > p.rows) rpi = p.rows;
  p.rows_per_item = (int32_t)rpi;
  p.items_per_unit = (p.rows + p.rows_per_item - 1) / p.rows_per_item;
  return p;
}

int cluster_params(const tpr_kv_cluster_t* cl, const tpr_kv_geometry_t* geo,
                   tpr::KvClusterParams* out) {
  if (!cl) return fail(TPR_EINVAL, "null cluster");
  if (cl->n_gpus <= 0 || cl->n_gpus > TPR_MAX_GPUS)
    return fail(TPR_EINVAL, "n_gpus=%d outside [1, %d]", cl->n_gpus, TPR_MAX_GPUS);
  std::memset(out, 0, sizeof(*out));
  for (int g = 0; g < cl->n_gpus; ++g) {
    out->pool[g] = cl->pool[g];
    out->block_table[g] = cl->block_table[g];
    out->free_ring[g] = cl->free_ring[g];
    out->ring_head[g] = cl->ring_head[g];
    out->ring_tail[g] = cl->ring_tail[g];
    out->units[g] = cl->units[g] > 0 ? cl->units[g] : geo->n_units;
    if (out->units[g] > geo->n_units)
      return fail(TPR_EINVAL, "slot %d: units %lld exceed geometry n_units %d", g,
                  (long long)out->units[g], geo->n_units);
  }
  return TPR_OK;
}

// TMA bulk engine by default: K1 at the measured HBM copy peak with one
// issuing thread per CTA (profiles/README.md); the vector engine stays
// selectable (tpr_set_copy_engine) for comparison.
std::atomic<int> g_engine{TPR_ENGINE_BULK};
// the engine the last K1 / K2 launch used (tpr_get_tuning "k1_engine_last" /
// "k2_engine_last"; -1 before the first launch)
std::atomic<int> g_k1_last{-1}, g_k2_last{-1};

// partial: the plan may contain partial pages (context not a multiple of the
// page size); only then does K1 need the pools' tensor maps. The TMA engine
// runs only when every pool of the cluster is the launching device's own HBM
// (tpr::all_local); a cluster with peer-mapped pools (one process per GPU,
// pools on other GPUs) takes the 16-byte vector engine.
cudaError_t run_k1(const tpr_kv_geometry_t* geo, int n_gpus, const tpr::KvCopyParams& p,
                   const tpr::KvClusterParams& cl, const int4* work, int64_t n, cudaStream_t st,
                   bool pdl, bool partial = true) {
  const bool bulk = g_engine.load() == TPR_ENGINE_BULK && tpr::all_local(cl.pool, n_gpus);
  g_k1_last.store(bulk ? TPR_ENGINE_BULK : TPR_ENGINE_VECTOR);
  return bulk ? tpr::launch_k1_bulk(p, cl, work, n, st, pdl, geo, n_gpus, partial)
              : tpr::launch_k1(p, cl, work, n, st, pdl);
}

bool any_partial(const int32_t* rec, int32_t n, int32_t block_tokens) {
  for (int32_t t = 0; t < n; ++t)
    if (rec[t * TPR_XFER_FIELDS + 5] % block_tokens) return true;
  return false;
}

// Records in caller memory the device can read directly: pinned (page-locked)
// host memory under unified addressing, or device memory. Then K3 reads them
// in place and the separate H2D copy disappears from the switch.
int64_t env_i64(const char* name, int64_t dflt);

// Launch-path knobs (process-wide): initialised from the environment, changed
// at run time with tpr_set_tuning (tests cover every combination).
std::atomic<int64_t> g_fuse{-1}, g_tensor{-1}, g_k31{-1}, g_k31_trace{0};

int64_t knob(std::atomic<int64_t>& k, const char* env, int64_t dflt) {
  int64_t v = k.load(std::memory_order_relaxed);
  if (v < 0) {
    v = env_i64(env, dflt);
    if (v < 0) v = 0;
    k.store(v, std::memory_order_relaxed);
  }
  return v;
}

// pinned or pageable host memory (the CPU can read it); not device memory.
// Host answers are cached per address: under unified addressing a host
// address is never a device address, so a cached "host" stays true.
bool host_readable(const int32_t* h) {
  thread_local const void* seen[8] = {nullptr};
  thread_local int next = 0;
  for (const void* s : seen)
    if (s == h) return true;
  cudaPointerAttributes a;
  bool host = true;  // unregistered host memory fails the query
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) cudaGetLastError();
  else host = a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
  if (host) {
    seen[next] = h;
    next = (next + 1) % 8;
  }
  return host;
}

const int32_t* device_view(const int32_t* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
      a.type == cudaMemoryTypeManaged)
    return static_cast<const int32_t*>(a.devicePointer);
  return nullptr;  // pageable
}

int64_t env_i64(const char* name, int64_t dflt) {
  const char* v = getenv(name);
  return (v && *v) ? strtoll(v, nullptr, 10) : dflt;
}

// local: every segment's source and destination is the launching device's
// own HBM (tpr_weight_reshard_host checks; tpr_weight_reshard, which only sees
// device-side segments, trusts the engine setting)
cudaError_t run_k2(const tpr_copy_seg_t* segs, const int64_t* prefix, int32_t n_segs,
                   int64_t n_items, int64_t chunk, int64_t* claim, cudaStream_t st,
                   bool local = true) {
  const bool bulk = g_engine.load() == TPR_ENGINE_BULK && local;
  g_k2_last.store(bulk ? TPR_ENGINE_BULK : TPR_ENGINE_VECTOR);
  return bulk ? tpr::launch_k2_bulk(segs, prefix, n_segs, n_items, chunk, claim, st)
              : tpr::launch_k2(segs, prefix, n_segs, n_items, chunk, st);
}

}  // namespace

namespace tpr {
// knob "tensor_partial": 0 row copies, 1 tensor boxes when a page is partial
// (default)
bool tensor_partial_enabled() { return knob(g_tensor, "TPR_TENSOR_PARTIAL", 1) != 0; }

// ---------------------------------------------------------------------------
// TMA tensor maps of the KV pools (K1 partial pages, tpr_internal.h).
// ---------------------------------------------------------------------------
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<EncodeTiled>(f);
  }();
  return fn;
}

struct MapKey {
  uint64_t pool;
  int64_t units;
  int32_t tok_bytes, block_tokens, rows, r_box;
  bool operator==(const MapKey& o) const {
    return pool == o.pool && units == o.units && tok_bytes == o.tok_bytes &&
           block_tokens == o.block_tokens && rows == o.rows && r_box == o.r_box;
  }
};

// one encoded map per pool, reused across switches (encoding costs ~us)
bool pool_map(const MapKey& k, CUtensorMap* out) {
  static std::mutex mu;
  static std::vector<std::pair<MapKey, CUtensorMap>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.first == k) {
      *out = e.second;
      return true;
    }
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(k.tok_bytes / 8), (cuuint64_t)k.block_tokens,
                              (cuuint64_t)k.units * (cuuint64_t)k.rows};
  const cuuint64_t strides[2] = {(cuuint64_t)k.tok_bytes,
                                 (cuuint64_t)k.tok_bytes * (cuuint64_t)k.block_tokens};
  const cuuint32_t box[3] = {(cuuint32_t)(k.tok_bytes / 8), 1u, (cuuint32_t)k.r_box};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  CUtensorMap m;
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, reinterpret_cast<void*>(k.pool), dims, strides,
          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() >= 256) cache.erase(cache.begin());
  cache.emplace_back(k, m);
  *out = m;
  return true;
}

// Programmatic dependent launch of K3b / K1 pays for small plans (its launch
// overlap is worth a few us); on a large K1 it was -2.5% under the static
// schedule and is neutral with dynamic claims (profiles/ab/r01_pdl_*), so
// large plans launch K1 normally.
bool pdl_for(int64_t n_units) { return n_units <= k3_fuse_units(); }

int64_t k31_trace_buffer() { return g_k31_trace.load(std::memory_order_relaxed); }

int64_t k3_fuse_units() {
  // one 1024-thread CTA expands up to 4 units per thread faster than a second
  // launch + dependency gap (measured, profiles/README.md)
  return knob(g_fuse, "TPR_K3_FUSE_UNITS", 4096);
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfail(code, fmt, ap);
  va_end(ap);
  return code;
}

// ---------------------------------------------------------------------------
// Pointer locality. The TMA engine (cp.async.bulk, tensor maps) is validated
// on the launching device's own HBM only; addresses that belong to another
// GPU (peer mappings over NVLink, CUDA-IPC handles of another device) are
// moved with plain 16-byte loads/stores. The owning device of an address is
// cached per allocation range (cuMemGetAddressRange), so a switch pays a few
// range compares, not a driver query per pointer.
// ---------------------------------------------------------------------------
using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

GetRange range_fn() {
  static GetRange fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<GetRange>(f);
  }();
  return fn;
}

struct DevRange {
  uint64_t lo, hi;
  int dev;
};
std::mutex g_range_mu;
std::vector<DevRange> g_ranges;

int ptr_device(uint64_t p) {
  {
    std::lock_guard<std::mutex> lock(g_range_mu);
    for (const DevRange& r : g_ranges)
      if (p >= r.lo && p < r.hi) return r.dev;
  }
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, reinterpret_cast<const void*>(p)) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  const int dev = a.type == cudaMemoryTypeDevice ? a.device : -1;
  CUdeviceptr base = 0;
  size_t size = 0;
  GetRange fn = range_fn();
  if (dev >= 0 && fn && fn(&base, &size, (CUdeviceptr)p) == CUDA_SUCCESS && size > 0) {
    std::lock_guard<std::mutex> lock(g_range_mu);
    if (g_ranges.size() >= 4096) g_ranges.clear();
    g_ranges.push_back(DevRange{(uint64_t)base, (uint64_t)base + size, dev});
  }
  return dev;
}

std::atomic<uint64_t> g_range_gen{0};  // bumped when allocations go away (memos below)

void forget_ranges() {
  std::lock_guard<std::mutex> lock(g_range_mu);
  g_ranges.clear();
  g_range_gen.fetch_add(1);
}

bool all_local(const uint64_t* ptrs, int n) {
  int cur = 0;
  cudaGetDevice(&cur);
  // the last answer per thread: a switch asks about the same pools every call
  thread_local int last_dev = -1, last_n = -1;
  thread_local uint64_t last_ptrs[TPR_MAX_GPUS], last_gen = ~0ull;
  thread_local bool last_local = false;
  const uint64_t gen = g_range_gen.load(std::memory_order_relaxed);
  if (n >= 0 && n <= TPR_MAX_GPUS && cur == last_dev && n == last_n && gen == last_gen &&
      memcmp(ptrs, last_ptrs, sizeof(uint64_t) * (size_t)n) == 0)
    return last_local;
  bool local = true;
  for (int i = 0; i < n && local; ++i)
    if (ptrs[i] && ptr_device(ptrs[i]) != cur) local = false;
  if (n >= 0 && n <= TPR_MAX_GPUS) {
    last_dev = cur;
    last_n = n;
    last_gen = gen;
    memcpy(last_ptrs, ptrs, sizeof(uint64_t) * (size_t)n);
    last_local = local;
  }
  return local;
}

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

void kv_tensor_maps(const tpr_kv_geometry_t& geo, const KvClusterParams& cl, int n_gpus,
                    uint32_t piece_bytes, KvTensorMaps* out) {
  // the last result per thread and ring piece (K1 and K31 ask with different
  // pieces): a switch asks about the same pools every call
  struct Memo {
    int dev = -1, n = -1, tok = 0, rows = 0, bt = 0, enabled_knob = -1;
    uint32_t piece = 0;
    uint64_t pool[TPR_MAX_GPUS];
    int64_t units[TPR_MAX_GPUS];
    KvTensorMaps tm;
  };
  thread_local Memo memo[2];
  int dev = 0;
  cudaGetDevice(&dev);
  const int knob_now = tensor_partial_enabled() ? 1 : 0;
  for (Memo& m : memo)
    if (m.dev == dev && m.n == n_gpus && m.piece == piece_bytes && m.enabled_knob == knob_now &&
        m.tok == geo.head_dim * geo.dtype_bytes && m.rows == 2 * geo.layers &&
        m.bt == geo.block_tokens && n_gpus >= 0 && n_gpus <= TPR_MAX_GPUS &&
        memcmp(m.pool, cl.pool, sizeof(uint64_t) * (size_t)n_gpus) == 0 &&
        memcmp(m.units, cl.units, sizeof(int64_t) * (size_t)n_gpus) == 0) {
      *out = m.tm;
      return;
    }
  kv_tensor_maps_uncached(geo, cl, n_gpus, piece_bytes, out);
  if (n_gpus < 0 || n_gpus > TPR_MAX_GPUS) return;
  Memo& m = memo[memo[0].piece == piece_bytes || memo[0].dev < 0 ? 0 : 1];
  m.dev = dev;
  m.n = n_gpus;
  m.piece = piece_bytes;
  m.enabled_knob = knob_now;
  m.tok = geo.head_dim * geo.dtype_bytes;
  m.rows = 2 * geo.layers;
  m.bt = geo.block_tokens;
  memcpy(m.pool, cl.pool, sizeof(uint64_t) * (size_t)n_gpus);
  memcpy(m.units, cl.units, sizeof(int64_t) * (size_t)n_gpus);
  m.tm = *out;
}

void kv_tensor_maps_uncached(const tpr_kv_geometry_t& geo, const KvClusterParams& cl, int n_gpus,
                             uint32_t piece_bytes, KvTensorMaps* out) {
  out->enabled = 0;
  const int32_t tok = geo.head_dim * geo.dtype_bytes;
  const int32_t rows = 2 * geo.layers;
  if (!tensor_partial_enabled() || tok % 16 || tok / 8 > 256 || geo.block_tokens > 256 ||
      n_gpus < 1 || n_gpus > TPR_MAX_GPUS)
    return;
  if (!all_local(cl.pool, n_gpus)) return;  // never a tensor map over a peer mapping
  // planes per tensor copy: the largest divisor of rows with <= 256 planes
  // whose box fits one ring stage
  int32_t r_box = 0;
  for (int32_t r = rows < 256 ? rows : 256; r >= 1; --r)
    if (rows % r == 0 && (int64_t)r * tok <= (int64_t)piece_bytes) {
      r_box = r;
      break;
    }
  if (r_box == 0 || (int64_t)r_box * tok % 128) return;
  for (int g = 0; g < n_gpus; ++g) {
    if (cl.pool[g] % 16) return;
    MapKey k{cl.pool[g], cl.units[g], tok, geo.block_tokens, rows, r_box};
    if (!pool_map(k, &out->map[g])) return;
  }
  out->r_box = r_box;
  out->n_pb = rows / r_box;
  out->enabled = 1;
}

int kv_switch_impl(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                   const int32_t* h_xfers, int32_t* d_xfers, int32_t n_xfers, int32_t filter_src,
                   int64_t* d_meta, int64_t* d_totals, int64_t n_units, int32_t* d_work,
                   int32_t* d_status, void* stream, int32_t* status_mirror,
                   void* const* k1_events, int32_t* records_async, int32_t* ticket) {
  if (records_async) *records_async = h_xfers != nullptr;
  if (ticket) *ticket = 0;
  int rc = check_geometry(geo);
  if (rc) return rc;
  KvClusterParams cp;
  if ((rc = cluster_params(cl, geo, &cp))) return rc;
  if (n_xfers < 0 || n_units < 0) return fail(TPR_EINVAL, "negative sizes");
  if (n_xfers == 0 && !status_mirror) return TPR_OK;
  if (!d_status || (n_xfers > 0 && (!d_xfers || !d_meta || !d_totals)) || (n_units > 0 && !d_work))
    return fail(TPR_EINVAL, "null device buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  bool mirrored = false;
  // small plans: the whole switch in one launch (K31), the records passed as
  // kernel parameters -- needs host records, the TMA engine on local pools
  if (n_xfers > 0 && n_units > 0 && h_xfers && n_xfers <= kK31Xfers && n_units <= k3_fuse_units() &&
      knob(g_k31, "TPR_K31", 1) && g_engine.load() == TPR_ENGINE_BULK &&
      all_local(cp.pool, cl->n_gpus) && host_readable(h_xfers)) {
    const bool timed = k1_events && k1_events[0] && k1_events[1];
    if (timed && (e = cudaEventRecord(static_cast<cudaEvent_t>(k1_events[0]), st)) != cudaSuccess)
      return cuda_fail(e, "tpr_kv_switch K31 start event");
    int32_t tk = 0;
    // a ticket is for a host that spins on it: only switches short enough to
    // spin through (<= 2048 pages, ~0.2 ms); longer ones wait on the stream
    if (ticket && status_mirror && n_units <= 2048) {  // nonzero, distinct from the last few calls
      static std::atomic<int32_t> g_ticket{0};
      tk = g_ticket.fetch_add(1) % 0x3fffffff + 1;
    }
    e = launch_k31(*geo, copy_params(geo), cp, h_xfers, n_xfers, filter_src, n_units, d_totals,
                   d_status, status_mirror, st, cl->n_gpus,
                   any_partial(h_xfers, n_xfers, geo->block_tokens), d_work,
                   (int)knob(g_k31, "TPR_K31", 1), tk);
    if (e == cudaSuccess) {
      if (ticket) *ticket = tk;
      g_k1_last.store(TPR_ENGINE_BULK);
      if (records_async) *records_async = 0;  // the launch copied them into its parameters
      if (timed && (e = cudaEventRecord(static_cast<cudaEvent_t>(k1_events[1]), st)) != cudaSuccess)
        return cuda_fail(e, "tpr_kv_switch K31 end event");
      return TPR_OK;
    }
    if (e != cudaErrorNotSupported) return cuda_fail(e, "tpr_kv_switch K31");
    cudaGetLastError();
  }
  if (n_xfers > 0 && n_units > 0) {
    // records K3 reads: pinned host records in place (zero-copy), else an
    // H2D copy into d_xfers first
    const int32_t* xin = d_xfers;
    if (h_xfers) {
      const int32_t* mapped = device_view(h_xfers);
      if (mapped) {
        xin = mapped;
      } else {
        e = cudaMemcpyAsync(d_xfers, h_xfers, sizeof(int32_t) * TPR_XFER_FIELDS * (size_t)n_xfers,
                            cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "tpr_kv_switch H2D");
      }
    }
    e = launch_k3(*geo, cp, xin, d_xfers, n_xfers, filter_src, d_meta, d_totals, n_units,
                  reinterpret_cast<int4*>(d_work), nullptr, d_status, st, status_mirror, &mirrored);
    if (e != cudaSuccess) return cuda_fail(e, "tpr_kv_switch K3");
    const bool timed = k1_events && k1_events[0] && k1_events[1];
    if (timed && (e = cudaEventRecord(static_cast<cudaEvent_t>(k1_events[0]), st)) != cudaSuccess)
      return cuda_fail(e, "tpr_kv_switch K1 start event");
    e = run_k1(geo, cl->n_gpus, copy_params(geo), cp, reinterpret_cast<const int4*>(d_work),
               n_units, st, pdl_for(n_units) && !timed,
               h_xfers ? any_partial(h_xfers, n_xfers, geo->block_tokens) : true);
    if (e != cudaSuccess) return cuda_fail(e, "tpr_kv_switch K1");
    if (timed && (e = cudaEventRecord(static_cast<cudaEvent_t>(k1_events[1]), st)) != cudaSuccess)
      return cuda_fail(e, "tpr_kv_switch K1 end event");
  } else if (h_xfers && n_xfers > 0) {
    // nothing to allocate or move: the records still land in d_xfers
    e = cudaMemcpyAsync(d_xfers, h_xfers, sizeof(int32_t) * TPR_XFER_FIELDS * (size_t)n_xfers,
                        cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "tpr_kv_switch H2D");
  }
  if (k1_events && k1_events[0] && k1_events[1] && !(n_xfers > 0 && n_units > 0)) {
    // no K1 this time: an empty, still-recorded interval
    cudaEventRecord(static_cast<cudaEvent_t>(k1_events[0]), st);
    cudaEventRecord(static_cast<cudaEvent_t>(k1_events[1]), st);
  }
  if (status_mirror && !mirrored) {
    e = cudaMemcpyAsync(status_mirror, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "tpr_kv_switch status D2H");
  }
  return TPR_OK;
}
}  // namespace tpr

extern "C" {

int tpr_version(void) { return TPR_ABI_VERSION; }

int tpr_set_copy_engine(int32_t engine) {
  if (engine != TPR_ENGINE_VECTOR && engine != TPR_ENGINE_BULK)
    return fail(TPR_EINVAL, "unknown copy engine %d", engine);
  g_engine.store(engine);
  return TPR_OK;
}

int tpr_get_copy_engine(void) { return g_engine.load(); }

int tpr_set_tuning(const char* key, int64_t value) {
  if (!key) return fail(TPR_EINVAL, "null tuning key");
  if (value < 0) return fail(TPR_EINVAL, "tuning value must be >= 0");
  if (!strcmp(key, "k3_fuse_units")) g_fuse.store(value);
  else if (!strcmp(key, "tensor_partial")) g_tensor.store(value > 1 ? 1 : value);
  else if (!strcmp(key, "k31")) g_k31.store(value > 3 ? 3 : value);
  else if (!strcmp(key, "k31_trace")) g_k31_trace.store(value);
  else return fail(TPR_EINVAL, "unknown tuning key '%s'", key);
  return TPR_OK;
}

int64_t tpr_get_tuning(const char* key) {
  if (!key) return -1;
  if (!strcmp(key, "k3_fuse_units")) return tpr::k3_fuse_units();
  if (!strcmp(key, "tensor_partial")) return knob(g_tensor, "TPR_TENSOR_PARTIAL", 1);
  if (!strcmp(key, "k31")) return knob(g_k31, "TPR_K31", 1);
  if (!strcmp(key, "k31_trace")) return g_k31_trace.load();
  if (!strcmp(key, "k1_engine_last")) return g_k1_last.load();
  if (!strcmp(key, "k2_engine_last")) return g_k2_last.load();
  return -1;
}

const char* tpr_last_error(void) { return g_err.c_str(); }

int tpr_device_info(int32_t* sm, int32_t* major, int32_t* minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int a = 0, b = 0, c = 0;
  cudaDeviceGetAttribute(&a, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&b, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&c, cudaDevAttrComputeCapabilityMinor, dev);
  if (sm) *sm = a;
  if (major) *major = b;
  if (minor) *minor = c;
  return TPR_OK;
}

// ---------------------------------------------------------------------------
// Native head planner. Ownership follows KvLayout (migration.py:25-47): rank r
// of a tp-N group owns heads [r*H/N, (r+1)*H/N). Ownership of both layouts is
// piecewise constant between multiples of H/N_old and H/N_new, so the planner
// walks those breakpoints instead of single heads and merges neighbouring
// pieces that share a (src, dst) pair. Pieces whose owner does not change are
// skipped and break runs, as in migration.py:112-133.
// ---------------------------------------------------------------------------
int tpr_plan_heads(int32_t n_req, const int64_t* req_ids, const int64_t* ctx,
                   const int32_t* old_off, const int32_t* old_tp, const int32_t* new_off,
                   const int32_t* new_tp, const int64_t* gpu_ids, int32_t total_heads,
                   int64_t kvb, int64_t capacity, int64_t* out, int64_t* n_out) {
  if (n_req < 0 || total_heads <= 0 || !n_out) return fail(TPR_EINVAL, "bad planner arguments");
  int64_t n = 0;
  for (int32_t i = 0; i < n_req; ++i) {
    const int32_t to = old_tp[i], tn = new_tp[i];
    if (to <= 0 || tn <= 0 || total_heads % to || total_heads % tn)
      return fail(TPR_EINVAL, "request %lld: total_heads=%d not divisible by tp",
                  (long long)req_ids[i], total_heads);
    const int32_t ho = total_heads / to, hn = total_heads / tn;
    const int64_t* go = gpu_ids + old_off[i];
    const int64_t* gn = gpu_ids + new_off[i];
    const int64_t per_head = ctx[i] * kvb;
    bool open = false;
    int64_t run_src = 0, run_dst = 0;
    int32_t run_lo = 0;
    int32_t p = 0;
    while (p <= total_heads) {
      int32_t next;
      bool moving = false;
      int64_t s = 0, d = 0;
      if (p < total_heads) {
        next = std::min((p / ho + 1) * ho, (p / hn + 1) * hn);
        s = go[p / ho];
        d = gn[p / hn];
        moving = s != d;
      } else {
        next = total_heads + 1;
      }
      const bool extends = open && moving && s == run_src && d == run_dst;
      if (open && !extends) {
        if (n >= capacity) return fail(TPR_ECAPACITY, "planner output capacity exhausted");
        int64_t* o = out + n * 6;
        o[0] = run_src;
        o[1] = run_dst;
        o[2] = req_ids[i];
        o[3] = run_lo;
        o[4] = p;
        o[5] = (int64_t)(p - run_lo) * per_head;
        ++n;
        open = false;
      }
      if (moving && !open) {
        open = true;
        run_src = s;
        run_dst = d;
        run_lo = p;
      }
      p = next;
    }
  }
  *n_out = n;
  return TPR_OK;
}

// ---------------------------------------------------------------------------
// K3 / K1 / K2 wrappers
// ---------------------------------------------------------------------------
int tpr_kv_remap(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl, const int32_t* d_xfers,
                 int32_t n_xfers, int32_t filter_src, int64_t* d_meta, int64_t* d_totals,
                 int64_t n_units_hint, int32_t* d_work, int32_t* d_work_ext, int32_t* d_status,
                 void* stream) {
  int rc = check_geometry(geo);
  if (rc) return rc;
  tpr::KvClusterParams cp;
  if ((rc = cluster_params(cl, geo, &cp))) return rc;
  if (n_xfers < 0) return fail(TPR_EINVAL, "n_xfers < 0");
  if (n_xfers == 0) return TPR_OK;
  if (!d_xfers || !d_meta || !d_totals || !d_work || !d_status)
    return fail(TPR_EINVAL, "null device buffer");
  cudaError_t e = tpr::launch_k3(*geo, cp, d_xfers, const_cast<int32_t*>(d_xfers), n_xfers, filter_src, d_meta,
                                 d_totals, n_units_hint, reinterpret_cast<int4*>(d_work),
                                 reinterpret_cast<int4*>(d_work_ext), d_status,
                                 static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_kv_remap launch");
}

int tpr_kv_migrate_ex(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                      const int32_t* d_work, int64_t n_units, int32_t flags, void* stream) {
  int rc = check_geometry(geo);
  if (rc) return rc;
  tpr::KvClusterParams cp;
  if ((rc = cluster_params(cl, geo, &cp))) return rc;
  if (n_units < 0) return fail(TPR_EINVAL, "n_units < 0");
  if (n_units > 0 && !d_work) return fail(TPR_EINVAL, "null work list");
  cudaError_t e = run_k1(geo, cl->n_gpus, copy_params(geo), cp, reinterpret_cast<const int4*>(d_work),
                         n_units, static_cast<cudaStream_t>(stream), tpr::pdl_for(n_units),
                         !(flags & TPR_MIGRATE_FULL_PAGES));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_kv_migrate launch");
}

int tpr_kv_migrate(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl, const int32_t* d_work,
                   int64_t n_units, void* stream) {
  return tpr_kv_migrate_ex(geo, cl, d_work, n_units, 0, stream);
}

int tpr_kv_switch(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl, const int32_t* h_xfers,
                  int32_t* d_xfers, int32_t n_xfers, int32_t filter_src, int64_t* d_meta,
                  int64_t* d_totals, int64_t n_units, int32_t* d_work, int32_t* d_status,
                  void* stream) {
  return tpr::kv_switch_impl(geo, cl, h_xfers, d_xfers, n_xfers, filter_src, d_meta, d_totals,
                             n_units, d_work, d_status, stream, nullptr);
}

int tpr_memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return TPR_OK;
  if (!dst || !src) return fail(TPR_EINVAL, "null pointer");
  cudaError_t e = cudaMemcpyAsync(reinterpret_cast<void*>(dst), src, bytes, cudaMemcpyHostToDevice,
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_memcpy_h2d");
}

int tpr_memcpy_d2h(void* dst, uint64_t src, uint64_t bytes, void* stream) {
  if (bytes == 0) return TPR_OK;
  if (!dst || !src) return fail(TPR_EINVAL, "null pointer");
  cudaError_t e = cudaMemcpyAsync(dst, reinterpret_cast<const void*>(src), bytes,
                                  cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_memcpy_d2h");
}

int tpr_event_record(void* event, void* stream) {
  if (!event) return fail(TPR_EINVAL, "null event");
  cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_event_record");
}

int tpr_copy_prepare(tpr_copy_seg_t* segs, int32_t n, int64_t chunk, int64_t* prefix,
                     int64_t* n_items) {
  if (n < 0 || !prefix || !n_items) return fail(TPR_EINVAL, "bad copy_prepare arguments");
  if (chunk <= 0 || chunk % 16) return fail(TPR_EINVAL, "chunk_bytes must be a positive multiple of 16");
  int64_t total = 0;
  prefix[0] = 0;
  for (int32_t i = 0; i < n; ++i) {
    tpr_copy_seg_t& s = segs[i];
    int64_t items = 0;
    if (s.rows > 0 && s.row_bytes > 0) {
      if (s.rows > 1 && s.src_pitch == s.row_bytes && s.dst_pitch == s.row_bytes) {
        s.row_bytes *= s.rows;
        s.rows = 1;
        s.src_pitch = s.dst_pitch = s.row_bytes;
      }
      if (s.rows == 1) s.src_pitch = s.dst_pitch = s.row_bytes;
      const bool aligned = ((s.src | s.dst) % 16 == 0) && s.row_bytes % 16 == 0 &&
                           s.src_pitch % 16 == 0 && s.dst_pitch % 16 == 0;
      s.flags = aligned ? TPR_SEG_ALIGNED16 : 0;
      if (s.row_bytes <= chunk) {
        const int64_t rpi = chunk / s.row_bytes;
        items = (s.rows + rpi - 1) / rpi;
      } else {
        items = s.rows * ((s.row_bytes + chunk - 1) / chunk);
      }
    } else {
      s.flags = 0;
    }
    total += items;
    prefix[i + 1] = total;
  }
  *n_items = total;
  return TPR_OK;
}

int tpr_weight_reshard(const tpr_copy_seg_t* d_segs, const int64_t* d_prefix, int32_t n_segs,
                       int64_t n_items, int64_t chunk, int64_t* d_claim, void* stream) {
  if (n_segs < 0 || n_items < 0 || chunk <= 0) return fail(TPR_EINVAL, "bad reshard arguments");
  if (n_items == 0) return TPR_OK;
  if (!d_segs || !d_prefix) return fail(TPR_EINVAL, "null segment buffers");
  cudaError_t e = run_k2(d_segs, d_prefix, n_segs, n_items, chunk, d_claim,
                         static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_weight_reshard launch");
}

int tpr_weight_reshard_host(tpr_copy_seg_t* h_buf, int32_t n_segs, int64_t chunk, uint64_t d_buf,
                            uint64_t d_buf_bytes, int64_t* n_items_out, void* stream) {
  if (n_segs < 0 || (n_segs > 0 && (!h_buf || !d_buf))) return fail(TPR_EINVAL, "bad reshard arguments");
  const size_t bytes = tpr_reshard_buffer_bytes(n_segs);
  if (d_buf_bytes < bytes) return fail(TPR_ECAPACITY, "device buffer %llu < %llu bytes",
                                       (unsigned long long)d_buf_bytes, (unsigned long long)bytes);
  int64_t* prefix = reinterpret_cast<int64_t*>(h_buf + n_segs);
  int64_t n_items = 0;
  int rc = tpr_copy_prepare(h_buf, n_segs, chunk, prefix, &n_items);
  if (rc) return rc;
  prefix[n_segs + 1] = 0;  // the dynamic-claim counter, 0 when K2 starts
  if (n_items_out) *n_items_out = n_items;
  if (n_items == 0) return TPR_OK;
  // TMA engine only when every byte K2 touches is this device's HBM
  std::vector<uint64_t> ptrs;
  ptrs.reserve(2 * (size_t)n_segs);
  for (int32_t i = 0; i < n_segs; ++i) {
    ptrs.push_back(h_buf[i].src);
    ptrs.push_back(h_buf[i].dst);
  }
  const bool local = tpr::all_local(ptrs.data(), (int)ptrs.size());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(reinterpret_cast<void*>(d_buf), h_buf, bytes,
                                  cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "tpr_weight_reshard_host H2D");
  const tpr_copy_seg_t* d_segs = reinterpret_cast<const tpr_copy_seg_t*>(d_buf);
  const int64_t* d_prefix = reinterpret_cast<const int64_t*>(d_segs + n_segs);
  e = run_k2(d_segs, d_prefix, n_segs, n_items, chunk, const_cast<int64_t*>(d_prefix) + n_segs + 1,
             st, local);
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_weight_reshard_host launch");
}

size_t tpr_reshard_buffer_bytes(int32_t n_segs) {
  return sizeof(tpr_copy_seg_t) * (size_t)(n_segs > 0 ? n_segs : 0) +
         sizeof(int64_t) * (size_t)((n_segs > 0 ? n_segs : 0) + 2);
}

// ---------------------------------------------------------------------------
// Synthetic data and checks
// ---------------------------------------------------------------------------
int tpr_kv_fill(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl, const int32_t* d_work,
                const int32_t* d_work_ext, int64_t n_units, uint64_t seed, void* stream) {
  int rc = check_geometry(geo);
  if (rc) return rc;
  tpr::KvClusterParams cp;
  if ((rc = cluster_params(cl, geo, &cp))) return rc;
  if (n_units > 0 && (!d_work || !d_work_ext)) return fail(TPR_EINVAL, "null buffer");
  cudaError_t e = tpr::launch_kv_fill(copy_params(geo), cp,
                                      reinterpret_cast<const int4*>(d_work),
                                      reinterpret_cast<const int4*>(d_work_ext), n_units, seed,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_kv_fill launch");
}

int tpr_pool_fill(const tpr_kv_geometry_t* geo, uint64_t pool, int32_t slot, uint64_t seed,
                  void* stream) {
  int rc = check_geometry(geo);
  if (rc) return rc;
  if (!pool) return fail(TPR_EINVAL, "null pool");
  cudaError_t e = tpr::launch_pool_fill(copy_params(geo), geo->n_units,
                                        reinterpret_cast<char*>(pool), slot, seed,
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_pool_fill launch");
}

int tpr_kv_verify(const tpr_kv_geometry_t* geo, uint64_t pool, const int32_t* d_bt,
                  const int32_t* d_ctx, const int32_t* d_owner, int32_t slot, uint64_t seed,
                  int64_t* d_counts, void* stream) {
  int rc = check_geometry(geo);
  if (rc) return rc;
  if (!pool || !d_bt || !d_ctx || !d_owner || !d_counts) return fail(TPR_EINVAL, "null buffer");
  cudaError_t e = tpr::launch_kv_verify(*geo, copy_params(geo), reinterpret_cast<const char*>(pool),
                                        d_bt, d_ctx, d_owner, slot, seed,
                                        reinterpret_cast<unsigned long long*>(d_counts),
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_kv_verify launch");
}

int tpr_matrix_fill(uint64_t buf, int64_t rows, int64_t cols, int64_t pitch, int64_t row0,
                    int64_t col0, int64_t full_cols, uint64_t key, int32_t elem_bytes,
                    void* stream) {
  if (!buf && rows > 0 && cols > 0) return fail(TPR_EINVAL, "null buffer");
  cudaError_t e = tpr::launch_matrix(reinterpret_cast<char*>(buf), rows, cols, pitch, row0, col0,
                                     full_cols, key, elem_bytes, false, nullptr,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_matrix_fill launch");
}

int tpr_matrix_verify(uint64_t buf, int64_t rows, int64_t cols, int64_t pitch, int64_t row0,
                      int64_t col0, int64_t full_cols, uint64_t key, int32_t elem_bytes,
                      int64_t* d_mismatch, void* stream) {
  if ((!buf && rows > 0 && cols > 0) || !d_mismatch) return fail(TPR_EINVAL, "null buffer");
  cudaError_t e = tpr::launch_matrix(reinterpret_cast<char*>(buf), rows, cols, pitch, row0, col0,
                                     full_cols, key, elem_bytes, true,
                                     reinterpret_cast<unsigned long long*>(d_mismatch),
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_matrix_verify launch");
}

// ---------------------------------------------------------------------------
// Peer memory
// ---------------------------------------------------------------------------
int tpr_baseline_copy_pages(const uint64_t* src, const uint64_t* dst, const uint64_t* bytes,
                            int64_t n, int32_t method, void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst || !bytes))) return fail(TPR_EINVAL, "bad page list");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (method == TPR_BASELINE_MEMCPY) {
    for (int64_t i = 0; i < n; ++i) {
      cudaError_t e = cudaMemcpyAsync(reinterpret_cast<void*>(dst[i]),
                                      reinterpret_cast<const void*>(src[i]), bytes[i],
                                      cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
    }
    return TPR_OK;
  }
  return fail(TPR_EINVAL, "unknown baseline method %d", method);
}

int tpr_device_barrier(const uint64_t* peer_flags, int32_t rank, int32_t world, uint64_t epoch,
                       uint64_t timeout_ns, int32_t* d_status, void* stream) {
  if (!peer_flags || world <= 0 || world > TPR_MAX_GPUS || rank < 0 || rank >= world)
    return fail(TPR_EINVAL, "bad barrier arguments (rank %d, world %d)", rank, world);
  cudaError_t e = tpr::launch_barrier(peer_flags, rank, world, epoch, timeout_ns, d_status,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "tpr_device_barrier launch");
}

int tpr_device_alloc(uint64_t bytes, uint64_t* dptr) {
  if (!dptr) return fail(TPR_EINVAL, "null output pointer");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  *dptr = reinterpret_cast<uint64_t>(p);
  return TPR_OK;
}

int tpr_device_free(uint64_t dptr) {
  tpr::forget_ranges();
  cudaError_t e = cudaFree(reinterpret_cast<void*>(dptr));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "cudaFree");
}

int tpr_ipc_get_handle(uint64_t dptr, uint8_t* handle64) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(dptr));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, 64);
  return TPR_OK;
}

int tpr_ipc_open(const uint8_t* handle64, uint64_t* dptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *dptr = reinterpret_cast<uint64_t>(p);
  return TPR_OK;
}

int tpr_ipc_close(uint64_t dptr) {
  tpr::forget_ranges();
  cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<void*>(dptr));
  return e == cudaSuccess ? TPR_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

}  // extern "C"
