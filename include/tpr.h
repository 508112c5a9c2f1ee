/*
 * tpr.h — C ABI of libtpr.so, the B200 (sm_100a) TP-reconfiguration data path.
 *
 * The reference (arxiv 2605.05467 artifact, `tpsim`) exposes this path as a pure
 * Python API in pkg/src/tpsim/migration.py; it has no FFI. Every entry point
 * below is what a binding for that API would call underneath, and each cites the
 * reference function it replaces or executes:
 *
 *   tpr_plan_heads        -> migration.py:101-134 head_transfers (run coalescing)
 *                            and migration.py:168-188 plan_repartition (plan order)
 *   tpr_kv_remap    (K3)  -> migration.py:192-207 apply_plan (placement replay),
 *                            executed on device: block-table remap + free-ring
 *                            allocation by warp-level prefix sums
 *   tpr_kv_migrate  (K1)  -> the Transfer list (migration.py:50-57) executed:
 *                            paged-KV head-shard movement, TMA bulk copies (or
 *                            16-B vectorised loads/stores) straight into the
 *                            destination pool (a peer mapping when the destination
 *                            is another GPU); partial pages as TMA tensor boxes
 *   tpr_weight_reshard (K2)-> migration.py:295-306 weight_memory("sharded", tp)
 *                            volumes realised: fetch only missing shard slices
 *   tpr_kv_switch_layouts -> migration.py:137-189 plan_repartition (or :101-134
 *                            head_transfers) + apply_plan (:192-207) in one call:
 *                            plan, records, capacity, K3 + K1, placement; the hook
 *                            engine.py:571-609 would call per reconfiguration
 *
 * Conventions: every call returns 0 on success and a negative tpr_status code on
 * failure; tpr_last_error() returns a thread-local message. Device pointers are
 * plain uint64 virtual addresses (local, or peer mappings opened with
 * tpr_ipc_open). Every device call is stream-ordered on the caller's
 * cudaStream_t (passed as void*) and launches on the caller's current device.
 * No torch types cross this boundary.
 */
#ifndef TPR_H_
#define TPR_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI 2 (round 2): tpr_switch_tables_t gained ring_head_io / ring_tail_io /
 * start_event and the ticket field; TPR_TOTALS_LEN grew by the small-switch
 * kernel's words; tpr_record_offsets and tpr_event_record are new. */
#define TPR_ABI_VERSION 2
#define TPR_MAX_GPUS 16

enum tpr_status {
  TPR_OK = 0,
  TPR_EINVAL = -1,     /* bad argument                                   */
  TPR_ECUDA = -2,      /* CUDA runtime error                             */
  TPR_ECAPACITY = -3,  /* output buffer too small                        */
  TPR_ENOTFOUND = -4,  /* input outside this fast path (an id outside the */
                       /* caller's tables, a repeated id): use the        */
                       /* caller's general path, which resolves or raises */
};

/* Device-side status bits written by the K3 remap kernel (status word). Each
 * K3 call (tpr_kv_remap, tpr_kv_switch, tpr_kv_switch_layouts) first zeroes
 * the word, so it reports that call only. A page with an error is not touched
 * (its work item has ntok = 0 and K1 skips it); the ring positions the host
 * counts are still written, so ring state stays defined (see tpr_kernels.cu
 * k3_page and oracle/kvmove.c for the exact rules). */
#define TPR_STATUS_WRONG_SOURCE 1  /* head not on src_gpu (migration.py:201-205) */
#define TPR_STATUS_DST_OCCUPIED 2  /* destination block-table slot already set   */
#define TPR_STATUS_OUT_OF_RANGE 8  /* request slot / head / page outside the
                                      block table (context longer than max_blocks) */
#define TPR_STATUS_RING_POISONED 16 /* a free-ring pop returned no valid unit (a
                                      slot an earlier error left poisoned)        */

/* Paged KV pool geometry. One pool unit = one KV head x one page of
 * `block_tokens` tokens x all layers x {K,V}, laid out [layer][kv][token][dim].
 * The pool shape is independent of the TP degree (KvLayout, migration.py:25-47,
 * only changes which GPU owns a head). */
typedef struct tpr_kv_geometry {
  int32_t layers;        /* L                                          */
  int32_t head_dim;      /* D                                          */
  int32_t dtype_bytes;   /* 2 for bf16                                 */
  int32_t block_tokens;  /* tokens per page                            */
  int32_t total_heads;   /* H (KV heads), KvLayout.total_heads         */
  int32_t max_blocks;    /* pages per (request slot, head) table row   */
  int32_t n_req_slots;   /* request slots per block table              */
  int32_t n_units;       /* units per pool == free-ring capacity       */
} tpr_kv_geometry_t;

/* The set of pools a plan touches, indexed by GPU slot (dense 0..n_gpus-1).
 * units[g] is slot g's pool capacity (= its free-ring length; 0 means
 * geometry.n_units). ring_head / ring_tail are monotonically increasing
 * counters owned by the host: the next allocation takes
 * ring[ring_head % units], the next release is stored at ring[ring_tail % units]. */
typedef struct tpr_kv_cluster {
  int32_t n_gpus;
  int32_t _pad;
  uint64_t pool[TPR_MAX_GPUS];        /* uint8 [units][unit_bytes]            */
  uint64_t block_table[TPR_MAX_GPUS]; /* int32 [n_req_slots][H][max_blocks]   */
  uint64_t free_ring[TPR_MAX_GPUS];   /* int32 [units]                        */
  int64_t ring_head[TPR_MAX_GPUS];
  int64_t ring_tail[TPR_MAX_GPUS];
  int64_t units[TPR_MAX_GPUS];
} tpr_kv_cluster_t;

/* One transfer record on device, int32 x 6:
 *   {src_slot, dst_slot, req_slot, head_lo, head_hi (excl.), context_len}
 * src_slot == -1 means "allocate only" (admission of a new request);
 * dst_slot == -1 means "release only" (request finished or evicted).       */
#define TPR_XFER_FIELDS 6

/* Per-transfer scan output of K3 (int64 x 4): {mine_off, alloc_off, rel_off, units} */
#define TPR_META_FIELDS 4

/* totals output of K3 (int64): [0] units processed by this caller,
 * [1+g] units allocated on slot g, [1+TPR_MAX_GPUS+g] units released on g;
 * [TPR_TOTALS_K31_DONE], [TPR_TOTALS_K31_STATUS], [TPR_TOTALS_K31_EPOCH] are
 * scratch words of the fused small-switch kernel. The caller zero-initialises
 * d_totals once; the kernel leaves DONE and STATUS zero between calls and
 * advances EPOCH (it tags the per-page reader counters K31 keeps in d_work). */
#define TPR_TOTALS_K31_DONE (1 + 2 * TPR_MAX_GPUS)
#define TPR_TOTALS_K31_STATUS (2 + 2 * TPR_MAX_GPUS)
#define TPR_TOTALS_K31_EPOCH (3 + 2 * TPR_MAX_GPUS)
/* [TPR_TOTALS_K31_PAR + 2k + parity], k = 0 claim counter, 1 CTAs decided,
 * 2 status bits, 3 CTAs finished: the dynamic small-switch kernel's words,
 * double-buffered by the launch parity the host tracks per d_totals (a launch
 * resets the other parity's words, which the previous launch on the stream
 * used). */
#define TPR_TOTALS_K31_PAR (4 + 2 * TPR_MAX_GPUS)
#define TPR_TOTALS_LEN (12 + 2 * TPR_MAX_GPUS)

/* ---- host utilities -------------------------------------------------- */
/* Copy engine of K1 and K2 (process-wide): TPR_ENGINE_BULK (default) = TMA
 * cp.async.bulk global->shared->global through an mbarrier ring, one issuing
 * thread per CTA; TPR_ENGINE_VECTOR = warp-wide 16-B ld/st. */
#define TPR_ENGINE_VECTOR 0
#define TPR_ENGINE_BULK 1
int tpr_set_copy_engine(int32_t engine);
int tpr_get_copy_engine(void);
/* Launch-path knobs of tpr_kv_switch (process-wide; initial values from the
 * environment variables in brackets):
 *   "k3_fuse_units" [TPR_K3_FUSE_UNITS, 4096]: plans up to this many units
 *                   run as one kernel (K31, below) or, when K31 does not
 *                   apply, K3 as one fused CTA (scan + remap) with K1 launched
 *                   behind it by programmatic dependent launch; 0 = never.
 *                   Larger plans run K3 scan + remap and a normally launched
 *                   K1 whose CTAs claim batches of 4 items dynamically;
 *   "tensor_partial" [TPR_TENSOR_PARTIAL, 1]: K1 / K31 (TMA engine) move
 *                   partial pages as TMA tensor boxes (token x planes)
 *                   instead of one short copy per plane: 0 never, 1 when a
 *                   page of the plan is partial (one K1 kernel either way);
 *   "k31"           [TPR_K31, 1]: a plan of at most k3_fuse_units pages and 96
 *                   transfers (host records, TMA engine, local pools) runs as
 *                   ONE kernel, K31, with the records and their three keyed
 *                   exclusive scans (done on the host) in its parameters and
 *                   two warps per CTA (ring TPR_BULK_K31 [3x32768], two CTAs
 *                   per SM). Two schedules: item shares (every CTA decides
 *                   the pages its equal share of 32 KiB items touches, the
 *                   last reader applies the bookkeeping; epoch-tagged
 *                   per-page counters in d_work, 8 bytes per page: a freshly
 *                   allocated d_work must be zeroed once) and dynamic (each
 *                   page decided once by its owner CTA, a grid-wide wait --
 *                   cooperative launch -- then K1's dynamic item claims).
 *                   0 = off, 1 = item shares below 512 pages and dynamic from
 *                   there, 2 = always dynamic, 3 = always item shares. The
 *                   fused path leaves d_xfers unfilled.
 * Diagnostics: "k31_trace" = the device address of an int64 [grid][8] buffer
 * (0 = off) where every K31 CTA stores globaltimer stamps of its phases
 * (item shares: entry, decisions, copies, bookkeeping; dynamic: entry,
 * decisions, grid-wide wait, copies) and the grid size in [7]
 * (tools/k31_trace.py).
 * tpr_get_tuning returns the current value, -1 for an unknown key. Two
 * read-only keys report the engine the last K1 / K2 launch used
 * ("k1_engine_last", "k2_engine_last": TPR_ENGINE_*, -1 before the first):
 * the TMA engine runs only when every pool (K1) or segment address
 * (tpr_weight_reshard_host) is the launching device's own HBM; peer mappings
 * of another GPU take the vector engine, and no tensor map is ever encoded
 * over a peer mapping.
 * Read once from the environment (TMA engine ring shapes, "<stages>x<bytes>"):
 *   TPR_BULK_K1 [3x65536], TPR_BULK_K2 [3x32768], TPR_BULK_K1_SMALL [3x32768]
 *   for K1s of at most 24 items per SM, TPR_BULK_K31 [3x32768]. */
int tpr_set_tuning(const char* key, int64_t value);
int64_t tpr_get_tuning(const char* key);
int tpr_version(void);
const char* tpr_last_error(void);
int tpr_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---- planner (host) --------------------------------------------------- */
/* Coalesced head-range transfers for n_req requests, in the given request
 * order. Request i moves from group gpu_ids[old_off[i] .. +old_tp[i]) to group
 * gpu_ids[new_off[i] .. +new_tp[i]); rank r of a tp-N group owns heads
 * [r*H/N, (r+1)*H/N). out is int64 [capacity][6] =
 * {src_gpu, dst_gpu, request_id, head_lo, head_hi, bytes}. Replaces
 * migration.py:101-134 (and the per-request loop of migration.py:168-188). */
int tpr_plan_heads(int32_t n_req, const int64_t* req_ids, const int64_t* ctx,
                   const int32_t* old_off, const int32_t* old_tp,
                   const int32_t* new_off, const int32_t* new_tp,
                   const int64_t* gpu_ids, int32_t total_heads, int64_t kvb,
                   int64_t capacity, int64_t* out, int64_t* n_out);

/* plan_repartition (migration.py:137-189) after its GPU-set / head-count
 * checks: layouts are flattened, layout j holding *_count[j] consecutive
 * requests (ids, context lengths) of group gpu_ids[*_goff[j] .. +*_tp[j]).
 * Checks that the new layouts carry exactly the old requests and that no
 * context length changed (the reference's messages, in its order), then plans
 * every new request in new-layout order as tpr_plan_heads. An old request id
 * that repeats returns TPR_ENOTFOUND (the reference's last-one-wins dict
 * semantics stay with the caller's general path). */
int tpr_plan_repartition(int32_t n_old, const int64_t* old_count, const int32_t* old_goff,
                         const int32_t* old_tp, const int64_t* old_req, const int64_t* old_ctx,
                         int32_t n_new, const int64_t* new_count, const int32_t* new_goff,
                         const int32_t* new_tp, const int64_t* new_req, const int64_t* new_ctx,
                         const int64_t* gpu_ids, int32_t total_heads, int64_t kvb,
                         int64_t capacity, int64_t* out, int64_t* n_out);

/* ---- K3: block-table remap + free-ring allocation (device) ------------- */
/* d_xfers: int32 [n][6] transfer records (device). d_meta: int64 [n][4]
 * scratch, d_totals: int64 [TPR_TOTALS_LEN] (device). filter_src = -1
 * processes every transfer (single-process, all pools visible); filter_src =
 * g processes only transfers leaving slot g (one process per GPU, push
 * model) while allocation offsets still follow the whole plan.
 * d_work: int32x4 [n_units + 1] {src_unit, dst_unit, src|dst<<16, ntok}; the
 * extra last entry is K1's claim counter (K3 zeroes it);
 * d_work_ext (nullable): int32x4 {req_slot, head, block, xfer}.
 * n_units_hint: host-computed number of units this caller processes (the
 * expand grid is sized from it). d_status: int32 (device), OR-ed status bits. */
int tpr_kv_remap(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                 const int32_t* d_xfers, int32_t n_xfers, int32_t filter_src,
                 int64_t* d_meta, int64_t* d_totals, int64_t n_units_hint,
                 int32_t* d_work, int32_t* d_work_ext, int32_t* d_status,
                 void* stream);

/* ---- K1: paged-KV head-shard migration (device) ------------------------ */
/* Copies the valid tokens of every work unit from pool[src] to pool[dst]. */
int tpr_kv_migrate(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                   const int32_t* d_work, int64_t n_units, void* stream);
/* tpr_kv_migrate with flags: TPR_MIGRATE_FULL_PAGES = the caller knows every
 * page of the plan is full (all context lengths are multiples of the page
 * size), so K1 launches without encoding the pools' tensor maps (the same
 * kernel; partial pages would then move as row copies). */
#define TPR_MIGRATE_FULL_PAGES 1
int tpr_kv_migrate_ex(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                      const int32_t* d_work, int64_t n_units, int32_t flags, void* stream);

/* ---- switch bookkeeping (host) ----------------------------------------- */
/* Plan rows -> K3 records, per-GPU-slot unit deltas and the plan checks of
 * migration.py:192-207, in one pass over the plan (replaces the per-transfer
 * Python walk between plan_repartition and the device).
 *   plan      int64 [n][6] {src_gpu, dst_gpu, request_id, head_lo, head_hi,
 *             bytes} (the MigrationPlan SoA, tpr_plan_heads' output)
 *   gpu_lut   [gpu id] -> slot, -1 absent;  gpu_ids [slot] -> gpu id
 *   req_lut   [request id] -> request slot, -1 absent
 *   slot_ctx  [request slot] -> context tokens
 *   owner     [request slot][total_heads] -> GPU slot holding the head
 *   validate  0: ids and head ranges only; 1: also bytes == (hi-lo)*ctx*kvb,
 *             no (request, head) moved twice, every head on its src_gpu
 *   records   int32 [n][6] {src slot, dst slot, request slot, lo, hi, ctx}
 *   in_units / out_units [n_slots]: units entering / leaving each slot;
 *   *total_units = units moved.
 * Errors: TPR_ENOTFOUND when an id is outside a table (the caller falls back
 * to its maps, which either resolve it or raise the reference error);
 * TPR_EINVAL with the reference's MigrationError text otherwise. */
int tpr_kv_records(const int64_t* plan, int64_t n, const int64_t* gpu_lut, int64_t gpu_lut_len,
                   const int64_t* gpu_ids, int32_t n_slots, const int64_t* req_lut,
                   int64_t req_lut_len, const int32_t* slot_ctx, const int32_t* owner,
                   int32_t n_req_slots, int32_t total_heads, int32_t block_tokens, int64_t kvb,
                   int32_t validate, int32_t* records, int64_t* in_units, int64_t* out_units,
                   int64_t* total_units);

/* K3's three keyed exclusive scans over n records, on the host (what the
 * one-launch small switch K31 passes in its parameters): meta[t] =
 * {units before t this caller moves (records with src == filter, or all when
 * filter < 0), units before t its destination ring hands out, units before t
 * its source ring takes back, units of t this caller moves} -- the int64 x 4
 * rows K3 writes to d_meta (TPR_META_FIELDS). *n_mine (nullable) = the total
 * this caller moves. */
int tpr_record_offsets(const int32_t* records, int64_t n, int32_t filter, int32_t block_tokens,
                       int64_t* meta, int64_t* n_mine);

/* After a switch is enqueued: owner[req slot][h] = dst slot for every head of
 * every record (apply_plan, migration.py:192-207, on the host placement). */
int tpr_kv_apply_owner(const int32_t* records, int64_t n, int32_t* owner, int32_t total_heads);

/* ---- one call per switch: layouts -> plan -> records -> K3 + K1 -------- */
/* Caller-owned state of one single-device cluster for tpr_kv_switch_layouts.
 * Lookup tables as in tpr_kv_records; plan/records are host outputs (records
 * pinned, so K3 reads them in place); the d_* buffers are device scratch. */
typedef struct tpr_switch_tables {
  const int64_t* gpu_lut;  /* [gpu id] -> slot, -1 absent                     */
  int64_t gpu_lut_len;
  const int64_t* gpu_ids;  /* [slot] -> gpu id                                */
  const int64_t* req_lut;  /* [request id] -> request slot, -1 absent         */
  int64_t req_lut_len;
  const int32_t* slot_ctx; /* [request slot] -> context tokens                */
  int32_t* owner;          /* [request slot][H] -> gpu slot; updated          */
  int64_t kvb;             /* kv_bytes_per_token_per_head                      */
  int32_t validate;        /* as tpr_kv_records                                */
  int32_t mode;            /* TPR_SWITCH_REPARTITION / TPR_SWITCH_HEAD_TRANSFERS */
  int64_t* plan;           /* out: int64 [plan_cap][6], the MigrationPlan SoA  */
  int64_t plan_cap;
  int32_t* records;        /* out: int32 [plan_cap][6] K3 records (pinned)     */
  int64_t in_units[TPR_MAX_GPUS];  /* out: units allocated per slot            */
  int64_t out_units[TPR_MAX_GPUS]; /* out: units released per slot             */
  int64_t n_plan;          /* out: transfers (or the plan_cap needed)          */
  int64_t total_units;     /* out: units moved (or the work_cap needed)        */
  int32_t* d_xfers;        /* device int32 [xfers_cap][6]                      */
  int64_t* d_meta;         /* device int64 [xfers_cap][4]                      */
  int64_t xfers_cap;
  int64_t* d_totals;       /* device int64 [TPR_TOTALS_LEN]                    */
  int32_t* d_work;         /* device int32x4 [work_cap], >= units + 1          */
  int64_t work_cap;
  int32_t* d_status;       /* device int32                                     */
  int64_t plan_bytes;      /* out: the plan's total bytes (MigrationPlan.total_bytes) */
  int32_t* h_status;       /* nullable pinned host int32 [2]: the status word is mirrored
                              there on the stream (fused K3 store or a 4-byte D2H),
                              so a synchronous caller needs no separate read-back */
  void* k1_events[2];      /* nullable cudaEvent_t pair recorded around K1 (timing) */
  int64_t n_records;       /* out: K3 records = the plan's + the release records */
  int32_t records_async;   /* out: 1 when the device reads `records` after the call
                              returns (keep them until the stream passes), 0 when
                              the launch took them (K31: kernel parameters)   */
  int32_t ticket;          /* in: nonzero asks for a completion ticket;
                              out: nonzero when the switch ran as K31 with h_status
                              and at most 2048 pages:
                              the kernel writes it to h_status[1] (h_status must
                              then hold 2 int32) after the status word, once every
                              copy and table write of the switch is done; a
                              synchronous caller may spin on it instead of an
                              event. 0: wait for the stream.                   */
  int64_t* ring_head_io;   /* nullable int64 [n_slots]: advanced by in_units    */
  int64_t* ring_tail_io;   /* nullable int64 [n_slots]: advanced by out_units
                              (both after the switch is enqueued; point them at
                              the cluster's own ring_head / ring_tail to keep
                              the host ring counters without a round trip)    */
  void* start_event;       /* nullable cudaEvent_t recorded on the stream right
                              before the switch's first launch (after planning) */
} tpr_switch_tables_t;

/* tpr_switch_tables_t.mode: the planner of the switch.
 *   TPR_SWITCH_REPARTITION     plan_repartition(old layouts, new layouts)
 *                              (migration.py:137-189): equal GPU sets, the new
 *                              layouts carry exactly the old requests;
 *   TPR_SWITCH_HEAD_TRANSFERS  head_transfers(old, new) (migration.py:101-134):
 *                              one old and one new layout, any GPU sets (the
 *                              engine's prefill->decode handoff, engine.py:571-589). */
#define TPR_SWITCH_REPARTITION 0
#define TPR_SWITCH_HEAD_TRANSFERS 1

/* The host half of a switch, no device work (plan_repartition,
 * migration.py:137-189, then tpr_kv_records and the capacity check).
 * `layouts` packs the old then the new KvLayouts as int64:
 *   n_old, n_new, then per layout: total_heads, tp, group[tp], count,
 *   (request id, context length) x count,
 * optionally followed by a release section: n_release, request id x n_release
 * -- resident requests (not in the layouts) whose pages the same switch frees
 * (destination KV-capacity eviction, engine.py:630-645). Their records (one per
 * run of heads on one slot, dst = -1) follow the plan's in `records`;
 * n_records counts both, n_plan the plan's transfers.
 * Returns TPR_ENOTFOUND when the switch needs the caller's general path: any
 * check the reference reports (GPU sets, head counts, carried requests,
 * context lengths, placement, capacity), a repeated old request id or an id
 * outside the tables; nothing is modified then. TPR_ECAPACITY: plan_cap too
 * small (n_plan = the capacity needed). */
int tpr_switch_prepare(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                       const int64_t* layouts, int64_t layouts_len, tpr_switch_tables_t* t);

/* tpr_switch_prepare, then K3 + K1 on `stream` (tpr_kv_switch over the
 * pinned records) and the host placement update (tpr_kv_apply_owner). The
 * caller commits in_units/out_units to its ring counters and keeps `records`
 * untouched until the stream passes. TPR_ECAPACITY also when the device
 * scratch is too small (n_plan / total_units = what is needed); nothing is
 * launched then. */
int tpr_kv_switch_layouts(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                          const int64_t* layouts, int64_t layouts_len, tpr_switch_tables_t* t,
                          void* stream);

/* ---- K3 + K1 in one call ----------------------------------------------- */
/* The switch fast path: K3 (remap) and K1 (page copy), all on `stream`.
 * h_xfers (may be NULL when d_xfers is already filled): when it is pinned host
 * memory, K3 reads the records in place over PCIe (zero-copy) and copies them
 * into d_xfers; pageable records are first copied H2D. Small plans run K3 as
 * one fused CTA; K3b and K1 use programmatic dependent launch. h_xfers must
 * stay untouched until the stream passes this call. Same arguments as
 * tpr_kv_remap; n_units must be the exact number of units this caller
 * processes. */
int tpr_kv_switch(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                  const int32_t* h_xfers, int32_t* d_xfers, int32_t n_xfers, int32_t filter_src,
                  int64_t* d_meta, int64_t* d_totals, int64_t n_units, int32_t* d_work,
                  int32_t* d_status, void* stream);

/* Stream-ordered host->device copy (pinned source for true asynchrony). */
int tpr_memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes, void* stream);
/* Stream-ordered device->host copy (pinned destination), e.g. the status word. */
int tpr_memcpy_d2h(void* dst, uint64_t src, uint64_t bytes, void* stream);

/* cudaEventRecord(event, stream) for a caller without its own CUDA binding
 * (the executor's end-of-switch event, ~0.5 us through ctypes). */
int tpr_event_record(void* event, void* stream);

/* ---- K2: weight reshard = batched 2-D strided copy (device) ------------ */
typedef struct tpr_copy_seg {
  uint64_t src;       /* device VA (local or peer)        */
  uint64_t dst;       /* device VA (local or peer)        */
  int64_t rows;
  int64_t row_bytes;
  int64_t src_pitch;
  int64_t dst_pitch;
  int64_t flags;      /* set by tpr_copy_prepare          */
  int64_t _pad;
} tpr_copy_seg_t;

/* Host: normalise segments in place (collapse contiguous ones, flag
 * unaligned ones) and fill prefix[n+1] with per-segment work-item counts for
 * the given chunk size. Returns the number of items in *n_items. */
int tpr_copy_prepare(tpr_copy_seg_t* segs, int32_t n, int64_t chunk_bytes,
                     int64_t* prefix, int64_t* n_items);
/* d_claim: optional device int64 that is 0 when the kernel starts (stream
 * order; e.g. uploaded with the segments). With it, CTAs claim batches of
 * items dynamically (no tail when CTAs run at different speeds); NULL keeps
 * the static grid-stride schedule. The kernel leaves it non-zero. */
int tpr_weight_reshard(const tpr_copy_seg_t* d_segs, const int64_t* d_prefix,
                       int32_t n_segs, int64_t n_items, int64_t chunk_bytes,
                       int64_t* d_claim, void* stream);

/* K2 in one call from host segments: `h_buf` (pinned host memory of
 * tpr_reshard_buffer_bytes(n_segs) bytes) holds the n_segs segments; the call
 * normalises them in place (tpr_copy_prepare), appends the item prefix and the
 * claim counter, copies the buffer to `d_buf` on `stream` and launches K2.
 * The copy engine follows the pointers: the TMA engine when every source and
 * destination is the launching device's own HBM, the 16-byte vector engine when
 * any is a peer mapping (another GPU). h_buf must stay untouched until the
 * stream passes this call. *n_items_out (nullable) = work items launched. */
size_t tpr_reshard_buffer_bytes(int32_t n_segs);
int tpr_weight_reshard_host(tpr_copy_seg_t* h_buf, int32_t n_segs, int64_t chunk, uint64_t d_buf,
                            uint64_t d_buf_bytes, int64_t* n_items_out, void* stream);

/* ---- synthetic data + full-size property checks (device) --------------- */
/* Pattern fill of every work unit's valid tokens in its destination pool
 * (typically the work list of an admission remap); the pattern is a function
 * of (seed, req_slot, head, block, offset) only, so it is placement-invariant. */
int tpr_kv_fill(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                const int32_t* d_work, const int32_t* d_work_ext, int64_t n_units,
                uint64_t seed, void* stream);
/* Whole-pool "garbage" fill keyed by (seed, slot, unit, offset). */
int tpr_pool_fill(const tpr_kv_geometry_t* geo, uint64_t pool, int32_t slot,
                  uint64_t seed, void* stream);
/* Checks one GPU's block table + pool: every (req, head, block) that
 * `owner[req][head] == slot` expects is present and carries the pattern, and
 * nothing else is present. d_ctx: int32 [n_req_slots] (-1 = empty slot).
 * d_counts: int64 [3] += {placement errors, word mismatches, units checked}. */
int tpr_kv_verify(const tpr_kv_geometry_t* geo, uint64_t pool, const int32_t* d_bt,
                  const int32_t* d_ctx, const int32_t* d_owner, int32_t slot,
                  uint64_t seed, int64_t* d_counts, void* stream);
/* 2-D weight slice fill/verify: element (i, j) of the buffer is element
 * (row0 + i, col0 + j) of the full matrix identified by key. */
int tpr_matrix_fill(uint64_t buf, int64_t rows, int64_t cols, int64_t pitch_elems,
                    int64_t row0, int64_t col0, int64_t full_cols, uint64_t key,
                    int32_t elem_bytes, void* stream);
int tpr_matrix_verify(uint64_t buf, int64_t rows, int64_t cols, int64_t pitch_elems,
                      int64_t row0, int64_t col0, int64_t full_cols, uint64_t key,
                      int32_t elem_bytes, int64_t* d_mismatch, void* stream);

/* ---- library baselines (measurement only) ------------------------------ */
/* The paper's straw-man ("cudaMemcpyAsync ... issue a
 * separate request for each memory page"): copy n (src, dst, bytes) pages with
 * one cudaMemcpyAsync each (method 0, the only method). Arrays are host memory. */
#define TPR_BASELINE_MEMCPY 0
int tpr_baseline_copy_pages(const uint64_t* src, const uint64_t* dst, const uint64_t* bytes,
                            int64_t n, int32_t method, void* stream);

/* ---- device-side barrier (one process per GPU) ------------------------ */
/* Stream-ordered barrier across `world` ranks without a host collective:
 * rank `rank` stores `epoch` into slot [rank] of every rank's flag array
 * (peer_flags[r] = device VA of rank r's uint64 [world] array, IPC-mapped;
 * release semantics at system scope), then spins until every slot of its own
 * array (peer_flags[rank]) reaches `epoch` (acquire). Epochs must increase.
 * A peer missing for timeout_ns ends the spin and ORs
 * TPR_STATUS_BARRIER_TIMEOUT into *d_status (device int32, nullable). */
#define TPR_STATUS_BARRIER_TIMEOUT 4
int tpr_device_barrier(const uint64_t* peer_flags, int32_t rank, int32_t world, uint64_t epoch,
                       uint64_t timeout_ns, int32_t* d_status, void* stream);

/* ---- peer memory (one process per GPU) -------------------------------- */
/* Whole-allocation device memory (cudaMalloc): the pointer is the allocation
 * base, so its IPC handle maps exactly this buffer in a peer process. */
int tpr_device_alloc(uint64_t bytes, uint64_t* dptr);
int tpr_device_free(uint64_t dptr);
int tpr_ipc_get_handle(uint64_t dptr, uint8_t* handle64);
int tpr_ipc_open(const uint8_t* handle64, uint64_t* dptr);
int tpr_ipc_close(uint64_t dptr);

#ifdef __cplusplus
}
#endif
#endif /* TPR_H_ */
