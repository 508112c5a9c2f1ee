// Host bookkeeping of one switch (include/tpr.h "switch bookkeeping"): plan
// rows -> K3 records + per-slot unit deltas + the plan checks of
// migration.py:192-207, and the host placement update after the enqueue.
// Replaces the per-transfer Python walk of kvcache.PagedKvCluster.records /
// _reserve (which stays as the fallback for ids outside the lookup tables).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "tpr.h"
#include "tpr_internal.h"

namespace {

// Generation-stamped (request slot, head) marks for the "moved twice" check,
// reused across calls so nothing is cleared per switch.
struct Stamps {
  std::vector<uint32_t> mark;
  uint32_t gen = 0;
  uint32_t* begin(size_t n) {
    if (mark.size() < n) mark.assign(n, 0), gen = 0;
    if (++gen == 0) {  // wrapped: clear once every 2^32 calls
      std::fill(mark.begin(), mark.end(), 0u);
      gen = 1;
    }
    return mark.data();
  }
};
thread_local Stamps g_stamps;

}  // namespace

extern "C" {

int tpr_kv_records(const int64_t* plan, int64_t n, const int64_t* gpu_lut, int64_t gpu_lut_len,
                   const int64_t* gpu_ids, int32_t n_slots, const int64_t* req_lut,
                   int64_t req_lut_len, const int32_t* slot_ctx, const int32_t* owner,
                   int32_t n_req_slots, int32_t total_heads, int32_t block_tokens, int64_t kvb,
                   int32_t validate, int32_t* records, int64_t* in_units, int64_t* out_units,
                   int64_t* total_units) {
  using tpr::set_error;
  if (n < 0 || (n > 0 && (!plan || !records)) || !in_units || !out_units || !total_units)
    return set_error(TPR_EINVAL, "bad tpr_kv_records arguments");
  if (n_slots < 1 || n_slots > TPR_MAX_GPUS || total_heads < 1 || block_tokens < 1)
    return set_error(TPR_EINVAL, "bad tpr_kv_records geometry");
  for (int s = 0; s < n_slots; ++s) in_units[s] = out_units[s] = 0;
  *total_units = 0;
  if (!gpu_lut || !req_lut || !slot_ctx || !owner) return set_error(TPR_ENOTFOUND, "no lookup tables");
  // pass 1 -- ids (all sources, all destinations, all requests: the order in
  // which the Python path would raise), the context of each request
  auto slot_of = [&](int64_t id) -> int64_t {
    return (id >= 0 && id < gpu_lut_len) ? gpu_lut[id] : -1;
  };
  for (int c = 0; c < 2; ++c)
    for (int64_t t = 0; t < n; ++t)
      if (slot_of(plan[t * 6 + c]) < 0) return set_error(TPR_ENOTFOUND, "gpu id not in table");
  for (int64_t t = 0; t < n; ++t) {
    const int64_t r = plan[t * 6 + 2];
    const int64_t rs = (r >= 0 && r < req_lut_len) ? req_lut[r] : -1;
    if (rs < 0 || rs >= n_req_slots) return set_error(TPR_ENOTFOUND, "request id not in table");
  }
  for (int64_t t = 0; t < n; ++t) {
    const int64_t lo = plan[t * 6 + 3], hi = plan[t * 6 + 4];
    if (lo < 0 || hi > total_heads || lo >= hi)
      return set_error(TPR_EINVAL, "head range outside [0, total_heads)");
  }
  if (validate) {
    for (int64_t t = 0; t < n; ++t) {
      const int64_t* p = plan + t * 6;
      const int64_t ctx = slot_ctx[req_lut[p[2]]];
      if (p[5] != (p[4] - p[3]) * ctx * kvb)
        return set_error(TPR_EINVAL,
                         "transfer bytes disagree with "
                         "(head_hi-head_lo)*context_len*kv_bytes_per_token_per_head");
    }
    uint32_t* mark = g_stamps.begin((size_t)n_req_slots * total_heads);
    const uint32_t gen = g_stamps.gen;
    for (int64_t t = 0; t < n; ++t) {
      const int64_t* p = plan + t * 6;
      uint32_t* row = mark + (size_t)req_lut[p[2]] * total_heads;
      for (int64_t h = p[3]; h < p[4]; ++h) {
        if (row[h] == gen) return set_error(TPR_EINVAL, "a (request, head) is moved twice in one plan");
        row[h] = gen;
      }
    }
    for (int64_t t = 0; t < n; ++t) {
      const int64_t* p = plan + t * 6;
      const int64_t rs = req_lut[p[2]], src = slot_of(p[0]);
      const int32_t* own = owner + (size_t)rs * total_heads;
      for (int64_t h = p[3]; h < p[4]; ++h) {
        if (own[h] == src) continue;
        if (own[h] >= 0 && own[h] < n_slots)
          return set_error(TPR_EINVAL, "transfer of request %lld head %lld from gpu %lld, but it is on %lld",
                           (long long)p[2], (long long)h, (long long)p[0],
                           (long long)gpu_ids[own[h]]);
        return set_error(TPR_EINVAL, "transfer of request %lld head %lld from gpu %lld, but it is on None",
                         (long long)p[2], (long long)h, (long long)p[0]);
      }
    }
  }
  // pass 2 -- records and unit deltas
  int64_t total = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t* p = plan + t * 6;
    const int32_t s = (int32_t)slot_of(p[0]), d = (int32_t)slot_of(p[1]);
    const int32_t rs = (int32_t)req_lut[p[2]];
    const int32_t ctx = slot_ctx[rs];
    const int64_t units = (p[4] - p[3]) * ((ctx + block_tokens - 1) / block_tokens);
    int32_t* rec = records + t * 6;
    rec[0] = s;
    rec[1] = d;
    rec[2] = rs;
    rec[3] = (int32_t)p[3];
    rec[4] = (int32_t)p[4];
    rec[5] = ctx;
    in_units[d] += units;
    out_units[s] += units;
    total += units;
  }
  *total_units = total;
  return TPR_OK;
}

int tpr_plan_repartition(int32_t n_old, const int64_t* old_count, const int32_t* old_goff,
                         const int32_t* old_tp, const int64_t* old_req, const int64_t* old_ctx,
                         int32_t n_new, const int64_t* new_count, const int32_t* new_goff,
                         const int32_t* new_tp, const int64_t* new_req, const int64_t* new_ctx,
                         const int64_t* gpu_ids, int32_t total_heads, int64_t kvb,
                         int64_t capacity, int64_t* out, int64_t* n_out) {
  using tpr::set_error;
  if (n_old < 0 || n_new < 0 || !n_out || total_heads < 1)
    return set_error(TPR_EINVAL, "bad tpr_plan_repartition arguments");
  thread_local std::vector<std::pair<int64_t, int32_t>> by_id;  // (old request id, old index)
  thread_local std::vector<int32_t> layout_of, match;
  thread_local std::vector<uint8_t> seen;
  thread_local std::vector<int32_t> meta;
  int64_t n_o = 0, n_n = 0;
  for (int32_t j = 0; j < n_old; ++j) n_o += old_count[j];
  for (int32_t j = 0; j < n_new; ++j) n_n += new_count[j];
  by_id.resize(n_o);
  layout_of.resize(n_o);
  for (int32_t j = 0, i = 0; j < n_old; ++j)
    for (int64_t k = 0; k < old_count[j]; ++k, ++i) {
      by_id[i] = {old_req[i], i};
      layout_of[i] = j;
    }
  std::sort(by_id.begin(), by_id.end());
  for (int64_t i = 1; i < n_o; ++i)
    if (by_id[i].first == by_id[i - 1].first)  // last-one-wins dict semantics: general path
      return set_error(TPR_ENOTFOUND, "old request id %lld repeats", (long long)by_id[i].first);
  // carried requests == old requests (migration.py:160-166)
  match.resize(n_n);
  seen.assign(n_o, 0);
  bool carried = n_n == n_o;
  for (int64_t i = 0; carried && i < n_n; ++i) {
    auto it = std::lower_bound(by_id.begin(), by_id.end(), std::make_pair(new_req[i], INT32_MIN));
    if (it == by_id.end() || it->first != new_req[i] || seen[it->second]) {
      carried = false;
      break;
    }
    seen[it->second] = 1;
    match[i] = it->second;
  }
  if (!carried) return set_error(TPR_EINVAL, "new layouts must carry exactly the old requests");
  for (int64_t i = 0; i < n_n; ++i)  // migration.py:172-173, in plan order
    if (old_ctx[match[i]] != new_ctx[i])
      return set_error(TPR_EINVAL, "request %lld: context length changed", (long long)new_req[i]);
  // per-request groups in plan order, then the head planner
  meta.resize(4 * n_n);
  for (int32_t j = 0, i = 0; j < n_new; ++j)
    for (int64_t k = 0; k < new_count[j]; ++k, ++i) {
      const int32_t oj = layout_of[match[i]];
      meta[i] = old_goff[oj];
      meta[n_n + i] = old_tp[oj];
      meta[2 * n_n + i] = new_goff[j];
      meta[3 * n_n + i] = new_tp[j];
    }
  if (n_n == 0) {
    *n_out = 0;
    return TPR_OK;
  }
  return tpr_plan_heads((int32_t)n_n, new_req, new_ctx, meta.data(), meta.data() + n_n,
                        meta.data() + 2 * n_n, meta.data() + 3 * n_n, gpu_ids, total_heads, kvb,
                        capacity, out, n_out);
}

// ---------------------------------------------------------------------------
// One call per switch (tpr_switch_prepare / tpr_kv_switch_layouts): the
// packed layouts are unpacked into the SoA that tpr_plan_repartition takes,
// planned, turned into K3 records and checked against ring capacity. Every
// failure the reference reports maps to TPR_ENOTFOUND: the caller's general
// path (plan_repartition + migrate) then raises it with the reference text.
// ---------------------------------------------------------------------------
int tpr_switch_prepare(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                       const int64_t* L, int64_t len, tpr_switch_tables_t* t) {
  using tpr::set_error;
  if (!geo || !cl || !t || (len > 0 && !L)) return set_error(TPR_EINVAL, "bad tpr_switch_prepare arguments");
  if (len < 2) return set_error(TPR_EINVAL, "layouts blob too short");
  const int32_t H = geo->total_heads;
  const int32_t n_slots = cl->n_gpus;
  if (n_slots < 1 || n_slots > TPR_MAX_GPUS || H < 1) return set_error(TPR_EINVAL, "bad geometry");
  thread_local std::vector<int64_t> cnt, req, ctx, gids, members[2];
  thread_local std::vector<int32_t> goff, tp;
  const int64_t n_old = L[0], n_new = L[1];
  if (n_old < 0 || n_new < 0 || n_old + n_new > INT32_MAX) return set_error(TPR_EINVAL, "bad layout counts");
  cnt.clear(), req.clear(), ctx.clear(), gids.clear(), goff.clear(), tp.clear();
  members[0].clear(), members[1].clear();
  int64_t pos = 2, n_old_req = 0;
  for (int64_t j = 0; j < n_old + n_new; ++j) {
    if (pos + 2 > len) return set_error(TPR_EINVAL, "layouts blob truncated");
    const int64_t h = L[pos++], k = L[pos++];
    if (h != H) return set_error(TPR_ENOTFOUND, "layout head count differs from the pools");
    if (k < 1 || pos + k + 1 > len) return set_error(TPR_EINVAL, "layouts blob truncated");
    goff.push_back((int32_t)gids.size());
    tp.push_back((int32_t)k);
    for (int64_t r = 0; r < k; ++r) {
      gids.push_back(L[pos]);
      members[j < n_old ? 0 : 1].push_back(L[pos]);
      ++pos;
    }
    const int64_t c = L[pos++];
    if (c < 0 || pos + 2 * c > len) return set_error(TPR_EINVAL, "layouts blob truncated");
    cnt.push_back(c);
    for (int64_t i = 0; i < c; ++i) {
      req.push_back(L[pos++]);
      ctx.push_back(L[pos++]);
    }
    if (j < n_old) n_old_req += c;
  }
  // optional release section: n_release, request ids (evicted requests whose
  // pages are freed in the same switch, engine.py:630-645)
  thread_local std::vector<int64_t> rel;
  rel.clear();
  if (pos < len) {
    const int64_t n_rel = L[pos++];
    if (n_rel < 0 || pos + n_rel != len) return set_error(TPR_EINVAL, "bad release section");
    rel.assign(L + pos, L + pos + n_rel);
    pos += n_rel;
  }
  if (pos != len) return set_error(TPR_EINVAL, "layouts blob has trailing data");
  for (auto& m : members) {  // "GPU sets differ" (migration.py:150-155)
    std::sort(m.begin(), m.end());
    m.erase(std::unique(m.begin(), m.end()), m.end());
  }
  const bool heads_mode = t->mode == TPR_SWITCH_HEAD_TRANSFERS;
  if (heads_mode && (n_old != 1 || n_new != 1))
    return set_error(TPR_EINVAL, "head_transfers mode takes one old and one new layout");
  if (!heads_mode && members[0] != members[1])  // plan_repartition only (migration.py:150-155)
    return set_error(TPR_ENOTFOUND, "GPU sets differ");
  const int64_t n_plan_req = heads_mode ? n_old_req : (int64_t)req.size() - n_old_req;
  const int64_t need = (std::max<int64_t>(n_plan_req, 1) + (int64_t)rel.size()) * H;
  if (!t->plan || !t->records || t->plan_cap < need) {
    t->n_plan = need;
    return set_error(TPR_ECAPACITY, "plan capacity %lld < %lld", (long long)t->plan_cap,
                     (long long)need);
  }
  int64_t n = 0;
  int rc;
  if (heads_mode) {
    // head_transfers(old, new) (migration.py:101-134): the old layout's
    // requests in order, from its group to the new group (any GPU sets)
    thread_local std::vector<int32_t> meta;
    meta.resize(4 * (size_t)n_old_req);
    for (int64_t i = 0; i < n_old_req; ++i) {
      meta[i] = goff[0];
      meta[n_old_req + i] = tp[0];
      meta[2 * n_old_req + i] = goff[1];
      meta[3 * n_old_req + i] = tp[1];
    }
    rc = n_old_req == 0 ? TPR_OK
                        : tpr_plan_heads((int32_t)n_old_req, req.data(), ctx.data(), meta.data(),
                                         meta.data() + n_old_req, meta.data() + 2 * n_old_req,
                                         meta.data() + 3 * n_old_req, gids.data(), H, t->kvb,
                                         t->plan_cap, t->plan, &n);
  } else {
    rc = tpr_plan_repartition(
        (int32_t)n_old, cnt.data(), goff.data(), tp.data(), req.data(), ctx.data(), (int32_t)n_new,
        cnt.data() + n_old, goff.data() + n_old, tp.data() + n_old, req.data() + n_old_req,
        ctx.data() + n_old_req, gids.data(), H, t->kvb, t->plan_cap, t->plan, &n);
  }
  if (rc == TPR_ECAPACITY) {
    t->n_plan = need;
    return rc;
  }
  if (rc != TPR_OK) return set_error(TPR_ENOTFOUND, "plan needs the general path");
  t->n_plan = n;
  int64_t plan_bytes = 0;
  for (int64_t i = 0; i < n; ++i) plan_bytes += t->plan[i * 6 + 5];
  t->plan_bytes = plan_bytes;
  rc = tpr_kv_records(t->plan, n, t->gpu_lut, t->gpu_lut_len, t->gpu_ids, n_slots, t->req_lut,
                      t->req_lut_len, t->slot_ctx, t->owner, geo->n_req_slots, H,
                      geo->block_tokens, t->kvb, t->validate, t->records, t->in_units,
                      t->out_units, &t->total_units);
  if (rc != TPR_OK) return set_error(TPR_ENOTFOUND, "records need the general path");
  // release records after the plan's: one per run of heads on the same slot
  // (dst = -1), in the order kvcache.release builds them
  int64_t n_rec = n;
  for (const int64_t rid : rel) {
    const int64_t rs = (rid >= 0 && rid < t->req_lut_len) ? t->req_lut[rid] : -1;
    if (rs < 0 || rs >= geo->n_req_slots) return set_error(TPR_ENOTFOUND, "released request not in table");
    const int32_t* own = t->owner + (size_t)rs * H;
    const int32_t ctx = t->slot_ctx[rs];
    const int64_t nblk = ctx > 0 ? (ctx + geo->block_tokens - 1) / geo->block_tokens : 0;
    for (int32_t h = 0; h < H;) {
      int32_t e = h;
      while (e < H && own[e] == own[h]) ++e;
      if (own[h] < 0 || own[h] >= n_slots) return set_error(TPR_ENOTFOUND, "released request not placed");
      int32_t* r = t->records + n_rec * 6;
      r[0] = own[h];
      r[1] = -1;
      r[2] = (int32_t)rs;
      r[3] = h;
      r[4] = e;
      r[5] = ctx;
      t->out_units[own[h]] += (e - h) * nblk;
      t->total_units += (e - h) * nblk;
      ++n_rec;
      h = e;
    }
  }
  t->n_records = n_rec;
  for (int s = 0; s < n_slots; ++s)  // capacity (kvcache._check_capacity)
    if (t->in_units[s] > cl->ring_tail[s] - cl->ring_head[s])
      return set_error(TPR_ENOTFOUND, "slot %d out of KV units", s);
  return TPR_OK;
}

int tpr_kv_switch_layouts(const tpr_kv_geometry_t* geo, const tpr_kv_cluster_t* cl,
                          const int64_t* L, int64_t len, tpr_switch_tables_t* t, void* stream) {
  int rc = tpr_switch_prepare(geo, cl, L, len, t);
  if (rc != TPR_OK) return rc;
  const int64_t n = t->n_records, units = t->total_units;  // plan + release records
  if (n > 0 && (n > t->xfers_cap || units + 1 > t->work_cap || !t->d_xfers || !t->d_meta ||
                !t->d_totals || !t->d_status || (units > 0 && !t->d_work)))
    return tpr::set_error(TPR_ECAPACITY, "device scratch too small: %lld transfers, %lld units",
                          (long long)n, (long long)units);
  t->records_async = 0;
  const bool want_ticket = t->ticket != 0;  // in: the caller will spin on a ticket
  t->ticket = 0;
  if (t->start_event) {  // the switch's device interval starts at its first launch
    cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(t->start_event),
                                    static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return tpr::set_error(TPR_ECUDA, "start event: %s", cudaGetErrorString(e));
  }
  if (n == 0 && !t->h_status) return TPR_OK;
  rc = tpr::kv_switch_impl(geo, cl, t->records, t->d_xfers, (int32_t)n, -1, t->d_meta,
                           t->d_totals, units, t->d_work, t->d_status, stream, t->h_status,
                           t->k1_events, &t->records_async, want_ticket ? &t->ticket : nullptr);
  if (rc != TPR_OK) return rc;
  if (n == 0) return TPR_OK;
  for (int32_t s = 0; s < cl->n_gpus; ++s) {  // the host ring counters
    if (t->ring_head_io) t->ring_head_io[s] += t->in_units[s];
    if (t->ring_tail_io) t->ring_tail_io[s] += t->out_units[s];
  }
  return tpr_kv_apply_owner(t->records, n, t->owner, geo->total_heads);
}

int tpr_record_offsets(const int32_t* records, int64_t n, int32_t filter, int32_t block_tokens,
                       int64_t* meta, int64_t* n_mine) {
  if (n < 0 || (n > 0 && (!records || !meta)) || block_tokens < 1)
    return tpr::set_error(TPR_EINVAL, "bad tpr_record_offsets arguments");
  int64_t mine = 0, in_u[TPR_MAX_GPUS] = {}, out_u[TPR_MAX_GPUS] = {};
  for (int64_t t = 0; t < n; ++t) {
    const int32_t* r = records + t * TPR_XFER_FIELDS;
    const int64_t nblk = r[5] > 0 ? (r[5] + block_tokens - 1) / block_tokens : 0;
    const int64_t u = (int64_t)(r[4] - r[3]) * nblk;
    const bool has_dst = r[1] >= 0 && r[1] < TPR_MAX_GPUS, has_src = r[0] >= 0 && r[0] < TPR_MAX_GPUS;
    const int64_t m = (filter < 0 || r[0] == filter) ? u : 0;
    int64_t* o = meta + t * TPR_META_FIELDS;
    o[0] = mine;
    o[1] = has_dst ? in_u[r[1]] : 0;
    o[2] = has_src ? out_u[r[0]] : 0;
    o[3] = m;
    mine += m;
    if (has_dst) in_u[r[1]] += u;
    if (has_src) out_u[r[0]] += u;
  }
  if (n_mine) *n_mine = mine;
  return TPR_OK;
}

int tpr_kv_apply_owner(const int32_t* records, int64_t n, int32_t* owner, int32_t total_heads) {
  if (n < 0 || (n > 0 && (!records || !owner)) || total_heads < 1)
    return tpr::set_error(TPR_EINVAL, "bad tpr_kv_apply_owner arguments");
  for (int64_t t = 0; t < n; ++t) {
    const int32_t* r = records + t * 6;
    int32_t* row = owner + (size_t)r[2] * total_heads;
    for (int32_t h = r[3]; h < r[4]; ++h) row[h] = r[1];
  }
  return TPR_OK;
}

}  // extern "C"
