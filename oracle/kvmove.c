/*
 * ORACLE -- test infrastructure only. Linked by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg; never by the product.
 *
 * CPU restatement of executing a KV migration plan on paged pools. The
 * reference has no KV memory (it prices plans, pkg/src/tpsim/migration.py:
 * 221-292), so the byte level is defined by the placement contract it does
 * pin: each transfer (src, dst, request, head_lo, head_hi) moves exactly the
 * heads [head_lo, head_hi) of that request from src to dst
 * (migration.py:50-57, 128-130), replayed in plan order (apply_plan,
 * migration.py:192-207). The paged layout, block tables and free rings are
 * ours; this file restates them sequentially:
 *
 *   for t in plan order, for h in [lo, hi), for b in pages of the request:
 *       u  = block_table[src][req][h][b]          (must be >= 0: "on src")
 *       block_table[src][req][h][b] = -1; ring[src][tail++] = u
 *       v  = ring[dst][head++];  block_table[dst][req][h][b] = v
 *       copy the valid tokens of page u (pool src) to page v (pool dst)
 *
 * The copies are independent once the mapping is known and are spread over
 * threads (OpenMP) for the CPU baseline.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int32_t layers, head_dim, dtype_bytes, block_tokens, total_heads, max_blocks, n_req_slots, n_units;
} oracle_geo;

typedef struct {
  int32_t su, du, src, dst, ntok;
} page_move;

/* Returns number of page moves, or -1 on allocation failure. status |= 1 for
 * a head not on src, |= 2 for an occupied destination entry, |= 8 for a page
 * outside the block table, |= 16 for a poisoned free-ring slot (the
 * TPR_STATUS_* bits of include/tpr.h). pools == NULL replays block tables,
 * free rings and ring counters only (no page bytes). */
int64_t oracle_kv_migrate(const oracle_geo* g, uint8_t** pools, int32_t** tables, int32_t** rings,
                          const int64_t* ring_len, int64_t* ring_head, int64_t* ring_tail,
                          const int64_t* xf, int64_t n, int32_t n_threads, int32_t* status) {
  const int64_t H = g->total_heads, MB = g->max_blocks, B = g->block_tokens;
  const int64_t tok = (int64_t)g->head_dim * g->dtype_bytes;
  const int64_t plane = B * tok, unit = plane * 2 * g->layers;
  int64_t total = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t ctx = xf[t * 6 + 5];
    total += (xf[t * 6 + 4] - xf[t * 6 + 3]) * ((ctx + B - 1) / B);
  }
  page_move* mv = (page_move*)malloc(sizeof(page_move) * (size_t)(total > 0 ? total : 1));
  if (!mv) return -1;
  int64_t k = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t* r = xf + t * 6;
    const int32_t src = (int32_t)r[0], dst = (int32_t)r[1];
    const int64_t req = r[2], ctx = r[5];
    const int64_t pages = (ctx + B - 1) / B;
    for (int64_t h = r[3]; h < r[4]; ++h) {
      for (int64_t b = 0; b < pages; ++b) {
        /* A page with an error is not touched (K1 skips it); the ring positions
         * are still consumed: a missing source is pushed as -1 (a poisoned
         * slot), a destination unit that cannot be placed leaks. */
        const int in_range = h >= 0 && h < H && b < MB && req >= 0 && req < g->n_req_slots;
        const int64_t idx = (req * H + h) * MB + b;
        int32_t su = -1;
        if (!in_range) *status |= 8;
        if (src >= 0) {
          if (in_range) {
            su = tables[src][idx];
            if (su < 0 || su >= ring_len[src]) {
              *status |= 1;
              su = -1;
            }
            tables[src][idx] = -1;
          }
          rings[src][ring_tail[src]++ % ring_len[src]] = su;
        }
        int32_t du = -1;
        if (dst >= 0) { /* dst < 0: release only */
          const int32_t v = rings[dst][ring_head[dst]++ % ring_len[dst]];
          if (v < 0 || v >= ring_len[dst]) {
            *status |= 16;
          } else if (!in_range) {
            /* leaked */
          } else if (tables[dst][idx] >= 0) {
            *status |= 2;
          } else if (!(src >= 0 && su < 0)) {
            tables[dst][idx] = v;
            du = v;
          }
        }
        mv[k].su = su;
        mv[k].du = du;
        mv[k].src = src;
        mv[k].dst = dst;
        mv[k].ntok = (int32_t)((b == pages - 1) ? ctx - b * B : B);
        ++k;
      }
    }
  }
  if (!pools) { /* tables-and-rings-only replay (full-size parity of K3) */
    free(mv);
    return total;
  }
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t i = 0; i < total; ++i) {
    const page_move m = mv[i];
    if (m.su < 0 || m.du < 0) continue;
    const uint8_t* s = pools[m.src] + (int64_t)m.su * unit;
    uint8_t* d = pools[m.dst] + (int64_t)m.du * unit;
    const int64_t nb = m.ntok * tok;
    if (nb == plane) {
      memcpy(d, s, (size_t)unit);
    } else {
      for (int32_t p = 0; p < 2 * g->layers; ++p) memcpy(d + p * plane, s + p * plane, (size_t)nb);
    }
  }
  free(mv);
  return total;
}

/* Threaded 2-D copy used by the CPU baseline for weight slices:
 * block i = rows[i] x row_bytes[i] from src[i] (pitch sp[i]) to dst[i]
 * (pitch dp[i]). Work is cut into <= 1 MiB pieces spread over threads. */
void oracle_copy_blocks(int64_t n, uint8_t* const* dst, const uint8_t* const* src,
                        const int64_t* rows, const int64_t* row_bytes, const int64_t* sp,
                        const int64_t* dp, int32_t n_threads) {
  const int64_t piece = 1 << 20;
  int64_t* first = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!first) return;
  first[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t per_row = (row_bytes[i] + piece - 1) / piece;
    first[i + 1] = first[i] + rows[i] * per_row;
  }
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t task = 0; task < first[n]; ++task) {
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) / 2;
      if (first[mid] <= task) lo = mid; else hi = mid;
    }
    const int64_t per_row = (row_bytes[lo] + piece - 1) / piece;
    const int64_t local = task - first[lo];
    const int64_t r = local / per_row, off = (local % per_row) * piece;
    const int64_t nb = row_bytes[lo] - off < piece ? row_bytes[lo] - off : piece;
    memcpy(dst[lo] + r * dp[lo] + off, src[lo] + r * sp[lo] + off, (size_t)nb);
  }
  free(first);
}

int32_t oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Threaded first touch of a host buffer (the CPU baseline's pools and arenas
 * are page-faulted here, outside its timed region). */
void oracle_fill(uint8_t* p, int64_t n, uint8_t v, int32_t n_threads) {
  const int64_t piece = 1 << 22;
  const int64_t tasks = (n + piece - 1) / piece;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t t = 0; t < tasks; ++t) {
    const int64_t off = t * piece;
    memset(p + off, v, (size_t)(n - off < piece ? n - off : piece));
  }
}
