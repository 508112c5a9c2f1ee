// Shared definitions for libtpr: synthetic-data pattern (host + device) and
// small device helpers. The pattern is mirrored in numpy by
// paper_2605_05467_b200/pattern.py; tests pin the two against each other.
#pragma once

#include <stdint.h>
#include "tpr.h"

#if defined(__CUDACC__)
#define TPR_HD __host__ __device__ __forceinline__
#else
#define TPR_HD inline
#endif

// splitmix64 finaliser (Steele et al.): a bijective 64-bit mix.
TPR_HD uint64_t tpr_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Key of one logical KV page: (request slot, kv head, page index). The key
// does not depend on which GPU or pool unit holds the page, so the content of
// a page is invariant under migration.
TPR_HD uint64_t tpr_page_key(uint64_t seed, uint32_t req_slot, uint32_t head,
                             uint32_t block) {
  const uint64_t id = ((uint64_t)req_slot << 40) ^ ((uint64_t)head << 24) ^ (uint64_t)block;
  return tpr_splitmix64(seed ^ tpr_splitmix64(id));
}

// Key of a raw pool unit (initial "garbage" content of free units).
TPR_HD uint64_t tpr_unit_key(uint64_t seed, uint32_t slot, uint32_t unit) {
  const uint64_t id = ((uint64_t)slot << 48) ^ (uint64_t)unit ^ 0x5A5A000000000000ull;
  return tpr_splitmix64(seed ^ tpr_splitmix64(id));
}

// 32-bit word `w` (byte offset 4*w inside the page/unit) of a keyed page.
TPR_HD uint32_t tpr_word(uint64_t key, uint64_t w) {
  return (uint32_t)(tpr_splitmix64(key + w) >> 16);
}

// Element (row, col) of a full weight matrix identified by key; truncated to
// the element width by the caller.
TPR_HD uint64_t tpr_matrix_elem(uint64_t key, uint64_t row, uint64_t col,
                                uint64_t full_cols) {
  return tpr_splitmix64(key + row * full_cols + col) >> 24;
}

// Flags of tpr_copy_seg_t.flags (set by tpr_copy_prepare).
#define TPR_SEG_ALIGNED16 1ll

#if defined(__CUDACC__)
// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may become resident while its
// predecessor on the stream is still running; griddepcontrol.wait blocks until
// that predecessor has completed and its memory is visible (a no-op after a
// normal launch). launch_dependents lets the dependent grid start early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif
