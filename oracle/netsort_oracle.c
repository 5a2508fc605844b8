/*
 * netsort_oracle.c — plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see netsort_oracle.h).  The product never links
 * this file.  Paths in citations are relative to /root/reference/proj.
 */
#include "netsort_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- input generation ------------------------------------------------- */

/* SplitMix64::next — include/netsort/datagen.hpp:33-38 */
uint64_t oracle_splitmix64_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* generate — src/datagen.cpp:18-50, written once for both widths. */
#define GEN_BODY(T, RANDOM_EXPR)                                              \
  if (kind == 2 && !(p >= 0.0 && p <= 1.0)) return -1;                       \
  if (kind == 0) {                                                           \
    uint64_t s = seed;                                                       \
    for (size_t i = 0; i < n; ++i) {                                         \
      uint64_t r = oracle_splitmix64_next(&s);                               \
      out[i] = (T)(RANDOM_EXPR);                                             \
    }                                                                        \
    return 0;                                                                \
  }                                                                          \
  for (size_t i = 0; i < n; ++i) out[i] = (T)i;                              \
  if (kind == 2) {                                                           \
    size_t swaps = (size_t)(p * (double)n);                                  \
    if (swaps == 0 && n >= 2 && p > 0.0) swaps = 1;                          \
    uint64_t s = seed;                                                       \
    for (size_t k = 0; k < swaps; ++k) {                                     \
      size_t i = (size_t)(oracle_splitmix64_next(&s) % n);                   \
      size_t j = (size_t)(oracle_splitmix64_next(&s) % n);                   \
      T t = out[i];                                                          \
      out[i] = out[j];                                                       \
      out[j] = t;                                                            \
    }                                                                        \
  }                                                                          \
  return 0;

int oracle_generate_i32(int kind, size_t n, uint64_t seed, double p, int32_t* out) {
  GEN_BODY(int32_t, r >> 33)
}

int oracle_generate_i64(int kind, size_t n, uint64_t seed, double p, int64_t* out) {
  GEN_BODY(int64_t, r)
}

size_t oracle_generate_batch_i32(size_t num_arrays, uint64_t seed, uint32_t* offsets,
                                 int32_t* keys) {
  uint64_t ls = seed;
  size_t total = 0;
  for (size_t a = 0; a < num_arrays; ++a) {
    if (offsets) offsets[a] = (uint32_t)total;
    total += 3 + (size_t)(oracle_splitmix64_next(&ls) % 6);
  }
  if (offsets) offsets[num_arrays] = (uint32_t)total;
  if (keys) {
    uint64_t ks = seed ^ 0x5bd1e995ull;
    for (size_t i = 0; i < total; ++i) keys[i] = (int32_t)(oracle_splitmix64_next(&ks) >> 33);
  }
  return total;
}

/* ---- networks ---------------------------------------------------------- */

/* Optimal-size comparator lists, widths 2..8 (sizes 1,3,5,9,12,16,19 as in
 * include/netsort/networks.hpp:49-72).  Any zero-one-complete network of the
 * same width yields the identical output; tests/test_oracle.py re-verifies
 * these exhaustively. */
static const uint8_t kW2[][2] = {{0, 1}};
static const uint8_t kW3[][2] = {{1, 2}, {0, 2}, {0, 1}};
static const uint8_t kW4[][2] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {1, 2}};
static const uint8_t kW5[][2] = {{0, 1}, {3, 4}, {2, 4}, {2, 3}, {0, 3},
                                 {0, 2}, {1, 4}, {1, 3}, {1, 2}};
static const uint8_t kW6[][2] = {{1, 2}, {4, 5}, {0, 2}, {3, 5}, {0, 1}, {3, 4},
                                 {2, 5}, {0, 3}, {1, 4}, {2, 4}, {1, 3}, {2, 3}};
static const uint8_t kW7[][2] = {{1, 2}, {3, 4}, {5, 6}, {0, 2}, {3, 5}, {4, 6},
                                 {0, 1}, {4, 5}, {2, 6}, {0, 4}, {1, 5}, {0, 3},
                                 {2, 5}, {1, 3}, {2, 4}, {2, 3}};
static const uint8_t kW8[][2] = {{0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6},
                                 {3, 7}, {0, 1}, {2, 3}, {4, 5}, {6, 7}, {2, 4}, {3, 5},
                                 {1, 4}, {3, 6}, {1, 2}, {3, 4}, {5, 6}};

static const uint8_t (*net_table(int w, int* count))[2] {
  switch (w) {
    case 2: *count = 1; return kW2;
    case 3: *count = 3; return kW3;
    case 4: *count = 5; return kW4;
    case 5: *count = 9; return kW5;
    case 6: *count = 12; return kW6;
    case 7: *count = 16; return kW7;
    case 8: *count = 19; return kW8;
    default: *count = -1; return NULL;
  }
}

int oracle_network(int width, uint8_t* pairs, int cap) {
  int count;
  const uint8_t(*t)[2] = net_table(width, &count);
  if (!t) return -1;
  for (int i = 0; i < count && i < cap; ++i) {
    pairs[2 * i] = t[i][0];
    pairs[2 * i + 1] = t[i][1];
  }
  return count;
}

/* base_case_applies — config.hpp:30-36 (fixed widths first, then varsort) */
int oracle_base_case_applies(int64_t size, uint32_t width_mask, int varsort_max) {
  if (size >= 2 && size <= 8 && ((width_mask >> size) & 1u)) return 1;
  return varsort_max != 0 && size >= 2 && size <= varsort_max;
}

static inline void st_depth(oracle_stats* s, int d) {
  if (s && d > s->max_depth) s->max_depth = d;
}

#define CAT2_(a, b) a##b
#define CAT_(a, b) CAT2_(a, b)

#define KEY int32_t
#define NAME(x) CAT_(x, _i32)
#include "netsort_oracle_sort.inc"
#undef KEY
#undef NAME

#define KEY int64_t
#define NAME(x) CAT_(x, _i64)
#include "netsort_oracle_sort.inc"
#undef KEY
#undef NAME

/* ---- stable key/payload merge sort (classical recursion) ---------------- */

static void merge_runs_pairs(int32_t* k, uint32_t* v, int64_t left, int64_t mid, int64_t right,
                             int32_t* sk, uint32_t* sv) {
  const int64_t left_len = mid - left + 1;
  memcpy(sk, k + left, (size_t)left_len * sizeof(int32_t));
  memcpy(sv, v + left, (size_t)left_len * sizeof(uint32_t));
  int64_t i = 0, j = mid + 1, out = left;
  while (i < left_len && j <= right) {
    if (k[j] < sk[i]) { k[out] = k[j]; v[out++] = v[j++]; }
    else { k[out] = sk[i]; v[out++] = sv[i++]; }
  }
  while (i < left_len) { k[out] = sk[i]; v[out++] = sv[i++]; }
}

static void ms_pairs_rec(int32_t* k, uint32_t* v, int64_t left, int64_t right, int32_t* sk,
                         uint32_t* sv) {
  if (left >= right) return;
  const int64_t mid = left + (right - left) / 2;
  ms_pairs_rec(k, v, left, mid, sk, sv);
  ms_pairs_rec(k, v, mid + 1, right, sk, sv);
  merge_runs_pairs(k, v, left, mid, right, sk, sv);
}

void oracle_stable_sort_pairs_i32(int32_t* keys, uint32_t* vals, int64_t n) {
  if (n < 2) return;
  int32_t* sk = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  uint32_t* sv = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  ms_pairs_rec(keys, vals, 0, n - 1, sk, sv);
  free(sk);
  free(sv);
}

/* ---- batch helpers ----------------------------------------------------- */

void oracle_sort_small_batch_i32(int32_t* keys, const uint32_t* offsets, size_t num_arrays) {
  for (size_t i = 0; i < num_arrays; ++i) {
    const int len = (int)(offsets[i + 1] - offsets[i]);
    oracle_sort_small_i32(keys + offsets[i], len);
  }
}

void oracle_segmented_quick_sort_i32(int32_t* keys, size_t num_segments, size_t seg_len,
                                     uint32_t mask, int vs) {
  for (size_t s = 0; s < num_segments; ++s)
    oracle_quick_sort_i32(keys + s * seg_len, 0, (int64_t)seg_len - 1, mask, vs, NULL);
}

/* ---- digest ------------------------------------------------------------ */

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_multiset_digest_i32(const int32_t* keys, size_t n, uint64_t out[2]) {
  uint64_t s = 0, x = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t m = mix64((uint64_t)(uint32_t)keys[i] + 0x9E3779B97F4A7C15ull);
    s += m;
    x ^= m;
  }
  out[0] = s;
  out[1] = x;
}

void oracle_multiset_digest_i64(const int64_t* keys, size_t n, uint64_t out[2]) {
  uint64_t s = 0, x = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t m = mix64((uint64_t)keys[i] + 0x9E3779B97F4A7C15ull);
    s += m;
    x ^= m;
  }
  out[0] = s;
  out[1] = x;
}
