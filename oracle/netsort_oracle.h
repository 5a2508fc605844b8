/*
 * netsort_oracle.h — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2503_05934_b200/,
 * include/) links or calls this.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker or the CPU baseline, never as the thing measured for the GPU.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - against the reference's own golden vectors (SplitMix64 KATs and frozen
 *     nearly-sorted outputs from proj/tests/test_datagen.cpp:25-35, 79-91);
 *   - against the reference compiled from /root/reference (oracle/_ref), whose
 *     outputs are frozen as digests under tests/golden/ by
 *     tests/golden/make_golden.py.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).
 */
#ifndef NETSORT_ORACLE_H
#define NETSORT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Dispatch counters — restates DispatchStats, include/netsort/hybrid.hpp:18-34 */
typedef struct oracle_stats {
  uint64_t network_hits[9]; /* indexed by width */
  uint64_t merges;
  uint64_t partitions;
  int32_t max_depth;
} oracle_stats;

/* SplitMix64 — include/netsort/datagen.hpp:29-42 */
uint64_t oracle_splitmix64_next(uint64_t* state);

/* int32 inputs (builder decision):
 *   kind 0 random        : (int32)(next() >> 33), U[0, 2^31)
 *   kind 1 sorted        : 0..n-1                       (datagen.cpp:31-34)
 *   kind 2 nearly_sorted : ramp + floor(p*n) swaps, min 1 (datagen.cpp:35-47)
 * returns 0, or -1 when p lies outside [0,1] (datagen.cpp:20-23). */
int oracle_generate_i32(int kind, size_t n, uint64_t seed, double p, int32_t* out);
/* The reference's own int64 stream (datagen.cpp:18-50), for the KATs. */
int oracle_generate_i64(int kind, size_t n, uint64_t seed, double p, int64_t* out);

/* Ragged batch for BASELINE config 2: lengths 3 + next()%6 from SplitMix64(seed),
 * keys (int32)(next()>>33) from SplitMix64(seed ^ 0x5bd1e995).  offsets has
 * num_arrays+1 entries; keys must hold offsets[num_arrays] values (call with
 * keys == NULL first to size it; returns the key count). */
size_t oracle_generate_batch_i32(size_t num_arrays, uint64_t seed, uint32_t* offsets,
                                 int32_t* keys);

/* Network tables: the comparator lists this oracle uses for widths 2..8.
 * Writes 2*count bytes (lo,hi pairs); returns count, or -1 for a bad width
 * (networks.hpp:89-104 throws std::invalid_argument there). */
int oracle_network(int width, uint8_t* pairs, int cap);

/* sort_small — networks.hpp:132-145 (size 2..8, otherwise no-op) */
void oracle_sort_small_i32(int32_t* v, int size);

/* base_case_applies — include/netsort/config.hpp:30-36 */
int oracle_base_case_applies(int64_t size, uint32_t width_mask, int varsort_max);

/* optimized_merge_sort over inclusive [left,right] — hybrid.hpp:156-165,
 * recursion 81-95, merge_runs 61-79.  stats may be NULL. */
void oracle_merge_sort_i32(int32_t* a, int64_t left, int64_t right, uint32_t width_mask,
                           int varsort_max, oracle_stats* stats);
/* merge — hybrid.hpp:186-193 */
void oracle_merge_i32(int32_t* a, int64_t left, int64_t mid, int64_t right);

/* median_of_three — hybrid.hpp:105-114; hoare_partition — hybrid.hpp:121-133 */
int32_t oracle_median_of_three_i32(int32_t* a, int64_t low, int64_t high);
int64_t oracle_hoare_partition_i32(int32_t* a, int64_t low, int64_t high, int32_t pivot);

/* optimized_quick_sort over inclusive [low,high] — hybrid.hpp:197-204,
 * recursion 137-150.  stats may be NULL. */
void oracle_quick_sort_i32(int32_t* a, int64_t low, int64_t high, uint32_t width_mask,
                           int varsort_max, oracle_stats* stats);

/* int64 keys — the reference's own benchmark type (bench.hpp:59-61); same
 * functions, same citations (the reference templates them on T). */
void oracle_sort_small_i64(int64_t* v, int size);
void oracle_merge_sort_i64(int64_t* a, int64_t left, int64_t right, uint32_t width_mask,
                           int varsort_max, oracle_stats* stats);
void oracle_merge_i64(int64_t* a, int64_t left, int64_t mid, int64_t right);
int64_t oracle_median_of_three_i64(int64_t* a, int64_t low, int64_t high);
int64_t oracle_hoare_partition_i64(int64_t* a, int64_t low, int64_t high, int64_t pivot);
void oracle_quick_sort_i64(int64_t* a, int64_t low, int64_t high, uint32_t width_mask,
                           int varsort_max, oracle_stats* stats);

/* Classical (stable) merge sort of key/payload pairs: merge_sort_rec with the
 * Classic config (hybrid.hpp:81-95, no networks: they are not stable) and
 * merge_runs carrying the payload (hybrid.hpp:61-79, left run wins ties).
 * The oracle for ns_sort_pairs_i32 / ns_argsort_i32. */
void oracle_stable_sort_pairs_i32(int32_t* keys, uint32_t* vals, int64_t n);

/* Batch / segmented helpers (no reference symbol):
 * sort_small per array, optimized_quick_sort per fixed-length segment. */
void oracle_sort_small_batch_i32(int32_t* keys, const uint32_t* offsets, size_t num_arrays);
void oracle_segmented_quick_sort_i32(int32_t* keys, size_t num_segments, size_t seg_len,
                                     uint32_t width_mask, int varsort_max);

/* Order-independent multiset digest used for the permutation property at
 * full sizes (sum of a 64-bit mix of every key, and xor of the same). */
void oracle_multiset_digest_i32(const int32_t* keys, size_t n, uint64_t out[2]);
/* int64: the mix is applied to the key's 64-bit pattern */
void oracle_multiset_digest_i64(const int64_t* keys, size_t n, uint64_t out[2]);

#ifdef __cplusplus
}
#endif
#endif
