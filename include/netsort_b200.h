/*
 * netsort_b200.h — C ABI of the B200 (sm_100a) hybrid network-base-case sort.
 *
 * This is the drop-in boundary under the reference's header-only C++ API
 * (/root/reference/proj/include/netsort/hybrid.hpp, config.hpp).  The
 * reference has no FFI of its own; its only injection point is the
 * `std::function<void(std::span<std::int64_t>)> sort_fn` that measure_loop
 * calls (bench.hpp:58-61, bound to run_variant at bench.cpp:94-96).  The C++
 * host layer include/netsort_b200.hpp keeps the reference's entry points
 * (optimized_merge_sort / optimized_quick_sort / run_variant, NetworkConfig /
 * find_config / base_case_applies) and calls down into these functions; a
 * ctypes / cgo / JNI binding would call them directly.
 *
 * Conventions
 *   - keys are int32_t (the BASELINE configs; *_i32) or int64_t (the
 *     reference's own benchmark type; *_i64), sorted ascending, in place;
 *   - ranges are half-open (ptr, n); the C++ layer converts the reference's
 *     inclusive [left, right] and keeps its "right < left is a no-op" rule
 *     (hybrid.hpp:160, 201);
 *   - d_* pointers are caller-owned device memory; `stream` is a
 *     cudaStream_t (NULL = legacy default stream); every device entry point
 *     is stream-ordered and asynchronous, never synchronises unless stated;
 *   - scratch is caller-provided: query *_temp_bytes(n) first;
 *   - a network configuration is (width_mask, varsort_max) exactly as
 *     NetworkConfig (config.hpp:20-26): bit w of width_mask enables the
 *     fixed width-w network, varsort_max != 0 enables widths 2..varsort_max;
 *   - no function throws; each returns an ns_status.  There is no CPU
 *     fallback: without a usable sm_100a device every compute call returns
 *     NS_ERR_CUDA.
 */
#ifndef NETSORT_B200_H
#define NETSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ns_status {
  NS_OK = 0,
  NS_ERR_INVALID = 1, /* bad argument / config (reference: std::invalid_argument) */
  NS_ERR_CUDA = 2,    /* CUDA runtime / launch error, or no device */
  NS_ERR_OOM = 3,     /* device or pinned-host allocation failed */
  NS_ERR_TEMP = 4,    /* caller scratch smaller than *_temp_bytes (or an output
                         buffer smaller than the result, see sample sort) */
  NS_ERR_NCCL = 5     /* NCCL unavailable or an NCCL call failed */
} ns_status;

typedef enum ns_algorithm { NS_MERGE_SORT = 0, NS_QUICK_SORT = 1 } ns_algorithm;

/* ---- library / configuration ------------------------------------------ */

/* Human-readable status; never NULL. */
const char* ns_status_string(int status);
/* Last CUDA error string recorded by this thread ("" if none). */
const char* ns_last_error(void);
/* ABI version (major*10000 + minor*100 + patch). */
int ns_version(void);

/* find_config — src/config.cpp:55-60.  Fills the (mask, varsort) pair of a
 * registry preset by case-sensitive name; NS_ERR_INVALID if unknown. */
int ns_find_config(const char* name, uint32_t* width_mask, int* varsort_max);
/* config_registry — src/config.cpp:35-53: number of presets and their names
 * in registry order (Classic, PowerOf2, ..., VarSort5). */
int ns_config_count(void);
const char* ns_config_name(int index);
/* base_case_applies — include/netsort/config.hpp:30-36. */
int ns_base_case_applies(int64_t size, uint32_t width_mask, int varsort_max);
/* Per-thread leaf width the kernels use for this config (8, 4, 2 or 1): the
 * reference recursion's shape on an 8-key window. */
int ns_leaf_width(uint32_t width_mask, int varsort_max);
/* The comparator list the kernels run for one width (bundled_network,
 * networks.hpp:89-104): writes `cap` (lo,hi) byte pairs at most and returns
 * the comparator count, or -1 for a width outside [2, 8]. */
int ns_network_comparators(int width, uint8_t* pairs, int cap);
/* DispatchStats of the reference's merge sort for n keys (hybrid.hpp:18-34,
 * recursion 81-95), computed from the recursion shape, which depends on n and
 * the config only: out12 = network_hits[0..8], merges, partitions (0),
 * max_depth.  Host-only; no device work. */
int ns_merge_sort_dispatch_stats(int64_t n, uint32_t width_mask, int varsort_max,
                                 uint64_t* out12);

/* ---- device entry points (caller-owned device memory) ----------------- */

/* optimized_merge_sort — include/netsort/hybrid.hpp:156-177. */
size_t ns_merge_sort_temp_bytes(size_t n);
int ns_merge_sort_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream);
/* The same for int64 keys, the type the reference's own benchmarks and
 * generator use (optimized_merge_sort<std::int64_t>, bench.hpp:59-61,
 * datagen.hpp:47). */
size_t ns_merge_sort_temp_bytes_i64(size_t n);
int ns_merge_sort_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream);

/* optimized_quick_sort — include/netsort/hybrid.hpp:197-216.  GPU form: a
 * sampled-pivot partition (the many-pivot analogue of median_of_three +
 * hoare_partition, hybrid.hpp:105-133; up to 127 pivots per segment and
 * level) recursing until buckets fit one CTA, whose on-chip sort uses the
 * config's network base case.  Bucket sizes are planned ON THE DEVICE (work
 * lists, upper-bound grids): the call never synchronises and can be captured
 * in a CUDA graph.  n < 2^32 per array. */
size_t ns_quick_sort_temp_bytes(size_t n);
int ns_quick_sort_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream);
/* int64 keys (optimized_quick_sort<std::int64_t>): always the multi-level
 * splitter partition. */
size_t ns_quick_sort_temp_bytes_i64(size_t n);
int ns_quick_sort_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream);

/* The reference's quick sort executed node for node (qs_trace.cu):
 * median_of_three (hybrid.hpp:105-114) + hoare_partition (121-133) at every
 * node of quick_sort_rec (137-150), the same pivots, swaps and splits, so the
 * DispatchStats counters equal the reference's (optimized_quick_sort(...,
 * stats), hybrid.hpp:197-204; run_variant 234-243).  out12 = network_hits
 * [0..8], merges (0), partitions, max_depth; n == 0 leaves them zero (no
 * call, hybrid.hpp:201).  This is the instrumentation path, not the timed
 * one: it synchronises the stream once per recursion level above 8192 keys.
 * n < 2^32.  Temp: ns_quick_sort_traced_temp_bytes(n) (either key type). */
size_t ns_quick_sort_traced_temp_bytes(size_t n);
int ns_quick_sort_traced_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                             uint64_t* out12, void* d_temp, size_t temp_bytes, void* stream);
int ns_quick_sort_traced_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                             uint64_t* out12, void* d_temp, size_t temp_bytes, void* stream);
/* hoare_partition — hybrid.hpp:121-133, on d_keys[low..high] (inclusive,
 * 0 <= low < high < n) of a device array of n keys: the same swaps in the
 * same cells and the same returned split (written to the HOST word *split,
 * absolute index; the call synchronises).  Two streaming passes, no
 * sequential scan.  The reference requires the pivot to occur in the range;
 * here a pivot above every key or below every key (where the reference's scan
 * would leave the range) is NS_ERR_INVALID with the keys untouched.
 * Temp: ns_hoare_partition_temp_bytes(high - low + 1). */
size_t ns_hoare_partition_temp_bytes(size_t len);
int ns_hoare_partition_i32(int32_t* d_keys, size_t n, int64_t low, int64_t high, int32_t pivot,
                           int64_t* split, void* d_temp, size_t temp_bytes, void* stream);
int ns_hoare_partition_i64(int64_t* d_keys, size_t n, int64_t low, int64_t high, int64_t pivot,
                           int64_t* split, void* d_temp, size_t temp_bytes, void* stream);
/* median_of_three — hybrid.hpp:105-114: the three compare-exchanges on cells
 * low, low+(high-low)/2, high (none when high-low < 2), pivot to the HOST
 * word *pivot (the call synchronises). */
int ns_median_of_three_i32(int32_t* d_keys, size_t n, int64_t low, int64_t high, int32_t* pivot,
                           void* stream);
int ns_median_of_three_i64(int64_t* d_keys, size_t n, int64_t low, int64_t high, int64_t* pivot,
                           void* stream);

/* Base-case batch (BASELINE config 2; no reference batch API — the
 * reference would loop sort_small, networks.hpp:132-145): num_arrays
 * independent arrays packed contiguously, array i = d_keys[d_offsets[i] ..
 * d_offsets[i+1]); every length must lie in [0, 8].  Each array of length
 * 2..8 is sorted by its own size-specific network; 0/1 are no-ops (the
 * reference's apply_varsort rule, networks.hpp:166-176).  A validation pass
 * over all offsets runs first: if any length lies outside [0, 8] NO key is
 * modified and the status is NS_ERR_INVALID.
 *   ns_sort_small_batch_async_i32: stream-ordered, never synchronises (CUDA-
 *     graph capturable); the status (NS_OK / NS_ERR_INVALID) is written to the
 *     caller's device word *d_status.
 *   ns_sort_small_batch_i32: the same, then reads the status back (one
 *     4-byte D2H + stream synchronise) and returns it. */
int ns_sort_small_batch_async_i32(int32_t* d_keys, const uint32_t* d_offsets, size_t num_arrays,
                                  int* d_status, void* stream);
int ns_sort_small_batch_i32(int32_t* d_keys, const uint32_t* d_offsets, size_t num_arrays,
                            void* stream);

/* Stable key-value sort and argsort.  The
 * reference's classical merge sort is stable (merge_runs keeps the left run
 * on ties, hybrid.hpp:61-79; test_hybrid.cpp:119-150) but has no payload API.
 * ns_sort_pairs_i32 sorts d_keys in place and applies the same stable
 * permutation to the 32-bit payload d_values (may be NULL).  ns_argsort_i32
 * writes d_perm with d_keys[d_perm[i]] stably ascending; d_keys is not
 * modified.  n < 2^32. */
size_t ns_sort_pairs_temp_bytes_i32(size_t n);
int ns_sort_pairs_i32(int32_t* d_keys, uint32_t* d_values, size_t n, void* d_temp,
                      size_t temp_bytes, void* stream);
size_t ns_argsort_temp_bytes_i32(size_t n);
int ns_argsort_i32(const int32_t* d_keys, uint32_t* d_perm, size_t n, void* d_temp,
                   size_t temp_bytes, void* stream);

/* Segmented sort of num_segments independent arrays of seg_len keys each,
 * stored back to back (BASELINE config 4's 65,536 x 16,384 batch).  The
 * reference would run `algorithm` once per segment.  Segments of up to 16384
 * keys are one CTA each; longer ones, with NS_QUICK_SORT, are all level-0
 * segments of ONE device-planned partition, with NS_MERGE_SORT one tile-sort
 * launch over every segment's tiles plus pairwise passes whose run pairs stay
 * inside their segment (no per-segment host loop either way; the merge path
 * needs the scratch of a merge sort of all the keys).
 * num_segments * seg_len overflowing is NS_ERR_INVALID. */
size_t ns_segmented_sort_temp_bytes(size_t num_segments, size_t seg_len);
int ns_segmented_sort_i32(int32_t* d_keys, size_t num_segments, size_t seg_len,
                          int algorithm, uint32_t width_mask, int varsort_max, void* d_temp,
                          size_t temp_bytes, void* stream);
size_t ns_segmented_sort_temp_bytes_i64(size_t num_segments, size_t seg_len);
int ns_segmented_sort_i64(int64_t* d_keys, size_t num_segments, size_t seg_len,
                          int algorithm, uint32_t width_mask, int varsort_max, void* d_temp,
                          size_t temp_bytes, void* stream);

/* ---- sample-sort building blocks (multi-GPU layer, BASELINE config 5) ---
 * The exchange itself is an NCCL all-to-all issued by the host layer; these
 * are the per-rank device steps around it. */

/* Regular sampling of a sorted shard: d_samples[k] = d_sorted[(k+1)*n/(s+1)]
 * for k < s (PSRS).  n must be >= 1. */
int ns_regular_samples_i32(const int32_t* d_sorted, size_t n, int s, int32_t* d_samples,
                           void* stream);
/* Sorts a small sample set (s <= 16384) in place and writes the g-1
 * splitters at regular positions: d_splitters[k] = d_samples[(k+1)*s/g]. */
int ns_select_splitters_i32(int32_t* d_samples, int s, int g, int32_t* d_splitters,
                            void* stream);
/* Bucket bounds of a sorted shard (int64): d_bounds[0] = 0, d_bounds[g] = n,
 * d_bounds[k] = number of keys < d_splitters[k-1] (lower_bound), so keys
 * equal to a splitter go to the upper bucket. */
int ns_bucket_bounds_i32(const int32_t* d_sorted, size_t n, const int32_t* d_splitters, int g,
                         int64_t* d_bounds, void* stream);
/* Merges `num_runs` sorted runs that lie back to back in d_keys (run r =
 * [d_run_offsets[r], d_run_offsets[r+1]) with host-side h_run_offsets the
 * same values) into one sorted array, in place. */
size_t ns_merge_runs_temp_bytes(size_t n, int num_runs);
int ns_merge_runs_i32(int32_t* d_keys, const int64_t* h_run_offsets, int num_runs,
                      void* d_temp, size_t temp_bytes, void* stream);
size_t ns_merge_runs_temp_bytes_i64(size_t n, int num_runs);
int ns_merge_runs_i64(int64_t* d_keys, const int64_t* h_run_offsets, int num_runs,
                      void* d_temp, size_t temp_bytes, void* stream);

/* Merges npairs (<= 32) independent pairs of sorted runs given by POINTERS:
 * pair p = (a_ptrs[p][0 .. a_lens[p]), b_ptrs[p][0 .. b_lens[p])) goes to
 * d_out[o_p .. o_p + a_lens[p] + b_lens[p]), o_p = sum of the earlier pairs'
 * lengths.  a_ptrs / b_ptrs / lengths are HOST arrays; the runs may live on
 * peer GPUs (pointers from ns_ipc_open_handle, read over NVLink), which fuses
 * the sample sort's all-to-all into its first merge round. */
size_t ns_merge_pairs_temp_bytes(int64_t total, int npairs);
int ns_merge_pairs_i32(const int32_t* const* a_ptrs, const int64_t* a_lens,
                       const int32_t* const* b_ptrs, const int64_t* b_lens, int npairs,
                       int32_t* d_out, void* d_temp, size_t temp_bytes, void* stream);

/* ---- multi-GPU, one host thread --------------
 * The sample sort of BASELINE config 5 over ngpu devices driven by ONE host
 * thread: shard d = d_shards[d][0 .. counts[d]) on device devices[d], its
 * stream streams[d] and scratch d_temps[d] (temp_bytes each, from
 * ns_sample_sort_multi_temp_bytes(ngpu, max shard, out_capacity)).  Steps:
 * local merge sort (the config's network base case) -> 255 regular samples
 * per shard -> all-gather -> g-1 common splitters -> bucket bounds ->
 * exchange -> g-way merge.  Device d receives the d-th key range of the
 * sorted array in d_out[d][0 .. out_counts[d]); concatenated in device order
 * the outputs are the sorted input.  The shards are sorted in place as a
 * side effect.
 *   exchange NS_EXCHANGE_NCCL: grouped ncclSend / ncclRecv over `comms`
 *     (one communicator per device, e.g. ns_nccl_comms_init_all = the
 *     single-process ncclCommInitAll), then a merge of the received runs;
 *   exchange NS_EXCHANGE_P2P: no receive buffer — each device merges the
 *     runs destined to it directly out of its peers' memory over NVLink
 *     (peer access; comms may be NULL; devices may repeat, e.g. several
 *     virtual ranks on one GPU).
 * The bucket bounds come to the host once (they size the exchange) and the
 * call synchronises every stream before returning (peers read the shards).
 * A result larger than out_capacity returns NS_ERR_TEMP with out_counts set.
 * NCCL is loaded at run time (libnccl.so.2); ns_nccl_available() says
 * whether it could be. */
typedef struct ncclComm* ns_nccl_comm; /* == ncclComm_t */
typedef enum ns_exchange { NS_EXCHANGE_NCCL = 0, NS_EXCHANGE_P2P = 1 } ns_exchange;
int ns_nccl_available(void);
int ns_nccl_comms_init_all(int ngpu, const int* devices, ns_nccl_comm* comms);
int ns_nccl_comms_destroy(int ngpu, ns_nccl_comm* comms);
/* Host-only exchange plan: bounds is ngpu rows of ngpu+1 bucket bounds (row
 * src = the sorted shard src cut for every destination); writes, per
 * destination dst, recv_offsets[dst*(ngpu+1) + src] = where src's run starts
 * in dst's output (row ends with the total) and recv_totals[dst]. */
int ns_sample_sort_plan(int ngpu, const int64_t* bounds, int64_t* recv_offsets,
                        int64_t* recv_totals);
size_t ns_sample_sort_multi_temp_bytes(int ngpu, size_t shard_keys, size_t out_capacity);
int ns_sample_sort_multi_i32(int ngpu, const int* devices, ns_nccl_comm* comms, int exchange,
                             int32_t* const* d_shards, const size_t* counts, int32_t* const* d_out,
                             size_t out_capacity, size_t* out_counts, uint32_t width_mask,
                             int varsort_max, void* const* d_temps, size_t temp_bytes,
                             void* const* streams);
/* Shard by array (BASELINE configs 2 and 4: independent arrays, no
 * collective).  ns_shard_batch_plan cuts a ragged batch (host offsets,
 * num_arrays + 1 entries) into nshards contiguous array ranges of about
 * equal key counts: shard k = arrays [array_begin[k], array_begin[k+1]).
 * The multi entry points then run the single-device call on every device's
 * shard (offsets rebased to the shard's first key; status per device). */
int ns_shard_batch_plan(const uint32_t* h_offsets, size_t num_arrays, int nshards,
                        size_t* array_begin);
int ns_sort_small_batch_multi_i32(int ngpu, const int* devices, int32_t* const* d_keys,
                                  const uint32_t* const* d_offsets, const size_t* num_arrays,
                                  int* const* d_status, void* const* streams);
int ns_segmented_sort_multi_i32(int ngpu, const int* devices, int32_t* const* d_keys,
                                const size_t* num_segments, size_t seg_len, int algorithm,
                                uint32_t width_mask, int varsort_max, void* const* d_temps,
                                const size_t* temp_bytes, void* const* streams);

/* CUDA IPC for the pull-based exchange: export the allocation that contains
 * d_ptr (64-byte handle + byte offset of d_ptr inside it), map a peer's
 * allocation (lazy peer access), unmap it. */
int ns_ipc_get_handle(const void* d_ptr, uint8_t* handle64, uint64_t* offset);
int ns_ipc_open_handle(const uint8_t* handle64, void** d_base);
int ns_ipc_close(void* d_base);

/* ---- checking helpers (used by tests and bench, not by the sort) ------- */

/* d_out[0] += sum of mix64(key), d_out[1] ^= xor of mix64(key) (uint64);
 * an order-independent multiset digest (matches the oracle's). */
int ns_multiset_digest_i32(const int32_t* d_keys, size_t n, uint64_t* d_out, void* stream);
/* d_out[0] += number of i with d_keys[i] > d_keys[i+1] (0 == sorted). */
int ns_count_inversions_i32(const int32_t* d_keys, size_t n, unsigned long long* d_out,
                            void* stream);
/* int64 forms of the two checking helpers (the digest mixes all 64 bits;
 * matches oracle_multiset_digest_i64). */
int ns_multiset_digest_i64(const int64_t* d_keys, size_t n, uint64_t* d_out, void* stream);
int ns_count_inversions_i64(const int64_t* d_keys, size_t n, unsigned long long* d_out,
                            void* stream);

/* Device generator for the seeded inputs (bench/tests): kind 0 = uniform
 * random int32 in [0, 2^31) = int32(SplitMix64(seed).next() >> 33) element by
 * element (datagen.hpp:29-42 narrowed as in SURVEY.md §8(d)); kind 1 = the
 * ramp 0..n-1.  Identical to oracle_generate_i32 for the same (kind, seed). */
int ns_generate_i32(int32_t* d_out, size_t n, int kind, uint64_t seed, void* stream);
/* Host-side forms (datagen.cpp): kind 0 random, 1 sorted (ramp), 2 nearly
 * sorted = the ramp after floor(p*n) seeded index-pair swaps (at least one
 * when p > 0) — generate(), src/datagen.cpp:18-50, at int32 (random =
 * int32(next() >> 33)) or at the reference's own int64 (random = next()).
 * The ragged batch of BASELINE config 2: lengths 3 + next() % 6 from stream
 * `seed`, keys int32(next() >> 33) from stream seed ^ 0x5bd1e995; writes
 * num_arrays + 1 offsets and returns the key count (either pointer may be
 * NULL to query it). */
int ns_generate_host_i32(int32_t* h_out, size_t n, int kind, uint64_t seed, double p);
int ns_generate_host_i64(int64_t* h_out, size_t n, int kind, uint64_t seed, double p);
size_t ns_generate_batch_host_i32(size_t num_arrays, uint64_t seed, uint32_t* h_offsets,
                                  int32_t* h_keys);

/* ---- instrumentation ----------------------------------------------------
 * ns_launch_count: kernels this library has launched since load (process-
 * wide).  The profiler, when enabled, records a CUDA event pair around every
 * launch on the launching stream, grouped by kernel class; ns_profile_read
 * synchronises those events and returns the summed device time and launch
 * count of one class.  ns_profile_enable(0|1) also clears the records. */
uint64_t ns_launch_count(void);
int ns_profile_enable(int on);
int ns_profile_kinds(void);
const char* ns_profile_kind_name(int kind);
int ns_profile_read(int kind, double* total_ms, uint64_t* launches);

/* ---- host-buffer entry points (the reference's own call shape) ---------
 * Sort a HOST array in place, exactly like optimized_merge_sort(span, cfg):
 * copies through pinned staging to the current device, sorts, copies back,
 * synchronises.  Device buffers are cached per thread (ns_release_cache). */
int ns_merge_sort_host_i32(int32_t* h_keys, size_t n, uint32_t width_mask, int varsort_max);
int ns_quick_sort_host_i32(int32_t* h_keys, size_t n, uint32_t width_mask, int varsort_max);
int ns_merge_sort_host_i64(int64_t* h_keys, size_t n, uint32_t width_mask, int varsort_max);
int ns_quick_sort_host_i64(int64_t* h_keys, size_t n, uint32_t width_mask, int varsort_max);
/* merge — hybrid.hpp:186-193: h_keys[0, n_left) and h_keys[n_left, n) are
 * sorted runs of a HOST array; merges them in place (stable, left run wins
 * ties).  n_left == 0 or n_left == n is a no-op. */
/* Stream-ordered host-array sorts: upload h_in, sort with the config's
 * network base case, download into h_out (h_out == h_in allowed), all
 * enqueued on `stream`; the call returns immediately (synchronise the stream
 * before reading h_out).  Device buffers are cached per (device, stream) and
 * reused only by later calls on the same stream.  With pinned host buffers,
 * sorts on two streams overlap one upload with the other's download. */
int ns_merge_sort_host_async_i32(const int32_t* h_in, int32_t* h_out, size_t n,
                                 uint32_t width_mask, int varsort_max, void* stream);
int ns_quick_sort_host_async_i32(const int32_t* h_in, int32_t* h_out, size_t n,
                                 uint32_t width_mask, int varsort_max, void* stream);
int ns_merge_host_i32(int32_t* h_keys, size_t n_left, size_t n);
int ns_merge_host_i64(int64_t* h_keys, size_t n_left, size_t n);
int ns_release_cache(void);
/* Host-array forms of the traced quick sort, hoare_partition and
 * median_of_three above (the reference's optimized_quick_sort(span, low,
 * high, cfg, stats) / hoare_partition(span, low, high, pivot) /
 * median_of_three(span, low, high) call shapes): the range goes to the
 * device, the device call runs, the range comes back; synchronous. */
int ns_quick_sort_traced_host_i32(int32_t* h_keys, size_t n, uint32_t width_mask, int varsort_max,
                                  uint64_t* out12);
int ns_quick_sort_traced_host_i64(int64_t* h_keys, size_t n, uint32_t width_mask, int varsort_max,
                                  uint64_t* out12);
int ns_hoare_partition_host_i32(int32_t* h_keys, size_t n, int64_t low, int64_t high,
                                int32_t pivot, int64_t* split);
int ns_hoare_partition_host_i64(int64_t* h_keys, size_t n, int64_t low, int64_t high,
                                int64_t pivot, int64_t* split);
int ns_median_of_three_host_i32(int32_t* h_keys, size_t n, int64_t low, int64_t high,
                                int32_t* pivot);
int ns_median_of_three_host_i64(int64_t* h_keys, size_t n, int64_t low, int64_t high,
                                int64_t* pivot);

#ifdef __cplusplus
}
#endif
#endif /* NETSORT_B200_H */
