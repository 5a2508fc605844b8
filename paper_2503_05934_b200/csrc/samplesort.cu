// samplesort.cu — per-rank device steps of the multi-GPU sample sort (PSRS)
// and the g-way merge of received runs.
//
// No reference counterpart: the reference is single-process (SURVEY.md §2.2,
// §8(e)).  The host layer (paper_2503_05934_b200/samplesort.py) runs, on every
// rank: local merge sort (ns_merge_sort_i32) -> ns_regular_samples_i32 ->
// all-gather of samples -> ns_select_splitters_i32 -> ns_bucket_bounds_i32 ->
// all-to-all of counts and keys over NCCL -> ns_merge_runs_i32.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "mergesort.cuh"

namespace nsb {

__global__ void regular_samples_kernel(const int32_t* __restrict__ sorted, int64_t n, int s,
                                       int32_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < s) out[k] = sorted[(int64_t)(k + 1) * n / (s + 1)];
}

__global__ void pick_splitters_kernel(const int32_t* __restrict__ samples, int s, int g,
                                      int32_t* __restrict__ spl) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < g - 1) spl[k] = samples[(int64_t)(k + 1) * s / g];
}

// bounds[k] = lower_bound(sorted, spl[k-1]) for 1 <= k < g; bounds[0] = 0,
// bounds[g] = n.  Keys equal to a splitter go to the upper bucket.
__global__ void bucket_bounds_kernel(const int32_t* __restrict__ sorted, int64_t n,
                                     const int32_t* __restrict__ spl, int g,
                                     int64_t* __restrict__ bounds) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > g) return;
  if (k == 0) { bounds[0] = 0; return; }
  if (k == g) { bounds[g] = n; return; }
  const int32_t key = spl[k - 1];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  bounds[k] = lo;
}

// ---- merge of pairs of runs given by POINTERS (possibly on peer GPUs) -----
// Pair p = (A_p[0..la_p), B_p[0..lb_p)) -> dst[out_off_p ..).  A_p/B_p may be
// peer addresses mapped over NVLink (ns_ipc_open_handle): the partition
// searches and the staging loads then read the peer's HBM directly, so the
// sample sort's all-to-all is fused into its first merge round (no receive
// buffer, no extra HBM pass, transfer overlapped with merging).  Tiles and
// the merge itself are the pairwise pass's (merge_staged_tile, mergesort.cuh):
// exactly NT*K outputs per full tile, odd K, +inf sentinels.
constexpr int kMaxPtrPairs = 32;
template <class Key>
struct PtrPairTable {
  int npairs;
  int contiguous;  // every B run directly follows its A run in one local buffer
  const Key* a[kMaxPtrPairs];
  const Key* b[kMaxPtrPairs];
  int64_t a_len[kMaxPtrPairs], b_len[kMaxPtrPairs], out_off[kMaxPtrPairs];
  int64_t tile0[kMaxPtrPairs + 1];
};

// tile shapes: int32 <256,29> (7424 keys, the pass default), int64 <256,15> (3840 keys)
template <class Key> struct PmShape;
template <> struct PmShape<int32_t> { static constexpr int NT = 256, K = 29; };
template <> struct PmShape<int64_t> { static constexpr int NT = 256, K = 15; };
template <class Key>
constexpr int pm_tile() { return PmShape<Key>::NT * PmShape<Key>::K; }

template <class Key>
__device__ __forceinline__ int ptr_pair_of(const PtrPairTable<Key>& t, int64_t tile) {
  int p = 0;
  while (p + 1 < t.npairs && t.tile0[p + 1] <= tile) ++p;
  return p;
}

template <class Key>
__global__ void ptr_pairs_partition_kernel(PtrPairTable<Key> t, int64_t* __restrict__ mp) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t.tile0[t.npairs]) return;
  const int p = ptr_pair_of(t, c);
  const int64_t diag = (c - t.tile0[p]) * pm_tile<Key>();
  mp[c] = merge_path<int64_t>(t.a[p], t.a_len[p], t.b[p], t.b_len[p], diag);
}

template <class Key>
__global__ void __launch_bounds__(PmShape<Key>::NT, v2_min_blocks(PmShape<Key>::NT, PmShape<Key>::K,
                                                                  (int)sizeof(Key)))
    ptr_pairs_merge_kernel(Key* __restrict__ dst, PtrPairTable<Key> t,
                           const int64_t* __restrict__ mp) {
  constexpr int NT = PmShape<Key>::NT, K = PmShape<Key>::K, TM = NT * K;
  constexpr int PV = kpv<Key>();
  constexpr int KB = (int)sizeof(Key);
  __shared__ __align__(128) Key sm[v2_smem_words(TM, K)];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int64_t s_out;
  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  const int p = ptr_pair_of(t, c);
  const int64_t pair_len = t.a_len[p] + t.b_len[p];
  const int64_t diag0 = (c - t.tile0[p]) * TM;
  const int64_t diag1 = min(diag0 + TM, pair_len);
  const int64_t a0 = mp[c];
  const int64_t a1 = (diag1 == pair_len) ? t.a_len[p] : mp[c + 1];
  const int la = (int)(a1 - a0);
  const int lb = (int)((diag1 - a1) - (diag0 - a0));
  const Key* A = t.a[p] + a0;
  const Key* B = t.b[p] + (diag0 - a0);
  // smem placement mirrors global 16-byte alignment (bulk copies need it)
  const uintptr_t a_addr = reinterpret_cast<uintptr_t>(A), b_addr = reinterpret_cast<uintptr_t>(B);
  const int a_shift = (int)((a_addr & 15) / KB), b_shift = (int)((b_addr & 15) / KB);
  const int b_off = (a_shift + la + v2_pad(K) + PV - 1) & ~(PV - 1);
  const Key* a_cov = A - a_shift;
  const Key* b_cov = B - b_shift;
  const int a_words = (a_shift + la + PV - 1) & ~(PV - 1), b_words = (b_shift + lb + PV - 1) & ~(PV - 1);
  // bulk copies only for local runs inside one buffer, cover within the pair's
  // extent; peer runs are read with plain coalesced loads over NVLink
  const Key* lo = t.a[p];
  const Key* hi = t.b[p] + t.b_len[p];
  const bool a_tma = t.contiguous && la > 0 && (a_addr % KB) == 0 && a_cov >= lo && a_cov + a_words <= hi;
  const bool b_tma = t.contiguous && lb > 0 && (b_addr % KB) == 0 && b_cov >= lo && b_cov + b_words <= hi;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    s_out = t.out_off[p] + diag0;
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t bytes = (a_tma ? a_words * (uint32_t)KB : 0u) + (b_tma ? b_words * (uint32_t)KB : 0u);
    mbar_arrive_expect_tx(&bar, bytes);
    if (a_tma) tma_load_1d(sm, a_cov, a_words * (uint32_t)KB, &bar);
    if (b_tma) tma_load_1d(sm + b_off, b_cov, b_words * (uint32_t)KB, &bar);
  }
  if (!a_tma)
    for (int i = tid; i < la; i += NT) sm[a_shift + i] = __ldcs(A + i);
  if (!b_tma)
    for (int i = tid; i < lb; i += NT) sm[b_off + b_shift + i] = __ldcs(B + i);
  mbar_wait(&bar, 0);
  __syncthreads();
  merge_staged_tile<NT, K>(sm, a_shift, la, b_off + b_shift, lb, dst, &s_out);
}

// Host side: merges up to kMaxPtrPairs pairs in one partition + one merge launch.
template <class Key>
static int merge_ptr_pairs(const PtrPairTable<Key>& t0, Key* dst, int64_t* mp, cudaStream_t s) {
  constexpr int TM = pm_tile<Key>();
  PtrPairTable<Key> t = t0;
  int64_t tiles = 0;
  for (int p = 0; p < t.npairs; ++p) {
    t.tile0[p] = tiles;
    tiles += (t.a_len[p] + t.b_len[p] + TM - 1) / TM;
  }
  t.tile0[t.npairs] = tiles;
  if (tiles == 0) return NS_OK;
  {
    Prof prof(PK_PARTITION, s);
    ptr_pairs_partition_kernel<Key><<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(t, mp);
  }
  NSB_TRY(check_launch("ptr_pairs_partition_kernel"));
  {
    Prof prof(PK_MERGE_PASS, s);
    ptr_pairs_merge_kernel<Key><<<(unsigned)tiles, PmShape<Key>::NT, 0, s>>>(dst, t, mp);
  }
  return check_launch("ptr_pairs_merge_kernel");
}

// Merges num_runs sorted runs lying back to back in d_keys: pairwise rounds,
// each one pointer-pair launch (up to kMaxPtrPairs pairs).
template <class Key>
static int merge_runs_t(Key* d_keys, const int64_t* h_run_offsets, int num_runs, void* d_temp,
                        size_t temp_bytes, size_t need, cudaStream_t s) {
  if (num_runs < 1 || num_runs > 2 * kMaxPtrPairs || !h_run_offsets) return NS_ERR_INVALID;
  const int64_t n = h_run_offsets[num_runs] - h_run_offsets[0];
  if (num_runs == 1 || n <= 1) return NS_OK;
  for (int r = 0; r < num_runs; ++r)
    if (h_run_offsets[r + 1] < h_run_offsets[r]) return NS_ERR_INVALID;
  if (!d_keys) return NS_ERR_INVALID;
  if (!d_temp || temp_bytes < need) return NS_ERR_TEMP;
  Key* base = d_keys + h_run_offsets[0];
  Key* tmp = static_cast<Key*>(d_temp);
  int64_t* mp =
      reinterpret_cast<int64_t*>(static_cast<char*>(d_temp) + align_up(n * sizeof(Key), 256));

  std::vector<int64_t> runs(h_run_offsets, h_run_offsets + num_runs + 1);
  for (auto& r : runs) r -= h_run_offsets[0];
  int rounds = 0;
  for (int k = num_runs; k > 1; k = (k + 1) / 2) ++rounds;
  // Pick the first destination so that the last round lands in d_keys.
  Key* cur = base;
  Key* other = tmp;
  if (rounds & 1) {
    // odd round count: start by staging into tmp so the final write hits base
    NSB_TRY(check_cuda(cudaMemcpyAsync(tmp, base, n * sizeof(Key), cudaMemcpyDeviceToDevice, s),
                       "copy"));
    cur = tmp;
    other = base;
  }
  while (runs.size() > 2) {
    const int nr = (int)runs.size() - 1;
    PtrPairTable<Key> t{};
    t.npairs = (nr + 1) / 2;
    t.contiguous = 1;
    std::vector<int64_t> next{0};
    for (int p = 0; p < t.npairs; ++p) {
      const int ra = 2 * p, rb = 2 * p + 1;
      t.a[p] = cur + runs[ra];
      t.a_len[p] = runs[ra + 1] - runs[ra];
      t.b[p] = cur + runs[ra + 1];
      t.b_len[p] = rb < nr ? runs[rb + 1] - runs[rb] : 0;
      t.out_off[p] = runs[ra];
      next.push_back(runs[std::min(rb + 1, nr)]);
    }
    NSB_TRY(merge_ptr_pairs(t, other, mp, s));
    std::swap(cur, other);
    runs.swap(next);
  }
  return NS_OK;
}

static size_t merge_runs_temp(size_t n, int num_runs, size_t key_bytes, int tile) {
  if (num_runs <= 1) return 0;
  return align_up(n * key_bytes, 256) + align_up((n / tile + 2 * kMaxPtrPairs + 2) * 8, 256);
}

}  // namespace nsb

using namespace nsb;

extern "C" {

int ns_regular_samples_i32(const int32_t* d_sorted, size_t n, int s, int32_t* d_samples,
                           void* stream) {
  if (n == 0 || s <= 0 || !d_sorted || !d_samples) return NS_ERR_INVALID;
  Prof prof(PK_PSRS, static_cast<cudaStream_t>(stream));
  regular_samples_kernel<<<(s + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_sorted, (int64_t)n, s, d_samples);
  return check_launch("regular_samples_kernel");
}

int ns_select_splitters_i32(int32_t* d_samples, int s, int g, int32_t* d_splitters,
                            void* stream) {
  if (s <= 0 || s > kSmallTile || g < 1 || !d_samples || (g > 1 && !d_splitters))
    return NS_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NSB_TRY(merge_sort_device(d_samples, (size_t)s, 8, nullptr, 0, st));
  if (g == 1) return NS_OK;
  Prof prof(PK_PSRS, st);
  pick_splitters_kernel<<<(g + 255) / 256, 256, 0, st>>>(d_samples, s, g, d_splitters);
  return check_launch("pick_splitters_kernel");
}

int ns_bucket_bounds_i32(const int32_t* d_sorted, size_t n, const int32_t* d_splitters, int g,
                         int64_t* d_bounds, void* stream) {
  if (g < 1 || !d_bounds || (n && !d_sorted) || (g > 1 && !d_splitters)) return NS_ERR_INVALID;
  Prof prof(PK_PSRS, static_cast<cudaStream_t>(stream));
  bucket_bounds_kernel<<<(g + 1 + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      d_sorted, (int64_t)n, d_splitters, g, d_bounds);
  return check_launch("bucket_bounds_kernel");
}

size_t ns_merge_pairs_temp_bytes(int64_t total, int npairs) {
  return align_up((size_t)(total / pm_tile<int32_t>() + npairs + 2) * 8, 256);
}

int ns_merge_pairs_i32(const int32_t* const* a_ptrs, const int64_t* a_lens,
                       const int32_t* const* b_ptrs, const int64_t* b_lens, int npairs,
                       int32_t* d_out, void* d_temp, size_t temp_bytes, void* stream) {
  if (npairs < 0 || npairs > kMaxPtrPairs || (npairs && (!a_ptrs || !a_lens || !b_ptrs || !b_lens)))
    return NS_ERR_INVALID;
  if (npairs == 0) return NS_OK;
  PtrPairTable<int32_t> t{};
  t.npairs = npairs;
  int64_t off = 0;
  for (int p = 0; p < npairs; ++p) {
    if (a_lens[p] < 0 || b_lens[p] < 0) return NS_ERR_INVALID;
    if ((a_lens[p] && !a_ptrs[p]) || (b_lens[p] && !b_ptrs[p])) return NS_ERR_INVALID;
    t.a[p] = a_ptrs[p];
    t.b[p] = b_ptrs[p] ? b_ptrs[p] : a_ptrs[p];
    t.a_len[p] = a_lens[p];
    t.b_len[p] = b_lens[p];
    t.out_off[p] = off;
    off += a_lens[p] + b_lens[p];
  }
  if (off == 0) return NS_OK;
  if (!d_out || !d_temp || temp_bytes < ns_merge_pairs_temp_bytes(off, npairs)) return NS_ERR_TEMP;
  return merge_ptr_pairs(t, d_out, static_cast<int64_t*>(d_temp),
                         static_cast<cudaStream_t>(stream));
}

size_t ns_merge_runs_temp_bytes(size_t n, int num_runs) {
  return merge_runs_temp(n, num_runs, 4, pm_tile<int32_t>());
}

size_t ns_merge_runs_temp_bytes_i64(size_t n, int num_runs) {
  return merge_runs_temp(n, num_runs, 8, pm_tile<int64_t>());
}

int ns_merge_runs_i32(int32_t* d_keys, const int64_t* h_run_offsets, int num_runs, void* d_temp,
                      size_t temp_bytes, void* stream) {
  const size_t n = (h_run_offsets && num_runs >= 1 && num_runs <= 2 * kMaxPtrPairs)
                       ? (size_t)(h_run_offsets[num_runs] - h_run_offsets[0]) : 0;
  return merge_runs_t(d_keys, h_run_offsets, num_runs, d_temp, temp_bytes,
                      ns_merge_runs_temp_bytes(n, num_runs), static_cast<cudaStream_t>(stream));
}

int ns_merge_runs_i64(int64_t* d_keys, const int64_t* h_run_offsets, int num_runs, void* d_temp,
                      size_t temp_bytes, void* stream) {
  const size_t n = (h_run_offsets && num_runs >= 1 && num_runs <= 2 * kMaxPtrPairs)
                       ? (size_t)(h_run_offsets[num_runs] - h_run_offsets[0]) : 0;
  return merge_runs_t(d_keys, h_run_offsets, num_runs, d_temp, temp_bytes,
                      ns_merge_runs_temp_bytes_i64(n, num_runs), static_cast<cudaStream_t>(stream));
}

}  // extern "C"
