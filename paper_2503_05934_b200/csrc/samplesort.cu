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

constexpr int kPmNT = 512, kPmK = 16, kPmT = kPmNT * kPmK;

// ---- merge of pairs of runs given by POINTERS (possibly on peer GPUs) -----
// Pair p = (A_p[0..la_p), B_p[0..lb_p)) -> dst[out_off_p ..).  A_p/B_p may be
// peer addresses mapped over NVLink (ns_ipc_open_handle): the partition
// searches and the staging loads then read the peer's HBM directly, so the
// sample sort's all-to-all is fused into its first merge round (no receive
// buffer, no extra HBM pass, transfer overlapped with merging).
constexpr int kMaxPtrPairs = 32;
struct PtrPairTable {
  int npairs;
  int contiguous;  // every B run directly follows its A run in one buffer
  const int32_t* a[kMaxPtrPairs];
  const int32_t* b[kMaxPtrPairs];
  int64_t a_len[kMaxPtrPairs], b_len[kMaxPtrPairs], out_off[kMaxPtrPairs];
  int64_t tile0[kMaxPtrPairs + 1];
};

__device__ __forceinline__ int ptr_pair_of(const PtrPairTable& t, int64_t tile) {
  int p = 0;
  while (p + 1 < t.npairs && t.tile0[p + 1] <= tile) ++p;
  return p;
}

template <int TM>
__global__ void ptr_pairs_partition_kernel(PtrPairTable t, int64_t* __restrict__ mp) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t.tile0[t.npairs]) return;
  const int p = ptr_pair_of(t, c);
  const int64_t diag = (c - t.tile0[p]) * TM;
  mp[c] = merge_path<int64_t>(t.a[p], t.a_len[p], t.b[p], t.b_len[p], diag);
}

template <int NT, int K>
__global__ void __launch_bounds__(NT)
    ptr_pairs_merge_kernel(int32_t* __restrict__ dst, PtrPairTable t,
                           const int64_t* __restrict__ mp) {
  constexpr int TM = NT * K;
  __shared__ __align__(16) int32_t sm[padded_words(TM)];
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
  const int32_t* A = t.a[p] + a0;
  const int32_t* B = t.b[p] + (diag0 - a0);
  const int total = la + lb;
  if (t.contiguous) {
    // one allocation: 128-bit staging bounded by the pair's own extent
    stage_slices<NT, TM>(t.a[p], t.b[p] + t.b_len[p], A, la, B, lb, sm);
  } else {
    // runs in different (possibly peer) allocations: scalar coalesced loads
#pragma unroll 8
    for (int i = tid; i < total; i += NT)
      sm[pad_idx(i)] = i < la ? __ldcs(A + i) : __ldcs(B + (i - la));
  }
  __syncthreads();
  const int diag = min(tid * K, total);
  const SmemRun<int32_t> SA{sm, 0}, SB{sm, la};
  const int a = merge_path<int>(SA, la, SB, lb, diag);
  int32_t v[K];
  serial_merge<K>(SA, la, SB, lb, a, diag - a, v);
  __syncthreads();
  regs_to_smem<K>(sm, v);
  __syncthreads();
  tile_store<NT, TM>(sm, dst + t.out_off[p] + diag0, total);
}

// Host side: merges up to kMaxPtrPairs pairs in one partition + one merge launch.
static int merge_ptr_pairs(const PtrPairTable& t0, int32_t* dst, int64_t* mp, cudaStream_t s) {
  PtrPairTable t = t0;
  int64_t tiles = 0;
  for (int p = 0; p < t.npairs; ++p) {
    t.tile0[p] = tiles;
    tiles += (t.a_len[p] + t.b_len[p] + kPmT - 1) / kPmT;
  }
  t.tile0[t.npairs] = tiles;
  if (tiles == 0) return NS_OK;
  {
    Prof prof(PK_PARTITION, s);
    ptr_pairs_partition_kernel<kPmT><<<(unsigned)((tiles + 255) / 256), 256, 0, s>>>(t, mp);
  }
  NSB_TRY(check_launch("ptr_pairs_partition_kernel"));
  {
    Prof prof(PK_MERGE_PASS, s);
    ptr_pairs_merge_kernel<kPmNT, kPmK><<<(unsigned)tiles, kPmNT, 0, s>>>(dst, t, mp);
  }
  return check_launch("ptr_pairs_merge_kernel");
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
  return align_up((size_t)(total / kPmT + npairs + 2) * 8, 256);
}

int ns_merge_pairs_i32(const int32_t* const* a_ptrs, const int64_t* a_lens,
                       const int32_t* const* b_ptrs, const int64_t* b_lens, int npairs,
                       int32_t* d_out, void* d_temp, size_t temp_bytes, void* stream) {
  if (npairs < 0 || npairs > kMaxPtrPairs || (npairs && (!a_ptrs || !a_lens || !b_ptrs || !b_lens)))
    return NS_ERR_INVALID;
  if (npairs == 0) return NS_OK;
  PtrPairTable t{};
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
  if (num_runs <= 1) return 0;
  return align_up(n * 4, 256) + align_up((n / kPmT + 2 * kMaxPtrPairs + 2) * 8, 256);
}

int ns_merge_runs_i32(int32_t* d_keys, const int64_t* h_run_offsets, int num_runs, void* d_temp,
                      size_t temp_bytes, void* stream) {
  if (num_runs < 1 || num_runs > 2 * kMaxPtrPairs || !h_run_offsets) return NS_ERR_INVALID;
  const int64_t n = h_run_offsets[num_runs] - h_run_offsets[0];
  if (num_runs == 1 || n <= 1) return NS_OK;
  for (int r = 0; r < num_runs; ++r)
    if (h_run_offsets[r + 1] < h_run_offsets[r]) return NS_ERR_INVALID;
  if (!d_temp || temp_bytes < ns_merge_runs_temp_bytes((size_t)n, num_runs)) return NS_ERR_TEMP;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* base = d_keys + h_run_offsets[0];
  int32_t* tmp = static_cast<int32_t*>(d_temp);
  int64_t* mp = reinterpret_cast<int64_t*>(static_cast<char*>(d_temp) + align_up(n * 4, 256));

  std::vector<int64_t> runs(h_run_offsets, h_run_offsets + num_runs + 1);
  for (auto& r : runs) r -= h_run_offsets[0];
  int rounds = 0;
  for (int k = num_runs; k > 1; k = (k + 1) / 2) ++rounds;
  // Pick the first destination so that the last round lands in d_keys.
  int32_t* cur = base;
  int32_t* other = tmp;
  if (rounds & 1) {
    // odd round count: start by staging into tmp so the final write hits base
    NSB_TRY(check_cuda(cudaMemcpyAsync(tmp, base, n * 4, cudaMemcpyDeviceToDevice, s), "copy"));
    cur = tmp;
    other = base;
  }
  while (runs.size() > 2) {
    const int nr = (int)runs.size() - 1;
    PtrPairTable t{};
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

}  // extern "C"
