// quicksort.cu — the quick-sort layer on sm_100a.
//
// Replaces /root/reference/proj/include/netsort/hybrid.hpp:105-150
// (median_of_three + hoare_partition + quick_sort_rec).  A single pivot and
// a two-cursor scan are inherently sequential, so the GPU partition step uses
// B-1 sampled splitters at once (a many-pivot quick sort, i.e. sample sort):
//   1. sample_kernel      : S = 16*B regularly spaced (jittered) keys;
//   2. the samples are sorted on chip and B-1 splitters picked at regular
//      ranks (the many-pivot analogue of median-of-three: a pivot is a
//      sample median, so sorted input still splits evenly);
//   3. count_kernel       : every key is classified into one of 2B-1 buckets
//      — "between" buckets (s[j-1] < k < s[j]) and "equal" buckets (k ==
//      s[j]); equal buckets are constant, which keeps heavy duplicates from
//      unbalancing the recursion (the job hoare_partition's j==high fix-up
//      does for a single pivot, hybrid.hpp:130);
//   4. scatter_kernel     : keys move to their bucket (warp-aggregated
//      atomics reserve slots);
//   5. bucket_sort_kernel : every bucket that fits one CTA is sorted on chip
//      by cta_sort with the config's network base case (try_base_case,
//      hybrid.hpp:48-56); larger buckets recurse (quick_sort_rec).
// Parity with the reference is on the sorted bytes, which are unique.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "mergesort.cuh"

namespace nsb {

constexpr int kQsMaxB = 4096;        // splitter slots (B-1 used, last is +inf pad)
constexpr int kQsOversample = 16;    // samples per bucket
constexpr int kQsTarget = 4096;      // target mean bucket size
constexpr int kQsNT = 512;
constexpr int kQsChunk = kQsNT * 32;  // keys per CTA in count / scatter
constexpr int kQsLut = 4096;          // prefix table slots

struct QsAux {  // carved from the caller's scratch, after the n-key buffer
  int32_t* samples;     // kQsMaxB * kQsOversample
  void* sample_temp;    // merge_sort_temp(samples)
  size_t sample_temp_bytes;
  int32_t* splitters;   // kQsMaxB
  uint32_t* totals;     // 2*kQsMaxB
  unsigned long long* fill;  // 2*kQsMaxB
  int64_t* jobs;        // 2 * 2*kQsMaxB
  int16_t* lut;         // kQsLut + 1 entries + {base, shift} header
};

static size_t qs_aux_bytes() {
  const size_t S = (size_t)kQsMaxB * kQsOversample;
  return align_up(S * 4, 256) + align_up(merge_sort_temp(S), 256) + align_up(kQsMaxB * 4, 256) +
         align_up(2 * kQsMaxB * 4, 256) + align_up(2 * kQsMaxB * 8, 256) +
         align_up(4 * kQsMaxB * 8, 256) + align_up((kQsLut + 1) * 2 + 16, 256);
}

static QsAux carve_aux(char* p) {
  QsAux a;
  const size_t S = (size_t)kQsMaxB * kQsOversample;
  a.samples = reinterpret_cast<int32_t*>(p);
  p += align_up(S * 4, 256);
  a.sample_temp = p;
  a.sample_temp_bytes = merge_sort_temp(S);
  p += align_up(a.sample_temp_bytes, 256);
  a.splitters = reinterpret_cast<int32_t*>(p);
  p += align_up(kQsMaxB * 4, 256);
  a.totals = reinterpret_cast<uint32_t*>(p);
  p += align_up(2 * kQsMaxB * 4, 256);
  a.fill = reinterpret_cast<unsigned long long*>(p);
  p += align_up(2 * kQsMaxB * 8, 256);
  a.jobs = reinterpret_cast<int64_t*>(p);
  p += align_up(4 * kQsMaxB * 8, 256);
  a.lut = reinterpret_cast<int16_t*>(p);
  return a;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void sample_kernel(const int32_t* __restrict__ keys, int64_t n, int S,
                              int32_t* __restrict__ samples) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int64_t stride = n / S;
  const int64_t pos = (int64_t)i * stride + (stride > 1 ? hash32((uint32_t)i) % stride : 0);
  samples[i] = keys[pos];
}

// spl[j] = samples[(j+1)*S/B - 1] for j < B-1; spl[B-1] = INT_MAX (pad).
__global__ void splitter_kernel(const int32_t* __restrict__ samples, int S, int B,
                                int32_t* __restrict__ spl) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B) return;
  spl[j] = j < B - 1 ? samples[(int64_t)(j + 1) * S / B - 1] : INT_MAX;
}

// Prefix lookup table that shortcuts the splitter search: keys are bucketed
// by (key - base) >> shift into kQsLut slots spanning [spl[0], spl[B-2]];
// lut[p] = number of splitters < base + (p << shift).  A key's lower_bound
// then lies in [lut[p], lut[p+1]] (p < kQsLut-1) — usually 0..2 candidates —
// instead of needing log2(B) dependent shared-memory loads.  Layout in global:
// int32 header {base, shift} then kQsLut+1 int16 entries.
__global__ void lut_kernel(const int32_t* __restrict__ spl, int B, int16_t* __restrict__ lut) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > kQsLut) return;
  const int32_t base = spl[0];
  const int64_t span = (int64_t)spl[max(B - 2, 0)] - base + 1;
  int shift = 0;
  while ((span >> shift) > kQsLut) ++shift;
  if (p == 0) {
    int32_t* hdr = reinterpret_cast<int32_t*>(lut);
    hdr[0] = base;
    hdr[1] = shift;
  }
  const int64_t bound = (int64_t)base + ((int64_t)p << shift);
  int lo = 0, hi = B - 1;  // lower_bound over the B-1 real splitters
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)spl[mid] < bound) lo = mid + 1;
    else hi = mid;
  }
  lut[8 + p] = (int16_t)lo;
}

struct Classifier {
  const int32_t* spl;  // smem, B entries (spl[B-1] = +inf pad)
  const int16_t* lut;  // smem, kQsLut+1 entries
  int B;
  int32_t base;
  int shift;
  // equal/between bucket id in [0, 2B-1)
  __device__ __forceinline__ int operator()(int32_t key) const {
    const int64_t d = (int64_t)key - base;
    int lo, hi;
    if (d < 0) {
      lo = hi = 0;
    } else {
      const int64_t pp = d >> shift;
      if (pp >= kQsLut - 1) {
        lo = lut[kQsLut - 1];
        hi = B - 1;
      } else {
        lo = lut[pp];
        hi = lut[pp + 1];
      }
    }
    while (lo < hi) {  // lower_bound in spl[lo..hi)
      const int mid = (lo + hi) >> 1;
      if (spl[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    return (lo < B - 1 && spl[lo] == key) ? 2 * lo + 1 : 2 * lo;
  }
};

__device__ __forceinline__ Classifier load_classifier(int32_t* sm, const int32_t* gspl,
                                                      const int16_t* glut, int B) {
  int32_t* spl = sm;
  int16_t* lut = reinterpret_cast<int16_t*>(sm + B);
  for (int i = threadIdx.x; i < B; i += blockDim.x) spl[i] = gspl[i];
  for (int i = threadIdx.x; i <= kQsLut; i += blockDim.x) lut[i] = glut[8 + i];
  const int32_t* hdr = reinterpret_cast<const int32_t*>(glut);
  return Classifier{spl, lut, B, hdr[0], hdr[1]};
}

constexpr int kQsClassifierWords = kQsMaxB + (kQsLut + 2) / 2 + 2;

__global__ void __launch_bounds__(kQsNT)
    count_kernel(const int32_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ gspl,
                 const int16_t* __restrict__ glut, int B, uint32_t* __restrict__ totals) {
  extern __shared__ int32_t qsm[];
  const Classifier cls = load_classifier(qsm, gspl, glut, B);
  uint32_t* hist = reinterpret_cast<uint32_t*>(qsm + kQsClassifierWords);
  const int NB = 2 * B - 1;
  for (int i = threadIdx.x; i < NB; i += kQsNT) hist[i] = 0;
  __syncthreads();
  const int64_t c0 = (int64_t)blockIdx.x * kQsChunk;
  const int64_t c1 = min(n, c0 + kQsChunk);
  const int lane = threadIdx.x & 31;
  for (int64_t i = c0 + threadIdx.x; i - threadIdx.x < c1; i += kQsNT) {
    const bool live = i < c1;
    const int b = live ? cls(__ldg(keys + i)) : -1;
    const unsigned peers = __match_any_sync(kFull, b);
    if (live && lane == __ffs(peers) - 1) atomicAdd(&hist[b], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += kQsNT)
    if (hist[i]) atomicAdd(&totals[i], hist[i]);
}

// Scatter with one global reservation per (CTA, bucket): the CTA classifies
// its chunk once (bucket ids stay in registers), builds a shared-memory
// histogram, reserves each non-empty bucket's range with ONE global atomic,
// then places every key at base + warp-aggregated shared-memory rank.
constexpr int kQsPer = 16;                  // keys per thread in scatter
constexpr int kQsSChunk = kQsPer * kQsNT;  // keys per CTA in scatter

__global__ void __launch_bounds__(kQsNT)
    scatter_kernel(const int32_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ gspl,
                   const int16_t* __restrict__ glut, int B, unsigned long long* __restrict__ fill,
                   int32_t* __restrict__ out) {
  extern __shared__ int32_t qsm[];
  const Classifier cls = load_classifier(qsm, gspl, glut, B);
  unsigned long long* pos =
      reinterpret_cast<unsigned long long*>(qsm + ((kQsClassifierWords + 3) & ~1));  // 8-byte aligned
  const int NB = 2 * B - 1;
  for (int i = threadIdx.x; i < NB; i += kQsNT) pos[i] = 0;
  __syncthreads();
  const int64_t c0 = (int64_t)blockIdx.x * kQsSChunk;
  const int lane = threadIdx.x & 31;
  int32_t k[kQsPer];
  int bk[kQsPer];
#pragma unroll
  for (int u = 0; u < kQsPer; ++u) {
    const int64_t i = c0 + u * kQsNT + threadIdx.x;
    k[u] = i < n ? __ldcs(keys + i) : 0;
  }
#pragma unroll
  for (int u = 0; u < kQsPer; ++u) {
    const int64_t i = c0 + u * kQsNT + threadIdx.x;
    bk[u] = i < n ? cls(k[u]) : -1;
    const unsigned peers = __match_any_sync(kFull, bk[u]);
    if (bk[u] >= 0 && lane == __ffs(peers) - 1) atomicAdd(&pos[bk[u]], (unsigned long long)__popc(peers));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += kQsNT) {
    const unsigned long long c = pos[b];
    if (c) pos[b] = atomicAdd(&fill[b], c);  // one global atomic per (CTA, bucket)
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kQsPer; ++u) {
    const int b = bk[u];
    const unsigned peers = __match_any_sync(kFull, b);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (b >= 0 && lane == leader) base = atomicAdd(&pos[b], (unsigned long long)__popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (b >= 0) out[base + __popc(peers & ((1u << lane) - 1))] = k[u];
  }
}

// One CTA per job (start, len <= T): sorts src[start..start+len) into dst.
template <int NT, int K, int LEAF>
__global__ void __launch_bounds__(NT)
    bucket_sort_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                       const int64_t* __restrict__ jobs) {
  extern __shared__ __align__(16) int32_t sm[];
  const int64_t start = jobs[2 * blockIdx.x];
  const int len = (int)jobs[2 * blockIdx.x + 1];
  cta_sort<NT, K, LEAF>(src + start, dst + start, len, sm);
}

template <int NT, int K, int LEAF>
static int launch_bucket_sort(const int32_t* src, int32_t* dst, const int64_t* jobs, int njobs,
                              cudaStream_t s) {
  if (njobs == 0) return NS_OK;
  constexpr int smem = padded_words(NT * K) * 4;
  auto* kern = bucket_sort_kernel<NT, K, LEAF>;
  static bool attr_set = false;
  if (!attr_set) {
    NSB_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            smem),
                       "cudaFuncSetAttribute(bucket_sort)"));
    attr_set = true;
  }
  {
    Prof prof(PK_QS_BUCKET, s);
    kern<<<njobs, NT, smem, s>>>(src, dst, jobs);
  }
  return check_launch("bucket_sort_kernel");
}

static int small_sort(int32_t* d_keys, size_t n, int leaf, cudaStream_t s) {
  // n <= kSmallTile: one CTA, in place (merge_sort_device's single-CTA path)
  return merge_sort_device(d_keys, n, leaf, nullptr, 0, s);
}

// Sorts keys[0..n) in place; tmp holds n keys of scratch; aux is reused by
// recursive calls only after this level has enqueued all its work.
static int quick_sort_level(int32_t* keys, int32_t* tmp, size_t n, int leaf, const QsAux& aux,
                            cudaStream_t s) {
  if (n <= (size_t)kSmallTile) return small_sort(keys, n, leaf, s);
  int B = 2;
  while (B < kQsMaxB && (size_t)B * kQsTarget < n) B *= 2;
  const int S = B * kQsOversample;
  const int NB = 2 * B - 1;

  {
    Prof prof(PK_QS_SAMPLE, s);
    sample_kernel<<<(S + 255) / 256, 256, 0, s>>>(keys, (int64_t)n, S, aux.samples);
  }
  NSB_TRY(check_launch("sample_kernel"));
  NSB_TRY(merge_sort_device(aux.samples, (size_t)S, 8, aux.sample_temp, aux.sample_temp_bytes, s));
  {
    Prof prof(PK_QS_SAMPLE, s);
    splitter_kernel<<<(B + 255) / 256, 256, 0, s>>>(aux.samples, S, B, aux.splitters);
  }
  NSB_TRY(check_launch("splitter_kernel"));
  {
    Prof prof(PK_QS_SAMPLE, s);
    lut_kernel<<<(kQsLut + 1 + 255) / 256, 256, 0, s>>>(aux.splitters, B, aux.lut);
  }
  NSB_TRY(check_launch("lut_kernel"));

  NSB_TRY(check_cuda(cudaMemsetAsync(aux.totals, 0, NB * sizeof(uint32_t), s), "memset"));
  const int64_t ctas = (int64_t)((n + kQsChunk - 1) / kQsChunk);
  const int count_smem = (kQsClassifierWords + NB) * 4;
  const int scatter_smem = ((kQsClassifierWords + 3) & ~1) * 4 + NB * 8;
  static bool attr_set = false;
  if (!attr_set) {
    NSB_TRY(check_cuda(cudaFuncSetAttribute(count_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (kQsClassifierWords + 2 * kQsMaxB) * 4),
                       "cudaFuncSetAttribute(count)"));
    NSB_TRY(check_cuda(cudaFuncSetAttribute(scatter_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            ((kQsClassifierWords + 3) & ~1) * 4 + 2 * kQsMaxB * 8),
                       "cudaFuncSetAttribute(scatter)"));
    attr_set = true;
  }
  {
    Prof prof(PK_QS_COUNT, s);
    count_kernel<<<(unsigned)ctas, kQsNT, count_smem, s>>>(keys, (int64_t)n, aux.splitters,
                                                           aux.lut, B, aux.totals);
  }
  NSB_TRY(check_launch("count_kernel"));

  // One device->host read per partition level: the bucket sizes drive the
  // launch plan, as the split point drives quick_sort_rec (hybrid.hpp:145-148).
  std::vector<uint32_t> totals(NB);
  NSB_TRY(check_cuda(cudaMemcpyAsync(totals.data(), aux.totals, NB * sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, s),
                     "cudaMemcpyAsync(totals)"));
  NSB_TRY(check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize"));

  std::vector<unsigned long long> starts(NB);
  unsigned long long acc = 0;
  for (int b = 0; b < NB; ++b) {
    starts[b] = acc;
    acc += totals[b];
  }
  if (acc != n) return NS_ERR_CUDA;  // classification lost keys: a device fault
  NSB_TRY(check_cuda(cudaMemcpyAsync(aux.fill, starts.data(), NB * sizeof(unsigned long long),
                                     cudaMemcpyHostToDevice, s),
                     "cudaMemcpyAsync(fill)"));
  {
    Prof prof(PK_QS_SCATTER, s);
    scatter_kernel<<<(unsigned)((n + kQsSChunk - 1) / kQsSChunk), kQsNT, scatter_smem, s>>>(
        keys, (int64_t)n, aux.splitters, aux.lut, B, aux.fill, tmp);
  }
  NSB_TRY(check_launch("scatter_kernel"));

  // Size classes: one CTA shape per class so small buckets do not pay for a
  // 16K-key tile.  Classes: <=2048, <=4096, <=8192, <=16384, larger.
  std::vector<int64_t> cls[4];
  std::vector<int> big;
  for (int b = 0; b < NB; ++b) {
    const int64_t len = totals[b];
    if (len == 0) continue;
    const int c = len <= 2048 ? 0 : len <= 4096 ? 1 : len <= 8192 ? 2 : len <= 16384 ? 3 : 4;
    if (c < 4) {
      cls[c].push_back((int64_t)starts[b]);
      cls[c].push_back(len);
    } else {
      big.push_back(b);
    }
  }
  std::vector<int64_t> jobs;
  int off[5] = {0, 0, 0, 0, 0};
  for (int c = 0; c < 4; ++c) {
    off[c] = (int)(jobs.size() / 2);
    jobs.insert(jobs.end(), cls[c].begin(), cls[c].end());
  }
  off[4] = (int)(jobs.size() / 2);
  if (!jobs.empty())
    NSB_TRY(check_cuda(cudaMemcpyAsync(aux.jobs, jobs.data(), jobs.size() * sizeof(int64_t),
                                       cudaMemcpyHostToDevice, s),
                       "cudaMemcpyAsync(jobs)"));
  NSB_TRY(with_leaf(leaf, [&](auto L) {
    constexpr int LF = decltype(L)::value;
    NSB_TRY((launch_bucket_sort<128, 16, LF>(tmp, keys, aux.jobs + 2 * off[0], off[1] - off[0], s)));
    NSB_TRY((launch_bucket_sort<256, 16, LF>(tmp, keys, aux.jobs + 2 * off[1], off[2] - off[1], s)));
    NSB_TRY((launch_bucket_sort<512, 16, LF>(tmp, keys, aux.jobs + 2 * off[2], off[3] - off[2], s)));
    return launch_bucket_sort<1024, 16, LF>(tmp, keys, aux.jobs + 2 * off[3], off[4] - off[3], s);
  }));
  // Oversized buckets: equal buckets are already sorted (constant); between
  // buckets recurse, using their own slice of tmp as scratch.
  for (int b : big) {
    const size_t st = starts[b], len = totals[b];
    NSB_TRY(check_cuda(cudaMemcpyAsync(keys + st, tmp + st, len * 4, cudaMemcpyDeviceToDevice, s),
                       "cudaMemcpyAsync(bucket)"));
    if ((b & 1) == 0) NSB_TRY(quick_sort_level(keys + st, tmp + st, len, leaf, aux, s));
  }
  return NS_OK;
}

size_t quick_sort_temp(size_t n) {
  if (n <= (size_t)kSmallTile) return 0;
  return align_up(n * 4, 256) + qs_aux_bytes();
}

}  // namespace nsb

using namespace nsb;

extern "C" {

size_t ns_quick_sort_temp_bytes(size_t n) { return quick_sort_temp(n); }

int ns_quick_sort_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream) {
  if (n > 0 && d_keys == nullptr) return NS_ERR_INVALID;
  if (n <= 1) return NS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int leaf = leaf_of(width_mask, varsort_max);
  if (n <= (size_t)kSmallTile) return small_sort(d_keys, n, leaf, s);
  if (!d_temp || temp_bytes < quick_sort_temp(n)) return NS_ERR_TEMP;
  int32_t* tmp = static_cast<int32_t*>(d_temp);
  const QsAux aux = carve_aux(static_cast<char*>(d_temp) + align_up(n * 4, 256));
  return quick_sort_level(d_keys, tmp, n, leaf, aux, s);
}

}  // extern "C"
