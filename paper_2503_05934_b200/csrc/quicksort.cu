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
#include <cstdlib>
#include <utility>
#include <climits>
#include <cstdint>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "mergesort.cuh"

namespace nsb {

constexpr int kQsMaxB = 4096;        // splitter slots (B-1 used, last is +inf pad)
#ifndef NSB_QS_OVERSAMPLE
#define NSB_QS_OVERSAMPLE 16
#endif
constexpr int kQsOversample = NSB_QS_OVERSAMPLE;  // samples per bucket
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

// Runs of equal bucket ids among consecutive lanes (consecutive keys in
// memory): one ballot finds the run heads, so a run — one lane for random
// input, the whole warp for sorted input — is charged with ONE shared-memory
// atomic by its head lane.  Equal ids in different runs of a warp just issue
// separate atomics.  (Replaces __match_any_sync, which measured as the
// bottleneck of these kernels.)  Lanes with b < 0 form their own runs and
// are skipped by the callers.
struct WarpRun {
  int head_lane;  // first lane of my run
  int len;        // my run's length (valid on every lane of the run)
  bool head;
};
__device__ __forceinline__ WarpRun warp_run(int b) {
  const int lane = threadIdx.x & 31;
  const int prev = __shfl_up_sync(kFull, b, 1);
  const bool head = lane == 0 || b != prev;
  const unsigned heads = __ballot_sync(kFull, head);
  const unsigned upto = heads & (0xffffffffu >> (31 - lane));      // heads at lanes <= mine
  const int hl = 31 - __clz(upto);
  const unsigned after = heads & ~(0xffffffffu >> (31 - lane));    // heads at lanes > mine
  const int next = after ? __ffs(after) - 1 : 32;
  return WarpRun{hl, next - hl, head};
}

// 2 CTAs/SM (<= 64 registers; the classifier + histogram take 57 KiB of
// shared memory each): measured at 112 registers and ONE CTA/SM the kernel
// ran at 25 % occupancy and 0.6 TB/s.
#ifndef NSB_QS_COUNT_MINB
#define NSB_QS_COUNT_MINB 2
#endif
__global__ void __launch_bounds__(kQsNT, NSB_QS_COUNT_MINB)
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
  constexpr int kU = kQsChunk / kQsNT;  // keys per thread
  constexpr int kG = 8;                 // loaded in groups of 8
#pragma unroll 1
  for (int g0 = 0; g0 < kU; g0 += kG) {
    int32_t k[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const int64_t i = c0 + (g0 + u) * kQsNT + threadIdx.x;
      k[u] = i < c1 ? __ldg(keys + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const int64_t i = c0 + (g0 + u) * kQsNT + threadIdx.x;
      const int b = i < c1 ? cls(k[u]) : -1;
      const WarpRun r = warp_run(b);
      if (b >= 0 && r.head) atomicAdd(&hist[b], (uint32_t)r.len);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += kQsNT)
    if (hist[i]) atomicAdd(&totals[i], hist[i]);
}

// Scatter with one global reservation per (CTA, bucket): the CTA classifies
// its chunk once (bucket ids stay in registers), builds a shared-memory
// histogram, reserves each non-empty bucket's range with ONE global atomic,
// then places every key at base + warp-aggregated shared-memory rank.
#ifndef NSB_QS_SNT
#define NSB_QS_SNT 512
#endif
constexpr int kQsSNT = NSB_QS_SNT;          // scatter threads (1024 measured no faster)
constexpr int kQsPer = 16;                  // keys per thread in scatter
constexpr int kQsSChunk = kQsPer * kQsSNT;  // keys per CTA in scatter

__global__ void __launch_bounds__(kQsSNT, 2)
    scatter_kernel(const int32_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ gspl,
                   const int16_t* __restrict__ glut, int B, uint32_t* __restrict__ fill,
                   int32_t* __restrict__ out) {
  extern __shared__ int32_t qsm[];
  const Classifier cls = load_classifier(qsm, gspl, glut, B);
  // 32-bit counters and positions: the single-level path sorts < 2^32 keys
  // (64-bit shared atomics measured as the bottleneck of this kernel)
  uint32_t* pos = reinterpret_cast<uint32_t*>(qsm + kQsClassifierWords);
  const int NB = 2 * B - 1;
  for (int i = threadIdx.x; i < NB; i += kQsSNT) pos[i] = 0;
  __syncthreads();
  const int64_t c0 = (int64_t)blockIdx.x * kQsSChunk;
  const int lane = threadIdx.x & 31;
  int32_t k[kQsPer];
  int bk[kQsPer];
#pragma unroll
  for (int u = 0; u < kQsPer; ++u) {
    const int64_t i = c0 + u * kQsSNT + threadIdx.x;
    k[u] = i < n ? __ldcs(keys + i) : 0;
  }
#pragma unroll
  for (int u = 0; u < kQsPer; ++u) {
    const int64_t i = c0 + u * kQsSNT + threadIdx.x;
    bk[u] = i < n ? cls(k[u]) : -1;
    const WarpRun r = warp_run(bk[u]);
    if (bk[u] >= 0 && r.head) atomicAdd(&pos[bk[u]], (uint32_t)r.len);
  }
  __syncthreads();
  {
    // one global reservation per (CTA, bucket); a thread's atomics are all
    // issued before any result is used, so their L2 round trips overlap
    // (one after another they were the kernel's critical path)
    constexpr int kR = (2 * kQsMaxB + kQsSNT - 1) / kQsSNT;
    uint32_t c[kR], r[kR];
#pragma unroll
    for (int q = 0; q < kR; ++q) {
      const int b = threadIdx.x + q * kQsSNT;
      c[q] = b < NB ? pos[b] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kR; ++q) r[q] = c[q] ? atomicAdd(&fill[threadIdx.x + q * kQsSNT], c[q]) : 0u;
#pragma unroll
    for (int q = 0; q < kR; ++q)
      if (c[q]) pos[threadIdx.x + q * kQsSNT] = r[q];
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kQsPer; ++u) {
    const int b = bk[u];
    const WarpRun r = warp_run(b);
    uint32_t base = 0;
    if (b >= 0 && r.head) base = atomicAdd(&pos[b], (uint32_t)r.len);
    base = __shfl_sync(kFull, base, r.head_lane);
    if (b >= 0) out[base + (lane - r.head_lane)] = k[u];
  }
}

// One CTA per job (start, len <= T): sorts src[start..start+len) into dst.
template <int NT, int K, int LEAF, class Key>
__global__ void __launch_bounds__(NT, (bs_min_blocks_tput<NT, K, Key>()))
    bucket_sort_kernel(const Key* __restrict__ src, Key* __restrict__ dst,
                       const int64_t* __restrict__ jobs) {
  extern __shared__ __align__(16) unsigned char bsm_raw[];
  Key* sm = reinterpret_cast<Key*>(bsm_raw);
  const int64_t start = jobs[2 * blockIdx.x];
  const int len = (int)jobs[2 * blockIdx.x + 1];
  cta_sort<NT, K, LEAF>(src + start, dst + start, len, sm);
}

template <int NT, int K, int LEAF, class Key>
static int launch_bucket_sort(const Key* src, Key* dst, const int64_t* jobs, int njobs,
                              cudaStream_t s) {
  if (njobs == 0) return NS_OK;
  constexpr int smem = tile_smem_bytes<NT, K, Key>();
  auto* kern = bucket_sort_kernel<NT, K, LEAF, Key>;
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(kern), smem,
                           "cudaFuncSetAttribute(bucket_sort)"));
  {
    Prof prof(PK_QS_BUCKET, s);
    kern<<<njobs, NT, smem, s>>>(src, dst, jobs);
  }
  return check_launch("bucket_sort_kernel");
}

// Job classes 1..3 (buckets of <= 4096, 8192, 16384 keys; class 0 is launched
// by the caller with <128,16>): int32 tiles as 32 keys per thread when
// seg_k32_enabled(), else 16.
template <int LF, class Key>
static int bucket_sort_classes(const Key* src, Key* dst, const int64_t* jobs, const int* off,
                               cudaStream_t s) {
  if (std::is_same_v<Key, int32_t> && seg_k32_enabled()) {
    NSB_TRY((launch_bucket_sort<128, 32, LF>(src, dst, jobs + 2 * off[1], off[2] - off[1], s)));
    NSB_TRY((launch_bucket_sort<256, 32, LF>(src, dst, jobs + 2 * off[2], off[3] - off[2], s)));
    return launch_bucket_sort<512, 32, LF>(src, dst, jobs + 2 * off[3], off[4] - off[3], s);
  }
  NSB_TRY((launch_bucket_sort<256, 16, LF>(src, dst, jobs + 2 * off[1], off[2] - off[1], s)));
  NSB_TRY((launch_bucket_sort<512, 16, LF>(src, dst, jobs + 2 * off[2], off[3] - off[2], s)));
  return launch_bucket_sort<1024, 16, LF>(src, dst, jobs + 2 * off[3], off[4] - off[3], s);
}

// n <= kSmallTile at the top level: the merge sort (one CTA up to 8192
// keys, else two tiles and a merge pass in the caller's scratch, which
// quick_sort_temp sizes for it).
template <class Key>
static int small_sort(Key* d_keys, size_t n, int leaf, void* d_temp, size_t temp_bytes,
                      cudaStream_t s) {
  return merge_sort_device(d_keys, n, leaf, d_temp, temp_bytes, s);
}

// Leaf jobs of a partition level.  Consecutive buckets hold disjoint,
// ascending key ranges, so a run of NEIGHBOURING buckets sorted as one tile
// is each bucket sorted: small buckets are packed greedily into tiles of up
// to kPackKeys keys, which removes the per-bucket tile padding (buckets of
// ~4 K keys in 4 K/8 K tiles wasted about a third of the bucket-sort work).
// Jobs are grouped by tile size class: <=2048, <=4096, <=8192, <=16384 keys.
constexpr int64_t kPackKeys = 8192;
struct JobPacker {
  std::vector<int64_t> cls[4];
  int64_t js = 0, jl = 0;
  static int class_of(int64_t len) { return len <= 2048 ? 0 : len <= 4096 ? 1 : len <= 8192 ? 2 : 3; }
  void flush() {
    if (jl > 0) {
      auto& c = cls[class_of(jl)];
      c.push_back(js);
      c.push_back(jl);
    }
    jl = 0;
  }
  // bucket [st, st+len), len <= kSmallTile
  void add(int64_t st, int64_t len) {
    if (len == 0) return;
    if (len > kPackKeys) {  // alone in the 16 K class
      flush();
      cls[3].push_back(st);
      cls[3].push_back(len);
      return;
    }
    if (jl > 0 && (js + jl != st || jl + len > kPackKeys)) flush();
    if (jl == 0) js = st;
    jl += len;
  }
};

// Sorts keys[0..n) in place; tmp holds n keys of scratch; aux is reused by
// recursive calls only after this level has enqueued all its work.
static int quick_sort_level(int32_t* keys, int32_t* tmp, size_t n, int leaf, const QsAux& aux,
                            cudaStream_t s) {
  if (n <= (size_t)kSmallTile) return merge_sort_device(keys, n, leaf, nullptr, 0, s);  // one CTA
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
  const int scatter_smem = (kQsClassifierWords + NB) * 4;
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(count_kernel),
                           (kQsClassifierWords + 2 * kQsMaxB) * 4, "cudaFuncSetAttribute(count)"));
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(scatter_kernel),
                           (kQsClassifierWords + 2 * kQsMaxB) * 4,
                           "cudaFuncSetAttribute(scatter)"));
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

  std::vector<uint32_t> starts(NB);
  uint64_t acc = 0;
  for (int b = 0; b < NB; ++b) {
    starts[b] = (uint32_t)acc;
    acc += totals[b];
  }
  if (acc != n) return NS_ERR_CUDA;  // classification lost keys: a device fault
  NSB_TRY(check_cuda(cudaMemcpyAsync(aux.fill, starts.data(), NB * sizeof(uint32_t),
                                     cudaMemcpyHostToDevice, s),
                     "cudaMemcpyAsync(fill)"));
  {
    Prof prof(PK_QS_SCATTER, s);
    scatter_kernel<<<(unsigned)((n + kQsSChunk - 1) / kQsSChunk), kQsSNT, scatter_smem, s>>>(
        keys, (int64_t)n, aux.splitters, aux.lut, B, reinterpret_cast<uint32_t*>(aux.fill), tmp);
  }
  NSB_TRY(check_launch("scatter_kernel"));

  // Size classes: one CTA shape per class so small buckets do not pay for a
  // 16K-key tile.  Classes: <=2048, <=4096, <=8192, <=16384, larger.
  JobPacker pk;
  std::vector<int> big;
  for (int b = 0; b < NB; ++b) {
    const int64_t len = totals[b];
    if (len == 0) continue;
    if (len <= kSmallTile) {
      pk.add((int64_t)starts[b], len);
    } else {
      pk.flush();
      big.push_back(b);
    }
  }
  pk.flush();
  auto& cls = pk.cls;
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
    return bucket_sort_classes<LF>(tmp, keys, aux.jobs, off, s);
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

// ===========================================================================
// Multi-level, multi-segment partition (default).  Every level partitions ALL
// oversized segments at once with at most 256 splitters per segment, so the
// count/scatter kernels stay cheap (8-step search, <= 511 buckets, coalesced
// ~32-key runs per bucket per CTA) and a whole level costs one host read,
// instead of one per bucket.  Segments ping-pong between the key buffer and
// tmp at fixed positions; buckets that fit one CTA are sorted straight into
// the key buffer (jobs), constant "equal" buckets are copied, the rest form
// the next level's segments.  Random input of 16M keys: 2 levels.
// ===========================================================================
constexpr int kMlMaxB = 256;

struct MlSeg {
  int64_t start, len;
  int B, spl_off, cnt_off;
  int64_t chunk0;  // first count/scatter chunk of this segment
  int64_t smp_off;
};

template <class Key>
struct MlAux {
  MlSeg* segs;
  Key* samples;
  Key* spl;
  uint32_t* counts;
  unsigned long long* fill;
  int64_t* jobs;
  size_t max_segs, max_samples, max_spl, max_cnt, max_jobs;
};

static size_t ml_max_segs(size_t n) { return n / (kSmallTile + 1) + 4; }
static size_t ml_max_spl(size_t n) { return n / 2048 + 2 * kMlMaxB * ml_max_segs(n) / 64 + 1024; }

static size_t ml_aux_bytes(size_t n, size_t kb = 4) {
  const size_t segs = ml_max_segs(n), spl = n / 2048 + 512 * segs / 64 + 4096;
  return align_up(segs * sizeof(MlSeg), 256) + align_up(16 * spl * kb, 256) +
         align_up(spl * kb, 256) + align_up(2 * spl * 4, 256) + align_up(2 * spl * 8, 256) +
         align_up(2 * (2 * spl + segs) * 8, 256);
}

template <class Key>
static MlAux<Key> carve_ml(char* p, size_t n) {
  MlAux<Key> a;
  a.max_segs = ml_max_segs(n);
  a.max_spl = n / 2048 + 512 * a.max_segs / 64 + 4096;
  a.max_samples = 16 * a.max_spl;
  a.max_cnt = 2 * a.max_spl;
  a.max_jobs = 2 * a.max_spl + a.max_segs;
  a.segs = reinterpret_cast<MlSeg*>(p);
  p += align_up(a.max_segs * sizeof(MlSeg), 256);
  a.samples = reinterpret_cast<Key*>(p);
  p += align_up(a.max_samples * sizeof(Key), 256);
  a.spl = reinterpret_cast<Key*>(p);
  p += align_up(a.max_spl * sizeof(Key), 256);
  a.counts = reinterpret_cast<uint32_t*>(p);
  p += align_up(a.max_cnt * 4, 256);
  a.fill = reinterpret_cast<unsigned long long*>(p);
  p += align_up(a.max_cnt * 8, 256);
  a.jobs = reinterpret_cast<int64_t*>(p);
  return a;
}

__device__ __forceinline__ int seg_of_chunk(const MlSeg* segs, int nseg, int64_t c) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].chunk0 <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int seg_of_sample(const MlSeg* segs, int nseg, int64_t i) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].smp_off <= i) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <class Key>
__global__ void ml_sample_kernel(const Key* __restrict__ X, const MlSeg* __restrict__ segs,
                                 int nseg, int64_t total, Key* __restrict__ samples) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const MlSeg sg = segs[seg_of_sample(segs, nseg, i)];
  const int S = kQsOversample * sg.B;
  const int64_t j = i - sg.smp_off;
  const int64_t stride = sg.len / S;
  const int64_t pos = j * stride + (stride > 1 ? hash32((uint32_t)j) % stride : 0);
  samples[i] = X[sg.start + pos];
}

template <class Key>
__global__ void ml_splitter_kernel(const Key* __restrict__ samples,
                                   const MlSeg* __restrict__ segs, int nseg,
                                   Key* __restrict__ spl) {
  const int sgi = blockIdx.x;
  if (sgi >= nseg) return;
  const MlSeg sg = segs[sgi];
  const int S = kQsOversample * sg.B;
  for (int j = threadIdx.x; j < sg.B; j += blockDim.x)
    spl[sg.spl_off + j] =
        j < sg.B - 1 ? samples[sg.smp_off + (int64_t)(j + 1) * S / sg.B - 1] : KeyT<Key>::kMax;
}

template <int LOGB, class Key>
__device__ __forceinline__ int ml_classify(const Key* spl, Key key) {
  constexpr int B = 1 << LOGB;
  int j = 0;
#pragma unroll
  for (int step = B >> 1; step >= 1; step >>= 1)
    if (spl[j + step - 1] < key) j += step;
  return (j < B - 1 && spl[j] == key) ? 2 * j + 1 : 2 * j;
}

constexpr int kMlNT = 512, kMlPer = 16, kMlChunk = kMlNT * kMlPer;

// Per-warp private histograms: a warp's lanes that share a bucket are
// combined with __match_any_sync and one lane updates the warp's own row, so
// no shared-memory atomics contend (with only 2B-1 <= 511 buckets, 16 warps
// hammering one shared histogram serialised on the atomic unit).
constexpr int kMlWarps = kMlNT / 32;

// Lanes of the warp holding the same bucket id, from one ballot per id bit
// (cheaper than __match_any_sync, which measured as the bottleneck of the
// count/scatter kernels).  Ids are < 2^nbits; an invalid lane passes -1 and
// lands in the all-ones group, which callers never use as a real id.
template <int NBITS>
__device__ __forceinline__ unsigned warp_peers(int b) {
  unsigned m = kFull;
#pragma unroll
  for (int i = 0; i < NBITS; ++i) {
    const bool bit = (b >> i) & 1;
    const unsigned bal = __ballot_sync(kFull, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

// Per-CTA bucket histogram: runs of equal ids among consecutive lanes are
// found with one ballot (warp_run) and charged with ONE shared atomic by the
// run's head lane; equal ids in different runs just add separately.
template <int LOGB, class Key>
__device__ __forceinline__ void ml_hist(const Key* spl, const Key (&k)[kMlPer],
                                        int (&bk)[kMlPer], int64_t c0, int64_t c1,
                                        uint32_t* hist) {
#pragma unroll
  for (int u = 0; u < kMlPer; ++u) {
    const int64_t i = c0 + u * kMlNT + threadIdx.x;
    bk[u] = i < c1 ? ml_classify<LOGB>(spl, k[u]) : -1;
    const WarpRun r = warp_run(bk[u]);
    if (bk[u] >= 0 && r.head) atomicAdd(&hist[bk[u]], (uint32_t)r.len);
  }
}

template <int LOGB, class Key>
__device__ __noinline__ void ml_count_body(const Key* __restrict__ X, const MlSeg& sg,
                                              const Key* spl, uint32_t* hist,
                                              uint32_t* __restrict__ counts) {
  const int NB = 2 * sg.B - 1;
  const int64_t c0 = sg.start + (blockIdx.x - sg.chunk0) * (int64_t)kMlChunk;
  const int64_t c1 = min(sg.start + sg.len, c0 + kMlChunk);
  Key k[kMlPer];
  int bk[kMlPer];
#pragma unroll
  for (int u = 0; u < kMlPer; ++u) {
    const int64_t i = c0 + u * kMlNT + threadIdx.x;
    k[u] = i < c1 ? __ldg(X + i) : 0;
  }
  ml_hist<LOGB>(spl, k, bk, c0, c1, hist);
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += kMlNT) {
    const uint32_t t = hist[b];
    if (t) atomicAdd(&counts[sg.cnt_off + b], t);
  }
}

#define NSB_LOGB_DISPATCH(B, CALL)        \
  switch (B) {                            \
    case 2: CALL(1); break;               \
    case 4: CALL(2); break;               \
    case 8: CALL(3); break;               \
    case 16: CALL(4); break;              \
    case 32: CALL(5); break;              \
    case 64: CALL(6); break;              \
    case 128: CALL(7); break;             \
    default: CALL(8); break;              \
  }

template <class Key>
__global__ void __launch_bounds__(kMlNT, 2)
    ml_count_kernel(const Key* __restrict__ X, const MlSeg* __restrict__ segs, int nseg,
                    const Key* __restrict__ gspl, uint32_t* __restrict__ counts) {
  __shared__ Key spl[kMlMaxB];
  __shared__ uint32_t hist[2 * kMlMaxB];
  const MlSeg sg = segs[seg_of_chunk(segs, nseg, blockIdx.x)];
  for (int i = threadIdx.x; i < sg.B; i += kMlNT) spl[i] = gspl[sg.spl_off + i];
  for (int i = threadIdx.x; i < 2 * sg.B - 1; i += kMlNT) hist[i] = 0;
  __syncthreads();
#define NSB_COUNT_CALL(L) ml_count_body<L>(X, sg, spl, hist, counts)
  NSB_LOGB_DISPATCH(sg.B, NSB_COUNT_CALL)
#undef NSB_COUNT_CALL
}

template <int LOGB, class Key>
__device__ __noinline__ void ml_scatter_body(const Key* __restrict__ X, const MlSeg& sg,
                                                const Key* spl, uint32_t* hist,
                                                unsigned long long* __restrict__ fill,
                                                Key* __restrict__ Y) {
  const int NB = 2 * sg.B - 1;
  const int lane = threadIdx.x & 31;
  const int64_t c0 = sg.start + (blockIdx.x - sg.chunk0) * (int64_t)kMlChunk;
  const int64_t c1 = min(sg.start + sg.len, c0 + kMlChunk);
  Key k[kMlPer];
  int bk[kMlPer];
#pragma unroll
  for (int u = 0; u < kMlPer; ++u) {
    const int64_t i = c0 + u * kMlNT + threadIdx.x;
    k[u] = i < c1 ? __ldcs(X + i) : 0;
  }
  ml_hist<LOGB>(spl, k, bk, c0, c1, hist);
  __syncthreads();
  // one global reservation per (CTA, bucket); cursors relative to the segment
  for (int b = threadIdx.x; b < NB; b += kMlNT) {
    const uint32_t t = hist[b];
    if (t)
      hist[b] = (uint32_t)(atomicAdd(&fill[sg.cnt_off + b], (unsigned long long)t) -
                           (unsigned long long)sg.start);
  }
  __syncthreads();
  Key* Ys = Y + sg.start;
#pragma unroll
  for (int u = 0; u < kMlPer; ++u) {
    const int b = bk[u];
    const WarpRun r = warp_run(b);
    uint32_t base = 0;
    if (b >= 0 && r.head) base = atomicAdd(&hist[b], (uint32_t)r.len);
    base = __shfl_sync(kFull, base, r.head_lane);
    if (b >= 0) Ys[base + (lane - r.head_lane)] = k[u];
  }
}

template <class Key>
__global__ void __launch_bounds__(kMlNT, 2)
    ml_scatter_kernel(const Key* __restrict__ X, const MlSeg* __restrict__ segs, int nseg,
                      const Key* __restrict__ gspl, unsigned long long* __restrict__ fill,
                      Key* __restrict__ Y) {
  __shared__ Key spl[kMlMaxB];
  __shared__ uint32_t hist[2 * kMlMaxB];  // counts, then cursors (relative to the segment)
  const MlSeg sg = segs[seg_of_chunk(segs, nseg, blockIdx.x)];
  for (int i = threadIdx.x; i < sg.B; i += kMlNT) spl[i] = gspl[sg.spl_off + i];
  for (int i = threadIdx.x; i < 2 * sg.B - 1; i += kMlNT) hist[i] = 0;
  __syncthreads();
#define NSB_SCATTER_CALL(L) ml_scatter_body<L>(X, sg, spl, hist, fill, Y)
  NSB_LOGB_DISPATCH(sg.B, NSB_SCATTER_CALL)
#undef NSB_SCATTER_CALL
}

// Copies jobs (start, len) from src to dst (constant "equal" buckets).
template <class Key>
__global__ void copy_jobs_kernel(const Key* __restrict__ src, Key* __restrict__ dst,
                                 const int64_t* __restrict__ jobs) {
  const int64_t st = jobs[2 * blockIdx.x], len = jobs[2 * blockIdx.x + 1];
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[st + i] = src[st + i];
}

template <class Key>
static int ml_quick_sort(Key* keys, Key* tmp, size_t n, int leaf, const MlAux<Key>& ax,
                         cudaStream_t s) {
  std::vector<std::pair<int64_t, int64_t>> cur{{0, (int64_t)n}};
  Key* X = keys;
  Key* Y = tmp;
  std::vector<MlSeg> segs;
  std::vector<uint32_t> counts;
  std::vector<unsigned long long> fill;
  while (!cur.empty()) {
    // ---- plan the level
    segs.clear();
    int spl = 0, cnt = 0;
    int64_t chunks = 0, smp = 0;
    for (auto [st, len] : cur) {
      MlSeg g{};
      g.start = st;
      g.len = len;
      int B = 2;
      while (B < kMlMaxB && (int64_t)B * kQsTarget < len) B *= 2;
      g.B = B;
      g.spl_off = spl;
      g.cnt_off = cnt;
      g.chunk0 = chunks;
      g.smp_off = smp;
      spl += B;
      cnt += 2 * B - 1;
      chunks += (len + kMlChunk - 1) / kMlChunk;
      smp += kQsOversample * B;
      segs.push_back(g);
    }
    const int nseg = (int)segs.size();
    if ((size_t)nseg > ax.max_segs || (size_t)spl > ax.max_spl || (size_t)cnt > ax.max_cnt ||
        (size_t)smp > ax.max_samples)
      return NS_ERR_TEMP;
    NSB_TRY(check_cuda(cudaMemcpyAsync(ax.segs, segs.data(), nseg * sizeof(MlSeg),
                                       cudaMemcpyHostToDevice, s),
                       "H2D(segs)"));
    // ---- splitters: sample, sort each segment's samples on chip, pick
    {
      Prof prof(PK_QS_SAMPLE, s);
      ml_sample_kernel<Key><<<(unsigned)((smp + 255) / 256), 256, 0, s>>>(X, ax.segs, nseg, smp,
                                                                       ax.samples);
    }
    NSB_TRY(check_launch("ml_sample_kernel"));
    std::vector<int64_t> sjobs;
    for (const auto& g : segs) {
      sjobs.push_back(g.smp_off);
      sjobs.push_back(kQsOversample * g.B);
    }
    NSB_TRY(check_cuda(cudaMemcpyAsync(ax.jobs, sjobs.data(), sjobs.size() * 8,
                                       cudaMemcpyHostToDevice, s),
                       "H2D(sample jobs)"));
    NSB_TRY((launch_bucket_sort<256, 16, 8>(ax.samples, ax.samples, ax.jobs, nseg, s)));
    {
      Prof prof(PK_QS_SAMPLE, s);
      ml_splitter_kernel<Key><<<nseg, 256, 0, s>>>(ax.samples, ax.segs, nseg, ax.spl);
    }
    NSB_TRY(check_launch("ml_splitter_kernel"));
    // ---- count
    NSB_TRY(check_cuda(cudaMemsetAsync(ax.counts, 0, cnt * 4, s), "memset"));
    {
      Prof prof(PK_QS_COUNT, s);
      ml_count_kernel<Key><<<(unsigned)chunks, kMlNT, 0, s>>>(X, ax.segs, nseg, ax.spl, ax.counts);
    }
    NSB_TRY(check_launch("ml_count_kernel"));
    // One device->host read per LEVEL: bucket sizes drive the plan, as the
    // split point drives quick_sort_rec (hybrid.hpp:145-148).
    counts.resize(cnt);
    NSB_TRY(check_cuda(cudaMemcpyAsync(counts.data(), ax.counts, cnt * 4, cudaMemcpyDeviceToHost,
                                       s),
                       "D2H(counts)"));
    NSB_TRY(check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize"));
    // ---- plan buckets: fill positions, jobs, next level
    fill.resize(cnt);
    JobPacker pk;
    std::vector<int64_t> copies;
    std::vector<std::pair<int64_t, int64_t>> next;
    for (const auto& g : segs) {
      int64_t acc = g.start;
      const int NB = 2 * g.B - 1;
      for (int b = 0; b < NB; ++b) {
        const int64_t len = counts[g.cnt_off + b];
        fill[g.cnt_off + b] = (unsigned long long)acc;
        if (len > 0) {
          if (len <= kSmallTile) {
            // leaf (a constant bucket too: sorting it from Y is its copy)
            pk.add(acc, len);
          } else if (b & 1) {  // large constant bucket: already sorted
            pk.flush();
            if (Y != keys) {
              copies.push_back(acc);
              copies.push_back(len);
            }
          } else {
            pk.flush();
            next.push_back({acc, len});
          }
        }
        acc += len;
      }
      if (acc != g.start + g.len) return NS_ERR_CUDA;  // lost keys: a device fault
    }
    NSB_TRY(check_cuda(cudaMemcpyAsync(ax.fill, fill.data(), cnt * 8, cudaMemcpyHostToDevice, s),
                       "H2D(fill)"));
    {
      Prof prof(PK_QS_SCATTER, s);
      ml_scatter_kernel<Key><<<(unsigned)chunks, kMlNT, 0, s>>>(X, ax.segs, nseg, ax.spl, ax.fill, Y);
    }
    NSB_TRY(check_launch("ml_scatter_kernel"));
    pk.flush();
    auto& cls = pk.cls;
    // ---- leaf buckets -> key buffer
    std::vector<int64_t> jobs;
    int off[6] = {0, 0, 0, 0, 0, 0};
    for (int c = 0; c < 4; ++c) {
      off[c] = (int)(jobs.size() / 2);
      jobs.insert(jobs.end(), cls[c].begin(), cls[c].end());
    }
    off[4] = (int)(jobs.size() / 2);
    jobs.insert(jobs.end(), copies.begin(), copies.end());
    off[5] = (int)(jobs.size() / 2);
    if ((size_t)off[5] > ax.max_jobs) return NS_ERR_TEMP;
    if (!jobs.empty())
      NSB_TRY(check_cuda(cudaMemcpyAsync(ax.jobs, jobs.data(), jobs.size() * 8,
                                         cudaMemcpyHostToDevice, s),
                         "H2D(jobs)"));
    NSB_TRY(with_leaf(leaf, [&](auto L) {
      constexpr int LF = decltype(L)::value;
      NSB_TRY((launch_bucket_sort<128, 16, LF>(Y, keys, ax.jobs + 2 * off[0], off[1] - off[0], s)));
      return bucket_sort_classes<LF>(Y, keys, ax.jobs, off, s);
    }));
    if (off[5] > off[4]) {
      copy_jobs_kernel<Key><<<off[5] - off[4], 256, 0, s>>>(Y, keys, ax.jobs + 2 * off[4]);
      NSB_TRY(check_launch("copy_jobs_kernel"));
    }
    // the jobs/fill/segs buffers are rewritten by the next level: the stream
    // orders that after this level's kernels; the host vectors are copied
    // by value into pageable H2D copies (staged before cudaMemcpyAsync returns)
    cur.swap(next);
    std::swap(X, Y);
  }
  return NS_OK;
}

size_t quick_sort_temp(size_t n) {
  if (n <= (size_t)kSmallTile) return merge_sort_temp(n);
  return align_up(n * 4, 256) + std::max(qs_aux_bytes(), ml_aux_bytes(n));
}

// int64 keys always take the multi-level partition (its classifier is a
// plain splitter search; the single-level prefix table is int32-specific)
size_t quick_sort_temp_i64(size_t n) {
  if (n <= (size_t)kSmallTile) return merge_sort_temp_i64(n);
  return align_up(n * 8, 256) + ml_aux_bytes(n, 8);
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
  if (n <= (size_t)kSmallTile) return small_sort(d_keys, n, leaf, d_temp, temp_bytes, s);
  if (!d_temp || temp_bytes < quick_sort_temp(n)) return NS_ERR_TEMP;
  int32_t* tmp = static_cast<int32_t*>(d_temp);
  char* auxp = static_cast<char*>(d_temp) + align_up(n * 4, 256);
  // Single level (up to 4096 splitters, measured faster while its buckets
  // fit one CTA) up to 2^25 keys; the multi-level partition above that,
  // where a single level would leave thousands of oversized buckets.
  // NSB_QS=1 / 2 forces one or the other.
  static const int mode = [] {
    const char* e = getenv("NSB_QS");
    return e ? atoi(e) : 0;
  }();
  const bool single = mode == 1 || (mode == 0 && n <= (size_t(1) << 25));
  if (single) return quick_sort_level(d_keys, tmp, n, leaf, carve_aux(auxp), s);
  return ml_quick_sort(d_keys, tmp, n, leaf, carve_ml<int32_t>(auxp, n), s);
}

size_t ns_quick_sort_temp_bytes_i64(size_t n) { return quick_sort_temp_i64(n); }

int ns_quick_sort_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream) {
  if (n > 0 && d_keys == nullptr) return NS_ERR_INVALID;
  if (n <= 1) return NS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int leaf = leaf_of(width_mask, varsort_max);
  if (n <= (size_t)kSmallTile) return small_sort(d_keys, n, leaf, d_temp, temp_bytes, s);
  if (!d_temp || temp_bytes < quick_sort_temp_i64(n)) return NS_ERR_TEMP;
  int64_t* tmp = static_cast<int64_t*>(d_temp);
  char* auxp = static_cast<char*>(d_temp) + align_up(n * 8, 256);
  return ml_quick_sort(d_keys, tmp, n, leaf, carve_ml<int64_t>(auxp, n), s);
}

}  // extern "C"
