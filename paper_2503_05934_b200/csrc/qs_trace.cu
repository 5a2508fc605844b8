// qs_trace.cu — the reference's quick sort executed node for node on the GPU.
//
// The timed quick sort (quicksort.cu) reaches the reference's OUTPUT with a
// many-pivot bucket recursion; its recursion tree is not the reference's, so
// it cannot report the reference's DispatchStats.  This file runs the
// reference's own recursion instead:
//   median_of_three  /root/reference/proj/include/netsort/hybrid.hpp:105-114
//   hoare_partition  hybrid.hpp:121-133
//   quick_sort_rec   hybrid.hpp:137-150 (try_base_case 48-56)
//   optimized_quick_sort(..., stats) hybrid.hpp:197-204, run_variant 234-243
// with the same pivot, the same swaps and the same split at every node, so
// the counters (network hits by width, partitions, max depth;
// DispatchStats, hybrid.hpp:18-34) and every intermediate arrangement are the
// reference's.
//
// Hoare partition in closed form (checked against the sequential loop in
// tests/test_oracle.py::test_hoare_closed_form).  Let L_1 < L_2 < ... be the
// positions with key >= pivot in ascending order and R_1 > R_2 > ... those
// with key <= pivot in descending order, both taken on the array as it is
// BEFORE the partition.  The k-th round of the two-cursor scan stops i at L_k
// and j at R_k as long as L_k < R_k (the cells between the cursors are
// untouched by earlier swaps), so the loop swaps exactly the pairs
// (L_k, R_k), k = 1..S, S = max{k : L_k < R_k}; the final j is
// max(R_{S+1}, L_S) and the split is j, or high-1 when j == high.  Every
// quantity is a rank or a prefix count, so a partition is two streaming
// passes (classify + compact the candidate positions, then swap S pairs) with
// no sequential scan.
//
// Schedule.  Segments longer than kTraceSmall keys are partitioned level by
// level by grid-wide kernels (median of three, count, scan, compact, find,
// swap; the host reads the splits back once per level to plan the next).
// A segment of at most kTraceSmall keys is finished by ONE CTA in shared
// memory: its 8 warps take nodes of the current level from a shared work
// list, each warp partitioning its node with ballots (compaction of the
// candidate positions, a binary search for S, the swaps), and push the
// children to the next level's list.  Base cases are sorted in place and
// counted exactly where try_base_case would count them.
//
// This is the instrumentation path (the reference's DispatchStats overload,
// not its timed NoStats path): it synchronises once per large level and is
// not graph-capturable.  It is NOT a fallback — the timed quick sort never
// calls it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "networks.cuh"

namespace nsb {
namespace {

constexpr int kTraceSmall = 8192;  // a segment up to this length is finished on chip
constexpr int kChunk = 4096;       // keys per CTA in the level kernels
constexpr int kThreads = 256;      // both kernel families
constexpr int kWarps = kThreads / 32;

struct Seg {  // one large segment of a level, inclusive bounds
  int64_t lo, hi;
};
struct Chunk {  // kChunk-key slice of a large segment
  int64_t start;
  int32_t len;
  int32_t seg;
  int32_t first;  // index of the segment's first chunk
  int32_t pad;
};
struct SmallSeg {  // segment finished by one CTA
  int64_t lo;
  int32_t len;
  int32_t depth;
};

// Counters on the device (the DispatchStats fields the CTAs accumulate).
enum { C_HITS = 0, C_PARTS = 9, C_MAXD = 10, C_NUM = 11 };

// ---------------------------------------------------------------------------
// level kernels (segments > kTraceSmall)

// median_of_three on each segment (hybrid.hpp:105-114): sorts the probed
// cells lo, mid, hi in place with the reference's three compare-exchanges.
template <class K>
__global__ void mot_kernel(K* __restrict__ a, const Seg* __restrict__ segs, int nseg,
                           K* __restrict__ piv) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int64_t lo = segs[s].lo, hi = segs[s].hi;
  if (hi - lo < 2) {
    piv[s] = a[lo];
    return;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  K x = a[lo], y = a[mid], z = a[hi];
  cx(x, y);
  cx(x, z);
  cx(y, z);
  a[lo] = x;
  a[mid] = y;
  a[hi] = z;
  piv[s] = y;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per chunk: how many keys are left candidates (>= pivot) and right
// candidates (<= pivot).
template <class K>
__global__ void __launch_bounds__(kThreads) count_kernel(const K* __restrict__ a,
                                                         const Chunk* __restrict__ ch,
                                                         const K* __restrict__ piv,
                                                         uint32_t* __restrict__ cnt) {
  const Chunk c = ch[blockIdx.x];
  const K p = piv[c.seg];
  uint32_t nl = 0, nr = 0;
  for (int i = threadIdx.x; i < c.len; i += kThreads) {
    const K v = a[c.start + i];
    nl += v >= p;
    nr += v <= p;
  }
  __shared__ uint32_t sl[kWarps], sr[kWarps];
  for (int o = 16; o; o >>= 1) {
    nl += __shfl_xor_sync(0xffffffffu, nl, o);
    nr += __shfl_xor_sync(0xffffffffu, nr, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sl[w] = nl, sr[w] = nr;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tl = 0, tr = 0;
    for (int i = 0; i < kWarps; ++i) tl += sl[i], tr += sr[i];
    cnt[2 * blockIdx.x] = tl;
    cnt[2 * blockIdx.x + 1] = tr;
  }
}

// Per segment: exclusive scan of its chunks' counts (in place) and the totals
// NL / NR.
__global__ void __launch_bounds__(kThreads) scan_kernel(const int32_t* __restrict__ first,
                                                        uint32_t* __restrict__ cnt,
                                                        int64_t* __restrict__ totals) {
  const int s = blockIdx.x;
  const int b = first[s], e = first[s + 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ uint32_t wl[kWarps], wr[kWarps];
  uint32_t runl = 0, runr = 0;
  for (int base = b; base < e; base += kThreads) {
    const int c = base + threadIdx.x;
    const uint32_t vl = c < e ? cnt[2 * c] : 0, vr = c < e ? cnt[2 * c + 1] : 0;
    uint32_t il = vl, ir = vr;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t tl = __shfl_up_sync(0xffffffffu, il, o);
      const uint32_t tr = __shfl_up_sync(0xffffffffu, ir, o);
      if (lane >= o) il += tl, ir += tr;
    }
    if (lane == 31) wl[w] = il, wr[w] = ir;
    __syncthreads();
    uint32_t pl = 0, pr = 0, tl = 0, tr = 0;
    for (int i = 0; i < kWarps; ++i) {
      if (i < w) pl += wl[i], pr += wr[i];
      tl += wl[i], tr += wr[i];
    }
    if (c < e) {
      cnt[2 * c] = runl + pl + il - vl;
      cnt[2 * c + 1] = runr + pr + ir - vr;
    }
    runl += tl;
    runr += tr;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[2 * s] = runl, totals[2 * s + 1] = runr;
}

// Per chunk: writes the segment-relative position of every left candidate at
// posL[lo + rank] (ascending) and of every right candidate at posR[lo + rank]
// (ascending; R_k is posR[lo + NR - k]).
template <class K>
__global__ void __launch_bounds__(kThreads) compact_kernel(const K* __restrict__ a,
                                                           const Chunk* __restrict__ ch,
                                                           const Seg* __restrict__ segs,
                                                           const K* __restrict__ piv,
                                                           const uint32_t* __restrict__ off,
                                                           uint32_t* __restrict__ posL,
                                                           uint32_t* __restrict__ posR) {
  const Chunk c = ch[blockIdx.x];
  const K p = piv[c.seg];
  const int64_t lo = segs[c.seg].lo;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  __shared__ uint32_t wl[kWarps], wr[kWarps];
  uint32_t basel = off[2 * blockIdx.x], baser = off[2 * blockIdx.x + 1];
  for (int r = 0; r < c.len; r += kThreads) {
    const int i = r + threadIdx.x;
    const bool ok = i < c.len;
    const K v = ok ? a[c.start + i] : K(0);
    const bool fl = ok && v >= p, fr = ok && v <= p;
    const uint32_t bl = __ballot_sync(0xffffffffu, fl), br = __ballot_sync(0xffffffffu, fr);
    if (lane == 0) wl[w] = __popc(bl), wr[w] = __popc(br);
    __syncthreads();
    uint32_t pl = 0, pr = 0, tl = 0, tr = 0;
    for (int k = 0; k < kWarps; ++k) {
      if (k < w) pl += wl[k], pr += wr[k];
      tl += wl[k], tr += wr[k];
    }
    const uint32_t rel = static_cast<uint32_t>(c.start + i - lo);
    if (fl) {
      const int64_t at = lo + basel + pl + __popc(bl & lt);
      NSB_DCHECK(at <= segs[c.seg].hi);
      posL[at] = rel;
    }
    if (fr) {
      const int64_t at = lo + baser + pr + __popc(br & lt);
      NSB_DCHECK(at <= segs[c.seg].hi);
      posR[at] = rel;
    }
    basel += tl;
    baser += tr;
    __syncthreads();
  }
}

// Per segment: S = max{k : L_k < R_k} by binary search (the predicate holds
// for a prefix of k), the final j = max(R_{S+1}, L_S) and the split.
// bad[0] is set when a segment has no left or no right candidate (the
// reference's scan would run off the range; only possible through the
// explicit-pivot entry point).
__global__ void find_kernel(const Seg* __restrict__ segs, int nseg,
                            const int64_t* __restrict__ totals, const uint32_t* __restrict__ posL,
                            const uint32_t* __restrict__ posR, int64_t* __restrict__ S_out,
                            int64_t* __restrict__ split, int* __restrict__ bad) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int64_t lo = segs[s].lo, hi = segs[s].hi;
  const int64_t NL = totals[2 * s], NR = totals[2 * s + 1];
  if (NL == 0 || NR == 0) {
    S_out[s] = 0;
    split[s] = -1;
    atomicExch(bad, 1);
    return;
  }
  int64_t a = 0, b = NL < NR ? NL : NR;
  while (a < b) {
    const int64_t m = (a + b + 1) / 2;
    if (posL[lo + m - 1] < posR[lo + NR - m]) a = m;
    else b = m - 1;
  }
  const int64_t S = a;
  int64_t j = -1;
  if (S + 1 <= NR) j = posR[lo + NR - S - 1];
  if (S >= 1) j = j > int64_t(posL[lo + S - 1]) ? j : int64_t(posL[lo + S - 1]);
  j += lo;
  S_out[s] = S;
  split[s] = j < hi ? j : hi - 1;
}

// The S swaps of each segment: chunk q of a segment performs pairs
// k = q*kChunk+1 .. (q+1)*kChunk (S <= len/2, so the chunks cover them).
template <class K>
__global__ void __launch_bounds__(kThreads) swap_kernel(K* __restrict__ a,
                                                        const Chunk* __restrict__ ch,
                                                        const Seg* __restrict__ segs,
                                                        const int64_t* __restrict__ totals,
                                                        const int64_t* __restrict__ S_in,
                                                        const uint32_t* __restrict__ posL,
                                                        const uint32_t* __restrict__ posR) {
  const Chunk c = ch[blockIdx.x];
  const int64_t lo = segs[c.seg].lo;
  const int64_t S = S_in[c.seg], NR = totals[2 * c.seg + 1];
  const int64_t k0 = int64_t(blockIdx.x - c.first) * kChunk;
  for (int i = threadIdx.x; i < kChunk; i += kThreads) {
    const int64_t k = k0 + i + 1;
    if (k > S) break;
    const int64_t x = lo + posL[lo + k - 1], y = lo + posR[lo + NR - k];
    NSB_DCHECK(x < y && y <= segs[c.seg].hi);
    const K t = a[x];
    a[x] = a[y];
    a[y] = t;
  }
}

// ---------------------------------------------------------------------------
// one-CTA finish of a segment of <= kTraceSmall keys

struct SmallShared {
  int cnt[2];
  int next;
  int maxd;
  unsigned long long hits[9];
  unsigned long long parts;
};

template <class K>
__device__ __forceinline__ void insertion_sort(K* s, int lo, int hi) {
  for (int i = lo + 1; i <= hi; ++i) {
    const K v = s[i];
    int j = i - 1;
    while (j >= lo && v < s[j]) {
      s[j + 1] = s[j];
      --j;
    }
    s[j + 1] = v;
  }
}

// The visit at the top of quick_sort_rec (hybrid.hpp:139-143): depth, then
// the base case or a partition at the next level.  One warp, uniform args.
template <class K>
__device__ __forceinline__ void visit(K* s, uint32_t* fr, SmallShared& sh, int slot, int lo, int hi,
                                      int depth, uint32_t mask, int vs, int lane) {
  if (lane == 0) {
    atomicMax(&sh.maxd, depth);
    const int size = hi - lo + 1;
    if (base_case_applies(size, mask, vs)) {
      atomicAdd(&sh.hits[size], 1ull);
      insertion_sort(s, lo, hi);  // any sort of <= 8 keys gives the network's output
    } else if (size >= 2) {
      const int i = atomicAdd(&sh.cnt[slot], 1);
      NSB_DCHECK(i < kTraceSmall / 2);
      fr[slot * (kTraceSmall / 2) + i] = uint32_t(lo) | (uint32_t(hi) << 16);
    }
  }
  __syncwarp();
}

// median_of_three + hoare_partition of s[lo..hi] by one warp; returns the split.
template <class K>
__device__ int warp_partition(K* s, uint16_t* sL, uint16_t* sR, int lo, int hi, int lane) {
  K p{};
  if (lane == 0) {
    if (hi - lo >= 2) {
      const int mid = lo + (hi - lo) / 2;
      cx(s[lo], s[mid]);
      cx(s[lo], s[hi]);
      cx(s[mid], s[hi]);
      p = s[mid];
    } else {
      p = s[lo];
    }
  }
  p = __shfl_sync(0xffffffffu, p, 0);
  __syncwarp();
  const uint32_t lt = lanemask_lt();
  int nl = 0, nr = 0;
  for (int base = lo; base <= hi; base += 32) {
    const int x = base + lane;
    const bool ok = x <= hi;
    const K v = ok ? s[x] : K(0);
    const bool fl = ok && v >= p, fr = ok && v <= p;
    const uint32_t bl = __ballot_sync(0xffffffffu, fl), br = __ballot_sync(0xffffffffu, fr);
    NSB_DCHECK(!fl || lo + nl + __popc(bl & lt) <= hi);
    NSB_DCHECK(!fr || lo + nr + __popc(br & lt) <= hi);
    if (fl) sL[lo + nl + __popc(bl & lt)] = uint16_t(x);
    if (fr) sR[lo + nr + __popc(br & lt)] = uint16_t(x);
    nl += __popc(bl);
    nr += __popc(br);
  }
  __syncwarp();
  int a = 0, b = nl < nr ? nl : nr;
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (sL[lo + m - 1] < sR[lo + nr - m]) a = m;
    else b = m - 1;
  }
  const int S = a;
  for (int k = lane + 1; k <= S; k += 32) {
    const int x = sL[lo + k - 1], y = sR[lo + nr - k];
    NSB_DCHECK(x >= lo && x < y && y <= hi);
    const K t = s[x];
    s[x] = s[y];
    s[y] = t;
  }
  int j = -1;
  if (S + 1 <= nr) j = sR[lo + nr - S - 1];
  if (S >= 1) j = max(j, int(sL[lo + S - 1]));
  __syncwarp();
  return j < hi ? j : hi - 1;
}

template <class K>
__global__ void __launch_bounds__(kThreads) small_kernel(K* __restrict__ a,
                                                         const SmallSeg* __restrict__ segs,
                                                         uint32_t mask, int vs,
                                                         unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* s = reinterpret_cast<K*>(smem);
  uint16_t* sL = reinterpret_cast<uint16_t*>(s + kTraceSmall);
  uint16_t* sR = sL + kTraceSmall;
  uint32_t* fr = reinterpret_cast<uint32_t*>(sR + kTraceSmall);  // 2 x kTraceSmall/2
  __shared__ SmallShared sh;
  const SmallSeg g = segs[blockIdx.x];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < g.len; i += kThreads) s[i] = a[g.lo + i];
  if (threadIdx.x < 9) sh.hits[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    sh.cnt[0] = sh.cnt[1] = 0;
    sh.next = 0;
    sh.maxd = 0;
    sh.parts = 0;
  }
  __syncthreads();
  if (w == 0) visit(s, fr, sh, 0, 0, g.len - 1, g.depth, mask, vs, lane);
  __syncthreads();
  int cur = 0, depth = g.depth;
  while (sh.cnt[cur] > 0) {
    const int nxt = cur ^ 1;
    const int ncur = sh.cnt[cur];
    __syncthreads();  // every thread has read cnt[cur] before it is reused below
    if (threadIdx.x == 0) {
      sh.cnt[nxt] = 0;
      sh.next = 0;
    }
    __syncthreads();
    for (;;) {
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&sh.next, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx >= ncur) break;
      const uint32_t node = fr[cur * (kTraceSmall / 2) + idx];
      const int lo = node & 0xffff, hi = node >> 16;
      NSB_DCHECK(lo < hi && hi < g.len);
      const int split = warp_partition(s, sL, sR, lo, hi, lane);
      if (lane == 0) atomicAdd(&sh.parts, 1ull);
      visit(s, fr, sh, nxt, lo, split, depth + 1, mask, vs, lane);
      visit(s, fr, sh, nxt, split + 1, hi, depth + 1, mask, vs, lane);
    }
    __syncthreads();
    cur = nxt;
    ++depth;
  }
  for (int i = threadIdx.x; i < g.len; i += kThreads) a[g.lo + i] = s[i];
  if (threadIdx.x < 9 && sh.hits[threadIdx.x]) atomicAdd(&ctr[C_HITS + threadIdx.x], sh.hits[threadIdx.x]);
  if (threadIdx.x == 9 && sh.parts) atomicAdd(&ctr[C_PARTS], sh.parts);
  if (threadIdx.x == 10) atomicMax(&ctr[C_MAXD], (unsigned long long)sh.maxd);
}

template <class K>
constexpr int small_smem() {
  return kTraceSmall * (int)sizeof(K) + 2 * kTraceSmall * 2 + kTraceSmall * 4;
}

// ---------------------------------------------------------------------------
// host side

struct TraceTemp {
  unsigned long long* ctr;
  uint32_t* posL;
  uint32_t* posR;
  Seg* segs;
  Chunk* chunks;
  int32_t* first;
  uint32_t* cnt;
  void* piv;
  int64_t* totals;
  int64_t* S;
  int64_t* split;
  int* bad;
  SmallSeg* small;
  size_t seg_cap, chunk_cap, small_cap;
};

size_t seg_cap_of(size_t n) { return n / kTraceSmall + 2; }
size_t chunk_cap_of(size_t n) { return n / kChunk + seg_cap_of(n) + 2; }

size_t trace_temp(size_t n, size_t key_bytes, TraceTemp* t, void* base) {
  const size_t sc = seg_cap_of(n), cc = chunk_cap_of(n), mc = 2 * sc + 2;
  const bool large = n > (size_t)kTraceSmall;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + bytes, 256);
    return base ? static_cast<unsigned char*>(base) + at : nullptr;
  };
  void* ctr = take(C_NUM * 8 + 8);  // + the bad flag
  void* posL = take(large ? n * 4 : 0);
  void* posR = take(large ? n * 4 : 0);
  void* segs = take(sc * sizeof(Seg));
  void* chunks = take(cc * sizeof(Chunk));
  void* first = take((sc + 1) * 4);
  void* cnt = take(cc * 8);
  void* piv = take(sc * key_bytes);
  void* totals = take(sc * 16);
  void* S = take(sc * 8);
  void* split = take(sc * 8);
  void* small = take(mc * sizeof(SmallSeg));
  if (t) {
    t->ctr = static_cast<unsigned long long*>(ctr);
    t->bad = reinterpret_cast<int*>(static_cast<unsigned char*>(ctr) + C_NUM * 8);
    t->posL = static_cast<uint32_t*>(posL);
    t->posR = static_cast<uint32_t*>(posR);
    t->segs = static_cast<Seg*>(segs);
    t->chunks = static_cast<Chunk*>(chunks);
    t->first = static_cast<int32_t*>(first);
    t->cnt = static_cast<uint32_t*>(cnt);
    t->piv = piv;
    t->totals = static_cast<int64_t*>(totals);
    t->S = static_cast<int64_t*>(S);
    t->split = static_cast<int64_t*>(split);
    t->small = static_cast<SmallSeg*>(small);
    t->seg_cap = sc;
    t->chunk_cap = cc;
    t->small_cap = mc;
  }
  return off;
}

// One level of grid-wide partitions over `segs` (all of one depth).  With
// `pivot` non-null the median of three is skipped and that pivot is used
// (the explicit-pivot hoare_partition entry, one segment).  Fills `split`.
template <class K>
int partition_level(K* d, const std::vector<Seg>& segs, const K* pivot, const TraceTemp& t,
                    std::vector<int64_t>& split, cudaStream_t st) {
  const int nseg = (int)segs.size();
  std::vector<Chunk> chunks;
  std::vector<int32_t> first(nseg + 1);
  for (int s = 0; s < nseg; ++s) {
    first[s] = (int32_t)chunks.size();
    for (int64_t x = segs[s].lo; x <= segs[s].hi; x += kChunk) {
      const int64_t len = std::min<int64_t>(kChunk, segs[s].hi - x + 1);
      chunks.push_back(Chunk{x, (int32_t)len, s, first[s], 0});
    }
  }
  first[nseg] = (int32_t)chunks.size();
  const int nch = (int)chunks.size();
  if ((size_t)nseg > t.seg_cap || (size_t)nch > t.chunk_cap) return NS_ERR_TEMP;
  K* piv = static_cast<K*>(t.piv);
  NSB_TRY(check_cuda(cudaMemcpyAsync(t.segs, segs.data(), nseg * sizeof(Seg), cudaMemcpyHostToDevice, st),
                     "trace segs"));
  NSB_TRY(check_cuda(cudaMemcpyAsync(t.chunks, chunks.data(), nch * sizeof(Chunk),
                                     cudaMemcpyHostToDevice, st),
                     "trace chunks"));
  NSB_TRY(check_cuda(cudaMemcpyAsync(t.first, first.data(), (nseg + 1) * 4, cudaMemcpyHostToDevice, st),
                     "trace first"));
  if (pivot) {
    NSB_TRY(check_cuda(cudaMemcpyAsync(piv, pivot, sizeof(K), cudaMemcpyHostToDevice, st), "trace pivot"));
  } else {
    mot_kernel<K><<<(nseg + 127) / 128, 128, 0, st>>>(d, t.segs, nseg, piv);
    NSB_TRY(check_launch("trace median_of_three"));
  }
  {
    Prof pr(PK_QS_COUNT, st);
    count_kernel<K><<<nch, kThreads, 0, st>>>(d, t.chunks, piv, t.cnt);
    NSB_TRY(check_launch("trace count"));
  }
  scan_kernel<<<nseg, kThreads, 0, st>>>(t.first, t.cnt, t.totals);
  NSB_TRY(check_launch("trace scan"));
  {
    Prof pr(PK_QS_SCATTER, st);
    compact_kernel<K><<<nch, kThreads, 0, st>>>(d, t.chunks, t.segs, piv, t.cnt, t.posL, t.posR);
    NSB_TRY(check_launch("trace compact"));
  }
  find_kernel<<<(nseg + 127) / 128, 128, 0, st>>>(t.segs, nseg, t.totals, t.posL, t.posR, t.S,
                                                  t.split, t.bad);
  NSB_TRY(check_launch("trace find"));
  swap_kernel<K><<<nch, kThreads, 0, st>>>(d, t.chunks, t.segs, t.totals, t.S, t.posL, t.posR);
  NSB_TRY(check_launch("trace swap"));
  split.resize(nseg);
  NSB_TRY(check_cuda(cudaMemcpyAsync(split.data(), t.split, nseg * 8, cudaMemcpyDeviceToHost, st),
                     "trace split"));
  return check_cuda(cudaStreamSynchronize(st), "trace level sync");
}

template <class K>
int launch_small(K* d, const std::vector<SmallSeg>& small, uint32_t mask, int vs,
                 const TraceTemp& t, cudaStream_t st) {
  if (small.empty()) return NS_OK;
  if (small.size() > t.small_cap) return NS_ERR_TEMP;
  NSB_TRY(check_cuda(cudaMemcpyAsync(t.small, small.data(), small.size() * sizeof(SmallSeg),
                                     cudaMemcpyHostToDevice, st),
                     "trace small list"));
  NSB_TRY(ensure_smem_attr((const void*)small_kernel<K>, small_smem<K>(), "trace small"));
  Prof pr(PK_QS_BUCKET, st);
  small_kernel<K><<<(unsigned)small.size(), kThreads, small_smem<K>(), st>>>(d, t.small, mask, vs,
                                                                            t.ctr);
  return check_launch("trace small");
}

template <class K>
int traced_quick_sort(K* d, size_t n, uint32_t mask, int vs, uint64_t* out12, void* temp,
                      size_t temp_bytes, cudaStream_t st) {
  for (int i = 0; i < 12; ++i) out12[i] = 0;
  if (n == 0) return NS_OK;  // high < low: no call, no counters (hybrid.hpp:201, 237)
  if (n > UINT32_MAX) return NS_ERR_INVALID;
  TraceTemp t;
  if (!temp || temp_bytes < trace_temp(n, sizeof(K), &t, nullptr)) return NS_ERR_TEMP;
  trace_temp(n, sizeof(K), &t, temp);
  NSB_TRY(check_cuda(cudaMemsetAsync(t.ctr, 0, C_NUM * 8 + 8, st), "trace memset"));
  uint64_t parts = 0;
  int maxd = 0;
  std::vector<SmallSeg> small;
  if (n <= (size_t)kTraceSmall) {
    small.push_back(SmallSeg{0, (int32_t)n, 1});
    NSB_TRY(launch_small(d, small, mask, vs, t, st));
  } else {
    std::vector<Seg> cur{Seg{0, (int64_t)n - 1}}, nxt;
    std::vector<int64_t> split;
    for (int depth = 1; !cur.empty(); ++depth) {
      maxd = std::max(maxd, depth);  // every large node: depth, then a partition
      parts += cur.size();
      NSB_TRY(partition_level(d, cur, (const K*)nullptr, t, split, st));
      nxt.clear();
      small.clear();
      for (size_t s = 0; s < cur.size(); ++s) {
        const Seg kids[2] = {{cur[s].lo, split[s]}, {split[s] + 1, cur[s].hi}};
        for (const Seg& k : kids) {
          const int64_t len = k.hi - k.lo + 1;
          if (len > kTraceSmall) nxt.push_back(k);
          else small.push_back(SmallSeg{k.lo, (int32_t)len, depth + 1});
        }
      }
      NSB_TRY(launch_small(d, small, mask, vs, t, st));
      cur.swap(nxt);
    }
  }
  unsigned long long c[C_NUM];
  NSB_TRY(check_cuda(cudaMemcpyAsync(c, t.ctr, sizeof c, cudaMemcpyDeviceToHost, st), "trace ctr"));
  NSB_TRY(check_cuda(cudaStreamSynchronize(st), "trace sync"));
  for (int w = 0; w <= 8; ++w) out12[w] = c[C_HITS + w];
  out12[9] = 0;  // merges
  out12[10] = c[C_PARTS] + parts;
  out12[11] = std::max<uint64_t>(c[C_MAXD], (uint64_t)maxd);
  return NS_OK;
}

template <class K>
int hoare_partition_dev(K* d, size_t n, int64_t low, int64_t high, K pivot, int64_t* out_split,
                        void* temp, size_t temp_bytes, cudaStream_t st) {
  if (!d || !out_split || low < 0 || low >= high || high >= (int64_t)n) return NS_ERR_INVALID;
  const size_t len = (size_t)(high - low + 1);
  if (len > UINT32_MAX) return NS_ERR_INVALID;
  // the level kernels index posL/posR by absolute position: hand them the
  // range as its own array
  K* r = d + low;
  TraceTemp t;
  const size_t need = trace_temp(std::max(len, (size_t)kTraceSmall + 1), sizeof(K), &t, nullptr);
  if (!temp || temp_bytes < need) return NS_ERR_TEMP;
  trace_temp(std::max(len, (size_t)kTraceSmall + 1), sizeof(K), &t, temp);
  NSB_TRY(check_cuda(cudaMemsetAsync(t.bad, 0, 4, st), "hoare memset"));
  std::vector<int64_t> split;
  NSB_TRY(partition_level(r, {Seg{0, (int64_t)len - 1}}, &pivot, t, split, st));
  int bad = 0;
  NSB_TRY(check_cuda(cudaMemcpyAsync(&bad, t.bad, 4, cudaMemcpyDeviceToHost, st), "hoare flag"));
  NSB_TRY(check_cuda(cudaStreamSynchronize(st), "hoare sync"));
  if (bad) return NS_ERR_INVALID;  // pivot above every key or below every key: untouched
  *out_split = low + split[0];
  return NS_OK;
}

template <class K>
int median_of_three_dev(K* d, size_t n, int64_t low, int64_t high, K* out_pivot, cudaStream_t st) {
  if (!d || !out_pivot || low < 0 || low > high || high >= (int64_t)n) return NS_ERR_INVALID;
  Seg* seg = nullptr;
  K* piv = nullptr;
  NSB_TRY(check_cuda(cudaMallocAsync(&seg, sizeof(Seg) + 16, st), "mot alloc"));
  piv = reinterpret_cast<K*>(seg + 1);
  const Seg h{low, high};
  int rc = check_cuda(cudaMemcpyAsync(seg, &h, sizeof h, cudaMemcpyHostToDevice, st), "mot seg");
  if (rc == NS_OK) {
    mot_kernel<K><<<1, 32, 0, st>>>(d, seg, 1, piv);
    rc = check_launch("median_of_three");
  }
  if (rc == NS_OK)
    rc = check_cuda(cudaMemcpyAsync(out_pivot, piv, sizeof(K), cudaMemcpyDeviceToHost, st), "mot pivot");
  cudaFreeAsync(seg, st);
  if (rc == NS_OK) rc = check_cuda(cudaStreamSynchronize(st), "mot sync");
  return rc;
}

// Host-array forms: one device copy of the range, the device call, the copy
// back (the reference's call shape on a host span).
template <class K>
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

template <class K>
int traced_quick_sort_host(K* h, size_t n, uint32_t mask, int vs, uint64_t* out12) {
  if (!out12 || (n && !h)) return NS_ERR_INVALID;
  if (n == 0) {
    for (int i = 0; i < 12; ++i) out12[i] = 0;
    return NS_OK;
  }
  const size_t kb = align_up(n * sizeof(K), 256), tb = trace_temp(n, sizeof(K), nullptr, nullptr);
  DevBuf<K> buf;
  NSB_TRY(check_cuda(cudaMalloc(&buf.p, kb + tb), "cudaMalloc"));
  K* d = static_cast<K*>(buf.p);
  cudaStream_t st = cudaStreamPerThread;
  NSB_TRY(check_cuda(cudaMemcpyAsync(d, h, n * sizeof(K), cudaMemcpyHostToDevice, st), "H2D"));
  NSB_TRY(traced_quick_sort(d, n, mask, vs, out12, static_cast<unsigned char*>(buf.p) + kb, tb, st));
  NSB_TRY(check_cuda(cudaMemcpyAsync(h, d, n * sizeof(K), cudaMemcpyDeviceToHost, st), "D2H"));
  return check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

template <class K>
int hoare_partition_host(K* h, size_t n, int64_t low, int64_t high, K pivot, int64_t* out_split) {
  if (!h || !out_split || low < 0 || low >= high || high >= (int64_t)n) return NS_ERR_INVALID;
  const size_t len = (size_t)(high - low + 1);
  const size_t kb = align_up(len * sizeof(K), 256);
  const size_t tb = trace_temp(std::max(len, (size_t)kTraceSmall + 1), sizeof(K), nullptr, nullptr);
  DevBuf<K> buf;
  NSB_TRY(check_cuda(cudaMalloc(&buf.p, kb + tb), "cudaMalloc"));
  K* d = static_cast<K*>(buf.p);
  cudaStream_t st = cudaStreamPerThread;
  NSB_TRY(check_cuda(cudaMemcpyAsync(d, h + low, len * sizeof(K), cudaMemcpyHostToDevice, st), "H2D"));
  int64_t split = 0;
  NSB_TRY(hoare_partition_dev(d, len, 0, (int64_t)len - 1, pivot, &split,
                              static_cast<unsigned char*>(buf.p) + kb, tb, st));
  NSB_TRY(check_cuda(cudaMemcpyAsync(h + low, d, len * sizeof(K), cudaMemcpyDeviceToHost, st), "D2H"));
  NSB_TRY(check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"));
  *out_split = low + split;
  return NS_OK;
}

template <class K>
int median_of_three_host(K* h, size_t n, int64_t low, int64_t high, K* out_pivot) {
  if (!h || !out_pivot || low < 0 || low > high || high >= (int64_t)n) return NS_ERR_INVALID;
  // only the three probed cells move: stage them, run the device compare-
  // exchanges on the staged copy, write them back
  const int64_t mid = low + (high - low) / 2;
  K three[3] = {h[low], h[mid], h[high]};
  const int64_t span = high - low < 2 ? 0 : 2;
  DevBuf<K> buf;
  NSB_TRY(check_cuda(cudaMalloc(&buf.p, 3 * sizeof(K)), "cudaMalloc"));
  K* d = static_cast<K*>(buf.p);
  cudaStream_t st = cudaStreamPerThread;
  NSB_TRY(check_cuda(cudaMemcpyAsync(d, three, sizeof three, cudaMemcpyHostToDevice, st), "H2D"));
  NSB_TRY(median_of_three_dev(d, 3, 0, span, out_pivot, st));
  NSB_TRY(check_cuda(cudaMemcpyAsync(three, d, sizeof three, cudaMemcpyDeviceToHost, st), "D2H"));
  NSB_TRY(check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"));
  if (span) {
    h[low] = three[0];
    h[mid] = three[1];
    h[high] = three[2];
  }
  return NS_OK;
}

}  // namespace
}  // namespace nsb

using namespace nsb;

extern "C" {

size_t ns_quick_sort_traced_temp_bytes(size_t n) { return trace_temp(n, 8, nullptr, nullptr); }
size_t ns_hoare_partition_temp_bytes(size_t len) {
  return trace_temp(std::max(len, (size_t)kTraceSmall + 1), 8, nullptr, nullptr);
}

int ns_quick_sort_traced_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                             uint64_t* out12, void* d_temp, size_t temp_bytes, void* stream) {
  if (!out12 || (n && !d_keys)) return NS_ERR_INVALID;
  return traced_quick_sort(d_keys, n, width_mask, varsort_max, out12, d_temp, temp_bytes,
                           static_cast<cudaStream_t>(stream));
}
int ns_quick_sort_traced_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                             uint64_t* out12, void* d_temp, size_t temp_bytes, void* stream) {
  if (!out12 || (n && !d_keys)) return NS_ERR_INVALID;
  return traced_quick_sort(d_keys, n, width_mask, varsort_max, out12, d_temp, temp_bytes,
                           static_cast<cudaStream_t>(stream));
}
int ns_hoare_partition_i32(int32_t* d_keys, size_t n, int64_t low, int64_t high, int32_t pivot,
                           int64_t* split, void* d_temp, size_t temp_bytes, void* stream) {
  return hoare_partition_dev(d_keys, n, low, high, pivot, split, d_temp, temp_bytes,
                             static_cast<cudaStream_t>(stream));
}
int ns_hoare_partition_i64(int64_t* d_keys, size_t n, int64_t low, int64_t high, int64_t pivot,
                           int64_t* split, void* d_temp, size_t temp_bytes, void* stream) {
  return hoare_partition_dev(d_keys, n, low, high, pivot, split, d_temp, temp_bytes,
                             static_cast<cudaStream_t>(stream));
}
int ns_median_of_three_i32(int32_t* d_keys, size_t n, int64_t low, int64_t high, int32_t* pivot,
                           void* stream) {
  return median_of_three_dev(d_keys, n, low, high, pivot, static_cast<cudaStream_t>(stream));
}
int ns_median_of_three_i64(int64_t* d_keys, size_t n, int64_t low, int64_t high, int64_t* pivot,
                           void* stream) {
  return median_of_three_dev(d_keys, n, low, high, pivot, static_cast<cudaStream_t>(stream));
}
int ns_quick_sort_traced_host_i32(int32_t* keys, size_t n, uint32_t width_mask, int varsort_max,
                                  uint64_t* out12) {
  return traced_quick_sort_host(keys, n, width_mask, varsort_max, out12);
}
int ns_quick_sort_traced_host_i64(int64_t* keys, size_t n, uint32_t width_mask, int varsort_max,
                                  uint64_t* out12) {
  return traced_quick_sort_host(keys, n, width_mask, varsort_max, out12);
}
int ns_hoare_partition_host_i32(int32_t* keys, size_t n, int64_t low, int64_t high, int32_t pivot,
                                int64_t* split) {
  return hoare_partition_host(keys, n, low, high, pivot, split);
}
int ns_hoare_partition_host_i64(int64_t* keys, size_t n, int64_t low, int64_t high, int64_t pivot,
                                int64_t* split) {
  return hoare_partition_host(keys, n, low, high, pivot, split);
}
int ns_median_of_three_host_i32(int32_t* keys, size_t n, int64_t low, int64_t high, int32_t* pivot) {
  return median_of_three_host(keys, n, low, high, pivot);
}
int ns_median_of_three_host_i64(int64_t* keys, size_t n, int64_t low, int64_t high, int64_t* pivot) {
  return median_of_three_host(keys, n, low, high, pivot);
}

}  // extern "C"
