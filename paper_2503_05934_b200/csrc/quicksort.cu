// quicksort.cu — the quick-sort layer on sm_100a, planned entirely on the
// device (no host round trip, so ns_quick_sort_* is stream-ordered and can
// be captured in a CUDA graph).
//
// Replaces /root/reference/proj/include/netsort/hybrid.hpp:105-150
// (median_of_three + hoare_partition + quick_sort_rec).  A single pivot and
// a two-cursor scan are inherently sequential, so one GPU partition level
// uses up to 255 sampled pivots at once (a many-pivot quick sort, i.e. a
// sample sort) on every oversized segment of the level:
//   sample  : one CTA per segment draws 16 jittered, regularly spaced samples
//             per bucket, sorts them on chip with the tile sort and keeps
//             every 16th as a pivot (the many-pivot analogue of
//             median_of_three: sorted input still splits evenly);
//   count   : every key is classified into 2B-1 buckets — "between" buckets
//             (s[j-1] < k < s[j]) and "equal" buckets (k == s[j]); an equal
//             bucket is constant, which keeps heavy duplicates from
//             unbalancing the recursion (the job of hoare_partition's j==high
//             fix-up for one pivot, hybrid.hpp:130); it stores every key's
//             one-byte bucket id and every chunk's bucket counts;
//   plan    : one CTA per segment scans its bucket counts into positions and
//             sorts the buckets out: the ones that fit a CTA become leaf jobs
//             (neighbouring small buckets packed into one tile, since they
//             hold disjoint ascending key ranges), large constant buckets are
//             already sorted, large between buckets become the next level's
//             segments (quick_sort_rec's two recursive calls, hybrid.hpp:
//             145-148), appended to device-side work lists;
//   scatter : keys move to their buckets through a shared-memory multisplit,
//             so each bucket's keys leave a CTA as one contiguous run
//             (coalesced stores) at a range reserved with one global atomic
//             per (chunk, bucket); the chunk's counts are scanned first, so
//             one shared atomic per key returns its staging position.
// The number of levels follows from n alone (each level divides a segment by
// up to 256); after the last level every leaf job is sorted on chip by
// cta_sort with the config's network base case (try_base_case,
// hybrid.hpp:48-56).  Launch grids are upper bounds and every kernel walks
// the device-side lists, so the host never reads a count.  A segment still
// larger than one CTA after the last level (only possible for adversarial
// sampling) is sorted by one CTA in global memory — correct, just slow.
// Parity with the reference is on the sorted bytes, which are unique.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "common.cuh"
#include "mergesort.cuh"

namespace nsb {

constexpr int kQsNT = 512;                   // count / scatter / plan threads
constexpr int kQsPer = 16;                   // keys per thread in count / scatter
constexpr int kQsChunk = kQsNT * kQsPer;     // keys per chunk (one CTA iteration)
constexpr int kQsMaxB = 128;                 // pivot slots per segment (B-1 real + pad):
                                             // 2B-1 <= 255 buckets, so a bucket id is one byte
constexpr int kQsOver = 16;                  // samples per bucket
constexpr int kQsHistStride = 2 * kQsMaxB;   // per-chunk histogram slots (2B-1 <= 255 used)
#ifndef NSB_QS_TARGET
#define NSB_QS_TARGET 4096
#endif
constexpr int64_t kQsTarget = NSB_QS_TARGET;  // mean bucket size a level aims for

// Buckets a segment of len keys is split into: the smallest power of two
// B >= 2 with B * kQsTarget >= len, at most kQsMaxB.
__host__ __device__ inline int qs_buckets(int64_t len) {
  int B = 2;
  while (B < kQsMaxB && (int64_t)B * kQsTarget < len) B <<= 1;
  return B;
}

// Partition levels for segments of len keys: expected bucket size after
// each level, until it fits one CTA.
static int qs_levels(int64_t len) {
  int levels = 0;
  for (int64_t s = len; s > kSmallTile / 2; s /= qs_buckets(s)) ++levels;
  return std::max(levels, 1);
}

struct QsSeg {
  int64_t start, len;
  int64_t chunk0;   // first chunk of this segment in its level's chunk list
  int64_t cnt_off;  // first bucket counter (2B-1 of them)
  int64_t spl_off;  // first pivot slot (B of them)
  int32_t B, nchunks;
};

struct QsJob {
  int64_t start, len;
  int32_t flags;  // bit 0: source is tmp; bits 1-2: 0 sort, 1 copy, 2 big
  int32_t pad;
};
enum { kJobSort = 0, kJobCopy = 1, kJobBig = 2 };
constexpr int64_t kQsCopyChunk = 32768;  // keys per copy job of a big constant bucket

struct QsCounters {  // device-side list lengths
  unsigned long long nseg[2], nchunk[2], nbkt[2], nspl[2];
  unsigned long long njobs[3];
};

template <class Key>
struct QsCtx {
  Key* keys;
  Key* tmp;
  int64_t n;
  // level 0: nseg0 uniform segments of len0 keys (no list: arithmetic)
  int64_t nseg0, len0, cps0;
  int32_t B0;
  QsCounters* ctr;
  QsSeg* segs[2];
  int32_t* chunk_seg[2];
  Key* spl[2];
  uint16_t* cells[2];  // 16 per pivot slot: the classifier's prefix cells
  uint8_t* ids;        // bucket id of every key of the level (count -> scatter)
  uint16_t* chist;     // per chunk: its kQsHistStride bucket counts (count -> scatter)
  uint32_t* cnt[2];
  unsigned long long* fill[2];  // bucket write cursors (absolute positions)
  QsJob* jobs[3];
  int64_t max_segs, max_chunks, max_bkt, max_spl, max_jobs;
};

// ---- level geometry (device) ----------------------------------------------
template <class Key>
__device__ __forceinline__ QsSeg qs_seg(const QsCtx<Key>& c, int level, int64_t s) {
  if (level == 0) {
    QsSeg g;
    g.start = s * c.len0;
    g.len = c.len0;
    g.B = c.B0;
    g.nchunks = (int32_t)c.cps0;
    g.chunk0 = s * c.cps0;
    g.cnt_off = s * (2 * c.B0 - 1);
    g.spl_off = s * c.B0;
    return g;
  }
  return c.segs[level & 1][s];
}
template <class Key>
__device__ __forceinline__ int64_t qs_nseg(const QsCtx<Key>& c, int level) {
  return level == 0 ? c.nseg0 : (int64_t)*(volatile unsigned long long*)&c.ctr->nseg[level & 1];
}
template <class Key>
__device__ __forceinline__ int64_t qs_nchunk(const QsCtx<Key>& c, int level) {
  return level == 0 ? c.nseg0 * c.cps0
                    : (int64_t)*(volatile unsigned long long*)&c.ctr->nchunk[level & 1];
}
template <class Key>
__device__ __forceinline__ int64_t qs_seg_of_chunk(const QsCtx<Key>& c, int level, int64_t ch) {
  return level == 0 ? ch / c.cps0 : (int64_t)c.chunk_seg[level & 1][ch];
}
// keys of level l live in X_l: the caller's buffer at even levels, tmp at odd
template <class Key>
__device__ __forceinline__ Key* qs_src(const QsCtx<Key>& c, int level) {
  return (level & 1) ? c.tmp : c.keys;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// ---- 1. sample + pivots -----------------------------------------------------
// Sample i of a segment sits at i*stride + jitter(i) (stride = len / S), so
// sorted input still yields evenly spaced pivots; the jitter is a hash scaled
// into [0, stride) with one multiply-high (a 64-bit modulo here measured as
// most of the sample kernel's time).
__device__ __forceinline__ int64_t qs_sample_pos(int i, int64_t stride, int level) {
  const uint32_t st = stride > 0xffffffffll ? 0xffffffffu : (uint32_t)stride;
  return (int64_t)i * stride + (int64_t)__umulhi(hash32((uint32_t)i * 2654435761u + (uint32_t)level), st);
}

// The classifier's prefix cells (see "classification" below): the pivots'
// key range [lo, hi] = [piv[0], piv[B-2]] cut into 16 B cells of 2^shift keys.
template <class Key>
__device__ __forceinline__ int qs_cell_shift(Key lo, Key hi, int ncell) {
  using U = std::make_unsigned_t<Key>;
  const U span = (U)hi - (U)lo;
  int shift = 0;
  while ((span >> shift) >= (U)ncell) ++shift;
  return shift;
}
template <class Key>
__device__ __forceinline__ int qs_cell_of(Key p, Key lo, int shift, int ncell) {
  using U = std::make_unsigned_t<Key>;
  const U cidx = ((U)p - (U)lo) >> shift;
  return cidx < (U)ncell ? (int)cidx : ncell - 1;
}

// Pivot j of S = 16 B sorted samples is sample 16 (j+1) - 1; slot B-1 is the
// key-maximum pad.  Also clears the segment's bucket counters.
template <class Key>
__device__ __forceinline__ void qs_write_pivots_zero(const QsCtx<Key>& c, int level, const QsSeg& g,
                                                     int i, int stride) {
  uint32_t* cnt = c.cnt[level & 1] + g.cnt_off;
  for (int b = i; b < 2 * g.B - 1; b += stride) cnt[b] = 0;
}

template <class Key>
__global__ void __launch_bounds__(256) qs_sample_kernel(QsCtx<Key> c, int level) {
  pdl_wait();  // everything below reads the previous kernels' lists / keys
  pdl_trigger();
  __shared__ __align__(16) Key tile[padded_words<Key>(2048)];
  __shared__ Key piv[kQsMaxB];
  __shared__ uint32_t ccount[16 * kQsMaxB];
  __shared__ uint32_t wsum[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x == 0 && tid == 0) {
    // the next level's lists are appended by this level's plan kernel
    const int nx = (level + 1) & 1;
    c.ctr->nseg[nx] = 0;
    c.ctr->nchunk[nx] = 0;
    c.ctr->nbkt[nx] = 0;
    c.ctr->nspl[nx] = 0;
    if (level == 0) c.ctr->njobs[0] = c.ctr->njobs[1] = c.ctr->njobs[2] = 0;
  }
  const Key* X = qs_src(c, level);
  Key* splb = c.spl[level & 1];
  const int64_t nseg = qs_nseg(c, level);
  // segments of B <= 32 pivots (S <= 512 samples): one warp each, sorted in
  // registers (16 per lane, network base case + warp bitonic stage); segment
  // s goes to CTA s mod grid first, so a level of few segments spreads over
  // the SMs instead of packing 8 warps onto one
  for (int64_t s = blockIdx.x + (int64_t)warp * gridDim.x; s < nseg;
       s += (int64_t)gridDim.x * 8) {
    {
      const QsSeg g = qs_seg(c, level, s);
      if (g.B <= 32) {
        const int S = kQsOver * g.B;
        const int64_t stride = g.len / S;
        Key v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int i = lane * 16 + u;
          v[u] = i < S ? X[g.start + qs_sample_pos(i, stride, level)] : KeyT<Key>::kMax;
        }
        thread_sort<8>(v);
        warp_bitonic<5>(v, lane);
        // lane l holds sorted samples [16 l, 16 l + 16): pivot j is lane j's last
        if (lane < g.B) splb[g.spl_off + lane] = lane < g.B - 1 ? v[15] : KeyT<Key>::kMax;
        qs_write_pivots_zero(c, level, g, lane, 32);
        // prefix cells: j0(c) = #pivots whose cell < c (cells of the sorted
        // pivots are non-decreasing: a 5-step shuffle search), k = j0(c+1) - j0(c)
        const Key lo = __shfl_sync(kFull, v[15], 0), hi = __shfl_sync(kFull, v[15], g.B - 2);
        const int ncell = 16 * g.B;
        const int shift = qs_cell_shift(lo, hi, ncell);
        const int cj = lane < g.B - 1 ? qs_cell_of(v[15], lo, shift, ncell) : ncell;
        uint16_t* cells = c.cells[level & 1] + 16 * g.spl_off;
        for (int c0 = 0; c0 < ncell; c0 += 32) {
          const int cc = c0 + lane;
          auto j0_of = [&](int x) {
            int l = 0, h = g.B - 1;
#pragma unroll
            for (int it = 0; it < 5; ++it) {
              const int m = (l + h) >> 1;
              const int cm = __shfl_sync(kFull, cj, m);
              if (l < h) {
                if (cm < x) l = m + 1;
                else h = m;
              }
            }
            return l;
          };
          const int j0 = j0_of(cc), j1 = j0_of(cc + 1);
          if (cc < ncell) cells[cc] = (uint16_t)(j0 | ((j1 - j0) << 8));
        }
      }
    }
  }
  // larger segments (B = 64, 128: S = 1024, 2048 samples), one CTA each: the
  // CTA gathers 8 samples per thread and sorts all S of them at once (network
  // base case, warp bitonic stage, three shared-memory merge levels), so the
  // pivots are exact regular quantiles of the samples: pivot j = sample
  // 16 (j+1) - 1 of the sorted S
  for (int64_t sb = blockIdx.x; sb < nseg; sb += gridDim.x) {
    {
      const QsSeg g = qs_seg(c, level, sb);
      if (g.B <= 32) continue;
      const int S = kQsOver * g.B;
      const int64_t stride = g.len / S;
      Key v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = tid * 8 + u;
        v[u] = i < S ? X[g.start + qs_sample_pos(i, stride, level)] : KeyT<Key>::kMax;
      }
      cta_sort_padded_regs<256, 8, 8>(v, tile);
      const int ncell = 16 * g.B;
      for (int i = tid; i < ncell; i += 256) ccount[i] = 0;
      for (int j = tid; j < g.B; j += 256) {
        const Key pv = j < g.B - 1 ? tile[pad_idx<Key>(16 * (j + 1) - 1)] : KeyT<Key>::kMax;
        splb[g.spl_off + j] = pv;
        piv[j] = pv;
      }
      qs_write_pivots_zero(c, level, g, tid, 256);
      __syncthreads();
      // prefix cells: count the pivots per cell, exclusive scan -> j0
      const Key lo = piv[0], hi = piv[g.B - 2];
      const int shift = qs_cell_shift(lo, hi, ncell);
      for (int j = tid; j < g.B - 1; j += 256) atomicAdd(&ccount[qs_cell_of(piv[j], lo, shift, ncell)], 1u);
      __syncthreads();
      {
        const int per = ncell / 256;  // 4 .. 16 cells per thread
        uint32_t run[16];
        uint32_t tot = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          run[q] = q < per ? ccount[tid * per + q] : 0u;
          tot += run[q];
        }
        // block exclusive scan of the per-thread totals (8 warps)
        uint32_t x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t before = 0;
        for (int w = 0; w < warp; ++w) before += wsum[w];
        uint32_t j0 = before + x - tot;
        uint16_t* cells = c.cells[level & 1] + 16 * g.spl_off;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q < per) {
            cells[tid * per + q] = (uint16_t)(j0 | (run[q] << 8));
            j0 += run[q];
          }
      }
      __syncthreads();  // sub / piv / ccount are reused by the next segment
    }
  }
}

// ---- classification ----------------------------------------------------------
// bucket(key): j = number of real pivots < key (lower_bound over the B-1 real
// pivots; slot B-1 is the key-maximum pad); equal bucket 2j+1 when
// piv[j] == key, else between bucket 2j.  Every key is classified ONCE per
// level (count kernel); its one-byte bucket id is stored for the scatter.
//
// Per segment every CTA loads, into shared memory,
//   - the pivot table REPLICATED across the banks: pivot i of lane l sits at
//     word i*R + l%R (R = 32 int32 / 16 int64 copies), so data-dependent
//     probes of the 32 lanes always hit 32 different banks (one copy: ~3.5
//     wavefronts per probe; ncu measured 76 % bank-conflict wavefronts);
//   - the prefix cells built by the sample kernel: the pivots' key range
//     [piv[0], piv[B-2]] cut into 16 B cells, cell c = (j0 = #pivots below
//     the cell, k = #pivots inside it).  A key finds its cell with one shift
//     and compares with the k pivots of its cell — usually none or one —
//     instead of log2(B) dependent probes.
template <class Key>
__host__ __device__ constexpr int qs_rep() { return sizeof(Key) == 4 ? 32 : 16; }
constexpr int kQsCellsMax = 16 * kQsMaxB;
template <class Key>
__host__ __device__ constexpr int qs_table_bytes() {
  // one more pivot slot than kQsMaxB: the classifier reads slot j + 1 <= B unclamped
  return (kQsMaxB + 1) * qs_rep<Key>() * (int)sizeof(Key) + kQsCellsMax * 2;
}

template <class Key>
struct QsClassifier {
  const Key* tab;        // replicated pivots, this lane's column
  const uint16_t* cell;  // j0 | k << 8
  Key lo, hi;
  int shift, ncell, B;
  __device__ __forceinline__ int operator()(Key key) const {
    constexpr int R = qs_rep<Key>();
    using U = std::make_unsigned_t<Key>;
    // the key clamped into the pivots' range [lo, hi] picks its cell: keys
    // below the first pivot use cell 0 (j0 = 0; its first candidate is the
    // first pivot, which they do not exceed), keys above the last pivot the
    // last pivot's cell (every pivot of it is smaller: j ends at B - 1);
    // (hi - lo) >> shift < ncell by the choice of shift
    const Key kc = min(max(key, lo), hi);
    const int ci = (int)(((U)kc - (U)lo) >> shift);
    const uint32_t e = cell[ci];
    int j = (int)(e & 255u);
    int k = (int)(e >> 8);
    // the first step without a branch (a cell holds 0 or 1 pivot almost
    // always): both candidate pivots are loaded at once (slots B-1 and B are
    // key-maximum pads, so j + 1 <= B stays in the table)
    const Key t0 = tab[j * R];
    const Key t1 = tab[(j + 1) * R];
    const bool s1 = (k > 0) & (t0 < key);
    j += s1;
    k -= s1;
    Key t = s1 ? t1 : t0;
#pragma unroll 1
    while (k > 0 && t < key) {  // cells with 2+ pivots (clustered pivots)
      ++j;
      --k;
      t = tab[j * R];
    }
    return 2 * j + ((j < B - 1) & (t == key));
  }
};

// Loads both tables of one segment (all threads of the CTA; the caller
// synchronises before and after).  The cells were built by the sample kernel.
template <class Key>
__device__ __forceinline__ QsClassifier<Key> qs_load_classifier(unsigned char* raw,
                                                                 const Key* __restrict__ spl,
                                                                 const uint16_t* __restrict__ cells,
                                                                 int B) {
  constexpr int R = qs_rep<Key>();
  Key* tab = reinterpret_cast<Key*>(raw);
  uint16_t* cell = reinterpret_cast<uint16_t*>(raw + (kQsMaxB + 1) * R * sizeof(Key));
  const Key lo = __ldg(spl), hi = __ldg(spl + (B >= 2 ? B - 2 : 0));
  const int ncell = 16 * B;
#pragma unroll 4
  for (int i = threadIdx.x; i < B * R; i += blockDim.x) tab[i] = __ldg(spl + i / R);
  if (threadIdx.x < R) tab[B * R + threadIdx.x] = KeyT<Key>::kMax;  // slot B: read, never selected
#pragma unroll 4
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) cell[i] = __ldg(cells + i);
  return QsClassifier<Key>{tab + (threadIdx.x & (R - 1)), cell, lo, hi, qs_cell_shift(lo, hi, ncell),
                           ncell, B};
}

// ---- 2. count (classify once, store the ids) ----------------------------------
// One shared increment per key: ptxas emits ATOMS.POPC.INC, which charges all
// lanes of a warp that hit the same bucket in one operation (sorted input).
__device__ __forceinline__ void qs_hist_add(uint32_t* hist, int b) {
  if (b >= 0) atomicAdd(&hist[b], 1u);
}

// Chunk staging for the count and scatter kernels: one elected thread copies
// the 16-byte-aligned cover of a chunk's keys (and, for the scatter, its
// one-byte bucket ids) into shared memory with a bulk copy (TMA 1D, mbarrier
// completion) as soon as the previous chunk has been moved into registers, so
// the next chunk's HBM read overlaps this chunk's classification / multisplit.
// A cover that would leave the array (a misaligned caller pointer at the
// first chunk, the array's last chunk) is read directly instead.
template <class T>
struct QsCover {
  const T* src;
  int phase;       // elements of the cover before the chunk's first
  uint32_t bytes;  // multiple of 16
  bool ok;
};
template <class T>
__device__ __forceinline__ QsCover<T> qs_cover(const T* X, int64_t n, int64_t c0, int64_t c1) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(X);
  const uintptr_t a = reinterpret_cast<uintptr_t>(X + c0) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(X + c1) + 15) & ~uintptr_t(15);
  QsCover<T> cv;
  cv.src = reinterpret_cast<const T*>(a);
  cv.phase = (int)((reinterpret_cast<uintptr_t>(X + c0) - a) / sizeof(T));
  cv.bytes = (uint32_t)(e - a);
  cv.ok = c1 > c0 && a >= x && e <= reinterpret_cast<uintptr_t>(X + n) && x % sizeof(T) == 0;
  return cv;
}
// staging buffer sizes: a chunk plus the cover's slack
template <class T>
__host__ __device__ constexpr int qs_stage_elems() { return kQsChunk + 32 / (int)sizeof(T); }

template <class Key>
__host__ __device__ constexpr int qs_count_smem() {
  return qs_table_bytes<Key>() + qs_stage_elems<Key>() * (int)sizeof(Key);
}

template <class Key>
__global__ void __launch_bounds__(kQsNT, 2) qs_count_kernel(QsCtx<Key> c, int level) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char qs_raw[];
  __shared__ uint32_t hist[2 * kQsMaxB];
  __shared__ __align__(8) uint64_t bar;
  Key* stage = reinterpret_cast<Key*>(qs_raw + qs_table_bytes<Key>());
  const int tid = threadIdx.x;
  const Key* X = qs_src(c, level);
  const int64_t nch = qs_nchunk(c, level);
  int64_t cur = -1;  // segment whose tables are loaded
  QsClassifier<Key> cls{};
  // contiguous chunk ranges per CTA: neighbouring chunks share a segment, so
  // the tables are reloaded only when the segment changes
  const int64_t per = (nch + gridDim.x - 1) / gridDim.x;
  const int64_t ch_begin = (int64_t)blockIdx.x * per;
  const int64_t ch_end = min(nch, ch_begin + per);
  auto range = [&](int64_t ch, int64_t& c0, int64_t& c1) {
    const QsSeg g = qs_seg(c, level, qs_seg_of_chunk(c, level, ch));
    c0 = g.start + (ch - g.chunk0) * kQsChunk;
    c1 = min(g.start + g.len, c0 + kQsChunk);
  };
  auto issue = [&](int64_t ch) {  // thread 0: stage chunk ch
    int64_t c0, c1;
    range(ch, c0, c1);
    const QsCover<Key> cv = qs_cover(X, c.n, c0, c1);
    if (cv.ok) {
      fence_proxy_async_smem();  // the previous chunk's generic reads of the buffer are done
      mbar_arrive_expect_tx(&bar, cv.bytes);
      tma_load_1d(stage, cv.src, cv.bytes, &bar);
    }
  };
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && ch_begin < ch_end) issue(ch_begin);
  uint32_t parity = 0;
  for (int64_t ch = ch_begin; ch < ch_end; ++ch) {
    const int64_t sid = qs_seg_of_chunk(c, level, ch);
    const QsSeg g = qs_seg(c, level, sid);
    const int NB = 2 * g.B - 1;
    const int64_t c0 = g.start + (ch - g.chunk0) * kQsChunk;
    const int64_t c1 = min(g.start + g.len, c0 + kQsChunk);
    const int cnt = (int)(c1 - c0);
    const QsCover<Key> cv = qs_cover(X, c.n, c0, c1);
    // this chunk's keys -> registers (from the staging buffer when staged)
    Key k[kQsPer];
    if (cv.ok) {
      mbar_wait(&bar, parity);
      parity ^= 1u;
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {
        const int j = u * kQsNT + tid;
        k[u] = j < cnt ? stage[cv.phase + j] : Key(0);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {
        const int j = u * kQsNT + tid;
        k[u] = j < cnt ? __ldg(X + c0 + j) : Key(0);
      }
    }
    __syncthreads();  // buffer, tables and hist free: the previous chunk is done
    if (tid == 0 && ch + 1 < ch_end) issue(ch + 1);  // overlaps this chunk's work
    if (sid != cur) {
      cls = qs_load_classifier<Key>(qs_raw, c.spl[level & 1] + g.spl_off,
                                    c.cells[level & 1] + 16 * g.spl_off, g.B);
      cur = sid;
    }
    for (int i = tid; i < NB; i += kQsNT) hist[i] = 0;
    __syncthreads();
    uint8_t* idp = c.ids + c0 + tid;
    if (cnt == kQsChunk) {  // full chunk (all but a segment's last): no per-key guard
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {
        const int b = cls(k[u]);
        NSB_DCHECK(b >= 0 && b < 2 * cls.B - 1);
        idp[u * kQsNT] = (uint8_t)b;
        atomicAdd(&hist[b], 1u);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {
        const int j = u * kQsNT + tid;
        const bool in = j < cnt;
        const int b = in ? cls(k[u]) : -1;
        NSB_DCHECK(b < 2 * cls.B - 1);
        if (in) idp[u * kQsNT] = (uint8_t)b;
        qs_hist_add(hist, b);
      }
    }
    __syncthreads();
    uint32_t* cn = c.cnt[level & 1] + g.cnt_off;
    uint16_t* chh = c.chist + ch * kQsHistStride;  // a chunk holds <= 8192 keys: counts fit 16 bits
    for (int b = tid; b < NB; b += kQsNT) {
      const uint32_t h = hist[b];
      chh[b] = (uint16_t)h;
      if (h) atomicAdd(&cn[b], h);
    }
  }
}

// ---- 3. plan ---------------------------------------------------------------------
// Block-wide exclusive scan of one value per thread (kQsNT threads) under an
// associative op with identity `id`.
template <class T, class Op>
__device__ __forceinline__ T qs_block_scan(T v, T id, Op op, T* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x = op(y, x);
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T t = lane < kQsNT / 32 ? warp_tot[lane] : id;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(kFull, t, o);
      if (lane >= o) t = op(y, t);
    }
    if (lane < kQsNT / 32) warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  T ex = __shfl_up_sync(kFull, x, 1);
  if (lane == 0) ex = id;
  const T r = warp > 0 ? op(warp_tot[warp - 1], ex) : ex;
  __syncthreads();  // warp_tot is reused by the caller's next scan
  return r;
}
__device__ __forceinline__ int64_t qs_block_scan(uint32_t v, int64_t* warp_tot) {
  return qs_block_scan<int64_t>((int64_t)v, 0, [](int64_t a, int64_t b) { return a + b; },
                                warp_tot);
}

#ifndef NSB_QS_PACK
#define NSB_QS_PACK 4096
#endif
// Leaf packing: neighbouring buckets of <= kQsPack keys whose start offsets
// in the segment fall in the same window of W keys form one leaf job, so a
// job is < W + kQsPack keys; the rule is evaluated by every bucket in
// parallel.
constexpr int kQsPack = NSB_QS_PACK;
static_assert(2 * kQsPack <= kSmallTile, "packed jobs must fit one tile");

__device__ __forceinline__ int qs_class_of(int64_t len) {
  return len <= 4096 ? 0 : len <= 8192 ? 1 : 2;
}

template <class Key>
__global__ void __launch_bounds__(kQsNT) qs_plan_kernel(QsCtx<Key> c, int level, int last) {
  pdl_wait();
  pdl_trigger();
  __shared__ int64_t s_wtot[kQsNT / 32];
  __shared__ uint32_t s_cnt[kQsNT];
  __shared__ int64_t s_pos[kQsNT];
  __shared__ uint8_t s_flag[kQsNT];  // 0 empty, 1 packed member, 2 job head, 3 big
  __shared__ uint32_t s_ccnt[3], s_nn;
  __shared__ uint32_t s_chunks, s_bk, s_sp;  // per segment: < 2^32 (32-bit shared atomics)
  __shared__ unsigned long long s_jbase[3], s_sbase, s_kbase, s_bbase, s_pbase;
  const int tid = threadIdx.x;
  const int nx = (level + 1) & 1;
  // buckets of this level land in Y_l (the scatter destination): tmp at even levels
  const int src_flag = (level & 1) ? 0 : 1;
  const int64_t nseg = qs_nseg(c, level);
  for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const QsSeg g = qs_seg(c, level, s);
    const int NB = 2 * g.B - 1;
    const uint32_t v = tid < NB ? __ldcg(c.cnt[level & 1] + g.cnt_off + tid) : 0u;
    const int64_t pos = g.start + qs_block_scan(v, s_wtot);
    // previous non-empty bucket (exclusive max-scan of indices)
    const int64_t prev = qs_block_scan<int64_t>(v ? tid : -1, -1,
                                                [](int64_t a, int64_t b) { return a > b ? a : b; },
                                                s_wtot);
    s_cnt[tid] = v;
    s_pos[tid] = pos;
    if (tid < NB) c.fill[level & 1][g.cnt_off + tid] = (unsigned long long)pos;
    if (tid == 0) {
      s_ccnt[0] = s_ccnt[1] = s_ccnt[2] = 0;
      s_nn = 0;
      s_chunks = s_bk = s_sp = 0;
    }
    __syncthreads();
    const bool small = v > 0 && v <= (uint32_t)kQsPack;
    // (W = kQsWinBig from kQsBigLeafN keys measured slower: 16M random
    // 0.45 -> 0.49 ms, the 16384-key leaf tiles cost more than they save)
    const int64_t W = kQsPack;
    const int64_t win = (pos - g.start) / W;
    bool head = false;
    if (small) {
      head = prev < 0 || s_cnt[prev] > (uint32_t)kQsPack || (s_pos[prev] - g.start) / W != win;
    }
    s_flag[tid] = head ? 2 : small ? 1 : v > 0 ? 3 : 0;
    __syncthreads();
    // this thread's job (packed run, own bucket, copy, fallback) or new segment
    int cls = -1, type = kJobSort;
    int64_t jstart = pos, jlen = 0;
    uint32_t jlocal = 0, njob = 1;
    int32_t nB = 0, nch = 0;
    uint32_t slocal = 0;
    uint32_t koff = 0, boff = 0, poff = 0;
    if (head) {
      int b = tid + 1;
      while (b < NB && s_flag[b] <= 1) ++b;
      jlen = (b < NB ? s_pos[b] : g.start + g.len) - pos;
      cls = qs_class_of(jlen);
    } else if (v > (uint32_t)kQsPack) {
      jlen = v;
      if (v <= (uint32_t)kSmallTile) {
        cls = qs_class_of(jlen);
      } else if (tid & 1) {  // constant bucket: already sorted; moved only if it sits in tmp
        if (src_flag) {
          cls = 2;
          type = kJobCopy;
          // a big constant bucket is copied by many CTAs, kQsCopyChunk keys each
          // (one job per bucket made all-equal input 25x slower than random)
          njob = (uint32_t)((jlen + kQsCopyChunk - 1) / kQsCopyChunk);
        }
      } else if (!last) {
        nB = qs_buckets(jlen);
        nch = (int32_t)((jlen + kQsChunk - 1) / kQsChunk);
        slocal = atomicAdd(&s_nn, 1u);
        koff = atomicAdd(&s_chunks, (uint32_t)nch);
        boff = atomicAdd(&s_bk, (uint32_t)(2 * nB - 1));
        poff = atomicAdd(&s_sp, (uint32_t)nB);
      } else {
        cls = 2;
        type = kJobBig;
      }
    }
    if (cls >= 0) jlocal = atomicAdd(&s_ccnt[cls], njob);
    __syncthreads();
    if (tid < 3) s_jbase[tid] = s_ccnt[tid] ? atomicAdd(&c.ctr->njobs[tid], (unsigned long long)s_ccnt[tid]) : 0ull;
    if (tid == 3 && s_nn) {
      s_sbase = atomicAdd(&c.ctr->nseg[nx], (unsigned long long)s_nn);
      s_kbase = atomicAdd(&c.ctr->nchunk[nx], (unsigned long long)s_chunks);
      s_bbase = atomicAdd(&c.ctr->nbkt[nx], (unsigned long long)s_bk);
      s_pbase = atomicAdd(&c.ctr->nspl[nx], (unsigned long long)s_sp);
    }
    __syncthreads();
    if (cls >= 0) {
      const unsigned long long at = s_jbase[cls] + jlocal;
      NSB_DCHECK(at + njob <= (unsigned long long)c.max_jobs);
      if (njob == 1) {
        if (at < (unsigned long long)c.max_jobs)
          c.jobs[cls][at] = QsJob{jstart, jlen, src_flag | (type << 1), 0};
      } else {
        for (uint32_t q = 0; q < njob; ++q)
          if (at + q < (unsigned long long)c.max_jobs)
            c.jobs[cls][at + q] =
                QsJob{jstart + (int64_t)q * kQsCopyChunk,
                      min((int64_t)kQsCopyChunk, jlen - (int64_t)q * kQsCopyChunk),
                      src_flag | (type << 1), 0};
      }
    }
    if (nB) {
      const unsigned long long sid = s_sbase + slocal, k0 = s_kbase + koff;
      NSB_DCHECK(sid < (unsigned long long)c.max_segs && k0 + nch <= (unsigned long long)c.max_chunks &&
                 s_bbase + boff + 2 * nB - 1 <= (unsigned long long)c.max_bkt &&
                 s_pbase + poff + nB <= (unsigned long long)c.max_spl);
      if (sid < (unsigned long long)c.max_segs) {
        QsSeg ns;
        ns.start = jstart;
        ns.len = jlen;
        ns.chunk0 = (int64_t)k0;
        ns.cnt_off = (int64_t)(s_bbase + boff);
        ns.spl_off = (int64_t)(s_pbase + poff);
        ns.B = nB;
        ns.nchunks = nch;
        c.segs[nx][sid] = ns;
        for (int j = 0; j < nch; ++j)
          if (k0 + j < (unsigned long long)c.max_chunks) c.chunk_seg[nx][k0 + j] = (int32_t)sid;
      }
    }
    __syncthreads();
  }
}

// ---- 4. scatter (shared-memory multisplit, coalesced bucket runs) -------------
template <class Key>
__host__ __device__ constexpr int qs_scatter_smem() {
  return kQsChunk * (int)sizeof(Key) + kQsChunk;  // keys + one-byte bucket ids
}

#ifndef NSB_QS_SCATTER_MINB
#define NSB_QS_SCATTER_MINB 2
#endif
template <class Key>
__global__ void __launch_bounds__(kQsNT, NSB_QS_SCATTER_MINB) qs_scatter_kernel(QsCtx<Key> c, int level) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t hist[2 * kQsMaxB];    // counts, then local starts
  __shared__ long long delta[2 * kQsMaxB];  // global position - local start
  __shared__ int64_t wtot[kQsNT / 32];
  extern __shared__ __align__(16) unsigned char qs_raw[];
  Key* skey = reinterpret_cast<Key*>(qs_raw);
  uint8_t* sbid = qs_raw + kQsChunk * sizeof(Key);
  const int tid = threadIdx.x, lane = tid & 31;
  const Key* X = qs_src(c, level);
  Key* Y = qs_src(c, level + 1);
  const int64_t nch = qs_nchunk(c, level);
  const int64_t per = (nch + gridDim.x - 1) / gridDim.x;  // contiguous chunk ranges
  const int64_t ch_end = min(nch, ((int64_t)blockIdx.x + 1) * per);
  for (int64_t ch = (int64_t)blockIdx.x * per; ch < ch_end; ++ch) {
    const QsSeg g = qs_seg(c, level, qs_seg_of_chunk(c, level, ch));
    const int NB = 2 * g.B - 1;
    const int64_t c0 = g.start + (ch - g.chunk0) * kQsChunk;
    const int64_t c1 = min(g.start + g.len, c0 + kQsChunk);
    // this chunk's keys and ids: in flight while the bucket starts are set up
    Key k[kQsPer];
    int b[kQsPer];
#pragma unroll
    for (int u = 0; u < kQsPer; ++u) {
      const int64_t i = c0 + u * kQsNT + tid;
      const bool in = i < c1;
      k[u] = in ? __ldcs(X + i) : Key(0);
      b[u] = in ? (int)__ldcs(c.ids + i) : -1;
    }
    // The count kernel left this chunk's bucket counts: their exclusive scan
    // gives every bucket's start in the staged chunk BEFORE any key is ranked,
    // so one shared atomic per key returns its final staging position (no
    // second pass over the keys, no rank kept in registers), and the global
    // range of every bucket is reserved up front (one atomic per bucket whose
    // round trip hides under the ranking).
    const uint32_t cnt = tid < NB ? (uint32_t)__ldcg(c.chist + ch * kQsHistStride + tid) : 0u;
    __syncthreads();  // the previous chunk's write-out is done with hist / delta / the stage
    const int64_t ls = qs_block_scan(cnt, wtot);
    unsigned long long* fill = c.fill[level & 1] + g.cnt_off;
    unsigned long long gb = 0ull;
    if (tid < NB) {
      if (cnt) gb = atomicAdd(&fill[tid], (unsigned long long)cnt);
      hist[tid] = (uint32_t)ls;
    }
    __syncthreads();
    const int total = (int)(c1 - c0);
    const bool full = total == kQsChunk;  // all but a segment's last chunk: no per-key guards
    const uint32_t hist_s = (uint32_t)__cvta_generic_to_shared(hist);
    if (full) {
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {
        int uni;
        __match_all_sync(kFull, b[u], &uni);
        uint32_t p;
        if (uni) {  // one bucket for the whole warp (sorted input): one atomic for 32 keys
          uint32_t base = 0;
          // (plain PTX: nvcc wraps a one-lane atomicAdd in its own warp aggregation)
          if (lane == 0)
            asm volatile("atom.shared.add.u32 %0, [%1], 32;"
                         : "=r"(base)
                         : "r"(hist_s + 4u * (uint32_t)b[u])
                         : "memory");
          p = __shfl_sync(kFull, base, 0) + (uint32_t)lane;
        } else {
          p = atomicAdd(&hist[b[u]], 1u);
        }
        NSB_DCHECK(b[u] >= 0 && b[u] < NB && p < (uint32_t)kQsChunk);
        skey[p] = k[u];
        sbid[p] = (uint8_t)b[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {  // a segment's last chunk: absent keys have b = -1
        int uni;
        __match_all_sync(kFull, b[u], &uni);
        uint32_t p = 0;
        if (uni) {
          uint32_t base = 0;
          if (lane == 0 && b[u] >= 0)
            asm volatile("atom.shared.add.u32 %0, [%1], 32;"
                         : "=r"(base)
                         : "r"(hist_s + 4u * (uint32_t)b[u])
                         : "memory");
          p = __shfl_sync(kFull, base, 0) + (uint32_t)lane;
        } else if (b[u] >= 0) {
          p = atomicAdd(&hist[b[u]], 1u);
        }
        if (b[u] >= 0) {
          NSB_DCHECK(b[u] < NB && p < (uint32_t)total);
          skey[p] = k[u];
          sbid[p] = (uint8_t)b[u];
        }
      }
    }
    if (tid < NB) delta[tid] = (long long)gb - (long long)ls;
    __syncthreads();
    if (full) {
#pragma unroll
      for (int u = 0; u < kQsPer; ++u) {
        const int i = u * kQsNT + tid;
        // every key lands inside its segment (the reserved bucket ranges)
        NSB_DCHECK(delta[sbid[i]] + i >= g.start && delta[sbid[i]] + i < g.start + g.len);
        Y[delta[sbid[i]] + i] = skey[i];
      }
    } else {
      for (int i = tid; i < total; i += kQsNT) {
        NSB_DCHECK(delta[sbid[i]] + i >= g.start && delta[sbid[i]] + i < g.start + g.len);
        Y[delta[sbid[i]] + i] = skey[i];
      }
    }
  }
}

// ---- 5. leaf jobs ---------------------------------------------------------------
// One CTA sorts a segment of any length in global memory (the fallback for a
// bucket still larger than one CTA after the last level): tiles sorted on
// chip, then pairwise merges of runs ping-ponging between the two buffers'
// ranges, the last pass landing in `keys`.  Plain loads/stores only (every
// key is re-read by this same CTA).
template <int NT, int K, int LEAF, class Key>
__device__ void qs_big_sort(Key* keys, Key* tmp, int64_t st, int64_t len, bool src_tmp, Key* sm) {
  static_assert(cta_sort_skewed<NT, K, Key>(), "the fallback reads the skewed tile from smem");
  constexpr int T = NT * K;
  const int tid = threadIdx.x;
  const int64_t tiles = (len + T - 1) / T;
  int passes = 0;
  for (int64_t r = tiles; r > 1; r = (r + 1) / 2) ++passes;
  Key* kb = keys + st;
  Key* tb = tmp + st;
  const Key* src = src_tmp ? tb : kb;
  Key* A = (passes & 1) ? tb : kb;
  Key* Bf = (passes & 1) ? kb : tb;
  for (int64_t t = 0; t < tiles; ++t) {
    const int valid = (int)min((int64_t)T, len - t * T);
    cta_sort<NT, K, LEAF>(src + t * T, (Key*)nullptr, valid, sm);
    __syncthreads();
    for (int i = tid; i < valid; i += NT) A[t * T + i] = sm[i];
    __syncthreads();
  }
  __shared__ int64_t s_split[2];
  constexpr int M = NT * 4;  // outputs per merge chunk, 4 per thread
  for (int64_t R = T; R < len; R *= 2) {
    for (int64_t p = 0; p < len; p += 2 * R) {
      const Key* a = A + p;
      const int64_t la = min(R, len - p);
      const Key* b = a + la;
      const int64_t lb = max((int64_t)0, min(R, len - p - R));
      for (int64_t d0 = 0; d0 < la + lb; d0 += M) {
        const int64_t d1 = min(d0 + M, la + lb);
        if (tid < 2) {
          const int64_t d = tid ? d1 : d0;
          int64_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldcg(a + mid) <= __ldcg(b + d - 1 - mid)) lo = mid + 1;
            else hi = mid;
          }
          s_split[tid] = lo;
        }
        __syncthreads();
        const int64_t a0 = s_split[0], a1 = s_split[1];
        const int na = (int)(a1 - a0), nb = (int)((d1 - a1) - (d0 - a0));
        for (int i = tid; i < na; i += NT) sm[i] = __ldcg(a + a0 + i);
        for (int i = tid; i < nb; i += NT) sm[na + i] = __ldcg(b + (d0 - a0) + i);
        __syncthreads();
        const int dd = min(tid * 4, na + nb);
        int lo = dd > nb ? dd - nb : 0, hi = dd < na ? dd : na;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (sm[mid] <= sm[na + dd - 1 - mid]) lo = mid + 1;
          else hi = mid;
        }
        int ia = lo, ib = dd - lo;
        for (int k = 0; k < 4 && dd + k < na + nb; ++k) {
          const bool ta = ib >= nb || (ia < na && sm[ia] <= sm[na + ib]);
          Bf[p + d0 + dd + k] = ta ? sm[ia++] : sm[na + ib++];
        }
        __syncthreads();
      }
    }
    std::swap(A, Bf);
  }
}

template <int NT, int K, int LEAF, class Key>
__global__ void __launch_bounds__(NT, (bs_min_blocks_tput<NT, K, Key>()))
    qs_leaf_kernel(QsCtx<Key> c, int cls) {
  extern __shared__ __align__(16) unsigned char qs_raw[];
  Key* sm = reinterpret_cast<Key*>(qs_raw);
  const int64_t nj = (int64_t)*(volatile unsigned long long*)&c.ctr->njobs[cls];
  const QsJob* jobs = c.jobs[cls];
  for (int64_t j = blockIdx.x; j < nj; j += gridDim.x) {
    const QsJob jb = jobs[j];
    const bool src_tmp = jb.flags & 1;
    const int type = (jb.flags >> 1) & 3;
    NSB_DCHECK(jb.start >= 0 && jb.len >= 0 && jb.start + jb.len <= c.n &&
               (type != kJobSort || jb.len <= (int64_t)NT * K));
    const Key* src = (src_tmp ? c.tmp : c.keys) + jb.start;
    Key* dst = c.keys + jb.start;
    if (type == kJobSort) {
      cta_sort<NT, K, LEAF>(src, dst, (int)jb.len, sm);
    } else if (type == kJobCopy) {
      for (int64_t i = threadIdx.x; i < jb.len; i += NT) dst[i] = src[i];
    } else {
      if constexpr (cta_sort_skewed<NT, K, Key>()) qs_big_sort<NT, K, LEAF>(c.keys, c.tmp, jb.start, jb.len, src_tmp, sm);
    }
    __syncthreads();
  }
}

// ---- host side ---------------------------------------------------------------------
constexpr int64_t kQsPdlMaxKeys = int64_t(1) << 22;
// Side streams + fork/join events for the concurrent leaf classes: one set
// per (host thread, device), so concurrent callers never share an event.
struct QsSide {
  cudaStream_t s[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
};
struct QsSideSet {
  QsSide d[64];
  ~QsSideSet() {
    for (auto& x : d) {
      for (int i = 0; i < 2; ++i) {
        if (x.s[i]) cudaStreamDestroy(x.s[i]);
        if (x.join[i]) cudaEventDestroy(x.join[i]);
      }
      if (x.fork) cudaEventDestroy(x.fork);
    }
  }
};
static thread_local QsSideSet t_side;

static int qs_side_streams(QsSide** out) {
  int dev = 0;
  NSB_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  if (dev < 0 || dev >= 64) return NS_ERR_INVALID;
  QsSide& x = t_side.d[dev];
  if (!x.fork) {
    for (int i = 0; i < 2; ++i) {
      NSB_TRY(check_cuda(cudaStreamCreateWithFlags(&x.s[i], cudaStreamNonBlocking), "cudaStreamCreate"));
      NSB_TRY(check_cuda(cudaEventCreateWithFlags(&x.join[i], cudaEventDisableTiming), "cudaEventCreate"));
    }
    NSB_TRY(check_cuda(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming), "cudaEventCreate"));
  }
  *out = &x;
  return NS_OK;
}

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Resident CTAs per SM of a kernel at (threads, dynamic smem), cached per device.
static int occupancy(const void* kern, int nt, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void*>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& e : cache)
    if (e.first.first == dev && e.first.second == kern) return e.second;
  int b = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, nt, smem) != cudaSuccess || b < 1) b = 1;
  cache.push_back({{dev, kern}, b});
  return b;
}

static unsigned grid_of(const void* kern, int nt, int smem, int64_t upper) {
  const int64_t g = (int64_t)sm_count() * occupancy(kern, nt, smem);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, upper));
}

struct QsSizes {
  int64_t max_segs, max_chunks, max_bkt, max_spl, max_jobs;
};

static QsSizes qs_sizes(int64_t nseg0, int64_t len0) {
  const int64_t n = nseg0 * len0;
  const int levels = qs_levels(len0);
  QsSizes z;
  // level >= 1 segments are buckets of > kSmallTile keys; level 0 is given
  z.max_segs = std::max<int64_t>(nseg0, n / (kSmallTile + 1) + 1);
  z.max_chunks = n / kQsChunk + z.max_segs + 1;
  // 2B-1 <= 4 len / kQsTarget + 3 buckets, B <= 2 len / kQsTarget + 2 pivots
  z.max_bkt = std::max<int64_t>(nseg0 * (2 * qs_buckets(len0) - 1), 4 * n / kQsTarget + 3 * z.max_segs) + 64;
  z.max_spl = std::max<int64_t>(nseg0 * qs_buckets(len0), 2 * n / kQsTarget + 2 * z.max_segs) + 64;
  // every job holds at least one non-empty bucket of one level
  z.max_jobs = std::max<int64_t>(nseg0 * (2 * qs_buckets(len0) - 1), 0) +
               (int64_t)levels * (4 * n / kQsTarget + 3 * z.max_segs) + 64;
  // plus the extra copy jobs of big constant buckets (one per kQsCopyChunk keys)
  z.max_jobs += (int64_t)levels * (n / kQsCopyChunk + 1);
  return z;
}

template <class Key>
static size_t qs_temp_bytes(int64_t nseg0, int64_t len0) {
  const int64_t n = nseg0 * len0;
  const QsSizes z = qs_sizes(nseg0, len0);
  size_t b = align_up((size_t)n * sizeof(Key), 256) + align_up(sizeof(QsCounters), 256);
  b += align_up((size_t)n, 256);
  b += align_up((size_t)z.max_chunks * kQsHistStride * 2, 256);
  b += 2 * align_up((size_t)z.max_segs * sizeof(QsSeg), 256);
  b += 2 * align_up((size_t)z.max_chunks * 4, 256);
  b += 2 * align_up((size_t)z.max_spl * sizeof(Key), 256);
  b += 2 * align_up((size_t)z.max_spl * 16 * 2, 256);
  b += 2 * align_up((size_t)z.max_bkt * 4, 256);
  b += 2 * align_up((size_t)z.max_bkt * 8, 256);
  b += 3 * align_up((size_t)z.max_jobs * sizeof(QsJob), 256);
  return b;
}

template <class Key>
static QsCtx<Key> qs_carve(Key* keys, void* d_temp, int64_t nseg0, int64_t len0) {
  const int64_t n = nseg0 * len0;
  const QsSizes z = qs_sizes(nseg0, len0);
  char* p = static_cast<char*>(d_temp);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align_up(bytes, 256);
    return r;
  };
  QsCtx<Key> c;
  c.keys = keys;
  c.tmp = reinterpret_cast<Key*>(take((size_t)n * sizeof(Key)));
  c.n = n;
  c.nseg0 = nseg0;
  c.len0 = len0;
  c.cps0 = (len0 + kQsChunk - 1) / kQsChunk;
  c.B0 = qs_buckets(len0);
  c.ctr = reinterpret_cast<QsCounters*>(take(sizeof(QsCounters)));
  c.ids = reinterpret_cast<uint8_t*>(take((size_t)n));
  c.chist = reinterpret_cast<uint16_t*>(take((size_t)z.max_chunks * kQsHistStride * 2));
  for (int i = 0; i < 2; ++i) c.segs[i] = reinterpret_cast<QsSeg*>(take((size_t)z.max_segs * sizeof(QsSeg)));
  for (int i = 0; i < 2; ++i) c.chunk_seg[i] = reinterpret_cast<int32_t*>(take((size_t)z.max_chunks * 4));
  for (int i = 0; i < 2; ++i) c.spl[i] = reinterpret_cast<Key*>(take((size_t)z.max_spl * sizeof(Key)));
  for (int i = 0; i < 2; ++i) c.cells[i] = reinterpret_cast<uint16_t*>(take((size_t)z.max_spl * 16 * 2));
  for (int i = 0; i < 2; ++i) c.cnt[i] = reinterpret_cast<uint32_t*>(take((size_t)z.max_bkt * 4));
  for (int i = 0; i < 2; ++i) c.fill[i] = reinterpret_cast<unsigned long long*>(take((size_t)z.max_bkt * 8));
  for (int i = 0; i < 3; ++i) c.jobs[i] = reinterpret_cast<QsJob*>(take((size_t)z.max_jobs * sizeof(QsJob)));
  c.max_segs = z.max_segs;
  c.max_chunks = z.max_chunks;
  c.max_bkt = z.max_bkt;
  c.max_spl = z.max_spl;
  c.max_jobs = z.max_jobs;
  return c;
}

// Leaf tile shapes per class (4096 / 8192 / 16384 keys): int32 at 32 keys per
// thread, int64 at 16.
template <class Key, int CLS> struct QsLeafShape;
template <> struct QsLeafShape<int32_t, 0> { static constexpr int NT = 128, K = 32; };
template <> struct QsLeafShape<int32_t, 1> { static constexpr int NT = 256, K = 32; };
template <> struct QsLeafShape<int32_t, 2> { static constexpr int NT = 512, K = 32; };
template <> struct QsLeafShape<int64_t, 0> { static constexpr int NT = 256, K = 16; };
template <> struct QsLeafShape<int64_t, 1> { static constexpr int NT = 512, K = 16; };
template <> struct QsLeafShape<int64_t, 2> { static constexpr int NT = 1024, K = 16; };

template <int CLS, int LF, class Key>
static int qs_launch_leaf(const QsCtx<Key>& c, int64_t upper, cudaStream_t s) {
  constexpr int NT = QsLeafShape<Key, CLS>::NT, K = QsLeafShape<Key, CLS>::K;
  constexpr int smem = tile_smem_bytes<NT, K, Key>();
  auto* kern = qs_leaf_kernel<NT, K, LF, Key>;
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(qs_leaf)"));
  {
    Prof prof(PK_QS_BUCKET, s);
    kern<<<grid_of(reinterpret_cast<const void*>(kern), NT, smem, upper), NT, smem, s>>>(c, CLS);
  }
  return check_launch("qs_leaf_kernel");
}

// Sorts nseg0 back-to-back segments of len0 (> kSmallTile) keys each.
template <class Key>
static int quick_sort_segments(Key* keys, int64_t nseg0, int64_t len0, int leaf, void* d_temp,
                               size_t temp_bytes, cudaStream_t s) {
  if (!d_temp || temp_bytes < qs_temp_bytes<Key>(nseg0, len0)) return NS_ERR_TEMP;
  const QsCtx<Key> c = qs_carve<Key>(keys, d_temp, nseg0, len0);
  const QsSizes z = qs_sizes(nseg0, len0);
  const int levels = qs_levels(len0);
  constexpr int sample_smem = 0;
  constexpr int scatter_smem = qs_scatter_smem<Key>();
  constexpr int count_smem = qs_count_smem<Key>();
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(qs_count_kernel<Key>), count_smem,
                           "cudaFuncSetAttribute(qs_count)"));
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(qs_scatter_kernel<Key>), scatter_smem,
                           "cudaFuncSetAttribute(qs_scatter)"));
  // programmatic dependent launch between the per-level kernels of
  // latency-bound sorts (every kernel waits for its predecessor on entry;
  // only the launch and CTA rasterisation overlap)
  const bool pdl = pdl_enabled(nseg0 * len0 >= kQsPdlMaxKeys ? INT64_MAX : 0);
  for (int l = 0; l < levels; ++l) {
    const int64_t segs_ub = l == 0 ? nseg0 : z.max_segs;
    const int64_t chunks_ub = l == 0 ? nseg0 * c.cps0 : z.max_chunks;
    {
      Prof prof(PK_QS_SAMPLE, s);
      NSB_TRY(check_cuda(launch_pdl_if(pdl, qs_sample_kernel<Key>,
                                       grid_of(reinterpret_cast<const void*>(qs_sample_kernel<Key>), 256,
                                               sample_smem, segs_ub),
                                       256, sample_smem, s, c, l),
                         "qs_sample_kernel"));
    }
    NSB_TRY(check_launch("qs_sample_kernel"));
    {
      Prof prof(PK_QS_COUNT, s);
      NSB_TRY(check_cuda(launch_pdl_if(pdl, qs_count_kernel<Key>,
                                       grid_of(reinterpret_cast<const void*>(qs_count_kernel<Key>), kQsNT,
                                               count_smem, chunks_ub),
                                       kQsNT, count_smem, s, c, l),
                         "qs_count_kernel"));
    }
    NSB_TRY(check_launch("qs_count_kernel"));
    {
      Prof prof(PK_QS_PLAN, s);
      NSB_TRY(check_cuda(launch_pdl_if(pdl, qs_plan_kernel<Key>,
                                       grid_of(reinterpret_cast<const void*>(qs_plan_kernel<Key>), kQsNT, 0,
                                               segs_ub),
                                       kQsNT, 0, s, c, l, (int)(l == levels - 1)),
                         "qs_plan_kernel"));
    }
    NSB_TRY(check_launch("qs_plan_kernel"));
    {
      Prof prof(PK_QS_SCATTER, s);
      NSB_TRY(check_cuda(launch_pdl_if(pdl, qs_scatter_kernel<Key>,
                                       grid_of(reinterpret_cast<const void*>(qs_scatter_kernel<Key>), kQsNT,
                                               scatter_smem, chunks_ub),
                                       kQsNT, scatter_smem, s, c, l),
                         "qs_scatter_kernel"));
    }
    NSB_TRY(check_launch("qs_scatter_kernel"));
  }
  // The three leaf classes are independent: they run concurrently on two
  // side streams forked from (and joined back into) the caller's stream, so
  // a small sort pays one tile-sort latency instead of three (the fork/join
  // is event-based and therefore also valid inside a CUDA-graph capture).
  QsSide* side = nullptr;
  NSB_TRY(qs_side_streams(&side));
  NSB_TRY(check_cuda(cudaEventRecord(side->fork, s), "cudaEventRecord(fork)"));
  for (int i = 0; i < 2; ++i)
    NSB_TRY(check_cuda(cudaStreamWaitEvent(side->s[i], side->fork, 0), "cudaStreamWaitEvent"));
  NSB_TRY(with_leaf(leaf, [&](auto L) {
    constexpr int LF = decltype(L)::value;
    NSB_TRY((qs_launch_leaf<0, LF>(c, z.max_jobs, side->s[0])));
    NSB_TRY((qs_launch_leaf<1, LF>(c, z.max_jobs, side->s[1])));
    return qs_launch_leaf<2, LF>(c, z.max_jobs, s);
  }));
  for (int i = 0; i < 2; ++i) {
    NSB_TRY(check_cuda(cudaEventRecord(side->join[i], side->s[i]), "cudaEventRecord(join)"));
    NSB_TRY(check_cuda(cudaStreamWaitEvent(s, side->join[i], 0), "cudaStreamWaitEvent"));
  }
  return NS_OK;
}

// The quick sort's base case.  Its recursion bottoms out where partitioning
// stops paying: an array (or segment) of up to qs_base_max() keys is finished
// by the merge layer — tile sort plus a few pairwise passes — instead of a
// partition level and bucket sorts.  Measured by graph replay (tools/
// qs_vs_ms.py): one partition level is a chain of five latency-bound kernels
// (38-45 us from 24 K to 512 K keys against 21-42 us for the merge layer; at
// 16385 keys 38 vs 16 us).  Default 2^19; NSB_QS_BASE_MAX overrides it (the
// tests set 16384 so that every partition path also runs at small sizes).
size_t qs_base_max() {
  static const size_t v = [] {
    const char* e = getenv("NSB_QS_BASE_MAX");
    const long long x = e ? atoll(e) : (1ll << 19);
    return (size_t)std::max<long long>(x, kSmallTile);
  }();
  return v;
}

size_t quick_sort_temp(size_t n) {
  if (n <= (size_t)kSmallTile) return merge_sort_temp(n);
  if (n <= qs_base_max()) return std::max(merge_sort_temp(n), qs_temp_bytes<int32_t>(1, (int64_t)n));
  return qs_temp_bytes<int32_t>(1, (int64_t)n);
}
size_t quick_sort_temp_i64(size_t n) {
  if (n <= (size_t)kSmallTile) return merge_sort_temp_i64(n);
  if (n <= qs_base_max()) return std::max(merge_sort_temp_i64(n), qs_temp_bytes<int64_t>(1, (int64_t)n));
  return qs_temp_bytes<int64_t>(1, (int64_t)n);
}
size_t quick_sort_segments_temp(size_t nseg, size_t len, size_t key_bytes) {
  if (len <= (size_t)kSmallTile) return 0;
  return key_bytes == 8 ? qs_temp_bytes<int64_t>((int64_t)nseg, (int64_t)len)
                        : qs_temp_bytes<int32_t>((int64_t)nseg, (int64_t)len);
}
int quick_sort_segments_device(int32_t* keys, size_t nseg, size_t len, int leaf, void* d_temp,
                               size_t temp_bytes, cudaStream_t s) {
  return quick_sort_segments(keys, (int64_t)nseg, (int64_t)len, leaf, d_temp, temp_bytes, s);
}
int quick_sort_segments_device(int64_t* keys, size_t nseg, size_t len, int leaf, void* d_temp,
                               size_t temp_bytes, cudaStream_t s) {
  return quick_sort_segments(keys, (int64_t)nseg, (int64_t)len, leaf, d_temp, temp_bytes, s);
}

}  // namespace nsb

using namespace nsb;

extern "C" {

size_t ns_quick_sort_temp_bytes(size_t n) { return quick_sort_temp(n); }

int ns_quick_sort_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream) {
  if (n > 0 && d_keys == nullptr) return NS_ERR_INVALID;
  if (n > (size_t)INT64_MAX / 8) return NS_ERR_INVALID;
  if (n <= 1) return NS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int leaf = leaf_of(width_mask, varsort_max);
  // the base case: the merge layer (one CTA, or tiles and a few passes)
  if (n <= qs_base_max()) return merge_sort_device(d_keys, n, leaf, d_temp, temp_bytes, s);
  return quick_sort_segments(d_keys, 1, (int64_t)n, leaf, d_temp, temp_bytes, s);
}

size_t ns_quick_sort_temp_bytes_i64(size_t n) { return quick_sort_temp_i64(n); }

int ns_quick_sort_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream) {
  if (n > 0 && d_keys == nullptr) return NS_ERR_INVALID;
  if (n > (size_t)INT64_MAX / 16) return NS_ERR_INVALID;
  if (n <= 1) return NS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int leaf = leaf_of(width_mask, varsort_max);
  if (n <= qs_base_max()) return merge_sort_device(d_keys, n, leaf, d_temp, temp_bytes, s);
  return quick_sort_segments(d_keys, 1, (int64_t)n, leaf, d_temp, temp_bytes, s);
}

}  // extern "C"
