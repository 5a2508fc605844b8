// kway.cuh — k-way merge pass (k = 4 or 8): one HBM pass merges k sorted runs
// into one, instead of log2(k) pairwise passes.
//
// Reference counterpart: merge_runs (hybrid.hpp:61-79) applied log2(k) times.
// The exact k-way split of an output tile cannot be found by one merge-path
// binary search, so tiles are cut at SAMPLES instead:
//   1. kway_sample_kernel   : every s-th key of every run becomes a 64-bit
//      composite sample (value, run-in-group, index) — a strict total order
//      that also breaks ties between equal keys (this is what makes the cuts
//      exact and consistent);
//   2. the samples of each group (k sorted sub-runs) are merged with log2(k)
//      small pairwise passes over 64-bit keys (simple_merge_pass_kernel);
//   3. kway_boundary_kernel : every m-th merged sample of a group is a tile
//      boundary; its cut in run i is the number of run-i keys that precede it
//      in the composite order (upper_bound for runs before the sample's run,
//      its own index for its run, lower_bound for runs after) — found by a
//      binary search over run i's samples, then over the <= s keys between two
//      samples;
//   4. kway_merge_kernel    : one CTA per tile stages the k slices with TMA
//      bulk copies as +inf-terminated runs and merges them in log2(k) shared-
//      memory levels (smem_merge.cuh); the output goes back with a bulk store.
// Tile size bound: between two boundaries m samples apart, run i contributes
// at most (c_i + 1)*s keys where sum c_i = m, so a tile holds <= (m + k)*s
// keys; m is chosen so that this fits the CTA's shared memory.
#pragma once
#include <climits>
#include <cstdint>

#include "mergesort.cuh"
#include "smem_merge.cuh"
#include "tma.cuh"

namespace nsb {

constexpr int kKwS = 128;          // sample spacing (keys)
constexpr int kKwCap = 7936;       // max keys per k-way tile
constexpr int kKwNT = 256;         // threads per k-way merge CTA

__host__ __device__ constexpr int kway_m(int k) { return kKwCap / kKwS - k; }

__device__ __forceinline__ uint64_t composite(int32_t v, int run, int j) {
  return ((uint64_t)((uint32_t)v ^ 0x80000000u) << 32) | ((uint64_t)run << 27) | (uint32_t)j;
}
__device__ __forceinline__ int32_t comp_value(uint64_t c) {
  return (int32_t)((uint32_t)(c >> 32) ^ 0x80000000u);
}
__device__ __forceinline__ int comp_run(uint64_t c) { return (int)((c >> 27) & 31); }
__device__ __forceinline__ int comp_index(uint64_t c) { return (int)(c & ((1u << 27) - 1)); }

// Geometry of one k-way pass over n keys in runs of R: groups of k runs.
struct KwPlan {
  int64_t n, R;
  int k;
  int64_t Ls;        // samples per full run = R / kKwS
  int64_t S;         // total samples
  int tiles_full;    // tiles of a full group
  int64_t groups;
  int64_t tiles;     // total tiles
};

__device__ __forceinline__ int64_t run_len(const KwPlan& P, int64_t r) {
  return max((int64_t)0, min(P.R, P.n - r * P.R));
}

// samples[r*Ls + j] = composite(run_r[j*s], r % k, j)
__global__ void kway_sample_kernel(const int32_t* __restrict__ src, KwPlan P,
                                   uint64_t* __restrict__ samples) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.S) return;
  const int64_t r = i / P.Ls;
  const int64_t j = i - r * P.Ls;
  samples[i] = composite(__ldg(src + r * P.R + j * kKwS), (int)(r % P.k), (int)j);
}

// ---- simple pairwise merge pass over 64-bit keys (for the samples) --------
template <class KT>
__global__ void simple_partition_kernel(const KT* __restrict__ src, int64_t n, int64_t R, int TM,
                                        int64_t tiles, int64_t* __restrict__ mp) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= tiles) return;
  const PassGeom g = pass_geom(c * TM, n, R);
  const KT* A = src + g.pair_base;
  mp[c] = merge_path<int64_t>(A, g.a_len, A + g.a_len, g.b_len, g.diag0);
}

// One CTA per output tile of `tm` keys (tm <= NT*K, tm a power of two that
// divides 2R, so a tile never straddles two run pairs).
template <class KT, int NT, int K>
__global__ void __launch_bounds__(NT)
    simple_merge_pass_kernel(const KT* __restrict__ src, KT* __restrict__ dst, int64_t n,
                             int64_t R, int tm, const int64_t* __restrict__ mp) {
  __shared__ KT sm[NT * K + 2];
  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  const PassGeom g = pass_geom(c * tm, n, R);
  const int64_t pair_len = g.a_len + g.b_len;
  const int64_t diag1 = min(g.diag0 + tm, pair_len);
  const int64_t a0 = mp[c];
  const int64_t a1 = (diag1 == pair_len) ? g.a_len : mp[c + 1];
  const int la = (int)(a1 - a0);
  const int lb = (int)((diag1 - a1) - (g.diag0 - a0));
  const KT* A = src + g.pair_base + a0;
  const KT* B = src + g.pair_base + g.a_len + (g.diag0 - a0);
  const int total = la + lb;
  for (int i = tid; i < total; i += NT) sm[i] = i < la ? A[i] : B[i - la];
  __syncthreads();
  const int per = (tm + NT - 1) / NT;
  const int diag = min(tid * per, total);
  const KT* SA = sm;
  const KT* SB = sm + la;
  int a = merge_path<int>(SA, la, SB, lb, diag);
  int b = diag - a;
  KT* out = dst + c * tm + diag;
  const int cnt = min(per, total - diag);
  for (int k = 0; k < cnt; ++k) {
    const bool take_a = b >= lb || (a < la && SA[a] <= SB[b]);
    out[k] = take_a ? SA[a] : SB[b];
    a += take_a;
    b += !take_a;
  }
}

// ---- tile boundaries -----------------------------------------------------
// cuts[(tile * k) + i] = keys of run i (of the tile's group) before the tile.
// One thread per (tile, run).  Tile 0 of a group starts at 0.
__global__ void kway_boundary_kernel(const int32_t* __restrict__ src,
                                     const uint64_t* __restrict__ raw,     // unmerged samples
                                     const uint64_t* __restrict__ merged,  // per-group sorted
                                     KwPlan P, int m, int32_t* __restrict__ cuts) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= P.tiles * P.k) return;
  const int64_t tile = gid / P.k;
  const int i = (int)(gid - tile * P.k);
  const int64_t g = tile / P.tiles_full;
  const int64_t t = tile - g * P.tiles_full;
  const int64_t r = g * P.k + i;           // global run index
  const int64_t len = run_len(P, r);
  if (t == 0) {
    cuts[gid] = 0;
    return;
  }
  const int64_t gs0 = g * P.k * P.Ls;      // first sample of the group
  const int64_t gs1 = min(P.S, gs0 + P.k * P.Ls);
  const int64_t bpos = gs0 + t * m;
  if (bpos >= gs1 || len == 0) {           // past the group's samples: whole run
    cuts[gid] = (int32_t)len;
    return;
  }
  const uint64_t bnd = merged[bpos];
  const int q = comp_run(bnd);
  if (q == i) {
    cuts[gid] = comp_index(bnd) * kKwS;
    return;
  }
  const int32_t v = comp_value(bnd);
  // run i's samples: number p of them that precede the boundary
  const uint64_t* rs = raw + r * P.Ls;
  const int64_t ns = (len + kKwS - 1) / kKwS;
  int64_t lo = 0, hi = ns;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rs[mid] < bnd) lo = mid + 1;
    else hi = mid;
  }
  // keys of run i before the boundary lie in ((lo-1)*s, lo*s]: search there
  const int32_t* run = src + r * P.R;
  int64_t a = lo == 0 ? 0 : (lo - 1) * kKwS + 1;
  int64_t b = min(len, lo * kKwS);
  // i < q: count keys <= v ; i > q: count keys < v
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    const int32_t x = run[mid];
    const bool before = i < q ? (x <= v) : (x < v);
    if (before) a = mid + 1;
    else b = mid;
  }
  cuts[gid] = (int32_t)a;
}

// Shared memory of one k-way tile: two ping-pong buffers with room for k
// sentinel slots and 16-byte alignment slack per run.
__host__ __device__ constexpr int kway_buf_words(int k) { return kKwCap + 8 * k + 16; }

__device__ __forceinline__ bool tma_ok(const int32_t* cov, int words, const int32_t* lo,
                                       const int32_t* hi) {
#ifdef NSB_KW_NO_TMA
  return false;
#else
  return cov >= lo && cov + words <= hi;
#endif
}

template <int K>
__global__ void __launch_bounds__(kKwNT)
    kway_merge_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst, KwPlan P,
                      const int32_t* __restrict__ cuts) {
  extern __shared__ __align__(128) int32_t kw_sm[];
  __shared__ RunSet rs[2];
  __shared__ __align__(8) uint64_t bar;
  int32_t* X = kw_sm;
  int32_t* Y = kw_sm + kway_buf_words(K);
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t g = tile / P.tiles_full;
  const int64_t t = tile - g * P.tiles_full;
  const int64_t gs0 = g * K * P.Ls;
  const int64_t gs1 = min(P.S, gs0 + K * P.Ls);
  const int64_t ntg = (gs1 - gs0 + kway_m(K) - 1) / kway_m(K);  // tiles of this group
  if (t >= ntg) return;
  const bool last_tile = t + 1 == ntg;

  // slice of run i: [c0_i, c1_i)
  __shared__ int c0s[K], c1s[K];
  __shared__ int64_t out_off_s;
  if (tid < K) {
    const int64_t r = g * K + tid;
    const int64_t len = run_len(P, r);
    c0s[tid] = cuts[tile * K + tid];
    c1s[tid] = last_tile ? (int)len : cuts[(tile + 1) * K + tid];
  }
  __syncthreads();
  if (tid == 0) {
    int64_t before = 0;
    int off = 0;
    rs[0].n = K;
    for (int i = 0; i < K; ++i) {
      before += c0s[i];
      const int64_t r = g * K + i;
      const int32_t* p = src + r * P.R + c0s[i];
      const int shift = (int)((reinterpret_cast<uintptr_t>(p) & 15) >> 2);
      off = ((off + 3) & ~3) + shift;  // mirror global 16-byte alignment
      rs[0].off[i] = off;
      rs[0].len[i] = c1s[i] - c0s[i];
      off += rs[0].len[i] + 1;         // + sentinel slot
    }
    out_off_s = g * K * P.R + before;
#ifdef NSB_DEBUG_KWAY
    int tot = 0;
    for (int i = 0; i < K; ++i) tot += rs[0].len[i];
    if (tot > kKwCap || off > kway_buf_words(K))
      printf("kway tile %lld g %lld t %lld: total %d off_end %d\n", (long long)tile, (long long)g,
             (long long)t, tot, off);
    for (int i = 0; i < K; ++i)
      if (rs[0].len[i] < 0)
        printf("kway tile %lld run %d: c0 %d c1 %d\n", (long long)tile, i, c0s[i], c1s[i]);
#endif
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // stage: one bulk copy per slice (16-byte-aligned cover), else plain loads
  const int32_t* lo = src;
  const int32_t* hi = src + P.n;
  uint32_t bytes = 0;
  if (tid == 0) {
    for (int i = 0; i < K; ++i) {
      const int len = rs[0].len[i];
      if (len == 0) continue;
      const int32_t* p = src + (g * K + i) * P.R + c0s[i];
      const int shift = (int)((reinterpret_cast<uintptr_t>(p) & 15) >> 2);
      const int words = (shift + len + 3) & ~3;
      const int32_t* cov = p - shift;
      if (tma_ok(cov, words, lo, hi)) bytes += words * 4u;
    }
    mbar_arrive_expect_tx(&bar, bytes);
    for (int i = 0; i < K; ++i) {
      const int len = rs[0].len[i];
      if (len == 0) continue;
      const int32_t* p = src + (g * K + i) * P.R + c0s[i];
      const int shift = (int)((reinterpret_cast<uintptr_t>(p) & 15) >> 2);
      const int words = (shift + len + 3) & ~3;
      const int32_t* cov = p - shift;
      if (tma_ok(cov, words, lo, hi)) tma_load_1d(X + rs[0].off[i] - shift, cov, words * 4u, &bar);
    }
  }
  // fallback plain loads for slices whose cover leaves the array
  for (int i = 0; i < K; ++i) {
    const int len = rs[0].len[i];
    if (len == 0) continue;
    const int32_t* p = src + (g * K + i) * P.R + c0s[i];
    const int shift = (int)((reinterpret_cast<uintptr_t>(p) & 15) >> 2);
    const int words = (shift + len + 3) & ~3;
    const int32_t* cov = p - shift;
    if (!tma_ok(cov, words, lo, hi))
      for (int j = tid; j < len; j += kKwNT) X[rs[0].off[i] + j] = p[j];
  }
  mbar_wait(&bar, 0);
  __syncthreads();
#ifdef NSB_DEBUG_KWAY
  if (tid < K && (rs[0].off[tid] + rs[0].len[tid] >= kway_buf_words(K) || rs[0].len[tid] < 0)) {
    dbg_record(4, tid, rs[0].off[tid], rs[0].len[tid]);
    return;
  }
#endif
  if (tid < K) X[rs[0].off[tid] + rs[0].len[tid]] = INT_MAX;  // sentinels
  int total = 0;
  for (int i = 0; i < K; ++i) total += rs[0].len[i];
  const int64_t out_off = out_off_s;
  const int out_shift = (int)(((reinterpret_cast<uintptr_t>(dst + out_off)) & 15) >> 2);

  // log2(K) pairwise levels; the last one writes contiguously at out_shift
  int cur = 0;
  int32_t* in_buf = X;
  int32_t* out_buf = Y;
#pragma unroll 1
  for (int nr = K; nr > 1; nr >>= 1) {
    const bool last = nr == 2;
    if (tid == 0) {
      RunSet& o = rs[cur ^ 1];
      o.n = nr / 2;
      int off = last ? out_shift : 0;
      for (int q = 0; q < o.n; ++q) {
        o.off[q] = off;
        o.len[q] = rs[cur].len[2 * q] + rs[cur].len[2 * q + 1];
        off += o.len[q] + (last ? 0 : 1);
      }
    }
    __syncthreads();
    merge_level<kKwNT>(in_buf, rs[cur], out_buf, rs[cur ^ 1], total, !last);
    __syncthreads();
    cur ^= 1;
    int32_t* tmp = in_buf;
    in_buf = out_buf;
    out_buf = tmp;
  }
  // in_buf holds the merged tile at [out_shift, out_shift + total)
  int32_t* out = dst + out_off;
  const int head = min(total, (4 - out_shift) & 3);
#ifdef NSB_KW_NO_TMA
  const int body = 0;
#else
  const int body = ((total - head) >> 2) << 2;
#endif
  if (body > 0) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tma_store_1d(out + head, in_buf + out_shift + head, (uint32_t)body * 4u);
      bulk_commit();
    }
  }
#ifdef NSB_DEBUG_KWAY
  if (out_off < 0 || out_off + total > P.n) {
    dbg_record(3, (int)tile, (int)out_off, total);
    return;
  }
#endif
  for (int j = tid; j < head; j += kKwNT) out[j] = in_buf[out_shift + j];
  for (int j = head + body + tid; j < total; j += kKwNT) out[j] = in_buf[out_shift + j];
  if (body > 0 && tid == 0) bulk_wait_read_all();
}

}  // namespace nsb
