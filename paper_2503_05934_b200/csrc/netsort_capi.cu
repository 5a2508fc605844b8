// netsort_capi.cu — C-ABI entry points of the merge layer, the base-case
// batch, the segmented sort and the checking helpers (include/netsort_b200.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "mergesort.cuh"
#include "networks.cuh"

namespace nsb {

// ---- tuning (sm_100a) -----------------------------------------------------
// Tile sort: 512 threads x 16 keys = 8192 keys (32 KiB smem), 2+ CTAs/SM.
constexpr int kBsNT = 512, kBsK = 16, kBsT = kBsNT * kBsK;
// Single-CTA sort for n <= 16384: 1024 threads x 16 keys (64 KiB smem).
constexpr int kSmNT = 1024, kSmK = 16, kSmT = kSmNT * kSmK;
static_assert(kSmT == kSmallTile, "small-tile size mismatch");


template <int NT, int K, int LEAF, class Key>
static int launch_blocksort(const Key* src, Key* dst, int64_t n, int stride, int64_t ctas,
                            cudaStream_t s, int64_t seg_len = 0, int tiles_per_seg = 1) {
  constexpr int smem = tile_smem_bytes<NT, K, Key>();
  auto* kern = blocksort_kernel<NT, K, LEAF, Key>;
  NSB_TRY(ensure_smem_attr(reinterpret_cast<const void*>(kern), smem,
                           "cudaFuncSetAttribute(blocksort)"));
  {
    Prof prof(PK_TILE_SORT, s);
    const cudaError_t e = launch_pdl(n, kern, (unsigned)ctas, NT, smem, s, src, dst, n, stride,
                                     seg_len, tiles_per_seg);
    if (e != cudaSuccess) return check_cuda(e, "blocksort_kernel");
  }
  return check_launch("blocksort_kernel");
}

// int32 sorts of at least 2^NSB_TILE16K_MIN_LOG2 keys use 16384-key tiles
#ifndef NSB_TILE16K_MIN_LOG2
#define NSB_TILE16K_MIN_LOG2 21
#endif
// Merge-pass tile shape: <256,29> = 7424 keys per tile (measured 0.5-4 %
// faster than <256,31> from 2^24 to 2^30, profiles/r01_tile_sort_v6_ab.txt);
// int64 keys take odd K as well (half-warp 64-bit cursors on distinct banks).
constexpr int kV2NT = 256, kV2K = 29, kV2T = kV2NT * kV2K;
// Run-time knobs (read once).  Only knobs that select between code paths
// every build carries anyway; the measured-dead tile shapes of round 1 are
// gone (DESIGN.md §4 lists what was measured).
//   NSB_FUSED_MAX     : passes with at most this many tiles search their
//                       merge-path splits in-kernel (no partition launch)
//   NSB_PART_WARP_MAX : passes of at most this many tiles find their splits
//                       with one warp per tile (merge_partition_v4_kernel),
//                       larger ones with one thread per tile (v3 / v2)
//   NSB_SAMPLES=0     : partition without the block samples (plain search)
//   NSB_SINGLE_MAX    : largest n sorted by one CTA (<= 16384; measured
//                       10,000 keys 22.9 us in one 1024-thread CTA, 15.9 us
//                       as two 8192-key tiles and one merge pass)
// The sanitizer-style tests use them to force every partition path at small
// sizes.
struct MergeTuning {
  int64_t fused_max_tiles = 4096;
  int samples = 1;
  int64_t single_max = kBsT;
  int64_t part_warp_max = 16384;
  MergeTuning() {
    if (const char* e = getenv("NSB_PART_WARP_MAX")) part_warp_max = atoll(e);
    if (const char* e = getenv("NSB_SINGLE_MAX")) single_max = std::min<int64_t>(atoll(e), kSmT);
    if (const char* e = getenv("NSB_SAMPLES")) samples = atoi(e);
    if (const char* e = getenv("NSB_FUSED_MAX")) fused_max_tiles = atoll(e);
  }
};
static const MergeTuning& tuning() {
  static const MergeTuning t;
  return t;
}

// Upper bound on merge-path splits of any pass (v2 tiles >= 3968 keys).
static size_t max_merge_tiles(size_t n) { return n / 1024 + 64; }

// block samples (first/last key of every 256-key block) for the partition
static size_t samples_bytes(size_t n, size_t kb) {
  return 2 * align_up(((n >> kSmpShiftMin) + 2) * kb, 256);
}

size_t merge_sort_temp(size_t n) {
  if (n <= (size_t)tuning().single_max) return 0;
  return align_up(n * sizeof(int32_t), 256) + align_up((max_merge_tiles(n) + 1) * 8, 256) +
         samples_bytes(n, 4);
}

// int64: ping-pong buffer + merge-path splits + block samples (no k-way scratch)
size_t merge_sort_temp_i64(size_t n) {
  if (n <= (size_t)tuning().single_max) return 0;
  return align_up(n * sizeof(int64_t), 256) + align_up((max_merge_tiles(n) + 1) * 8, 256) +
         samples_bytes(n, 8);
}

// Block samples of the pass outputs of one sort: recorded by every merge
// pass, used by the next pass's partition when `have` (the array's previous
// pass recorded them for the same n).
struct SmpCtx {
  void* base = nullptr;  // first[] then last[]
  int64_t n = 0;
  bool have = false;
  int shift = kSmpShift;  // block size the last recording pass used
  template <class Key>
  BlockSamples<Key> get(int sh) const {
    if (!base) return BlockSamples<Key>{nullptr, nullptr, 0, sh};
    Key* f = static_cast<Key*>(base);
    Key* l = reinterpret_cast<Key*>(static_cast<char*>(base) +
                                    align_up((((size_t)n >> kSmpShiftMin) + 2) * sizeof(Key), 256));
    return BlockSamples<Key>{f, l, n, sh};
  }
};

// Tiles of exactly NT*K outputs (a multiple of 4 keys, so every tile starts
// 16-byte aligned); only the last tile of a run pair is partial.  A full tile
// gives every thread exactly K outputs, which the merge loop exploits.
static PassPlan plan_pass(int64_t n, int64_t R, int nt = kV2NT, int k = kV2K, int64_t seg_len = 0) {
  PassPlan P;
  P.R = R;
  P.n = n;
  const int64_t two_r = 2 * R;
  P.tmp = nt * k;
  P.tpp = (int)((two_r + P.tmp - 1) / P.tmp);
  P.kp = k;
  P.seg_len = seg_len;
  P.pps = seg_len > 0 ? (seg_len + two_r - 1) / two_r : 0;
  return P;
}

// One pairwise merge pass (v2): runs of R in src -> runs of 2R in dst.
template <int NT, int K, class Key>
static int v2_pass_t(const Key* src, Key* dst, int64_t n, int64_t R, int64_t* mp,
                     cudaStream_t s, SmpCtx* sc = nullptr, int64_t seg_len = 0) {
  const MergeTuning& tu = tuning();
  const PassPlan P = plan_pass(n, R, NT, K, seg_len);
  // segmented passes (seg_len > 0): every segment's runs pair up on their own;
  // they neither read nor record block samples (sc == nullptr)
  const int64_t pairs = seg_len > 0 ? (n / seg_len) * P.pps : (n + 2 * R - 1) / (2 * R);
  const int64_t mt = pairs * P.tpp;
  // samples: only for the whole array of a sort (sc->n == n); tiles must be
  // whole 256-key blocks (NT*K a multiple of 256)
  // block = 256 keys when the tile is a multiple of it, else 128 (every
  // shape's NT is a multiple of 128)
  constexpr int kShift = ((NT * K) % 256 == 0) ? kSmpShift : kSmpShiftMin;
  const bool rec = sc && sc->base && sc->n == n && ((NT * K) % (1 << kShift)) == 0;
  const BlockSamples<Key> bs =
      rec ? sc->get<Key>(kShift) : BlockSamples<Key>{nullptr, nullptr, 0, kShift};
  // in-kernel search up to 4096 tiles of <= 4096 keys, 2048 larger tiles
  // (tools/fused_ab.sh: 2^24 keys in 2114 <256,31> tiles 480 -> 473 us with
  // the partition kernel; 2^23 in 2850 <128,23> tiles 235 vs 261 us fused)
  // int64 keys: 1024 (measured: 2^23 keys in 2850 <128,23> tiles 540 us fused
  // vs 419 us with the partition kernel, 2^22 261 vs 242 us; equal below)
  const int64_t fused_max = sizeof(Key) == 8 ? tu.fused_max_tiles / 4
                            : NT * K > 4096  ? tu.fused_max_tiles / 2
                                             : tu.fused_max_tiles;
  if (mt <= fused_max) {
    // few tiles: every CTA finds its own split (no partition launch)
    {
      Prof prof(PK_MERGE_PASS, s);
      const cudaError_t e = launch_pdl(n, merge_pass_v2_kernel<NT, K, true, Key>, (unsigned)mt, NT,
                                       0, s, src, dst, P, (const int64_t*)nullptr, bs);
      if (e != cudaSuccess) return check_cuda(e, "merge_pass_v2_kernel<fused>");
    }
    if (sc) {
      sc->have = rec;
      sc->shift = kShift;
    }
    return check_launch("merge_pass_v2_kernel<fused>");
  }
  {
    Prof prof(PK_PARTITION, s);
    cudaError_t e;
    const bool smp = sc && sc->have && rec && tu.samples;
    if (mt <= tu.part_warp_max)  // few tiles: latency-bound, one warp per search
      e = launch_pdl(n, merge_partition_v4_kernel<Key>, (unsigned)((mt + 7) / 8), 256, 0, s,
                     src, P, mt, mp,
                     smp ? sc->get<Key>(sc->shift) : BlockSamples<Key>{nullptr, nullptr, 0, kShift});
    else if (smp)
      e = launch_pdl(n, merge_partition_v3_kernel<Key>, (unsigned)((mt + 255) / 256), 256, 0, s,
                     src, P, mt, mp, sc->get<Key>(sc->shift));
    else
      e = launch_pdl(n, merge_partition_v2_kernel<Key>, (unsigned)((mt + 255) / 256), 256, 0, s,
                     src, P, mt, mp);
    if (e != cudaSuccess) return check_cuda(e, "merge_partition_kernel");
  }
  NSB_TRY(check_launch("merge_partition_kernel"));
  {
    Prof prof(PK_MERGE_PASS, s);
    const cudaError_t e = launch_pdl(n, merge_pass_v2_kernel<NT, K, false, Key>, (unsigned)mt, NT, 0,
                                     s, src, dst, P, (const int64_t*)mp, bs);
    if (e != cudaSuccess) return check_cuda(e, "merge_pass_v2_kernel");
  }
  if (sc) {
    sc->have = rec;
    sc->shift = kShift;
  }
  return check_launch("merge_pass_v2_kernel");
}

// One pairwise merge pass (v2): runs of R in src -> runs of 2R in dst.
// Tile shape by array size (tools/mid_sweep.sh on B200): up to 2^23 keys a
// pass is latency bound and smaller tiles (<128,23>, 2944 keys, 12 CTAs/SM)
// win by 5-10 %; above, <256,29>.  int64 (tools/i64_sweep.sh): <128,15> up
// to 2^20 keys, <128,23> up to 2^25, <128,31> above.
static int v2_pass(const int32_t* src, int32_t* dst, int64_t n, int64_t R, int64_t* mp,
                   cudaStream_t s, SmpCtx* sc = nullptr, int64_t seg_len = 0) {
  return n <= (int64_t(1) << 23) ? v2_pass_t<128, 23>(src, dst, n, R, mp, s, sc, seg_len)
                                 : v2_pass_t<kV2NT, kV2K>(src, dst, n, R, mp, s, sc, seg_len);
}
static int v2_pass(const int64_t* src, int64_t* dst, int64_t n, int64_t R, int64_t* mp,
                   cudaStream_t s, SmpCtx* sc = nullptr, int64_t seg_len = 0) {
  if (n <= (int64_t(1) << 20)) return v2_pass_t<128, 15>(src, dst, n, R, mp, s, sc, seg_len);
  if (n <= (int64_t(1) << 25)) return v2_pass_t<128, 23>(src, dst, n, R, mp, s, sc, seg_len);
  return v2_pass_t<128, 31>(src, dst, n, R, mp, s, sc, seg_len);
}

// Pairwise passes over existing sorted runs of length R0 (the last may be
// shorter) until one run remains; *result = the buffer holding it (keys or tmp).
template <class Key>
static int merge_existing_runs_t(Key* keys, Key* tmp, size_t n, int64_t R0, void* d_temp,
                                 cudaStream_t s, Key** result) {
  int64_t* mp = reinterpret_cast<int64_t*>(static_cast<char*>(d_temp) +
                                           align_up(n * sizeof(Key), 256));
  Key* cur = keys;
  Key* other = tmp;
  for (int64_t R = R0; R < (int64_t)n; R *= 2) {
    NSB_TRY(v2_pass(cur, other, (int64_t)n, R, mp, s));
    std::swap(cur, other);
  }
  *result = cur;
  return NS_OK;
}
int merge_existing_runs(int32_t* keys, int32_t* tmp, size_t n, int64_t R0, void* d_temp,
                        cudaStream_t s, int32_t** result) {
  return merge_existing_runs_t(keys, tmp, n, R0, d_temp, s, result);
}
int merge_existing_runs(int64_t* keys, int64_t* tmp, size_t n, int64_t R0, void* d_temp,
                        cudaStream_t s, int64_t** result) {
  return merge_existing_runs_t(keys, tmp, n, R0, d_temp, s, result);
}

template <class Key>
static int merge_sort_device_t(Key* d_keys, size_t n, int leaf, void* d_temp, size_t temp_bytes,
                               cudaStream_t s) {
  constexpr bool k32 = std::is_same_v<Key, int32_t>;
  if (n <= 1) return NS_OK;
  if (n <= (size_t)kSmT && (n <= (size_t)tuning().single_max || d_temp == nullptr)) {
    // one CTA sized to the array: fewer threads and merge levels for small n
    // (also up to 16384 keys when the caller passes no scratch)
    return with_leaf(leaf, [&](auto L) {
      constexpr int LF = decltype(L)::value;
      if (n <= 512) return launch_blocksort<32, 16, LF>(d_keys, d_keys, (int64_t)n, 512, 1, s);
      if (n <= 2048) return launch_blocksort<128, 16, LF>(d_keys, d_keys, (int64_t)n, 2048, 1, s);
      if (n <= 4096) return launch_blocksort<256, 16, LF>(d_keys, d_keys, (int64_t)n, 4096, 1, s);
      if (n <= 8192) return launch_blocksort<512, 16, LF>(d_keys, d_keys, (int64_t)n, 8192, 1, s);
      return launch_blocksort<kSmNT, kSmK, LF>(d_keys, d_keys, (int64_t)n, kSmT, 1, s);
    });
  }
  const size_t need = k32 ? merge_sort_temp(n) : merge_sort_temp_i64(n);
  if (temp_bytes < need || d_temp == nullptr) return NS_ERR_TEMP;
  Key* tmp = static_cast<Key*>(d_temp);
  int64_t* mp = reinterpret_cast<int64_t*>(static_cast<char*>(d_temp) +
                                           align_up(n * sizeof(Key), 256));
  // int32 tile: 16384 keys (<512,32>) from 2^21 keys up (one merge pass
  // fewer; with 32 keys per thread it has the 8192-key tile's four
  // shared-memory levels), 8192 (<256,32>) below; int64: 8192 (<512,16>)
  const int T = (k32 && n >= (size_t(1) << NSB_TILE16K_MIN_LOG2)) ? kSmT : kBsT;
  const int64_t tiles = (int64_t)((n + T - 1) / T);
  // pairwise passes until one run remains
  int passes = 0;
  for (int64_t runs = tiles; runs > 1; runs = (runs + 1) / 2) ++passes;
  // Pick the tile-sort destination so the last pass lands in d_keys.
  Key* cur = (passes & 1) ? tmp : d_keys;
  Key* other = (cur == d_keys) ? tmp : d_keys;
  NSB_TRY(with_leaf(leaf, [&](auto L) {
    constexpr int LF = decltype(L)::value;
    if constexpr (!k32) {
      return launch_blocksort<512, 16, LF>(d_keys, cur, (int64_t)n, T, tiles, s);
    } else {
      if (T == kBsT) return launch_blocksort<256, 32, LF>(d_keys, cur, (int64_t)n, T, tiles, s);
      return launch_blocksort<512, 32, LF>(d_keys, cur, (int64_t)n, T, tiles, s);
    }
  }));
  SmpCtx sc;
  {
    const size_t off =
        align_up(n * sizeof(Key), 256) + align_up((max_merge_tiles(n) + 1) * 8, 256);
    sc.base = static_cast<char*>(d_temp) + off;
    sc.n = (int64_t)n;
  }
  int64_t R = T;
  for (int pi = 0; pi < passes; ++pi) {
    NSB_TRY(v2_pass(cur, other, (int64_t)n, R, mp, s, &sc));
    std::swap(cur, other);
    R *= 2;
  }
  return NS_OK;
}

int merge_sort_device(int32_t* d_keys, size_t n, int leaf, void* d_temp, size_t temp_bytes,
                      cudaStream_t s) {
  return merge_sort_device_t(d_keys, n, leaf, d_temp, temp_bytes, s);
}
int merge_sort_device(int64_t* d_keys, size_t n, int leaf, void* d_temp, size_t temp_bytes,
                      cudaStream_t s) {
  return merge_sort_device_t(d_keys, n, leaf, d_temp, temp_bytes, s);
}

// Segments of up to 512 keys: 2^LV lanes of a warp per segment (16 keys per
// lane, missing keys padded with the key maximum), so a warp sorts 32 >> LV
// segments at once and a CTA of 8 warps 256 >> LV of them — a batch of tiny
// segments is not one 32-thread CTA per segment (2^23 segments of 8 keys:
// 14.8 ms that way).  Each lane sorts its 16 keys with the config's base case
// and in-register merges, LV warp-bitonic levels join the lanes of a segment;
// no shared memory.
template <int LV, int LEAF, class Key>
__global__ void __launch_bounds__(256) small_segments_kernel(Key* __restrict__ keys, int64_t nseg,
                                                             int seg_len) {
  constexpr int G = 1 << LV;     // lanes per segment
  constexpr int SPW = 32 >> LV;  // segments per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t seg = ((int64_t)blockIdx.x * 8 + warp) * SPW + (lane >> LV);
  const int j = lane & (G - 1);
  pdl_wait();
  pdl_trigger();
  const int cnt = seg < nseg ? max(0, min(16, seg_len - 16 * j)) : 0;
  Key* p = keys + (seg < nseg ? seg * seg_len + 16 * j : 0);
  // a lane's keys lie inside its own segment
  NSB_DCHECK(cnt == 0 || (16 * j + cnt <= seg_len && seg * seg_len + 16 * j + cnt <= nseg * seg_len));
  // (16-byte vector loads / stores of a lane's 16 keys measured slower: 0.55
  // vs 0.32 ms for 2^20 segments of 64 keys)
  Key v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = k < cnt ? p[k] : KeyT<Key>::kMax;
  thread_sort<LEAF>(v);  // the network base case (try_base_case, hybrid.hpp:48-56)
  if constexpr (LV > 0) warp_bitonic<LV>(v, lane);
  // the segment's lanes hold its sorted keys blocked, the pads at the end
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (k < cnt) p[k] = v[k];
}

template <int LV, int LEAF, class Key>
static int launch_small_segments(Key* d_keys, int64_t nseg, int seg_len, cudaStream_t s) {
  const int64_t per_cta = 8 * (32 >> LV);
  const int64_t ctas = (nseg + per_cta - 1) / per_cta;
  if (ctas > INT_MAX) return NS_ERR_INVALID;
  {
    Prof prof(PK_TILE_SORT, s);
    const cudaError_t e = launch_pdl(nseg * seg_len, small_segments_kernel<LV, LEAF, Key>,
                                     (unsigned)ctas, 256, 0, s, d_keys, nseg, seg_len);
    if (e != cudaSuccess) return check_cuda(e, "small_segments_kernel");
  }
  return check_launch("small_segments_kernel");
}

// One CTA per segment, the tile sized to the segment (a 100-key segment does
// not pay for an 8192-key tile); segments of up to 512 keys share warps.
template <class Key>
static int tile_sort_segments_t(Key* d_keys, size_t num_segments, size_t seg_len, int leaf,
                                cudaStream_t s) {
  if (seg_len > (size_t)kSmT) return NS_ERR_INVALID;
  const int64_t n = (int64_t)(num_segments * seg_len);
  const int st = (int)seg_len;
  const int64_t g = (int64_t)num_segments;
  return with_leaf(leaf, [&](auto L) {
    constexpr int LF = decltype(L)::value;
    if (seg_len <= 16) return launch_small_segments<0, LF>(d_keys, g, st, s);
    if (seg_len <= 32) return launch_small_segments<1, LF>(d_keys, g, st, s);
    if (seg_len <= 64) return launch_small_segments<2, LF>(d_keys, g, st, s);
    if (seg_len <= 128) return launch_small_segments<3, LF>(d_keys, g, st, s);
    if (seg_len <= 256) return launch_small_segments<4, LF>(d_keys, g, st, s);
    // (a whole warp per segment: the staged one-warp tile is faster, 0.23 vs 0.39 ms per 2^26 keys)
    if (seg_len <= 512) return launch_blocksort<32, 16, LF>(d_keys, d_keys, n, st, g, s);
    if (seg_len <= 2048) return launch_blocksort<128, 16, LF>(d_keys, d_keys, n, st, g, s);
    if constexpr (std::is_same_v<Key, int32_t>) {
      // 32 keys per thread: 1024-key warp runs, one shared-memory merge level
      // fewer than 16 keys per thread
      if (seg_len <= 4096) return launch_blocksort<128, 32, LF>(d_keys, d_keys, n, st, g, s);
      if (seg_len <= (size_t)kBsT) return launch_blocksort<256, 32, LF>(d_keys, d_keys, n, st, g, s);
      return launch_blocksort<512, 32, LF>(d_keys, d_keys, n, st, g, s);
    } else {
      if (seg_len <= 4096) return launch_blocksort<256, 16, LF>(d_keys, d_keys, n, st, g, s);
      if (seg_len <= (size_t)kBsT) return launch_blocksort<kBsNT, kBsK, LF>(d_keys, d_keys, n, st, g, s);
      return launch_blocksort<kSmNT, kSmK, LF>(d_keys, d_keys, n, st, g, s);
    }
  });
}
// Segments longer than one tile, merge-sorted ALL AT ONCE: one tile-sort
// launch over every segment's tiles (each segment starts a tile; its last
// tile is partial), then ceil(log2(tiles per segment)) pairwise passes whose
// run pairs never cross a segment boundary (PassPlan::seg_len) — no
// per-segment host loop.  Scratch: that of a merge sort of all the keys.
template <class Key>
static int merge_sort_segments_t(Key* d_keys, size_t num_segments, size_t seg_len, int leaf,
                                 void* d_temp, size_t temp_bytes, cudaStream_t s) {
  constexpr bool k32 = std::is_same_v<Key, int32_t>;
  const size_t n = num_segments * seg_len;
  const size_t need = k32 ? merge_sort_temp(n) : merge_sort_temp_i64(n);
  if (temp_bytes < need || d_temp == nullptr) return NS_ERR_TEMP;
  Key* tmp = static_cast<Key*>(d_temp);
  int64_t* mp = reinterpret_cast<int64_t*>(static_cast<char*>(d_temp) +
                                           align_up(n * sizeof(Key), 256));
  const int T = k32 ? kSmT : kBsT;
  const int tps = (int)((seg_len + T - 1) / T);
  int passes = 0;
  for (int64_t runs = tps; runs > 1; runs = (runs + 1) / 2) ++passes;
  Key* cur = (passes & 1) ? tmp : d_keys;
  Key* other = (cur == d_keys) ? tmp : d_keys;
  const int64_t ctas = (int64_t)num_segments * tps;
  NSB_TRY(with_leaf(leaf, [&](auto L) {
    constexpr int LF = decltype(L)::value;
    if constexpr (!k32)
      return launch_blocksort<512, 16, LF>(d_keys, cur, (int64_t)n, T, ctas, s, (int64_t)seg_len, tps);
    else
      return launch_blocksort<512, 32, LF>(d_keys, cur, (int64_t)n, T, ctas, s, (int64_t)seg_len, tps);
  }));
  int64_t R = T;
  for (int pi = 0; pi < passes; ++pi) {
    NSB_TRY(v2_pass(cur, other, (int64_t)n, R, mp, s, nullptr, (int64_t)seg_len));
    std::swap(cur, other);
    R *= 2;
  }
  return NS_OK;
}

int tile_sort_segments(int32_t* d_keys, size_t num_segments, size_t seg_len, int leaf,
                       cudaStream_t s) {
  return tile_sort_segments_t(d_keys, num_segments, seg_len, leaf, s);
}

// ---------------------------------------------------------------------------
// Base-case batch: each ragged array (length 0..8) sorted by its own network.
// A CTA owns kBaArr consecutive arrays; their keys (<= 8 per array) are staged
// in shared memory with coalesced loads, each thread sorts its arrays in
// registers with the size-specific network, and the CTA stores them back.
// ---------------------------------------------------------------------------
#ifndef NSB_BATCH_PER
#define NSB_BATCH_PER 4
#endif
#ifndef NSB_BATCH_MINB
#define NSB_BATCH_MINB 1
#endif
constexpr int kBaNT = 256, kBaPer = NSB_BATCH_PER, kBaArr = kBaNT * kBaPer;

// Lanes of a warp that sort arrays of different lengths would serialise the
// seven network paths, so each CTA first splits its arrays by length (a
// 9-way block multisplit with warp ballots: deterministic and stable, so the
// arrays one warp receives are same-length neighbours ~6 arrays apart in
// memory, i.e. on different banks), then thread t sorts the t-th array of
// that order and a warp runs one network width almost always.  Keys are
// staged in shared memory at the same 16-byte phase as in HBM so the
// 128-bit loads and stores of the aligned body are bank-conflict free.
// Lanes of the warp whose len equals this lane's (len in -1..8; -1 = no
// array): one ballot per bit of the 4-bit length.
__device__ __forceinline__ unsigned match_len4(int len) {
  const unsigned u = (unsigned)len & 15u;
  unsigned eq = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const unsigned m = __ballot_sync(0xffffffffu, (u >> b) & 1u);
    eq &= ((u >> b) & 1u) ? m : ~m;
  }
  return eq;
}

// One chunk of kBaArr consecutive arrays (first = its first array), sorted
// by one CTA.  Returns false (keys untouched) if a length is out of range —
// unreachable after the validation phase, kept as a bounds guard.
__device__ __forceinline__ bool batch_chunk(int32_t* __restrict__ keys,
                                            const uint32_t* __restrict__ offsets,
                                            int64_t num_arrays, int64_t first, uint64_t* bar,
                                            uint32_t& tma_uses, const int* status) {
  constexpr int NW = kBaNT / 32;
  __shared__ __align__(16) int32_t sk[kBaArr * 8 + 8];
  // length-grouped order: (shared-memory key offset << 4) | length per slot
  __shared__ uint32_t perm[kBaArr];
  // per (warp, length, round) counts -> bases; warp-major so the scan rows
  // (one per (length, round), across warps) are read conflict-free
  __shared__ int wcnt[NW][9][kBaPer];
  __shared__ int s_bad;
  __shared__ uint32_t s_k0, s_k1, s_kt;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int cnt = (int)min((int64_t)kBaArr, num_arrays - first);
  if (tid == 0) {
    s_bad = 0;
    s_k0 = __ldg(offsets + first);
    s_k1 = __ldg(offsets + first + cnt);
    s_kt = __ldg(offsets + num_arrays);  // end of the key array
    if (s_k1 < s_k0 || s_k1 - s_k0 > 8u * (uint32_t)cnt) s_bad = 1;
  }
  __syncthreads();
  const uint32_t k0 = s_k0;
  const int nk = s_bad ? 0 : (int)(s_k1 - k0);
  // The keys are staged by one bulk copy (TMA) of their 16-byte-aligned
  // cover, placed in shared memory at the same 16-byte phase as in HBM; the
  // neighbours' keys it drags in are never written back.  A cover that would
  // leave the key array falls back to per-thread loads.
  const int32_t* kp = keys + k0;
  const int phase = (int)((reinterpret_cast<uintptr_t>(kp) & 15) >> 2);  // key i -> sk[i + phase]
  const int head = min(nk, (4 - phase) & 3);
  const int body = (nk - head) >> 2;
  const int tail = nk - head - 4 * body;
  const int32_t* cov = kp - phase;
  const int cov_words = (phase + nk + 3) & ~3;
  const bool use_tma = nk > 0 && cov >= keys && cov + cov_words <= keys + s_kt;
  if (use_tma) {
    if (tid == 0) {
      mbar_arrive_expect_tx(bar, (uint32_t)cov_words * 4u);
      tma_load_1d(sk, cov, (uint32_t)cov_words * 4u, bar);
    }
  } else {
    for (int i = tid; i < nk; i += kBaNT) sk[phase + i] = __ldcs(kp + i);
  }
  // this thread's array starts (coalesced; each array's end is the next
  // lane's start, lane 31 loads its own)
  uint32_t ofa[kBaPer], ofb[kBaPer];
#pragma unroll
  for (int r = 0; r < kBaPer; ++r) {
    const int j = r * kBaNT + tid;
    ofa[r] = j <= cnt ? __ldg(offsets + first + j) : 0u;
    ofb[r] = (lane == 31 && j + 1 <= cnt) ? __ldg(offsets + first + j + 1) : 0u;
  }
#pragma unroll
  for (int r = 0; r < kBaPer; ++r) {
    const uint32_t nx = __shfl_down_sync(0xffffffffu, ofa[r], 1);
    if (lane != 31) ofb[r] = nx;
  }
  int4* sk4 = reinterpret_cast<int4*>(sk + phase + head);  // 16-byte aligned
  // the barrier (initialised once per CTA) completes one phase per staged chunk
  if (use_tma) mbar_wait(bar, tma_uses++ & 1u);
  __syncthreads();
  // validate (lengths outside [0, 8] -> error, nothing is touched) and count
  // lengths per (round, warp) with ballots
  int mylen[kBaPer];
  uint32_t myoff[kBaPer];
  unsigned myeq[kBaPer];
#pragma unroll
  for (int r = 0; r < kBaPer; ++r) {
    const int j = r * kBaNT + tid;
    int len = -1;
    myoff[r] = 0;
    if (j < cnt) {
      const uint32_t a = ofa[r], b = ofb[r];
      if (b < a || b - a > 8) s_bad = 1;
      else len = (int)(b - a);
      myoff[r] = a - k0 + (uint32_t)phase;  // < 2^14 when the CTA's range is valid
    }
    mylen[r] = len;
    // lanes with this lane's length (4 ballots on the length bits instead of
    // one per length); the group's lowest lane records the group's size
    const unsigned eq = match_len4(len);
    myeq[r] = eq;
    if (lane <= 8) wcnt[warp][lane][r] = 0;
    __syncwarp();
    if (len >= 0 && (eq & ((1u << lane) - 1u)) == 0) wcnt[warp][len][r] = __popc(eq);
  }
  __syncthreads();
  if (s_bad) return false;  // unreachable after the validation phase
  // exclusive scan in (length, round, warp) order (stable): each of the
  // 9*kBaPer rows of NW counts is scanned by one thread, then one warp scans
  // the row totals
  __shared__ int rowtot[9 * kBaPer];
  if (tid < 9 * kBaPer) {  // row tid = (length, round), stride 9*kBaPer across warps
    int* row = &wcnt[0][0][0] + tid;
    int acc = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int c = row[w * 9 * kBaPer];
      row[w * 9 * kBaPer] = acc;
      acc += c;
    }
    rowtot[tid] = acc;
  }
  __syncthreads();
  if (warp == 0) {
    int v0 = lane < 9 * kBaPer ? rowtot[lane] : 0;
    int v1 = lane + 32 < 9 * kBaPer ? rowtot[lane + 32] : 0;
    int x0 = v0, x1 = v1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(0xffffffffu, x0, o), y1 = __shfl_up_sync(0xffffffffu, x1, o);
      if (lane >= o) {
        x0 += y0;
        x1 += y1;
      }
    }
    const int tot0 = __shfl_sync(0xffffffffu, x0, 31);
    if (lane < 9 * kBaPer) rowtot[lane] = x0 - v0;
    if (lane + 32 < 9 * kBaPer) rowtot[lane + 32] = tot0 + x1 - v1;
  }
  __syncthreads();
  if (tid < 9 * kBaPer) {
    int* row = &wcnt[0][0][0] + tid;
    const int base = rowtot[tid];
#pragma unroll
    for (int w = 0; w < NW; ++w) row[w * 9 * kBaPer] += base;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kBaPer; ++r) {
    const int len = mylen[r];
    const int rank = __popc(myeq[r] & ((1u << lane) - 1u));
    if (len >= 0) perm[wcnt[warp][len][r] + rank] = (myoff[r] << 4) | (uint32_t)len;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kBaPer; ++r) {
    const int slot = r * kBaNT + tid;
    if (slot < cnt) {
      const uint32_t pk = perm[slot];  // one load: no second look at the offsets
      const int off = (int)(pk >> 4);
      const int len = (int)(pk & 15u);
      NSB_DCHECK(len <= 8 && off + len <= kBaArr * 8 + 8);
      sort_small_in_place(sk + off, len);  // warp-uniform almost always (grouped by length)
    }
  }
  // Only now wait for the validation kernel (programmatic dependent launch:
  // everything above overlapped it) and write nothing if it flagged the batch.
  pdl_wait();
  __shared__ int s_skip;
  if (tid == 0) s_skip = *reinterpret_cast<const volatile int*>(status);
  __syncthreads();
  if (s_skip) return true;
  int32_t* kw = keys + k0;
  if (body > 0) {  // aligned interior: one bulk store; head/tail keys one by one
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tma_store_1d(kw + head, sk4, (uint32_t)body * 16u);
      bulk_commit();
      bulk_wait_read_all();
    }
  }
  if (tid < head) kw[tid] = sk[phase + tid];
  if (tid < tail) kw[head + 4 * body + tid] = sk[phase + head + 4 * body + tid];
  // the shared buffers are reused by this CTA's next chunk, whose staging
  // bulk copy (async proxy) overwrites keys this chunk wrote generically
  fence_proxy_async_smem();
  __syncthreads();
  return true;
}

// Length check of the whole batch BEFORE any key moves (networks.hpp:99-103
// throws before touching the window): *status = NS_ERR_INVALID if some array
// is longer than 8 keys or its offsets decrease.  A pure stream over the
// offsets: every thread checks 4 consecutive arrays per 16-byte load (the
// 5th offset comes from the next lane), 4 loads in flight per thread.
__global__ void __launch_bounds__(256) batch_validate_kernel(const uint32_t* __restrict__ offsets,
                                                             int64_t num_arrays,
                                                             int* __restrict__ status) {
  pdl_trigger();  // the sort kernel may start staging and sorting right away
  const int lane = threadIdx.x & 31;
  bool bad = false;
  // offsets[0, head) one by one until a 16-byte boundary, then quads
  const int head = (int)min(num_arrays, (int64_t)(((16 - (reinterpret_cast<uintptr_t>(offsets) & 15)) & 15) >> 2));
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  if (gtid < head) {
    const uint32_t a = __ldg(offsets + gtid), b = __ldg(offsets + gtid + 1);
    bad |= b < a || b - a > 8u;
  }
  const uint4* q = reinterpret_cast<const uint4*>(offsets + head);
  const int64_t nq = (num_arrays - head) / 4;  // whole quads of arrays
  constexpr int U = 4;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U; base < nq; base += nthreads * U) {
    // one round trip per iteration: the quads and, for the lanes whose
    // neighbour does not hold it, the 5th offset are all loaded up front
    uint4 v[U];
    uint32_t own[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x + threadIdx.x;
      v[u] = i < nq ? __ldcs(q + i) : make_uint4(0, 0, 0, 0);
      own[u] = (i < nq && (lane == 31 || i + 1 >= nq)) ? __ldg(offsets + head + 4 * i + 4) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x + threadIdx.x;
      uint32_t n = __shfl_down_sync(0xffffffffu, v[u].x, 1);
      if (lane == 31 || i + 1 >= nq) n = own[u];
      if (i < nq) {
        const uint4 x = v[u];
        bad |= x.y < x.x || x.y - x.x > 8u || x.z < x.y || x.z - x.y > 8u || x.w < x.z ||
               x.w - x.z > 8u || n < x.w || n - x.w > 8u;
      }
    }
  }
  // the last (num_arrays - head) % 4 arrays one by one
  const int64_t t0 = head + 4 * nq;
  if (gtid < num_arrays - t0) {
    const uint32_t a = __ldg(offsets + t0 + gtid), b = __ldg(offsets + t0 + gtid + 1);
    bad |= b < a || b - a > 8u;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(status, NS_ERR_INVALID);
}

// One CTA per chunk of kBaArr arrays.  Launched as a programmatic dependent
// of the validation kernel: it stages and sorts its chunk while the
// validation still runs and writes nothing if the validation flagged the
// batch (batch_chunk).
__global__ void __launch_bounds__(kBaNT, NSB_BATCH_MINB)
    sort_small_batch_kernel(int32_t* __restrict__ keys, const uint32_t* __restrict__ offsets,
                            int64_t num_arrays, int* __restrict__ status) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t tma_uses = 0;
  if (!batch_chunk(keys, offsets, num_arrays, (int64_t)blockIdx.x * kBaArr, &bar, tma_uses,
                   status) &&
      threadIdx.x == 0)
    atomicExch(status, NS_ERR_INVALID);
}

// Validation flag + pinned host mirror per (host thread, device), allocated
// once: concurrent calls from different host threads never share a flag, and
// one thread's calls are serialised by the read-back that ends each call.
struct BatchFlag {
  int* dev = nullptr;
  int* host = nullptr;
};
struct BatchFlags {
  BatchFlag f[64];
  ~BatchFlags() {
    for (auto& x : f) {
      if (x.dev) cudaFree(x.dev);
      if (x.host) cudaFreeHost(x.host);
    }
  }
};
static thread_local BatchFlags t_flags;

static int batch_flag(BatchFlag** out) {
  int dev = 0;
  NSB_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  if (dev < 0 || dev >= 64) return NS_ERR_INVALID;
  BatchFlag& f = t_flags.f[dev];
  if (!f.dev) {
    NSB_TRY(check_cuda(cudaMalloc(reinterpret_cast<void**>(&f.dev), sizeof(int)), "cudaMalloc"));
    NSB_TRY(check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&f.host), sizeof(int),
                                     cudaHostAllocDefault),
                       "cudaHostAlloc"));
  }
  *out = &f;
  return NS_OK;
}

// ---------------------------------------------------------------------------
// Checking helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// key bit pattern fed to the digest mix: uint32 for int32 (oracle_multiset_
// digest_i32), the full 64 bits for int64
__device__ __forceinline__ uint64_t key_bits(int32_t k) { return (uint64_t)(uint32_t)k; }
__device__ __forceinline__ uint64_t key_bits(int64_t k) { return (uint64_t)k; }

template <class Key>
__global__ void digest_kernel(const Key* __restrict__ keys, int64_t n,
                              unsigned long long* __restrict__ out) {
  unsigned long long s = 0, x = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t m = mix64(key_bits(keys[i]) + 0x9E3779B97F4A7C15ull);
    s += m;
    x ^= m;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(kFull, s, o);
    x ^= __shfl_xor_sync(kFull, x, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, s);
    atomicXor(out + 1, x);
  }
}

template <class Key>
__global__ void inversions_kernel(const Key* __restrict__ keys, int64_t n,
                                  unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += keys[i] > keys[i + 1];
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

static int sm_count_of_current() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static int grid_for(int64_t n, int nt) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + nt - 1) / nt;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

// Segments of up to one CTA (16384 keys) are tile-sorted one CTA each; larger
// segments go, all at once, through the quick sort's device-planned partition
// (every segment is a level-0 segment of one batched launch sequence) or, for
// the merge sort, through one merge sort per segment (stream-ordered).
template <class Key>
static size_t segmented_temp(size_t num_segments, size_t seg_len) {
  if (seg_len <= (size_t)kSmT || num_segments == 0) return 0;
  if (num_segments > SIZE_MAX / seg_len) return 0;
  // the merge path sorts every segment at once: a merge sort's scratch for all keys
  const size_t n = num_segments * seg_len;
  const size_t ms = sizeof(Key) == 4 ? merge_sort_temp(n) : merge_sort_temp_i64(n);
  return std::max(ms, quick_sort_segments_temp(num_segments, seg_len, sizeof(Key)));
}

template <class Key>
static int segmented_sort(Key* d_keys, size_t num_segments, size_t seg_len, int algorithm,
                          uint32_t width_mask, int varsort_max, void* d_temp, size_t temp_bytes,
                          cudaStream_t s) {
  if (algorithm != NS_MERGE_SORT && algorithm != NS_QUICK_SORT) return NS_ERR_INVALID;
  if (num_segments == 0 || seg_len <= 1) return NS_OK;
  if (!d_keys) return NS_ERR_INVALID;
  if (num_segments > (size_t)INT64_MAX / sizeof(Key) / seg_len) return NS_ERR_INVALID;
  const int leaf = leaf_of(width_mask, varsort_max);
  if (seg_len <= (size_t)kSmT) return tile_sort_segments_t(d_keys, num_segments, seg_len, leaf, s);
  // quick sort: segments of up to qs_base_max() keys are its base case (the
  // merge layer, all segments at once: 0.57-0.9 ms per 2^26 keys against 1.1)
  if (algorithm == NS_QUICK_SORT && seg_len > qs_base_max())
    return quick_sort_segments_device(d_keys, num_segments, seg_len, leaf, d_temp, temp_bytes, s);
  return merge_sort_segments_t(d_keys, num_segments, seg_len, leaf, d_temp, temp_bytes, s);
}

}  // namespace nsb

using namespace nsb;

extern "C" {

const char* ns_status_string(int status) {
  switch (status) {
    case NS_OK: return "ok";
    case NS_ERR_INVALID: return "invalid argument";
    case NS_ERR_CUDA: return "CUDA error";
    case NS_ERR_OOM: return "out of memory";
    case NS_ERR_TEMP: return "scratch buffer too small";
    case NS_ERR_NCCL: return "NCCL unavailable or failed";
    default: return "unknown status";
  }
}

int ns_version(void) { return 100; }

#if NSB_CHECKED
// Checked build only (not in the header): a kernel whose NSB_DCHECK fails on
// purpose, so the tests can show that the device-side checks are live (the
// launch must end in a trap and the message must name the condition).
__global__ void nsb_checked_selftest_kernel(int bound) {
  const int i = (int)threadIdx.x;
  NSB_DCHECK(i < bound);
}
int ns_checked_selftest(void) {
  nsb_checked_selftest_kernel<<<1, 32>>>(16);
  const cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? NS_OK : NS_ERR_CUDA;
}
#endif


int ns_leaf_width(uint32_t width_mask, int varsort_max) { return leaf_of(width_mask, varsort_max); }

int ns_network_comparators(int width, uint8_t* pairs, int cap) {
  auto emit = [&](const Pair* p, int cnt) {
    for (int i = 0; i < cnt && i < cap; ++i) {
      pairs[2 * i] = p[i].lo;
      pairs[2 * i + 1] = p[i].hi;
    }
    return cnt;
  };
  switch (width) {
    case 2: return emit(Net<2>::P, Net<2>::N);
    case 3: return emit(Net<3>::P, Net<3>::N);
    case 4: return emit(Net<4>::P, Net<4>::N);
    case 5: return emit(Net<5>::P, Net<5>::N);
    case 6: return emit(Net<6>::P, Net<6>::N);
    case 7: return emit(Net<7>::P, Net<7>::N);
    case 8: return emit(Net<8>::P, Net<8>::N);
    default: return -1;
  }
}

size_t ns_merge_sort_temp_bytes(size_t n) { return merge_sort_temp(n); }

int ns_merge_sort_i32(int32_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream) {
  if (n > 0 && d_keys == nullptr) return NS_ERR_INVALID;
  if (n > (size_t)INT64_MAX / 4) return NS_ERR_INVALID;
  return merge_sort_device(d_keys, n, leaf_of(width_mask, varsort_max), d_temp, temp_bytes,
                           static_cast<cudaStream_t>(stream));
}

size_t ns_merge_sort_temp_bytes_i64(size_t n) { return merge_sort_temp_i64(n); }

int ns_merge_sort_i64(int64_t* d_keys, size_t n, uint32_t width_mask, int varsort_max,
                      void* d_temp, size_t temp_bytes, void* stream) {
  if (n > 0 && d_keys == nullptr) return NS_ERR_INVALID;
  if (n > (size_t)INT64_MAX / 8) return NS_ERR_INVALID;
  return merge_sort_device(d_keys, n, leaf_of(width_mask, varsort_max), d_temp, temp_bytes,
                           static_cast<cudaStream_t>(stream));
}

int ns_sort_small_batch_async_i32(int32_t* d_keys, const uint32_t* d_offsets, size_t num_arrays,
                                  int* d_status, void* stream) {
  if (!d_status) return NS_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  NSB_TRY(check_cuda(cudaMemsetAsync(d_status, 0, sizeof(int), s), "cudaMemsetAsync"));
  if (num_arrays == 0) return NS_OK;
  if (!d_keys || !d_offsets) return NS_ERR_INVALID;
  if (num_arrays >= (size_t)UINT32_MAX) return NS_ERR_INVALID;
  {
    Prof prof(PK_BATCH, s);
    // four CTAs per SM: the sort CTAs share the SMs with it (PDL)
    const int64_t vg = std::min<int64_t>((int64_t)(num_arrays / 4096 + 1), 4 * sm_count_of_current());
    batch_validate_kernel<<<(unsigned)vg, 256, 0, s>>>(d_offsets, (int64_t)num_arrays, d_status);
  }
  NSB_TRY(check_launch("batch_validate_kernel"));
  const int64_t ctas = (int64_t)((num_arrays + kBaArr - 1) / kBaArr);
  {
    Prof prof(PK_BATCH, s);
    const cudaError_t e = launch_pdl(0, sort_small_batch_kernel, (unsigned)ctas, kBaNT, 0, s, d_keys,
                                     d_offsets, (int64_t)num_arrays, d_status);
    if (e != cudaSuccess) return check_cuda(e, "sort_small_batch_kernel");
  }
  return check_launch("sort_small_batch_kernel");
}

int ns_sort_small_batch_i32(int32_t* d_keys, const uint32_t* d_offsets, size_t num_arrays,
                            void* stream) {
  if (num_arrays == 0) return NS_OK;
  if (!d_keys || !d_offsets) return NS_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  BatchFlag* f = nullptr;
  NSB_TRY(batch_flag(&f));
  NSB_TRY(ns_sort_small_batch_async_i32(d_keys, d_offsets, num_arrays, f->dev, stream));
  // reading the status back is the only device->host traffic of this call
  NSB_TRY(check_cuda(cudaMemcpyAsync(f->host, f->dev, sizeof(int), cudaMemcpyDeviceToHost, s),
                     "cudaMemcpyAsync"));
  NSB_TRY(check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize"));
  return *f->host ? NS_ERR_INVALID : NS_OK;
}

size_t ns_segmented_sort_temp_bytes(size_t num_segments, size_t seg_len) {
  return segmented_temp<int32_t>(num_segments, seg_len);
}

int ns_segmented_sort_i32(int32_t* d_keys, size_t num_segments, size_t seg_len, int algorithm,
                          uint32_t width_mask, int varsort_max, void* d_temp,
                          size_t temp_bytes, void* stream) {
  return segmented_sort(d_keys, num_segments, seg_len, algorithm, width_mask, varsort_max, d_temp,
                        temp_bytes, static_cast<cudaStream_t>(stream));
}

size_t ns_segmented_sort_temp_bytes_i64(size_t num_segments, size_t seg_len) {
  return segmented_temp<int64_t>(num_segments, seg_len);
}

int ns_segmented_sort_i64(int64_t* d_keys, size_t num_segments, size_t seg_len, int algorithm,
                          uint32_t width_mask, int varsort_max, void* d_temp,
                          size_t temp_bytes, void* stream) {
  return segmented_sort(d_keys, num_segments, seg_len, algorithm, width_mask, varsort_max, d_temp,
                        temp_bytes, static_cast<cudaStream_t>(stream));
}

int ns_multiset_digest_i32(const int32_t* d_keys, size_t n, uint64_t* d_out, void* stream) {
  if (!d_out || (n && !d_keys)) return NS_ERR_INVALID;
  if (n == 0) return NS_OK;
  Prof prof(PK_CHECK, static_cast<cudaStream_t>(stream));
  digest_kernel<<<grid_for((int64_t)n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_keys, (int64_t)n, reinterpret_cast<unsigned long long*>(d_out));
  return check_launch("digest_kernel");
}

int ns_count_inversions_i32(const int32_t* d_keys, size_t n, unsigned long long* d_out,
                            void* stream) {
  if (!d_out || (n && !d_keys)) return NS_ERR_INVALID;
  if (n < 2) return NS_OK;
  Prof prof(PK_CHECK, static_cast<cudaStream_t>(stream));
  inversions_kernel<<<grid_for((int64_t)n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_keys, (int64_t)n, d_out);
  return check_launch("inversions_kernel");
}

int ns_multiset_digest_i64(const int64_t* d_keys, size_t n, uint64_t* d_out, void* stream) {
  if (!d_out || (n && !d_keys)) return NS_ERR_INVALID;
  if (n == 0) return NS_OK;
  Prof prof(PK_CHECK, static_cast<cudaStream_t>(stream));
  digest_kernel<<<grid_for((int64_t)n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_keys, (int64_t)n, reinterpret_cast<unsigned long long*>(d_out));
  return check_launch("digest_kernel");
}

int ns_count_inversions_i64(const int64_t* d_keys, size_t n, unsigned long long* d_out,
                            void* stream) {
  if (!d_out || (n && !d_keys)) return NS_ERR_INVALID;
  if (n < 2) return NS_OK;
  Prof prof(PK_CHECK, static_cast<cudaStream_t>(stream));
  inversions_kernel<<<grid_for((int64_t)n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      d_keys, (int64_t)n, d_out);
  return check_launch("inversions_kernel");
}

}  // extern "C"
