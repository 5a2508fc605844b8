// mergesort.cuh — the merge layer on sm_100a.
//
// Replaces the reference's merge sort (/root/reference/proj/include/netsort/
// hybrid.hpp): the top-down recursion merge_sort_rec (81-95) and the stable
// two-cursor merge_runs (61-79) become
//   1. blocksort_kernel : one CTA sorts a tile of T = NT*K keys entirely on
//      chip — 128-bit loads into registers, the config-shaped network base
//      case per thread (networks.cuh), a warp-level bitonic stage on
//      __shfl_xor_sync that turns 32 per-thread runs into one 32*K run, then
//      merge-path merges in shared memory up to T;
//   2. merge passes     : merge_partition_kernel finds the merge-path split
//      of every output tile with one binary search in HBM/L2, and
//      merge_pass_kernel stages the two input slices of its tile in shared
//      memory and merges them, ping-ponging between the key buffer and one
//      scratch buffer of n keys (the reference's `new T[n]`, hybrid.hpp:163).
// The recursion shape does not need to be mirrored: for int32 keys every
// correct sort yields the same bytes, which the parity tests
// check bit-for-bit against the oracle.
#pragma once
#include <cstdint>
#include <climits>
#include <cstring>

#include "common.cuh"
#include "networks.cuh"
#include "tma.cuh"

namespace nsb {

constexpr unsigned kFull = 0xffffffffu;

// Warp bitonic merge stage: on entry every lane holds K sorted keys
// (blocked: lane l owns warp positions [l*K, l*K+K)); after LEVELS levels
// every aligned group of 2^LEVELS lanes holds one sorted run.
template <int LEVELS, int K, class T>
__device__ __forceinline__ void warp_bitonic(T (&v)[K], int lane) {
#pragma unroll
  for (int s = 0; s < LEVELS; ++s) {
    // flip step: (lane, i) <-> (lane ^ (2^(s+1)-1), K-1-i).  Positions i and
    // K-1-i exchange with each other, so they are done as a pair: two
    // temporaries live instead of K (the 40-register tile sort spilled here)
    {
      const int fm = (2 << s) - 1;
      const bool upper = (lane >> s) & 1;
#pragma unroll
      for (int i = 0; i < K / 2; ++i) {
        const T ti = __shfl_xor_sync(kFull, v[K - 1 - i], fm);
        const T tj = __shfl_xor_sync(kFull, v[i], fm);
        v[i] = upper ? max(v[i], ti) : min(v[i], ti);
        v[K - 1 - i] = upper ? max(v[K - 1 - i], tj) : min(v[K - 1 - i], tj);
      }
    }
    // cross-lane half-cleaners
#pragma unroll
    for (int j = s - 1; j >= 0; --j) {
      const bool upper = (lane >> j) & 1;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const T o = __shfl_xor_sync(kFull, v[i], 1 << j);
        v[i] = upper ? max(v[i], o) : min(v[i], o);
      }
    }
    // intra-thread half-cleaners
#pragma unroll
    for (int st = K / 2; st >= 1; st >>= 1) {
#pragma unroll
      for (int i = 0; i < K; ++i)
        if ((i & st) == 0) cx(v[i], v[i + st]);
    }
  }
}

// Shared-memory layout: one pad word after every 32 keys.  Thread cursors in
// the merge levels sit ~K/2 keys apart (K = keys per thread), i.e. on the same
// bank every 32/(K/2) lanes without padding; with it every warp-wide blocked
// access (thread t touching t*K + k) and every coalesced access is bank
// conflict free, and data-dependent merge cursors spread across banks.
//
// Keys are int32 (the BASELINE configs) or int64 (the reference's own
// benchmark type, datagen.hpp:47).  An int64 key covers two banks, and 64-bit
// shared accesses are served per half-warp, so its pad is one key per 16.
template <class Key>
struct KeyT;
template <>
struct KeyT<int32_t> {
  static constexpr int32_t kMax = INT_MAX;
  static constexpr int kPadShift = 5;
};
template <>
struct KeyT<int64_t> {
  static constexpr int64_t kMax = INT64_MAX;
  static constexpr int kPadShift = 4;
};
// keys per 16-byte vector
template <class Key>
__host__ __device__ constexpr int kpv() { return 16 / (int)sizeof(Key); }

template <class Key = int32_t>
__host__ __device__ constexpr int pad_idx(int i) { return i + (i >> KeyT<Key>::kPadShift); }
template <class Key = int32_t>
__host__ __device__ constexpr int padded_words(int T) { return T + (T >> KeyT<Key>::kPadShift) + 8; }
// bytes of dynamic shared memory a padded T-key tile needs
template <class Key>
__host__ __device__ constexpr int padded_bytes(int T) { return padded_words<Key>(T) * (int)sizeof(Key); }

// 16 bytes <-> kpv<Key>() keys (register moves only)
template <class Key>
__device__ __forceinline__ void unpack16(const int4& x, Key (&e)[kpv<Key>()]) {
  memcpy(e, &x, 16);
}
template <class Key>
__device__ __forceinline__ int4 pack16(const Key (&e)[kpv<Key>()]) {
  int4 x;
  memcpy(&x, e, 16);
  return x;
}

// Read-only view of a run that starts at logical index `off` of padded smem.
template <class Key = int32_t>
struct SmemRun {
  const Key* s;
  int off;
  __device__ __forceinline__ Key operator[](int i) const { return s[pad_idx<Key>(off + i)]; }
};

// Merge-path split: number of elements taken from A among the first `diag`
// outputs of merge(A, B) when A wins ties (same rule as merge_runs,
// hybrid.hpp:71-75).
template <class IDX, class PA, class PB>
__device__ __forceinline__ IDX merge_path(PA A, IDX a_len, PB B, IDX b_len, IDX diag) {
  IDX lo = diag > b_len ? diag - b_len : 0;
  IDX hi = diag < a_len ? diag : a_len;
  while (lo < hi) {
    const IDX mid = (lo + hi) >> 1;
    if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Serial merge of K outputs starting at (a, b).
template <int K, class SA, class SB, class Key>
__device__ __forceinline__ void serial_merge(SA A, int a_len, SB B, int b_len, int a, int b,
                                             Key (&v)[K]) {
  // clamped indices keep every read inside the staged tile; the clamped
  // value is never selected because the exhausted side loses every test
  const int a_last = max(a_len - 1, 0), b_last = max(b_len - 1, 0);
  Key ka = A[min(a, a_last)];
  Key kb = B[min(b, b_last)];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool take_a = (b >= b_len) || (a < a_len && ka <= kb);
    v[k] = take_a ? ka : kb;
    if (take_a) {
      ++a;
      ka = A[min(a, a_last)];
    } else {
      ++b;
      kb = B[min(b, b_last)];
    }
  }
}

// Blocked registers <-> padded smem (thread t owns logical [t*K, t*K+K)).
template <int K, class Key>
__device__ __forceinline__ void regs_to_smem(Key* sm, const Key (&v)[K]) {
  const int base = threadIdx.x * K;
#pragma unroll
  for (int k = 0; k < K; ++k) sm[pad_idx<Key>(base + k)] = v[k];
}
template <int K, class Key>
__device__ __forceinline__ void smem_to_regs(const Key* sm, Key (&v)[K]) {
  const int base = threadIdx.x * K;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = sm[pad_idx<Key>(base + k)];
}

// Coalesced global -> padded smem for a T-key tile (`valid` live keys, the
// rest padded with the key maximum, which sorts to the tail).
template <int NT, int T, class Key>
__device__ __forceinline__ void tile_load(const Key* in, int valid, Key* sm) {
  constexpr int PV = kpv<Key>();
  const int tid = threadIdx.x;
  if (valid == T && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    const int4* p = reinterpret_cast<const int4*>(in);
#pragma unroll
    for (int q = 0; q < T / PV / NT; ++q) {
      const int j = q * NT + tid;
      Key e[PV];
      unpack16<Key>(__ldcs(p + j), e);  // streamed: every key is read exactly once
      const int i = pad_idx<Key>(PV * j);  // one vector never straddles a pad
#pragma unroll
      for (int u = 0; u < PV; ++u) sm[i + u] = e[u];
    }
  } else {
#pragma unroll 4
    for (int i = tid; i < T; i += NT) sm[pad_idx<Key>(i)] = i < valid ? in[i] : KeyT<Key>::kMax;
  }
}

// Stage the two input slices of a merge tile, A = a_ptr[0, la) followed by
// B = b_ptr[0, lb), into padded smem [0, la + lb).  The slices start at
// arbitrary key offsets, so each is covered by 16-byte-aligned chunks that
// are loaded with 128-bit LDGs — ALL of a thread's chunks are issued before
// the first shared-memory store, so every thread keeps up to CH loads in
// flight — and the keys outside the slice are dropped.  [lo, hi) bounds the
// underlying array: a chunk that would cross it is read key by key.
template <int NT, int TM>
__device__ __forceinline__ void stage_slices(const int32_t* lo, const int32_t* hi,
                                             const int32_t* a_ptr, int la, const int32_t* b_ptr,
                                             int lb, int32_t* sm) {
  constexpr int CH = (TM / 4 + 3 + NT - 1) / NT;
  const int tid = threadIdx.x;
  const int32_t* a_al = reinterpret_cast<const int32_t*>(reinterpret_cast<uintptr_t>(a_ptr) & ~uintptr_t(15));
  const int32_t* b_al = reinterpret_cast<const int32_t*>(reinterpret_cast<uintptr_t>(b_ptr) & ~uintptr_t(15));
  const int a_shift = (int)(a_ptr - a_al), b_shift = (int)(b_ptr - b_al);
  const int ca = la ? (a_shift + la + 3) >> 2 : 0;
  const int cb = lb ? (b_shift + lb + 3) >> 2 : 0;
  int4 x[CH];
#pragma unroll
  for (int u = 0; u < CH; ++u) {
    const int c = u * NT + tid;
    if (c < ca + cb) {
      const int32_t* p = c < ca ? a_al + 4 * c : b_al + 4 * (c - ca);
      if (p >= lo && p + 4 <= hi) {
        x[u] = __ldcs(reinterpret_cast<const int4*>(p));
      } else {
        x[u].x = (p + 0 >= lo && p + 0 < hi) ? p[0] : 0;
        x[u].y = (p + 1 >= lo && p + 1 < hi) ? p[1] : 0;
        x[u].z = (p + 2 >= lo && p + 2 < hi) ? p[2] : 0;
        x[u].w = (p + 3 >= lo && p + 3 < hi) ? p[3] : 0;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < CH; ++u) {
    const int c = u * NT + tid;
    if (c < ca + cb) {
      const bool in_a = c < ca;
      const int first = in_a ? 4 * c - a_shift : la + 4 * (c - ca) - b_shift;
      const int lim_lo = in_a ? 0 : la, lim_hi = in_a ? la : la + lb;
      const int32_t e[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = first + q;
        if (i >= lim_lo && i < lim_hi) sm[pad_idx(i)] = e[q];
      }
    }
  }
}

// Coalesced padded smem -> global for the first `valid` keys of a T-key tile.
template <int NT, int T, class Key>
__device__ __forceinline__ void tile_store(const Key* sm, Key* out, int valid) {
  constexpr int PV = kpv<Key>();
  const int tid = threadIdx.x;
  if (valid == T && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    int4* p = reinterpret_cast<int4*>(out);
#pragma unroll
    for (int q = 0; q < T / PV / NT; ++q) {
      const int j = q * NT + tid;
      const int i = pad_idx<Key>(PV * j);
      Key e[PV];
#pragma unroll
      for (int u = 0; u < PV; ++u) e[u] = sm[i + u];
      __stcs(p + j, pack16<Key>(e));
    }
  } else {
#pragma unroll 4
    for (int i = tid; i < valid; i += NT) out[i] = sm[pad_idx<Key>(i)];
  }
}

// ---------------------------------------------------------------------------
// Tile sort: one CTA sorts `valid` <= T = NT*K keys from `in` into `out` (in
// place allowed) on chip.  Shared by the tiled merge sort, the segmented sort
// and the quick-sort bucket sort.
// ---------------------------------------------------------------------------

// Padded variant (one pad word per 32 keys, serial merge with clamped
// indices): the fallback for shapes the skewed variant below does not cover
// (32-thread tiles, int64 tiles other than 8 or 16 keys per thread).  int32
// tiles of up to 1024 threads and int64 tiles of 8 / 16 keys per thread use
// the skewed variant.
// From registers (thread t holds K of the tile's keys, any assignment, pads
// the key maximum): the sorted tile is left in padded smem, logical key i at
// sm[pad_idx(i)].
template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort_padded_regs(Key (&v)[K], Key* sm) {
  constexpr int T = NT * K;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  thread_sort<LEAF>(v);  // the network base case (try_base_case, hybrid.hpp:48-56)
  if constexpr (NT >= 32) warp_bitonic<5>(v, lane);
#pragma unroll 1
  for (int R = 32 * K; R < T; R *= 2) {
    __syncthreads();
    regs_to_smem<K>(sm, v);
    __syncthreads();
    const int pos = tid * K;
    const int pair = pos & ~(2 * R - 1);
    const int diag = pos - pair;
    const SmemRun<Key> A{sm, pair}, B{sm, pair + R};
    const int a = merge_path<int>(A, R, B, R, diag);
    serial_merge<K>(A, R, B, R, a, diag - a, v);
  }
  __syncthreads();
  regs_to_smem<K>(sm, v);
  __syncthreads();
}

template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort_padded(const Key* in, Key* out, int valid, Key* sm) {
  constexpr int T = NT * K;
  const int tid = threadIdx.x;
  const int lane = tid & 31;

  tile_load<NT, T>(in, valid, sm);
  __syncthreads();
  Key v[K];
  smem_to_regs<K>(sm, v);

  thread_sort<LEAF>(v);  // the network base case (try_base_case, hybrid.hpp:48-56)
  if constexpr (NT >= 32) warp_bitonic<5>(v, lane);

  // shared-memory merge-path levels: runs of 32*K up to T
#pragma unroll 1
  for (int R = 32 * K; R < T; R *= 2) {
    __syncthreads();
    regs_to_smem<K>(sm, v);
    __syncthreads();
    const int pos = tid * K;
    const int pair = pos & ~(2 * R - 1);
    const int diag = pos - pair;
    const SmemRun<Key> A{sm, pair}, B{sm, pair + R};
    const int a = merge_path<int>(A, R, B, R, diag);
    serial_merge<K>(A, R, B, R, a, diag - a, v);
  }

  __syncthreads();
  regs_to_smem<K>(sm, v);
  __syncthreads();
  tile_store<NT, T>(sm, out, valid);
}

//
// Merge levels (v5).  After the warp bitonic stage every warp holds one
// sorted 512-key run (16 keys per lane, blocked).  The runs go to shared
// memory in a GAP layout — run r at r*(R+4), its +inf sentinel right after
// it — so each level can use the pass kernel's merge loop: byte-offset
// cursors clamped at the sentinel, no bounds tests, no index arithmetic.
// Output diagonals are skewed inside each warp (lane l starts at
// 16l + ((l>>1)&15) and emits 16 or 17 keys; lane 31 emits the last one), so
// for any k the 32 lanes' k-th output stores fall on 32 different banks
// without padding words; every lane runs the same 17 unguarded merge steps
// and only the stores are predicated.
#ifndef NSB_SKEW_MAX_NT
#define NSB_SKEW_MAX_NT 1024
#endif
// int64 tiles of 16 keys per thread (<512,16>) in the skewed layout: with
// the producer/loser loop they fit 64 registers without spills; measured
// equal for the merge-sort tile and 8 % faster for the 16 M int64 quick-sort
// bucket tiles (tools/i64_ab.sh)
// Warp bitonic levels of the skewed tile sort: 4 = 16-lane runs and one more
// shared-memory merge level than 5 (a warp run).  Measured (tools/ab_all.sh,
// tools/i64_quick_ab.sh): int32 2^30 tile sort 7.72 -> 7.48 ms, segmented
// 7.60 -> 7.47 ms; int64 2^28 tile sort 5.06 -> 4.57 ms, int64 16M quick-sort
// buckets 538 -> 478 us (a bitonic level costs more ALU than a merge level
// costs shared-memory wavefronts).
#ifndef NSB_TS_WARP_LEVELS
#define NSB_TS_WARP_LEVELS 4
#endif
#ifndef NSB_SKEW64_K16
#define NSB_SKEW64_K16 1
#endif
template <int NT, int K, class Key>
__host__ __device__ constexpr bool cta_sort_skewed() {
  return ((sizeof(Key) == 4 && (K == 16 || K == 32)) || (sizeof(Key) == 8 && (K == 8 || (NSB_SKEW64_K16 && K == 16)))) &&
         NT > 32 && NT <= NSB_SKEW_MAX_NT;
}

// Sentinel pad after every run of the skewed layout: a lane's producer
// cursor can run at most K+1 keys past its run's end (all-key-maximum
// tail, see the merge loop), so K+4 sentinels (16-byte multiple) keep every
// read inside sentinels without a clamp.
template <int K>
__host__ __device__ constexpr int skew_pad() { return K + 4; }

// Bitonic levels of the skewed tile sort and its sentinel pad (see
// cta_sort_skewed_body).
template <int NT, int K, class Key>
__host__ __device__ constexpr int ts_warp_levels() {
  return NT <= 32 ? 5
         : (NSB_TS_WARP_LEVELS >= 4 || 128 / (int)sizeof(Key) == K) ? NSB_TS_WARP_LEVELS
                                                                      : 4;
}
template <int NT, int K, class Key>
__host__ __device__ constexpr int ts_gap() {
  return (ts_warp_levels<NT, K, Key>() == 3 && sizeof(Key) == 4) ? 48 : skew_pad<K>();
}

// Dynamic shared memory of a tile-sort CTA (either layout).
template <int NT, int K, class Key>
__host__ __device__ constexpr int tile_smem_bytes() {
  constexpr int T = NT * K;
  constexpr int pw = padded_words<Key>(T);
  constexpr int sw = T + (NT > 32 ? (NT >> ts_warp_levels<NT, K, Key>()) : 1) * ts_gap<NT, K, Key>() + 8;
  return (cta_sort_skewed<NT, K, Key>() && sw > pw ? sw : pw) * (int)sizeof(Key);
}

template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort_skewed_body(const Key* in, Key* out, int valid, Key* sm);

template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort(const Key* in, Key* out, int valid, Key* sm) {
  if constexpr (!cta_sort_skewed<NT, K, Key>()) {
    cta_sort_padded<NT, K, LEAF>(in, out, valid, sm);
  } else {
    cta_sort_skewed_body<NT, K, LEAF>(in, out, valid, sm);
  }
}

template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort_regs(Key (&v)[K], Key* out, int valid, Key* sm);

// Global -> registers for the skewed tile sort.  A full, 16-byte-aligned
// tile (every tile of a merge sort but the last) skips the shared-memory
// staging: the register stage accepts any assignment of keys to threads, so
// thread t takes vector q*NT + t and every warp-wide load is one coalesced
// 512-byte row.  Partial or unaligned tiles are staged through shared memory
// into the BLOCKED assignment (thread t owns [t*K, t*K + K), pads the key
// maximum), which keeps cta_sort_regs' all-padding-warp skip valid.
template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort_skewed_body(const Key* in, Key* out, int valid, Key* sm) {
  constexpr int T = NT * K;
  constexpr int PV = kpv<Key>();
  Key v[K];
  if (valid == T && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    const int4* p = reinterpret_cast<const int4*>(in);
#pragma unroll
    for (int q = 0; q < K / PV; ++q) {
      Key e[PV];
      unpack16<Key>(__ldcs(p + q * NT + threadIdx.x), e);  // streamed: read once
#pragma unroll
      for (int u = 0; u < PV; ++u) v[q * PV + u] = e[u];
    }
  } else {
    tile_load<NT, T>(in, valid, sm);
    __syncthreads();
    smem_to_regs<K>(sm, v);
  }
  cta_sort_regs<NT, K, LEAF>(v, out, valid, sm);
}

// v as NQ quads of PV keys: quad i <- quad (i + r) mod NQ, branch-free (one
// conditional cyclic shift per bit of r, walked cycle by cycle so one
// temporary quad is live at a time).
template <int NQ, int PV, class Key, int K>
__device__ __forceinline__ void rotate_quads(Key (&v)[K], int r) {
#pragma unroll
  for (int b = 1; b < NQ; b <<= 1) {
    const bool on = (r & b) != 0;
#pragma unroll
    for (int c0 = 0; c0 < b; ++c0) {  // gcd(NQ, b) = b cycles of length NQ / b
      Key t[PV];
#pragma unroll
      for (int u = 0; u < PV; ++u) t[u] = v[c0 * PV + u];
#pragma unroll
      for (int j = 0; j < NQ / b - 1; ++j) {
        const int i = c0 + j * b, nx = i + b;
#pragma unroll
        for (int u = 0; u < PV; ++u) v[i * PV + u] = on ? v[nx * PV + u] : v[i * PV + u];
      }
      const int last = c0 + (NQ / b - 1) * b;
#pragma unroll
      for (int u = 0; u < PV; ++u) v[last * PV + u] = on ? t[u] : v[last * PV + u];
    }
  }
}

// The skewed tile sort from registers: thread t holds K of the tile's T keys
// (any assignment — the result is the sorted multiset; pad with the key
// maximum), `valid` keys are stored to out (nullptr: left in sm[0, T)).
template <int NT, int K, int LEAF, class Key>
__device__ __forceinline__ void cta_sort_regs(Key (&v)[K], Key* out, int valid, Key* sm) {
  static_assert(cta_sort_skewed<NT, K, Key>(), "cta_sort_regs is the skewed layout");
  constexpr int T = NT * K;
  const int tid = threadIdx.x;
  const int lane = tid & 31;

  // Tile positions >= valid hold the key maximum at every stage (a sorted run
  // keeps its pads at its end), so a warp whose keys are all padding skips the
  // register stage and a lane whose outputs all lie at or past `valid` writes
  // the maximum without merging: a partial tile costs about its valid keys.
  const bool warp_pad = (tid & ~31) * K >= valid;
  constexpr int WL = ts_warp_levels<NT, K, Key>();
  static_assert(WL >= 3 && WL <= 5, "the merge levels take runs of 8, 16 or 32 lanes");
  if (!warp_pad) {
    thread_sort<LEAF>(v);  // the network base case (try_base_case, hybrid.hpp:48-56)
    // NSB_TS_WARP_LEVELS bitonic levels: runs of 2^levels lanes (5: one run per
    // warp; 4: one per half-warp and one more shared-memory level)
    // 3 levels only where a bank row holds exactly K keys (int32 x 32, int64 x 16):
    // the sub-warp merge level's skew pattern is proven for that shape alone
    if constexpr (NT >= 32) warp_bitonic<WL>(v, lane);
  }

  if constexpr (NT <= 32) {
    __syncthreads();
    regs_to_smem<K>(sm, v);
    __syncthreads();
    tile_store<NT, T>(sm, out, valid);
  } else {
    // a bank row holds S = 128/KB keys.  Lanes whose diagonals are K apart
    // hit S/K residues of a row: the skew spreads them over all of it —
    // (l>>1) when S == 2K, l itself when S == K
    constexpr int S = 128 / (int)sizeof(Key);
    static_assert(S == 2 * K || S == K, "skew pattern needs 128/sizeof(Key) in {K, 2K}");
    constexpr int W = 32 * K;  // warp run
    // sentinels after every run; keeps every run 16-byte aligned.  With two
    // output runs per warp (8-lane input runs, int32) the second run's
    // stores must land 16 banks away from the first's: GAP = 16 (mod 32)
    constexpr int GAP = ts_gap<NT, K, Key>();
    static_assert(GAP >= K + 2 && GAP % 4 == 0, "sentinel pad");
    constexpr int PV = kpv<Key>();
    constexpr int KB = (int)sizeof(Key);
    constexpr int KM = K + 1;
    const int warp = tid >> 5;
    constexpr int L0 = K << WL;             // run length after the warp stage
    constexpr int LPR = 1 << WL;            // lanes per run
    __syncthreads();  // every thread is done reading the padded tile
    {
      const int run = (warp << (5 - WL)) + (lane >> WL);
      Key* dst = sm + run * (L0 + GAP) + K * (lane & (LPR - 1));
      const int li = lane & (LPR - 1);
      // Lane li's K keys are 16-byte quads at a stride of K*KB bytes, so at
      // equal q the lanes of a quarter-warp would hit the same 16-byte bank
      // group (8-way conflict for 128-byte lane blocks).  Each lane rotates
      // its quads by r (three conditional cyclic shifts, one temporary quad)
      // and stores quad (q + r) mod NQ at step q: eight distinct groups.
      constexpr int NQ = K / PV;
      static_assert(NQ >= 1 && NQ <= 8 && (NQ & (NQ - 1)) == 0, "quads per lane");
      const int r = NQ == 1 ? 0 : (li / (8 / NQ)) & (NQ - 1);
      rotate_quads<NQ, PV>(v, r);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        Key e[PV];
#pragma unroll
        for (int u = 0; u < PV; ++u) e[u] = v[q * PV + u];
        *reinterpret_cast<int4*>(dst + ((q + r) & (NQ - 1)) * PV) = pack16<Key>(e);
      }
      for (int i = li; i < GAP; i += LPR) sm[run * (L0 + GAP) + L0 + i] = KeyT<Key>::kMax;
    }
    __syncthreads();
    auto skew_of = [](int l) { return S == 2 * K ? ((l >> 1) & (K - 1)) : (l & (S - 1)); };
    const char* smc = reinterpret_cast<const char*>(sm);
#pragma unroll 1
    for (int R = L0; R < T; R *= 2) {
      const int S = R + GAP, S2 = 2 * R + GAP;
      // G lanes per output run (a run of 2R keys; G = 32 and several warps
      // per run once 2R >= W)
      const int G = 2 * R / K < 32 ? 2 * R / K : 32;
      const int li = lane & (G - 1);
      const int RW = G * K;  // outputs of one lane group
      const int skew = skew_of(li);
      const int cnt = li == G - 1 ? RW - (K * (G - 1) + skew_of(G - 1)) : K + skew_of(li + 1) - skew;
      const int wpp = G < 32 ? 1 : 2 * R / W;  // warps per output run
      const int p = G < 32 ? warp * (32 / G) + (lane / G) : warp / wpp;
      const int wi = G < 32 ? 0 : warp - p * wpp;
      const int d = W * wi + K * li + skew;
      const int a_pos = 2 * p * S, b_pos = a_pos + S;
      Key w[KM];
      if (p * 2 * R + d >= valid) {  // every output of this lane is padding
#pragma unroll
        for (int k = 0; k < KM; ++k) w[k] = KeyT<Key>::kMax;
      } else {
      const int a = merge_path<int>(sm + a_pos, R, sm + b_pos, R, d);
      // Producer/loser form of the merge: m is the head of the run that did
      // not emit the last key, ptr the next key of the run that did, mnext
      // the key after m.  Per output: one LDS, a compare, min/max and two
      // cursor selects — no per-side bookkeeping and no clamp (an exhausted
      // run is followed by GAP sentinels; a cursor only passes its first
      // sentinel once m is the key maximum too, i.e. every key left is the
      // maximum).  Ties may come from either run: for keys alone any greedy
      // merge from a merge-path split emits the same values.
      uint32_t ptr = (uint32_t)(a_pos + a) * KB;
      uint32_t mnext = (uint32_t)(b_pos + d - a + 1) * KB;
      Key m = sm[b_pos + d - a];
      NSB_DCHECK(a >= 0 && a <= R && d - a >= 0 && d - a <= R);
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        // a cursor stays inside its run + GAP sentinels (runs at a_pos, b_pos)
        NSB_DCHECK((ptr >= (uint32_t)a_pos * KB && ptr < (uint32_t)(a_pos + R + GAP) * KB) ||
                   (ptr >= (uint32_t)b_pos * KB && ptr < (uint32_t)(b_pos + R + GAP) * KB));
        const Key x = *reinterpret_cast<const Key*>(smc + ptr);
        const bool t = x <= m;
        w[k] = t ? x : m;
        const uint32_t q = ptr + (uint32_t)KB;
        ptr = t ? q : mnext;
        mnext = t ? mnext : q;
        m = t ? m : x;
      }
      }
      __syncthreads();  // every thread is done reading this level's input
      Key* o = sm + p * S2 + d;
      NSB_DCHECK(p * S2 + 2 * R + GAP <= tile_smem_bytes<NT, K, Key>() / KB && d + cnt <= 2 * R);
#pragma unroll
      for (int k = 0; k < KM; ++k)
        if (k < cnt) o[k] = w[k];
      if (wi == 0)
        for (int i = li; i < GAP; i += G) sm[p * S2 + 2 * R + i] = KeyT<Key>::kMax;
      __syncthreads();
    }
    // the sorted tile is sm[0, T); out == nullptr leaves it there (the
    // quick-sort splitter selection and big-bucket fallback read it on chip)
    if (out == nullptr) return;
    if (valid == T && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tma_store_1d(out, sm, (uint32_t)T * (uint32_t)KB);
        bulk_commit();
        bulk_wait_read_all();
      }
    } else {
      for (int i = tid; i < valid; i += NT) out[i] = sm[i];
    }
  }
}

// CTA b sorts [b*stride, b*stride + min(stride, n - b*stride)), stride <= T
// (stride == T for plain tiling, the segment length for segmented sorts).
// Resident CTAs per SM requested for a tile-sort CTA of NT threads.
#ifndef NSB_BS_THREADS_PER_SM
#define NSB_BS_THREADS_PER_SM 2048
#endif
// 32 keys per thread: 512-thread tiles (16384 keys) at 3 CTAs per SM (40
// registers; measured 2^30 tile sort 8.02 -> 7.60 ms, segmented 65,536 x
// 16,384 8.07 -> 7.61 ms), smaller tiles at 1024 threads per SM (64
// registers: the latency-bound sorts of < 2^21 keys run them, and 40
// registers measured slower there, 2^20 49 -> 53 us)
#ifndef NSB_BS_THREADS_PER_SM_K32
#define NSB_BS_THREADS_PER_SM_K32 1536
#endif
#ifndef NSB_BS_THREADS_PER_SM_K32_SMALL
#define NSB_BS_THREADS_PER_SM_K32_SMALL 1024
#endif
#ifndef NSB_BS_THREADS_PER_SM_64
#define NSB_BS_THREADS_PER_SM_64 1024  // int64: 64 registers per thread
#endif
template <int NT, int K, class Key>
__host__ __device__ constexpr int bs_min_blocks() {
  // 0 = no minimum (the padded variant keeps the compiler's own choice)
  // threads per SM by key size and keys per thread (the macros above)
  constexpr int tps = sizeof(Key) == 8 ? NSB_BS_THREADS_PER_SM_64
                                       : (K >= 32 ? (NT >= 512 ? NSB_BS_THREADS_PER_SM_K32
                                                               : NSB_BS_THREADS_PER_SM_K32_SMALL)
                                                  : NSB_BS_THREADS_PER_SM);
  return !cta_sort_skewed<NT, K, Key>() || NT >= tps ? 0 : tps / NT;
}

// Throughput-bound tile sorts (quick-sort buckets: many CTAs, no latency
// floor): 32-key int32 tiles of every size at NSB_BS_THREADS_PER_SM_K32.
#ifndef NSB_BUCKET_TPUT
#define NSB_BUCKET_TPUT 0  // measured: 16M bucket sorts 207 -> 205 us, 1M quick sort 155 -> 164 us
#endif
template <int NT, int K, class Key>
__host__ __device__ constexpr int bs_min_blocks_tput() {
  if constexpr (NSB_BUCKET_TPUT && sizeof(Key) == 4 && K >= 32 && cta_sort_skewed<NT, K, Key>() &&
                NT < NSB_BS_THREADS_PER_SM_K32)
    return NSB_BS_THREADS_PER_SM_K32 / NT;
  return bs_min_blocks<NT, K, Key>();
}

template <int NT, int K, int LEAF, class Key = int32_t>
__global__ void __launch_bounds__(NT, (bs_min_blocks<NT, K, Key>()))
    blocksort_kernel(const Key* src, Key* dst, int64_t n, int stride, int64_t seg_len,
                     int tiles_per_seg) {  // src == dst ok
  extern __shared__ __align__(16) unsigned char sm_raw[];
  Key* sm = reinterpret_cast<Key*>(sm_raw);
  // seg_len > 0: back-to-back segments of seg_len keys, tiles_per_seg tiles
  // each (the last one of a segment partial); else tiles of `stride` keys
  int64_t base;
  int valid;
  if (seg_len > 0) {
    const int64_t sg = blockIdx.x / tiles_per_seg;
    const int t = (int)(blockIdx.x - sg * tiles_per_seg);
    base = sg * seg_len + (int64_t)t * stride;
    valid = (int)min((int64_t)stride, seg_len - (int64_t)t * stride);
  } else {
    base = (int64_t)blockIdx.x * stride;
    valid = (int)min((int64_t)stride, n - base);
  }
  pdl_wait();     // src may be the previous kernel's output
  pdl_trigger();
  cta_sort<NT, K, LEAF>(src + base, dst + base, valid, sm);
}

// ---------------------------------------------------------------------------
// Merge pass: runs of length R in src are merged pairwise into dst.
// ---------------------------------------------------------------------------
struct PassGeom {
  int64_t pair_base, a_len, b_len, diag0;
};

__device__ __forceinline__ PassGeom pass_geom(int64_t pos0, int64_t n, int64_t R) {
  PassGeom g;
  g.pair_base = (pos0 / (2 * R)) * (2 * R);
  g.a_len = min(R, n - g.pair_base);
  g.b_len = max((int64_t)0, min(R, n - g.pair_base - R));
  g.diag0 = pos0 - g.pair_base;
  return g;
}

}  // namespace nsb

// ===========================================================================
// Merge pass v2: pair-local tiles, TMA bulk staging, sentinel merge.
//
// Every run pair (A = [p*2R, p*2R+R), B = the next R keys) is cut into tpp
// output tiles of TMp keys (TMp <= NT*K, a multiple of 4, as even as the pair
// allows), so no tile straddles two pairs and K can be odd: with an odd
// per-thread output count the merge cursors of neighbouring lanes land on
// different shared-memory banks without any padding, which keeps the layout
// TMA-compatible.  One elected thread stages the 16-byte-aligned cover of
// each input slice with a single cp.async.bulk (complete_tx on an mbarrier),
// places +inf sentinels after both slices (no bounds tests in the merge
// loop), and after the merge writes the tile back with one bulk store.
// Slices whose cover would leave the array fall back to plain loads.
// ===========================================================================
#include "tma.cuh"

namespace nsb {

struct PassPlan {
  int64_t R;    // run length being merged
  int64_t n;    // keys
  int tpp;      // tiles per pair
  int tmp;      // keys per tile (<= NT*K, multiple of 4)
  int kp;       // outputs per thread = ceil(tmp / NT)
  int64_t seg_len = 0;  // > 0: runs live in back-to-back segments of seg_len keys
  int64_t pps = 0;      // run pairs per segment (segmented passes)
};

struct TileGeom {
  int64_t pair_base, a_len, b_len, diag0, diag1;
};

__device__ __forceinline__ TileGeom tile_geom(const PassPlan& P, int64_t c) {
  TileGeom g;
  const int64_t pair = c / P.tpp;
  const int64_t lt = c - pair * P.tpp;
  int64_t end = P.n;  // end of the keys this pair belongs to
  if (P.seg_len > 0) {
    const int64_t sg = pair / P.pps;
    const int64_t seg0 = sg * P.seg_len;
    g.pair_base = seg0 + (pair - sg * P.pps) * 2 * P.R;
    end = seg0 + P.seg_len;
  } else {
    g.pair_base = pair * 2 * P.R;
  }
  g.a_len = min(P.R, end - g.pair_base);
  g.b_len = max((int64_t)0, min(P.R, end - g.pair_base - P.R));
  const int64_t pair_len = g.a_len + g.b_len;
  g.diag0 = min(lt * P.tmp, pair_len);
  g.diag1 = min(g.diag0 + P.tmp, pair_len);
  return g;
}

// Merge-path split found by a whole warp with a 32-ary search: each round
// every lane evaluates the predicate A[a] <= B[diag-1-a] at one of 32 evenly
// spaced candidates and a ballot narrows the range 32x — log32 instead of
// log2 dependent global loads (used when a merge pass has too few tiles for a
// separate partition kernel to pay for its launch).  All lanes return the
// split.
template <class Key>
__device__ __forceinline__ int64_t warp_merge_path(const Key* A, int64_t a_len, const Key* B,
                                                   int64_t b_len, int64_t diag) {
  const int lane = threadIdx.x & 31;
  int64_t lo = diag > b_len ? diag - b_len : 0;
  int64_t hi = diag < a_len ? diag : a_len;
  while (lo < hi) {
    const int64_t span = hi - lo;
    const int64_t step = span <= 32 ? 1 : (span + 31) / 32;
    const int64_t a = lo + lane * step;
    const bool valid = a < hi;
    const bool p = valid && (A[a] <= B[diag - 1 - a]);
    const unsigned m = __ballot_sync(0xffffffffu, p);
    const int c = __popc(m);  // P holds on a prefix of the candidates
    if (step == 1) return lo + c;
    const int64_t new_lo = c == 0 ? lo : lo + (int64_t)(c - 1) * step + 1;
    const int64_t new_hi = min(hi, lo + (int64_t)c * step);
    lo = new_lo;
    hi = new_hi;
  }
  return lo;
}

template <class Key>
__global__ void merge_partition_v2_kernel(const Key* __restrict__ src, PassPlan P,
                                          int64_t num_tiles, int64_t* __restrict__ mp) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();  // src is the previous pass's output
  pdl_trigger();
  if (c >= num_tiles) return;
  const TileGeom g = tile_geom(P, c);
  const Key* A = src + g.pair_base;
  mp[c] = merge_path<int64_t>(A, g.a_len, A + g.a_len, g.b_len, g.diag0);
}

// Merge of one staged tile: A = sm[a_pos, a_pos+la), B = sm[b_pos, b_pos+lb)
// (each with one free slot after it for its +inf sentinel), the la+lb merged
// keys written to dst + *s_out_off.  Shared by the pairwise passes and the
// pointer-pair merge (samplesort.cu).  Must be called by all NT threads after
// the staged slices are visible to the CTA.
// Block samples of a pass's output, for the next pass's partition search
// (merge_partition_v3_kernel): for every 256-key block j of the output,
// first[j] = out[256j] and last[j] = out[min(256j + 255, n - 1)].  They are
// 1/128 of the keys and stay L2-resident.
constexpr int kSmpShift = 8;     // 256-key blocks when the tile size allows
constexpr int kSmpShiftMin = 7;  // 128-key blocks otherwise (sizes the buffer)
template <class Key>
struct BlockSamples {
  Key* first;   // nullptr: not recorded
  Key* last;
  int64_t n;    // keys in the whole array
  int shift;    // log2 of the block size
};

// NSB_PASS_PL=1: the pass merge loop in producer/loser form over K-sentinel
// pads (one LDS per output, no clamps), as in the tile sort.
#ifndef NSB_PASS_PL
#define NSB_PASS_PL 1
#endif
// sentinel words after each staged slice of a K-output-per-thread merge
__host__ __device__ constexpr int v2_pad(int K) { return NSB_PASS_PL ? K : 1; }

template <int NT, int K, class Key>
__device__ __forceinline__ void merge_staged_tile(Key* sm, int a_pos, int la, int b_pos, int lb,
                                                  Key* dst, const int64_t* s_out_off,
                                                  BlockSamples<Key> bs = {nullptr, nullptr, 0, kSmpShift}) {
  constexpr int TM = NT * K;
  constexpr int PV = kpv<Key>();
  constexpr int KB = (int)sizeof(Key);
  const int tid = threadIdx.x;
  constexpr int PAD = v2_pad(K);
  for (int q = tid; q < PAD; q += NT) {
    sm[a_pos + la + q] = KeyT<Key>::kMax;  // sentinels: the merge loop has no bounds tests
    sm[b_pos + lb + q] = KeyT<Key>::kMax;
  }
  __syncthreads();

  const Key* SA = sm + a_pos;
  const Key* SB = sm + b_pos;
  const int total = la + lb;
  NSB_DCHECK(la >= 0 && lb >= 0 && total <= TM &&
             (a_pos + la + PAD <= b_pos || b_pos + lb + PAD <= a_pos));
  // full tiles (every tile but the last of a pair) give every thread exactly
  // K outputs: that path has no per-output guard at all
  const int d = min(tid * K, total);
  const int cnt = min(K, total - d);
  const int a = merge_path<int>(SA, la, SB, lb, d);
  const char* smc = reinterpret_cast<const char*>(sm);
  Key v[K];
#if NSB_PASS_PL
  // producer/loser form (see cta_sort_skewed_body): one LDS per output; a
  // cursor runs at most K keys into its slice's K sentinels
  uint32_t ptr = (uint32_t)(a_pos + a) * KB;
  uint32_t mnext = (uint32_t)(b_pos + d - a + 1) * KB;
  Key m = *reinterpret_cast<const Key*>(smc + mnext - KB);
  auto step = [&]() {
    NSB_DCHECK((ptr >= (uint32_t)a_pos * KB && ptr < (uint32_t)(a_pos + la + PAD) * KB) ||
               (ptr >= (uint32_t)b_pos * KB && ptr < (uint32_t)(b_pos + lb + PAD) * KB));
    const Key x = *reinterpret_cast<const Key*>(smc + ptr);
    const bool t = x <= m;
    const Key out = t ? x : m;
    const uint32_t q = ptr + (uint32_t)KB;
    ptr = t ? q : mnext;
    mnext = t ? mnext : q;
    m = t ? m : x;
    return out;
  };
#else
  // cursors are byte offsets into shared memory (LDS [reg + base] needs no
  // index arithmetic), clamped at their slice's +inf sentinel
  uint32_t oa = (uint32_t)(a_pos + a) * KB, ob = (uint32_t)(b_pos + d - a) * KB;
  const uint32_t ea = (uint32_t)(a_pos + la) * KB, eb = (uint32_t)(b_pos + lb) * KB;
  Key ka = *reinterpret_cast<const Key*>(smc + oa), kb = *reinterpret_cast<const Key*>(smc + ob);
  auto step = [&]() {
    const bool take_a = ka <= kb;  // A wins ties (merge_runs, hybrid.hpp:71-75)
    const Key out = take_a ? ka : kb;
    if (take_a) {
      oa = min(oa + (uint32_t)KB, ea);  // an exhausted side keeps re-reading its sentinel
      ka = *reinterpret_cast<const Key*>(smc + oa);
    } else {
      ob = min(ob + (uint32_t)KB, eb);
      kb = *reinterpret_cast<const Key*>(smc + ob);
    }
    return out;
  };
#endif
  const bool full = total == TM;
  if (full) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = step();
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (k < cnt) v[k] = step();
  }
  __syncthreads();  // every thread is done reading the staged inputs
  if (full) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[d + k] = v[k];
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (k < cnt) sm[d + k] = v[k];
  }

  Key* out = dst + *s_out_off;
  const bool o_tma = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && (total % PV) == 0;
  __syncthreads();
  if (bs.first) {  // tiles start on block boundaries (TM and 2R are multiples of the block)
    const int sh = bs.shift;
    const int nb = (total + (1 << sh) - 1) >> sh;
    const int64_t b0 = *s_out_off >> sh;
    for (int t = tid; t < nb; t += NT) {
      bs.first[b0 + t] = sm[t << sh];
      bs.last[b0 + t] = sm[min((t << sh) + (1 << sh) - 1, total - 1)];
    }
  }
  if (o_tma) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tma_store_1d(out, sm, (uint32_t)total * (uint32_t)KB);
      bulk_commit();
      bulk_wait_read_all();
    }
  } else {
    for (int i = tid; i < total; i += NT) out[i] = sm[i];
  }
}

// Partition with the previous pass's block samples.  For a pair of two FULL
// runs (the bulk of every pass) the split a for diagonal d (a multiple of
// 256) is bracketed on the samples first: the predicate
// A[mid] <= B[d-1-mid] at mid = 256j reads A's first[] and B's last[] of
// block (d/256 - j - 1), both L2-resident; then 8 steps on the keys finish
// inside one 256-key block.  Other pairs (the array's short last pair) use
// the plain search.  Same result as merge_path, fewer DRAM round trips.
template <class Key>
__global__ void merge_partition_v3_kernel(const Key* __restrict__ src, PassPlan P,
                                          int64_t num_tiles, int64_t* __restrict__ mp,
                                          BlockSamples<Key> bs) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  pdl_trigger();
  if (c >= num_tiles) return;
  const TileGeom g = tile_geom(P, c);
  const Key* A = src + g.pair_base;
  const Key* B = A + g.a_len;
  const int64_t diag = g.diag0;
  const int sh = bs.shift;
  const int64_t bm = (int64_t(1) << sh) - 1;
  if (g.a_len != P.R || g.b_len != P.R || (diag & bm) != 0) {
    mp[c] = merge_path<int64_t>(A, g.a_len, B, g.b_len, diag);
    return;
  }
  const int64_t R = P.R;
  int64_t lo = diag > R ? diag - R : 0;
  int64_t hi = diag < R ? diag : R;
  // coarse over block starts mid = j*blk in [lo, hi): find the first j where
  // P(mid) = A[mid] <= B[diag - 1 - mid] fails; B's element is the LAST key
  // of block (diag/blk - j - 1) because diag is a block multiple
  const int64_t abase = g.pair_base >> sh, bbase = (g.pair_base + R) >> sh;
  const int64_t dblk = diag >> sh;
  int64_t jl = (lo + bm) >> sh, jh = (hi + bm) >> sh;  // candidates j in [jl, jh)
  while (jl < jh) {
    const int64_t jm = (jl + jh) >> 1;
    const bool p = (jm << sh) < hi && bs.first[abase + jm] <= bs.last[bbase + dblk - jm - 1];
    if (p) jl = jm + 1;
    else jh = jm;
  }
  // P holds at block starts j < jl and fails from jl: a in (blk(jl-1), blk*jl]
  int64_t flo = jl > 0 ? max(lo, ((jl - 1) << sh) + 1) : lo;
  int64_t fhi = min(hi, jl << sh);
  if (flo > fhi) flo = fhi;
  while (flo < fhi) {
    const int64_t mid = (flo + fhi) >> 1;
    if (A[mid] <= B[diag - 1 - mid]) flo = mid + 1;
    else fhi = mid;
  }
  mp[c] = flo;
}

// First index in [lo, hi) where a monotone (true ... true false ... false)
// predicate fails, found by the whole warp with 32-ary rounds: each round
// every lane evaluates one of 32 evenly spaced candidates and a ballot
// narrows the range 32x.  All lanes return the result.
template <class F>
__device__ __forceinline__ int64_t warp_first_false(int64_t lo, int64_t hi, F pred) {
  const int lane = threadIdx.x & 31;
  while (lo < hi) {
    const int64_t span = hi - lo;
    const int64_t step = span <= 32 ? 1 : (span + 31) / 32;
    const int64_t i = lo + lane * step;
    const unsigned m = __ballot_sync(0xffffffffu, i < hi && pred(i));
    const int c = __popc(m);
    if (step == 1) return lo + c;
    const int64_t nlo = c == 0 ? lo : lo + (int64_t)(c - 1) * step + 1;
    hi = min(hi, lo + (int64_t)c * step);
    lo = nlo;
  }
  return lo;
}

// Partition v4: one WARP per tile, the search of v3 (or of v2 without block
// samples) in 32-ary rounds: about 7 dependent L2/HBM round trips instead of
// ~29 serial probes.  It moves 32x the probe sectors, so it only pays where
// the partition is latency-bound — passes of few tiles (measured: 2^30 keys,
// 135 K tiles, 2x slower than v3; 2^24 keys, 2 K tiles, see the host policy).
template <class Key>
__global__ void merge_partition_v4_kernel(const Key* __restrict__ src, PassPlan P,
                                          int64_t num_tiles, int64_t* __restrict__ mp,
                                          BlockSamples<Key> bs) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  pdl_wait();
  pdl_trigger();
  if (c >= num_tiles) return;  // whole warps exit together
  const TileGeom g = tile_geom(P, c);
  const Key* A = src + g.pair_base;
  const Key* B = A + g.a_len;
  const int64_t diag = g.diag0;
  const int sh = bs.shift;
  const int64_t bm = (int64_t(1) << sh) - 1;
  const int64_t R = P.R;
  int64_t flo = diag > g.b_len ? diag - g.b_len : 0;
  int64_t fhi = diag < g.a_len ? diag : g.a_len;
  if (bs.first && g.a_len == R && g.b_len == R && (diag & bm) == 0) {
    // coarse: first block start j*blk where A[j*blk] <= B[diag-1-j*blk]
    // fails; B's key there is the LAST key of block (diag/blk - j - 1)
    const int64_t lo = flo, hi = fhi;
    const int64_t abase = g.pair_base >> sh, bbase = (g.pair_base + R) >> sh;
    const int64_t dblk = diag >> sh;
    const Key* first = bs.first;
    const Key* last = bs.last;
    const int64_t jl = warp_first_false((lo + bm) >> sh, (hi + bm) >> sh, [&](int64_t j) {
      return (j << sh) < hi && first[abase + j] <= last[bbase + dblk - j - 1];
    });
    flo = jl > 0 ? max(lo, ((jl - 1) << sh) + 1) : lo;
    fhi = min(hi, jl << sh);
    if (flo > fhi) flo = fhi;
  }
  const int64_t a = warp_first_false(flo, fhi, [&](int64_t m) { return A[m] <= B[diag - 1 - m]; });
  if ((threadIdx.x & 31) == 0) mp[c] = a;
}

// Keys of shared memory a v2 tile needs: two slices with up to 3 keys of
// alignment slack each, a sentinel after each, 16-byte rounding.
__host__ __device__ constexpr int v2_smem_words(int TM, int K = 0) { return TM + 16 + 2 * v2_pad(K); }

// Resident CTAs per SM the launch bounds ask for: as many as shared memory
// (228 KiB per SM, 1 KiB reserved per CTA), the 2048-thread limit and a
// register floor allow.  <256,29> / <256,31>: 6 CTAs/SM at 40 registers (measured
// best; 7 CTAs force 32 registers and spill).
#ifndef NSB_V2_REGS
#define NSB_V2_REGS 40  // register budget per thread assumed for int32 tiles of <= 31 keys
#endif
__host__ __device__ constexpr int v2_min_blocks(int NT, int K, int key_bytes) {
  const int smem = v2_smem_words(NT * K, K) * key_bytes + 1024;
  int b = 228 * 1024 / smem;
  if (b > 2048 / NT) b = 2048 / NT;
  // the K outputs stay in registers until the store (2 registers per int64)
  const int regs = key_bytes == 8 ? 2 * K + 17 : (K <= 31 ? NSB_V2_REGS : K + 17);
  if (b > 65536 / (NT * regs)) b = 65536 / (NT * regs);
  if (b > 32) b = 32;
  return b < 1 ? 1 : b;
}

// Stage + merge + store of one tile of a pairwise pass whose merge-path
// splits (a0 at diag0, a1 at diag1) are known: both input slices go to shared
// memory by bulk copy (TMA 1D, completion on *bar at `parity`), the merge is
// merge_staged_tile's.  `init_bar`: the caller has not initialised *bar
// (the one-tile kernel does it here; the persistent flow kernel once).
template <int NT, int K, class Key>
__device__ __forceinline__ void merge_tile_v2(const Key* __restrict__ src, Key* __restrict__ dst,
                                              const PassPlan& P, const TileGeom& g, int64_t a0,
                                              int64_t a1, BlockSamples<Key> bs, Key* sm,
                                              uint64_t* bar, uint32_t parity, bool init_bar) {
  constexpr int TM = NT * K;
  constexpr int PV = kpv<Key>();
  constexpr int KB = (int)sizeof(Key);
  const int tid = threadIdx.x;
  const int la = (int)(a1 - a0);
  const int lb = (int)((g.diag1 - a1) - (g.diag0 - a0));
  // the splits lie on the pair's merge path and the slices fit the tile
  NSB_DCHECK(a0 >= 0 && a0 <= a1 && a1 <= g.a_len && g.diag0 - a0 >= 0 && g.diag1 - a1 <= g.b_len &&
             lb >= 0 && la + lb == (int)(g.diag1 - g.diag0) && la + lb <= TM);
  const Key* A = src + g.pair_base + a0;
  const Key* B = src + g.pair_base + g.a_len + (g.diag0 - a0);
  const Key* lo = src;
  const Key* hi = src + P.n;

  // smem placement mirrors global 16-byte alignment so one bulk copy per slice
  const uintptr_t a_addr = reinterpret_cast<uintptr_t>(A), b_addr = reinterpret_cast<uintptr_t>(B);
  const int a_shift = (int)((a_addr & 15) / KB), b_shift = (int)((b_addr & 15) / KB);
  const int b_off = (a_shift + la + v2_pad(K) + PV - 1) & ~(PV - 1);  // B cover starts 16-byte aligned
  const Key* a_cov = A - a_shift;
  const Key* b_cov = B - b_shift;
  const int a_words = (a_shift + la + PV - 1) & ~(PV - 1), b_words = (b_shift + lb + PV - 1) & ~(PV - 1);
  const bool a_tma = la > 0 && (a_addr % KB) == 0 && a_cov >= lo && a_cov + a_words <= hi;
  const bool b_tma = lb > 0 && (b_addr % KB) == 0 && b_cov >= lo && b_cov + b_words <= hi;
  NSB_DCHECK(b_off + b_words + v2_pad(K) <= v2_smem_words(TM, K) && a_shift + la + v2_pad(K) <= b_off);

  // the output offset crosses the merge loop through shared memory, so no
  // 64-bit geometry stays live in registers next to the K outputs
  __shared__ int64_t s_out;
  if (tid == 0) {
    if (init_bar) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
    s_out = g.pair_base + g.diag0;
  }
  __syncthreads();
  if (tid == 0) {
    fence_proxy_async_smem();  // earlier generic accesses of sm before the bulk writes
    const uint32_t bytes = (a_tma ? a_words * (uint32_t)KB : 0u) + (b_tma ? b_words * (uint32_t)KB : 0u);
    mbar_arrive_expect_tx(bar, bytes);
    if (a_tma) tma_load_1d(sm, a_cov, a_words * (uint32_t)KB, bar);
    if (b_tma) tma_load_1d(sm + b_off, b_cov, b_words * (uint32_t)KB, bar);
  }
  if (!a_tma)
    for (int i = tid; i < la; i += NT) sm[a_shift + i] = __ldcs(A + i);
  if (!b_tma)
    for (int i = tid; i < lb; i += NT) sm[b_off + b_shift + i] = __ldcs(B + i);
  mbar_wait(bar, parity);
  __syncthreads();
  merge_staged_tile<NT, K>(sm, a_shift, la, b_off + b_shift, lb, dst, &s_out, bs);
}

template <int NT, int K, bool FUSED = false, class Key = int32_t>
__global__ void __launch_bounds__(NT, v2_min_blocks(NT, K, (int)sizeof(Key)))
    merge_pass_v2_kernel(const Key* __restrict__ src, Key* __restrict__ dst, PassPlan P,
                         const int64_t* __restrict__ mp, BlockSamples<Key> bs) {
  constexpr int TM = NT * K;
  static_assert(TM % 4 == 0, "tiles must start 16-byte aligned");
  __shared__ __align__(128) Key sm[v2_smem_words(TM, K)];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  const TileGeom g = tile_geom(P, c);
  pdl_wait();  // src / mp come from the previous kernels
  pdl_trigger();
  if (g.diag0 >= g.diag1) return;  // empty trailing tile of a short last pair
  const bool last_in_pair = g.diag1 == g.a_len + g.b_len;
  int64_t a0, a1;
  if constexpr (FUSED) {
    // splits found here by warps 0 and 1 instead of a partition kernel
    __shared__ int64_t splits[2];
    const int warp = tid >> 5;
    const Key* PA = src + g.pair_base;
    if (warp == 0) {
      const int64_t v = warp_merge_path(PA, g.a_len, PA + g.a_len, g.b_len, g.diag0);
      if (tid == 0) splits[0] = v;
    } else if (warp == 1) {
      const int64_t v = last_in_pair
                            ? g.a_len
                            : warp_merge_path(PA, g.a_len, PA + g.a_len, g.b_len, g.diag1);
      if (tid == 32) splits[1] = v;
    }
    __syncthreads();
    a0 = splits[0];
    a1 = splits[1];
  } else {
    a0 = mp[c];
    a1 = last_in_pair ? g.a_len : mp[c + 1];
  }
  merge_tile_v2<NT, K>(src, dst, P, g, a0, a1, bs, sm, &bar, 0u, true);
}


}  // namespace nsb
