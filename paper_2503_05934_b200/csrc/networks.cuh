// networks.cuh — register-resident sorting networks (widths 2..8) and the
// config-shaped per-thread base case.
//
// Replaces the reference's base-case layer:
//   compare_exchange  /root/reference/proj/include/netsort/networks.hpp:25-32
//   sort_exact<W>     networks.hpp:122-128
//   sort_small        networks.hpp:132-145
//   try_base_case     /root/reference/proj/include/netsort/hybrid.hpp:48-56
//
// Every comparator is a pair of IMNMX on registers; all indices are
// compile-time constants, so a network never touches local memory.  The
// comparator tables are optimal-size (1,3,5,9,12,16,19) and are exported
// through ns_network_comparators() so the CPU tests can verify them with the
// zero-one principle without a GPU.
#pragma once
#include <cstdint>
#include <utility>

namespace nsb {

#define NSB_HD __host__ __device__ __forceinline__

template <class T>
NSB_HD void cx(T& a, T& b) {
  const T lo = a < b ? a : b;
  const T hi = a < b ? b : a;
  a = lo;
  b = hi;
}

struct Pair {
  uint8_t lo, hi;
};

// Comparator tables (lo, hi) for widths 2..8.
template <int W>
struct Net;
template <> struct Net<2> { static constexpr int N = 1;  static constexpr Pair P[N] = {{0, 1}}; };
template <> struct Net<3> { static constexpr int N = 3;  static constexpr Pair P[N] = {{1, 2}, {0, 2}, {0, 1}}; };
template <> struct Net<4> { static constexpr int N = 5;  static constexpr Pair P[N] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {1, 2}}; };
template <> struct Net<5> { static constexpr int N = 9;  static constexpr Pair P[N] = {{0, 1}, {3, 4}, {2, 4}, {2, 3}, {0, 3}, {0, 2}, {1, 4}, {1, 3}, {1, 2}}; };
template <> struct Net<6> { static constexpr int N = 12; static constexpr Pair P[N] = {{1, 2}, {4, 5}, {0, 2}, {3, 5}, {0, 1}, {3, 4}, {2, 5}, {0, 3}, {1, 4}, {2, 4}, {1, 3}, {2, 3}}; };
template <> struct Net<7> { static constexpr int N = 16; static constexpr Pair P[N] = {{1, 2}, {3, 4}, {5, 6}, {0, 2}, {3, 5}, {4, 6}, {0, 1}, {4, 5}, {2, 6}, {0, 4}, {1, 5}, {0, 3}, {2, 5}, {1, 3}, {2, 4}, {2, 3}}; };
template <> struct Net<8> { static constexpr int N = 19; static constexpr Pair P[N] = {{0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}, {0, 1}, {2, 3}, {4, 5}, {6, 7}, {2, 4}, {3, 5}, {1, 4}, {3, 6}, {1, 2}, {3, 4}, {5, 6}}; };

// sort_exact<W> equivalent: width-W network on v[OFF .. OFF+W).
// Comparator I of the width-W network on the window at OFF.  The indices are
// constant expressions, so the table never exists in device memory.
template <int W, int OFF, int I, class T, int K>
NSB_HD void net_step(T (&v)[K]) {
  constexpr int lo = OFF + Net<W>::P[I].lo;
  constexpr int hi = OFF + Net<W>::P[I].hi;
  cx(v[lo], v[hi]);
}

template <int W, int OFF, class T, int K, int... I>
NSB_HD void sort_net_seq(T (&v)[K], std::integer_sequence<int, I...>) {
  (net_step<W, OFF, I>(v), ...);
}

template <int W, int OFF = 0, class T, int K>
NSB_HD void sort_net(T (&v)[K]) {
  static_assert(W >= 2 && W <= 8 && OFF + W <= K, "bad network window");
  sort_net_seq<W, OFF>(v, std::make_integer_sequence<int, Net<W>::N>{});
}

// Merge two sorted adjacent runs v[OFF..OFF+H) and v[OFF+H..OFF+2H) held in
// registers (flip step + half-cleaners; H a power of two).
template <int H, int OFF = 0, class T, int K>
NSB_HD void reg_merge(T (&v)[K]) {
#pragma unroll
  for (int i = 0; i < H; ++i) cx(v[OFF + i], v[OFF + 2 * H - 1 - i]);
#pragma unroll
  for (int s = H / 2; s >= 1; s >>= 1) {
#pragma unroll
    for (int i = 0; i < 2 * H; ++i)
      if ((i & s) == 0) cx(v[OFF + i], v[OFF + i + s]);
  }
}

// Host/device mirror of base_case_applies (config.hpp:30-36).
NSB_HD constexpr bool base_case_applies(int size, uint32_t mask, int varsort_max) {
  return (size >= 2 && size <= 8 && ((mask >> size) & 1u)) ||
         (varsort_max != 0 && size >= 2 && size <= varsort_max);
}

// Leaf shape of the reference recursion (merge_sort_rec, hybrid.hpp:81-95)
// applied to an 8-key window: the largest power-of-two size the config sends
// to a network (8, 4 or 2), or 1 when the recursion bottoms out at single
// elements (Classic, Odd, "3").  The GPU per-thread base case follows exactly
// this shape: LEAF-wide networks, then in-register merges up to 8.
NSB_HD constexpr int leaf_of(uint32_t mask, int varsort_max) {
  return base_case_applies(8, mask, varsort_max)   ? 8
         : base_case_applies(4, mask, varsort_max) ? 4
         : base_case_applies(2, mask, varsort_max) ? 2
                                                   : 1;
}

// Applies the width-W network to every W-aligned window of v.
template <int W, int OFF, class T, int K>
NSB_HD void windows(T (&v)[K]) {
  if constexpr (OFF + W <= K) {
    sort_net<W, OFF>(v);
    windows<W, OFF + W>(v);
  }
}

// Batcher's odd-even merge of the two sorted halves of v[LO..HI] (HI
// inclusive; R is the recursion's comparator distance, 1 at the top): 9, 25
// and 65 comparators for 2 x 4, 2 x 8 and 2 x 16 keys, against 12, 32 and 80
// for a bitonic flip + half-cleaner merge.
template <int LO, int HI, int R, class T, int K>
NSB_HD void oe_merge(T (&v)[K]) {
  constexpr int STEP = 2 * R;
  if constexpr (STEP < HI - LO) {
    oe_merge<LO, HI, STEP>(v);
    oe_merge<LO + R, HI, STEP>(v);
#pragma unroll
    for (int i = LO + R; i < HI - R; i += STEP) cx(v[i], v[i + R]);
  } else {
    cx(v[LO], v[LO + R]);
  }
}

// Merges sorted runs of H keys pairwise up to one sorted run of K.
template <int H, class T, int K, int... B>
NSB_HD void merge_level(T (&v)[K], std::integer_sequence<int, B...>) {
  (oe_merge<B * 2 * H, B * 2 * H + 2 * H - 1, 1>(v), ...);
}
template <int H, int K, class T>
NSB_HD void thread_merges(T (&v)[K]) {
  if constexpr (H < K) {
    merge_level<H>(v, std::make_integer_sequence<int, K / (2 * H)>{});
    thread_merges<2 * H, K>(v);
  }
}

// Per-thread sort of K (power of two, >= 8) register-resident keys: each
// 8-key window is sorted by the config-shaped base case, then the windows are
// merged in registers.
template <int LEAF, int K, class T>
NSB_HD void thread_sort(T (&v)[K]) {
  static_assert(K >= 8 && (K & (K - 1)) == 0, "K must be a power of two >= 8");
  if constexpr (LEAF == 8 || LEAF == 4) windows<LEAF, 0>(v);
  if constexpr (LEAF == 2) {
#pragma unroll
    for (int i = 0; i < K; i += 2) cx(v[i], v[i + 1]);
  }
  // merges from LEAF up to K (LEAF==1 starts from single elements)
  thread_merges<(LEAF < 1 ? 1 : LEAF), K>(v);
  static_assert(K <= 32, "thread_sort supports up to 32 keys per thread");
}

// The width-L network (sort_exact<L>, networks.hpp:122-128) on L keys in
// memory: L loads, the network in registers, L stores.
template <int L, class T>
__device__ __forceinline__ void sort_in_place(T* p) {
  T v[L];
#pragma unroll
  for (int k = 0; k < L; ++k) v[k] = p[k];
  sort_net<L>(v);
#pragma unroll
  for (int k = 0; k < L; ++k) p[k] = v[k];
}

// Runtime-width network for one ragged array of `len` keys at p (the
// reference's sort_small switch, networks.hpp:132-145; lengths 0 and 1 are
// no-ops).  Exactly `len` loads and stores.
template <class T>
__device__ __forceinline__ void sort_small_in_place(T* p, int len) {
  switch (len) {
    case 2: sort_in_place<2>(p); break;
    case 3: sort_in_place<3>(p); break;
    case 4: sort_in_place<4>(p); break;
    case 5: sort_in_place<5>(p); break;
    case 6: sort_in_place<6>(p); break;
    case 7: sort_in_place<7>(p); break;
    case 8: sort_in_place<8>(p); break;
    default: break;
  }
}

}  // namespace nsb
