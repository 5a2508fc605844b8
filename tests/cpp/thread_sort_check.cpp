// Host-compiled check of the per-thread base case in networks.cuh (built by
// tests/test_library.py with g++; the __host__/__device__ qualifiers are
// defined away).  thread_sort<LEAF, K> is exhaustive under the zero-one
// principle for K <= 16; for K = 32 every odd-even merge it is built from
// is checked on all zero-one inputs with sorted halves, and thread_sort on
// random permutations.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <random>

#include "networks.cuh"

using namespace nsb;

template <int LEAF, int K>
static bool exhaustive() {
  for (unsigned long bits = 0; bits < (1ul << K); ++bits) {
    int v[K];
    for (int i = 0; i < K; ++i) v[i] = (bits >> i) & 1;
    thread_sort<LEAF>(v);
    if (!std::is_sorted(v, v + K)) return false;
  }
  return true;
}

template <int H>
static bool merge_zero_one() {
  for (int a = 0; a <= H; ++a)
    for (int b = 0; b <= H; ++b) {
      int v[2 * H];
      for (int i = 0; i < H; ++i) v[i] = i >= H - a;
      for (int i = 0; i < H; ++i) v[H + i] = i >= H - b;
      oe_merge<0, 2 * H - 1, 1>(v);
      if (!std::is_sorted(v, v + 2 * H)) return false;
    }
  return true;
}

template <int LEAF, int K>
static bool random_perms(int reps) {
  std::mt19937 rng(LEAF * 131 + K);
  for (int r = 0; r < reps; ++r) {
    int v[K];
    for (int i = 0; i < K; ++i) v[i] = (int)(rng() % 7) - 3 + i * (r & 1);
    std::shuffle(v, v + K, rng);
    thread_sort<LEAF>(v);
    if (!std::is_sorted(v, v + K)) return false;
  }
  return true;
}

int main() {
  bool ok = true;
  ok &= merge_zero_one<1>() && merge_zero_one<2>() && merge_zero_one<4>() &&
        merge_zero_one<8>() && merge_zero_one<16>();
  ok &= exhaustive<1, 8>() && exhaustive<2, 8>() && exhaustive<4, 8>() && exhaustive<8, 8>();
  ok &= exhaustive<1, 16>() && exhaustive<2, 16>() && exhaustive<4, 16>() && exhaustive<8, 16>();
  ok &= random_perms<1, 32>(20000) && random_perms<2, 32>(20000) && random_perms<4, 32>(20000) &&
        random_perms<8, 32>(20000);
  std::printf(ok ? "thread_sort ok\n" : "thread_sort FAILED\n");
  return ok ? 0 : 1;
}
