// datagen.cpp — host-side seeded inputs.
//
// The reference generates int64 inputs only (generate, src/datagen.cpp:18-50,
// SplitMix64 at include/netsort/datagen.hpp:29-42).  The BASELINE configs are
// int32, narrowed as SURVEY.md §8(d) fixes it: random = int32(next() >> 33),
// i.e. U[0, 2^31); sorted = 0..n-1; nearly sorted = the ramp after
// floor(p*n) seeded index-pair swaps (at least one when p > 0), exactly the
// reference's swap rule.  The ragged base-case batch (BASELINE config 2) draws
// lengths 3 + next() % 6 from stream `seed` and keys from stream
// seed ^ 0x5bd1e995.  These are the inputs bench.py and the tests feed the
// device path; ns_generate_i32 (prof.cu) produces kinds 0/1 on the device.
#include <cstddef>
#include <cstdint>
#include <utility>

#include "../../include/netsort_b200.h"

namespace {

struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

template <class T, class R>
int generate(T* out, size_t n, int kind, uint64_t seed, double p, R rnd) {
  if (n && !out) return NS_ERR_INVALID;
  if (kind < 0 || kind > 2) return NS_ERR_INVALID;
  if (kind == 2 && !(p >= 0.0 && p <= 1.0)) return NS_ERR_INVALID;
  if (kind == 0) {
    SplitMix64 g{seed};
    for (size_t i = 0; i < n; ++i) out[i] = rnd(g.next());
    return NS_OK;
  }
  for (size_t i = 0; i < n; ++i) out[i] = static_cast<T>(i);
  if (kind == 2) {
    size_t swaps = static_cast<size_t>(p * static_cast<double>(n));
    if (swaps == 0 && n >= 2 && p > 0.0) swaps = 1;
    SplitMix64 g{seed};
    for (size_t k = 0; k < swaps; ++k) {
      const size_t i = g.next() % n;
      const size_t j = g.next() % n;
      std::swap(out[i], out[j]);
    }
  }
  return NS_OK;
}

}  // namespace

extern "C" {

int ns_generate_host_i32(int32_t* h_out, size_t n, int kind, uint64_t seed, double p) {
  return generate(h_out, n, kind, seed, p, [](uint64_t r) { return static_cast<int32_t>(r >> 33); });
}

int ns_generate_host_i64(int64_t* h_out, size_t n, int kind, uint64_t seed, double p) {
  return generate(h_out, n, kind, seed, p, [](uint64_t r) { return static_cast<int64_t>(r); });
}

size_t ns_generate_batch_host_i32(size_t num_arrays, uint64_t seed, uint32_t* h_offsets,
                                  int32_t* h_keys) {
  SplitMix64 ls{seed};
  size_t total = 0;
  for (size_t a = 0; a < num_arrays; ++a) {
    if (h_offsets) h_offsets[a] = static_cast<uint32_t>(total);
    total += 3 + static_cast<size_t>(ls.next() % 6);
  }
  if (h_offsets) h_offsets[num_arrays] = static_cast<uint32_t>(total);
  if (h_keys) {
    SplitMix64 ks{seed ^ 0x5bd1e995ull};
    for (size_t i = 0; i < total; ++i) h_keys[i] = static_cast<int32_t>(ks.next() >> 33);
  }
  return total;
}

}  // extern "C"
