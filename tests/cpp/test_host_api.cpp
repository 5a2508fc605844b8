// C++ host-API test: the reference's own call shapes (hybrid.hpp / config.hpp)
// against netsort_b200.hpp, mirroring the predicates of the reference's
// tests/test_hybrid.cpp (restated, not copied).  Exit status = #failures.
//   argv[1] == "--no-gpu": only the host-side checks (registry, configs).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

#include "netsort_b200.hpp"

namespace ns = netsort_b200;

static int failures = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

static std::vector<int32_t> random_values(size_t n, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<int32_t> v(n);
  for (auto& x : v) x = static_cast<int32_t>(rng() >> 33);
  return v;
}

static void host_side() {
  // test_hybrid.cpp:48-100 restated: registry, names, width sets
  const auto& reg = ns::config_registry();
  CHECK(reg.size() == 12);
  CHECK(reg.front().name == "Classic" && reg.front().is_classic());
  CHECK(ns::find_config("9To12") == nullptr);
  CHECK(ns::find_config("classic") == nullptr);
  CHECK(ns::bundled_variants().size() == 24);
  CHECK(ns::base_case_applies(7, *ns::find_config("6To8")));
  CHECK(!ns::base_case_applies(5, *ns::find_config("6To8")));
  CHECK(ns::base_case_applies(2, *ns::find_config("VarSort5")));
  CHECK(!ns::base_case_applies(6, *ns::find_config("VarSort5")));
  CHECK(ns::base_case_applies(8, *ns::find_config("PowerOf2")));
  CHECK(!ns::base_case_applies(2, *ns::find_config("3")));
  for (int s = 0; s <= 10; ++s) CHECK(!ns::base_case_applies(s, ns::classic_config()));
  bool threw = false;
  try {
    ns::make_fixed_config("bad", {2});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    ns::make_varsort_config("bad", 6);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  // C ABI agrees with the C++ registry
  for (const auto& c : reg) {
    uint32_t m = 0;
    int v = 0;
    CHECK(ns_find_config(c.name.c_str(), &m, &v) == NS_OK);
    CHECK(m == c.width_mask && v == c.varsort_max);
  }
}

static void device_side() {
  // every variant on random arrays (test_hybrid.cpp:306-318)
  for (size_t n : {0u, 1u, 2u, 3u, 4u, 7u, 16u, 33u, 64u, 501u, 1000u, 20000u, 300000u}) {
    const auto input = random_values(n, 3000 + n);
    auto expect = input;
    std::sort(expect.begin(), expect.end());
    for (const auto& var : ns::bundled_variants()) {
      auto v = input;
      ns::run_variant(var, std::span<int32_t>(v));
      CHECK(v == expect);
    }
  }
  // classical sorts (test_hybrid.cpp:102-117)
  for (size_t n : {0u, 1u, 2u, 3u, 5u, 17u, 64u, 1000u, 10000u}) {
    auto m = random_values(n, 1000 + n), q = m, e = m;
    std::sort(e.begin(), e.end());
    ns::classical_merge_sort(std::span<int32_t>(m));
    ns::classical_quick_sort(std::span<int32_t>(q));
    CHECK(m == e && q == e);
  }
  // ternary arrays up to length 6 through all 24 variants (test_hybrid.cpp:283-304)
  for (int len = 0; len <= 6; ++len) {
    int total = 1;
    for (int i = 0; i < len; ++i) total *= 3;
    for (int code = 0; code < total; ++code) {
      std::vector<int32_t> base(static_cast<size_t>(len));
      int rest = code;
      for (int i = 0; i < len; ++i) {
        base[static_cast<size_t>(i)] = rest % 3;
        rest /= 3;
      }
      auto expect = base;
      std::sort(expect.begin(), expect.end());
      for (const auto& var : {ns::SortVariant{ns::Algorithm::merge_sort, *ns::find_config("6To8")},
                              ns::SortVariant{ns::Algorithm::quick_sort, *ns::find_config("3To5")}}) {
        auto v = base;
        ns::run_variant(var, std::span<int32_t>(v));
        CHECK(v == expect);
      }
    }
  }
  // range sorts leave the outside untouched; inverted ranges are no-ops
  // (test_hybrid.cpp:320-354)
  auto base = random_values(40, 17);
  for (auto& x : base) x %= 100;
  std::vector<int32_t> window(base.begin() + 10, base.begin() + 30);
  std::sort(window.begin(), window.end());
  for (const char* name : {"Classic", "3To8", "VarSort4"}) {
    const auto& cfg = *ns::find_config(name);
    auto m = base, q = base;
    ns::optimized_merge_sort(std::span<int32_t>(m), 10, 29, cfg);
    ns::optimized_quick_sort(std::span<int32_t>(q), 10, 29, cfg);
    for (int k = 0; k < 40; ++k) {
      if (k >= 10 && k < 30) continue;
      CHECK(m[static_cast<size_t>(k)] == base[static_cast<size_t>(k)]);
      CHECK(q[static_cast<size_t>(k)] == base[static_cast<size_t>(k)]);
    }
    CHECK(std::equal(window.begin(), window.end(), m.begin() + 10));
    CHECK(std::equal(window.begin(), window.end(), q.begin() + 10));
  }
  std::vector<int32_t> v{3, 1, 2};
  ns::optimized_merge_sort(std::span<int32_t>(v), 2, 1, *ns::find_config("3To8"));
  ns::optimized_quick_sort(std::span<int32_t>(v), 2, 1, *ns::find_config("3To8"));
  CHECK((v == std::vector<int32_t>{3, 1, 2}));
  // device spans with caller scratch
  ns::DeviceScratch scratch;
  const auto big = random_values(1 << 20, 5);
  int32_t* d = nullptr;
  CHECK(cudaMalloc(&d, big.size() * 4) == cudaSuccess);
  cudaMemcpy(d, big.data(), big.size() * 4, cudaMemcpyHostToDevice);
  ns::device_merge_sort(d, big.size(), *ns::find_config("6To8"), scratch);
  std::vector<int32_t> back(big.size());
  cudaMemcpy(back.data(), d, big.size() * 4, cudaMemcpyDeviceToHost);
  auto e = big;
  std::sort(e.begin(), e.end());
  CHECK(back == e);
  cudaMemcpy(d, big.data(), big.size() * 4, cudaMemcpyHostToDevice);
  ns::device_quick_sort(d, big.size(), *ns::find_config("3To5"), scratch);
  cudaMemcpy(back.data(), d, big.size() * 4, cudaMemcpyDeviceToHost);
  CHECK(back == e);
  cudaFree(d);

  // DispatchStats overloads (hybrid.hpp:158-165, 234-243) and merge (186-193)
  {
    auto v = random_values(100000, 77);
    ns::DispatchStats st;
    ns::run_variant(ns::SortVariant{ns::Algorithm::merge_sort, *ns::find_config("6To8")},
                    std::span<int32_t>(v), st);
    CHECK(std::is_sorted(v.begin(), v.end()));
    CHECK(st.merges == 16383 && st.network_hits[6] == 14688 && st.network_hits[7] == 1696);
    CHECK(st.max_depth == 15);  // SURVEY.md A.2 (100,000 keys, 6To8)
    // quick sort with stats: the reference recursion traced on the GPU; the
    // depth bound on sorted input (test_hybrid.cpp:271-281)
    std::vector<int32_t> sorted_in(10000);
    std::iota(sorted_in.begin(), sorted_in.end(), 0);
    for (const char* name : {"Classic", "3To5"}) {
      ns::DispatchStats qs;
      auto q = sorted_in;
      ns::run_variant(ns::SortVariant{ns::Algorithm::quick_sort, *ns::find_config(name)},
                      std::span<int32_t>(q), qs);
      CHECK(q == sorted_in);
      CHECK(qs.partitions > 0 && qs.merges == 0);
      CHECK(qs.max_depth >= 1 && qs.max_depth <= 4 * 13.3 + 16);
    }
    // hoare_partition / median_of_three contract (test_hybrid.cpp:204-269)
    for (int t = 0; t < 50; ++t) {
      auto b = random_values(64, 300 + t);
      for (auto& x : b) x %= 5;
      auto u = b;
      const int32_t p = ns::median_of_three(std::span<int32_t>(u), 3, 60);
      CHECK(u[3] <= p && p <= u[60] && u[31] == p);
      const auto j = ns::hoare_partition(std::span<int32_t>(u), 3, 60, p);
      CHECK(j >= 3 && j < 60);
      for (std::ptrdiff_t k = 3; k <= j; ++k) CHECK(u[static_cast<size_t>(k)] <= p);
      for (std::ptrdiff_t k = j + 1; k <= 60; ++k) CHECK(u[static_cast<size_t>(k)] >= p);
    }
    auto m = random_values(5000, 78);
    std::sort(m.begin(), m.begin() + 2000);
    std::sort(m.begin() + 2000, m.end());
    auto em = m;
    std::sort(em.begin(), em.end());
    ns::merge(std::span<int32_t>(m), 0, 1999, 4999);
    CHECK(m == em);
  }

  // int64: the reference's benchmark type, bound exactly as measure_loop's
  // sort_fn (std::function<void(std::span<std::int64_t>)>, bench.hpp:58-61;
  // bench.cpp:94-96 binds it to run_variant)
  std::mt19937_64 rng64(99);
  for (size_t n : {0u, 1u, 5u, 8u, 100u, 4097u, 70000u, 300000u}) {
    std::vector<int64_t> in(n);
    for (auto& x : in) x = static_cast<int64_t>(rng64());  // full 64-bit range, as datagen.cpp:27-29
    auto expect = in;
    std::sort(expect.begin(), expect.end());
    for (const auto& var : ns::bundled_variants()) {
      auto v = in;
      std::function<void(std::span<std::int64_t>)> sort_fn =
          [&var](std::span<std::int64_t> s) { ns::run_variant(var, s); };
      sort_fn(std::span<int64_t>(v));
      CHECK(v == expect);
    }
  }
  {
    const size_t n = size_t(1) << 21;
    std::vector<int64_t> h(n);
    for (auto& x : h) x = static_cast<int64_t>(rng64());
    auto e64 = h;
    std::sort(e64.begin(), e64.end());
    int64_t* d64 = nullptr;
    CHECK(cudaMalloc(&d64, n * 8) == cudaSuccess);
    std::vector<int64_t> back64(n);
    cudaMemcpy(d64, h.data(), n * 8, cudaMemcpyHostToDevice);
    ns::device_merge_sort(d64, n, *ns::find_config("6To8"), scratch);
    cudaMemcpy(back64.data(), d64, n * 8, cudaMemcpyDeviceToHost);
    CHECK(back64 == e64);
    cudaMemcpy(d64, h.data(), n * 8, cudaMemcpyHostToDevice);
    ns::device_quick_sort(d64, n, *ns::find_config("3To5"), scratch);
    cudaMemcpy(back64.data(), d64, n * 8, cudaMemcpyDeviceToHost);
    CHECK(back64 == e64);
    cudaFree(d64);
  }

  // several GPUs behind one host thread (BASELINE config 5's shape): the NCCL
  // exchange on the devices present, the peer-memory exchange with several
  // virtual ranks on device 0 (both checked against std::sort)
  {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    std::mt19937 r32(5);
    for (size_t n : {size_t(0), size_t(1), size_t(1000), size_t(3000017)}) {
      std::vector<int32_t> in(n);
      for (auto& x : in) x = static_cast<int32_t>(r32() >> 1);
      auto expect = in;
      std::sort(expect.begin(), expect.end());
      std::vector<int> all;
      for (int d = 0; d < ndev; ++d) all.push_back(d);
      if (ns_nccl_available()) {
        auto v = in;
        ns::sample_sort_multi(std::span<int32_t>(v), all, *ns::find_config("6To8"),
                              ns::Exchange::nccl);
        CHECK(v == expect);
      }
      for (int g : {1, 2, 3, 4}) {
        auto v = in;
        ns::sample_sort_multi(std::span<int32_t>(v), std::vector<int>(g, 0),
                              *ns::find_config("6To8"), ns::Exchange::p2p);
        CHECK(v == expect);
      }
    }
  }
}

int main(int argc, char** argv) {
  host_side();
  if (!(argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0)) device_side();
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
  return failures;
}
