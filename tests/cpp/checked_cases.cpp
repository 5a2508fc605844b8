// checked_cases.cpp — every kernel family of the library at small sizes,
// driven through the C ABI, linked against the CHECKED build
// (libnetsort_b200_checked.so: NSB_CHECKED=1 device-side bounds checks that
// trap; tests/test_checked_build.py).  SURVEY.md §5 asks for sanitizer CI in
// place of the reference's debug asserts (networks.hpp:36, 134, 153;
// hybrid.hpp:107, 124, 161, 189, 202); compute-sanitizer is closed on this
// GPU pool, so this driver adds what it would catch from the outside:
//   - guard zones: every device buffer (keys, offsets, scratch) sits between
//     two 4 KiB guards filled with a pattern that is verified after the case
//     (out-of-bounds writes);
//   - poisoned scratch: the caller scratch is filled with a pattern before
//     the call, so a read of scratch nobody wrote shows up in the output;
//   - every output is compared with std::sort of the input.
// Exit status = number of failed cases.
//   argv[1] (optional): a substring; only cases whose name contains it run.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "netsort_b200.h"

static int failures = 0;
static const char* filter = nullptr;

#define CK(x)                                                                          \
  do {                                                                                 \
    const int st_ = (x);                                                               \
    if (st_ != NS_OK) {                                                                \
      std::printf("FAIL %s:%d: %s -> %s (%s)\n", __FILE__, __LINE__, #x,               \
                  ns_status_string(st_), ns_last_error());                              \
      ++failures;                                                                      \
      return;                                                                          \
    }                                                                                  \
  } while (0)
#define CU(x)                                                                          \
  do {                                                                                 \
    const cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                           \
      std::printf("FAIL %s:%d: %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      ++failures;                                                                      \
      return;                                                                          \
    }                                                                                  \
  } while (0)

template <class T>
static std::vector<T> values(size_t n, uint64_t seed, int dist) {
  std::mt19937_64 rng(seed);
  std::vector<T> v(n);
  for (size_t i = 0; i < n; ++i) {
    if (dist == 0) v[i] = static_cast<T>(rng() >> (sizeof(T) == 4 ? 33 : 1));
    else if (dist == 1) v[i] = static_cast<T>(i);
    else v[i] = static_cast<T>(rng() % 7);  // heavy duplicates
  }
  return v;
}

// A device buffer between two guard zones.  The guards (and, for scratch,
// the buffer itself) are filled with a byte pattern; ~Dev verifies the guards.
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5, kPoisonByte = 0xC3;
static const char* g_case = "";
template <class T>
struct Dev {
  T* p = nullptr;
  unsigned char* base = nullptr;
  size_t bytes = 0;
  explicit Dev(size_t count, bool poison = false) : bytes(std::max<size_t>(count, 1) * sizeof(T)) {
    if (cudaMalloc(&base, bytes + 2 * kGuard) != cudaSuccess) {
      base = nullptr;
      return;
    }
    cudaMemset(base, kGuardByte, kGuard);
    cudaMemset(base + kGuard + bytes, kGuardByte, kGuard);
    if (poison) cudaMemset(base + kGuard, kPoisonByte, bytes);
    p = reinterpret_cast<T*>(base + kGuard);
  }
  ~Dev() {
    if (!base) return;
    std::vector<unsigned char> g(2 * kGuard);
    cudaDeviceSynchronize();
    if (cudaMemcpy(g.data(), base, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(g.data() + kGuard, base + kGuard + bytes, kGuard, cudaMemcpyDeviceToHost) !=
            cudaSuccess) {
      std::printf("FAIL %s: guard read-back failed (%s)\n", g_case,
                  cudaGetErrorString(cudaGetLastError()));
      ++failures;
    } else {
      for (size_t i = 0; i < g.size(); ++i)
        if (g[i] != kGuardByte) {
          std::printf("FAIL %s: guard byte %zu %s the buffer overwritten\n", g_case,
                      i < kGuard ? kGuard - i : i - kGuard, i < kGuard ? "before" : "after");
          ++failures;
          break;
        }
    }
    cudaFree(base);
  }
};

static std::string g_case_buf;
static bool run(const char* name) {
  if (filter && !std::strstr(name, filter)) return false;
  g_case_buf = name;
  g_case = g_case_buf.c_str();
  std::printf("case %s\n", name);
  std::fflush(stdout);
  return true;
}

template <class T>
static void expect_sorted_copy(const char* name, const std::vector<T>& in, const T* d, size_t n) {
  std::vector<T> got(n), want(in);
  std::sort(want.begin(), want.end());
  if (cudaMemcpy(got.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess ||
      got != want) {
    std::printf("FAIL %s: output differs from std::sort\n", name);
    ++failures;
  }
}

// merge sort / quick sort of one array through the device entry points
template <class T>
static void one_sort(const char* tag, int algo, size_t n, int dist) {
  char name[96];
  std::snprintf(name, sizeof name, "%s/%s/%s/n=%zu/dist=%d", tag, algo ? "quick" : "merge",
                sizeof(T) == 4 ? "i32" : "i64", n, dist);
  if (!run(name)) return;
  const auto in = values<T>(n, 1000 + n + dist, dist);
  Dev<T> d(n);
  CU(cudaMemcpy(d.p, in.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  uint32_t mask;
  int vs;
  CK(ns_find_config(algo ? "3To5" : "6To8", &mask, &vs));
  size_t tb;
  if constexpr (sizeof(T) == 4)
    tb = algo ? ns_quick_sort_temp_bytes(n) : ns_merge_sort_temp_bytes(n);
  else
    tb = algo ? ns_quick_sort_temp_bytes_i64(n) : ns_merge_sort_temp_bytes_i64(n);
  Dev<char> tmp(tb, true);
  if constexpr (sizeof(T) == 4) {
    CK(algo ? ns_quick_sort_i32(d.p, n, mask, vs, tmp.p, tb, nullptr)
            : ns_merge_sort_i32(d.p, n, mask, vs, tmp.p, tb, nullptr));
  } else {
    CK(algo ? ns_quick_sort_i64(d.p, n, mask, vs, tmp.p, tb, nullptr)
            : ns_merge_sort_i64(d.p, n, mask, vs, tmp.p, tb, nullptr));
  }
  CU(cudaDeviceSynchronize());
  expect_sorted_copy(name, in, d.p, n);
}

// the traced quick sort (qs_trace.cu): the reference recursion node for
// node; checked sorted (its counters are checked against the oracle by
// tests/test_gpu_qs_trace.py)
template <class T>
static void traced_case(size_t n, int dist) {
  char name[96];
  std::snprintf(name, sizeof name, "traced/%s/n=%zu/dist=%d", sizeof(T) == 4 ? "i32" : "i64", n,
                dist);
  if (!run(name)) return;
  const auto in = values<T>(n, 3000 + n + dist, dist);
  Dev<T> d(n);
  CU(cudaMemcpy(d.p, in.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  uint32_t mask;
  int vs;
  CK(ns_find_config("3To5", &mask, &vs));
  const size_t tb = ns_quick_sort_traced_temp_bytes(n);
  Dev<char> tmp(tb, true);
  uint64_t st[12];
  if constexpr (sizeof(T) == 4)
    CK(ns_quick_sort_traced_i32(d.p, n, mask, vs, st, tmp.p, tb, nullptr));
  else
    CK(ns_quick_sort_traced_i64(d.p, n, mask, vs, st, tmp.p, tb, nullptr));
  CU(cudaDeviceSynchronize());
  expect_sorted_copy(name, in, d.p, n);
  // one explicit-pivot partition over the middle of a fresh copy
  if (n >= 3) {
    CU(cudaMemcpy(d.p, in.data(), n * sizeof(T), cudaMemcpyHostToDevice));
    const size_t hb = ns_hoare_partition_temp_bytes(n);
    Dev<char> ht(hb, true);
    int64_t split = -1;
    const int64_t lo = 1, hi = (int64_t)n - 1;
    if constexpr (sizeof(T) == 4)
      CK(ns_hoare_partition_i32(d.p, n, lo, hi, in[n / 2], &split, ht.p, hb, nullptr));
    else
      CK(ns_hoare_partition_i64(d.p, n, lo, hi, in[n / 2], &split, ht.p, hb, nullptr));
    if (split < lo || split >= hi) {
      std::printf("FAIL %s: split %lld outside [%lld, %lld)\n", name, (long long)split,
                  (long long)lo, (long long)hi);
      ++failures;
    }
  }
}

static void batch_case(size_t arrays, bool bad) {
  char name[64];
  std::snprintf(name, sizeof name, "batch/arrays=%zu/%s", arrays, bad ? "invalid" : "valid");
  if (!run(name)) return;
  std::vector<uint32_t> offs(arrays + 1);
  const size_t keys = ns_generate_batch_host_i32(arrays, 42, offs.data(), nullptr);
  std::vector<int32_t> in(keys);
  ns_generate_batch_host_i32(arrays, 42, offs.data(), in.data());
  if (bad) {  // one length of 9 in the second CTA's range
    // array i absorbs the next two (>= 9 keys), which become empty
    const size_t i = std::min<size_t>(arrays - 3, 1500);
    offs[i + 1] = offs[i + 2] = offs[i + 3];
  }
  Dev<int32_t> d(keys);
  Dev<uint32_t> o(arrays + 1);
  Dev<int> st(1);
  CU(cudaMemcpy(d.p, in.data(), keys * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(o.p, offs.data(), (arrays + 1) * 4, cudaMemcpyHostToDevice));
  CK(ns_sort_small_batch_async_i32(d.p, o.p, arrays, st.p, nullptr));
  int status = -1;
  CU(cudaMemcpy(&status, st.p, 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> got(keys);
  CU(cudaMemcpy(got.data(), d.p, keys * 4, cudaMemcpyDeviceToHost));
  if (bad) {
    if (status != NS_ERR_INVALID || got != in) {
      std::printf("FAIL %s: status %d, keys %s\n", name, status, got == in ? "kept" : "modified");
      ++failures;
    }
    return;
  }
  auto want = in;
  for (size_t i = 0; i < arrays; ++i) std::sort(want.begin() + offs[i], want.begin() + offs[i + 1]);
  if (status != NS_OK || got != want) {
    std::printf("FAIL %s: status %d\n", name, status);
    ++failures;
  }
}

template <class T>
static void segmented_case(size_t segs, size_t len, int algo) {
  char name[80];
  std::snprintf(name, sizeof name, "segmented/%s/%s/%zux%zu", algo ? "quick" : "merge",
                sizeof(T) == 4 ? "i32" : "i64", segs, len);
  if (!run(name)) return;
  const size_t n = segs * len;
  const auto in = values<T>(n, 77 + n, 0);
  Dev<T> d(n);
  CU(cudaMemcpy(d.p, in.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  uint32_t mask;
  int vs;
  CK(ns_find_config(algo ? "3To5" : "6To8", &mask, &vs));
  size_t tb;
  if constexpr (sizeof(T) == 4) tb = ns_segmented_sort_temp_bytes(segs, len);
  else tb = ns_segmented_sort_temp_bytes_i64(segs, len);
  Dev<char> tmp(tb, true);
  if constexpr (sizeof(T) == 4)
    CK(ns_segmented_sort_i32(d.p, segs, len, algo, mask, vs, tmp.p, tb, nullptr));
  else
    CK(ns_segmented_sort_i64(d.p, segs, len, algo, mask, vs, tmp.p, tb, nullptr));
  std::vector<T> got(n);
  CU(cudaMemcpy(got.data(), d.p, n * sizeof(T), cudaMemcpyDeviceToHost));
  auto want = in;
  for (size_t s = 0; s < segs; ++s) std::sort(want.begin() + s * len, want.begin() + (s + 1) * len);
  if (got != want) {
    std::printf("FAIL %s\n", name);
    ++failures;
  }
}

static void pairs_case(size_t n) {
  char name[48];
  std::snprintf(name, sizeof name, "pairs/n=%zu", n);
  if (!run(name)) return;
  auto in = values<int32_t>(n, 5 + n, 2);
  Dev<int32_t> k(n);
  Dev<uint32_t> v(n);
  std::vector<uint32_t> pos(n);
  for (size_t i = 0; i < n; ++i) pos[i] = (uint32_t)i;
  CU(cudaMemcpy(k.p, in.data(), n * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(v.p, pos.data(), n * 4, cudaMemcpyHostToDevice));
  const size_t tb = ns_sort_pairs_temp_bytes_i32(n);
  Dev<char> tmp(tb, true);
  CK(ns_sort_pairs_i32(k.p, v.p, n, tmp.p, tb, nullptr));
  std::vector<int32_t> gk(n);
  std::vector<uint32_t> gv(n);
  CU(cudaMemcpy(gk.data(), k.p, n * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(gv.data(), v.p, n * 4, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> want(pos);
  std::stable_sort(want.begin(), want.end(), [&](uint32_t a, uint32_t b) { return in[a] < in[b]; });
  bool ok = gv == want;
  for (size_t i = 0; ok && i < n; ++i) ok = gk[i] == in[want[i]];
  // argsort of the same input
  Dev<uint32_t> perm(n);
  CU(cudaMemcpy(k.p, in.data(), n * 4, cudaMemcpyHostToDevice));
  const size_t ta = ns_argsort_temp_bytes_i32(n);
  Dev<char> tmp2(ta, true);
  CK(ns_argsort_i32(k.p, perm.p, n, tmp2.p, ta, nullptr));
  CU(cudaMemcpy(gv.data(), perm.p, n * 4, cudaMemcpyDeviceToHost));
  ok = ok && gv == want;
  if (!ok) {
    std::printf("FAIL %s\n", name);
    ++failures;
  }
}

static void merge_runs_case(size_t n, int runs) {
  char name[48];
  std::snprintf(name, sizeof name, "merge_runs/n=%zu/runs=%d", n, runs);
  if (!run(name)) return;
  auto in = values<int32_t>(n, 9 + n, 0);
  std::vector<int64_t> off(runs + 1);
  for (int r = 0; r <= runs; ++r) off[r] = (int64_t)(n * (size_t)r * (size_t)r / ((size_t)runs * runs));
  for (int r = 0; r < runs; ++r) std::sort(in.begin() + off[r], in.begin() + off[r + 1]);
  Dev<int32_t> d(n);
  CU(cudaMemcpy(d.p, in.data(), n * 4, cudaMemcpyHostToDevice));
  const size_t tb = ns_merge_runs_temp_bytes(n, runs);
  Dev<char> tmp(tb, true);
  CK(ns_merge_runs_i32(d.p, off.data(), runs, tmp.p, tb, nullptr));
  CU(cudaDeviceSynchronize());
  expect_sorted_copy(name, in, d.p, n);

  // the pointer-pair merge (sample sort's fused exchange) on odd offsets
  if (runs >= 2) {
    Dev<int32_t> a(n), out(n);
    CU(cudaMemcpy(a.p, in.data(), n * 4, cudaMemcpyHostToDevice));
    const int32_t* ap[2] = {a.p + off[0], a.p + off[1]};
    const int32_t* bp[2] = {a.p + off[1], a.p + off[2]};
    int64_t al[2] = {off[1] - off[0], 0};
    int64_t bl[2] = {off[2] - off[1], 0};
    const size_t tp = ns_merge_pairs_temp_bytes(al[0] + bl[0], 1);
    Dev<char> t2(tp, true);
    CK(ns_merge_pairs_i32(ap, al, bp, bl, 1, out.p, t2.p, tp, nullptr));
    CU(cudaDeviceSynchronize());
    std::vector<int32_t> sub(in.begin() + off[0], in.begin() + off[2]);
    expect_sorted_copy("merge_pairs", sub, out.p, sub.size());
  }
}

static void host_case(size_t n) {
  char name[48];
  std::snprintf(name, sizeof name, "host/n=%zu", n);
  if (!run(name)) return;
  auto in = values<int32_t>(n, 21 + n, 0);
  auto a = in;
  uint32_t mask;
  int vs;
  CK(ns_find_config("6To8", &mask, &vs));
  CK(ns_merge_sort_host_i32(a.data(), n, mask, vs));
  auto b = in;
  CK(ns_quick_sort_host_i32(b.data(), n, mask, vs));
  auto want = in;
  std::sort(want.begin(), want.end());
  if (a != want || b != want) {
    std::printf("FAIL %s\n", name);
    ++failures;
  }
  CK(ns_release_cache());
}

int main(int argc, char** argv) {
  if (argc > 1) filter = argv[1];
  // merge sort: one-CTA shapes, two tiles + fused pass, 8192- and 16384-key
  // tiles with partition-kernel passes (NSB_FUSED_MAX=0 in the test forces
  // the separate partition on every pass), ragged tails
  for (size_t n : {5u, 100u, 3000u, 9000u, 20000u, 250001u}) one_sort<int32_t>("ms", 0, n, 0);
  one_sort<int32_t>("ms", 0, 250001, 2);
  one_sort<int32_t>("ms", 0, (1u << 21) + 4099, 0);
  for (size_t n : {700u, 50000u}) one_sort<int64_t>("ms", 0, n, 0);
  // quick sort: one tile, one partition level, two levels; sorted and
  // duplicate-heavy inputs (equal buckets)
  for (size_t n : {5000u, 200000u}) {
    one_sort<int32_t>("qs", 1, n, 0);
    one_sort<int32_t>("qs", 1, n, 1);
    one_sort<int32_t>("qs", 1, n, 2);
  }
  one_sort<int32_t>("qs", 1, 1500000, 0);
  one_sort<int64_t>("qs", 1, 100000, 0);
  for (size_t n : {1u, 7u, 3000u, 8192u, 8193u, 60000u}) traced_case<int32_t>(n, 0);
  traced_case<int32_t>(100000, 1);
  traced_case<int32_t>(100000, 2);
  traced_case<int64_t>(30000, 0);
  batch_case(3000, false);
  batch_case(3000, true);
  segmented_case<int32_t>(24, 5000, 0);
  segmented_case<int32_t>(6, 16384, 1);
  segmented_case<int32_t>(3, 40000, 1);
  segmented_case<int32_t>(3, 40000, 0);
  segmented_case<int32_t>(2, 70001, 0);
  segmented_case<int64_t>(3, 20000, 0);
  segmented_case<int64_t>(5, 3000, 0);
  // segments that share warps (small_segments_kernel): every lane-group size,
  // a ragged last warp / CTA; the guard zones catch a lane that stores past
  // its segment or a group that touches the next segment's keys
  for (size_t len : {1, 7, 16, 17, 33, 100, 129, 256})
    for (size_t segs : {1, 37, 300}) {
      segmented_case<int32_t>(segs, len, 0);
      segmented_case<int64_t>(segs, len, 1);
    }
  segmented_case<int32_t>(50, 257, 0);
  segmented_case<int32_t>(50, 512, 1);
  pairs_case(30000);
  merge_runs_case(100000, 3);
  host_case(10000);
  host_case(70000);
  std::printf("%s (%d failure(s))\n", failures ? "FAILED" : "PASSED", failures);
  return failures;
}
