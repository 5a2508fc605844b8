// netsort_b200.hpp — C++20 host API with the reference's entry points.
//
// Mirrors /root/reference/proj/include/netsort/{config,hybrid}.hpp for int32
// and int64 keys so that a user of the reference can switch by changing the namespace:
//   NetworkConfig, base_case_applies      config.hpp:20-36
//   config_registry, find_config, ...     src/config.cpp:11-70
//   optimized_merge_sort (3 overloads)    hybrid.hpp:156-177
//   classical_merge_sort                  hybrid.hpp:180-183
//   optimized_quick_sort (3 overloads)    hybrid.hpp:197-216
//   classical_quick_sort                  hybrid.hpp:220-223
//   run_variant                           hybrid.hpp:225-232
// The spans are HOST memory sorted in place, as in the reference; the work
// runs on the current CUDA device through the C ABI (netsort_b200.h).  The
// device_* overloads take caller-owned device memory and a stream instead.
// Errors: config errors throw std::invalid_argument (as the reference does,
// config.cpp:16-19, networks.hpp:99-114); device errors throw
// std::runtime_error.  There is no CPU fallback.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "netsort_b200.h"

namespace netsort_b200 {

inline constexpr int kMinNetworkWidth = 2;
inline constexpr int kMaxNetworkWidth = 8;

enum class Algorithm { merge_sort, quick_sort };
std::string_view algorithm_name(Algorithm a);

struct NetworkConfig {
  std::string name;
  std::uint32_t width_mask = 0;
  int varsort_max = 0;
  bool is_classic() const { return width_mask == 0 && varsort_max == 0; }
};

inline bool base_case_applies(std::ptrdiff_t size, const NetworkConfig& cfg) {
  if (size >= kMinNetworkWidth && size <= kMaxNetworkWidth && ((cfg.width_mask >> size) & 1u))
    return true;
  return cfg.varsort_max != 0 && size >= 2 && size <= cfg.varsort_max;
}

NetworkConfig make_fixed_config(std::string name, std::initializer_list<int> widths);
NetworkConfig make_varsort_config(std::string name, int max_width);
NetworkConfig classic_config();
const std::vector<NetworkConfig>& config_registry();
const NetworkConfig* find_config(std::string_view name);

struct SortVariant {
  Algorithm algorithm;
  NetworkConfig config;
};
std::vector<SortVariant> bundled_variants();

// DispatchStats — hybrid.hpp:18-34 (same fields and helpers).
struct DispatchStats {
  std::array<std::uint64_t, kMaxNetworkWidth + 1> network_hits{};  // by width
  std::uint64_t merges = 0;
  std::uint64_t partitions = 0;
  int max_depth = 0;
  std::uint64_t total_network_hits() const {
    std::uint64_t t = 0;
    for (std::uint64_t h : network_hits) t += h;
    return t;
  }
  void network(int width) { ++network_hits[static_cast<std::size_t>(width)]; }
  void merge() { ++merges; }
  void partition() { ++partitions; }
  void depth(int d) { max_depth = d > max_depth ? d : max_depth; }
};

// The counters the reference's merge sort would record for a range of n keys
// (its recursion shape depends on n and the config only).  The GPU kernels do
// not recurse; this reproduces the reference's instrumentation exactly.
// Quick sort's counters depend on the data's pivot splits and have no GPU
// equivalent.
DispatchStats merge_sort_dispatch_stats(std::ptrdiff_t n, const NetworkConfig& cfg);

namespace detail {
inline void check(int status, const char* what) {
  if (status == NS_OK) return;
  std::string msg = std::string(what) + ": " + ns_status_string(status);
  const char* cuda = ns_last_error();
  if (cuda && *cuda) msg += std::string(" (") + cuda + ")";
  if (status == NS_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// ---- host spans (the reference's own call shape) --------------------------
// Overloads for int32 (the BASELINE configs) and int64 (the reference's own
// benchmark type: measure_loop's sort_fn takes std::span<std::int64_t>,
// bench.hpp:58-61, so run_variant below binds to it directly).

namespace detail {
inline int host_sort(std::int32_t* p, size_t n, const NetworkConfig& c, Algorithm a) {
  return a == Algorithm::merge_sort ? ns_merge_sort_host_i32(p, n, c.width_mask, c.varsort_max)
                                    : ns_quick_sort_host_i32(p, n, c.width_mask, c.varsort_max);
}
inline int host_sort(std::int64_t* p, size_t n, const NetworkConfig& c, Algorithm a) {
  return a == Algorithm::merge_sort ? ns_merge_sort_host_i64(p, n, c.width_mask, c.varsort_max)
                                    : ns_quick_sort_host_i64(p, n, c.width_mask, c.varsort_max);
}
// accumulates like the reference's Stats object across calls
inline void add_stats(DispatchStats& into, const DispatchStats& s) {
  for (std::size_t w = 0; w < into.network_hits.size(); ++w) into.network_hits[w] += s.network_hits[w];
  into.merges += s.merges;
  into.partitions += s.partitions;
  into.depth(s.max_depth);
}
inline int host_merge(std::int32_t* p, size_t n_left, size_t n) {
  return ns_merge_host_i32(p, n_left, n);
}
inline int host_merge(std::int64_t* p, size_t n_left, size_t n) {
  return ns_merge_host_i64(p, n_left, n);
}
// merge — hybrid.hpp:186-193: left <= mid <= right required (the reference
// asserts it; here it is std::invalid_argument)
template <class Key>
void merge_range(std::span<Key> a, std::ptrdiff_t left, std::ptrdiff_t mid, std::ptrdiff_t right) {
  if (!(left >= 0 && left <= mid && mid <= right && right < static_cast<std::ptrdiff_t>(a.size())))
    throw std::invalid_argument("merge: need 0 <= left <= mid <= right < size");
  check(host_merge(a.data() + left, static_cast<size_t>(mid - left + 1),
                   static_cast<size_t>(right - left + 1)),
        "merge");
}
inline int host_traced(std::int32_t* p, size_t n, const NetworkConfig& c, std::uint64_t* o) {
  return ns_quick_sort_traced_host_i32(p, n, c.width_mask, c.varsort_max, o);
}
inline int host_traced(std::int64_t* p, size_t n, const NetworkConfig& c, std::uint64_t* o) {
  return ns_quick_sort_traced_host_i64(p, n, c.width_mask, c.varsort_max, o);
}
inline int host_mot(std::int32_t* p, size_t n, std::int64_t lo, std::int64_t hi, std::int32_t* v) {
  return ns_median_of_three_host_i32(p, n, lo, hi, v);
}
inline int host_mot(std::int64_t* p, size_t n, std::int64_t lo, std::int64_t hi, std::int64_t* v) {
  return ns_median_of_three_host_i64(p, n, lo, hi, v);
}
inline int host_hoare(std::int32_t* p, size_t n, std::int64_t lo, std::int64_t hi, std::int32_t v,
                      std::int64_t* j) {
  return ns_hoare_partition_host_i32(p, n, lo, hi, v, j);
}
inline int host_hoare(std::int64_t* p, size_t n, std::int64_t lo, std::int64_t hi, std::int64_t v,
                      std::int64_t* j) {
  return ns_hoare_partition_host_i64(p, n, lo, hi, v, j);
}
// optimized_quick_sort(a, low, high, cfg, stats) — hybrid.hpp:197-204
template <class Key>
void traced_quick_sort(std::span<Key> a, std::ptrdiff_t low, std::ptrdiff_t high,
                       const NetworkConfig& cfg, DispatchStats& stats) {
  if (high < low) return;  // hybrid.hpp:201
  if (low < 0 || high >= static_cast<std::ptrdiff_t>(a.size()))
    throw std::invalid_argument("optimized_quick_sort: range outside the span");
  std::uint64_t o[12] = {};
  check(host_traced(a.data() + low, static_cast<size_t>(high - low + 1), cfg, o),
        "optimized_quick_sort(stats)");
  DispatchStats s;
  for (std::size_t w = 0; w < s.network_hits.size(); ++w) s.network_hits[w] = o[w];
  s.merges = o[9];
  s.partitions = o[10];
  s.max_depth = static_cast<int>(o[11]);
  add_stats(stats, s);
}
template <class Key>
Key median_of_three(std::span<Key> a, std::ptrdiff_t low, std::ptrdiff_t high) {
  if (!(low >= 0 && low <= high && high < static_cast<std::ptrdiff_t>(a.size())))
    throw std::invalid_argument("median_of_three: need 0 <= low <= high < size");
  Key v{};
  check(host_mot(a.data(), a.size(), low, high, &v), "median_of_three");
  return v;
}
template <class Key>
std::ptrdiff_t hoare_partition(std::span<Key> a, std::ptrdiff_t low, std::ptrdiff_t high, Key pivot) {
  if (!(low >= 0 && low < high && high < static_cast<std::ptrdiff_t>(a.size())))
    throw std::invalid_argument("hoare_partition: need 0 <= low < high < size");
  std::int64_t j = 0;
  check(host_hoare(a.data(), a.size(), low, high, pivot, &j), "hoare_partition");
  return static_cast<std::ptrdiff_t>(j);
}
template <class Key>
void sort_range(std::span<Key> a, std::ptrdiff_t lo, std::ptrdiff_t hi, const NetworkConfig& cfg,
                Algorithm alg) {
  const char* what =
      alg == Algorithm::merge_sort ? "optimized_merge_sort" : "optimized_quick_sort";
  if (hi < lo) return;  // hybrid.hpp:160, 201
  if (lo < 0 || hi >= static_cast<std::ptrdiff_t>(a.size()))
    throw std::invalid_argument(std::string(what) + ": range outside the span");
  check(host_sort(a.data() + lo, static_cast<size_t>(hi - lo + 1), cfg, alg), what);
}
}  // namespace detail

#define NETSORT_B200_HOST_OVERLOADS(KEY)                                                  \
  inline void optimized_merge_sort(std::span<KEY> a, std::ptrdiff_t left,                 \
                                   std::ptrdiff_t right, const NetworkConfig& cfg) {      \
    detail::sort_range(a, left, right, cfg, Algorithm::merge_sort);                       \
  }                                                                                       \
  inline void optimized_merge_sort(std::span<KEY> a, const NetworkConfig& cfg) {          \
    optimized_merge_sort(a, 0, static_cast<std::ptrdiff_t>(a.size()) - 1, cfg);           \
  }                                                                                       \
  inline void classical_merge_sort(std::span<KEY> a) {                                    \
    optimized_merge_sort(a, classic_config());                                            \
  }                                                                                       \
  inline void optimized_quick_sort(std::span<KEY> a, std::ptrdiff_t low,                  \
                                   std::ptrdiff_t high, const NetworkConfig& cfg) {       \
    detail::sort_range(a, low, high, cfg, Algorithm::quick_sort);                         \
  }                                                                                       \
  inline void optimized_quick_sort(std::span<KEY> a, const NetworkConfig& cfg) {          \
    optimized_quick_sort(a, 0, static_cast<std::ptrdiff_t>(a.size()) - 1, cfg);           \
  }                                                                                       \
  inline void classical_quick_sort(std::span<KEY> a) {                                    \
    optimized_quick_sort(a, classic_config());                                            \
  }                                                                                       \
  inline void run_variant(const SortVariant& v, std::span<KEY> a) {                       \
    if (v.algorithm == Algorithm::merge_sort) optimized_merge_sort(a, v.config);          \
    else optimized_quick_sort(a, v.config);                                               \
  }                                                                                       \
  /* stats overloads (hybrid.hpp:158-165, 197-204, 234-243); quick sort runs  */         \
  /* the reference's recursion node for node on the GPU (qs_trace.cu)          */         \
  inline void optimized_merge_sort(std::span<KEY> a, std::ptrdiff_t left,                 \
                                   std::ptrdiff_t right, const NetworkConfig& cfg,        \
                                   DispatchStats& stats) {                                \
    detail::sort_range(a, left, right, cfg, Algorithm::merge_sort);                       \
    if (right >= left) detail::add_stats(stats, merge_sort_dispatch_stats(right - left + 1, cfg)); \
  }                                                                                       \
  inline void optimized_quick_sort(std::span<KEY> a, std::ptrdiff_t low,                  \
                                   std::ptrdiff_t high, const NetworkConfig& cfg,         \
                                   DispatchStats& stats) {                                \
    detail::traced_quick_sort(a, low, high, cfg, stats);                                  \
  }                                                                                       \
  inline void run_variant(const SortVariant& v, std::span<KEY> a, DispatchStats& stats) { \
    if (a.empty()) return;                                                                \
    const auto hi = static_cast<std::ptrdiff_t>(a.size()) - 1;                            \
    if (v.algorithm == Algorithm::merge_sort) optimized_merge_sort(a, 0, hi, v.config, stats); \
    else optimized_quick_sort(a, 0, hi, v.config, stats);                                 \
  }                                                                                       \
  /* median_of_three / hoare_partition, hybrid.hpp:105-133 (on the GPU) */                \
  inline KEY median_of_three(std::span<KEY> a, std::ptrdiff_t low, std::ptrdiff_t high) { \
    return detail::median_of_three(a, low, high);                                         \
  }                                                                                       \
  inline std::ptrdiff_t hoare_partition(std::span<KEY> a, std::ptrdiff_t low,             \
                                        std::ptrdiff_t high, KEY pivot) {                 \
    return detail::hoare_partition(a, low, high, pivot);                                  \
  }                                                                                       \
  inline void merge(std::span<KEY> a, std::ptrdiff_t left, std::ptrdiff_t mid,             \
                    std::ptrdiff_t right) {                                               \
    detail::merge_range(a, left, mid, right);                                             \
  }

NETSORT_B200_HOST_OVERLOADS(std::int32_t)
NETSORT_B200_HOST_OVERLOADS(std::int64_t)
#undef NETSORT_B200_HOST_OVERLOADS

// ---- device spans (caller-owned device memory, stream-ordered) ------------

class DeviceScratch {
 public:
  DeviceScratch() = default;
  DeviceScratch(const DeviceScratch&) = delete;
  DeviceScratch& operator=(const DeviceScratch&) = delete;
  ~DeviceScratch();
  void* reserve(size_t bytes);  // grows, never shrinks
  size_t size() const { return bytes_; }

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
};

void device_merge_sort(std::int32_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream = nullptr);
void device_quick_sort(std::int32_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream = nullptr);
void device_merge_sort(std::int64_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream = nullptr);
void device_quick_sort(std::int64_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream = nullptr);

// ---- several GPUs, one host thread (BASELINE config 5) ---------------------
// optimized_merge_sort's call shape (a HOST array sorted in place,
// hybrid.hpp:174-177) over several devices: the array is cut into even
// shards, one per entry of `devices`, uploaded, sample-sorted
// (ns_sample_sort_multi_i32) and the devices' key ranges are read back in
// order.  Exchange::nccl creates single-process communicators
// (ncclCommInitAll; devices must be distinct); Exchange::p2p merges out of
// the peers' memory over NVLink (devices may repeat).
enum class Exchange { nccl = NS_EXCHANGE_NCCL, p2p = NS_EXCHANGE_P2P };
void sample_sort_multi(std::span<std::int32_t> a, const std::vector<int>& devices,
                       const NetworkConfig& cfg, Exchange exchange = Exchange::nccl);

}  // namespace netsort_b200
