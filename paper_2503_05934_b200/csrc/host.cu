// host.cu — host-buffer entry points (the reference's own call shape:
// optimized_merge_sort(span, cfg) sorts a host array in place,
// /root/reference/proj/include/netsort/hybrid.hpp:174-177) and the C++
// DeviceScratch / device_* helpers declared in include/netsort_b200.hpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/netsort_b200.hpp"
#include "common.cuh"

namespace nsb {
size_t quick_sort_temp(size_t n);
size_t quick_sort_temp_i64(size_t n);

// Per-thread device staging: keys + scratch, grown on demand, plus one
// non-blocking stream.  Mirrors the reference's per-call `new T[n]` scratch
// (hybrid.hpp:163) without paying an allocation on every call.
constexpr int kMaxChunks = 8;

struct HostCache {
  void* dev = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t copy = nullptr;    // host->device chunks
  cudaEvent_t ev[kMaxChunks] = {};
  ~HostCache() { release(); }
  void release() {
    if (dev) cudaFree(dev);
    if (stream) cudaStreamDestroy(stream);
    if (copy) cudaStreamDestroy(copy);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : ev) e = nullptr;
    dev = nullptr;
    bytes = 0;
    stream = nullptr;
    copy = nullptr;
  }
  int ensure(size_t need) {
    if (!stream) {
      NSB_TRY(check_cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking),
                         "cudaStreamCreate"));
      NSB_TRY(check_cuda(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking),
                         "cudaStreamCreate"));
      for (auto& e : ev)
        NSB_TRY(check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming),
                           "cudaEventCreate"));
    }
    if (bytes >= need) return NS_OK;
    if (dev) cudaFree(dev);
    dev = nullptr;
    bytes = 0;
    NSB_TRY(check_cuda(cudaMalloc(&dev, need), "cudaMalloc"));
    bytes = need;
    return NS_OK;
  }
};
static thread_local HostCache g_host;

// Host-buffer sort.  Large merge sorts overlap the PCIe upload with compute:
// the array is cut into up to 8 chunks (multiples of the 8192-key tile); each
// chunk is merge-sorted on the compute stream as soon as its copy (on the copy
// stream) lands, so the tile sort and all intra-chunk merge passes hide under
// the host->device transfer; log2(chunks) pairwise passes then merge the
// chunks and the result is read back from whichever buffer holds it.
static size_t dev_temp(const int32_t*, int algorithm, size_t n) {
  return algorithm == NS_MERGE_SORT ? merge_sort_temp(n) : quick_sort_temp(n);
}
static size_t dev_temp(const int64_t*, int algorithm, size_t n) {
  return algorithm == NS_MERGE_SORT ? merge_sort_temp_i64(n) : quick_sort_temp_i64(n);
}
static int dev_sort(int32_t* d, size_t n, uint32_t mask, int vs, void* t, size_t tb, int algorithm,
                    cudaStream_t s) {
  return algorithm == NS_MERGE_SORT ? ns_merge_sort_i32(d, n, mask, vs, t, tb, s)
                                    : ns_quick_sort_i32(d, n, mask, vs, t, tb, s);
}
static int dev_sort(int64_t* d, size_t n, uint32_t mask, int vs, void* t, size_t tb, int algorithm,
                    cudaStream_t s) {
  return algorithm == NS_MERGE_SORT ? ns_merge_sort_i64(d, n, mask, vs, t, tb, s)
                                    : ns_quick_sort_i64(d, n, mask, vs, t, tb, s);
}

template <class Key>
static int host_sort(Key* h_keys, size_t n, uint32_t mask, int vs, int algorithm) {
  if (n <= 1) return NS_OK;
  if (!h_keys) return NS_ERR_INVALID;
  constexpr size_t KB = sizeof(Key);
  const size_t kb = align_up(n * KB, 256);
  const size_t tb = dev_temp(h_keys, algorithm, n);
  NSB_TRY(g_host.ensure(kb + tb));
  cudaStream_t s = g_host.stream;
  Key* d = static_cast<Key*>(g_host.dev);
  void* t = static_cast<char*>(g_host.dev) + kb;
  const size_t chunk_min = (size_t(1) << 24) / KB;  // 16 MiB
  Key* result = d;
  if (algorithm == NS_MERGE_SORT && n >= 2 * chunk_min) {
    int chunks = (int)std::min<size_t>(kMaxChunks, n / chunk_min);
    size_t clen = (n + chunks - 1) / chunks;
    clen = (clen + 8191) / 8192 * 8192;
    chunks = (int)((n + clen - 1) / clen);
    for (int c = 0; c < chunks; ++c) {
      const size_t off = c * clen, len = std::min(clen, n - off);
      NSB_TRY(check_cuda(cudaMemcpyAsync(d + off, h_keys + off, len * KB, cudaMemcpyHostToDevice,
                                         g_host.copy),
                         "H2D"));
      NSB_TRY(check_cuda(cudaEventRecord(g_host.ev[c], g_host.copy), "cudaEventRecord"));
    }
    for (int c = 0; c < chunks; ++c) {
      const size_t off = c * clen, len = std::min(clen, n - off);
      NSB_TRY(check_cuda(cudaStreamWaitEvent(s, g_host.ev[c], 0), "cudaStreamWaitEvent"));
      const int st = dev_sort(d + off, len, mask, vs, t, tb, NS_MERGE_SORT, s);
      if (st != NS_OK) {
        cudaStreamSynchronize(s);
        return st;
      }
    }
    NSB_TRY(merge_existing_runs(d, static_cast<Key*>(t), n, (int64_t)clen, t, s, &result));
  } else {
    NSB_TRY(check_cuda(cudaMemcpyAsync(d, h_keys, n * KB, cudaMemcpyHostToDevice, s), "H2D"));
    const int st = dev_sort(d, n, mask, vs, t, tb, algorithm, s);
    if (st != NS_OK) {
      cudaStreamSynchronize(s);
      return st;
    }
  }
  NSB_TRY(check_cuda(cudaMemcpyAsync(h_keys, result, n * KB, cudaMemcpyDeviceToHost, s), "D2H"));
  return check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

// merge (hybrid.hpp:186-193) on a host array: upload, one two-run merge, read back.
static size_t merge_temp(const int32_t*, size_t n) { return ns_merge_runs_temp_bytes(n, 2); }
static size_t merge_temp(const int64_t*, size_t n) { return ns_merge_runs_temp_bytes_i64(n, 2); }
static int merge_dev(int32_t* d, const int64_t* offs, void* t, size_t tb, cudaStream_t s) {
  return ns_merge_runs_i32(d, offs, 2, t, tb, s);
}
static int merge_dev(int64_t* d, const int64_t* offs, void* t, size_t tb, cudaStream_t s) {
  return ns_merge_runs_i64(d, offs, 2, t, tb, s);
}

template <class Key>
static int host_merge(Key* h_keys, size_t n_left, size_t n) {
  if (n_left > n) return NS_ERR_INVALID;
  if (n_left == 0 || n_left == n) return NS_OK;
  if (!h_keys) return NS_ERR_INVALID;
  constexpr size_t KB = sizeof(Key);
  const size_t kb = align_up(n * KB, 256);
  const size_t tb = merge_temp(h_keys, n);
  NSB_TRY(g_host.ensure(kb + tb));
  cudaStream_t s = g_host.stream;
  Key* d = static_cast<Key*>(g_host.dev);
  void* t = static_cast<char*>(g_host.dev) + kb;
  const int64_t offs[3] = {0, (int64_t)n_left, (int64_t)n};
  NSB_TRY(check_cuda(cudaMemcpyAsync(d, h_keys, n * KB, cudaMemcpyHostToDevice, s), "H2D"));
  const int st = merge_dev(d, offs, t, tb, s);
  if (st != NS_OK) {
    cudaStreamSynchronize(s);
    return st;
  }
  NSB_TRY(check_cuda(cudaMemcpyAsync(h_keys, d, n * KB, cudaMemcpyDeviceToHost, s), "D2H"));
  return check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

}  // namespace nsb

extern "C" {

int ns_merge_host_i32(int32_t* h_keys, size_t n_left, size_t n) {
  return nsb::host_merge(h_keys, n_left, n);
}

int ns_merge_host_i64(int64_t* h_keys, size_t n_left, size_t n) {
  return nsb::host_merge(h_keys, n_left, n);
}


int ns_merge_sort_host_i32(int32_t* h_keys, size_t n, uint32_t width_mask, int varsort_max) {
  return nsb::host_sort(h_keys, n, width_mask, varsort_max, NS_MERGE_SORT);
}

int ns_quick_sort_host_i32(int32_t* h_keys, size_t n, uint32_t width_mask, int varsort_max) {
  return nsb::host_sort(h_keys, n, width_mask, varsort_max, NS_QUICK_SORT);
}

int ns_merge_sort_host_i64(int64_t* h_keys, size_t n, uint32_t width_mask, int varsort_max) {
  return nsb::host_sort(h_keys, n, width_mask, varsort_max, NS_MERGE_SORT);
}

int ns_quick_sort_host_i64(int64_t* h_keys, size_t n, uint32_t width_mask, int varsort_max) {
  return nsb::host_sort(h_keys, n, width_mask, varsort_max, NS_QUICK_SORT);
}

int ns_release_cache(void) {
  nsb::g_host.release();
  return NS_OK;
}

}  // extern "C"

namespace netsort_b200 {

DeviceScratch::~DeviceScratch() {
  if (ptr_) cudaFree(ptr_);
}

void* DeviceScratch::reserve(size_t bytes) {
  if (bytes <= bytes_) return ptr_;
  if (ptr_) cudaFree(ptr_);
  ptr_ = nullptr;
  bytes_ = 0;
  if (bytes == 0) return nullptr;
  detail::check(nsb::check_cuda(cudaMalloc(&ptr_, bytes), "cudaMalloc"), "DeviceScratch");
  bytes_ = bytes;
  return ptr_;
}

void device_merge_sort(std::int32_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream) {
  const size_t tb = ns_merge_sort_temp_bytes(n);
  void* t = scratch.reserve(tb);
  detail::check(ns_merge_sort_i32(d_keys, n, cfg.width_mask, cfg.varsort_max, t, tb, stream),
                "device_merge_sort");
}

void device_quick_sort(std::int32_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream) {
  const size_t tb = ns_quick_sort_temp_bytes(n);
  void* t = scratch.reserve(tb);
  detail::check(ns_quick_sort_i32(d_keys, n, cfg.width_mask, cfg.varsort_max, t, tb, stream),
                "device_quick_sort");
}

void device_merge_sort(std::int64_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream) {
  const size_t tb = ns_merge_sort_temp_bytes_i64(n);
  void* t = scratch.reserve(tb);
  detail::check(ns_merge_sort_i64(d_keys, n, cfg.width_mask, cfg.varsort_max, t, tb, stream),
                "device_merge_sort");
}

void device_quick_sort(std::int64_t* d_keys, size_t n, const NetworkConfig& cfg,
                       DeviceScratch& scratch, void* stream) {
  const size_t tb = ns_quick_sort_temp_bytes_i64(n);
  void* t = scratch.reserve(tb);
  detail::check(ns_quick_sort_i64(d_keys, n, cfg.width_mask, cfg.varsort_max, t, tb, stream),
                "device_quick_sort");
}

}  // namespace netsort_b200
