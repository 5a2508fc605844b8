// host.cu — host-buffer entry points (the reference's own call shape:
// optimized_merge_sort(span, cfg) sorts a host array in place,
// /root/reference/proj/include/netsort/hybrid.hpp:174-177) and the C++
// DeviceScratch / device_* helpers declared in include/netsort_b200.hpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

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
  // small arrays (<= kSmallTile keys): pinned, device-mapped staging that the
  // one-CTA sort reads and writes in place over PCIe (zero-copy): one launch
  // and one synchronise per call, no DMA round trips
  void* pinned = nullptr;
  void* mapped = nullptr;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t copy = nullptr;    // host->device chunks
  cudaEvent_t ev[kMaxChunks] = {};
  ~HostCache() { release(); }
  void release() {
    if (pinned) cudaFreeHost(pinned);
    pinned = mapped = nullptr;
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
  int ensure_pinned() {
    if (pinned) return NS_OK;
    NSB_TRY(check_cuda(cudaHostAlloc(&pinned, (size_t)kSmallTile * 8, cudaHostAllocMapped),
                       "cudaHostAlloc"));
    return check_cuda(cudaHostGetDevicePointer(&mapped, pinned, 0), "cudaHostGetDevicePointer");
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
    if (need == 0) return NS_OK;
    if (bytes >= need) return NS_OK;
    if (dev) cudaFree(dev);
    dev = nullptr;
    bytes = 0;
    NSB_TRY(check_cuda(cudaMalloc(&dev, need), "cudaMalloc"));
    bytes = need;
    return NS_OK;
  }
};
// One cache per (host thread, device): a thread that switches devices gets
// that device's own buffers and streams.
struct HostCaches {
  HostCache d[64];
};
static thread_local HostCaches g_hosts;
static int host_cache(HostCache** out) {
  int dev = 0;
  NSB_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  if (dev < 0 || dev >= 64) return NS_ERR_INVALID;
  *out = &g_hosts.d[dev];
  return NS_OK;
}

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
  HostCache* hc = nullptr;
  NSB_TRY(host_cache(&hc));
  HostCache& g_host = *hc;
  if (n <= (size_t)kSmallTile) {
    // the keys stay in the mapped staging buffer (zero-copy over PCIe: one
    // launch sequence and one synchronise per call, no DMA round trips); up to
    // 8192 keys one CTA sorts them there, above that the tiled path reads them
    // once (tile sort -> device scratch) and writes them once (the merge pass's
    // bulk store into mapped memory); quick sort delegates to the merge sort
    // at these sizes
    const size_t tb = dev_temp(h_keys, algorithm, n);
    NSB_TRY(g_host.ensure(tb));
    NSB_TRY(g_host.ensure_pinned());
    std::memcpy(g_host.pinned, h_keys, n * KB);
    const int st = dev_sort(static_cast<Key*>(g_host.mapped), n, mask, vs, tb ? g_host.dev : nullptr,
                            tb, algorithm, g_host.stream);
    NSB_TRY(check_cuda(cudaStreamSynchronize(g_host.stream), "cudaStreamSynchronize"));
    if (st != NS_OK) return st;
    std::memcpy(h_keys, g_host.pinned, n * KB);
    return NS_OK;
  }
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
  HostCache* hc = nullptr;
  NSB_TRY(host_cache(&hc));
  HostCache& g_host = *hc;
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

// ---- stream-ordered host-array sort ------------------------------------------
// H2D of h_in, the device sort, D2H into h_out, all enqueued on the caller's
// stream; the call returns at once.  Device keys + scratch come from a cache
// keyed by (device, stream): a buffer is only reused by later calls on the
// same stream, so stream order is the only synchronisation it needs.  With
// pinned host buffers, sorts issued on two streams overlap one's upload with
// the other's download (PCIe is full duplex).
struct AsyncSlot {
  int dev = -1;
  cudaStream_t stream = nullptr;
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t copy = nullptr;  // chunked uploads of large merge sorts
  cudaEvent_t start = nullptr, ev[kMaxChunks] = {};
};
static std::mutex g_async_mu;
static std::vector<AsyncSlot> g_async;
// Uploads of the async calls on one device are serialised in issue order
// (each waits for the previous call's last H2D): one host link cannot upload
// two arrays faster than one after the other, and staggering them lets call
// k+1's upload run under call k's download instead of both uploading, then
// both downloading.
static cudaEvent_t g_upload_done[64] = {};

static void release_async_slots() {
  std::lock_guard<std::mutex> lk(g_async_mu);
  for (auto& a : g_async) {
    if (a.ptr) {
      cudaStreamSynchronize(a.stream);
      cudaFree(a.ptr);
    }
    if (a.copy) cudaStreamDestroy(a.copy);  // (g_upload_done events are kept)
    if (a.start) cudaEventDestroy(a.start);
    for (auto& e : a.ev)
      if (e) cudaEventDestroy(e);
  }
  g_async.clear();
}

template <class Key>
static int host_sort_async(const Key* h_in, Key* h_out, size_t n, uint32_t mask, int vs,
                           int algorithm, cudaStream_t s) {
  if (n == 0) return NS_OK;
  if (!h_in || !h_out) return NS_ERR_INVALID;
  constexpr size_t KB = sizeof(Key);
  const size_t kb = align_up(n * KB, 256);
  const size_t tb = dev_temp(h_in, algorithm, n);
  int dev = 0;
  NSB_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  void* buf = nullptr;
  AsyncSlot sl;
  {
    std::lock_guard<std::mutex> lk(g_async_mu);
    AsyncSlot* slot = nullptr;
    for (auto& a : g_async)
      if (a.dev == dev && a.stream == s) slot = &a;
    if (!slot) {
      g_async.push_back(AsyncSlot{});
      slot = &g_async.back();
      slot->dev = dev;
      slot->stream = s;
      NSB_TRY(check_cuda(cudaStreamCreateWithFlags(&slot->copy, cudaStreamNonBlocking),
                         "cudaStreamCreate"));
      NSB_TRY(check_cuda(cudaEventCreateWithFlags(&slot->start, cudaEventDisableTiming),
                         "cudaEventCreate"));
      for (auto& e : slot->ev)
        NSB_TRY(check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate"));
    }
    if (dev < 0 || dev >= 64) return NS_ERR_INVALID;
    if (!g_upload_done[dev])
      NSB_TRY(check_cuda(cudaEventCreateWithFlags(&g_upload_done[dev], cudaEventDisableTiming),
                         "cudaEventCreate"));
    if (slot->bytes < kb + tb) {
      if (slot->ptr) {
        NSB_TRY(check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize"));  // earlier work on it
        cudaFree(slot->ptr);
        slot->ptr = nullptr;
        slot->bytes = 0;
      }
      NSB_TRY(check_cuda(cudaMalloc(&slot->ptr, kb + tb), "cudaMalloc"));
      slot->bytes = kb + tb;
    }
    buf = slot->ptr;
    sl = *slot;
  }
  // issue order of the uploads (see g_upload_done); the enqueueing below is
  // under the lock so two host threads cannot interleave their event chain
  std::lock_guard<std::mutex> lk(g_async_mu);
  cudaEvent_t& up = g_upload_done[dev];
  Key* d = static_cast<Key*>(buf);
  void* t = static_cast<char*>(buf) + kb;
  Key* result = d;
  const size_t chunk_min = (size_t(1) << 24) / KB;  // 16 MiB
  if (algorithm == NS_MERGE_SORT && n >= 2 * chunk_min) {
    // as host_sort: chunks uploaded on the slot's copy stream, each merge-
    // sorted on `s` as soon as it lands, then the chunks merged.  The copy
    // stream first waits for everything earlier on `s` (the previous sort on
    // this slot may still be downloading from d).
    int chunks = (int)std::min<size_t>(kMaxChunks, n / chunk_min);
    size_t clen = (n + chunks - 1) / chunks;
    clen = (clen + 8191) / 8192 * 8192;
    chunks = (int)((n + clen - 1) / clen);
    NSB_TRY(check_cuda(cudaEventRecord(sl.start, s), "cudaEventRecord"));
    NSB_TRY(check_cuda(cudaStreamWaitEvent(sl.copy, sl.start, 0), "cudaStreamWaitEvent"));
    NSB_TRY(check_cuda(cudaStreamWaitEvent(sl.copy, up, 0), "cudaStreamWaitEvent"));
    for (int c = 0; c < chunks; ++c) {
      const size_t off = c * clen, len = std::min(clen, n - off);
      NSB_TRY(check_cuda(cudaMemcpyAsync(d + off, h_in + off, len * KB, cudaMemcpyHostToDevice,
                                         sl.copy),
                         "H2D"));
      NSB_TRY(check_cuda(cudaEventRecord(sl.ev[c], sl.copy), "cudaEventRecord"));
    }
    NSB_TRY(check_cuda(cudaEventRecord(up, sl.copy), "cudaEventRecord"));
    for (int c = 0; c < chunks; ++c) {
      const size_t off = c * clen, len = std::min(clen, n - off);
      NSB_TRY(check_cuda(cudaStreamWaitEvent(s, sl.ev[c], 0), "cudaStreamWaitEvent"));
      NSB_TRY(dev_sort(d + off, len, mask, vs, t, tb, NS_MERGE_SORT, s));
    }
    NSB_TRY(merge_existing_runs(d, static_cast<Key*>(t), n, (int64_t)clen, t, s, &result));
  } else {
    NSB_TRY(check_cuda(cudaStreamWaitEvent(s, up, 0), "cudaStreamWaitEvent"));
    NSB_TRY(check_cuda(cudaMemcpyAsync(d, h_in, n * KB, cudaMemcpyHostToDevice, s), "H2D"));
    NSB_TRY(check_cuda(cudaEventRecord(up, s), "cudaEventRecord"));
    NSB_TRY(dev_sort(d, n, mask, vs, tb ? t : nullptr, tb, algorithm, s));
  }
  return check_cuda(cudaMemcpyAsync(h_out, result, n * KB, cudaMemcpyDeviceToHost, s), "D2H");
}

}  // namespace nsb

extern "C" {

int ns_merge_sort_host_async_i32(const int32_t* h_in, int32_t* h_out, size_t n, uint32_t width_mask,
                                 int varsort_max, void* stream) {
  return nsb::host_sort_async(h_in, h_out, n, width_mask, varsort_max, NS_MERGE_SORT,
                              static_cast<cudaStream_t>(stream));
}

int ns_quick_sort_host_async_i32(const int32_t* h_in, int32_t* h_out, size_t n, uint32_t width_mask,
                                 int varsort_max, void* stream) {
  return nsb::host_sort_async(h_in, h_out, n, width_mask, varsort_max, NS_QUICK_SORT,
                              static_cast<cudaStream_t>(stream));
}

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
  for (auto& c : nsb::g_hosts.d) c.release();
  nsb::release_async_slots();
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

void sample_sort_multi(std::span<std::int32_t> a, const std::vector<int>& devices,
                       const NetworkConfig& cfg, Exchange exchange) {
  const int g = (int)devices.size();
  if (g < 1) throw std::invalid_argument("sample_sort_multi: no devices");
  const size_t n = a.size();
  std::vector<size_t> counts(g), start(g + 1, 0);
  for (int d = 0; d < g; ++d) {
    start[d + 1] = n * (size_t)(d + 1) / (size_t)g;
    counts[d] = start[d + 1] - start[d];
  }
  const size_t shard_max = *std::max_element(counts.begin(), counts.end());
  size_t cap = std::min(n, 2 * shard_max + (size_t)4096 * g);
  if (cap == 0) cap = 1;
  std::vector<int32_t*> shards(g, nullptr), outs(g, nullptr);
  std::vector<void*> temps(g, nullptr), streams(g, nullptr);
  std::vector<ns_nccl_comm> comms(g, nullptr);
  int prev = 0;
  cudaGetDevice(&prev);
  auto cleanup = [&] {
    for (int d = 0; d < g; ++d) {
      cudaSetDevice(devices[d]);
      if (shards[d]) cudaFree(shards[d]);
      if (outs[d]) cudaFree(outs[d]);
      if (temps[d]) cudaFree(temps[d]);
      if (streams[d]) cudaStreamDestroy(static_cast<cudaStream_t>(streams[d]));
    }
    if (exchange == Exchange::nccl && comms[0]) ns_nccl_comms_destroy(g, comms.data());
    cudaSetDevice(prev);
  };
  int st = NS_OK;
  size_t tb = 0;
  std::vector<size_t> oc(g, 0);
  for (int attempt = 0; attempt < 2; ++attempt) {
    tb = ns_sample_sort_multi_temp_bytes(g, shard_max, cap);
    for (int d = 0; d < g && st == NS_OK; ++d) {
      st = nsb::check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice");
      cudaStream_t s = static_cast<cudaStream_t>(streams[d]);
      if (st == NS_OK && !s) {
        st = nsb::check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        streams[d] = s;
      }
      if (st == NS_OK && !shards[d])
        st = nsb::check_cuda(cudaMalloc(&shards[d], std::max<size_t>(counts[d], 1) * 4), "cudaMalloc");
      if (outs[d]) cudaFree(outs[d]);
      if (temps[d]) cudaFree(temps[d]);
      outs[d] = nullptr;
      temps[d] = nullptr;
      if (st == NS_OK) st = nsb::check_cuda(cudaMalloc(&outs[d], cap * 4), "cudaMalloc");
      if (st == NS_OK) st = nsb::check_cuda(cudaMalloc(&temps[d], tb), "cudaMalloc");
      if (st == NS_OK)
        st = nsb::check_cuda(cudaMemcpyAsync(shards[d], a.data() + start[d], counts[d] * 4,
                                             cudaMemcpyHostToDevice, s),
                             "H2D");
    }
    if (st == NS_OK && exchange == Exchange::nccl && !comms[0])
      st = ns_nccl_comms_init_all(g, devices.data(), comms.data());
    if (st == NS_OK)
      st = ns_sample_sort_multi_i32(g, devices.data(),
                                    exchange == Exchange::nccl ? comms.data() : nullptr,
                                    (int)exchange, shards.data(), counts.data(), outs.data(), cap,
                                    oc.data(), cfg.width_mask, cfg.varsort_max, temps.data(), tb,
                                    streams.data());
    if (st == NS_ERR_TEMP && *std::max_element(oc.begin(), oc.end()) > cap) {
      cap = *std::max_element(oc.begin(), oc.end());  // a bucket above the PSRS estimate
      st = NS_OK;
      continue;
    }
    break;
  }
  size_t at = 0;
  for (int d = 0; d < g && st == NS_OK; ++d) {
    st = nsb::check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice");
    if (st == NS_OK && oc[d])
      st = nsb::check_cuda(cudaMemcpy(a.data() + at, outs[d], oc[d] * 4, cudaMemcpyDeviceToHost), "D2H");
    at += oc[d];
  }
  cleanup();
  detail::check(st, "sample_sort_multi");
  if (at != n) throw std::runtime_error("sample_sort_multi: lost keys");
}

}  // namespace netsort_b200
