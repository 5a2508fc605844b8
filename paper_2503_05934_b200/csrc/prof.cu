// prof.cu — launch accounting, the built-in per-kernel-class profiler and the
// device input generator.
//
// The profiler exists so bench.py can report the dominant kernel's average
// launch duration measured live, with CUDA events recorded on the stream each
// kernel is launched on (torch.cuda.Event would only see torch's stream).
// Off by default: one relaxed atomic load per launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace nsb {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};
static std::atomic<bool> g_prof_on{false};

struct ProfRecord {
  int kind;
  cudaEvent_t begin, end;
};
static std::mutex g_prof_mu;
static std::vector<ProfRecord> g_prof;

void set_last_error(const char* where, cudaError_t e) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled(int64_t n) {
  static const int mode = [] {
    const char* e = getenv("NSB_PDL");
    return e ? atoi(e) : 1;
  }();
  return mode == 2 || (mode == 1 && n <= kPdlMaxKeys);
}

int ensure_smem_attr(const void* kern, int bytes, const char* what) {
  static std::mutex mu;
  static std::vector<std::pair<int, const void*>> done;
  int dev = 0;
  NSB_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& d : done)
    if (d.first == dev && d.second == kern) return NS_OK;
  NSB_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                     what));
  // prefer the largest shared-memory carveout: these kernels are sized by
  // their shared memory, and a small default carveout can cap residency at
  // one CTA per SM
  NSB_TRY(check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          (int)cudaSharedmemCarveoutMaxShared),
                     what));
  done.emplace_back(dev, kern);
  return NS_OK;
}

Prof::Prof(int k, cudaStream_t s) : kind(k), stream(s) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  if (cudaEventCreate(&begin) != cudaSuccess) {
    begin = nullptr;
    return;
  }
  cudaEventRecord(begin, stream);
}

Prof::~Prof() {
  if (!begin) return;
  cudaEvent_t end = nullptr;
  if (cudaEventCreate(&end) != cudaSuccess) {
    cudaEventDestroy(begin);
    return;
  }
  cudaEventRecord(end, stream);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({kind, begin, end});
}

static void prof_clear() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.begin);
    cudaEventDestroy(r.end);
  }
  g_prof.clear();
}

static const char* kKindNames[PK_NUM_KINDS] = {
    "tile_sort", "merge_partition", "merge_pass", "sort_small_batch", "qs_sample",
    "qs_count",  "qs_scatter",      "qs_bucket_sort", "psrs",         "check",
    "qs_plan"};

// SplitMix64 output i of a stream seeded with `seed` is mix(seed + (i+1)*gamma)
// (include/netsort/datagen.hpp:33-38), so the stream is counter-based and the
// generator is embarrassingly parallel.  kind 0: int32(next() >> 33); kind 1:
// the ramp 0..n-1 (datagen.cpp:31-34).  Same values as oracle_generate_i32.
__global__ void generate_kernel(int32_t* __restrict__ out, int64_t n, int kind, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (kind == 1) {
      out[i] = (int32_t)i;
    } else {
      uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      out[i] = (int32_t)(z >> 33);
    }
  }
}

}  // namespace nsb

using namespace nsb;

extern "C" {

const char* ns_last_error(void) { return g_last_error.c_str(); }

uint64_t ns_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int ns_profile_enable(int on) {
  prof_clear();
  g_prof_on.store(on != 0);
  return NS_OK;
}

int ns_profile_kinds(void) { return PK_NUM_KINDS; }

const char* ns_profile_kind_name(int kind) {
  return (kind >= 0 && kind < PK_NUM_KINDS) ? kKindNames[kind] : nullptr;
}

int ns_profile_read(int kind, double* total_ms, uint64_t* launches) {
  if (kind < 0 || kind >= PK_NUM_KINDS || !total_ms || !launches) return NS_ERR_INVALID;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double ms = 0;
  uint64_t cnt = 0;
  for (auto& r : g_prof) {
    if (r.kind != kind) continue;
    NSB_TRY(check_cuda(cudaEventSynchronize(r.end), "cudaEventSynchronize"));
    float t = 0;
    NSB_TRY(check_cuda(cudaEventElapsedTime(&t, r.begin, r.end), "cudaEventElapsedTime"));
    ms += t;
    ++cnt;
  }
  *total_ms = ms;
  *launches = cnt;
  return NS_OK;
}

int ns_ipc_get_handle(const void* d_ptr, uint8_t* handle64, uint64_t* offset) {
  if (!d_ptr || !handle64 || !offset) return NS_ERR_INVALID;
  // cuMemGetAddressRange through the runtime's driver entry point, so the
  // library does not link libcuda (it must load on GPU-less build hosts)
  using range_fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static range_fn get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<range_fn>(fn);
  }();
  if (!get_range) return NS_ERR_CUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
    return NS_ERR_CUDA;
  cudaIpcMemHandle_t h;
  NSB_TRY(check_cuda(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)),
                     "cudaIpcGetMemHandle"));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle64, &h, 64);
  *offset = reinterpret_cast<uint64_t>(d_ptr) - static_cast<uint64_t>(base);
  return NS_OK;
}

int ns_ipc_open_handle(const uint8_t* handle64, void** d_base) {
  if (!handle64 || !d_base) return NS_ERR_INVALID;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  return check_cuda(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess),
                    "cudaIpcOpenMemHandle");
}

int ns_ipc_close(void* d_base) {
  if (!d_base) return NS_ERR_INVALID;
  return check_cuda(cudaIpcCloseMemHandle(d_base), "cudaIpcCloseMemHandle");
}

int ns_generate_i32(int32_t* d_out, size_t n, int kind, uint64_t seed, void* stream) {
  if ((n && !d_out) || (kind != 0 && kind != 1)) return NS_ERR_INVALID;
  if (n == 0) return NS_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Prof prof(PK_CHECK, s);
  generate_kernel<<<sms * 8, 256, 0, s>>>(d_out, (int64_t)n, kind, seed);
  return check_launch("generate_kernel");
}

}  // extern "C"
