// common.cuh — status plumbing shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "../../include/netsort_b200.h"

// Checked build (NSB_CHECKED=1, libnetsort_b200_checked.so): device-side
// bounds checks on every data-dependent shared / global index of the hot
// kernels (merge cursors against their slice + sentinel pad, staged slice
// extents, bucket ids and scatter positions, job-list capacities).  A failed
// check prints the condition and traps (cudaErrorLaunchFailure for the
// caller).  This stands in for compute-sanitizer, which this GPU pool does
// not allow (tests/test_checked_build.py); the default build compiles the
// checks out.
#ifndef NSB_CHECKED
#define NSB_CHECKED 0
#endif
#if NSB_CHECKED
#include <cstdio>
#define NSB_DCHECK(...)                                                                 \
  do {                                                                                  \
    if (!(__VA_ARGS__)) {                                                                      \
      printf("NSB_DCHECK failed %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, \
             #__VA_ARGS__, (int)blockIdx.x, (int)threadIdx.x);                                 \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define NSB_DCHECK(...) \
  do {                   \
  } while (0)
#endif

namespace nsb {

void set_last_error(const char* where, cudaError_t e);
void count_launch();

// Kernel classes for the built-in launch profiler (ns_profile_*).
enum ProfKind {
  PK_TILE_SORT = 0,  // blocksort_kernel
  PK_PARTITION,      // merge-path partition searches
  PK_MERGE_PASS,     // merge_pass_kernel / pairs_merge_kernel
  PK_BATCH,          // sort_small_batch_kernel
  PK_QS_SAMPLE,      // sampling + splitter selection
  PK_QS_COUNT,       // count_kernel
  PK_QS_SCATTER,     // scatter_kernel
  PK_QS_BUCKET,      // bucket_sort_kernel
  PK_PSRS,           // multi-GPU sample-sort helpers
  PK_CHECK,          // digest / inversions / generator
  PK_QS_PLAN,        // quick-sort level planning (bucket positions, work lists)
  PK_NUM_KINDS
};

// RAII: when profiling is on, records a CUDA event pair around one launch on
// the launching stream (so the timing sees exactly that stream's work).
struct Prof {
  Prof(int kind, cudaStream_t s);
  ~Prof();
  int kind;
  cudaStream_t stream;
  cudaEvent_t begin = nullptr;
};

// Returns NS_OK, or records the pending launch/runtime error.
inline int check_launch(const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    count_launch();
    return NS_OK;
  }
  set_last_error(where, e);
  return e == cudaErrorMemoryAllocation ? NS_ERR_OOM : NS_ERR_CUDA;
}

inline int check_cuda(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return NS_OK;
  set_last_error(where, e);
  return e == cudaErrorMemoryAllocation ? NS_ERR_OOM : NS_ERR_CUDA;
}

#define NSB_TRY(expr)                 \
  do {                                \
    const int _st = (expr);           \
    if (_st != NS_OK) return _st;     \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Programmatic dependent launch (sm_90+): kernels of one sort are launched
// with programmatic stream serialization, so the next kernel's CTAs can be
// scheduled while the previous kernel drains; each kernel runs its
// input-independent prologue, then pdl_wait() (griddepcontrol.wait: the
// previous grid has completed and its writes are visible) before touching
// data the previous kernel produced, and pdl_trigger() lets the following
// kernel start launching.  Both are no-ops for a kernel launched without
// the attribute.  Measured (profiles/r01_pdl_ab.txt): 3-8 % faster for sorts
// of 2^16..2^19 keys (launch-latency bound), 5-8 % SLOWER from 2^25 up, so the
// merge sort uses it only below kPdlMaxKeys.  NSB_PDL=0 / 2 forces off / on.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
constexpr int64_t kPdlMaxKeys = int64_t(1) << 19;
bool pdl_enabled(int64_t n);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int64_t n, void (*kern)(KArgs...), unsigned grid, unsigned block,
                              size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(n) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// The same with the attribute chosen by the caller.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_if(bool on, void (*kern)(KArgs...), unsigned grid, unsigned block,
                                 size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device,
// once per (device, kernel): the attribute is per device, so a process that
// drives several GPUs must set it on each.
int ensure_smem_attr(const void* kern, int bytes, const char* what);

inline int ceil_log2(uint64_t x) {
  int p = 0;
  while ((uint64_t(1) << p) < x) ++p;
  return p;
}

// Per-leaf-width template dispatch (networks.cuh leaf_of).
template <class F>
inline int with_leaf(int leaf, F&& f) {
  switch (leaf) {
    case 8: return f(std::integral_constant<int, 8>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 2: return f(std::integral_constant<int, 2>{});
    default: return f(std::integral_constant<int, 1>{});
  }
}

// Device-side sort primitives shared between translation units.
int merge_sort_device(int32_t* d_keys, size_t n, int leaf, void* d_temp, size_t temp_bytes,
                      cudaStream_t s);
int tile_sort_segments(int32_t* d_keys, size_t num_segments, size_t seg_len, int leaf,
                       cudaStream_t s);
int merge_sort_device(int64_t* d_keys, size_t n, int leaf, void* d_temp, size_t temp_bytes,
                      cudaStream_t s);
size_t merge_sort_temp(size_t n);
size_t merge_sort_temp_i64(size_t n);
int merge_existing_runs(int32_t* keys, int32_t* tmp, size_t n, int64_t R0, void* d_temp,
                        cudaStream_t s, int32_t** result);
int merge_existing_runs(int64_t* keys, int64_t* tmp, size_t n, int64_t R0, void* d_temp,
                        cudaStream_t s, int64_t** result);
constexpr int kSmallTile = 16384;  // largest array one CTA sorts on chip
// quick sort of nseg back-to-back segments of len (> kSmallTile) keys each,
// planned on the device (quicksort.cu)
size_t quick_sort_segments_temp(size_t nseg, size_t len, size_t key_bytes);
// largest array / segment the quick sort hands to the merge layer (quicksort.cu)
size_t qs_base_max();
int quick_sort_segments_device(int32_t* keys, size_t nseg, size_t len, int leaf, void* d_temp,
                               size_t temp_bytes, cudaStream_t s);
int quick_sort_segments_device(int64_t* keys, size_t nseg, size_t len, int leaf, void* d_temp,
                               size_t temp_bytes, cudaStream_t s);

}  // namespace nsb
