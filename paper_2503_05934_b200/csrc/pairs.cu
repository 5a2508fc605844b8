// pairs.cu — stable key-value sort and argsort.
//
// The reference's classical merge sort is stable (merge_runs takes the left
// run on ties, hybrid.hpp:61-79; test_hybrid.cpp:119-150 checks it on
// key/tag pairs).  Its network base case is not, and the reference has no
// payload API.  A keys-only sort of int32 gives unique bytes, so stability
// only matters once a payload rides along.  This file provides that
// capability on the GPU:
//   composite[i] = (int64(key[i]) << 32) | i
// is unique per element, and the int64 ordering of the composites is the
// (key, original position) lexicographic order.  Any correct sort of the
// composites is therefore THE stable order.  The composites go through the
// int64 merge sort (networks.cuh base case, merge passes); then one pass
// splits them into keys and the permutation and gathers the payload.
//
// Traffic: pack 4n read + 8n write; the int64 sort; unpack 8n read + 4n + 4n
// write + a 4n-byte payload gather.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace nsb {

size_t merge_sort_temp_i64(size_t n);

__global__ void pack_pairs_kernel(const int32_t* __restrict__ keys, int64_t n,
                                  int64_t* __restrict__ comp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    comp[i] = (int64_t)((uint64_t)(int64_t)__ldcs(keys + i) << 32 | (uint64_t)(uint32_t)i);
}

// keys_out / perm_out may be null; values_out[i] = values_in[perm[i]] when
// both value pointers are set.
__global__ void unpack_pairs_kernel(const int64_t* __restrict__ comp, int64_t n,
                                    int32_t* __restrict__ keys_out, uint32_t* __restrict__ perm_out,
                                    const uint32_t* __restrict__ values_in,
                                    uint32_t* __restrict__ values_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = __ldcs(comp + i);
    const uint32_t p = (uint32_t)c;
    if (keys_out) keys_out[i] = (int32_t)(c >> 32);
    if (perm_out) perm_out[i] = p;
    if (values_out) values_out[i] = __ldg(values_in + p);
  }
}

static unsigned grid_of(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return (unsigned)(want < (int64_t)sms * 16 ? (want < 1 ? 1 : want) : (int64_t)sms * 16);
}

// scratch: composites (8n) | int64 merge-sort temp | payload copy (4n)
static size_t pairs_temp(size_t n) {
  return align_up(n * 8, 256) + align_up(merge_sort_temp_i64(n), 256) + align_up(n * 4, 256);
}

static int sort_composites(const int32_t* keys, size_t n, void* d_temp, cudaStream_t s,
                           int64_t** comp_out) {
  int64_t* comp = static_cast<int64_t*>(d_temp);
  char* mst = static_cast<char*>(d_temp) + align_up(n * 8, 256);
  {
    Prof prof(PK_CHECK, s);
    pack_pairs_kernel<<<grid_of((int64_t)n), 256, 0, s>>>(keys, (int64_t)n, comp);
  }
  NSB_TRY(check_launch("pack_pairs_kernel"));
  NSB_TRY(merge_sort_device(comp, n, 8, mst, merge_sort_temp_i64(n), s));
  *comp_out = comp;
  return NS_OK;
}

}  // namespace nsb

using namespace nsb;

extern "C" {

size_t ns_sort_pairs_temp_bytes_i32(size_t n) { return n <= 1 ? 0 : pairs_temp(n); }

int ns_sort_pairs_i32(int32_t* d_keys, uint32_t* d_values, size_t n, void* d_temp,
                      size_t temp_bytes, void* stream) {
  if (n > 0 && !d_keys) return NS_ERR_INVALID;
  if (n > (size_t)UINT32_MAX) return NS_ERR_INVALID;  // positions are 32-bit
  if (n <= 1) return NS_OK;
  if (!d_temp || temp_bytes < pairs_temp(n)) return NS_ERR_TEMP;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t* comp = nullptr;
  NSB_TRY(sort_composites(d_keys, n, d_temp, s, &comp));
  uint32_t* vcopy = nullptr;
  if (d_values) {
    vcopy = reinterpret_cast<uint32_t*>(static_cast<char*>(d_temp) + align_up(n * 8, 256) +
                                        align_up(merge_sort_temp_i64(n), 256));
    NSB_TRY(check_cuda(cudaMemcpyAsync(vcopy, d_values, n * 4, cudaMemcpyDeviceToDevice, s),
                       "copy values"));
  }
  {
    Prof prof(PK_CHECK, s);
    unpack_pairs_kernel<<<grid_of((int64_t)n), 256, 0, s>>>(comp, (int64_t)n, d_keys, nullptr,
                                                            vcopy, d_values);
  }
  return check_launch("unpack_pairs_kernel");
}

size_t ns_argsort_temp_bytes_i32(size_t n) { return n <= 1 ? 0 : pairs_temp(n); }

int ns_argsort_i32(const int32_t* d_keys, uint32_t* d_perm, size_t n, void* d_temp,
                   size_t temp_bytes, void* stream) {
  if (n > 0 && (!d_keys || !d_perm)) return NS_ERR_INVALID;
  if (n > (size_t)UINT32_MAX) return NS_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return NS_OK;
  if (n == 1) return check_cuda(cudaMemsetAsync(d_perm, 0, 4, s), "memset");
  if (!d_temp || temp_bytes < pairs_temp(n)) return NS_ERR_TEMP;
  int64_t* comp = nullptr;
  NSB_TRY(sort_composites(d_keys, n, d_temp, s, &comp));
  {
    Prof prof(PK_CHECK, s);
    unpack_pairs_kernel<<<grid_of((int64_t)n), 256, 0, s>>>(comp, (int64_t)n, nullptr, d_perm,
                                                            nullptr, nullptr);
  }
  return check_launch("unpack_pairs_kernel");
}

}  // extern "C"
