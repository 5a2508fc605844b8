// multigpu.cu — the multi-GPU layer behind ONE host thread (SURVEY.md §8(b)
// "ns_sample_sort_multi_i32(int ngpu, ncclComm_t* comms, int32_t** d_shards,
// ...)", §8(e)).
//
// The reference is single-process and single-threaded; its
// entry shape is optimized_merge_sort(std::span<T>, cfg) (hybrid.hpp:156-177)
// over one array.  Here one array of BASELINE config 5 is sharded over
// ngpu devices and sorted by regular-sampling sample sort (PSRS):
//   1. local merge sort of every shard (the 6To8 network base case);
//   2. s = min(255, shard) regular samples per shard;
//   3. all-gather of the samples (ncclAllGather, or peer copies);
//   4. every device sorts the g*s samples and picks the same g-1 splitters;
//   5. bucket bounds of every sorted shard (lower_bound: keys equal to a
//      splitter go to the upper bucket); the g x (g+1) bounds come to the
//      host (the only synchronisation: they size the exchange);
//   6. exchange:
//        NS_EXCHANGE_NCCL: grouped ncclSend / ncclRecv (all-to-all over
//          NVLink / NVSwitch) into d_out, then a g-way merge of the received
//          runs (ns_merge_runs_i32);
//        NS_EXCHANGE_P2P: no receive step — device d merges the runs destined
//          to it straight out of its peers' HBM (peer access over NVLink) with
//          the pointer-pair merge (ns_merge_pairs_i32), which fuses the
//          all-to-all into the first merge round; later rounds are local.
// Device d ends with the d-th key range of the sorted array in d_out[d].
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, reusing one already in
// the process, e.g. PyTorch's), so single-GPU users do not depend on it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace nsb {

// ---- NCCL, resolved at run time --------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // one already loaded wins
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      return fp != nullptr;
    };
    api.ok = sym(api.GroupStart, "ncclGroupStart") && sym(api.GroupEnd, "ncclGroupEnd") &&
             sym(api.Send, "ncclSend") && sym(api.Recv, "ncclRecv") &&
             sym(api.AllGather, "ncclAllGather") && sym(api.CommInitAll, "ncclCommInitAll") &&
             sym(api.CommDestroy, "ncclCommDestroy") && sym(api.GetErrorString, "ncclGetErrorString");
  });
  return api;
}

static int nccl_check(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return NS_OK;
  set_last_error(where, cudaErrorUnknown);
  return NS_ERR_NCCL;
}

// ---- layout of one device's scratch ------------------------------------------
constexpr int kSamplesPerShard = 255;

struct MultiTemp {
  void* sort_temp;
  size_t sort_bytes;
  int32_t* samples;  // g * s (all-gathered)
  int32_t* splitters;
  int64_t* bounds;   // g + 1
  void* merge_temp;
  size_t merge_bytes;
};

static size_t multi_merge_bytes(int g, size_t cap) {
  const int np = std::max(1, (g + 1) / 2);
  return std::max({ns_merge_runs_temp_bytes(cap, g), ns_merge_runs_temp_bytes(cap, np),
                   ns_merge_pairs_temp_bytes((int64_t)cap, np)});
}

static size_t multi_temp_bytes(int g, size_t shard, size_t cap) {
  return align_up(merge_sort_temp(shard), 256) + align_up((size_t)g * kSamplesPerShard * 4, 256) +
         align_up((size_t)g * 4, 256) + align_up((size_t)(g + 1) * 8, 256) +
         align_up(multi_merge_bytes(g, cap), 256);
}

static MultiTemp carve_multi(void* base, int g, size_t shard, size_t cap) {
  char* p = static_cast<char*>(base);
  MultiTemp t;
  t.sort_temp = p;
  t.sort_bytes = merge_sort_temp(shard);
  p += align_up(t.sort_bytes, 256);
  t.samples = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)g * kSamplesPerShard * 4, 256);
  t.splitters = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)g * 4, 256);
  t.bounds = reinterpret_cast<int64_t*>(p);
  p += align_up((size_t)(g + 1) * 8, 256);
  t.merge_temp = p;
  t.merge_bytes = multi_merge_bytes(g, cap);
  return t;
}

// restores the caller's current device on scope exit
struct DeviceGuard {
  int prev = 0;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

__global__ void fill_kernel(int32_t* p, int n, int32_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace nsb

using namespace nsb;

extern "C" {

int ns_nccl_available(void) { return nccl().ok ? 1 : 0; }

int ns_nccl_comms_init_all(int ngpu, const int* devices, ns_nccl_comm* comms) {
  if (ngpu < 1 || !devices || !comms) return NS_ERR_INVALID;
  const NcclApi& api = nccl();
  if (!api.ok) return NS_ERR_NCCL;
  DeviceGuard guard;
  return nccl_check(api.CommInitAll(reinterpret_cast<ncclComm_t*>(comms), ngpu, devices),
                    "ncclCommInitAll");
}

int ns_nccl_comms_destroy(int ngpu, ns_nccl_comm* comms) {
  if (ngpu < 1 || !comms) return NS_ERR_INVALID;
  const NcclApi& api = nccl();
  if (!api.ok) return NS_ERR_NCCL;
  for (int g = 0; g < ngpu; ++g)
    if (comms[g]) {
      NSB_TRY(nccl_check(api.CommDestroy(reinterpret_cast<ncclComm_t>(comms[g])), "ncclCommDestroy"));
      comms[g] = nullptr;
    }
  return NS_OK;
}

int ns_sample_sort_plan(int ngpu, const int64_t* bounds, int64_t* recv_offsets,
                        int64_t* recv_totals) {
  if (ngpu < 1 || !bounds || !recv_offsets || !recv_totals) return NS_ERR_INVALID;
  const int g = ngpu;
  for (int src = 0; src < g; ++src) {
    const int64_t* b = bounds + (size_t)src * (g + 1);
    if (b[0] != 0) return NS_ERR_INVALID;
    for (int k = 0; k < g; ++k)
      if (b[k + 1] < b[k]) return NS_ERR_INVALID;
  }
  for (int dst = 0; dst < g; ++dst) {
    int64_t* ro = recv_offsets + (size_t)dst * (g + 1);
    ro[0] = 0;
    for (int src = 0; src < g; ++src) {
      const int64_t* b = bounds + (size_t)src * (g + 1);
      ro[src + 1] = ro[src] + (b[dst + 1] - b[dst]);
    }
    recv_totals[dst] = ro[g];
  }
  return NS_OK;
}

size_t ns_sample_sort_multi_temp_bytes(int ngpu, size_t shard_keys, size_t out_capacity) {
  if (ngpu < 1) return 0;
  return multi_temp_bytes(ngpu, shard_keys, out_capacity);
}

int ns_sample_sort_multi_i32(int ngpu, const int* devices, ns_nccl_comm* comms, int exchange,
                             int32_t* const* d_shards, const size_t* counts, int32_t* const* d_out,
                             size_t out_capacity, size_t* out_counts, uint32_t width_mask,
                             int varsort_max, void* const* d_temps, size_t temp_bytes,
                             void* const* streams) {
  const int g = ngpu;
  if (g < 1 || g > 64 || !devices || !d_shards || !counts || !d_out || !out_counts || !d_temps ||
      !streams)
    return NS_ERR_INVALID;
  if (exchange != NS_EXCHANGE_NCCL && exchange != NS_EXCHANGE_P2P) return NS_ERR_INVALID;
  if (exchange == NS_EXCHANGE_NCCL && (!comms || !nccl().ok)) return comms ? NS_ERR_NCCL : NS_ERR_INVALID;
  size_t shard_max = 0;
  for (int d = 0; d < g; ++d) {
    if (counts[d] && !d_shards[d]) return NS_ERR_INVALID;
    shard_max = std::max(shard_max, counts[d]);
  }
  if (temp_bytes < multi_temp_bytes(g, shard_max, out_capacity)) return NS_ERR_TEMP;
  DeviceGuard guard;
  auto S = [&](int d) { return static_cast<cudaStream_t>(streams[d]); };
  std::vector<MultiTemp> tm(g);
  const int s = kSamplesPerShard;

  // 1-2. local sort and regular samples (an empty shard contributes INT_MAX)
  for (int d = 0; d < g; ++d) {
    NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
    tm[d] = carve_multi(d_temps[d], g, shard_max, out_capacity);
    NSB_TRY(ns_merge_sort_i32(d_shards[d], counts[d], width_mask, varsort_max, tm[d].sort_temp,
                              tm[d].sort_bytes, S(d)));
    int32_t* mine = tm[d].samples + (size_t)d * s;
    if (counts[d]) {
      NSB_TRY(ns_regular_samples_i32(d_shards[d], counts[d], s, mine, S(d)));
    } else {
      fill_kernel<<<1, 256, 0, S(d)>>>(mine, s, INT32_MAX);
      NSB_TRY(check_launch("fill_kernel"));
    }
  }
  // 3. all-gather of the samples
  if (exchange == NS_EXCHANGE_NCCL) {
    const NcclApi& api = nccl();
    NSB_TRY(nccl_check(api.GroupStart(), "ncclGroupStart"));
    for (int d = 0; d < g; ++d)
      NSB_TRY(nccl_check(api.AllGather(tm[d].samples + (size_t)d * s, tm[d].samples, (size_t)s,
                                       ncclInt32, reinterpret_cast<ncclComm_t>(comms[d]), S(d)),
                         "ncclAllGather"));
    NSB_TRY(nccl_check(api.GroupEnd(), "ncclGroupEnd"));
  } else {
    for (int d = 0; d < g; ++d) NSB_TRY(check_cuda(cudaStreamSynchronize(S(d)), "cudaStreamSynchronize"));
    for (int d = 0; d < g; ++d) {
      NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
      for (int p = 0; p < g; ++p)
        if (p != d)
          NSB_TRY(check_cuda(cudaMemcpyPeerAsync(tm[d].samples + (size_t)p * s, devices[d],
                                                 tm[p].samples + (size_t)p * s, devices[p],
                                                 (size_t)s * 4, S(d)),
                             "cudaMemcpyPeerAsync"));
    }
  }
  // 4-5. splitters and bucket bounds; the bounds come to the host
  std::vector<int64_t> bounds((size_t)g * (g + 1));
  for (int d = 0; d < g; ++d) {
    NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
    if (g > 1)
      NSB_TRY(ns_select_splitters_i32(tm[d].samples, g * s, g, tm[d].splitters, S(d)));
    NSB_TRY(ns_bucket_bounds_i32(d_shards[d], counts[d], g > 1 ? tm[d].splitters : nullptr, g,
                                 tm[d].bounds, S(d)));
    NSB_TRY(check_cuda(cudaMemcpyAsync(bounds.data() + (size_t)d * (g + 1), tm[d].bounds,
                                       (size_t)(g + 1) * 8, cudaMemcpyDeviceToHost, S(d)),
                       "cudaMemcpyAsync(bounds)"));
  }
  for (int d = 0; d < g; ++d) {
    NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
    NSB_TRY(check_cuda(cudaStreamSynchronize(S(d)), "cudaStreamSynchronize"));
  }
  std::vector<int64_t> roff((size_t)g * (g + 1)), rtot(g);
  NSB_TRY(ns_sample_sort_plan(g, bounds.data(), roff.data(), rtot.data()));
  bool fits = true;
  for (int d = 0; d < g; ++d) {
    out_counts[d] = (size_t)rtot[d];
    fits = fits && (size_t)rtot[d] <= out_capacity;
  }
  if (!fits) return NS_ERR_TEMP;
  auto cnt = [&](int src, int dst) {
    return bounds[(size_t)src * (g + 1) + dst + 1] - bounds[(size_t)src * (g + 1) + dst];
  };
  auto off = [&](int src, int dst) { return bounds[(size_t)src * (g + 1) + dst]; };

  // 6. exchange + merge
  if (exchange == NS_EXCHANGE_NCCL) {
    const NcclApi& api = nccl();
    NSB_TRY(nccl_check(api.GroupStart(), "ncclGroupStart"));
    for (int d = 0; d < g; ++d) {
      const ncclComm_t cm = reinterpret_cast<ncclComm_t>(comms[d]);
      for (int p = 0; p < g; ++p) {
        if (cnt(d, p))
          NSB_TRY(nccl_check(api.Send(d_shards[d] + off(d, p), (size_t)cnt(d, p), ncclInt32, p, cm,
                                      S(d)),
                             "ncclSend"));
        if (cnt(p, d))
          NSB_TRY(nccl_check(api.Recv(d_out[d] + roff[(size_t)d * (g + 1) + p], (size_t)cnt(p, d),
                                      ncclInt32, p, cm, S(d)),
                             "ncclRecv"));
      }
    }
    NSB_TRY(nccl_check(api.GroupEnd(), "ncclGroupEnd"));
    for (int d = 0; d < g; ++d) {
      NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
      NSB_TRY(ns_merge_runs_i32(d_out[d], roff.data() + (size_t)d * (g + 1), g, tm[d].merge_temp,
                                tm[d].merge_bytes, S(d)));
    }
  } else {
    // peer access between distinct devices (virtual ranks on one device need none)
    for (int d = 0; d < g; ++d)
      for (int p = 0; p < g; ++p)
        if (devices[p] != devices[d]) {
          NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[p], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else NSB_TRY(check_cuda(e, "cudaDeviceEnablePeerAccess"));
        }
    const int np = (g + 1) / 2;
    for (int d = 0; d < g; ++d) {
      NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
      std::vector<const int32_t*> ap(np), bp(np);
      std::vector<int64_t> al(np), bl(np), po(np + 1, 0);
      for (int q = 0; q < np; ++q) {
        const int pa = 2 * q, pb = 2 * q + 1;
        ap[q] = d_shards[pa] + off(pa, d);
        al[q] = cnt(pa, d);
        bp[q] = pb < g ? d_shards[pb] + off(pb, d) : ap[q] + al[q];
        bl[q] = pb < g ? cnt(pb, d) : 0;
        po[q + 1] = po[q] + al[q] + bl[q];
      }
      NSB_TRY(ns_merge_pairs_i32(ap.data(), al.data(), bp.data(), bl.data(), np, d_out[d],
                                 tm[d].merge_temp, tm[d].merge_bytes, S(d)));
      if (np > 1)
        NSB_TRY(ns_merge_runs_i32(d_out[d], po.data(), np, tm[d].merge_temp, tm[d].merge_bytes,
                                  S(d)));
    }
  }
  // every device reads its peers' shards (P2P) or its send buffers are in
  // flight (NCCL): the caller's buffers must stay untouched until all is done
  for (int d = 0; d < g; ++d) {
    NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
    NSB_TRY(check_cuda(cudaStreamSynchronize(S(d)), "cudaStreamSynchronize"));
  }
  return NS_OK;
}

// ---- shard by array (base-case batch, segmented batch) -----------------------
int ns_shard_batch_plan(const uint32_t* h_offsets, size_t num_arrays, int nshards,
                        size_t* array_begin) {
  if (nshards < 1 || !array_begin || (num_arrays && !h_offsets)) return NS_ERR_INVALID;
  array_begin[0] = 0;
  const uint64_t total = num_arrays ? h_offsets[num_arrays] - h_offsets[0] : 0;
  size_t a = 0;
  for (int k = 1; k < nshards; ++k) {
    // first array whose start reaches k/nshards of the keys (arrays stay whole)
    const uint64_t target = h_offsets ? h_offsets[0] + total * (uint64_t)k / (uint64_t)nshards : 0;
    while (a < num_arrays && h_offsets[a] < target) ++a;
    array_begin[k] = std::max(a, array_begin[k - 1]);
  }
  array_begin[nshards] = num_arrays;
  return NS_OK;
}

int ns_sort_small_batch_multi_i32(int ngpu, const int* devices, int32_t* const* d_keys,
                                  const uint32_t* const* d_offsets, const size_t* num_arrays,
                                  int* const* d_status, void* const* streams) {
  if (ngpu < 1 || !devices || !d_keys || !d_offsets || !num_arrays || !d_status || !streams)
    return NS_ERR_INVALID;
  DeviceGuard guard;
  for (int d = 0; d < ngpu; ++d) {
    NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
    NSB_TRY(ns_sort_small_batch_async_i32(d_keys[d], d_offsets[d], num_arrays[d], d_status[d],
                                          streams[d]));
  }
  return NS_OK;
}

int ns_segmented_sort_multi_i32(int ngpu, const int* devices, int32_t* const* d_keys,
                                const size_t* num_segments, size_t seg_len, int algorithm,
                                uint32_t width_mask, int varsort_max, void* const* d_temps,
                                const size_t* temp_bytes, void* const* streams) {
  if (ngpu < 1 || !devices || !d_keys || !num_segments || !d_temps || !temp_bytes || !streams)
    return NS_ERR_INVALID;
  DeviceGuard guard;
  for (int d = 0; d < ngpu; ++d) {
    NSB_TRY(check_cuda(cudaSetDevice(devices[d]), "cudaSetDevice"));
    NSB_TRY(ns_segmented_sort_i32(d_keys[d], num_segments[d], seg_len, algorithm, width_mask,
                                  varsort_max, d_temps[d], temp_bytes[d], streams[d]));
  }
  return NS_OK;
}

}  // extern "C"
