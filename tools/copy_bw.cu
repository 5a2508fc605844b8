// Streaming-copy bandwidth on this B200: what a read-once/write-once pass
// (the merge pass's byte pattern) can reach.  nvcc -O3 -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_v4(const int4* __restrict__ a, int4* __restrict__ b, long n4) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
// each CTA copies one contiguous tile with 128-bit loads held in registers
template <int PER>
__global__ void copy_tile(const int4* __restrict__ a, int4* __restrict__ b, long n4) {
  const long base = (long)blockIdx.x * blockDim.x * PER;
  int4 v[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const long i = base + (long)u * blockDim.x + threadIdx.x;
    if (i < n4) v[u] = __ldcs(a + i);
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const long i = base + (long)u * blockDim.x + threadIdx.x;
    if (i < n4) __stcs(b + i, v[u]);
  }
}

int main() {
  const long n = 1L << 30;  // int32 keys
  const long n4 = n / 4;
  int4 *a, *b;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaMemset(a, 1, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s %.3f ms  %.1f GB/s (8n bytes)\n", name, ms, 8.0 * n / (ms * 1e-3) / 1e9);
  };
  run("grid-stride v4, 148*8x256", [&] { copy_v4<<<sms * 8, 256>>>(a, b, n4); });
  run("grid-stride v4, 148*16x512", [&] { copy_v4<<<sms * 16, 512>>>(a, b, n4); });
  run("tile 256x8 int4", [&] { copy_tile<8><<<(unsigned)((n4 + 2047) / 2048), 256>>>(a, b, n4); });
  run("tile 256x16 int4", [&] { copy_tile<16><<<(unsigned)((n4 + 4095) / 4096), 256>>>(a, b, n4); });
  run("cudaMemcpyD2D", [&] { cudaMemcpyAsync(b, a, n * 4, cudaMemcpyDeviceToDevice); });
  return 0;
}
