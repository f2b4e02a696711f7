// Microbenchmark: tcgen05.ld (TMEM -> registers) bandwidth on one SM with
// W warps (lane quarter = warp % 4), each loading 32x32b.x32 (4 KB) per op.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

__global__ void bench(int reps, int per_wait, long long* out, float* sink) {
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + 32 * ((warp >> 2) & 7);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t v0[32], v1[32], v2[32], v3[32];
    tmem_ld32(T, v0);
    if (per_wait > 1) tmem_ld32(T + 64, v1);
    if (per_wait > 2) {
      tmem_ld32(T + 128, v2);
      tmem_ld32(T + 192, v3);
    }
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += __uint_as_float(v0[i]);
    if (per_wait > 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(v1[i]);
    }
    if (per_wait > 2) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(v2[i]) + __uint_as_float(v3[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[0] = t1 - t0;
  if (acc == 12345.f) sink[tid] = acc;
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(taddr_s);
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4 * 1024);
  const int reps = 400;
  for (int warps : {1, 4, 8, 16})
    for (int pw : {1, 2, 4}) {
      bench<<<1, 32 * warps>>>(reps, pw, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)reps * pw * warps * 4096;
      printf("warps=%2d loads/wait=%d : %7.1f bytes/cycle  (%6.1f cycles per 4 KB load per warp) %s\n", warps, pw,
             bytes / h, (double)h / (reps * pw), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
