// Microbenchmark 5: the SKUT P.V / P.a issue pattern -- a group of G
// tcgen05.mma (kind::f16, M = 128, N = 64, K = 16, A in TMEM at advancing
// column offsets, 3 per k-step as in the split products) into one
// accumulator, then commit + wait; cycles from the first issue to the
// mbarrier completion, per B-operand layout:
//   0: K-major B (LBO = N*16, SBO = 128)
//   1: MN-major B, core matrices k-group-major (LBO = 1024, SBO = 128): skut_tc3 V'
//   2: MN-major B, core matrices n-group-major (LBO = 128, SBO = K*16): skut_tc4 keys
// Also the plain latency of one MMA + commit + wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench5 tools/mma_bench5.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

__global__ void __launch_bounds__(256, 1) bench(int layout, int ksteps, int reps, int noise, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 16; i += 256) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;
  __shared__ volatile int stop;
  if (tid == 0) stop = 0;
  __syncthreads();
  if (warp >= 4 && noise) {  // other warps: TMEM loads (noise 1) or FFMA chains (noise 2) meanwhile
    const uint32_t ta = T + ((uint32_t)(32 * (warp & 3)) << 16) + 384;
    float acc = 0.f;
    uint32_t v[32];
    while (!stop) {
      if (noise == 1) {
        tmem_ld32(ta, v);
        tmem_ld_wait();
        acc += __uint_as_float(v[tid & 31]);
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) acc = fmaf(acc, 1.0001f, 0.5f);
      }
    }
    if (acc == 12345.f) out[1] = 1;
  }
  if (warp == 0) {
    const uint32_t id = idesc_bf16(128, 64, 0, layout != 0);
    const uint32_t bhi = smem_u32(sm), blo = smem_u32(sm + 48 * 1024);
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      __syncwarp();
      const long long t0 = clock64();
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        if (j >= ksteps) break;
        uint64_t bh, bl;
        if (layout == 0) {
          bh = sdesc(bhi + 2 * j * 64 * 16, 64 * 16, 128);
          bl = sdesc(blo + 2 * j * 64 * 16, 64 * 16, 128);
        } else if (layout == 1) {
          bh = sdesc(bhi + 2 * j * 1024, 1024, 128);
          bl = sdesc(blo + 2 * j * 1024, 1024, 128);
        } else {
          bh = sdesc(bhi + 2 * j * 128, 128, 192 * 16);
          bl = sdesc(blo + 2 * j * 128, 128, 192 * 16);
        }
        mma_bf16_ts_w(T + 256, T + 16 * j, bh, id, j > 0);
        mma_bf16_ts_w(T + 256, T + 16 * j, bl, id, 1);
        mma_bf16_ts_w(T + 256, T + 16 * j + 8, bh, id, 1);
      }
      commit_w(&bar);
      mbar_wait(&bar, r & 1);
      tot += clock64() - t0;
    }
    if (tid == 0) out[0] = tot / reps;
    if (tid == 0) stop = 1;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(T);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int noise = 0; noise < 3; ++noise)
  for (int layout = 0; layout < 3; layout += 1)
    for (int ks : {1, 4, 6, 12}) {
      bench<<<1, 256, 96 * 1024>>>(layout, ks, 64, noise, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("noise %d layout %d  k-steps %2d (%2d MMAs, N=64): %6lld cycles issue->complete  (%5.1f per MMA) %s\n", noise, layout, ks,
             3 * ks, h, (double)h / (3 * ks), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  return 0;
}
