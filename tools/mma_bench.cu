// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion time on one SM
// for the shapes the NN scan and SKUT use (data = zeros; timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I include -o /tmp/mma_bench tools/mma_bench.cu -lcuda && /tmp/mma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

// mode 0: SS (A,B smem), 1: TS (A TMEM); chain: number of independent
// accumulators the MMAs rotate over; layout: 0 no swizzle, 2 = 128B swizzle
__global__ void __launch_bounds__(128, 1) bench(int mode, int N, int chain, int layout, int reps,
                                                int sync_each, int elect_mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 * 1024 / 16; i += 128) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar, elect_mode >= 2 ? elect_mode : 1);
    mbar_fence_init();
  }
  if (tid < 32) tmem_alloc<512>(&taddr_s);
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;
  const int issuers = elect_mode >= 2 ? elect_mode : 1;  // elect_mode k >= 2: k issuing warps
  const int wq = tid >> 5;
  if (elect_mode ? wq < issuers : tid == 0) {
    const uint32_t id = idesc_bf16(128, N);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 16384);
    const uint32_t lbo_a = layout ? 16 : 128 * 16, lbo_b = layout ? 16 : N * 16;
    const uint32_t sbo = layout ? 1024 : 128;
    uint32_t dd[6];
    uint64_t ad[2], bd[2];
#pragma unroll
    for (int j = 0; j < 6; ++j) dd[j] = T + (uint32_t)((j % chain) * N) + (uint32_t)(wq * 128);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      bd[j] = sdesc(b + j * 32, lbo_b, sbo, layout);
      ad[j] = sdesc(a + j * 32, lbo_a, sbo, layout);
    }
    const uint32_t ta0 = T + 384, ta1 = T + 392;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        if (elect_mode) {
          if (mode == 0) {
            asm volatile(
                "{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;}\n" ::"r"(dd[j]), "l"(ad[j & 1]),
                "l"(bd[j & 1]), "r"(id));
          } else {
            asm volatile(
                "{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;}\n" ::"r"(dd[j]),
                "r"((j & 1) ? ta1 : ta0), "l"(bd[j & 1]), "r"(id));
          }
        } else if (mode == 0) {
          mma_bf16_ss(dd[j], ad[j & 1], bd[j & 1], id, 1);
        } else {
          mma_bf16_ts(dd[j], (j & 1) ? ta1 : ta0, bd[j & 1], id, 1);
        }
      }
      if (sync_each) {
        commit(&bar);
        mbar_wait(&bar, r & 1);
      }
    }
    if (!sync_each) {
      if (elect_mode) {
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}\n" ::"r"(smem_u32(&bar))
                     : "memory");
      } else {
        commit(&bar);
      }
      mbar_wait(&bar, 0);
    }
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  }
  fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<512>(T);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 200;
  for (int elect_mode : {1, 2, 3})
  for (int sync_each = 0; sync_each < 1; ++sync_each)
  for (int mode = 0; mode < 2; ++mode)
    for (int layout : {0})
      for (int N : {64, 128, 256})
        for (int chain : {1}) {
          if (N * chain > 128 && elect_mode >= 2) continue;
          bench<<<1, 128, 64 * 1024>>>(mode, N, chain, layout, reps, sync_each, elect_mode, d);
          cudaError_t e = cudaDeviceSynchronize();
          long long h = 0;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("%s %s %s %-9s N=%3d chain=%d : %7.1f cycles per MMA (floor %d)  %s\n", elect_mode == 1 ? "1 warp    " : elect_mode == 2 ? "2 warps   " : "3 warps   ", sync_each ? "commit+wait/6" : "stream      ", mode ? "TS" : "SS",
                 layout ? "swz128" : "noswz", N, chain, (double)h / (reps * 6 * (elect_mode >= 2 ? elect_mode : 1)), 128 * N / 256,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
          if (e != cudaSuccess) return 1;
        }
  return 0;
}
