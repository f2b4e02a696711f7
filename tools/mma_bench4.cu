// Microbenchmark 4: tcgen05.mma issue cost from one warp as a function of
// how the issue is coded (the SKUT kernels issue chains of 2..36 small-N
// MMAs from one thread):
//   variant 0: warp-converged, elect.sync inside the asm, all descriptors
//              warp-uniform (kernel parameters + compile-time offsets),
//              unrolled -> no R2UR waterfall per MMA
//   variant 1: same, but only thread 0 enters (divergent `if`) -> the
//              compiler wraps every MMA in an ELECT/R2UR.BROADCAST loop
//   variant 2: warp-converged + elect.sync, descriptors computed per MMA from
//              a per-thread register (R2UR per MMA)
// Each issues reps x 12 MMAs (M = 128, K = 16, bf16, A in TMEM) into one
// accumulator (chain) or 3 rotating accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_bench4 tools/mma_bench4.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{.reg .pred p, e; setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}

template <int N, int ROT>
__global__ void __launch_bounds__(128, 1) bench(int variant, int reps, uint32_t bsm_off, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 16; i += 128) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
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
  constexpr uint32_t id = idesc_bf16(128, N);
  const uint32_t bs = smem_u32(sm) + bsm_off;
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    if (variant == 0) {
      t0 = clock64();
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int j = 0; j < 12; ++j)
          mma_ts_elect(T + (j % ROT) * N, T + 448 + 8 * (j & 1), sdesc(bs + 256 * (j & 3), N * 16, 128), id, 1);
      }
      asm volatile(
          "{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}\n" ::"r"(smem_u32(&bar))
          : "memory");
      mbar_wait(&bar, 0);
      t1 = clock64();
    } else if (variant == 1) {
      if (tid == 0) {
        t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
          for (int j = 0; j < 12; ++j)
            mma_bf16_ts(T + (j % ROT) * N, T + 448 + 8 * (j & 1), sdesc(bs + 256 * (j & 3), N * 16, 128), id, 1);
        }
        commit(&bar);
        mbar_wait(&bar, 0);
        t1 = clock64();
      }
    } else {
      const uint32_t lane_b = bs + 0 * tid;  // per-thread register copy
      uint32_t bb = lane_b;
      asm volatile("mov.b32 %0, %0;" : "+r"(bb));
      t0 = clock64();
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int j = 0; j < 12; ++j)
          mma_ts_elect(T + (j % ROT) * N, T + 448 + 8 * (j & 1), sdesc(bb + 256 * (j & 3), N * 16, 128), id, 1);
      }
      asm volatile(
          "{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}\n" ::"r"(smem_u32(&bar))
          : "memory");
      mbar_wait(&bar, 0);
      t1 = clock64();
    }
    if (tid == 0) out[0] = t1 - t0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(T);
}

template <int N, int ROT>
void run(long long* d, int variant) {
  const int reps = 64;
  cudaFuncSetAttribute(bench<N, ROT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  bench<N, ROT><<<1, 128, 64 * 1024>>>(variant, reps, 16384, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("variant %d N=%3d accumulators=%d : %6.1f cyc/MMA (floor %d) %s\n", variant, N, ROT,
         (double)h / (reps * 12), 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int v = 0; v < 3; ++v) {
    run<32, 1>(d, v);
    run<64, 1>(d, v);
    run<64, 3>(d, v);
    run<128, 1>(d, v);
    run<128, 3>(d, v);
    run<256, 1>(d, v);
  }
  return 0;
}
