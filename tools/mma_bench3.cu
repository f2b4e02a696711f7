// Microbenchmark 3: what limits back-to-back tcgen05.mma (kind::f16, A in
// TMEM, M = 128) at the small N the SKUT kernels use.
//   (a) one issuing thread, `chain` independent accumulators rotated per MMA
//       (chain = 1: every MMA accumulates into the same D)
//   (b) several issuing warps (warp mask), each on its own accumulator --
//       same SM sub-partition (warps 0, 4) vs different ones (0, 1)
//   (c) FFMA filler between MMAs in the issuing thread: is the issue slot
//       blocking the warp or only the tensor pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_bench3 tools/mma_bench3.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

__global__ void __launch_bounds__(256, 1) bench(int N, int chain, unsigned warp_mask, int reps, int filler,
                                                int ss, long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar[8];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 16; i += 256) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
  if (tid < 8) mbar_init(&bar[tid], 1);
  if (tid == 0) mbar_fence_init();
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;
  int slot = __popc(warp_mask & ((1u << warp) - 1));  // this warp's accumulator set
  if (((warp_mask >> warp) & 1u) && (tid & 31) == 0) {
    const uint32_t id = idesc_bf16(128, N);
    const uint32_t b = smem_u32(sm + 16384), a = smem_u32(sm);
    const uint64_t bd = sdesc(b, N * 16, 128);
    const uint64_t ad = sdesc(a, 128 * 16, 128);
    const uint32_t ta = T + 448;  // A operand columns (bf16 K=16: 8 columns)
    const uint32_t dbase = T + (uint32_t)(slot * chain * N);
    float f0 = 1.0f + tid, f1 = 2.0f;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int j = 0; j < chain; ++j) {
        if (ss) mma_bf16_ss(dbase + j * N, ad, bd, id, 1);
        else mma_bf16_ts(dbase + j * N, ta, bd, id, 1);
        for (int f = 0; f < filler; ++f) f0 = fmaf(f0, f1, 0.5f);
      }
    }
    const long long t_issue = clock64() - t0;
    commit(&bar[slot]);
    mbar_wait(&bar[slot], 0);
    long long t1 = clock64();
    out[2 * warp] = t1 - t0;
    out[2 * warp + 1] = t_issue;
    sink[tid] = f0;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(T);
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 8 * 16);
  cudaMalloc(&sink, 4 * 256);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 96;
  auto run = [&](int N, int chain, unsigned mask, int filler, int ss) {
    cudaMemset(d, 0, 8 * 16);
    bench<<<1, 256, 64 * 1024>>>(N, chain, mask, reps, filler, ss, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, d, 8 * 16, cudaMemcpyDeviceToHost);
    long long mx = 0, mi = 0;
    int nw = 0;
    for (int w = 0; w < 8; ++w)
      if ((mask >> w) & 1u) {
        mx = h[2 * w] > mx ? h[2 * w] : mx;
        mi = h[2 * w + 1] > mi ? h[2 * w + 1] : mi;
        ++nw;
      }
    const double per = (double)mx / (reps * chain * nw);
    printf("%s N=%3d chain=%d warps=0x%02x filler=%3d : %6.1f cyc/MMA (SM-wide), per-warp issue %6.1f cyc/MMA, floor %d %s\n",
           ss ? "SS" : "TS", N, chain, mask, filler, per, (double)mi / (reps * chain), 128 * N / 256,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int ss = 0; ss < 2; ++ss)
    for (int N : {32, 64, 128, 256})
      for (int chain : {1, 2, 3, 4}) {
        if (N * chain > 448) continue;
        run(N, chain, 0x1, 0, ss);
      }
  for (int N : {32, 64, 128})
    for (unsigned mask : {0x3u, 0x11u, 0xfu, 0x33u, 0xffu}) {
      if (N * __builtin_popcount(mask) > 448) continue;
      run(N, 1, mask, 0, 0);
    }
  for (int filler : {0, 16, 32, 64, 128}) run(64, 1, 0x1, filler, 0);
  for (int filler : {0, 16, 32, 64, 128}) run(64, 2, 0x1, filler, 0);
  return 0;
}
