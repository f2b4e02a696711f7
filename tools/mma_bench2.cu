// Microbenchmark 2: the NN-scan MMA pattern -- per 256-token tile 2 fp16 MMAs
// (M=128, N=256, K=16, A/B in smem), one commit per tile, 2 TMEM buffers,
// B rotating over 6 stages; grid 1 or 148 CTAs.  Prints cycles per tile.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

__global__ void __launch_bounds__(576, 1) bench(int tiles, int rotate_b, int wait_each, int epi, int tma,
                                                const uint8_t* gsrc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar[2], tempty[2], full[6], empty[6];
  const int tid = threadIdx.x;
  for (int i = tid; i < 112 * 1024 / 16; i += blockDim.x) reinterpret_cast<int4*>(sm)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&tempty[0], 512);
    mbar_init(&tempty[1], 512);
    for (int q = 0; q < 6; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    mbar_fence_init();
  }
  if (tid < 32) tmem_alloc<512>(&taddr_s);  // (warp 0)
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;
  const int warp = tid >> 5;
  if (warp < 16) {  // epilogue warps: wait tile, load 64 columns, release the buffer
    if (epi) {
      float acc = 0.f;
      for (int i = 0; i < tiles; ++i) {
        const int bb = i & 1;
        mbar_wait(&bar[bb], (i >> 1) & 1);
        fence_after();
        uint32_t v[64];
        const uint32_t ta = T + ((uint32_t)(32 * (warp & 3)) << 16) + bb * 256 + 64 * (warp >> 2);
        tmem_ld32(ta, v);
        tmem_ld32(ta + 32, v + 32);
        tmem_ld_wait();
        fence_before();
        mbar_arrive(&tempty[bb]);
#pragma unroll
        for (int e = 0; e < 64; ++e) acc = fmaxf(acc, __uint_as_float(v[e]));
      }
      if (acc == 1234.f) out[1] = 0;
    }
  } else if (tid == 544) {  // producer
    if (tma)
      for (int i = 0; i < tiles; ++i) {
        const int q = i % 6;
        mbar_wait(&empty[q], ((i / 6) & 1) ^ 1);
        mbar_expect_tx(&full[q], 16384);
        bulk_g2s(sm + 8192 + q * 16384, gsrc + (size_t)(blockIdx.x * 16 + i % 16) * 16384, 16384, &full[q]);
      }
  } else if (tid == 512) {
    const uint32_t id = idesc_f16(128, 256);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 8192);
    long long t0 = clock64();
    for (int i = 0; i < tiles; ++i) {
      const int bb = i & 1;
      if (i >= 2 && epi) mbar_wait(&tempty[bb], ((i >> 1) - 1) & 1);       // epilogue released the buffer
      else if (i >= 2 && wait_each) mbar_wait(&bar[bb], ((i >> 1) - 1) & 1);  // buffer free (no epilogue)
      const uint32_t bs = b + (rotate_b ? (i % 6) * 16384 : 0);
      if (tma) {
        mbar_wait(&full[i % 6], (i / 6) & 1);
        fence_after();
      }
      for (int j = 0; j < 2; ++j)
        mma_bf16_ss(T + bb * 256, sdesc(a + 2 * j * 2048, 2048, 128), sdesc(bs + 2 * j * 4096, 4096, 128), id, j > 0);
      commit(&bar[bb]);
      if (tma) commit(&empty[i % 6]);
    }
    if (!epi) mbar_wait(&bar[(tiles - 1) & 1], (((tiles - 1) >> 1)) & 1);
    else mbar_wait(&tempty[(tiles - 1) & 1], (((tiles - 1) >> 1)) & 1);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;  // (tid 512)
  }
  fence_before();
  __syncthreads();
  if (tid < 32) tmem_free<512>(T);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);  // A 8 KB + 6 x 16 KB
  const int tiles = 64;
  uint8_t* g;
  cudaMalloc(&g, (size_t)148 * 16 * 16384);
  cudaMemset(g, 0, (size_t)148 * 16 * 16384);
  for (int grid : {1, 148})
    for (int rot : {1})
      for (int we : {1})
       for (int epi : {1})
        for (int tma : {0, 1}) {
        bench<<<grid, 576, 112 * 1024>>>(tiles, rot, we, epi, tma, g, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("grid=%3d epilogue=%d tma=%d : %7.1f cycles per 2-MMA tile %s\n", grid, epi, tma,
               (double)mx / tiles, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
