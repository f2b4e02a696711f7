// Microbenchmark of the SKUT softmax exp loop (skut_tc3.cu P3b): per warp,
// NCH chunks of 16 TMEM columns: ld16 (double-buffered) -> exp2(s - m) ->
// mask -> row sum -> bf16 hi/lo split -> 2 x st8 in place.  Variants switch
// off the stores / the ex2 to find what bounds the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/exp_bench tools/exp_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2506_02267_b200/csrc/tc_common.cuh"

using namespace tav2::tc;

template <bool ST, bool EX, bool LD>
__global__ void bench(int reps, int nch, long long* out, float* sink) {
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t cs = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + 256 * ((warp >> 2) & 1);
  const float2 nmb = make_float2(-1.0f, -1.0f);
  float2 l2 = make_float2(0.f, 0.f);
  const uint32_t vmask = 0xfff7u ^ (uint32_t)tid;
  __syncthreads();
  long long t0 = clock64();
  for (int rr = 0; rr < reps; ++rr) {
    uint32_t sa[16], sb[16];
    if (LD) tmem_ld16(cs, sa);
    else
      for (int i = 0; i < 16; ++i) sa[i] = __float_as_uint(0.01f * i);
    for (int j = 0; j < nch; j += 2) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int jj = j + u;
        if (jj >= nch) break;
        uint32_t* cur = u == 0 ? sa : sb;
        uint32_t* nxt = u == 0 ? sb : sa;
        if (LD) {
          tmem_ld_wait();
          if (jj + 1 < nch) tmem_ld16(cs + 16 * (jj + 1), nxt);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) nxt[i] = cur[i] ^ 1u;
        }
        const uint32_t vm = vmask >> (jj & 7);
        float pv[16];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float2 d = __fadd2_rn(make_float2(__uint_as_float(cur[e]), __uint_as_float(cur[e + 1])), nmb);
          float p0, p1;
          if (EX) {
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(d.x));
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(d.y));
          } else {
            p0 = d.x * 1.5f;
            p1 = d.y * 1.5f;
          }
          pv[e] = ((vm >> e) & 1u) ? p0 : 0.0f;
          pv[e + 1] = ((vm >> (e + 1)) & 1u) ? p1 : 0.0f;
          l2 = __fadd2_rn(l2, make_float2(pv[e], pv[e + 1]));
        }
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) split_pair_t(pv[2 * i], pv[2 * i + 1], hi[i], lo[i]);
        if (ST) {
          tmem_st8(cs + 16 * jj, hi);
          tmem_st8(cs + 16 * jj + 8, lo);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) l2.x += __uint_as_float(hi[i] ^ lo[i]);
        }
      }
    }
    if (ST) tmem_st_wait();
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[0] = t1 - t0;
  if (l2.x + l2.y == 12345.f) sink[tid] = l2.x;
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(taddr_s);
}

template <bool ST, bool EX, bool LD>
void run(const char* name, int warps, long long* d, float* sink) {
  const int reps = 200, nch = 12;
  bench<ST, EX, LD><<<1, 32 * warps>>>(reps, nch, d, sink);
  cudaDeviceSynchronize();
  bench<ST, EX, LD><<<1, 32 * warps>>>(reps, nch, d, sink);
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s warps %d: %7.1f cycles / chunk (per warp)\n", name, warps, (double)c / (reps * nch));
}

int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 4096 * 4);
  for (int w : {4, 8}) {
    run<true, true, true>("full", w, d, sink);
    run<false, true, true>("no st", w, d, sink);
    run<true, false, true>("no ex2", w, d, sink);
    run<true, true, false>("no ld", w, d, sink);
    run<false, false, false>("alu only", w, d, sink);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
}
