// pool (encoder.py:265-273) over caller-provided encoder outputs: y = U W_out
// for every valid row, elementwise max over the valid rows, zeros when no row
// is valid.  (The ranking path fuses this into the SKUT epilogue; this kernel
// serves the module-level encoder.pool / trainer.model_forward API.)
//
// One CTA per item, 256 threads = 4 row groups x 64 output columns; W_out
// (16 KB) and 32-row chunks of U staged in shared memory; f32 accumulation.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "tav2_common.cuh"

namespace tav2 {

__global__ void __launch_bounds__(256) pool_kernel(const float* U, const uint8_t* mask, const float* W, int S,
                                                   float* out) {
  __shared__ float w_s[kDModel * kDModel];
  __shared__ float u_s[32][kDModel + 1];
  __shared__ float red_s[4][kDModel];
  __shared__ int any_s;
  const int item = blockIdx.x, tid = threadIdx.x;
  const int j = tid & 63, g = tid >> 6;
  for (int i = tid; i < kDModel * kDModel; i += 256) w_s[i] = W[i];
  if (tid == 0) any_s = 0;
  const float* u = U + (size_t)item * S * kDModel;
  const uint8_t* m = mask + (size_t)item * S;
  float best = -INFINITY;
  for (int r0 = 0; r0 < S; r0 += 32) {
    __syncthreads();
    for (int i = tid; i < 32 * kDModel; i += 256) {
      const int rr = i >> 6, c = i & 63;
      u_s[rr][c] = r0 + rr < S ? u[(size_t)(r0 + rr) * kDModel + c] : 0.0f;
    }
    __syncthreads();
    for (int rr = g; rr < 32 && r0 + rr < S; rr += 4) {
      if (!m[r0 + rr]) continue;
      float acc = 0.0f;
#pragma unroll 16
      for (int k = 0; k < kDModel; ++k) acc = fmaf(u_s[rr][k], w_s[k * kDModel + j], acc);
      best = fmaxf(best, acc);
      any_s = 1;
    }
  }
  red_s[g][j] = best;
  __syncthreads();
  if (tid < kDModel) {
    const float v = fmaxf(fmaxf(red_s[0][tid], red_s[1][tid]), fmaxf(red_s[2][tid], red_s[3][tid]));
    out[(size_t)item * kDModel + tid] = any_s ? v : 0.0f;
  }
}

cudaError_t launch_pool(const float* U, const uint8_t* mask, const float* out_linear, int n, int S, float* pooled,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pool_kernel<<<n, 256, 0, s>>>(U, mask, out_linear, S, pooled);
  return cudaGetLastError();
}

}  // namespace tav2
