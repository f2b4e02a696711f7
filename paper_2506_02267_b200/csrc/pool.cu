// pool (encoder.py:265-273) over caller-provided encoder outputs: y = U W_out
// for every valid row, elementwise max over the valid rows, zeros when no row
// is valid.  (The ranking path fuses this into the SKUT epilogue; this kernel
// serves the module-level encoder.pool / trainer.model_forward API.)
//
// One CTA per item, 256 threads = 4 row groups x 64 output columns; W_out
// (16 KB) and 32-row chunks of U staged in shared memory; f32 accumulation.
#include <cuda_runtime.h>

#include <algorithm>
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

// CTR head (trainer.py:361-366) over the pooled vectors skut_tc3 wrote:
// z = [pooled | unit(c) | ctx] (104), h = ReLU(z W1 + b1), logits = h W2 + b2.
// Warp per candidate, W1 / b1 / W2 staged in shared memory once per CTA.
// The summation order is skut_tc3's former in-kernel head (two halves of 52
// inputs, even / odd accumulators, then an 8-lane tree per head), so the
// logits are bit-identical to it.  Split out of the transformer kernel: its
// ~2.9K cycles per candidate sat on tile 0 at every candidate boundary and
// delayed the next candidate's first K/V handover to the critical tile.
// spin (the pooled workspace of a fused run): no wait for the whole
// transformer grid -- each lane polls its two pooled entries until they are
// no longer kPooledEmpty (a value written by a plain store is read whole, so
// no flag and no fence is needed), so the heads of the early candidates run
// on the SMs the transformer's tail frees; the entries are reset to
// kPooledEmpty after use.  Otherwise griddep_wait up front.
constexpr int kHeadWarps = 8;
__global__ void __launch_bounds__(32 * kHeadWarps) head_kernel(Params p, Staged st, float* pooled, int n,
                                                              float* logits, int spin) {
  __shared__ float w1_s[(kDModel + kEmbed + kCtx) * kHidden];  // 26 KB
  __shared__ float w2_s[kHidden * kHeads];
  __shared__ float b1_s[kHidden];
  __shared__ float z_s[kHeadWarps][kDModel + kEmbed + kCtx];
  __shared__ float hid_s[kHeadWarps][kHidden];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (kDModel + kEmbed + kCtx) * kHidden; i += 32 * kHeadWarps) w1_s[i] = p.head_w1[i];
  for (int i = tid; i < kHidden * kHeads; i += 32 * kHeadWarps) w2_s[i] = p.head_w2[i];
  if (tid < kHidden) b1_s[tid] = p.head_b1[tid];
  griddep_launch();
  if (!spin) griddep_wait();  // pooled vectors written
  __syncthreads();
  for (int item = blockIdx.x * kHeadWarps + warp; item < n; item += gridDim.x * kHeadWarps) {
    float* z = z_s[warp];
    float* pv = pooled + (size_t)item * kDModel;
    float v0, v1;
    if (spin) {
      const volatile uint32_t* pu = reinterpret_cast<const volatile uint32_t*>(pv);
      uint32_t u0, u1;
      while ((u0 = pu[lane]) == kPooledEmpty || (u1 = pu[lane + 32]) == kPooledEmpty) __nanosleep(64);
      v0 = __uint_as_float(u0);
      v1 = __uint_as_float(u1);
      pv[lane] = __uint_as_float(kPooledEmpty);  // for the next run
      pv[lane + 32] = __uint_as_float(kPooledEmpty);
    } else {
      v0 = pv[lane];
      v1 = pv[lane + 32];
    }
    z[lane] = v0;
    z[lane + 32] = v1;
    z[kDModel + lane] = st.cand_unit[(size_t)item * kEmbed + lane];
    if (lane < kCtx) z[kDModel + kEmbed + lane] = st.ctx[st.item_req[item] * kCtx + lane];
    __syncwarp();
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {  // hidden units lane, lane + 32
      const int hu = lane + 32 * hh;
      float hp[2];
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int i = 0; i < 52; i += 2) {
          a0 = fmaf(z[52 * part + i], w1_s[(52 * part + i) * kHidden + hu], a0);
          a1 = fmaf(z[52 * part + i + 1], w1_s[(52 * part + i + 1) * kHidden + hu], a1);
        }
        hp[part] = a0 + a1;
      }
      hid_s[warp][hu] = fmaxf((hp[0] + hp[1]) + b1_s[hu], 0.0f);
    }
    __syncwarp();
    {  // lane: head (lane & 3), hidden slice 8 * (lane >> 2) .. + 8
      const int hd = lane & 3, j0 = 8 * (lane >> 2);
      float o = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) o = fmaf(hid_s[warp][j0 + j], w2_s[(j0 + j) * kHeads + hd], o);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) o += __shfl_xor_sync(0xffffffffu, o, off);
      if (lane < kHeads) logits[(size_t)item * kHeads + lane] = o + __ldg(p.head_b2 + lane);
    }
    __syncwarp();
  }
  // completion implies the transformer grid's (the next kernel's griddep_wait)
  if (spin) griddep_wait();
}

cudaError_t launch_head(const Params& p, const Staged& st, float* pooled, int n, float* logits, bool spin,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  // a warp per candidate, at most SMs / 4 CTAs whose warps then loop: fewer
  // weight stagings and fewer SM slots held by polling warps while the
  // transformer's tail runs (measured at C2: SMs / 4 -> step -0.8% against
  // one CTA per 8 candidates; SMs / 8 gives the gain back)
  const int blocks = std::min((n + kHeadWarps - 1) / kHeadWarps, std::max(device_sms() / 4, 1));
  return launch_pdl(head_kernel, dim3(blocks), dim3(32 * kHeadWarps), 0, s, p, st, pooled, n, logits, (int)spin);
}

cudaError_t launch_pool(const float* U, const uint8_t* mask, const float* out_linear, int n, int S, float* pooled,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pool_kernel<<<n, 256, 0, s>>>(U, mask, out_linear, S, pooled);
  return cudaGetLastError();
}

}  // namespace tav2
