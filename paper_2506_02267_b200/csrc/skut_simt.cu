// fp32 parity mode of the scoring path: gather + Eq. 4 encode (K3), the
// 2-layer pre-norm causal transformer (K4) and linear + masked max-pool +
// CTR head (K5), SIMT fp32, one block per candidate.
//
// Reference: encoder.py:161-188 (encode_batch), :196-211 (layer_norm,
// masked_softmax), :314-462 (forward_fused), :265-273 (pool);
// trainer.py:354-366 (batched pool + head).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "encode.cuh"
#include "tav2_common.cuh"

namespace tav2 {

constexpr int kSkutThreads = 256;  // one row per thread up to S = 256
constexpr int kSkutWarps = kSkutThreads / 32;
constexpr float kLnEps = 1e-5f;  // encoder.py:19

// out[j] = sum_i a[i] * W[i, j]   (W row-major [IN, OUT] f32 in global)
template <int IN, int OUT>
__device__ __forceinline__ void matvec(const float* a, const float* __restrict__ W, float* out) {
#pragma unroll
  for (int j = 0; j < OUT; ++j) out[j] = 0.0f;
#pragma unroll 4
  for (int i = 0; i < IN; ++i) {
    const float ai = a[i];
    const float4* w = reinterpret_cast<const float4*>(W + i * OUT);
#pragma unroll
    for (int j = 0; j < OUT / 4; ++j) {
      float4 v = __ldg(w + j);
      out[4 * j] = fmaf(ai, v.x, out[4 * j]);
      out[4 * j + 1] = fmaf(ai, v.y, out[4 * j + 1]);
      out[4 * j + 2] = fmaf(ai, v.z, out[4 * j + 2]);
      out[4 * j + 3] = fmaf(ai, v.w, out[4 * j + 3]);
    }
  }
}

// encoder.py:196-200 (biased variance, eps 1e-5)
__device__ __forceinline__ void layer_norm64(const float* x, const float* __restrict__ g,
                                             const float* __restrict__ b, float* y) {
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < kDModel; ++j) s += x[j];
  const float mu = s / 64.0f;
  float v = 0.0f;
#pragma unroll
  for (int j = 0; j < kDModel; ++j) {
    float c = x[j] - mu;
    v = fmaf(c, c, v);
  }
  const float den = sqrtf(v / 64.0f + kLnEps);
#pragma unroll
  for (int j = 0; j < kDModel; ++j) y[j] = (x[j] - mu) / den * __ldg(g + j) + __ldg(b + j);
}

__device__ __forceinline__ void load64(const float* src, float* dst) {
  const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float4 v = s[j];
    dst[4 * j] = v.x; dst[4 * j + 1] = v.y; dst[4 * j + 2] = v.z; dst[4 * j + 3] = v.w;
  }
}
__device__ __forceinline__ void store64(float* dst, const float* src) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int j = 0; j < 16; ++j) d[j] = make_float4(src[4 * j], src[4 * j + 1], src[4 * j + 2], src[4 * j + 3]);
}

// ---------------------------------------------------------------------------
// Encode kernel (tav2_encode parity entry): one thread per (item, slot).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) encode_kernel(Staged st, NNCfg nn, Params p,
                                                     const int32_t* idx, float* F, uint8_t* mask) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= st.n_items * nn.seq_len) return;
  int item = g / nn.seq_len, r = g % nn.seq_len;
  int tok = slot_token(st, nn, idx, item, r);
  float f[kDModel];
  if (tok >= 0) {
    encode_row(st, p, item, tok, r, f);
  } else {
#pragma unroll
    for (int j = 0; j < kDModel; ++j) f[j] = 0.0f;
  }
  store64(F + (size_t)g * kDModel, f);
  mask[g] = tok >= 0;
}

cudaError_t launch_encode(const Staged& st, const NNCfg& nn, const Params& p, const int32_t* idx,
                          float* F, uint8_t* mask, cudaStream_t s) {
  int n = st.n_items * nn.seq_len;
  if (n == 0) return cudaSuccess;
  encode_kernel<<<(n + 127) / 128, 128, 0, s>>>(st, nn, p, idx, F, mask);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// SKUT (SIMT fp32).  Block = one candidate at a time (grid-stride over
// candidates), thread-per-row.  K and V of the whole sequence live in
// shared memory; the residual stream X and Q are row-private and live in a
// per-block global scratch (L2-resident).  Padded query rows are skipped:
// keys mask them and pooling ignores them.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSkutThreads, 1) skut_simt_kernel(
    Params p, NNCfg nn, Staged st, int use_staged, const int32_t* idx, const float* Fin,
    const uint8_t* fmask, int n, float* scratch, float* U, float* logits, float* pooled_out, int cs_shift,
    const uint8_t* extra, long long extra_stride) {
  __shared__ unsigned kmax_s;  // max_j ||k_j||^2 of the layer (single-pass shift)
  extern __shared__ __align__(16) float sm[];
  const int S = nn.seq_len;
  float* Ks = sm;                    // [S][64]
  float* Vs = sm + S * kDModel;      // [S][64]
  float* red = Vs + S * kDModel;     // [warps][64] pool partials
  float* zs = red + kSkutWarps * kDModel;  // [104] head input
  float* hs = zs + 112;              // [64]  head hidden
  int* valid_s = reinterpret_cast<int*>(hs + kHidden);  // [kMaxSeq] mask
  float* X = scratch + (size_t)blockIdx.x * 2 * S * kDModel;
  float* Q = X + (size_t)S * kDModel;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int item = blockIdx.x; item < n; item += gridDim.x) {
    // ---- K3: gather + encode (or load caller features) ----
    for (int r = tid; r < S; r += kSkutThreads) {
      float f[kDModel];
      int ok;
      if (use_staged) {
        int tok = slot_token(st, nn, idx, item, r);
        ok = tok >= 0;
        if (ok) encode_row(st, p, item, tok, r, f);
      } else {
        ok = fmask[(size_t)item * S + r] != 0;
        if (ok) load64(Fin + ((size_t)item * S + r) * kDModel, f);
      }
      valid_s[r] = ok;
      if (ok) store64(X + r * kDModel, f);
    }
    __syncthreads();

    for (int L = 0; L < p.num_layers; ++L) {
      if (tid == 0) kmax_s = 0u;
      __syncthreads();
      // ---- LN1 + Q/K/V projections (encoder.py:386-392, :398, :412-413) ----
      for (int r = tid; r < S; r += kSkutThreads) {
        if (!valid_s[r]) continue;
        float x[kDModel], a[kDModel], o[kDModel];
        load64(X + r * kDModel, x);
        layer_norm64(x, p.ln1_scale[L], p.ln1_shift[L], a);
        matvec<kDModel, kDModel>(a, p.wq[L], o);
        store64(Q + r * kDModel, o);
        matvec<kDModel, kDModel>(a, p.wk[L], o);
        store64(Ks + r * kDModel, o);
        if (cs_shift) {
          float kn2 = 0.0f;
#pragma unroll
          for (int j = 0; j < kDModel; ++j) kn2 = fmaf(o[j], o[j], kn2);
          atomicMax(&kmax_s, __float_as_uint(kn2));
        }
        matvec<kDModel, kDModel>(a, p.wv[L], o);
        store64(Vs + r * kDModel, o);
      }
      __syncthreads();
      // ---- causal key-masked softmax attention + Wo + LN2 + FFN ----
      for (int r0 = 0; r0 < S; r0 += kSkutThreads) {
        const int r = r0 + tid;
        const bool mine = r < S && valid_s[r];
        // warp-uniform key bound so the K/V broadcast reads stay converged
        int rmax = mine ? r : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        if (rmax < 0) continue;
        float q[kDModel], acc[kDModel];
        if (mine) load64(Q + r * kDModel, q);
        // encoder.py:366-377 custom mask (extra_mask, NAL training): key j is
        // allowed for row r only where extra[r, j] is set (2-D: shared)
        const uint8_t* xrow = (extra && mine) ? extra + (size_t)item * extra_stride + (size_t)r * S : nullptr;
#pragma unroll
        for (int j = 0; j < kDModel; ++j) acc[j] = 0.0f;
        float l = 0.0f;
        if (cs_shift) {
          // single pass: p_j = exp(s_j - m') with the Cauchy-Schwarz bound
          // m' = ||q_r|| max_j ||k_j|| / 8 >= s_j (shift invariance keeps 1/l
          // the exact normaliser; the host enables it only when m' provably
          // keeps every exponent in the normal range) -- no running max, no
          // per-key rescale of the accumulator
          float qn2 = 0.0f;
#pragma unroll
          for (int e = 0; e < kDModel; ++e) qn2 = fmaf(q[e], q[e], qn2);
          const float mb = sqrtf(qn2 * __uint_as_float(kmax_s)) * 0.125f;
          for (int j = 0; j <= rmax; ++j) {
            if (!valid_s[j]) continue;  // warp-uniform
            const float4* kr = reinterpret_cast<const float4*>(Ks + j * kDModel);
            float sdot = 0.0f;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float4 kv = kr[e];
              sdot = fmaf(q[4 * e], kv.x, sdot);
              sdot = fmaf(q[4 * e + 1], kv.y, sdot);
              sdot = fmaf(q[4 * e + 2], kv.z, sdot);
              sdot = fmaf(q[4 * e + 3], kv.w, sdot);
            }
            const float pj = (mine && j <= r && (!xrow || xrow[j])) ? expf(sdot * 0.125f - mb) : 0.0f;
            l += pj;
            const float4* vr = reinterpret_cast<const float4*>(Vs + j * kDModel);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float4 vv = vr[e];
              acc[4 * e] = fmaf(pj, vv.x, acc[4 * e]);
              acc[4 * e + 1] = fmaf(pj, vv.y, acc[4 * e + 1]);
              acc[4 * e + 2] = fmaf(pj, vv.z, acc[4 * e + 2]);
              acc[4 * e + 3] = fmaf(pj, vv.w, acc[4 * e + 3]);
            }
          }
        } else {
          float m = -INFINITY;
          for (int j = 0; j <= rmax; ++j) {
            if (!valid_s[j]) continue;  // warp-uniform
            const float4* kr = reinterpret_cast<const float4*>(Ks + j * kDModel);
            float sdot = 0.0f;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float4 kv = kr[e];
              sdot = fmaf(q[4 * e], kv.x, sdot);
              sdot = fmaf(q[4 * e + 1], kv.y, sdot);
              sdot = fmaf(q[4 * e + 2], kv.z, sdot);
              sdot = fmaf(q[4 * e + 3], kv.w, sdot);
            }
            const bool use = mine && j <= r && (!xrow || xrow[j]);
            const float sc = sdot * 0.125f;  // 1/sqrt(64)
            const float mn = use ? fmaxf(m, sc) : m;
            const float alpha = use ? expf(m - mn) : 1.0f;
            const float pj = use ? expf(sc - mn) : 0.0f;
            m = mn;
            l = l * alpha + pj;
            const float4* vr = reinterpret_cast<const float4*>(Vs + j * kDModel);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float4 vv = vr[e];
              acc[4 * e] = fmaf(pj, vv.x, acc[4 * e] * alpha);
              acc[4 * e + 1] = fmaf(pj, vv.y, acc[4 * e + 1] * alpha);
              acc[4 * e + 2] = fmaf(pj, vv.z, acc[4 * e + 2] * alpha);
              acc[4 * e + 3] = fmaf(pj, vv.w, acc[4 * e + 3] * alpha);
            }
          }
        }
        if (!mine) continue;
        // row r is a valid key of itself, so l > 0 and row_any = 1 -- unless
        // an extra mask disallows every key: zero attention output (:379-381)
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
#pragma unroll
        for (int j = 0; j < kDModel; ++j) acc[j] *= inv;
        float x[kDModel], t[kDModel];
        load64(X + r * kDModel, x);
        matvec<kDModel, kDModel>(acc, p.wo[L], t);  // (:449-450)
#pragma unroll
        for (int j = 0; j < kDModel; ++j) x[j] += t[j];
        layer_norm64(x, p.ln2_scale[L], p.ln2_shift[L], t);  // (:452-454)
        float h[kFfn];
        matvec<kDModel, kFfn>(t, p.w1[L], h);
#pragma unroll
        for (int j = 0; j < kFfn; ++j) h[j] = fmaxf(h[j], 0.0f);
        matvec<kFfn, kDModel>(h, p.w2[L], t);  // (:455-460)
#pragma unroll
        for (int j = 0; j < kDModel; ++j) x[j] += t[j];
        store64(X + r * kDModel, x);
      }
      __syncthreads();
    }

    if (U) {  // forward_fused output (valid rows; padded rows written as 0)
      for (int r = tid; r < S; r += kSkutThreads) {
        float x[kDModel];
        if (valid_s[r]) {
          load64(X + r * kDModel, x);
        } else {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) x[j] = 0.0f;
        }
        store64(U + ((size_t)item * S + r) * kDModel, x);
      }
    }
    if (logits) {
      // ---- K5: y = U W_out, max over valid rows (trainer.py:354-359) ----
      float pm[kDModel];
#pragma unroll
      for (int j = 0; j < kDModel; ++j) pm[j] = -INFINITY;
      int any = 0;
      for (int r = tid; r < S; r += kSkutThreads) {
        if (!valid_s[r]) continue;
        any = 1;
        float x[kDModel], y[kDModel];
        load64(X + r * kDModel, x);
        matvec<kDModel, kDModel>(x, p.out_linear, y);
#pragma unroll
        for (int j = 0; j < kDModel; ++j) pm[j] = fmaxf(pm[j], y[j]);
      }
      any = __syncthreads_or(any);
#pragma unroll
      for (int j = 0; j < kDModel; ++j) {
        float v = pm[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[warp * kDModel + j] = v;
      }
      __syncthreads();
      if (tid < kDModel) {
        float v = red[tid];
#pragma unroll
        for (int w = 1; w < kSkutWarps; ++w) v = fmaxf(v, red[w * kDModel + tid]);
        v = any ? v : 0.0f;  // empty user -> pooled = 0 (trainer.py:358-359)
        zs[tid] = v;
        if (pooled_out) pooled_out[(size_t)item * kDModel + tid] = v;
      } else if (tid < kDModel + kEmbed) {
        zs[tid] = use_staged ? st.cand_unit[(size_t)item * kEmbed + tid - kDModel] : 0.0f;
      } else if (tid < kDModel + kEmbed + kCtx) {
        zs[tid] = use_staged ? st.ctx[st.item_req[item] * kCtx + tid - kDModel - kEmbed] : 0.0f;
      }
      __syncthreads();
      // ---- CTR head: ReLU(z W1 + b1) W2 + b2 (trainer.py:361-366) ----
      if (tid < kHidden) {
        float h = 0.0f;
        for (int i = 0; i < kDModel + kEmbed + kCtx; ++i) h = fmaf(zs[i], __ldg(p.head_w1 + i * kHidden + tid), h);
        hs[tid] = fmaxf(h + __ldg(p.head_b1 + tid), 0.0f);
      }
      __syncthreads();
      if (tid < kHeads) {
        float o = 0.0f;
        for (int j = 0; j < kHidden; ++j) o = fmaf(hs[j], __ldg(p.head_w2 + j * kHeads + tid), o);
        logits[(size_t)item * kHeads + tid] = o + __ldg(p.head_b2 + tid);
      }
    }
    __syncthreads();
  }
}

int skut_simt_grid(int n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return n < sms ? n : sms;
}

size_t skut_simt_scratch_floats(int seq_len) { return (size_t)2 * seq_len * kDModel; }

cudaError_t launch_skut_simt(const Params& p, const NNCfg& nn, const Staged* st,
                             const int32_t* idx, const float* F, const uint8_t* fmask, int n,
                             float* scratch, float* U, float* logits, float* pooled, int cs_shift,
                             cudaStream_t s, const uint8_t* extra, long long extra_stride) {
  if (n == 0) return cudaSuccess;
  const int S = nn.seq_len;
  size_t smem = (size_t)(2 * S * kDModel + kSkutWarps * kDModel + 112 + kHidden) * 4 + kMaxSeq * 4;
  cudaError_t e = set_max_dyn_smem((const void*)skut_simt_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  Staged dummy{};
  skut_simt_kernel<<<skut_simt_grid(n), kSkutThreads, smem, s>>>(
      p, nn, st ? *st : dummy, st != nullptr, idx, F, fmask, n, scratch, U, logits, pooled, cs_shift, extra,
      extra_stride);
  return cudaGetLastError();
}

}  // namespace tav2
