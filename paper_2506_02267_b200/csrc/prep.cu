// K1: token and candidate prep for the NN scan and the encoder.
//
// Reference: nnsearch.py:274-286 (_unit_rows_into), :313-320 (candidate
// normalisation); core.py:54-79 (dequantize / l2_normalize_rows /
// unit_embeddings).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"
#include "dbg.cuh"

namespace tav2 {

// ---------------------------------------------------------------------------
// K1: per token  unit(dequantize(q)) in f32 with the reference's rounding
// steps (core.py:54-57 then :69-74), its fp16 tile image for the tensor-core
// scan and (with parameters) its Eq. 4 feature part for the SKUT gather; per
// candidate  l2_normalize_rows (nnsearch.py:313-320).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float sumsq8(const float* v) {
  // 8 interleaved accumulators, adjacent-pair combine (a fixed order; the
  // reference's einsum order is BLAS-internal, differences are <= 1 ulp).
  float a[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) a[l] = __fmul_rn(v[l], v[l]);
#pragma unroll
  for (int j = 8; j < kEmbed; ++j) a[j & 7] = __fadd_rn(a[j & 7], __fmul_rn(v[j], v[j]));
  float b0 = __fadd_rn(a[0], a[1]), b1 = __fadd_rn(a[2], a[3]);
  float b2 = __fadd_rn(a[4], a[5]), b3 = __fadd_rn(a[6], a[7]);
  return __fadd_rn(__fadd_rn(b0, b1), __fadd_rn(b2, b3));
}

__global__ void __launch_bounds__(256) prep_kernel(Staged st, Params p, int with_feat) {
  cta_stamp(kDbgPrep, 0);
  griddep_launch();
  griddep_wait();  // the previous step's kernels may still read tok_unit / cand_unit
  cta_stamp(kDbgPrep, 2);
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < st.n_tok) {
    const int4* src = reinterpret_cast<const int4*>(st.emb + (size_t)i * kEmbed);
    int4 raw[2] = {src[0], src[1]};
    const int8_t* q = reinterpret_cast<const int8_t*>(raw);
    float d[kEmbed];
#pragma unroll
    for (int j = 0; j < kEmbed; ++j) {
      int qi = q[j];
      d[j] = __fmul_rn(__fdiv_rn((float)qi, 127.0f), 0.65f);
    }
    float nrm = __fsqrt_rn(sumsq8(d));
    if (nrm == 0.0f) nrm = 1.0f;
    float u[kEmbed];
#pragma unroll
    for (int j = 0; j < kEmbed; ++j) u[j] = __fdiv_rn(d[j], nrm);
    float4* dst = reinterpret_cast<float4*>(st.tok_unit + (size_t)i * kEmbed);
#pragma unroll
    for (int j = 0; j < kEmbed; j += 4) dst[j / 4] = make_float4(u[j], u[j + 1], u[j + 2], u[j + 3]);
    // fp16 image of the unit row, pre-tiled for the tensor-core NN scan
    // (kScanTile-token tiles, UMMA K-major no-swizzle B-operand layout,
    // tav2_common.cuh), one bulk copy per tile
    uint8_t* tile = reinterpret_cast<uint8_t*>(st.tok_img) + (size_t)(i / kScanTile) * kScanTileBytes +
                    (i % kScanTile) * 16;
#pragma unroll
    for (int j = 0; j < kEmbed; j += 8) {
      uint32_t h[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __half2 p = __floats2half2_rn(u[j + 2 * e], u[j + 2 * e + 1]);
        h[e] = *reinterpret_cast<const uint32_t*>(&p);
      }
      *reinterpret_cast<uint4*>(tile + (j / 8) * (kScanTile * 16)) = make_uint4(h[0], h[1], h[2], h[3]);
    }
    if (with_feat) {  // token part of Eq. 4 (encoder.py:171-187): [unit(q) | 0] + bits @ action + surface
      float f[kDModel];
#pragma unroll
      for (int j = 0; j < kEmbed; ++j) {
        f[j] = u[j];
        f[kEmbed + j] = 0.0f;
      }
      const unsigned act = st.action[i];
      float asum[kDModel];
#pragma unroll
      for (int j = 0; j < kDModel; ++j) asum[j] = 0.0f;
      for (int b = 0; b < p.action_rows; ++b)
        if ((act >> b) & 1u) {
          const float4* row = reinterpret_cast<const float4*>(p.action_table + b * kDModel);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 v = __ldg(row + j);
            asum[4 * j] += v.x; asum[4 * j + 1] += v.y; asum[4 * j + 2] += v.z; asum[4 * j + 3] += v.w;
          }
        }
      const int surf = min((int)st.surface[i], 3);  // SURFACE_OTHER fold (encoder.py:178)
      const float4* srow = reinterpret_cast<const float4*>(p.surface_table + surf * kDModel);
      float4* fd = reinterpret_cast<float4*>(st.tok_feat + (size_t)i * kDModel);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float4 sv = __ldg(srow + j);
        fd[j] = make_float4((f[4 * j] + asum[4 * j]) + sv.x, (f[4 * j + 1] + asum[4 * j + 1]) + sv.y,
                            (f[4 * j + 2] + asum[4 * j + 2]) + sv.z, (f[4 * j + 3] + asum[4 * j + 3]) + sv.w);
      }
    }
    return;
  }
  i -= st.n_tok;
  if (i < st.n_items) {
    const float4* src = reinterpret_cast<const float4*>(st.cand + (size_t)i * kEmbed);
    float c[kEmbed];
#pragma unroll
    for (int j = 0; j < kEmbed; j += 4) {
      float4 v = src[j / 4];
      c[j] = v.x; c[j + 1] = v.y; c[j + 2] = v.z; c[j + 3] = v.w;
    }
    float nrm = __fsqrt_rn(sumsq8(c));
    if (nrm == 0.0f) nrm = 1.0f;
    float4* dst = reinterpret_cast<float4*>(st.cand_unit + (size_t)i * kEmbed);
#pragma unroll
    for (int j = 0; j < kEmbed; j += 4)
      dst[j / 4] = make_float4(__fdiv_rn(c[j], nrm), __fdiv_rn(c[j + 1], nrm),
                               __fdiv_rn(c[j + 2], nrm), __fdiv_rn(c[j + 3], nrm));
  }
}

cudaError_t set_dbg_cta_prep(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t launch_prep(const Staged& st, const Params* p, cudaStream_t s) {
  int n = st.n_tok + st.n_items;
  if (n == 0) return cudaSuccess;
  const Params pz{};
  return launch_pdl(prep_kernel, dim3((n + 255) / 256), dim3(256), 0, s, st, p ? *p : pz, (int)(p != nullptr));
}

}  // namespace tav2
