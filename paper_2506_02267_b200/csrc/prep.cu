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

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// ---------------------------------------------------------------------------
// K1: per token  unit(dequantize(q)) in f32 with the reference's rounding
// steps (core.py:54-57 then :69-74), its fp16 tile image for the tensor-core
// scan and (with parameters) its Eq. 4 feature part for the SKUT gather; per
// candidate  l2_normalize_rows (nnsearch.py:313-320).
// ---------------------------------------------------------------------------
// Sum of squares of a 32-vector held by a quad of threads (thread g holds
// elements 8g..8g+7) in numpy's exact einsum("ij,ij->i", dtype=f32) order
// (core.py:72, nnsearch.py:282 / :317), probed bit for bit on this image's
// numpy (tools/einsum_order.py): four 4-lane accumulators, lane l summing
// x[l + 4m]^2 in the unrolled-by-4 reverse order m = 3,2,1,0 then 7,6,5,4
// (separately rounded products and additions), then (l0 + l1) + (l2 + l3).
// Every thread of the quad gathers all 32 squares and returns the same value.
__device__ __forceinline__ float quad_sumsq(const float* v, unsigned qm) {  // (qm: the participating lanes)
  float s[32];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float sq = __fmul_rn(v[i], v[i]);
#pragma unroll
    for (int t = 0; t < 4; ++t) s[8 * t + i] = __shfl_sync(qm, sq, t, 4);
  }
  float lane[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    float a = s[12 + l];
    a = __fadd_rn(s[8 + l], a);
    a = __fadd_rn(s[4 + l], a);
    a = __fadd_rn(s[l], a);
    a = __fadd_rn(s[28 + l], a);
    a = __fadd_rn(s[24 + l], a);
    a = __fadd_rn(s[20 + l], a);
    a = __fadd_rn(s[16 + l], a);
    lane[l] = a;
  }
  return __fadd_rn(__fadd_rn(lane[0], lane[1]), __fadd_rn(lane[2], lane[3]));
}

// One quad of threads per token row (then per candidate row); thread g owns
// elements 8g..8g+7 of the 32-vector and features 16g..16g+15 of the 64-d
// Eq. 4 token part.
__device__ __forceinline__ void prep_body(const Staged& st, int with_feat, const float* tab_s, int action_rows,
                                          int2 raw, unsigned act, int surf_raw, float4 c0, float4 c1,
                                          const float* deq_s);

__global__ void __launch_bounds__(256) prep_kernel(Staged st, Params p, int with_feat, uint32_t* epoch_bump) {
  cta_stamp(kDbgPrep, 0);
  griddep_launch();
  griddep_wait();  // the previous step's kernels may still read tok_unit / cand_unit
  // a fresh select-flag epoch for this run (SelFlags): the previous run's
  // select / SKUT grids are complete here; the epoch is never 0 (the flags'
  // reset value)
  if (epoch_bump && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t e = *epoch_bump + 1u;
    *epoch_bump = e ? e : 1u;
    epoch_bump[1] = 0u;  // the SKUT's dynamic item counter (SelFlags::next_item)
  }
  cta_stamp(kDbgPrep, 2);
  // this thread's global inputs, requested before the table staging so the
  // round trips overlap
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = gt >> 2;
  int2 raw = make_int2(0, 0);
  unsigned act = 0u;
  int surf = 0;
  float4 c0 = make_float4(0.f, 0.f, 0.f, 0.f), c1 = c0;
  if (row < st.n_tok) {
    raw = reinterpret_cast<const int2*>(st.emb + (size_t)row * kEmbed)[gt & 3];
    if (with_feat) {
      act = st.action[row];
      surf = st.surface[row];
    }
  } else if (row - st.n_tok < st.n_items) {
    const float4* src = reinterpret_cast<const float4*>(st.cand + (size_t)(row - st.n_tok) * kEmbed + 8 * (gt & 3));
    c0 = src[0];
    c1 = src[1];
  }
  // action (<= 16 rows) and surface (4 rows) tables staged in shared memory:
  // a token sums up to 16 action rows, read from here instead of one
  // dependent global round trip per set bit
  __shared__ __align__(16) float tab_s[(16 + 4) * kDModel];
  if (with_feat) {
    for (int i = threadIdx.x; i < (p.action_rows + 4) * kDModel / 4; i += blockDim.x) {
      const int r = i / (kDModel / 4);
      const float4* srcp = r < p.action_rows ? reinterpret_cast<const float4*>(p.action_table) + i
                                             : reinterpret_cast<const float4*>(p.surface_table) + (i - p.action_rows * kDModel / 4);
      reinterpret_cast<float4*>(tab_s)[r < p.action_rows ? i : 16 * kDModel / 4 + (i - p.action_rows * kDModel / 4)] =
          __ldg(srcp);
    }
  }
  // dequantize (core.py:54-57) as a 256-entry table: one IEEE division per
  // thread per CTA instead of eight per row (bit-identical: the same two
  // correctly rounded operations per int8 value)
  __shared__ float deq_s[256];
  deq_s[threadIdx.x] = __fmul_rn(__fdiv_rn((float)((int)threadIdx.x - 128), 127.0f), 0.65f);
  __syncthreads();
  prep_body(st, with_feat, tab_s, p.action_rows, raw, act, surf, c0, c1, deq_s);
  if (kDebug) {
    __syncthreads();
    cta_stamp(kDbgPrep, 1);
  }
}

__device__ __forceinline__ void prep_body(const Staged& st, int with_feat, const float* tab_s, int action_rows,
                                          int2 raw, unsigned act, int surf_raw, float4 v0, float4 v1,
                                          const float* deq_s) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  int i = gt >> 2;
  const int g = gt & 3;
  // The quad's sum of squares at a point every lane of the warp reaches (a
  // warp may hold token rows, candidate rows and padding): full-mask
  // shuffles, not quad-masked ones inside the branches (each of which
  // compiled to a divergence check)
  const bool is_tok = i < st.n_tok;
  const int8_t* q = reinterpret_cast<const int8_t*>(&raw);
  float d[8];
  if (is_tok) {
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = deq_s[(int)q[j] + 128];  // core.py:54-57
  } else {
    d[0] = v0.x; d[1] = v0.y; d[2] = v0.z; d[3] = v0.w; d[4] = v1.x; d[5] = v1.y; d[6] = v1.z; d[7] = v1.w;
  }
  const float ss = quad_sumsq(d, 0xffffffffu);
  // unit rows of tokens and candidates alike (core.py:69-74, nnsearch.py:313-320;
  // zero rows stay zero; padding lanes compute zeros and store nothing)
  float nrm = __fsqrt_rn(ss);
  if (nrm == 0.0f) nrm = 1.0f;
  float u[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) u[j] = __fdiv_rn(d[j], nrm);
  // features 0..31 of a token's Eq. 4 part = unit(q): thread g < 2 takes
  // elements 16g..16g+15, held by threads 2g and 2g+1 (full-mask shuffles,
  // every lane; g >= 2 and non-token lanes discard)
  float fq[16];
  if (with_feat) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float lo = __shfl_sync(0xffffffffu, u[j], 2 * (g & 1), 4);
      const float hi = __shfl_sync(0xffffffffu, u[j], 2 * (g & 1) + 1, 4);
      fq[j] = g < 2 ? lo : 0.0f;
      fq[8 + j] = g < 2 ? hi : 0.0f;
    }
  }
  if (is_tok) {
    float4* dst = reinterpret_cast<float4*>(st.tok_unit + (size_t)i * kEmbed + 8 * g);
    dst[0] = make_float4(u[0], u[1], u[2], u[3]);
    dst[1] = make_float4(u[4], u[5], u[6], u[7]);
    // fp16 image of the unit row, pre-tiled for the tensor-core NN scan
    // (kScanTile-token tiles, UMMA K-major no-swizzle B-operand layout,
    // tav2_common.cuh): this thread's 8 elements are one 16-byte chunk
    uint8_t* tile = reinterpret_cast<uint8_t*>(st.tok_img) + (size_t)(i / kScanTile) * kScanTileBytes +
                    (i % kScanTile) * 16 + g * (kScanTile * 16);
    *reinterpret_cast<uint4*>(tile) = make_uint4(pack_h2(u[0], u[1]), pack_h2(u[2], u[3]), pack_h2(u[4], u[5]),
                                                 pack_h2(u[6], u[7]));
    if (with_feat) {  // token part of Eq. 4 (encoder.py:171-187): [unit(q) | 0] + bits @ action + surface
      const float* f = fq;
      float asum[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) asum[j] = 0.0f;
      for (int b = 0; b < action_rows; ++b)
        if ((act >> b) & 1u) {
          const float4* row = reinterpret_cast<const float4*>(tab_s + b * kDModel + 16 * g);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 v = row[j];
            asum[4 * j] += v.x; asum[4 * j + 1] += v.y; asum[4 * j + 2] += v.z; asum[4 * j + 3] += v.w;
          }
        }
      const int surf = min(surf_raw, 3);  // SURFACE_OTHER fold (encoder.py:178)
      const float4* srow = reinterpret_cast<const float4*>(tab_s + (16 + surf) * kDModel + 16 * g);
      float4* fd = reinterpret_cast<float4*>(st.tok_feat + (size_t)i * kDModel + 16 * g);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 sv = srow[j];
        fd[j] = make_float4((f[4 * j] + asum[4 * j]) + sv.x, (f[4 * j + 1] + asum[4 * j + 1]) + sv.y,
                            (f[4 * j + 2] + asum[4 * j + 2]) + sv.z, (f[4 * j + 3] + asum[4 * j + 3]) + sv.w);
      }
    }
    return;
  }
  i -= st.n_tok;
  if (i < st.n_items) {  // l2_normalize_rows of the candidates (nnsearch.py:313-320)
    float4* dst = reinterpret_cast<float4*>(st.cand_unit + (size_t)i * kEmbed + 8 * g);
    dst[0] = make_float4(u[0], u[1], u[2], u[3]);
    dst[1] = make_float4(u[4], u[5], u[6], u[7]);
  }
}

cudaError_t set_dbg_cta_prep(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t launch_prep(const Staged& st, const Params* p, cudaStream_t s, uint32_t* epoch_bump) {
  int n = st.n_tok + st.n_items;
  if (n == 0) return cudaSuccess;
  const Params pz{};
  return launch_pdl(prep_kernel, dim3((4 * n + 255) / 256), dim3(256), 0, s, st, p ? *p : pz, (int)(p != nullptr),
                    epoch_bump);
}

}  // namespace tav2
