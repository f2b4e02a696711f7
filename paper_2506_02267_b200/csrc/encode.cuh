// Gather + Eq. 4 early-fusion encode of one layout slot (shared by the SIMT
// and tensor-core SKUT kernels).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

// Which source and token does layout slot `r` of `item` hold?  Returns the
// global token id or -1 for padding (nnsearch.py:153-180 segment order).
__device__ __forceinline__ int slot_token(const Staged& st, const NNCfg& nn, const int32_t* idx,
                                          int item, int r) {
  int t = idx[(size_t)item * nn.seq_len + r];
  if (t < 0) return -1;
  const ReqInfo& rq = st.req[st.item_req[item]];
  int src = r < nn.seg_start[1] ? 0 : (r < nn.seg_start[3] ? 1 : 2);
  return rq.tok_off[src] + t;
}

// Eq. 4 (encoder.py:171-187): [unit(q) | unit(c)] + (bits @ action_table)
// + surface_table[min(s,3)] + position_table[r]; masked rows are zero.
__device__ __forceinline__ void encode_row(const Staged& st, const Params& p, int item, int tok,
                                           int r, float* f) {
  const float4* tu = reinterpret_cast<const float4*>(st.tok_unit + (size_t)tok * kEmbed);
  const float4* cu = reinterpret_cast<const float4*>(st.cand_unit + (size_t)item * kEmbed);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float4 a = tu[j], b = cu[j];
    f[4 * j] = a.x; f[4 * j + 1] = a.y; f[4 * j + 2] = a.z; f[4 * j + 3] = a.w;
    f[32 + 4 * j] = b.x; f[33 + 4 * j] = b.y; f[34 + 4 * j] = b.z; f[35 + 4 * j] = b.w;
  }
  const unsigned act = st.action[tok];
  int surf = st.surface[tok];
  surf = surf > 3 ? 3 : surf;  // SURFACE_OTHER fold (encoder.py:178)
  float asum[kDModel];
#pragma unroll
  for (int j = 0; j < kDModel; ++j) asum[j] = 0.0f;
  for (int b = 0; b < p.action_rows; ++b) {
    if ((act >> b) & 1u) {
      const float4* row = reinterpret_cast<const float4*>(p.action_table + b * kDModel);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float4 v = __ldg(row + j);
        asum[4 * j] += v.x; asum[4 * j + 1] += v.y; asum[4 * j + 2] += v.z; asum[4 * j + 3] += v.w;
      }
    }
  }
  const float4* srow = reinterpret_cast<const float4*>(p.surface_table + surf * kDModel);
  const float4* prow = reinterpret_cast<const float4*>(p.position_table + r * kDModel);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float4 s4 = __ldg(srow + j), p4 = __ldg(prow + j);
    f[4 * j] = (f[4 * j] + asum[4 * j]) + s4.x;
    f[4 * j + 1] = (f[4 * j + 1] + asum[4 * j + 1]) + s4.y;
    f[4 * j + 2] = (f[4 * j + 2] + asum[4 * j + 2]) + s4.z;
    f[4 * j + 3] = (f[4 * j + 3] + asum[4 * j + 3]) + s4.w;
    f[4 * j] += p4.x; f[4 * j + 1] += p4.y; f[4 * j + 2] += p4.z; f[4 * j + 3] += p4.w;
  }
}

// The same row from prep's precomputed token part (tok_feat = [unit(q) | 0]
// + bits @ action_table + surface_table[min(s,3)]): x = (tok_feat + [0 |
// unit(c)]) + position_table[r], with 32-byte loads (LDG.256: one sector
// per lane).  f32 sums in another order than encode_row (<= 1 ulp apart);
// the bf16 tensor-core kernels use it, the fp32 parity path keeps encode_row.
__device__ __forceinline__ void encode_feat(const Staged& st, const Params& p, int item, int tok, int r,
                                            float* f) {
  const float* tf = st.tok_feat + (size_t)tok * kDModel;
  const float* cu = st.cand_unit + (size_t)item * kEmbed;
  const float* pr = p.position_table + (size_t)r * kDModel;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float a[8], b[8], c[8];
    tc::ldg256(tf + 8 * j, a);
    tc::ldg256(pr + 8 * j, b);
    if (j >= 4) {
      tc::ldg256(cu + 8 * (j - 4), c);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) c[e] = 0.0f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) f[8 * j + e] = (a[e] + c[e]) + b[e];
  }
}

}  // namespace tav2
