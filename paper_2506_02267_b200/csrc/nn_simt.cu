// K1 token/candidate prep, K2 NN scoring (SIMT, reference-faithful f64
// scores) with per-candidate streaming top-k, and the top-k merge that
// writes the Eq. 2 index layout.
//
// Reference: nnsearch.py:274-286 (_unit_rows_into), :289-369
// (fused_assemble), :114-118 (_nn_segment_indices), :153-180 (_layout);
// core.py:54-79 (dequantize / l2_normalize_rows / unit_embeddings).
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

// ---------------------------------------------------------------------------
// K1: per token  unit(dequantize(q)) in f32 with the reference's rounding
// steps (core.py:54-57 then :69-74) and 2^-27/||q|| in f64 for the i8-limb
// tensor-core path; per candidate  l2_normalize_rows (nnsearch.py:313-320).
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

__global__ void __launch_bounds__(256) prep_kernel(Staged st) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < st.n_tok) {
    const int4* src = reinterpret_cast<const int4*>(st.emb + (size_t)i * kEmbed);
    int4 raw[2] = {src[0], src[1]};
    const int8_t* q = reinterpret_cast<const int8_t*>(raw);
    float d[kEmbed];
    int isq = 0;
#pragma unroll
    for (int j = 0; j < kEmbed; ++j) {
      int qi = q[j];
      isq += qi * qi;
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
    // bf16 hi/lo image of the unit row, pre-tiled for the tensor-core NN
    // scores: 64-token tiles of 8 KB = [8 chunks (hi 0-3, lo 4-7)][64 rows][16 B]
    // (the UMMA K-major no-swizzle B-operand layout), one bulk copy per tile
    uint8_t* tile = reinterpret_cast<uint8_t*>(st.tok_bf16) + (size_t)(i >> 6) * 8192 + (i & 63) * 16;
#pragma unroll
    for (int j = 0; j < kEmbed; j += 8) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) tc::split_pair(u[j + 2 * e], u[j + 2 * e + 1], hi[e], lo[e]);
      *reinterpret_cast<uint4*>(tile + (j / 8) * 1024) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(tile + (4 + j / 8) * 1024) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    (void)isq;
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

cudaError_t launch_prep(const Staged& st, cudaStream_t s) {
  int n = st.n_tok + st.n_items;
  if (n == 0) return cudaSuccess;
  prep_kernel<<<(n + 255) / 256, 256, 0, s>>>(st);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2 (SIMT): one block per NNWork unit = (64-candidate tile, source, token
// chunk).  Thread c owns candidate c: f64 dot of the f32 unit vectors
// (nnsearch.py:344-347) for every token of the chunk, streamed through a
// per-thread min-heap of the best k keys (ties -> lower index).  Token rows
// are staged through shared memory and read as warp-wide broadcasts.
// ---------------------------------------------------------------------------
constexpr int kSimtTile = 64;
constexpr int kTokTile = 64;

__global__ void __launch_bounds__(kSimtTile) nn_simt_kernel(Staged st, NNCfg nn, uint64_t* part,
                                                            int kmax, int tile_size) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* toks = reinterpret_cast<float*>(smem);                         // [kTokTile][32]
  uint64_t* heap = reinterpret_cast<uint64_t*>(smem + kTokTile * kEmbed * 4);  // [k][64]
  const NNWork w = st.work[blockIdx.x];
  const NNTile tile = st.tiles[w.tile];
  const ReqInfo rq = st.req[tile.req];
  const int c = threadIdx.x;
  const int lc = blockIdx.y * kSimtTile + c;  // candidate within the tile
  const int k = nn.k[w.source];
  const int src = w.source;  // 0 LL, 1 RT (tail range), 2 IMP
  if (blockIdx.y * kSimtTile >= tile.n) return;  // block-uniform
  const float* tok_base = st.tok_unit + (size_t)rq.tok_off[src] * kEmbed;

  double uc[kEmbed];
  const bool active = lc < tile.n;
  {
    const float* cu = st.cand_unit + (size_t)(tile.item0 + (active ? lc : 0)) * kEmbed;
#pragma unroll
    for (int j = 0; j < kEmbed; ++j) uc[j] = (double)cu[j];
  }
  for (int i = 0; i < k; ++i) heap[i * kSimtTile + c] = 0ull;
  uint64_t root = 0ull;

  for (int t0 = w.t0; t0 < w.t1; t0 += kTokTile) {
    const int nt = min(kTokTile, w.t1 - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * (kEmbed / 4); e += blockDim.x) {
      reinterpret_cast<float4*>(toks)[e] =
          reinterpret_cast<const float4*>(tok_base + (size_t)t0 * kEmbed)[e];
    }
    __syncthreads();
    if (!active) continue;
    for (int j = 0; j < nt; ++j) {
      const float4* row = reinterpret_cast<const float4*>(toks + j * kEmbed);
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kEmbed / 4; ++q) {
        float4 v = row[q];
        s = fma((double)v.x, uc[4 * q], s);
        s = fma((double)v.y, uc[4 * q + 1], s);
        s = fma((double)v.z, uc[4 * q + 2], s);
        s = fma((double)v.w, uc[4 * q + 3], s);
      }
      uint64_t key = score_key(s, t0 + j);
      if (key > root) {
        heap_replace_root(heap + c, kSimtTile, k, key);
        root = heap[c];
      }
    }
  }
  if (!active) return;
  uint64_t* out = part + part_offset(tile, src, lc, blockIdx.x - tile.work0[src], kmax, tile_size);
  for (int i = 0; i < k; ++i) out[i] = heap[i * kSimtTile + c];
}

cudaError_t launch_nn_simt(const Staged& st, const NNCfg& nn, uint64_t* part, int kmax,
                           int tile_size, cudaStream_t s) {
  if (st.n_work == 0) return cudaSuccess;
  size_t smem = kTokTile * kEmbed * 4 + (size_t)kmax * kSimtTile * 8;
  cudaError_t e = cudaFuncSetAttribute(nn_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(st.n_work, tile_size / kSimtTile);
  nn_simt_kernel<<<grid, kSimtTile, smem, s>>>(st, nn, part, kmax, tile_size);
  return cudaGetLastError();
}

}  // namespace tav2
