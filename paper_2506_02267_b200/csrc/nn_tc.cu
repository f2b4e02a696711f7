// K2 on the tensor cores: NN scores of a 128-candidate tile against a token
// chunk as an exact int8 GEMM (tcgen05.mma kind::i8, s32 accumulation in
// TMEM), fused with the per-candidate streaming top-k.
//
// Reference semantics (nnsearch.py:274-286, :313-347): score(t, c) =
// unit(dequantize(q_t)) . unit(c).  Since normalisation removes the int8
// scale, score = (q_t . u_c) / ||q_t||.  The candidate unit vector u_c is
// written as a 2^-27 fixed-point integer split into four balanced int8
// limbs (base 128), so q . u_c = sum_l 2^(7(3-l)) (q . d_l) is EXACT in four
// s32 accumulators; the epilogue recombines them in f64 and multiplies by
// 2^-27/||q|| (f64).  Score error <= 2^-28 * ||q||_1/||q|| ~ 2e-8, i.e. an
// order of magnitude below the reference's own f32 rounding noise.
//
// Roles (192 threads): warps 0-3 epilogue (thread = candidate = TMEM lane),
// warp 4 TMA producer (64-token x 32-byte tiles, 4-stage ring), warp 5 MMA
// issuer.  TMEM: 2 buffers x 4 limbs x 64 columns = 512.
//
// Exact top-k over a source split into `nw` chunks runs in two passes so the
// per-element work is a handful of f32 instructions:
//   pass 1: each chunk keeps, in registers, its top-M APPROXIMATE scores
//           (exact int64 dot rounded once to f32, |err| <= 3 ulp < 2e-7),
//           M in {8, 16} with nw*M >= k (planner), and publishes the M-th
//           one.  T = min over chunks: >= nw*M >= k elements have approx >= T,
//           so the exact k-th best g >= T - eps and every exact top-k element
//           has approx >= T - 2 eps.
//   pass 2: each chunk builds exact f64 keys only for approx >= T - 2 eps
//           and keeps the best k of them (append, heapify when full).
// A single-chunk source (nw == 1) is done exactly in pass 1.
// The merge folds the per-chunk lists (nn_merge.cu).
#include <cuda.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

constexpr int kNT = 64;      // tokens per MMA tile (N)
constexpr int kStages = 4;   // smem ring depth
constexpr int kTcThreads = 192;

struct NNTcSmem {
  static constexpr int kA = 4 * 128 * 32;   // 4 limbs x 128 rows x 32 B
  static constexpr int kB = kNT * 32;       // one token tile
};

constexpr int kTopM = 16;        // register top-m capacity of pass 1
constexpr float kApproxEps = 1e-6f;  // > 3x the f32 recombination error bound


template <int M>  // pass-1 register list size (compile time: branch-free bubble)
__global__ void __launch_bounds__(kTcThreads, 1) nn_tc_kernel(Staged st, NNCfg nn,
                                                              const __grid_constant__ CUtensorMap emb_map,
                                                              uint64_t* part, float* part1,
                                                              int kmax, int tile_size, int pass) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;                                      // [4][2 chunks][128][16]
  uint8_t* Bs = sm + NNTcSmem::kA;                       // [kStages][2][64][16]
  uint64_t* heap = reinterpret_cast<uint64_t*>(Bs + kStages * NNTcSmem::kB);  // [k][cpb]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
  __shared__ uint32_t taddr_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const NNWork w = st.work[blockIdx.x];
  const NNTile tile = st.tiles[w.tile];
  const ReqInfo rq = st.req[tile.req];
  const int src = w.source;
  const int nw = tile.nwork[src];
  if (pass == 2 && nw == 1) return;  // pass 1 was already exact (block-uniform)
  const int k = nn.k[src];
  const bool exact = pass == 2 || nw == 1;  // exact keys + heap, else approx top-m
  const int jchunk = blockIdx.x - tile.work0[src];
  const int cpb = tile_size / gridDim.y;  // candidates owned by this CTA
  const int c_lo = blockIdx.y * cpb;
  const int ntiles = (w.t1 - w.t0 + kNT - 1) / kNT;
  const int row0 = rq.tok_off[src] + w.t0;

  // ---- prologue: candidate limbs (A operand), heaps, barriers, TMEM ----
  if (warp < 4) {
    const int c = tid;
    int32_t C[kEmbed];
    const bool real = c < tile.n;
    const float* cu = st.cand_unit + (size_t)(tile.item0 + (real ? c : 0)) * kEmbed;
#pragma unroll
    for (int j = 0; j < kEmbed; ++j) C[j] = real ? __float2int_rn(cu[j] * 134217728.0f) : 0;  // 2^27
    uint32_t limb[4][8];
#pragma unroll
    for (int l = 3; l >= 0; --l) {
#pragma unroll
      for (int j = 0; j < kEmbed; j += 4) {
        uint32_t packed = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int x = C[j + e];
          int d = l == 0 ? x : ((x + 64) & 127) - 64;  // balanced base-128 digit
          C[j + e] = (x - d) >> 7;
          packed |= (uint32_t)(uint8_t)(int8_t)d << (8 * e);
        }
        limb[l][j / 4] = packed;
      }
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      *reinterpret_cast<uint4*>(As + l * 4096 + c * 16) = make_uint4(limb[l][0], limb[l][1], limb[l][2], limb[l][3]);
      *reinterpret_cast<uint4*>(As + l * 4096 + 2048 + c * 16) =
          make_uint4(limb[l][4], limb[l][5], limb[l][6], limb[l][7]);
    }
    if (exact && c >= c_lo && c < c_lo + cpb) {
      uint64_t* hh = heap + (c - c_lo);
      for (int i = 0; i < k; ++i) hh[i * cpb] = 0ull;
    }
  } else if (warp == 4) {
    if (lane == 0) {
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], 128);
      }
      mbar_fence_init();
      tma_prefetch_desc(&emb_map);
    }
  } else {
    tmem_alloc<512>(&taddr_s);
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;

  if (warp == 4) {
    // ---- TMA producer ----
    if (lane == 0) {
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], NNTcSmem::kB);
        tma_load_3d(Bs + s * NNTcSmem::kB, &emb_map, &full[s], 0, row0 + i * kNT, 0);
      }
    }
  } else if (warp == 5) {
    // ---- MMA issuer ----
    if (lane == 0) {
      const uint32_t id = idesc_i8(128, kNT);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages, b = i & 1;
        mbar_wait(&full[s], (i / kStages) & 1);
        mbar_wait(&tempty[b], ((i >> 1) & 1) ^ 1);
        fence_after();
        const uint64_t bd = sdesc(smem_u32(Bs + s * NNTcSmem::kB), kNT * 16, 128);
#pragma unroll
        for (int l = 0; l < 4; ++l)
          mma_i8_ss(T + b * 256 + l * kNT, sdesc(smem_u32(As + l * 4096), 128 * 16, 128), bd, id, 0);
        commit(&empty[s]);
        commit(&tfull[b]);
      }
    }
  } else {
    // ---- epilogue: recombine limbs -> score -> top-m (pass 1) / top-k (exact) ----
    const int c = tid;
    const bool mine = c >= c_lo && c < c_lo + cpb && c < tile.n;
    uint64_t* h = heap + (c - c_lo);
    uint64_t root = 0ull;
    int hn = 0;  // heap fill (append mode until k, then heapify)
    float top[M];  // descending
#pragma unroll
    for (int i = 0; i < M; ++i) top[i] = -INFINITY;
    float thr = -FLT_MAX;  // approx-score gate (-inf marks columns past the chunk)
    if (pass == 2 && mine) {
      const float* p1 = part1 + part_offset(tile, src, c, 0, 1, tile_size);
      float t = INFINITY;
      for (int j = 0; j < nw; ++j) t = fminf(t, p1[j]);
      thr = t - 2.0f * kApproxEps;
    }
    const uint32_t lane_base = T + ((uint32_t)(warp * 32) << 16);
    const double* rn = st.tok_rnorm + rq.tok_off[src];
    const float* rnf = st.tok_rnorm_f + rq.tok_off[src];
    for (int i = 0; i < ntiles; ++i) {
      const int b = i & 1;
      const int tb = w.t0 + i * kNT;
      // this tile's 64 norms: two per lane, broadcast by shuffle below
      const float rf0 = tb + lane < w.t1 ? __ldg(rnf + tb + lane) : 0.0f;
      const float rf1 = tb + 32 + lane < w.t1 ? __ldg(rnf + tb + 32 + lane) : 0.0f;
      mbar_wait(&tfull[b], (i >> 1) & 1);
      fence_after();
#pragma unroll 1
      for (int q = 0; q < kNT / 16; ++q) {
        uint32_t r0[16], r1[16], r2[16], r3[16];
        const uint32_t ta = lane_base + b * 256 + q * 16;
        tmem_ld16(ta, r0);
        tmem_ld16(ta + kNT, r1);
        tmem_ld16(ta + 2 * kNT, r2);
        tmem_ld16(ta + 3 * kNT, r3);
        tmem_ld_wait();
        if (q == kNT / 16 - 1) {
          fence_before();
          mbar_arrive(&tempty[b]);
        }
        const float rsrc = q < 2 ? rf0 : rf1;
        float sf[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float rv = __shfl_sync(0xffffffffu, rsrc, (q & 1) * 16 + e);
          const int hi = (int)r0[e] * 128 + (int)r1[e];
          const int lo = (int)r2[e] * 128 + (int)r3[e];
          const int t = tb + q * 16 + e;
          // exact int64 dot, one rounding to f32, one product: |err| <= 3 ulp(|score|)
          const long long d = (long long)hi * 16384 + lo;
          sf[e] = t < w.t1 ? __fmul_rn(__ll2float_rn(d), rv) : -INFINITY;
        }
        if (!mine) continue;
        if (!exact) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x = sf[e];
            if (x > top[M - 1]) {  // sorted insert, register bubble
#pragma unroll
              for (int j = 0; j < M; ++j) {
                const float hiv = fmaxf(top[j], x);
                x = fminf(top[j], x);
                top[j] = hiv;
              }
            }
          }
          continue;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          if (!(sf[e] >= thr)) continue;
          const int t = tb + q * 16 + e;
          const int hi = (int)r0[e] * 128 + (int)r1[e];
          const int lo = (int)r2[e] * 128 + (int)r3[e];
          const double dot = fma((double)hi, 16384.0, (double)lo);
          const uint64_t key = score_key(dot * __ldg(rn + t), t);
          if (hn < k) {
            h[hn * cpb] = key;
            if (++hn == k) {  // heapify, then replace-root mode
              for (int p = k / 2 - 1; p >= 0; --p) heap_sift_min(h, cpb, k, p);
              root = h[0];
            }
          } else if (key > root) {
            heap_replace_root(h, cpb, k, key);
            root = h[0];
          }
        }
      }
    }
    if (mine) {
      if (!exact) {
        part1[part_offset(tile, src, c, jchunk, 1, tile_size)] = top[M - 1];
      } else {
        // full heap: slot 0 = root (k-th best); partial: slot 0 = 0, entries from slot 1
        uint64_t* out = part + part_offset(tile, src, c, jchunk, kmax, tile_size);
        if (hn == k) {
          for (int i = 0; i < k; ++i) out[i] = h[i * cpb];
        } else {
          out[0] = 0ull;
          for (int i = 0; i < k - 1; ++i) out[i + 1] = i < hn ? h[i * cpb] : 0ull;
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 5) tmem_free<512>(T);
}

cudaError_t launch_nn_tc(const Staged& st, const NNCfg& nn, const CUtensorMap& emb_map,
                         uint64_t* part, float* part1, int kmax, int tile_size, int pass,
                         cudaStream_t s) {
  if (st.n_work == 0) return cudaSuccess;
  // heap of cpb x (kmax+1) u64 per CTA: split the 128-candidate tile over 2
  // CTAs when kmax > 128 so that it fits in shared memory
  const int halves = kmax > 128 ? 2 : 1;
  const size_t smem = NNTcSmem::kA + kStages * NNTcSmem::kB + (size_t)kmax * (tile_size / halves) * 8;
  // pass-1 list size chosen by the planner so that nw * M >= k for every
  // chunked source (tav2_stage)
  auto kern = st.p1_m <= 8 ? nn_tc_kernel<8> : nn_tc_kernel<kTopM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(st.n_work, halves);
  kern<<<grid, kTcThreads, smem, s>>>(st, nn, emb_map, part, part1, kmax, tile_size, pass);
  return cudaGetLastError();
}

}  // namespace tav2
