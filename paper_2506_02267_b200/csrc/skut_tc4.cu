// SKUT v4 on the 5th-gen tensor cores for long layouts (192 < S <= 384,
// <= 2 layers; the k_ll = 128 / 256 points of the C5 sweep): one candidate
// per CTA (S_pad <= 256) or per 2-CTA cluster (S_pad <= 384) iteration,
// persistent over candidates.
//
// Reference: encoder.py:161-188 (encode_batch), :196-211 (layer_norm,
// masked_softmax), :314-462 (forward_fused), trainer.py:354-366 (pool + head).
//
// Why a cluster: at S = 352 the keys alone take 352 x 64 x 2 x 2 B = 90 KB of
// shared memory (bf16 hi/lo) and the folded weight images 112 KB, and 352
// row threads with a 64-float residual row each do not fit one SM's register
// file next to the 2 x 128-lane TMEM tiles.  So the S rows are split over
// two SMs (16 row blocks of rpw = S_pad/16 rows; CTA 0 takes blocks 0-3 and
// 12-15, CTA 1 blocks 4-11, so both see the same causal work), and every
// row's key is written to its own CTA's key buffer and, over distributed
// shared memory, to the peer's when the peer's rows can see it.
//
// Same folded algebra and bf16x3 split GEMMs as skut_tc3, with one more
// re-association so that no V' buffer is needed:
//   scores  (a Wq)(a Wk)^T / 8 = (a Wqk) a^T,  Wqk = Wq Wk^T log2(e)/8
//   output  P (a Wv) Wo = (P a) Wvo             (O'' = P a, then O'' Wvo)
// -> the key buffer (a, K-major for S = Q' a^T) is also the B operand of
//    P a, read MN-major (tc_selftest case 5).  S and P live in TMEM in
//    key chunks of <= 128 (the fixed Cauchy-Schwarz shift makes the chunks
//    independent: P = exp2(s - m'), l summed over chunks, O'' accumulated
//    in TMEM), so a 256-column tile holds A (64) + S/P chunk (128) + O'' (64).
//
// Synchronisation: per tile simt/mma mbarriers as skut_tc3; kvready (512
// arrivals: every thread of both CTAs, after its key row, validity bits and
// ||a||^2 are written -- remote ones with release.cluster) and kvfree (4
// tcgen05.commit arrivals multicast to both CTAs: every tile's last P.a of
// the layer) couple the two CTAs; the pooled maxima of the non-head CTA go
// to the head CTA (alternating per item) through DSMEM + poolready.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "encode.cuh"
#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

constexpr int kT4Warps = 8;
constexpr int kT4Threads = 32 * kT4Warps;
constexpr float kLnEps4 = 1e-5f;
constexpr int kT4Chunk = 128;  // keys per S/P chunk
// TMEM columns per tile (base 256 t): D [0, 128): M1 out Q' [0, 64) / S,P
// chunk / M3b out O' [0, 64) / H [0, 32) / ReLU A2 [32, 64) / W2 out
// [64, 128) / pool out [0, 64); O'' = P a accumulator [128, 192); A region
// [192, 256): LN1 out / Q' / O'' split / LN2 out / x (pool).
constexpr uint32_t k4CD = 0, k4CO = 128, k4CA = 192, k4CA2 = 32, k4CW2 = 64;
constexpr int kW4Layer = kImg3WA + kImg3WB;  // the skut_tc3 images, 48 KB per layer

// ---- cluster / distributed shared memory primitives ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_dsmem_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_dsmem_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void atom_or_dsmem(uint32_t addr, uint32_t v) {
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void atom_max_dsmem(uint32_t addr, uint32_t v) {
  asm volatile("red.shared::cluster.max.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_dsmem(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
// wait with cluster-scope acquire (the phase may be completed by arrivals
// of the peer CTA that release its distributed shared memory writes)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{.reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITC_%=;}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(20000u)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// tcgen05.commit arriving on the mbarrier at this offset in every CTA of `mask`
__device__ __forceinline__ void commit_mc_w(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

struct T4Bars {
  uint64_t simt[2], mma[2], m3[2], kvready, kvfree, wfull, poolready[2], order;
};
__shared__ T4Bars t4;

// branch-free row masking (as skut_tc3's t3_keep)
__device__ __forceinline__ float t4_keep(float v, uint32_t m) { return __uint_as_float(__float_as_uint(v) & m); }

static __device__ __forceinline__ uint32_t allowed16_4(uint32_t bits, int k0, int r) {
  const int n = r - k0 + 1;
  const uint32_t causal = 0xffffu >> min(max(16 - n, 0), 16);  // branch-free (skut_tc3)
  return bits & causal;
}

template <bool F16>
__device__ __forceinline__ void t4_split(float a, float b, uint32_t& hi, uint32_t& lo) {
  if constexpr (F16) split_pair_h(a, b, hi, lo);
  else split_pair(a, b, hi, lo);
}
template <bool F16>
__host__ __device__ constexpr uint32_t t4_idesc(int M, int N, int a_mn = 0, int b_mn = 0) {
  return F16 ? idesc_f16(M, N, a_mn, b_mn) : idesc_bf16(M, N, a_mn, b_mn);
}
template <int N, bool F16>
__device__ __forceinline__ void t4_st_split(uint32_t ta, const float* v) {
#pragma unroll
  for (int c = 0; c < N / 16; ++c) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t4_split<F16>(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
    tmem_st8(ta + 8 * c, hi);
    tmem_st8(ta + N / 2 + 8 * c, lo);
  }
}
__device__ __forceinline__ void t4_ld64(uint32_t ta, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  tmem_ld32(ta, r);
  tmem_ld32(ta + 32, r + 32);
  tmem_ld_wait();
}
// pre-norm LayerNorm (encoder.py:196-200, biased variance, eps 1e-5)
__device__ __forceinline__ void t4_layer_norm(const float* x, const float* g, const float* b, float* y) {
  float2 s = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < kDModel; j += 4) {
    s = __fadd2_rn(s, make_float2(x[j], x[j + 1]));
    s1 = __fadd2_rn(s1, make_float2(x[j + 2], x[j + 3]));
  }
  const float mu = ((s.x + s.y) + (s1.x + s1.y)) * (1.0f / 64.0f);
  const float2 nmu = make_float2(-mu, -mu);
  float2 v = make_float2(0.f, 0.f), v1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < kDModel; j += 4) {
    const float2 c = __fadd2_rn(make_float2(x[j], x[j + 1]), nmu);
    const float2 c1 = __fadd2_rn(make_float2(x[j + 2], x[j + 3]), nmu);
    v = __ffma2_rn(c, c, v);
    v1 = __ffma2_rn(c1, c1, v1);
  }
  const float rs = rsqrtf(((v.x + v.y) + (v1.x + v1.y)) * (1.0f / 64.0f) + kLnEps4);
  const float2 rs2 = make_float2(rs, rs);
  const float2* g2 = reinterpret_cast<const float2*>(g);
  const float2* b2 = reinterpret_cast<const float2*>(b);
#pragma unroll
  for (int j = 0; j < kDModel; j += 2) {
    const float2 c = __fmul2_rn(__fadd2_rn(make_float2(x[j], x[j + 1]), nmu), rs2);
    const float2 o = __ffma2_rn(c, g2[j / 2], b2[j / 2]);
    y[j] = o.x;
    y[j + 1] = o.y;
  }
}
// D += A(TMEM hi/lo) x B(smem hi/lo, K-major slabs), 3 terms per k-step
template <int KSTEPS>
__device__ __forceinline__ void t4_mma3(uint32_t d, uint32_t a_col, uint32_t a_lo_off, uint32_t b_hi,
                                        uint32_t b_lo, uint32_t lbo, uint32_t idesc) {
  // k-step-0 descriptors once; k-step j adds j * 2 lbo / 16 to the 14-bit
  // start-address field (as skut_tc3: no per-k-step address rebuild)
  const uint64_t bh0 = sdesc(b_hi, lbo, 128), bl0 = sdesc(b_lo, lbo, 128);
  const uint32_t step16 = (2 * lbo) >> 4;
#pragma unroll
  for (int j = 0; j < KSTEPS; ++j) {
    const uint64_t bh = bh0 + (uint64_t)(j * step16);
    const uint64_t bl = bl0 + (uint64_t)(j * step16);
    mma_bf16_ts_w(d, a_col + 8 * j, bh, idesc, j > 0);
    mma_bf16_ts_w(d, a_col + 8 * j, bl, idesc, 1);
    mma_bf16_ts_w(d, a_col + a_lo_off + 8 * j, bh, idesc, 1);
  }
}

// CL = 2: the 2-CTA cluster layout above (256 < S_pad <= 384).  CL = 1:
// one CTA holds all rows (192 < S_pad <= 256: 8 blocks of S_pad/8 rows,
// tile 0 = blocks 0-3, tile 1 = 7-4 as in skut_tc3), keys 64 KB + weights
// 112 KB; no distributed shared memory.
template <bool F16, int CL>
__global__ void __launch_bounds__(kT4Threads, 1) skut_tc4_kernel(Params p, SkutImages3 img, NNCfg nn, Staged st,
                                                                 const int32_t* idx, int n, float* logits,
                                                                 float* pooled_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ uint32_t valid_w[2][12];  // [item parity] key-validity bitmask, bit r of word r/32
  __shared__ unsigned kmax_s[2][2];    // [item parity][layer] max ||a_j||^2 (f32 bits) over both CTAs
  __shared__ __align__(16) float lnp_s[2][4][kDModel];
  __shared__ float red_s[kT4Warps][kDModel];
  __shared__ float pool_s[2][kDModel];  // [item parity] the peer's column maxima (head CTA)
  __shared__ int pany_s[2];
  __shared__ float z_s[kDModel + kEmbed + kCtx];
  __shared__ float hpart_s[4][kHidden];
  __shared__ float hid_s[kHidden];
  __shared__ int any_s;

  const int S = nn.seq_len;
  const int S_pad = (S + 15) & ~15;
  const int rpw = CL == 2 ? S_pad >> 4 : S_pad >> 3;  // rows per warp block (8 blocks per CTA)
  const int NL = p.num_layers;
  const int wbytes = NL * kW4Layer + kImg3WO;
  uint8_t* Wsm = sm;
  uint8_t* Khi = sm + wbytes;
  uint8_t* Klo = Khi + S_pad * 128;
  const uint32_t wsm = smem_u32(Wsm);
  const uint32_t khi = smem_u32(Khi), klo = smem_u32(Klo);

  const uint32_t crank = CL == 2 ? cluster_rank() : 0u, peer = crank ^ 1u;
  const int pair = CL == 2 ? blockIdx.x >> 1 : blockIdx.x, npairs = CL == 2 ? gridDim.x >> 1 : gridDim.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = warp >> 2, q = warp & 3;
  // row blocks: CTA 0 = {q, 15 - q}, CTA 1 = {4 + q, 11 - q} (tile 0, tile 1)
  const int kb = CL == 1 ? (t == 0 ? q : 7 - q)
                         : (crank == 0 ? (t == 0 ? q : 15 - q) : (t == 0 ? 4 + q : 11 - q));
  const int maxblk = CL == 1 ? (t == 0 ? 3 : 7) : (crank == 0 ? (t == 0 ? 3 : 15) : (t == 0 ? 7 : 11));
  const int NK = (((maxblk + 1) * rpw) + 15) & ~15;  // keys this tile's rows can see
  const int nchunks = (NK + kT4Chunk - 1) / kT4Chunk;
  const bool mapped = lane < rpw;
  const int r = rpw * kb + lane;
  const bool in_seq = mapped && r < S;
  // does the peer's tile see this row's key?  (CTA 1 sees keys < 12 rpw)
  const bool to_peer = CL == 2 && (crank == 1 || t == 0);

  if (tid == 0) {
    mbar_init(&t4.simt[0], 128);
    mbar_init(&t4.simt[1], 128);
    mbar_init(&t4.mma[0], 1);
    mbar_init(&t4.mma[1], 1);
    mbar_init(&t4.m3[0], 1);
    mbar_init(&t4.m3[1], 1);
    mbar_init(&t4.kvready, CL * kT4Threads);
    mbar_init(&t4.kvfree, 2 * CL);
    mbar_init(&t4.wfull, 1);
    mbar_init(&t4.order, 1);
    mbar_init(&t4.poolready[0], kDModel + 1);
    mbar_init(&t4.poolready[1], kDModel + 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  if (tid < 24) (&valid_w[0][0])[tid] = 0u;
  if (tid < 4) (&kmax_s[0][0])[tid] = 0u;
  for (int i = tid; i < NL * 4 * kDModel; i += kT4Threads) {
    const int L = i / (4 * kDModel), w = (i / kDModel) % 4, j = i % kDModel;
    const float* src = w == 0 ? p.ln1_scale[L] : w == 1 ? p.ln1_shift[L] : w == 2 ? p.ln2_scale[L] : p.ln2_shift[L];
    lnp_s[L][w][j] = src[j];
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (taddr_s != 0u) __trap();
  // key rows no CTA writes (a tile's key range rounded up to 16 may reach
  // rows the peer keeps to itself) must hold finite values: P = 0 there,
  // but 0 x NaN would poison P.a
  for (int i = tid; i < S_pad * 16; i += kT4Threads) reinterpret_cast<uint4*>(Khi)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) {  // all weight images, once per CTA (input independent: before the PDL wait)
    mbar_expect_tx(&t4.wfull, (uint32_t)wbytes);
    for (int L = 0; L < NL; ++L) bulk_g2s(Wsm + L * kW4Layer, img.w[L], kW4Layer, &t4.wfull);
    bulk_g2s(Wsm + NL * kW4Layer, img.wout, kImg3WO, &t4.wfull);
  }
  if constexpr (CL == 2) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrival
  else __syncthreads();

  // peer addresses (distributed shared memory)
  uint32_t p_khi = 0, p_klo = 0, p_valid = 0, p_kmax = 0, p_kvready = 0, p_pool = 0, p_pany = 0, p_poolready = 0;
  if constexpr (CL == 2) {
    p_khi = dsmem_addr(khi, peer);
    p_klo = dsmem_addr(klo, peer);
    p_valid = dsmem_addr(smem_u32(&valid_w[0][0]), peer);
    p_kmax = dsmem_addr(smem_u32(&kmax_s[0][0]), peer);
    p_kvready = dsmem_addr(smem_u32(&t4.kvready), peer);
    p_pool = dsmem_addr(smem_u32(&pool_s[0][0]), peer);
    p_pany = dsmem_addr(smem_u32(&pany_s[0]), peer);
    p_poolready = dsmem_addr(smem_u32(&t4.poolready[0]), peer);
  }

  const bool issue_warp = q == 0;
  const uint32_t R = 256u * t;
  const uint32_t lanebase = ((uint32_t)(32 * q) << 16) + R;
  const uint32_t cA = lanebase + k4CA;
  uint32_t n_mma = 0, n_m3 = 0, n_kv = 0, ph_simt = 0, ph_order = 0;
  // tile 1 (the later rows: more keys) is the critical path; tile 0's
  // issuer queues its M1 / first M2 after tile 1's (as skut_tc3)
  // (CL = 2: measured slower -- the cluster-wide kvready couples all four
  // tiles, so no single tile is critical)
  auto order_after_tile1 = [&]() {
#ifndef TAV2_NO_TILE_ORDER
    if (CL == 2) return;
    if (t == 0) {
      mbar_wait(&t4.order, ph_order);
      ph_order ^= 1u;
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&t4.order);
    }
#endif
  };
  auto wait_mma = [&]() {
    __syncwarp();
    mbar_wait_sleep(&t4.mma[t], n_mma & 1);
    ++n_mma;
    fence_after();
  };
  auto done = [&]() {
    fence_before();
    mbar_arrive(&t4.simt[t]);
  };
  auto issuer_wait_simt = [&]() {
    mbar_wait(&t4.simt[t], ph_simt);
    ph_simt ^= 1u;
    fence_after();
  };
  auto wa = [&](int L) { return wsm + L * kW4Layer; };
  auto wb = [&](int L) { return wsm + L * kW4Layer + kImg3WA; };

  griddep_launch();
  griddep_wait();  // idx (select) and tok_feat / cand_unit (prep) complete
  if (issue_warp) {
    mbar_wait(&t4.wfull, 0);
    fence_after();
  }
  const float* pos = p.position_table + (size_t)(in_seq ? r : 0) * kDModel;

  int k = 0;  // local item counter (identical in both CTAs of the pair)
  for (int item = pair; item < n; item += npairs, ++k) {
    const int par = k & 1;
    // the other parity's exchange words are reused by item k + 1: every
    // peer write of item k - 1 is ordered before this CTA's item k (kvready)
    if (tid < 12) valid_w[par ^ 1][tid] = 0u;
    if (tid < 2) kmax_s[par ^ 1][tid] = 0u;
    // ---- K3: gather + encode: x = tok_feat[tok] + [0 | unit(c)] + pos[r] ----
    const int tok = in_seq ? slot_token(st, nn, idx, item, r) : -1;
    const bool ok = in_seq && tok >= 0;
    float x[kDModel];
    {
      const float* tf = st.tok_feat + (size_t)(ok ? tok : 0) * kDModel;
      const float* cu = st.cand_unit + (size_t)item * kEmbed;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float a8[8], b8[8], c8[8];
        ldg256(tf + 8 * j, a8);
        ldg256(pos + 8 * j, b8);
        if (j >= 4) {
          ldg256(cu + 8 * (j - 4), c8);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) c8[e] = 0.0f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) x[8 * j + e] = ok ? (a8[e] + c8[e]) + b8[e] : 0.0f;
      }
    }
    {
      const unsigned b = __ballot_sync(0xffffffffu, ok);  // lanes >= rpw are never ok
      if (lane == 0 && b) {
        const int r0 = rpw * kb;
        const unsigned long long w = (unsigned long long)b << (r0 & 31);
        const int w0 = r0 >> 5;
        atomicOr(&valid_w[par][w0], (uint32_t)w);
        if (CL == 2) atom_or_dsmem(p_valid + 4u * (uint32_t)(12 * par + w0), (uint32_t)w);
        if ((uint32_t)(w >> 32)) {
          atomicOr(&valid_w[par][w0 + 1], (uint32_t)(w >> 32));
          if (CL == 2) atom_or_dsmem(p_valid + 4u * (uint32_t)(12 * par + w0 + 1), (uint32_t)(w >> 32));
        }
      }
    }

    for (int L = 0; L < NL; ++L) {
      // ---- P1: a = LN1(x) -> A (TMEM) and this row's key (both CTAs' smem) ----
      if (n_kv > 0) mbar_wait_cl(&t4.kvfree, (n_kv - 1) & 1);  // every tile's previous P.a retired
      {
        float a[kDModel];
        t4_layer_norm(x, lnp_s[L][0], lnp_s[L][1], a);
        const uint32_t okm = ok ? 0xffffffffu : 0u;
#pragma unroll
        for (int j = 0; j < kDModel; ++j) a[j] = t4_keep(a[j], okm);
        float an2 = 0.0f;
#pragma unroll
        for (int j = 0; j < kDModel; ++j) an2 = fmaf(a[j], a[j], an2);
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) t4_split<F16>(a[2 * i], a[2 * i + 1], hi[i], lo[i]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tmem_st8(cA + 8 * c, hi + 8 * c);
          tmem_st8(cA + 32 + 8 * c, lo + 8 * c);
        }
        if (mapped) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int off = c * (S_pad * 16) + r * 16;
            const uint4 vh = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
            const uint4 vl = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
            *reinterpret_cast<uint4*>(Khi + off) = vh;
            *reinterpret_cast<uint4*>(Klo + off) = vl;
            if (to_peer) {
              st_dsmem_v4(p_khi + off, vh);
              st_dsmem_v4(p_klo + off, vl);
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) an2 = fmaxf(an2, __shfl_xor_sync(0xffffffffu, an2, o));
        if (lane == 0) {
          atomicMax(&kmax_s[par][L], __float_as_uint(an2));
          if (CL == 2) atom_max_dsmem(p_kmax + 4u * (uint32_t)(2 * par + L), __float_as_uint(an2));
        }
        tmem_st_wait();
        fence_proxy_async_all();  // generic-proxy key writes (both CTAs) -> tensor core
        done();
        mbar_arrive(&t4.kvready);
        if (CL == 2) mbar_arrive_dsmem(p_kvready);
      }
      if (issue_warp) {  // M1: Q' = A Wqk   (N = 64: the first 64 rows of the [Wqk|Wvo] image)
        issuer_wait_simt();
        if (t == 0) order_after_tile1();
        t4_mma3<4>(R + k4CD, R + k4CA, 32, wa(L), wa(L) + kImg3WA / 2, 128 * 16, t4_idesc<F16>(128, 64));
        commit_w(&t4.mma[t]);
        if (t == 1) order_after_tile1();
      }
      // ---- P2: Q' -> A; ||q'||^2 (and s_rr = q'_r . a_r in fp32 mode) ----
      wait_mma();
      float qn2 = 0.0f, s_rr = 0.0f;
      {
        float v[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld32(lanebase + k4CD + 32 * h, reinterpret_cast<uint32_t*>(v));
          tmem_ld_wait();
          // (rows that are not ok have a = 0 in A, so Q' is exactly 0)
#pragma unroll
          for (int i = 0; i < 32; ++i) qn2 = fmaf(v[i], v[i], qn2);
          if (F16 && mapped) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int off = (4 * h + c) * (S_pad * 16) + r * 16;
              const uint4 kh = *reinterpret_cast<const uint4*>(Khi + off);
              const uint4 kl = *reinterpret_cast<const uint4*>(Klo + off);
              const uint32_t khw[4] = {kh.x, kh.y, kh.z, kh.w}, klw[4] = {kl.x, kl.y, kl.z, kl.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 a0 = __half22float2(*reinterpret_cast<const __half2*>(&khw[i]));
                const float2 a1 = __half22float2(*reinterpret_cast<const __half2*>(&klw[i]));
                s_rr = fmaf(v[8 * c + 2 * i], a0.x + a1.x, s_rr);
                s_rr = fmaf(v[8 * c + 2 * i + 1], a0.y + a1.y, s_rr);
              }
            }
          }
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) t4_split<F16>(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
            tmem_st8(cA + 16 * h + 8 * c, hi);
            tmem_st8(cA + 32 + 16 * h + 8 * c, lo);
          }
        }
        tmem_st_wait();
        done();
      }
      if (issue_warp) {  // M2 (chunk 0): S = Q' a^T over keys [0, min(NK, 128))
        issuer_wait_simt();
        mbar_wait_cl(&t4.kvready, n_kv & 1);  // every key of this layer in place (both CTAs)
        fence_after();
        const int cc = NK < kT4Chunk ? NK : kT4Chunk;
        if (t == 0) order_after_tile1();
        t4_mma3<4>(R + k4CD, R + k4CA, 32, khi, klo, S_pad * 16, t4_idesc<F16>(128, cc));
        commit_w(&t4.mma[t]);
        if (t == 1) order_after_tile1();
      }
      // ---- P3: causal key-masked softmax over key chunks; O'' = P a in TMEM ----
      // Single pass with the Cauchy-Schwarz shift m' = ||q'_r|| max_j ||a_j||
      // (>= every exp2-domain score of the row): shift invariance makes 1/l
      // the exact normaliser of encoder.py:203-211, and the chunks are
      // independent of each other.
      mbar_wait_cl(&t4.kvready, n_kv & 1);  // kmax_s / valid_w complete (already passed)
      const float m2 = qn2 * __uint_as_float(kmax_s[par][L]);
      float mb = m2 > 0.0f ? m2 * rsqrtf(m2) : 0.0f;  // (no sqrtf slow-path branch; skut_tc3)
      if constexpr (F16) mb = ok ? fmaxf(s_rr, mb - 15.0f) : 0.0f;  // as skut_tc3's fp32 mode
      const float2 nmb = make_float2(-mb, -mb);
      float2 l2 = make_float2(0.f, 0.f);
      const uint32_t cs = lanebase + k4CD;
      for (int c = 0; c < nchunks; ++c) {
        const int k0 = kT4Chunk * c;
        const int cc = min(NK - k0, kT4Chunk);
        const int nch = cc >> 4;
        wait_mma();  // S of chunk c
        // the warp's causal bound in this chunk (warp-uniform): sub-chunks
        // [0, jlast] hold keys <= the warp's last row
        const int wlast = rpw * kb + rpw - 1;
        const int jlast = wlast < k0 ? -1 : min(nch - 1, (wlast - k0) >> 4);
        auto chunk16 = [&](const uint32_t* cur, uint32_t vm, uint32_t tcol) {
          float pv[16];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float2 d = __fadd2_rn(make_float2(__uint_as_float(cur[e]), __uint_as_float(cur[e + 1])), nmb);
            float p0, p1;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(d.x));
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(d.y));
            p0 = ((vm >> e) & 1u) ? p0 : 0.0f;
            p1 = ((vm >> (e + 1)) & 1u) ? p1 : 0.0f;
            pv[e] = p0;
            pv[e + 1] = p1;
            l2 = __fadd2_rn(l2, make_float2(p0, p1));
          }
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if constexpr (F16) split_pair_h(pv[2 * i], pv[2 * i + 1], hi[i], lo[i]);
            else split_pair_t(pv[2 * i], pv[2 * i + 1], hi[i], lo[i]);
          }
          tmem_st8(tcol, hi);
          tmem_st8(tcol + 8, lo);
        };
        if (jlast >= 0) {
          uint32_t sa[16], sb[16];
          tmem_ld16(cs, sa);
          for (int j = 0; j <= jlast; j += 2) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int jj = j + u;
              if (jj > jlast) break;
              tmem_ld_wait();
              uint32_t* cur = u == 0 ? sa : sb;
              uint32_t* nxt = u == 0 ? sb : sa;
              if (jj + 1 <= jlast) tmem_ld16(cs + 16 * (jj + 1), nxt);  // warp-uniform
              const int g = (k0 >> 4) + jj;  // global 16-key sub-chunk
              const uint32_t vw = valid_w[par][g >> 1] >> ((g & 1) * 16);
              const uint32_t vm = allowed16_4(vw, 16 * g, r) & (ok ? 0xffffffffu : 0u);
              chunk16(cur, vm, cs + 16 * jj);
            }
          }
        }
        {  // sub-chunks past the warp's causal bound: P = 0 (P.a reads all cc keys)
          const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          for (int j = jlast + 1; j < nch; ++j) {
            tmem_st8(cs + 16 * j, z);
            tmem_st8(cs + 16 * j + 8, z);
          }
        }
        tmem_st_wait();
        done();
        if (issue_warp) {  // M3 (chunk c): O'' += P a[k0, k0 + cc)  (N = 64, K = cc; a MN-major)
          issuer_wait_simt();
          const uint32_t id = t4_idesc<F16>(128, 64, 0, 1);
          const uint32_t sbo = (uint32_t)S_pad * 16;
          // (16 keys = 2 groups of 8 keys x 128 B per k-step: +16 in the address field)
          const uint64_t bh0 = sdesc(khi + (uint32_t)k0 * 16, 128, sbo), bl0 = sdesc(klo + (uint32_t)k0 * 16, 128, sbo);
          for (int j = 0; j < nch; ++j) {
            const uint64_t bh = bh0 + (uint64_t)(16 * j);
            const uint64_t bl = bl0 + (uint64_t)(16 * j);
            mma_bf16_ts_w(R + k4CO, R + k4CD + 16 * j, bh, id, (c > 0 || j > 0) ? 1u : 0u);
            mma_bf16_ts_w(R + k4CO, R + k4CD + 16 * j, bl, id, 1);
            mma_bf16_ts_w(R + k4CO, R + k4CD + 16 * j + 8, bh, id, 1);
          }
          if (c + 1 < nchunks) {
            // S of the next chunk overwrites P of this one: wait for this
            // chunk's P.a to retire before issuing it
            commit_w(&t4.m3[t]);
            mbar_wait(&t4.m3[t], n_m3 & 1);
            ++n_m3;
            fence_after();
            const int k1 = k0 + kT4Chunk;
            const int c1 = min(NK - k1, kT4Chunk);
            t4_mma3<4>(R + k4CD, R + k4CA, 32, khi + k1 * 16, klo + k1 * 16, S_pad * 16, t4_idesc<F16>(128, c1));
            commit_w(&t4.mma[t]);
          } else {
            commit_w(&t4.mma[t]);
            if (CL == 2) commit_mc_w(&t4.kvfree, 0x3);  // this tile no longer reads either CTA's keys
            else commit_w(&t4.kvfree);
          }
        }
      }
      ++n_kv;
      const float l = l2.x + l2.y;
      const float inv_l = l > 0.0f ? __fdividef(1.0f, l) : 0.0f;  // a valid row always sees itself
      // ---- P4a: O'' -> A (hi/lo) ----
      wait_mma();
      {
        float d[kDModel];
        t4_ld64(lanebase + k4CO, d);
        t4_st_split<64, F16>(cA, d);
        tmem_st_wait();
        done();
      }
      if (issue_warp) {  // M3b: O' = O'' Wvo   (N = 64: rows 64..127 of the [Wqk|Wvo] image)
        issuer_wait_simt();
        t4_mma3<4>(R + k4CD, R + k4CA, 32, wa(L) + 64 * 16, wa(L) + kImg3WA / 2 + 64 * 16, 128 * 16,
                   t4_idesc<F16>(128, 64));
        commit_w(&t4.mma[t]);
      }
      // ---- P4b: x += O' / l ; LN2 -> A ----
      wait_mma();
      {
        float d[kDModel];
        t4_ld64(lanebase + k4CD, d);
        // (a row that is not ok has P = 0: O' = 0 and inv_l = 0, x stays 0)
#pragma unroll
        for (int j = 0; j < kDModel; j += 2) {
          const float2 o = __ffma2_rn(make_float2(d[j], d[j + 1]), make_float2(inv_l, inv_l), make_float2(x[j], x[j + 1]));
          x[j] = o.x;
          x[j + 1] = o.y;
        }
        t4_layer_norm(x, lnp_s[L][2], lnp_s[L][3], d);
        const uint32_t okm = ok ? 0xffffffffu : 0u;
#pragma unroll
        for (int j = 0; j < kDModel; ++j) d[j] = t4_keep(d[j], okm);
        t4_st_split<64, F16>(cA, d);
        tmem_st_wait();
        done();
      }
      if (issue_warp) {  // M4: H = A W1   (N = 32, K = 64)
        issuer_wait_simt();
        t4_mma3<4>(R + k4CD, R + k4CA, 32, wb(L), wb(L) + 4096, 32 * 16, t4_idesc<F16>(128, 32));
        commit_w(&t4.mma[t]);
      }
      // ---- P5: ReLU(H) -> A2 ----
      wait_mma();
      {
        float h[kFfn];
        tmem_ld32(lanebase + k4CD, reinterpret_cast<uint32_t*>(h));
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < kFfn; ++j) h[j] = ok ? fmaxf(h[j], 0.0f) : 0.0f;
        t4_st_split<32, F16>(lanebase + k4CA2, h);
        tmem_st_wait();
        done();
      }
      if (issue_warp) {  // M5: D2 = ReLU(H) W2   (N = 64, K = 32)
        issuer_wait_simt();
        t4_mma3<2>(R + k4CW2, R + k4CA2, 16, wb(L) + 8192, wb(L) + 8192 + 4096, 64 * 16, t4_idesc<F16>(128, 64));
        commit_w(&t4.mma[t]);
      }
      // ---- P6: x += D2 ----
      wait_mma();
      {
        float d[kDModel];
        t4_ld64(lanebase + k4CW2, d);
        // (a row that is not ok has ReLU(H) = 0: D2 = 0, x stays 0)
#pragma unroll
        for (int j = 0; j < kDModel; j += 2) {
          const float2 o = __fadd2_rn(make_float2(d[j], d[j + 1]), make_float2(x[j], x[j + 1]));
          x[j] = o.x;
          x[j + 1] = o.y;
        }
      }
    }

    // ---- K5: y = x out_linear, masked max over rows (both CTAs), CTR head ----
    t4_st_split<64, F16>(cA, x);  // invalid rows carry x = 0
    tmem_st_wait();
    done();
    if (issue_warp) {
      issuer_wait_simt();
      t4_mma3<4>(R + k4CD, R + k4CA, 32, wsm + NL * kW4Layer, wsm + NL * kW4Layer + 8192, 64 * 16,
                 t4_idesc<F16>(128, 64));
      commit_w(&t4.mma[t]);
    }
    wait_mma();
    const bool head = CL == 1 || (uint32_t)par == crank;  // the head alternates between the pair's CTAs
    {
      float y[kDModel];
      t4_ld64(lanebase + k4CD, y);
      if (tid == 0) any_s = 0;
      named_bar_sync(1, kT4Threads);
      if (ok) any_s = 1;
#pragma unroll
      for (int j = 0; j < kDModel; ++j) {
        const float v = warp_max_f32(ok ? y[j] : -INFINITY);
        if (lane == 0) red_s[warp][j] = v;
      }
    }
    named_bar_sync(1, kT4Threads);
    float v = -INFINITY;
    if (tid < kDModel) {
#pragma unroll
      for (int w = 0; w < kT4Warps; ++w) v = fmaxf(v, red_s[w][tid]);
    }
    if (!head) {  // column maxima + any-valid flag -> the head CTA's pool_s[par]
      if (tid < kDModel) {
        st_dsmem_f32(p_pool + 4u * (uint32_t)(kDModel * par + tid), v);
        mbar_arrive_dsmem(p_poolready + 8u * (uint32_t)par);
      } else if (tid == kDModel) {
        st_dsmem_u32(p_pany + 4u * (uint32_t)par, (uint32_t)any_s);
        mbar_arrive_dsmem(p_poolready + 8u * (uint32_t)par);
      }
      continue;
    }
    // head CTA: combine with the peer's maxima (trainer.py:354-359)
    if (CL == 2) mbar_wait_cl(&t4.poolready[par], (k >> 1) & 1);
    if (tid < kDModel) {
      if (CL == 2) v = fmaxf(v, pool_s[par][tid]);
      const bool any = any_s || (CL == 2 && pany_s[par]);
      v = any ? v : 0.0f;  // empty user -> pooled = 0 (trainer.py:358-359)
      z_s[tid] = v;
      if (pooled_out) pooled_out[(size_t)item * kDModel + tid] = v;
    } else if (tid < kDModel + kEmbed) {
      z_s[tid] = st.cand_unit[(size_t)item * kEmbed + tid - kDModel];
    } else if (tid < kDModel + kEmbed + kCtx) {
      z_s[tid] = st.ctx[st.item_req[item] * kCtx + tid - kDModel - kEmbed];
    }
    named_bar_sync(1, kT4Threads);
    {  // head (trainer.py:361-365): 4 threads per hidden unit
      const int hu = tid & 63, part = tid >> 6;
      float acc = 0.0f;
#pragma unroll
      for (int i = 0; i < 26; ++i) acc = fmaf(z_s[26 * part + i], __ldg(p.head_w1 + (26 * part + i) * kHidden + hu), acc);
      hpart_s[part][hu] = acc;
    }
    named_bar_sync(1, kT4Threads);
    if (tid < kHidden) {
      const float hsum = ((hpart_s[0][tid] + hpart_s[1][tid]) + (hpart_s[2][tid] + hpart_s[3][tid])) +
                         __ldg(p.head_b1 + tid);
      hid_s[tid] = fmaxf(hsum, 0.0f);
    }
    named_bar_sync(1, kT4Threads);
    if (warp == 0) {
      const int hd = lane & 3, j0 = 8 * (lane >> 2);
      float o = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) o = fmaf(hid_s[j0 + j], __ldg(p.head_w2 + (j0 + j) * kHeads + hd), o);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) o += __shfl_xor_sync(0xffffffffu, o, off);
      if (lane < kHeads) logits[(size_t)item * kHeads + lane] = o + __ldg(p.head_b2 + lane);
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (CL == 2) cluster_sync_all();  // no distributed shared memory traffic targets an exited CTA
  if (warp == 0) tmem_free<512>(0u);
}


bool skut_tc4_supported(const NNCfg& nn, const Params& p) {
  const int S_pad = (nn.seq_len + 15) & ~15;
  return S_pad > 192 && S_pad <= 384 && p.num_layers >= 1 && p.num_layers <= 2;
}

cudaError_t launch_skut_tc4(const Params& p, const SkutImages3& img, const NNCfg& nn, const Staged& st,
                            const int32_t* idx, int n, float* logits, float* pooled, bool f16, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int S_pad = (nn.seq_len + 15) & ~15;
  const size_t smem = (size_t)p.num_layers * kW4Layer + kImg3WO + 2 * (size_t)S_pad * 128;
  const int CL = S_pad > 256 ? 2 : 1;
  auto kern = CL == 2 ? (f16 ? skut_tc4_kernel<true, 2> : skut_tc4_kernel<false, 2>)
                      : (f16 ? skut_tc4_kernel<true, 1> : skut_tc4_kernel<false, 1>);
  cudaError_t e = set_max_dyn_smem((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int units_max = device_sms() / CL;
  const int units = n < units_max ? n : units_max;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CL * units);
  cfg.blockDim = dim3(kT4Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (CL == 2) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, p, img, nn, st, idx, n, logits, pooled);
}

}  // namespace tav2
