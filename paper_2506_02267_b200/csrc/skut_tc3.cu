// SKUT v3 on the 5th-gen tensor cores (S <= 192, <= 2 layers): gather +
// Eq. 4 encode, 2 x pre-norm causal transformer layers, linear + masked
// max-pool, one candidate per CTA iteration (persistent).  The CTR head on
// the pooled vectors is head_kernel (pool.cu), which starts per candidate
// as the pooled vectors land.
//
// Reference: encoder.py:161-188 (encode_batch), :196-211 (layer_norm,
// masked_softmax), :221-246 / :314-462 (forward_reference / forward_fused),
// trainer.py:354-366 (pool + head).
//
// Versus the reference's layer (encoder.py:229-246) the kernel uses two
// exact algebraic re-associations, folded into the bf16x3 weight images at
// load time (tav2_load_params, f64 products):
//   scores  (a Wq)(a Wk)^T / 8 = (a Wqk) a^T,  Wqk = Wq Wk^T log2(e) / 8
//           -> K is the LN1 output itself and the scores land in the exp2
//              domain of the softmax;
//   output  (P (a Wv)) Wo = P (a Wvo),  Wvo = Wv Wo
//           -> no separate Wo GEMM: x += (P V') / l.
// Per layer this is five MMA <-> SIMT round trips (tc2: six) and ~20% fewer
// tcgen05.mma instructions.  Numerics ("bf16 mode"): every GEMM is a 3-term
// split-bf16 product (a_hi b_hi + a_hi b_lo + a_lo b_hi, f32 accumulation
// in TMEM); residual stream, LN, softmax statistics and the head are f32.
//
// Layout: thread = sequence row; the S_pad rows form 8 blocks of rpw = S_pad/8
// and warp (t, q) owns block q (tile 0) or 7 - q (tile 1): every SM
// sub-partition holds one early and one late block, and tile 0 only needs
// the keys < S_pad/2 (half the score / P.V MMA work).  Two independent
// tiles (warps 4t..4t+3), each with its own TMEM half (256 columns), its own
// simt/mma barriers and issuing warp (warp 4t); they couple only through the
// K/V operands (kready: every row's K and ||a||^2 after P1; kvready: every
// row's V' after P2; kvfree).  All weight images stay resident in
// shared memory for the CTA's lifetime (loaded once); the token features of
// the gather come precomputed from prep_kernel (tok_feat).
//
// TMEM per tile (base 256t): D region [0, 192): QV' out [0,128) / S,P [0,NK)
// / H = W1 out [0,32) / ReLU A2 [32,64) / W2 out [64,128) / pool out [0,64);
// A region [192, 256): LN1 out / Q' / O' (PV out) / LN2 out / x (pool).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "dbg.cuh"
#include "encode.cuh"
#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

constexpr int kT3Warps = 8;
constexpr int kT3Threads = 32 * kT3Warps;
constexpr float kLnEps3 = 1e-5f;
constexpr uint32_t kCA = 192, kCD = 0, kCA2 = 32, kCW2 = 64;

// weight image offsets inside the shared-memory weight region
constexpr int kW3Layer = kImg3WA + kImg3WB;  // 48 KB per layer

// Debug (libtav2_debug.so): clock64 accumulated per code segment of the two
// tile leaders (thread 0 / 128: row thread + MMA issuer) of CTA 0 over all its
// candidates: g_dbg_skut3[32 * tile + segment], [32 * tile + 31] = items.
__device__ long long* g_dbg_skut3 = nullptr;

struct T3Bars {
  uint64_t simt[2], mma[2], kready, kvready, kvfree, wfull, order;
};
__shared__ __align__(8) T3Bars t3;

// allowed keys k0..k0+15 for query row r: key-valid bits (low 16 of `bits`)
// AND causal (key <= r)
static __device__ __forceinline__ uint32_t allowed16(uint32_t bits, int k0, int r) {
  const int n = r - k0 + 1;  // keys k0..r are causal-visible
  // branch-free: the select form compiled to a divergent branch around the
  // mask in every exp-loop chunk (measured: skut_tc3 -2.9%)
  const uint32_t causal = 0xffffu >> min(max(16 - n, 0), 16);
  return bits & causal;
}

// v if m = ~0, +0 if m = 0: branch-free row masking (an `if (!ok)` block
// around a register array is a divergent branch in every warp: its lanes
// >= rows-per-warp are never ok)
__device__ __forceinline__ float t3_keep(float v, uint32_t m) { return __uint_as_float(__float_as_uint(v) & m); }

__device__ __forceinline__ void t3_ld64(uint32_t ta, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  tmem_ld32(ta, r);
  tmem_ld32(ta + 32, r + 32);
  tmem_ld_wait();
}
// The operand format: F16 = false: bf16 hi/lo parts (bf16 mode); true: fp16
// hi/lo parts (fp32 mode: 11-bit significands, ~2^-22 per 3-term product;
// the softmax then uses the true row max so P stays in [0, 1], inside fp16's
// normal range -- tools/split_precision_err.py).
template <bool F16>
__device__ __forceinline__ void t3_split(float a, float b, uint32_t& hi, uint32_t& lo) {
  if constexpr (F16) split_pair_h(a, b, hi, lo);
  else split_pair(a, b, hi, lo);
}
template <bool F16>
__host__ __device__ constexpr uint32_t t3_idesc(int M, int N, int a_mn = 0, int b_mn = 0) {
  return F16 ? idesc_f16(M, N, a_mn, b_mn) : idesc_bf16(M, N, a_mn, b_mn);
}
// split n floats into packed hi/lo pairs: hi at [0, n/2), lo at [n/2, n)
template <int N, bool F16>
__device__ __forceinline__ void t3_st_split(uint32_t ta, const float* v) {
#pragma unroll
  for (int c = 0; c < N / 16; ++c) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t3_split<F16>(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
    tmem_st8(ta + 8 * c, hi);
    tmem_st8(ta + N / 2 + 8 * c, lo);
  }
}
template <bool F16>
__device__ __forceinline__ void t3_split8_store(uint8_t* hi_dst, uint8_t* lo_dst, const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) t3_split<F16>(v[2 * i], v[2 * i + 1], h[i], l[i]);
  *reinterpret_cast<uint4*>(hi_dst) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(lo_dst) = make_uint4(l[0], l[1], l[2], l[3]);
}
// pre-norm LayerNorm (encoder.py:196-200, biased variance, eps 1e-5)
// (paired f32x2 arithmetic: FADD2 / FMUL2 / FFMA2 on sm_100)
__device__ __forceinline__ void t3_layer_norm(const float* x, const float* g, const float* b, float* y) {
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
  const float rs = rsqrtf(((v.x + v.y) + (v1.x + v1.y)) * (1.0f / 64.0f) + kLnEps3);
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

// D += A(TMEM hi/lo) x B(smem hi/lo, K-major slabs), 3 terms per k-step;
// warp-collective (one elected lane issues), fully unrolled.  bh0 / bl0 are
// the k-step-0 B descriptors (precomputed per CTA in desc_s); k-step j adds
// j * step16 to the 14-bit start-address field (step16 = 2 lbo / 16; smem
// addresses < 256 KB never carry out of the field).  (Building each
// descriptor from the shared-window address instead cost an S2R + LDC +
// address chain per k-step: the register-starved kernel rematerialises it.)
template <int KSTEPS, bool ACC = false>  // ACC: accumulate onto D from the first k-step
__device__ __forceinline__ void t3_mma3(uint32_t d, uint32_t a_col, uint32_t a_lo_off, uint64_t bh0,
                                        uint64_t bl0, uint32_t step16, uint32_t idesc) {
#pragma unroll
  for (int j = 0; j < KSTEPS; ++j) {
    const uint64_t bh = bh0 + (uint64_t)(j * step16);
    const uint64_t bl = bl0 + (uint64_t)(j * step16);
    mma_bf16_ts_w(d, a_col + 8 * j, bh, idesc, ACC || j > 0);
    mma_bf16_ts_w(d, a_col + 8 * j, bl, idesc, 1);
    mma_bf16_ts_w(d, a_col + a_lo_off + 8 * j, bh, idesc, 1);
  }
}

template <bool F16>
__global__ void __launch_bounds__(kT3Threads, 1) skut_tc3_kernel(
    Params p, SkutImages3 img, NNCfg nn, Staged st, const int32_t* idx, int n, float* logits,
    float* pooled_out, SelFlags sel) {
  extern __shared__ __align__(1024) uint8_t sm[];
  cta_stamp(kDbgSkut, 0);
  __shared__ uint32_t taddr_s;
  // B-operand descriptors of every GEMM at k-step 0: [2L, 2L+1] M1 (layer L
  // hi / lo), [4, 5] M2 keys, [6, 7] M3 V', [8 + 2L ..] M4, [12 + 2L ..] M5,
  // [16, 17] pool, [18, 19] W2 W_out (the fused last-layer pool GEMM)
  __shared__ uint64_t desc_s[20];
  __shared__ uint32_t valid_w[8];  // key-validity bitmask, bit r of word r/32
  __shared__ __align__(16) float lnp_s[2][4][kDModel];
  __shared__ float red_s[kT3Warps][kDModel];
  __shared__ int any_s;
  __shared__ int nx_s;  // the item after the next one (dynamic rounds)
  __shared__ unsigned kmax_s[2];

  const int S = nn.seq_len;
  const int S_pad = (S + 15) & ~15;
  const int NL = p.num_layers;
  const int wbytes = NL * kW3Layer + kImg3WO + kImg3W2O;
  uint8_t* Wsm = sm;
  uint8_t* Khi = sm + wbytes;
  uint8_t* Klo = Khi + S_pad * 128;
  uint8_t* Vhi = Klo + S_pad * 128;
  uint8_t* Vlo = Vhi + S_pad * 128;
  const uint32_t wsm = smem_u32(Wsm);
  const uint32_t khi = smem_u32(Khi), klo = smem_u32(Klo), vhi = smem_u32(Vhi), vlo = smem_u32(Vlo);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = warp >> 2, q = warp & 3;
  const int rpw = S_pad >> 3;
  // row blocks: tile 0 = blocks 0-3 (keys < S_pad/2 only), tile 1 = 7-4, so
  // each SM sub-partition q holds one early and one late block
  const int kb = t == 0 ? q : 7 - q;
  const bool mapped = lane < rpw;
  const int r = rpw * kb + lane;
  const int NK = t == 0 ? (((S_pad >> 1) + 15) & ~15) : S_pad;  // keys this tile's rows can see
  if (tid == 0) {
    mbar_init(&t3.simt[0], 128);
    mbar_init(&t3.simt[1], 128);
    mbar_init(&t3.mma[0], 1);
    mbar_init(&t3.mma[1], 1);
    mbar_init(&t3.kready, kT3Threads);
    mbar_init(&t3.kvready, kT3Threads);
    mbar_init(&t3.kvfree, 2);
    mbar_init(&t3.wfull, 1);
    mbar_init(&t3.order, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  if (tid < 8) valid_w[tid] = 0u;
  if (tid < 2) kmax_s[tid] = 0u;
  if (tid == 0) {
    for (int L = 0; L < NL; ++L) {
      const uint32_t a = wsm + L * kW3Layer, b = a + kImg3WA;
      desc_s[2 * L] = sdesc(a, 128 * 16, 128);
      desc_s[2 * L + 1] = sdesc(a + kImg3WA / 2, 128 * 16, 128);
      desc_s[8 + 2 * L] = sdesc(b, 32 * 16, 128);
      desc_s[9 + 2 * L] = sdesc(b + 4096, 32 * 16, 128);
      desc_s[12 + 2 * L] = sdesc(b + 8192, 64 * 16, 128);
      desc_s[13 + 2 * L] = sdesc(b + 8192 + 4096, 64 * 16, 128);
    }
    desc_s[4] = sdesc(khi, S_pad * 16, 128);
    desc_s[5] = sdesc(klo, S_pad * 16, 128);
    desc_s[6] = sdesc(vhi, 1024, 128);
    desc_s[7] = sdesc(vlo, 1024, 128);
    desc_s[16] = sdesc(wsm + NL * kW3Layer, 64 * 16, 128);
    desc_s[17] = sdesc(wsm + NL * kW3Layer + 8192, 64 * 16, 128);
    desc_s[18] = sdesc(wsm + NL * kW3Layer + kImg3WO, 64 * 16, 128);
    desc_s[19] = sdesc(wsm + NL * kW3Layer + kImg3WO + 4096, 64 * 16, 128);
  }
  for (int i = tid; i < NL * 4 * kDModel; i += kT3Threads) {
    const int L = i / (4 * kDModel), w = (i / kDModel) % 4, j = i % kDModel;
    const float* src = w == 0 ? p.ln1_scale[L] : w == 1 ? p.ln1_shift[L] : w == 2 ? p.ln2_scale[L] : p.ln2_shift[L];
    lnp_s[L][w][j] = src[j];
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (taddr_s != 0u) __trap();  // a 512-column allocation always starts at column 0
  if (tid == 0) {  // all weight images, once per CTA (input independent: before the PDL wait)
    mbar_expect_tx(&t3.wfull, (uint32_t)wbytes);
    for (int L = 0; L < NL; ++L) bulk_g2s(Wsm + L * kW3Layer, img.w[L], kW3Layer, &t3.wfull);
    bulk_g2s(Wsm + NL * kW3Layer, img.wout, kImg3WO, &t3.wfull);
    bulk_g2s(Wsm + NL * kW3Layer + kImg3WO, img.w2out, kImg3W2O, &t3.wfull);
  }

  const bool issuer = (tid & 127) == 0;  // debug stamps only
  const bool issue_warp = q == 0;         // warp 4t issues tile t's MMAs (warp-collective)
  long long* dbg = (kDebug && blockIdx.x == 0 && issuer && g_dbg_skut3) ? g_dbg_skut3 + 32 * (tid >> 7) : nullptr;
  long long t_last = 0, dbg_m3 = 0;
  auto stamp = [&](int id) {
    if (kDebug && dbg) {
      const long long now = clock64();
      dbg[id] += now - t_last;
      t_last = now;
    }
  };
  const uint32_t R = 256u * t;
  const uint32_t lanebase = ((uint32_t)(32 * q) << 16) + R;
  const uint32_t cA = lanebase + kCA;
  const bool in_seq = mapped && r < S;
  uint32_t n_mma = 0, n_kv = 0;
  uint32_t ph_simt = 0, ph_order = 0;
  // Tile 1 (the late rows: twice the attention work) is the critical path;
  // the two tiles share the SM's tensor pipe and issue M1 and M2 at the
  // same moments, so tile 0's issuer waits until tile 1's MMAs of that
  // phase are queued (tile 0 has slack: it waits at kvfree / the pool).
  auto order_after_tile1 = [&]() {
#ifndef TAV2_NO_TILE_ORDER
    if (t == 0) {
      mbar_wait(&t3.order, ph_order);
      ph_order ^= 1u;
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&t3.order);
    }
#endif
  };
  auto wait_mma = [&]() {
    __syncwarp();
    mbar_wait_sleep(&t3.mma[t], n_mma & 1);
    ++n_mma;
    fence_after();
  };
  auto done = [&]() {
    fence_before();
    mbar_arrive(&t3.simt[t]);
  };
  auto issuer_wait_simt = [&]() {
    mbar_wait(&t3.simt[t], ph_simt);
    ph_simt ^= 1u;
    fence_after();
  };

  griddep_launch();
  // NN selection (idx) and prep (tok_feat, cand_unit) complete: the whole
  // select grid, or (SelFlags) prep .. scan2 -- the select kernel lets this
  // grid launch only after its griddep_wait -- plus, per candidate, its
  // three select flags (sel_ready, checked before the candidate's idx reads)
  if (!sel.done) griddep_wait();
  if (sel.done && (int)blockIdx.x < n && tid < 3) {  // the first candidate's three selections
    const uint32_t ep = ld_acquire_gpu(sel.epoch);  // this run's epoch (bumped by prep)
    while (ld_acquire_gpu(sel.done + 3 * blockIdx.x + tid) != ep) __nanosleep(100);
  }
  if (sel.done) __syncthreads();
  bool sel_all = !sel.done;  // the whole select grid is complete and visible
  cta_stamp(kDbgSkut, 2);
  if (issue_warp) {
    mbar_wait(&t3.wfull, 0);
    fence_after();
    cta_stamp(8, 2);  // (debug) weights landed
  }
  const float4* pos4 = reinterpret_cast<const float4*>(p.position_table + (size_t)(in_seq ? r : 0) * kDModel);

  // the gather's index chain (idx -> token) of the next candidate is resolved
  // during the last layer of the current one
  int tok_pf = (in_seq && (int)blockIdx.x < n) ? slot_token(st, nn, idx, blockIdx.x, r) : -1;
  int pf_idx = -1, pf_req = 0, pf_off = 0;  // the next item's index chain, in flight
  const int r_src = r < nn.seg_start[1] ? 0 : (r < nn.seg_start[3] ? 1 : 2);  // this row's source
  // Tile 1's rows' position embeddings stay in TMEM for the kernel's
  // lifetime: tile 0's columns [128, 192) are never used by tile 0 (its
  // scores span <= 96 keys, its widest output 128 columns), and tile 1's
  // warp q shares tile 0's warp q lane quadrant.  Saves tile 1 -- the
  // critical tile -- 16 of its 40 row-per-thread global loads per item.
  const uint32_t pos_t = ((uint32_t)(32 * q) << 16) + 128u;
  if (t == 1) {
    float pp[kDModel];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float4 b = in_seq ? __ldg(pos4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
      pp[4 * j] = b.x; pp[4 * j + 1] = b.y; pp[4 * j + 2] = b.z; pp[4 * j + 3] = b.w;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_st16(pos_t + 16 * c, reinterpret_cast<const uint32_t*>(pp + 16 * c));
    tmem_st_wait();
  }
  // this row's token features of the item about to be encoded: loaded for the
  // first item here, for the next one during the current item's pooling
  // (its 32-byte loads then overlap the pool and head phases)
  float tfv[kDModel];
  {
    const size_t tr = (in_seq && tok_pf >= 0) ? (size_t)tok_pf : 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) ldg256(st.tok_feat + tr * kDModel + 8 * j, tfv + 8 * j);
  }
  // Items: the first two rounds round-robin, then a counter (sel.next_item,
  // zeroed by prep): a CTA that started late or ran slow takes fewer of the
  // last rounds' items.  The claim for item k+2 is made in item k's last
  // layer and handed over in nx_s at its pool barrier; the next item is then
  // known a whole layer ahead (its index chain is prefetched there).
  int nx = 0;
  uint32_t claim = 0u;
  for (int item = blockIdx.x; item < n; item = nx) {
    if (kDebug && dbg) {
      dbg[31] += 1;
      t_last = clock64();
    }
    // ---- K3: gather + encode: x = tok_feat[tok] + pos[r] + [0 | unit(c)] ----
    // (the token row tfv was loaded during the previous item's head; x is
    // built 16 columns at a time so x and tfv do not both stay live)
    float x[kDModel];
    const bool ok = in_seq && tok_pf >= 0;
    {
      const float* cu = st.cand_unit + (size_t)item * kEmbed;
      const float* pr = p.position_table + (size_t)(in_seq ? r : 0) * kDModel;
#pragma unroll
      for (int c16 = 0; c16 < 4; ++c16) {
        float pp[16], cc[16];
        if (t == 1) {  // position rows from TMEM (warp-uniform branch)
          tmem_ld16(pos_t + 16 * c16, reinterpret_cast<uint32_t*>(pp));
          tmem_ld_wait();
        } else {
          ldg256(pr + 16 * c16, pp);
          ldg256(pr + 16 * c16 + 8, pp + 8);
        }
        if (c16 >= 2) {
          ldg256(cu + 16 * (c16 - 2), cc);
          ldg256(cu + 16 * (c16 - 2) + 8, cc + 8);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) cc[e] = 0.0f;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) x[16 * c16 + e] = (tfv[16 * c16 + e] + cc[e]) + pp[e];
      }
    }
    const uint32_t okm = ok ? 0xffffffffu : 0u;  // this row's mask for the item
#pragma unroll
    for (int j = 0; j < kDModel; ++j) x[j] = t3_keep(x[j], okm);
    {
      const unsigned b = __ballot_sync(0xffffffffu, ok);  // lanes >= rpw are never ok
      if (lane == 0 && b) {
        const int r0 = rpw * kb;
        const unsigned long long w = (unsigned long long)b << (r0 & 31);
        atomicOr(&valid_w[r0 >> 5], (uint32_t)w);
        if ((uint32_t)(w >> 32)) atomicOr(&valid_w[(r0 >> 5) + 1], (uint32_t)(w >> 32));
      }
    }
    stamp(0);
    // (no barrier: valid_w is read only in the softmax, after kready -- every
    // thread arrives there after its own validity bits)
    stamp(1);

    for (int L = 0; L < NL; ++L) {
      if (L == NL - 1) {
        if (!sel_all) {
          cta_stamp(9, 1);  // (debug) first item's last layer reached
          griddep_wait();
          cta_stamp(9, 0);  // (debug) select grid complete
          sel_all = true;
        }
        // (nx_s was written by tid 0 before the previous item's pool barrier)
        nx = (sel.next_item == nullptr || item < (int)gridDim.x) ? item + (int)gridDim.x : nx_s;
        if (sel.next_item != nullptr && tid == 0) claim = atomicAdd(sel.next_item, 1u);  // consumed at the pool
#ifdef TAV2_OLD_PF
        tok_pf = (in_seq && nx < n) ? slot_token(st, nn, idx, nx, r) : -1;
#else
        // The next item's index chain (slot_token: idx -> item_req -> req
        // tok_off) in three steps whose loads are consumed a phase later:
        // here idx and item_req (independent), the request's token offset
        // after P2, the sum at the pool.  (slot_token here put its dependent
        // L2 round trips on the critical tile's path at the layer top.)
        pf_idx = (in_seq && nx < n) ? idx[(size_t)nx * S + r] : -1;
        pf_req = nx < n ? st.item_req[nx] : 0;
#endif
      }
      // ---- P1: a = LN1(x) -> A (TMEM) and K = a (smem); ||a||^2 -> kmax ----
      if (n_kv > 0) mbar_wait_sleep(&t3.kvfree, (n_kv - 1) & 1);  // both tiles' previous P.V retired
      stamp(2);
      {
        float a[kDModel];
        t3_layer_norm(x, lnp_s[L][0], lnp_s[L][1], a);
        float an2 = 0.0f;
#pragma unroll
        for (int j = 0; j < kDModel; ++j) a[j] = t3_keep(a[j], okm);
#pragma unroll
        {  // the shift's max ||a_j||: paired FFMA2 chains (a 64-deep FMA chain was ~260 cycles)
          float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < kDModel; j += 4) {
            s0 = __ffma2_rn(make_float2(a[j], a[j + 1]), make_float2(a[j], a[j + 1]), s0);
            s1 = __ffma2_rn(make_float2(a[j + 2], a[j + 3]), make_float2(a[j + 2], a[j + 3]), s1);
          }
          an2 = (s0.x + s0.y) + (s1.x + s1.y);
        }
        // one bf16 hi/lo split of a, stored twice: the M1 A operand (TMEM,
        // warp-collective: never under a divergent branch) and this row's K
        // (K-major smem slabs: chunk c of row r at c*(S_pad*16) + r*16)
        {
          uint32_t hi[32], lo[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) t3_split<F16>(a[2 * i], a[2 * i + 1], hi[i], lo[i]);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tmem_st8(cA + 8 * c, hi + 8 * c);
            tmem_st8(cA + 32 + 8 * c, lo + 8 * c);
          }
          if (mapped) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const int off = c * (S_pad * 16) + r * 16;
              *reinterpret_cast<uint4*>(Khi + off) = make_uint4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
              *reinterpret_cast<uint4*>(Klo + off) = make_uint4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) an2 = fmaxf(an2, __shfl_xor_sync(0xffffffffu, an2, o));
        if (lane == 0) atomicMax(&kmax_s[L], __float_as_uint(an2));
        tmem_st_wait();
        fence_proxy_async();  // K (smem) -> the M2s of both tiles
        fence_before();
        mbar_arrive(&t3.kready);
        done();
      }
      stamp(3);
      if (issue_warp) {  // M1: [Q' | V'] = A [Wqk | Wvo]   (N = 128, K = 64)
        issuer_wait_simt();
        stamp(28);
        if (t == 0) order_after_tile1();
        t3_mma3<4>(R + kCD, R + kCA, 32, desc_s[2 * L], desc_s[2 * L + 1], (2 * 128 * 16) >> 4, t3_idesc<F16>(128, 128));
        commit_w(&t3.mma[t]);
        if (t == 1) order_after_tile1();
      }
      stamp(4);
      // ---- P2: Q' -> A, V' -> smem (MN-major) ----
#ifndef TAV2_OLD_PF
      if (L == NL - 1 && in_seq) pf_off = st.req[pf_req].tok_off[r_src];
#endif
      wait_mma();
      stamp(5);
      float s_rr = 0.0f, qn2;
      float2 qa = make_float2(0.f, 0.f), qb = make_float2(0.f, 0.f);  // ||q'||^2 in paired chains
      {
        float v[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          tmem_ld32(lanebase + kCD + 32 * h, reinterpret_cast<uint32_t*>(v));
          tmem_ld_wait();
          // (rows that are not ok have a = 0 in A, so Q' and V' are exactly 0)
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            qa = __ffma2_rn(make_float2(v[i], v[i + 1]), make_float2(v[i], v[i + 1]), qa);
            qb = __ffma2_rn(make_float2(v[i + 2], v[i + 3]), make_float2(v[i + 2], v[i + 3]), qb);
          }
          if (F16 && mapped) {  // s_rr = q'_r . a_r from this row's K (fp16 hi + lo parts)
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
            for (int i = 0; i < 8; ++i) t3_split<F16>(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
            tmem_st8(cA + 16 * h + 8 * c, hi);
            tmem_st8(cA + 32 + 16 * h + 8 * c, lo);
          }
        }
        qn2 = (qa.x + qa.y) + (qb.x + qb.y);
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // V': (key r, d) at (r/8)*1024 + (d/8)*128 + (r%8)*16 + (d%8)*2
          tmem_ld32(lanebase + kCD + 64 + 32 * h, reinterpret_cast<uint32_t*>(v));
          tmem_ld_wait();
          if (mapped) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int off = (r >> 3) * 1024 + (4 * h + c) * 128 + (r & 7) * 16;
              t3_split8_store<F16>(Vhi + off, Vlo + off, v + 8 * c);
            }
          }
        }
        tmem_st_wait();
        fence_proxy_async();
        fence_before();
        mbar_arrive(&t3.kvready);  // this row's V' is in place (the M3s)
        done();                    // this tile's Q' is in place (its M2)
      }
      stamp(6);
      if (issue_warp) {  // M2: S = Q' K^T   (N = keys of this tile, K = 64)
        // this tile's Q' plus every row's K (P1): the M2 no longer waits for
        // the other tile's P2 (V' is needed only by the M3s)
        issuer_wait_simt();
        mbar_wait(&t3.kready, n_kv & 1);
        fence_after();
        if (t == 0) order_after_tile1();
        t3_mma3<4>(R + kCD, R + kCA, 32, desc_s[4], desc_s[5], 2 * S_pad, t3_idesc<F16>(128, NK));
        commit_w(&t3.mma[t]);
        if (t == 1) order_after_tile1();
      }
      stamp(7);
      // ---- P3: causal key-masked softmax -> P (bf16 hi/lo, in place over S) ----
      // Single pass with the Cauchy-Schwarz shift m' = ||q'_r|| max_j ||a_j||
      // (>= q'_r . a_j, the exp2-domain score): shift invariance makes 1/l the
      // exact normaliser of encoder.py:203-211.
      wait_mma();
      stamp(8);
      float inv_l = 0.0f;
      {
        const uint32_t cs = lanebase + kCD;
        const int nch = NK / 16;
        const int jlast = min(nch - 1, (rpw * kb + rpw - 1) / 16);  // warp-uniform causal bound
        float mb;
        mbar_wait_sleep(&t3.kready, n_kv & 1);  // kmax_s[L] complete (already passed)
        stamp(24);
        {  // Cauchy-Schwarz: >= every score of the row (up to the MUFU rsqrt's
           // ~2 ulp: any shift works, this one keeps exp2 in range)
          const float m2 = qn2 * __uint_as_float(kmax_s[L]);
          mb = m2 > 0.0f ? m2 * rsqrtf(m2) : 0.0f;
        }
        if constexpr (F16) {
          // fp32 mode (fp16 P parts): shift by the row's own diagonal score
          // where the bound allows, m' = max(s_rr, m_cs - 15): then P_rr = 1
          // (no underflow of the largest P's in fp16) unless the bound
          // overshoots the diagonal by > 15 binades, and always
          // P <= 2^(m_cs - m') <= 2^15 < fp16 max (no overflow)
          mb = ok ? fmaxf(s_rr, mb - 15.0f) : 0.0f;
        }
        const float2 nmb = make_float2(-mb, -mb);
        float2 l2 = make_float2(0.f, 0.f);
        // p = exp2(s - m') for one 16-key chunk, masked keys -> 0 (MASK: the
        // warp has a causal-diagonal or invalid key in the chunk)
        auto chunk = [&](const uint32_t* cur, uint32_t vm, uint32_t tcol, auto mask) {
          float pv[16];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float2 d = __fadd2_rn(make_float2(__uint_as_float(cur[e]), __uint_as_float(cur[e + 1])), nmb);
            float p0, p1;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(d.x));
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(d.y));
            if constexpr (decltype(mask)::value) {
              p0 = ((vm >> e) & 1u) ? p0 : 0.0f;
              p1 = ((vm >> (e + 1)) & 1u) ? p1 : 0.0f;
            }
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
        // the causal chunks, one at a time with the next chunk's TMEM load in
        // flight while this one is exponentiated (2-deep software pipeline)
        // 32-key pairs of chunks per TMEM load: tcgen05.wait::ld waits for
        // every load in flight, so a pair in flight while the previous pair
        // is exponentiated doubles the latency each load can hide (-1.5%
        // against 16-key chunks once the mask was branch-free)
        auto exp_pass = [&]() {
          uint32_t sa[32], sb[32];
          tmem_ld32(cs, sa);
          for (int j = 0; j <= jlast; j += 4) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int jj = j + 2 * u;  // this pair's first chunk
              if (jj > jlast) break;
              tmem_ld_wait();
              uint32_t* cur = u == 0 ? sa : sb;
              uint32_t* nxt = u == 0 ? sb : sa;
              if (jj + 2 <= jlast) tmem_ld32(cs + 16 * (jj + 2), nxt);  // warp-uniform
              const uint32_t vw = valid_w[jj >> 1];
              chunk(cur, allowed16(vw, 16 * jj, r) & okm, cs + 16 * jj, std::true_type{});
              if (jj + 1 <= jlast) chunk(cur + 16, allowed16(vw >> 16, 16 * (jj + 1), r) & okm, cs + 16 * (jj + 1), std::true_type{});
            }
          }
        };

        exp_pass();
        const int jz = jlast + 1;
        stamp(25);
        {  // chunks past the warp's causal bound: P = 0 (the P.V MMA reads all NK keys)
          const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          for (int j = jz; j < nch; ++j) {
            tmem_st8(cs + 16 * j, z);
            tmem_st8(cs + 16 * j + 8, z);
          }
        }
        const float l = l2.x + l2.y;
        stamp(26);
        // a valid row always sees itself (l >= P_rr > 0); the approximate
        // reciprocal (2 ulp) keeps the IEEE division's slow-path branch out
        inv_l = l > 0.0f ? __fdividef(1.0f, l) : 0.0f;
        tmem_st_wait();
        done();
      }
      stamp(9);
      if (issue_warp) {  // M3: O' = P V'   (N = 64, K = keys; V' MN-major)
        issuer_wait_simt();
        mbar_wait(&t3.kvready, n_kv & 1);  // every row's V' (tile 0's keys may reach into tile 1's rows)
        fence_after();
        stamp(29);
        const uint32_t id = t3_idesc<F16>(128, 64, 0, 1);
        const int nk16 = NK / 16;  // <= 12 (S_pad <= 192); unrolled, warp-uniform bound
        const uint64_t bv_hi = desc_s[6], bv_lo = desc_s[7];
        const long long t_iss = kDebug ? clock64() : 0;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          if (j < nk16) {
            const uint64_t bh = bv_hi + (uint64_t)(j * ((2 * 1024) >> 4));
            const uint64_t bl = bv_lo + (uint64_t)(j * ((2 * 1024) >> 4));
            mma_bf16_ts_w(R + kCA, R + kCD + 16 * j, bh, id, j > 0);
            mma_bf16_ts_w(R + kCA, R + kCD + 16 * j, bl, id, 1);
            mma_bf16_ts_w(R + kCA, R + kCD + 16 * j + 8, bh, id, 1);
          }
        }
        commit_w(&t3.mma[t]);
        commit_w(&t3.kvfree);  // this tile no longer reads K / V' of this layer
        if (kDebug) dbg_m3 += clock64() - t_iss;  // the M3 issue alone, no stamp in between
      }
      stamp(10);
      ++n_kv;
      // ---- P4: x += O' / l ; LN2 -> A ----
      wait_mma();
      stamp(11);
      {
        float d[kDModel];
        t3_ld64(cA, d);
        // (a row that is not ok has P = 0: O' = 0 and inv_l = 0, x stays 0)
#pragma unroll
        for (int j = 0; j < kDModel; j += 2) {
          const float2 o = __ffma2_rn(make_float2(d[j], d[j + 1]), make_float2(inv_l, inv_l), make_float2(x[j], x[j + 1]));
          x[j] = o.x;
          x[j + 1] = o.y;
        }
        t3_layer_norm(x, lnp_s[L][2], lnp_s[L][3], d);
#pragma unroll
        for (int j = 0; j < kDModel; ++j) d[j] = t3_keep(d[j], okm);
        t3_st_split<64, F16>(cA, d);
        tmem_st_wait();
        done();
      }
      stamp(12);
      if (issue_warp) {  // M4: H = A W1   (N = 32, K = 64)
        issuer_wait_simt();
        stamp(30);
        t3_mma3<4>(R + kCD, R + kCA, 32, desc_s[8 + 2 * L], desc_s[9 + 2 * L], (2 * 32 * 16) >> 4, t3_idesc<F16>(128, 32));
        commit_w(&t3.mma[t]);
      }
      stamp(13);
      // ---- P5: ReLU(H) -> A2 ----
      wait_mma();
      stamp(14);
      {
        float h[kFfn];
        tmem_ld32(lanebase + kCD, reinterpret_cast<uint32_t*>(h));
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < kFfn; ++j) h[j] = t3_keep(fmaxf(h[j], 0.0f), okm);
        t3_st_split<32, F16>(lanebase + kCA2, h);
#ifndef TAV2_POOL_UNFUSED
        // last layer: x_mid -> A as well (M4 has consumed LN2's output): the
        // pooled projection of the layer output x_mid + ReLU(H) W2 is
        // x_mid W_out + ReLU(H) (W2 W_out) -- one GEMM, no M5 / P6 / pool store
        if (L == NL - 1) t3_st_split<64, F16>(cA, x);  // invalid rows carry x = 0
#endif
        tmem_st_wait();
        done();
      }
      stamp(15);
#ifndef TAV2_POOL_UNFUSED
      if (L == NL - 1) {
        if (issue_warp) {  // pool: Y = A x_mid W_out + A2 ReLU(H) W2'  (N = 64, K = 64 + 32) -> D [64, 128)
          issuer_wait_simt();
          t3_mma3<4>(R + kCW2, R + kCA, 32, desc_s[16], desc_s[17], (2 * 64 * 16) >> 4, t3_idesc<F16>(128, 64));
          t3_mma3<2, true>(R + kCW2, R + kCA2, 16, desc_s[18], desc_s[19], (2 * 64 * 16) >> 4,
                           t3_idesc<F16>(128, 64));
          commit_w(&t3.mma[t]);
        }
        stamp(16);
        break;  // (the last layer ends here)
      }
#endif
      if (issue_warp) {  // M5: D2 = ReLU(H) W2   (N = 64, K = 32)
        issuer_wait_simt();
        t3_mma3<2>(R + kCW2, R + kCA2, 16, desc_s[12 + 2 * L], desc_s[13 + 2 * L], (2 * 64 * 16) >> 4, t3_idesc<F16>(128, 64));
        commit_w(&t3.mma[t]);
      }
      stamp(16);
      // ---- P6: x += D2 ----
      wait_mma();
      stamp(17);
      {
        float d[kDModel];
        t3_ld64(lanebase + kCW2, d);
        // (a row that is not ok has ReLU(H) = 0: D2 = 0, x stays 0)
#pragma unroll
        for (int j = 0; j < kDModel; j += 2) {
          const float2 o = __fadd2_rn(make_float2(d[j], d[j + 1]), make_float2(x[j], x[j + 1]));
          x[j] = o.x;
          x[j + 1] = o.y;
        }
      }
      stamp(18);
    }

    // ---- K5: y = x out_linear, masked max over rows ----
#ifdef TAV2_POOL_UNFUSED
    t3_st_split<64, F16>(cA, x);  // invalid rows carry x = 0
    tmem_st_wait();
    done();
    stamp(19);
    if (issue_warp) {
      issuer_wait_simt();
      t3_mma3<4>(R + kCD, R + kCA, 32, desc_s[16], desc_s[17], (2 * 64 * 16) >> 4,
                 t3_idesc<F16>(128, 64));
      commit_w(&t3.mma[t]);
    }
    constexpr uint32_t kCY = kCD;
#else
    constexpr uint32_t kCY = kCW2;  // issued in the last layer
#endif
    stamp(20);
    wait_mma();
    stamp(21);
    {
      float y[kDModel];
      t3_ld64(lanebase + kCY, y);
      if (tid == 0) any_s = 0;
      named_bar_sync(1, kT3Threads);  // every row is past its last softmax (valid_w, kmax_s free)
      if (ok) any_s = 1;
      if (tid < 8) valid_w[tid] = 0u;
      if (tid < 2) kmax_s[tid] = 0u;
#pragma unroll
      for (int j = 0; j < kDModel; ++j) {
        const float v = warp_max_f32(ok ? y[j] : -INFINITY);
        if (lane == 0) red_s[warp][j] = v;
      }
    }
    // (every thread read nx_s at this item's last-layer top, before its
    // kready arrival, which tid 0 has waited on since)
    if (sel.next_item != nullptr && tid == 0) nx_s = 2 * (int)gridDim.x + (int)claim;
#ifndef TAV2_OLD_PF
    tok_pf = pf_idx >= 0 ? pf_off + pf_idx : -1;
#endif
    {  // the next item's token row (tok_pf resolved in the last layer), under
       // the pool barrier; always overwritten (row 0 for padding slots) so tfv
       // is dead through the layers
      const size_t tr = (in_seq && tok_pf >= 0) ? (size_t)tok_pf : 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) ldg256(st.tok_feat + tr * kDModel + 8 * j, tfv + 8 * j);
    }
    named_bar_sync(1, kT3Threads);
    stamp(22);
    // pooled vector -> pooled_out (the CTR head is head_kernel, pool.cu, which
    // may already be polling it: plain stores, no fence)
    if (tid < kDModel) {
      float v = -INFINITY;
#pragma unroll
      for (int w = 0; w < kT3Warps; ++w) v = fmaxf(v, red_s[w][tid]);
      pooled_out[(size_t)item * kDModel + tid] = any_s ? v : 0.0f;  // empty user -> 0 (trainer.py:358-359)
    }
    // (red_s is rewritten only after the next item's pool barrier)
    stamp(23);
    if (item == (int)blockIdx.x) cta_stamp(8, 0);  // (debug) first item pooled
  }
  if (kDebug && dbg) dbg[27] += dbg_m3;
  cta_stamp(8, 1);  // (debug) last item pooled
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(0u);
  cta_stamp(kDbgSkut, 1);
}

cudaError_t set_dbg_cta_skut3(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t set_debug_skut3(long long* dev) { return cudaMemcpyToSymbol(g_dbg_skut3, &dev, sizeof(dev)); }

bool skut_tc3_supported(const NNCfg& nn, const Params& p) {
  const int S_pad = (nn.seq_len + 15) & ~15;
  return S_pad <= 192 && p.num_layers >= 1 && p.num_layers <= 2;
}

cudaError_t launch_skut_tc3(const Params& p, const SkutImages3& img, const NNCfg& nn, const Staged& st,
                            const int32_t* idx, int n, float* logits, float* pooled, SelFlags sel, bool f16,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int S_pad = (nn.seq_len + 15) & ~15;
  const size_t smem = (size_t)p.num_layers * kW3Layer + kImg3WO + kImg3W2O + 4 * (size_t)S_pad * 128;
  auto kern = f16 ? skut_tc3_kernel<true> : skut_tc3_kernel<false>;
  cudaError_t e = set_max_dyn_smem((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int sms = device_sms();
  return launch_pdl(kern, dim3(n < sms ? n : sms), dim3(kT3Threads), smem, s, p, img, nn, st, idx, n, logits,
                    pooled, sel);
}

}  // namespace tav2
