// SKUT on the 5th-gen tensor cores: gather + Eq. 4 encode, 2 x pre-norm
// causal transformer layers, linear + masked max-pool and the CTR head for
// one candidate per CTA iteration (persistent over candidates).
//
// Reference: encoder.py:161-188 (encode_batch), :196-211 (layer_norm,
// masked_softmax), :314-462 (forward_fused), trainer.py:354-366 (pool + head).
//
// Numerics ("bf16 mode"): every GEMM is a 3-term split-bf16 product
// a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi (x_hi = bf16(x), x_lo = bf16(x -
// x_hi)) accumulated in f32 in TMEM (~2^-16 relative per product, SURVEY
// App. B: logits within 5e-5 vs the 2e-3 budget).  Residual stream, LN,
// softmax statistics and the head stay f32 in registers.
//
// Layout: thread = sequence row.  Rows 0..127 are tile 0 (warps 0-3), rows
// 128..255 tile 1 (warps 4-7); warp w owns TMEM lanes 32*(w%4)..+31.  The
// residual row x[64] lives in registers.  A operands (LN outputs, Q, P,
// O/l, ReLU(h)) are written by the row threads straight into TMEM as packed
// bf16 hi/lo pairs (tcgen05.st); B operands (weights, K, V) live in shared
// memory in the UMMA no-swizzle canonical layouts (tc_common.cuh).  Weight
// images are streamed with cp.async.bulk into two buffers (WA: Wqkv or
// out_linear, WB: Wo|W1|W2) one phase ahead.  Thread 0 also issues all
// MMAs and bulk copies; row threads and the issuer hand off through
// mbarriers (8 warps = 2 per SM sub-partition -> up to 255 registers).
//
// TMEM columns (512): A/Q/O/LN2-A at 384+64t; D_qkv at 192t; S/P at 0 (tile
// 0, 128 keys) and 128 (tile 1, S_pad keys); D_wo at 64t; D_w1 at 128+32t;
// ReLU-A at 192+32t; D_w2 at 256+64t; pool D at 64t.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "encode.cuh"
#include "tav2_common.cuh"
#include "tc_common.cuh"
#include "dbg.cuh"

namespace tav2 {

using namespace tc;

constexpr int kSkRowWarps = 8;
constexpr int kSkThreads = 32 * kSkRowWarps;
constexpr int kRowThreads = 32 * kSkRowWarps;
constexpr float kLnEpsTc = 1e-5f;
constexpr float kLog2e = 1.4426950408889634f;

constexpr uint32_t kColA = 384, kColQKV = 0, kColS1 = 128, kColWo = 0, kColW1 = 128, kColA2 = 192,
                   kColW2 = 256, kColOut = 0;

// Debug timeline (tav2_debug_timeline): %globaltimer stamps of CTA 0's
// first candidate: slot 2p = SIMT phase p done (thread 0), 2p+1 = MMA phase p
// issued; 64 + p = MMA phase p observed complete by thread 0.
__device__ long long* g_dbg_skut = nullptr;
__device__ __forceinline__ long long sk_time() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- row-thread helpers (warp-collective TMEM access) ----
__device__ __forceinline__ void ld64(uint32_t ta, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  tmem_ld32(ta, r);
  tmem_ld32(ta + 32, r + 32);
  tmem_ld_wait();
}
__device__ __forceinline__ void ld32f(uint32_t ta, float* v) {
  tmem_ld32(ta, reinterpret_cast<uint32_t*>(v));
  tmem_ld_wait();
}
// split n (multiple of 16) floats into packed bf16 hi/lo pairs and store:
// hi pairs at columns [0, n/2), lo pairs at [n/2, n) relative to `ta`
template <int N>
__device__ __forceinline__ void st_split(uint32_t ta, const float* v) {
#pragma unroll
  for (int c = 0; c < N / 16; ++c) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) split_pair(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
    tmem_st8(ta + 8 * c, hi);
    tmem_st8(ta + N / 2 + 8 * c, lo);
  }
}
__device__ __forceinline__ void layer_norm_reg(const float* x, const float* g, const float* b,
                                               float* y) {
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < kDModel; ++j) s += x[j];
  const float mu = s * (1.0f / 64.0f);
  float v = 0.0f;
#pragma unroll
  for (int j = 0; j < kDModel; ++j) {
    const float c = x[j] - mu;
    v = fmaf(c, c, v);
  }
  const float rs = 1.0f / sqrtf(v * (1.0f / 64.0f) + kLnEpsTc);
#pragma unroll
  for (int j = 0; j < kDModel; ++j) y[j] = fmaf((x[j] - mu) * rs, g[j], b[j]);
}
// 16 bytes of 8 bf16 elements (from 8 floats)
__device__ __forceinline__ void split8_store(uint8_t* hi_dst, uint8_t* lo_dst, const float* v) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_pair(v[2 * i], v[2 * i + 1], h[i], l[i]);
  *reinterpret_cast<uint4*>(hi_dst) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(lo_dst) = make_uint4(l[0], l[1], l[2], l[3]);
}

// ---- issuer helpers: D += A(TMEM hi/lo) x B(smem hi/lo), 3 terms per k-step ----
// A: hi at a_col + 8j, lo at a_col + a_lo_off + 8j (k-step j covers 16 K)
// B (K-major slabs): hi at b_hi + 2j*lbo, lo at b_lo + 2j*lbo
__device__ __forceinline__ void mma3_kmajor(uint32_t d, uint32_t a_col, uint32_t a_lo_off,
                                            uint32_t b_hi, uint32_t b_lo, uint32_t lbo, int ksteps,
                                            uint32_t idesc) {
  for (int j = 0; j < ksteps; ++j) {
    const uint64_t bh = sdesc(b_hi + 2 * j * lbo, lbo, 128);
    const uint64_t bl = sdesc(b_lo + 2 * j * lbo, lbo, 128);
    mma_bf16_ts(d, a_col + 8 * j, bh, idesc, j > 0);
    mma_bf16_ts(d, a_col + 8 * j, bl, idesc, 1);
    mma_bf16_ts(d, a_col + a_lo_off + 8 * j, bh, idesc, 1);
  }
}

// allowed keys k0..k0+15 for query row r: key-valid bits (low 16 of `bits`)
// AND causal (key <= r)
static __device__ __forceinline__ uint32_t allowed16(uint32_t bits, int k0, int r) {
  const int n = r - k0 + 1;  // keys k0..r are causal-visible
  const uint32_t causal = 0xffffu >> min(max(16 - n, 0), 16);  // branch-free (skut_tc3)
  return bits & causal;
}

// MMA / bulk-copy issuer state, driven by thread 0 between its own
// arrive on bar_simt and its wait on bar_mma (the CTA has no spare warp:
// 8 warps keep 2 per SM sub-partition and so up to 255 registers each).
struct Issuer {
  uint32_t T, wa, wb, khi, klo, vhi, vlo;
  uint32_t ph_simt = 0, ph_wa = 0, ph_wb = 0, n_mma = 0;
  uint64_t *bar_simt, *bar_mma, *bar_wa, *bar_wb;
  uint8_t *WA, *WB;
  int NT, S_pad;

  int n_ws = 0;
  __device__ void wait_simt() {
    mbar_wait(bar_simt, ph_simt);
    if (dbg && n_ws < 32) dbg[160 + n_ws] = sk_time();
    ++n_ws;
    ph_simt ^= 1;
    fence_after();
  }
  long long* dbg = nullptr;
  __device__ void commit_mma() {
    commit(bar_mma);
    if (dbg && n_mma < 32) dbg[2 * n_mma + 1] = sk_time();
    ++n_mma;
  }
  __device__ void wait_mma() { mbar_wait(bar_mma, (n_mma - 1) & 1); }
  __device__ void load_wa(const void* src, uint32_t bytes) {
    mbar_expect_tx(bar_wa, bytes);
    bulk_g2s(WA, src, bytes, bar_wa);
  }
  __device__ void load_wb(const void* src) {
    mbar_expect_tx(bar_wb, kImgWB);
    bulk_g2s(WB, src, kImgWB, bar_wb);
  }
  __device__ void need_wa() {
    mbar_wait(bar_wa, ph_wa);
    ph_wa ^= 1;
    fence_after();
  }
  __device__ void need_wb() {
    mbar_wait(bar_wb, ph_wb);
    ph_wb ^= 1;
    fence_after();
  }
  __device__ int nkeys(int t) const { return t == 0 ? (S_pad < 128 ? S_pad : 128) : S_pad; }

  // QKV = LN1(x) [Wq|Wk|Wv]   (N = 192, K = 64)
  __device__ void qkv() {
    for (int t = 0; t < NT; ++t)
      mma3_kmajor(T + kColQKV + 192 * t, T + kColA + 64 * t, 32, wa, wa + kImgWA / 2, 192 * 16, 4,
                  idesc_bf16(128, 192));
  }
  // S_t = Q_t K^T  (N = keys of tile t, K = 64)
  __device__ void scores() {
    for (int t = 0; t < NT; ++t)
      mma3_kmajor(T + (t == 0 ? 0u : kColS1), T + kColA + 64 * t, 32, khi, klo, S_pad * 16, 4,
                  idesc_bf16(128, nkeys(t)));
  }
  // O_t = P_t V  (N = 64, K = keys; V is MN-major)
  __device__ void pv() {
    const uint32_t id = idesc_bf16(128, 64, 0, 1);
    for (int t = 0; t < NT; ++t) {
      const uint32_t pc = T + (t == 0 ? 0u : kColS1), d = T + kColA + 64 * t;
      for (int j = 0; j < nkeys(t) / 16; ++j) {
        const uint64_t bh = sdesc(vhi + 2 * j * 1024, 1024, 128);
        const uint64_t bl = sdesc(vlo + 2 * j * 1024, 1024, 128);
        mma_bf16_ts(d, pc + 16 * j, bh, id, j > 0);
        mma_bf16_ts(d, pc + 16 * j, bl, id, 1);
        mma_bf16_ts(d, pc + 16 * j + 8, bh, id, 1);
      }
    }
  }
  __device__ void wo() {
    for (int t = 0; t < NT; ++t)
      mma3_kmajor(T + kColWo + 64 * t, T + kColA + 64 * t, 32, wb, wb + 8192, 64 * 16, 4, idesc_bf16(128, 64));
  }
  __device__ void w1() {
    for (int t = 0; t < NT; ++t)
      mma3_kmajor(T + kColW1 + 32 * t, T + kColA + 64 * t, 32, wb + 16384, wb + 16384 + 4096, 32 * 16, 4,
                  idesc_bf16(128, 32));
  }
  __device__ void w2() {
    for (int t = 0; t < NT; ++t)
      mma3_kmajor(T + kColW2 + 64 * t, T + kColA2 + 32 * t, 16, wb + 24576, wb + 24576 + 4096, 64 * 16, 2,
                  idesc_bf16(128, 64));
  }
  __device__ void pool() {
    for (int t = 0; t < NT; ++t)
      mma3_kmajor(T + kColOut + 64 * t, T + kColA + 64 * t, 32, wa, wa + 8192, 64 * 16, 4, idesc_bf16(128, 64));
  }
};

__global__ void __launch_bounds__(kSkThreads, 1) skut_tc_kernel(
    Params p, SkutImages img, NNCfg nn, Staged st, int use_staged, const int32_t* idx,
    const float* Fin, const uint8_t* fmask, int n, float* U, float* logits, float* pooled_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar_simt, bar_mma, bar_wa, bar_wb;
  __shared__ uint32_t taddr_s;
  __shared__ uint32_t valid_w[8];  // key-validity bitmask, bit r of word r/32
  __shared__ __align__(16) float lnp_s[kMaxLayers][4][kDModel];  // ln1 g/b, ln2 g/b
  __shared__ float red_s[kSkRowWarps][kDModel];
  __shared__ float z_s[kDModel + kEmbed + kCtx];
  __shared__ float hid_s[kHidden];
  __shared__ int any_s;
  __shared__ unsigned kmax_s[kMaxLayers];  // per layer: max over rows of ||k_r||^2 (f32 bits)
  __shared__ float qn2_s[256];             // ||q_r||^2 per row (softmax shift)
  __shared__ float lsum_s[2][256];         // softmax row sums: [owner warp | helper warp]

  const int S = nn.seq_len;
  const int S_pad = (S + 15) & ~15;
  const int NT = (S + 127) / 128;  // 1 or 2 row tiles
  const int NL = p.num_layers;
  uint8_t* WA = sm;
  uint8_t* WB = sm + kImgWA;
  uint8_t* Khi = WB + kImgWB;
  uint8_t* Klo = Khi + S_pad * 128;
  uint8_t* Vhi = Klo + S_pad * 128;
  uint8_t* Vlo = Vhi + S_pad * 128;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar_simt, kRowThreads);
    mbar_init(&bar_mma, 1);
    mbar_init(&bar_wa, 1);
    mbar_init(&bar_wb, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  for (int i = tid; i < NL * 4 * kDModel; i += kSkThreads) {
    const int L = i / (4 * kDModel), w = (i / kDModel) % 4, j = i % kDModel;
    const float* src = w == 0 ? p.ln1_scale[L] : w == 1 ? p.ln1_shift[L] : w == 2 ? p.ln2_scale[L] : p.ln2_shift[L];
    lnp_s[L][w][j] = src[j];
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;

  Issuer is;
  const bool issuer = tid == 0;
  if (issuer) {
    is.T = T;
    is.WA = WA;
    is.WB = WB;
    is.wa = smem_u32(WA);
    is.wb = smem_u32(WB);
    is.khi = smem_u32(Khi);
    is.klo = smem_u32(Klo);
    is.vhi = smem_u32(Vhi);
    is.vlo = smem_u32(Vlo);
    is.bar_simt = &bar_simt;
    is.bar_mma = &bar_mma;
    is.bar_wa = &bar_wa;
    is.bar_wb = &bar_wb;
    is.NT = NT;
    is.S_pad = S_pad;
    is.dbg = kDebug && blockIdx.x == 0 ? g_dbg_skut : nullptr;
    is.load_wa(img.wa[0], kImgWA);
    is.load_wb(img.wb[0]);
  }

  const int t = warp >> 2, q = warp & 3;
  const int r = 128 * t + 32 * q + lane;  // sequence row
  const uint32_t lanebase = T + ((uint32_t)(32 * q) << 16);
  const uint32_t cA = lanebase + kColA + 64 * t;
  const bool in_seq = r < S;
  uint32_t n_mma = 0, n_done = 0;
  long long* dbg = (kDebug && blockIdx.x == 0 && tid == 0) ? g_dbg_skut : nullptr;
  auto wait_mma = [&]() {
    __syncwarp();
    mbar_wait_sleep(&bar_mma, n_mma & 1);
    if (dbg && n_mma < 64) dbg[64 + n_mma] = sk_time();
    ++n_mma;
    fence_after();
  };
  auto done = [&]() {
    fence_before();
    mbar_arrive(&bar_simt);
    if (dbg && n_done < 32) dbg[2 * n_done] = sk_time();
    ++n_done;
  };

  griddep_launch();
  griddep_wait();  // NN selection (idx) and prep (tok_unit, cand_unit) complete
  cta_stamp(kDbgSkut, 2);
  for (int item = blockIdx.x; item < n; item += gridDim.x) {
    // ---- K3: gather + encode this row (or load caller features) ----
    float x[kDModel];
    bool ok = false;
    if (in_seq) {
      if (use_staged) {
        const int tok = slot_token(st, nn, idx, item, r);
        ok = tok >= 0;
        if (ok) encode_feat(st, p, item, tok, r, x);
      } else {
        ok = fmask[(size_t)item * S + r] != 0;
        if (ok) {
          const float4* src = reinterpret_cast<const float4*>(Fin + ((size_t)item * S + r) * kDModel);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 v = src[j];
            x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
          }
        }
      }
    }
    if (!ok) {
#pragma unroll
      for (int j = 0; j < kDModel; ++j) x[j] = 0.0f;
    }
    {
      const unsigned b = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) valid_w[warp] = b;
      if (tid < kMaxLayers) kmax_s[tid] = 0u;
    }
    named_bar_sync(1, kRowThreads);
    const int wmax_row = 128 * t + 32 * q + 31;  // warp-uniform causal bound

    for (int L = 0; L < NL; ++L) {
      float qn2 = 0.0f;  // ||q_r||^2 of this row (QKV epilogue -> softmax)
      // ---- LN1 -> A ----
      {
        float y[kDModel];
        layer_norm_reg(x, lnp_s[L][0], lnp_s[L][1], y);
        if (!ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) y[j] = 0.0f;
        }
        st_split<64>(cA, y);  // warp-collective: never under a divergent branch
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.need_wa();
        is.qkv();
        is.commit_mma();
        is.wait_mma();  // WA free: prefetch the next Wqkv (or out_linear)
        if (L + 1 < NL) is.load_wa(img.wa[L + 1], kImgWA);
        else is.load_wa(img.wout, kImgWO);
      }
      // ---- QKV epilogue: Q -> TMEM A, K/V -> smem ----
      wait_mma();
      {
        const uint32_t cq = lanebase + kColQKV + 192 * t;
        float v[32];
        qn2 = 0.0f;
        float kn2 = 0.0f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          ld32f(cq + 32 * h, v);
          if (!ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0f;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) qn2 = fmaf(v[i], v[i], qn2);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) split_pair(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
            tmem_st8(cA + 16 * h + 8 * c, hi);
            tmem_st8(cA + 32 + 16 * h + 8 * c, lo);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // K: K-major slabs, chunk c of row r at c*(S_pad*16) + r*16
          ld32f(cq + 64 + 32 * h, v);
          if (r < S_pad) {
            if (!ok) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.0f;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) kn2 = fmaf(v[i], v[i], kn2);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int off = (4 * h + c) * (S_pad * 16) + r * 16;
              split8_store(Khi + off, Klo + off, v + 8 * c);
            }
          }
        }
        // max_j ||k_j||^2 over the valid keys: shift bound of the softmax below
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) kn2 = fmaxf(kn2, __shfl_xor_sync(0xffffffffu, kn2, o));
        if (lane == 0) atomicMax(&kmax_s[L], __float_as_uint(kn2));
        qn2_s[r] = qn2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // V: MN-major (key r, d) at (r/8)*1024 + (d/8)*128 + (r%8)*16 + (d%8)*2
          ld32f(cq + 128 + 32 * h, v);
          if (r < S_pad) {
            if (!ok) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.0f;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int off = (r >> 3) * 1024 + (4 * h + c) * 128 + (r & 7) * 16;
              split8_store(Vhi + off, Vlo + off, v + 8 * c);
            }
          }
        }
        tmem_st_wait();
        fence_proxy_async();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.scores();
        is.commit_mma();
      }
      // ---- causal key-masked softmax -> P (bf16 hi/lo, in place over S) ----
      // Single pass: softmax is shift invariant, so instead of the row max we
      // subtract its Cauchy-Schwarz bound m' = ||q_r|| max_j ||k_j|| / 8 >=
      // q_r.k_j / 8 (m' - max stays far inside the f32 exp range for
      // LN-scaled activations; 1/l normalises exactly as encoder.py:203-211).
      // No row max also means a row's key chunks can be split across the two
      // warps that share its TMEM lanes (q and q+4): the chunks of tile-0 rows
      // 32q.. and tile-1 rows 128+32q.. are dealt out evenly between them and
      // the two partial row sums are combined through shared memory.
      wait_mma();
      {
        named_bar_sync(1, kRowThreads);  // kmax_s[L], qn2_s complete
        const float kmax2 = __uint_as_float(kmax_s[L]);
        const int nkt[2] = {S_pad < 128 ? S_pad : 128, S_pad};
        const int nA = 32 * q < S ? min(nkt[0] / 16, (32 * q + 31) / 16 + 1) : 0;        // tile-0 chunks
        const int nB = 128 + 32 * q < S ? min(nkt[1] / 16, (128 + 32 * q + 31) / 16 + 1) : 0;  // tile-1
        const int half = (nA + nB + 1) / 2;
        const int s0 = t == 0 ? 0 : half, s1 = t == 0 ? half : nA + nB;  // this warp's chunk slots
        float lpart[2] = {0.0f, 0.0f};
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const int base = tt == 0 ? 0 : nA;
          const int j_lo = max(s0 - base, 0), j_hi = min(s1 - base, tt == 0 ? nA : nB);
          const int rr = 128 * tt + 32 * q + lane;
          const bool okr = (valid_w[rr >> 5] >> lane) & 1u;
          const float mb = sqrtf(qn2_s[rr] * kmax2) * (0.125f * kLog2e);
          const uint32_t cs = lanebase + (tt == 0 ? 0u : kColS1);
          for (int j0 = j_lo; j0 < j_hi; j0 += 2) {
            uint32_t s32[32];
            const bool two = j0 + 1 < j_hi;  // warp-uniform
            tmem_ld16(cs + 16 * j0, s32);
            if (two) tmem_ld16(cs + 16 * (j0 + 1), s32 + 16);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j = j0 + u;
              if (u == 1 && !two) break;
              const uint32_t vm = okr ? allowed16(valid_w[j >> 1] >> ((j & 1) * 16), 16 * j, rr) : 0u;
              float pv[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                float p;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p) : "f"(fmaf(__uint_as_float(s32[16 * u + e]), 0.125f * kLog2e, -mb)));
                pv[e] = ((vm >> e) & 1u) ? p : 0.0f;
                lpart[tt] += pv[e];
              }
              uint32_t hi[8], lo[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) split_pair(pv[2 * i], pv[2 * i + 1], hi[i], lo[i]);
              tmem_st8(cs + 16 * j, hi);
              tmem_st8(cs + 16 * j + 8, lo);
            }
          }
        }
        // the row owner zero-fills its tile's chunks past the causal range
        {
          const uint32_t cs = lanebase + (t == 0 ? 0u : kColS1);
          const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          for (int j = t == 0 ? nA : nB; j < nkt[t] / 16; ++j) {
            tmem_st8(cs + 16 * j, z);
            tmem_st8(cs + 16 * j + 8, z);
          }
        }
        lsum_s[0][r] = lpart[t];                          // owner's part of row r
        lsum_s[1][128 * (1 - t) + 32 * q + lane] = lpart[1 - t];  // helper's part of the other tile's row
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.pv();
        is.commit_mma();
      }
      // ---- O / l -> A ----
      wait_mma();
      {
        named_bar_sync(1, kRowThreads);  // lsum_s complete
        const float l = lsum_s[0][r] + lsum_s[1][r];
        const float inv_l = l > 0.0f ? 1.0f / l : 0.0f;  // a valid row always sees itself
        float o[kDModel];
        ld64(cA, o);
#pragma unroll
        for (int j = 0; j < kDModel; ++j) o[j] = ok ? o[j] * inv_l : 0.0f;
        st_split<64>(cA, o);
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.need_wb();
        is.wo();
        is.commit_mma();
      }
      // ---- x += O Wo ; LN2 -> A ----
      wait_mma();
      {
        float d[kDModel];
        ld64(lanebase + kColWo + 64 * t, d);
        if (ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) x[j] += d[j];
        }
        layer_norm_reg(x, lnp_s[L][2], lnp_s[L][3], d);
        if (!ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) d[j] = 0.0f;
        }
        st_split<64>(cA, d);
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.w1();
        is.commit_mma();
      }
      // ---- ReLU(h) -> A2 ----
      wait_mma();
      {
        float h[kFfn];
        ld32f(lanebase + kColW1 + 32 * t, h);
#pragma unroll
        for (int j = 0; j < kFfn; ++j) h[j] = ok ? fmaxf(h[j], 0.0f) : 0.0f;
        st_split<32>(lanebase + kColA2 + 32 * t, h);
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.w2();
        is.commit_mma();
        is.wait_mma();  // WB free: prefetch the next layer's (or candidate's) Wo|W1|W2
        is.load_wb(img.wb[(L + 1) % NL]);
      }
      // ---- x += ReLU(h) W2 ----
      wait_mma();
      {
        float d[kDModel];
        ld64(lanebase + kColW2 + 64 * t, d);
        if (ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) x[j] += d[j];
        }
      }
    }

    if (U && in_seq) {  // forward_fused output rows (padded rows are zero)
      float4* dst = reinterpret_cast<float4*>(U + ((size_t)item * S + r) * kDModel);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        dst[j] = ok ? make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // ---- K5: y = x out_linear, masked max over rows, CTR head ----
    st_split<64>(cA, x);  // invalid rows carry x = 0
    tmem_st_wait();
    done();
    if (issuer) {
      is.wait_simt();
      is.need_wa();
      is.pool();
      is.commit_mma();
      is.wait_mma();  // WA free: next candidate's layer-0 Wqkv
      is.load_wa(img.wa[0], kImgWA);
    }
    wait_mma();
    {
      float y[kDModel];
      ld64(lanebase + kColOut + 64 * t, y);
      if (tid == 0) any_s = 0;
      named_bar_sync(1, kRowThreads);
      if (ok) any_s = 1;
#pragma unroll
      for (int j = 0; j < kDModel; ++j) {
        const float v = warp_max_f32(ok ? y[j] : -INFINITY);
        if (lane == 0) red_s[warp][j] = v;
      }
    }
    named_bar_sync(1, kRowThreads);
    if (logits) {
      if (tid < kDModel) {
        float v = -INFINITY;
#pragma unroll
        for (int w = 0; w < kSkRowWarps; ++w) v = fmaxf(v, red_s[w][tid]);
        v = any_s ? v : 0.0f;  // empty user -> pooled = 0 (trainer.py:358-359)
        z_s[tid] = v;
        if (pooled_out) pooled_out[(size_t)item * kDModel + tid] = v;
      } else if (tid < kDModel + kEmbed) {
        z_s[tid] = use_staged ? st.cand_unit[(size_t)item * kEmbed + tid - kDModel] : 0.0f;
      } else if (tid < kDModel + kEmbed + kCtx) {
        z_s[tid] = use_staged ? st.ctx[st.item_req[item] * kCtx + tid - kDModel - kEmbed] : 0.0f;
      }
      named_bar_sync(1, kRowThreads);
      if (tid < kHidden) {
        float h = 0.0f;
        for (int i = 0; i < kDModel + kEmbed + kCtx; ++i) h = fmaf(z_s[i], __ldg(p.head_w1 + i * kHidden + tid), h);
        hid_s[tid] = fmaxf(h + __ldg(p.head_b1 + tid), 0.0f);
      }
      named_bar_sync(1, kRowThreads);
      if (tid < kHeads) {
        float o = 0.0f;
        for (int j = 0; j < kHidden; ++j) o = fmaf(hid_s[j], __ldg(p.head_w2 + j * kHeads + tid), o);
        logits[(size_t)item * kHeads + tid] = o + __ldg(p.head_b2 + tid);
      }
    }
    named_bar_sync(1, kRowThreads);  // smem (valid_w, red_s, z_s) reuse by the next item
  }
  if (issuer) {  // drain the last prefetches before the CTA retires
    is.need_wa();
    is.need_wb();
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(T);
}

// ===========================================================================
// Tile-decoupled SKUT (S <= 192): two independent row tiles.
//
// Rows are laid out in 8 blocks of S_pad/8 (see the kernel prologue) so
// every SM sub-partition carries equal causal work.  Each tile t (warps
// 4t..4t+3) owns a 256-column TMEM region, its own simt/mma mbarriers and its
// own issuer lane (thread 128t), so one tile's SIMT epilogue runs while the
// tensor core executes the other tile's MMAs.  Coupling points: K/V of a
// layer are complete when all 256 rows arrived on bar_kvready (both tiles'
// score MMAs need every key), the next layer's K/V may be written once both
// tiles' P.V MMAs retired (bar_kvfree), and the shared weight buffers are
// refilled (by tile 1's issuer) once both tiles' MMAs released them.
//
// TMEM per tile (base 256t): A/Q/O/LN2-A at +192 (64 cols); D_qkv at +0
// (192); S/P at +0 (S_pad <= 192); D_wo / pool D at +0; D_w1 at +64;
// ReLU-A at +96; D_w2 at +128.
// ===========================================================================
constexpr uint32_t kTA = 192, kTD = 0, kTW1 = 64, kTA2 = 96, kTW2 = 128;

struct Tc2Bars {
  uint64_t simt[2], mma[2], kvready, kvfree, wa_full, wb_full, wa_free, wb_free;
};
__shared__ __align__(8) Tc2Bars tc2;  // one set per CTA (static shared, only skut_tc2 uses it)

// MMA issue for tile t (thread 128t).  Only phase bits live in registers: the
// barrier and operand addresses are static shared / derivable from S_pad.
struct TileIssuer {
  uint32_t R;       // TMEM column base of the tile
  uint32_t S_pad;
  uint32_t NK;      // keys this tile's rows can see (multiple of 16)
  uint32_t ph = 0;  // bit0 simt, bit1 wa_full, bit2 wb_full, bit3 wa_free, bit4 wb_free
  int n_commit = 0;
  bool dbg = false;

  __device__ static uint32_t base() {
    extern __shared__ __align__(1024) uint8_t sm[];
    return smem_u32(sm);
  }
  __device__ uint32_t wa() const { return base(); }
  __device__ uint32_t wb() const { return base() + kImgWA; }
  __device__ uint32_t khi() const { return base() + kImgWA + kImgWB; }
  __device__ uint32_t klo() const { return khi() + S_pad * 128; }
  __device__ uint32_t vhi() const { return khi() + 2 * S_pad * 128; }
  __device__ uint32_t vlo() const { return khi() + 3 * S_pad * 128; }
  __device__ void wait_ph(uint64_t* bar, int bit) {
    mbar_wait(bar, (ph >> bit) & 1u);
    ph ^= 1u << bit;
  }
  __device__ void wait_simt() {
    wait_ph(&tc2.simt[R >> 8], 0);
    fence_after();
  }
  __device__ void commit_mma() {
    commit(&tc2.mma[R >> 8]);
    if (dbg && n_commit < 32) g_dbg_skut[2 * n_commit + 1] = sk_time();
    ++n_commit;
  }
  __device__ void need_wa() { wait_ph(&tc2.wa_full, 1); fence_after(); }
  __device__ void need_wb() { wait_ph(&tc2.wb_full, 2); fence_after(); }
  // loader role (tile 1): refill once both tiles released the buffer
  __device__ void refill_wa(const void* src, uint32_t bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    wait_ph(&tc2.wa_free, 3);
    mbar_expect_tx(&tc2.wa_full, bytes);
    bulk_g2s(sm, src, bytes, &tc2.wa_full);
  }
  __device__ void refill_wb(const void* src) {
    extern __shared__ __align__(1024) uint8_t sm[];
    wait_ph(&tc2.wb_free, 4);
    mbar_expect_tx(&tc2.wb_full, kImgWB);
    bulk_g2s(sm + kImgWA, src, kImgWB, &tc2.wb_full);
  }
  __device__ void qkv() { mma3_kmajor(R + kTD, R + kTA, 32, wa(), wa() + kImgWA / 2, 192 * 16, 4, idesc_bf16(128, 192)); }
  __device__ void scores() { mma3_kmajor(R + kTD, R + kTA, 32, khi(), klo(), S_pad * 16, 4, idesc_bf16(128, NK)); }
  __device__ void pv() {
    const uint32_t id = idesc_bf16(128, 64, 0, 1);
    for (int j = 0; j < (int)NK / 16; ++j) {
      const uint64_t bh = sdesc(vhi() + 2 * j * 1024, 1024, 128);
      const uint64_t bl = sdesc(vlo() + 2 * j * 1024, 1024, 128);
      mma_bf16_ts(R + kTA, R + kTD + 16 * j, bh, id, j > 0);
      mma_bf16_ts(R + kTA, R + kTD + 16 * j, bl, id, 1);
      mma_bf16_ts(R + kTA, R + kTD + 16 * j + 8, bh, id, 1);
    }
  }
  __device__ void wo() { mma3_kmajor(R + kTD, R + kTA, 32, wb(), wb() + 8192, 64 * 16, 4, idesc_bf16(128, 64)); }
  __device__ void w1() { mma3_kmajor(R + kTW1, R + kTA, 32, wb() + 16384, wb() + 16384 + 4096, 32 * 16, 4, idesc_bf16(128, 32)); }
  __device__ void w2() { mma3_kmajor(R + kTW2, R + kTA2, 16, wb() + 24576, wb() + 24576 + 4096, 64 * 16, 2, idesc_bf16(128, 64)); }
  __device__ void pool() { mma3_kmajor(R + kTD, R + kTA, 32, wa(), wa() + 8192, 64 * 16, 4, idesc_bf16(128, 64)); }
};

__global__ void __launch_bounds__(kSkThreads, 1) skut_tc2_kernel(
    Params p, SkutImages img, NNCfg nn, Staged st, int use_staged, const int32_t* idx,
    const float* Fin, const uint8_t* fmask, int n, float* U, float* logits, float* pooled_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  cta_stamp(kDbgSkut, 0);
  __shared__ uint32_t taddr_s;
  __shared__ uint32_t valid_w[8];  // key-validity bitmask, bit r of word r/32
  __shared__ __align__(16) float lnp_s[kMaxLayers][4][kDModel];
  __shared__ float red_s[kSkRowWarps][kDModel];
  __shared__ float z_s[kDModel + kEmbed + kCtx];
  __shared__ float hid_s[kHidden];
  __shared__ int any_s;
  __shared__ unsigned kmax_s[kMaxLayers];

  const int S = nn.seq_len;
  const int S_pad = (S + 15) & ~15;
  const int NL = p.num_layers;
  uint8_t* WA = sm;
  uint8_t* WB = sm + kImgWA;
  uint8_t* Khi = WB + kImgWB;
  uint8_t* Klo = Khi + S_pad * 128;
  uint8_t* Vhi = Klo + S_pad * 128;
  uint8_t* Vlo = Vhi + S_pad * 128;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = warp >> 2, q = warp & 3;
  const int li = 32 * q + lane;  // TMEM lane within the tile
  // Row blocks: S_pad rows in 8 blocks of rpw = S_pad/8 (<= 24); warp (t, q)
  // takes block kb = q (tile 0) or 7 - q (tile 1), lanes >= rpw are padding.
  // Each SM sub-partition q thus holds one early and one late block, so the
  // causal softmax work is balanced across sub-partitions, no warp is pure
  // padding, and tile 0 (rows < S_pad/2) only needs keys < NK0.
  const int rpw = S_pad >> 3;
  const int kb = t == 0 ? q : 7 - q;
  const bool mapped = lane < rpw;   // lane carries a row < S_pad
  const int r = rpw * kb + lane;    // sequence row (when mapped)
  const int NK0 = ((S_pad >> 1) + 15) & ~15;
  if (tid == 0) {
    mbar_init(&tc2.simt[0], 128);
    mbar_init(&tc2.simt[1], 128);
    mbar_init(&tc2.mma[0], 1);
    mbar_init(&tc2.mma[1], 1);
    mbar_init(&tc2.kvready, kRowThreads);
    mbar_init(&tc2.kvfree, 2);
    mbar_init(&tc2.wa_full, 1);
    mbar_init(&tc2.wb_full, 1);
    mbar_init(&tc2.wa_free, 2);
    mbar_init(&tc2.wb_free, 2);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  if (tid < 8) valid_w[tid] = 0u;
  for (int i = tid; i < NL * 4 * kDModel; i += kSkThreads) {
    const int L = i / (4 * kDModel), w = (i / kDModel) % 4, j = i % kDModel;
    const float* src = w == 0 ? p.ln1_scale[L] : w == 1 ? p.ln1_shift[L] : w == 2 ? p.ln2_scale[L] : p.ln2_shift[L];
    lnp_s[L][w][j] = src[j];
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (taddr_s != 0u) __trap();  // a 512-column allocation always starts at column 0

  const bool issuer = li == 0;  // thread 128t issues tile t's MMAs
  TileIssuer is;
  is.R = 256u * t;
  is.S_pad = S_pad;
  is.NK = t == 0 ? NK0 : S_pad;
  is.dbg = kDebug && issuer && blockIdx.x == 0 && t == 0 && g_dbg_skut != nullptr;
  if (issuer && t == 1) {  // loader: initial fills
    mbar_expect_tx(&tc2.wa_full, kImgWA);
    bulk_g2s(WA, img.wa[0], kImgWA, &tc2.wa_full);
    mbar_expect_tx(&tc2.wb_full, kImgWB);
    bulk_g2s(WB, img.wb[0], kImgWB, &tc2.wb_full);
  }

  const uint32_t lanebase = ((uint32_t)(32 * q) << 16) + 256u * t;
  const uint32_t cA = lanebase + kTA;
  const bool in_seq = mapped && r < S;
  uint32_t n_mma = 0, n_kv = 0, n_done = 0;
  long long* dbg = (kDebug && blockIdx.x == 0 && tid == 0) ? g_dbg_skut : nullptr;
  auto wait_mma = [&]() {
    __syncwarp();
    mbar_wait_sleep(&tc2.mma[t], n_mma & 1);
    if (dbg && n_mma < 64) dbg[64 + n_mma] = sk_time();
    ++n_mma;
    fence_after();
  };
  auto done = [&]() {
    fence_before();
    mbar_arrive(&tc2.simt[t]);
    if (dbg && n_done < 32) dbg[2 * n_done] = sk_time();
    ++n_done;
  };
  // warp-uniform causal bound: the largest row of this warp
  const int wmax_row = rpw * kb + rpw - 1;

  griddep_launch();
  griddep_wait();  // NN selection (idx) and prep (tok_unit, cand_unit) complete
  cta_stamp(kDbgSkut, 2);
  for (int item = blockIdx.x; item < n; item += gridDim.x) {
    // ---- K3: gather + encode this row (or load caller features) ----
    float x[kDModel];
    bool ok = false;
    if (in_seq) {
      if (use_staged) {
        const int tok = slot_token(st, nn, idx, item, r);
        ok = tok >= 0;
        if (ok) encode_feat(st, p, item, tok, r, x);
      } else {
        ok = fmask[(size_t)item * S + r] != 0;
        if (ok) {
          const float4* src = reinterpret_cast<const float4*>(Fin + ((size_t)item * S + r) * kDModel);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float4 v = src[j];
            x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
          }
        }
      }
    }
    if (!ok) {
#pragma unroll
      for (int j = 0; j < kDModel; ++j) x[j] = 0.0f;
    }
    {
      const unsigned b = __ballot_sync(0xffffffffu, ok);  // lanes >= rpw are never ok
      if (lane == 0 && b) {
        const int r0 = rpw * kb;
        const unsigned long long w = (unsigned long long)b << (r0 & 31);
        atomicOr(&valid_w[r0 >> 5], (uint32_t)w);
        if ((uint32_t)(w >> 32)) atomicOr(&valid_w[(r0 >> 5) + 1], (uint32_t)(w >> 32));
      }
      if (tid < kMaxLayers) kmax_s[tid] = 0u;
    }
    named_bar_sync(1, kRowThreads);

    for (int L = 0; L < NL; ++L) {
      float qn2 = 0.0f;
      // ---- LN1 -> A ----
      {
        float y[kDModel];
        layer_norm_reg(x, lnp_s[L][0], lnp_s[L][1], y);
        if (!ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) y[j] = 0.0f;
        }
        st_split<64>(cA, y);  // warp-collective: never under a divergent branch
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.need_wa();
        is.qkv();
        is.commit_mma();
        commit(&tc2.wa_free);
        if (t == 1) {  // WA free once both tiles' QKV retired: next Wqkv (or out_linear)
          if (L + 1 < NL) is.refill_wa(img.wa[L + 1], kImgWA);
          else is.refill_wa(img.wout, kImgWO);
        }
      }
      // ---- QKV epilogue: Q -> TMEM A, K/V -> smem (once both tiles' previous P.V retired) ----
      wait_mma();
      {
        if (n_kv > 0) mbar_wait_sleep(&tc2.kvfree, (n_kv - 1) & 1);
        const uint32_t cq = lanebase + kTD;
        float v[32];
        float kn2 = 0.0f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          ld32f(cq + 32 * h, v);
          if (!ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0f;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) qn2 = fmaf(v[i], v[i], qn2);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) split_pair(v[16 * c + 2 * i], v[16 * c + 2 * i + 1], hi[i], lo[i]);
            tmem_st8(cA + 16 * h + 8 * c, hi);
            tmem_st8(cA + 32 + 16 * h + 8 * c, lo);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // K: K-major slabs, chunk c of row r at c*(S_pad*16) + r*16
          ld32f(cq + 64 + 32 * h, v);
          if (mapped) {
            if (!ok) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.0f;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) kn2 = fmaf(v[i], v[i], kn2);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int off = (4 * h + c) * (S_pad * 16) + r * 16;
              split8_store(Khi + off, Klo + off, v + 8 * c);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // V: MN-major (key r, d) at (r/8)*1024 + (d/8)*128 + (r%8)*16 + (d%8)*2
          ld32f(cq + 128 + 32 * h, v);
          if (mapped) {
            if (!ok) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.0f;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int off = (r >> 3) * 1024 + (4 * h + c) * 128 + (r & 7) * 16;
              split8_store(Vhi + off, Vlo + off, v + 8 * c);
            }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) kn2 = fmaxf(kn2, __shfl_xor_sync(0xffffffffu, kn2, o));
        if (lane == 0) atomicMax(&kmax_s[L], __float_as_uint(kn2));
        tmem_st_wait();
        fence_proxy_async();
        fence_before();
        mbar_arrive(&tc2.kvready);  // this row's K/V (and Q) are in place
      }
      if (issuer) {
        mbar_wait(&tc2.kvready, n_kv & 1);  // every key of the layer present
        fence_after();
        is.scores();
        is.commit_mma();
      }
      // ---- causal key-masked softmax -> P (bf16 hi/lo, in place over S) ----
      // single pass with the Cauchy-Schwarz shift m' = ||q_r|| max_j ||k_j|| / 8
      wait_mma();
      float inv_l = 0.0f;
      {
        mbar_wait_sleep(&tc2.kvready, n_kv & 1);  // kmax_s[L] complete (already passed)
        const float mb = sqrtf(qn2 * __uint_as_float(kmax_s[L])) * (0.125f * kLog2e);
        const uint32_t cs = lanebase + kTD;
        const int nch = (t == 0 ? NK0 : S_pad) / 16;
        const int jlast = min(nch - 1, wmax_row / 16);
        float l = 0.0f;
        for (int j0 = 0; j0 < nch; j0 += 2) {
          uint32_t s32[32];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (j0 + u <= jlast) tmem_ld16(cs + 16 * (j0 + u), s32 + 16 * u);  // warp-uniform
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = j0 + u;
            if (j >= nch) break;
            uint32_t hi[8], lo[8];
            uint32_t vm = 0u;
            if (ok && j <= jlast) vm = allowed16(valid_w[j >> 1] >> ((j & 1) * 16), 16 * j, r);
            float pv[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float pe;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(pe) : "f"(fmaf(__uint_as_float(s32[16 * u + e]), 0.125f * kLog2e, -mb)));
              pv[e] = ((vm >> e) & 1u) ? pe : 0.0f;
              l += pv[e];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) split_pair(pv[2 * i], pv[2 * i + 1], hi[i], lo[i]);
            tmem_st8(cs + 16 * j, hi);
            tmem_st8(cs + 16 * j + 8, lo);
          }
        }
        inv_l = l > 0.0f ? 1.0f / l : 0.0f;  // a valid row always sees itself
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.pv();
        is.commit_mma();
        commit(&tc2.kvfree);  // this tile no longer reads K/V of this layer
      }
      ++n_kv;
      // ---- O / l -> A ----
      wait_mma();
      {
        float o[kDModel];
        ld64(cA, o);
#pragma unroll
        for (int j = 0; j < kDModel; ++j) o[j] = ok ? o[j] * inv_l : 0.0f;
        st_split<64>(cA, o);
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.need_wb();
        is.wo();
        is.commit_mma();
      }
      // ---- x += O Wo ; LN2 -> A ----
      wait_mma();
      {
        float d[kDModel];
        ld64(lanebase + kTD, d);
        if (ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) x[j] += d[j];
        }
        layer_norm_reg(x, lnp_s[L][2], lnp_s[L][3], d);
        if (!ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) d[j] = 0.0f;
        }
        st_split<64>(cA, d);
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.w1();
        is.commit_mma();
      }
      // ---- ReLU(h) -> A2 ----
      wait_mma();
      {
        float h[kFfn];
        ld32f(lanebase + kTW1, h);
#pragma unroll
        for (int j = 0; j < kFfn; ++j) h[j] = ok ? fmaxf(h[j], 0.0f) : 0.0f;
        st_split<32>(lanebase + kTA2, h);
        tmem_st_wait();
        done();
      }
      if (issuer) {
        is.wait_simt();
        is.w2();
        is.commit_mma();
        commit(&tc2.wb_free);
        if (t == 1) is.refill_wb(img.wb[(L + 1) % NL]);  // next layer's (or candidate's) Wo|W1|W2
      }
      // ---- x += ReLU(h) W2 ----
      wait_mma();
      {
        float d[kDModel];
        ld64(lanebase + kTW2, d);
        if (ok) {
#pragma unroll
          for (int j = 0; j < kDModel; ++j) x[j] += d[j];
        }
      }
    }

    if (U && in_seq) {  // forward_fused output rows (padded rows are zero)
      float4* dst = reinterpret_cast<float4*>(U + ((size_t)item * S + r) * kDModel);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        dst[j] = ok ? make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3])
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // ---- K5: y = x out_linear, masked max over rows, CTR head ----
    st_split<64>(cA, x);  // invalid rows carry x = 0
    tmem_st_wait();
    done();
    if (issuer) {
      is.wait_simt();
      is.need_wa();
      is.pool();
      is.commit_mma();
      commit(&tc2.wa_free);
      if (t == 1) is.refill_wa(img.wa[0], kImgWA);  // next candidate's layer-0 Wqkv
    }
    wait_mma();
    {
      float y[kDModel];
      ld64(lanebase + kTD, y);
      if (tid == 0) any_s = 0;
      named_bar_sync(1, kRowThreads);  // every row is past its last softmax
      if (ok) any_s = 1;
      if (tid < 8) valid_w[tid] = 0u;
#pragma unroll
      for (int j = 0; j < kDModel; ++j) {
        const float v = warp_max_f32(ok ? y[j] : -INFINITY);
        if (lane == 0) red_s[warp][j] = v;
      }
    }
    named_bar_sync(1, kRowThreads);
    if (logits) {
      if (tid < kDModel) {
        float v = -INFINITY;
#pragma unroll
        for (int w = 0; w < kSkRowWarps; ++w) v = fmaxf(v, red_s[w][tid]);
        v = any_s ? v : 0.0f;  // empty user -> pooled = 0 (trainer.py:358-359)
        z_s[tid] = v;
        if (pooled_out) pooled_out[(size_t)item * kDModel + tid] = v;
      } else if (tid < kDModel + kEmbed) {
        z_s[tid] = use_staged ? st.cand_unit[(size_t)item * kEmbed + tid - kDModel] : 0.0f;
      } else if (tid < kDModel + kEmbed + kCtx) {
        z_s[tid] = use_staged ? st.ctx[st.item_req[item] * kCtx + tid - kDModel - kEmbed] : 0.0f;
      }
      named_bar_sync(1, kRowThreads);
      if (tid < kHidden) {
        float h = 0.0f;
        for (int i = 0; i < kDModel + kEmbed + kCtx; ++i) h = fmaf(z_s[i], __ldg(p.head_w1 + i * kHidden + tid), h);
        hid_s[tid] = fmaxf(h + __ldg(p.head_b1 + tid), 0.0f);
      }
      named_bar_sync(1, kRowThreads);
      if (tid < kHeads) {
        float o = 0.0f;
        for (int j = 0; j < kHidden; ++j) o = fmaf(hid_s[j], __ldg(p.head_w2 + j * kHeads + tid), o);
        logits[(size_t)item * kHeads + tid] = o + __ldg(p.head_b2 + tid);
      }
    }
    named_bar_sync(1, kRowThreads);  // smem (valid_w, red_s, z_s, kmax_s) reuse by the next item
  }
  if (issuer && t == 1) {  // drain the loader's last prefetches before the CTA retires
    mbar_wait(&tc2.wa_full, (is.ph >> 1) & 1u);
    mbar_wait(&tc2.wb_full, (is.ph >> 2) & 1u);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(0u);
  cta_stamp(kDbgSkut, 1);
}

cudaError_t set_dbg_cta_skut(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t set_debug_skut(long long* dev) { return cudaMemcpyToSymbol(g_dbg_skut, &dev, sizeof(dev)); }

cudaError_t launch_skut_tc(const Params& p, const SkutImages& img, const NNCfg& nn,
                           const Staged* st, const int32_t* idx, const float* F,
                           const uint8_t* fmask, int n, float* U, float* logits, float* pooled,
                           cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int S_pad = (nn.seq_len + 15) & ~15;
  const size_t smem = (size_t)kImgWA + kImgWB + 4 * (size_t)S_pad * 128;
  // S <= 192: tile-decoupled kernel; 192 < S <= 256: the coupled 2-tile kernel
  auto kern = S_pad <= 192 ? skut_tc2_kernel : skut_tc_kernel;
  cudaError_t e = set_max_dyn_smem((const void*)kern, (int)smem);
  if (e != cudaSuccess) return e;
  const int sms = device_sms();
  Staged dummy{};
  e = launch_pdl(kern, dim3(n < sms ? n : sms), dim3(kSkThreads), smem, s, p, img, nn, st ? *st : dummy,
                 (int)(st != nullptr), idx, F, fmask, n, U, logits, pooled);
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr, "skut_tc launch failed: regs=%d maxThreads=%d static_smem=%zu dyn_smem=%zu local=%zu\n",
            fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, smem, fa.localSizeBytes);
  }
  return e;
}

}  // namespace tav2
