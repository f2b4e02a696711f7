// K2 on the tensor cores: candidate-anchored NN scores of a 128-candidate
// tile against a token chunk, as a threshold scan (no per-thread top-k).
//
// Reference semantics (nnsearch.py:274-286, :313-347): score(t, c) =
// f64(unit(dequantize(q_t))) . f64(unit(c)), top-k by (score desc, index asc).
//
// Tensor-core part: approximate scores for every (candidate, token) as an
// fp16 GEMM of the f32 unit vectors rounded to fp16, M = 128 candidates x
// N = 256 tokens x K = 32 per tile, f32 accumulation in TMEM:
// |approx - exact| < 9.8e-4 < kGateEps (tav2_common.cuh).  The margin only
// widens the gate: the score density near the k-th is low, so the gate keeps
// ~130 of 16,384 LL tokens for k = 96 (bf16x3 products would keep ~105 for
// three times the tensor work and twice the token bytes).
//
//   pass 1 (group max): every (candidate, source) splits the source into
//          groups of G = 2^glog consecutive tokens (G-aligned in the global
//          token index, glog chosen by the planner so that a source has
//          about 4k..8k groups) and writes each group's approximate maximum.
//   nn_bound_kernel: T <= the k-th largest group maximum (bisection).  k
//          distinct groups hold a token with approx >= T, so the exact k-th
//          best score is >= T - eps and every exact top-k token has approx
//          >= T - 2 eps.
//   pass 2 (gate): every token with approx >= T - 2 eps is appended (source
//          index, u16) to the (candidate, source) survivor list.
//   nn_select_kernel (nn_select.cu) re-scores the survivors exactly (f64,
//          the reference formula) and selects the top k.
// Both scan passes are branch-light per score (a max or a compare), so the
// epilogue keeps pace with the tensor core instead of running a divergent
// per-thread insertion sort.
//
// MMA: N = 256 tokens per instruction.  One warp issues a tcgen05.mma only
// every ~120 cycles whatever its N (tools/mma_bench.cu: the tensor core
// itself needs 32 / 64 / 128 cycles at N = 64 / 128 / 256), so N = 256 is the
// first shape where a single issuer keeps the tensor core busy: 2 MMAs
// (2 k-steps of 16) per 256-token tile.
// Roles (576 threads): warps 0-15 epilogue in two groups of 8 on alternate
// tiles (warp w reads TMEM lanes 32*(w%4).. = candidates, column half
// (w%8)/4 = 128 tokens of its group's tiles in two rounds of two tcgen05.ld +
// one wait; the TMEM load latency, ~0.25 us, dominates a round, and the two
// groups overlap it), warp 16 producer
// (one 16 KB cp.async.bulk per pre-tiled 256-token fp16 image written by
// prep_kernel, 6-stage ring), warp 17 MMA issuer.  TMEM: 2 accumulator
// buffers x 256 columns.  Chunk boundaries are tile aligned (planner), so
// every group is scanned by exactly one CTA.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "dbg.cuh"
#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

constexpr int kNT = kScanTile;   // tokens per tile and MMA (N = 256)
constexpr int kStages = 6;       // smem ring depth
constexpr int kAcc = 2;          // TMEM accumulator buffers (2 x 256 columns)
constexpr int kTcThreads = 576;
constexpr int kProdWarp = 16, kMmaWarp = 17;
constexpr int kEpiThreads = 512;
constexpr int kGrpThreads = 256;  // epilogue group: warps 0-7 take even tiles, 8-15 odd tiles
constexpr int kBTile = kScanTileBytes;      // 4 chunks x 256 rows x 16 B = 16 KB
constexpr int kASlab = 128 * 16;            // one 16-byte K chunk of 128 candidate rows
constexpr int kATile = 4 * kASlab;          // 32 fp16 of 128 rows (8 KB)
constexpr int kSurvBuf = 16;                // pass-2 survivors buffered per thread before a flush

// Debug timeline (tav2_debug_timeline): %globaltimer stamps of work unit
// g_dbg_block: slot 160*(pass-1) + {0 inputs ready, 8+i producer copy of tile
// i, 40+i MMA issue, 72+i epilogue thread 0 sees tile i, 104+i thread 0 done
// with tile i, 150 CTA end}.
__device__ long long* g_dbg_timeline = nullptr;
__device__ int g_dbg_block = 0;
#define SCAN_STAMP(slot)                                                             \
  do {                                                                               \
    if (kDebug && dbgp) {                                                            \
      long long t_;                                                                  \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                          \
      dbgp[(slot) + 160 * (pass - 1)] = t_;                                          \
    }                                                                                \
  } while (0)
// pass-1 per-warp stamps: slot 1100 + (tile * 16 + warp) * 6 + which, tiles < 4
#define WARP_STAMP(tile_, which)                                                     \
  do {                                                                               \
    if (kDebug && dbgp && pass == 1 && lane == 0 && (tile_) < 4) {                   \
      long long t_;                                                                  \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                          \
      dbgp[1100 + ((tile_) * 16 + warp) * 6 + (which)] = t_;                          \
    }                                                                                \
  } while (0)

// Store the group maxima of one 32-column quarter v[32].  dst is the
// (candidate, source) row indexed by global group - gbase (gbase = 8-aligned
// first group), so a quarter's 32 >> GL groups are contiguous and 16-byte
// aligned whenever there are >= 4 of them: a quarter inside the chunk stores
// vectors.
template <int GL>
__device__ __forceinline__ void write_groups(const float* v, float* dst, int g_first, int g_lo,
                                             int g_hi, bool whole) {
  constexpr int G = 1 << GL, NG = 32 >> GL;
  float m[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) m[g] = max_run<G>(v + g * G);
  float* d = dst + g_first;
  if (whole) {
    if constexpr (NG >= 4) {
#pragma unroll
      for (int g = 0; g < NG; g += 4) *reinterpret_cast<float4*>(d + g) = make_float4(m[g], m[g + 1], m[g + 2], m[g + 3]);
    } else if constexpr (NG == 2) {
      *reinterpret_cast<float2*>(d) = make_float2(m[0], m[1]);
    } else {
      d[0] = m[0];
    }
    return;
  }
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int gg = g_first + g;  // global group index
    if (gg >= g_lo && gg <= g_hi) d[g] = m[g];
  }
}

// valid-column mask of the 32 columns starting at col0 within [g0, g1)
__device__ __forceinline__ uint32_t range_mask(int col0, int g0, int g1) {
  const int a = max(g0 - col0, 0), z = min(g1 - col0, 32);
  if (a >= z) return 0u;
  return (z >= 32 ? 0xffffffffu : ((1u << z) - 1u)) & ~((1u << a) - 1u);
}

__global__ void __launch_bounds__(kTcThreads, 1) nn_scan_kernel(Staged st, NNCfg nn, NNScan sc,
                                                                int pass) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;          // candidates: 4 chunks x 128 rows x 16 B (fp16)
  uint8_t* Bs = sm + kATile;  // [kStages][16 KB token image]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[kAcc], tempty[kAcc];
  __shared__ uint32_t taddr_s;
  __shared__ uint16_t sbuf[kSurvBuf][kEpiThreads];  // pass 2: per-thread survivor buffer
  __shared__ __align__(16) float gstage[kAcc][2][128][kNT / 32];  // pass 1, G = 32: [group][tile parity]

  cta_stamp(pass == 1 ? kDbgScan1 : kDbgScan2, 0);
  long long* const dbgp = kDebug && blockIdx.x == g_dbg_block ? g_dbg_timeline : nullptr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const NNWork w = st.work[blockIdx.x];
  const NNTile tile = st.tiles[w.tile];
  const ReqInfo& rq = st.req[tile.req];  // (global: indexed by a runtime source)
  const int src = w.source;
  const int tok_off = rq.tok_off[src], tok_off0 = rq.tok_off[0], glog = rq.glog[src];
  // global token ranges: the source's scanned range and this chunk
  const int s_lo = tok_off + (src == 1 ? nn.recent : 0);
  const int s_hi = tok_off + rq.len[src];
  const int g0 = tok_off + w.t0, g1 = tok_off + w.t1;
  const int tile0 = g0 / kNT;
  const int ntiles = (g1 + kNT - 1) / kNT - tile0;

  // ---- prologue: barriers, TMEM (input independent) ----
  if (warp == kProdWarp) {
    if (lane == 0) {
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);  // the MMA commit frees the stage
      }
      for (int b = 0; b < kAcc; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], kGrpThreads);
      }
      mbar_fence_init();
    }
  } else if (warp == kMmaWarp) {
    tmem_alloc<512>(&taddr_s);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;
  griddep_launch();
  griddep_wait();  // prep (cand_unit, tok_img) / bound (gate) complete
  cta_stamp(pass == 1 ? kDbgScan1 : kDbgScan2, 2);
  if (tid == 0) SCAN_STAMP(0);
  // ---- candidates fp16 (A operand, smem K-major slabs) ----
  if (warp < 4) {
    const int c = tid;
    const bool real = c < tile.n;
    const float4* cu = reinterpret_cast<const float4*>(st.cand_unit + (size_t)(tile.item0 + (real ? c : 0)) * kEmbed);
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {  // 8 elements per 16-byte chunk
      const float4 v0 = cu[2 * ch], v1 = cu[2 * ch + 1];
      const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      uint32_t h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __half2 p = __floats2half2_rn(real ? f[2 * i] : 0.f, real ? f[2 * i + 1] : 0.f);
        h[i] = *reinterpret_cast<const uint32_t*>(&p);
      }
      *reinterpret_cast<uint4*>(As + ch * kASlab + c * 16) = make_uint4(h[0], h[1], h[2], h[3]);
    }
  }
  fence_proxy_async();
  __syncthreads();

  if (warp == kProdWarp) {
    // ---- producer: one bulk copy per pre-tiled 16 KB token tile ----
    if (lane == 0) {
      const uint8_t* img = reinterpret_cast<const uint8_t*>(st.tok_img);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        if (i < 32) SCAN_STAMP(8 + i);
        mbar_expect_tx(&full[s], kBTile);
        bulk_g2s(Bs + s * kBTile, img + (size_t)(tile0 + i) * kBTile, kBTile, &full[s]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer: 2 k-steps per tile ----
    if (lane == 0) {
      const uint32_t id = idesc_f16(128, kNT);
      const uint32_t a0 = smem_u32(As);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages, b = i % kAcc;
        mbar_wait(&full[s], (i / kStages) & 1);
        mbar_wait(&tempty[b], ((i / kAcc) & 1) ^ 1);
        fence_after();
        if (i < 32) SCAN_STAMP(40 + i);
        const uint32_t b0 = smem_u32(Bs + s * kBTile);
        const uint32_t d = T + b * kNT;
#pragma unroll
        for (int j = 0; j < 2; ++j)
          mma_bf16_ss(d, sdesc(a0 + 2 * j * kASlab, kASlab, 128), sdesc(b0 + 2 * j * kNT * 16, kNT * 16, 128), id,
                      j > 0);
        commit(&empty[s]);
        commit(&tfull[b]);
        if (kDebug && dbgp && i < 32) {  // MMA completion latency (debug builds only)
          mbar_wait(&tfull[b], (i / kAcc) & 1);
          SCAN_STAMP(520 - 120 * (pass - 1) + i);  // dbgp[520 + 40 * (pass - 1) + i]
        }
      }
    }
  } else {
    // ---- epilogue: two groups of 8 warps on alternate tiles (accumulator
    // buffer = group), so one group's TMEM loads overlap the other's
    // processing; thread = (candidate, 128-column half), two 64-column rounds
    // per tile ----
    const int grp = warp >> 3, gw = warp & 7, gtid = tid & (kGrpThreads - 1);
    const int c = tid & 127;
    const bool mine = c < tile.n;
    const int item = tile.item0 + (mine ? c : 0);
    const int gl_lo = s_lo >> glog, gl_hi = (s_hi - 1) >> glog;  // the source's global groups
    float* gdst = sc.gmax + ((size_t)item * 3 + src) * sc.gcap - (gl_lo & ~7);
    unsigned* cnt = sc.count + (size_t)item * 3 + src;
    uint16_t* sdst = sc.surv + (size_t)item * sc.surv_stride + (tok_off - tok_off0);
    const float gate = pass == 2 ? sc.bound[(size_t)item * 3 + src] - 2.0f * kGateEps : 0.0f;
    int nb = 0;  // pass 2: survivors buffered in sbuf[.][tid]
    auto flush = [&]() {
      const unsigned pos = atomicAdd(cnt, (unsigned)nb);
      for (int j = 0; j < nb; ++j) sdst[pos + j] = sbuf[j][tid];
      nb = 0;
    };
    const uint32_t lane_base = T + ((uint32_t)((warp & 3) * 32) << 16) + 128 * (gw >> 2);
    for (int i = grp; i < ntiles; i += kAcc) {
      const int b = grp;
      float(*const gs)[kNT / 32] = gstage[b][(i / kAcc) & 1];
      mbar_wait_sleep(&tfull[b], (i / kAcc) & 1);
      fence_after();
      if (gtid == 0 && i < 32) SCAN_STAMP(72 + i);
#pragma unroll 1
      for (int hq = 0; hq < 2; ++hq) {
        const int cq = 2 * (gw >> 2) + hq;  // 64-column quarter of the tile
        float v[64];
        tmem_ld32(lane_base + b * kNT + 64 * hq, reinterpret_cast<uint32_t*>(v));
        tmem_ld32(lane_base + b * kNT + 64 * hq + 32, reinterpret_cast<uint32_t*>(v + 32));
        tmem_ld_wait();
        WARP_STAMP(i, 2 * hq);
        if (hq == 1) {
          fence_before();
          mbar_arrive(&tempty[b]);
          if (gtid == 0 && i < 32) SCAN_STAMP(104 + i);
        }
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {  // two 32-column quarters
          const int col0 = (tile0 + i) * kNT + 64 * cq + 32 * qq;  // global token of column 0
          if (col0 + 32 <= g0 || col0 >= g1 || !mine) {
            if (pass == 1 && glog == 5) gs[c][2 * cq + qq] = -INFINITY;
            continue;
          }
          const bool partial = col0 < g0 || col0 + 32 > g1;
          const uint32_t valid = partial ? range_mask(col0, g0, g1) : 0xffffffffu;
          float* q = v + 32 * qq;
          if (pass == 1) {
            if (glog == 5) {  // one group per quarter: staged, written coalesced below
              float m;
              if (!partial) {
                m = max_run<32>(q);
              } else {
                m = -INFINITY;
#pragma unroll
                for (int e = 0; e < 32; ++e) m = fmaxf(m, ((valid >> e) & 1u) ? q[e] : -INFINITY);
              }
              gs[c][2 * cq + qq] = m;
              continue;
            }
            if (partial) {
#pragma unroll
              for (int e = 0; e < 32; ++e) q[e] = ((valid >> e) & 1u) ? q[e] : -INFINITY;
            }
            const int gf = col0 >> glog;
            switch (glog) {
              case 0: write_groups<0>(q, gdst, gf, gl_lo, gl_hi, !partial); break;
              case 1: write_groups<1>(q, gdst, gf, gl_lo, gl_hi, !partial); break;
              case 2: write_groups<2>(q, gdst, gf, gl_lo, gl_hi, !partial); break;
              case 3: write_groups<3>(q, gdst, gf, gl_lo, gl_hi, !partial); break;
              case 4: write_groups<4>(q, gdst, gf, gl_lo, gl_hi, !partial); break;
              default: write_groups<5>(q, gdst, gf, gl_lo, gl_hi, !partial); break;
            }
          } else {
            // survivors are rare: test the quarter's maximum first
            if (!(max_run<32>(q) >= gate)) continue;
            uint32_t m = 0u;
#pragma unroll
            for (int e = 0; e < 32; ++e) m |= (q[e] >= gate ? 1u : 0u) << e;
            m &= valid;
            const int base = col0 - tok_off;  // source index of column 0
            while (m) {  // rare: ~k survivors per (candidate, source) in total
              const int e = __ffs(m) - 1;
              m &= m - 1;
              sbuf[nb++][tid] = (uint16_t)(base + e);
              if (nb == kSurvBuf) flush();
            }
          }
        }
        WARP_STAMP(i, 2 * hq + 1);
      }
      if (pass == 1 && glog == 5) {
        // coalesced write-out of this tile's group maxima: thread -> (candidate,
        // 4-group half); the group row of a candidate is contiguous in gmax
        named_bar_sync(1 + grp, kGrpThreads);
        WARP_STAMP(i, 4);
        const int cc = gtid >> 1, hh = gtid & 1;
        const int gg0 = (tile0 + i) * (kNT / 32) + 4 * hh;  // global group index of the 4
        if (cc < tile.n) {
          float* dst = sc.gmax + ((size_t)(tile.item0 + cc) * 3 + src) * sc.gcap - (gl_lo & ~7);
          const float* sv = &gs[cc][4 * hh];
          if (gg0 >= gl_lo && gg0 + 3 <= gl_hi) {
            *reinterpret_cast<float4*>(dst + gg0) = *reinterpret_cast<const float4*>(sv);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (gg0 + k >= gl_lo && gg0 + k <= gl_hi) dst[gg0 + k] = sv[k];
          }
        }
        WARP_STAMP(i, 5);
      }
    }
    if (pass == 2 && nb > 0) flush();
  }
  fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_free<512>(T);
  cta_stamp(pass == 1 ? kDbgScan1 : kDbgScan2, 1);
  if (tid == 0) SCAN_STAMP(150);
}

// Gate bound of a (candidate, source): T <= the k-th largest group maximum,
// by bisection on the value range with warp-wide counts (values held in
// registers, kBoundPer per lane; no shared-memory histograms).  The
// invariant count(g >= lo) >= k keeps lo a valid bound; ~14 halvings of
// [min, max] leave it within 1e-4 of the exact k-th value.  Also resets the
// pass-2 survivor counter.
constexpr int kBoundWarps = 4;
constexpr int kBoundPer = 72;  // values per lane: ng <= 8k + 2 <= 2304

__device__ __forceinline__ void nn_bound_body(const Staged& st, const NNCfg& nn, const NNScan& sc);

__global__ void __launch_bounds__(32 * kBoundWarps) nn_bound_kernel(Staged st, NNCfg nn, NNScan sc) {
  nn_bound_body(st, nn, sc);
  __syncthreads();
  cta_stamp(kDbgBound, 1);
}

template <int PER>
__device__ __forceinline__ float bisect_kth(const float* g, int ng, int k, int lane) {
  float v[PER];
  float mn = INFINITY, mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = j * 32 + lane;
    v[j] = i < ng ? __ldg(g + i) : -INFINITY;
    mx = fmaxf(mx, v[j]);
    if (i < ng) mn = fminf(mn, v[j]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  // four independent counters: one counter compiled to a PER-long chain of
  // dependent predicated increments per bisection step (step 0.2062 ->
  // 0.2060 ms; a CTA of 4 warps per (candidate, source) instead, 3000 CTAs,
  // was slower: 0.2067 ms, the CTA launches of the grid set the bound's end)
  static_assert(PER % 4 == 0, "PER must be a multiple of 4");
  auto count_ge = [&](float x) {
    int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int j = 0; j < PER; j += 4) {
      c0 += v[j] >= x ? 1 : 0;
      c1 += v[j + 1] >= x ? 1 : 0;
      c2 += v[j + 2] >= x ? 1 : 0;
      c3 += v[j + 3] >= x ? 1 : 0;
    }
    return (int)__reduce_add_sync(0xffffffffu, (unsigned)((c0 + c1) + (c2 + c3)));
  };
  if (count_ge(mx) >= k) return mx;
  // T only has to stay <= the k-th largest maximum: stop once the bracket is
  // 1e-4 wide (a tenth of the gate margin: a handful of extra survivors at
  // most) or a midpoint counts exactly k
  float lo = mn, hi = mx;  // count(>= lo) >= k > count(>= hi)
#pragma unroll 1
  while (hi - lo > 1e-4f) {
    const float mid = 0.5f * (lo + hi);
    if (!(mid > lo && mid < hi)) break;  // adjacent floats
    const int c = count_ge(mid);
    if (c >= k) {
      lo = mid;
      if (c == k) break;
    } else {
      hi = mid;
    }
  }
  return lo;
}

__device__ __forceinline__ void nn_bound_body(const Staged& st, const NNCfg& nn, const NNScan& sc) {
  cta_stamp(kDbgBound, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kBoundWarps + warp;
  const int s = blockIdx.y;
  griddep_launch();
  // the request's source ranges come from the staged plan (copied before the
  // chain started): read before the wait, their round trips overlap it
  int lo = 0, hi = 0, glog = 0;
  if (item < st.n_items) {
    const ReqInfo& rq = st.req[st.item_req[item]];
    lo = rq.tok_off[s] + (s == 1 ? min(nn.recent, rq.len[1]) : 0);
    hi = rq.tok_off[s] + rq.len[s];
    glog = rq.glog[s];
  }
  griddep_wait();  // scan pass 1 complete (and the previous select is done with count)
  cta_stamp(kDbgBound, 2);
  if (item >= st.n_items) return;
  if (lane == 0) sc.count[(size_t)item * 3 + s] = 0u;
  const int k = nn.k[s];
  if (!nn_scanned(hi - lo, k)) return;  // no scan (nn_select takes every token)
  const int ng = ((hi - 1) >> glog) - (lo >> glog) + 1;
  float* out = sc.bound + (size_t)item * 3 + s;
  const float* g = sc.gmax + ((size_t)item * 3 + s) * sc.gcap + ((lo >> glog) & 7);
  float T;
  if (ng < k) T = -INFINITY;
  else if (ng <= 256) T = bisect_kth<8>(g, ng, k, lane);
  else if (ng <= 512) T = bisect_kth<16>(g, ng, k, lane);
  else if (ng <= 1024) T = bisect_kth<32>(g, ng, k, lane);
  else T = bisect_kth<kBoundPer>(g, ng, k, lane);
  if (lane == 0) *out = T;
}

cudaError_t set_dbg_cta_scan(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t set_debug_timeline(long long* dev, int block) {
  cudaError_t e = cudaMemcpyToSymbol(g_dbg_block, &block, sizeof(block));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_dbg_timeline, &dev, sizeof(dev));
}

cudaError_t launch_nn_scan(const Staged& st, const NNCfg& nn, const NNScan& sc, int pass,
                           cudaStream_t s) {
  if (st.n_work == 0) return cudaSuccess;
  const size_t smem = kATile + (size_t)kStages * kBTile;
  cudaError_t e = set_max_dyn_smem((const void*)nn_scan_kernel, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(nn_scan_kernel, dim3(st.n_work), dim3(kTcThreads), smem, s, st, nn, sc, pass);
}

cudaError_t launch_nn_bound(const Staged& st, const NNCfg& nn, const NNScan& sc, cudaStream_t s) {
  if (st.n_items == 0) return cudaSuccess;
  dim3 grid((st.n_items + kBoundWarps - 1) / kBoundWarps, 3);
  return launch_pdl(nn_bound_kernel, grid, dim3(32 * kBoundWarps), 0, s, st, nn, sc);
}

}  // namespace tav2
