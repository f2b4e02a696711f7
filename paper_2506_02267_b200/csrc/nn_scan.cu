// K2 on the tensor cores: candidate-anchored NN scores of a 128-candidate
// tile against a token chunk, as a threshold scan (no per-thread top-k).
//
// Reference semantics (nnsearch.py:274-286, :313-347): score(t, c) =
// f64(unit(dequantize(q_t))) . f64(unit(c)), top-k by (score desc, index asc).
//
// Tensor-core part: approximate scores for every (candidate, token) as a
// bf16x3 GEMM of the f32 unit vectors (x = hi + lo, a.b ~= ah.bh + ah.bl +
// al.bh), M = 128 candidates x N = 64 tokens x K = 32 per tile, f32
// accumulation in TMEM.  |approx - exact| <= 3*2^-18*sum|a_j b_j| + f32
// accumulation <= 2.3e-5 for unit vectors (measured max 5.7e-6,
// tools/measure_bf16x3_err.py) < kGateEps.
//
//   pass 1 (group max): every (candidate, source) splits the source into
//          groups of G = 2^glog consecutive tokens (G-aligned in the global
//          token index, glog chosen by the planner so that a source has
//          about 4k..8k groups) and writes each group's approximate maximum.
//   nn_bound_kernel: T = k-th largest group maximum.  k distinct groups hold
//          a token with approx >= T, so the exact k-th best score is >= T -
//          eps and every exact top-k token has approx >= T - 2 eps.
//   pass 2 (compaction): every token with approx >= T - 2 eps is appended
//          (source index, u16) to the (candidate, source) survivor list.
//   nn_select_kernel (nn_select.cu) re-scores the survivors exactly (f64,
//          the reference formula) and selects the top k.
// Both scan passes are branch-light per score (a max or a compare), so the
// epilogue keeps pace with the tensor core instead of running a divergent
// per-thread insertion sort.
//
// Roles (320 threads): warps 0-7 epilogue (warp w reads TMEM lanes
// 32*(w%4).. = candidates, column half w/4 of every tile), warp 8 producer
// (one 8 KB cp.async.bulk per pre-tiled 64-token bf16 hi/lo image written by
// prep_kernel, 8-stage ring), warp 9 MMA issuer.  TMEM: 4 accumulator
// buffers x 64 columns.  Chunk boundaries are 64-token aligned (planner), so
// every group is scanned by exactly one CTA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

constexpr int kNT = 64;          // tokens per MMA tile (N)
constexpr int kStages = 8;       // smem ring depth
constexpr int kAcc = 4;          // TMEM accumulator buffers
constexpr int kTcThreads = 320;
constexpr int kProdWarp = 8, kMmaWarp = 9;
constexpr int kEpiThreads = 256;

constexpr int kASlab = 128 * 16;            // one 16-byte K chunk of 128 candidate rows
constexpr int kAHalf = 4 * kASlab;          // 32 bf16 of 128 rows (8 KB)
constexpr int kBTile = 8 * kNT * 16;        // token tile: 8 chunks (hi 0-3, lo 4-7) x 64 rows (8 KB)

__device__ long long* g_dbg_timeline = nullptr;
__device__ int g_dbg_block = 0;

// max over groups of G = 2^GL consecutive values of v[32] -> out[32 >> GL]
template <int GL>
__device__ __forceinline__ void group_max(const float* v, float* out) {
  constexpr int G = 1 << GL;
#pragma unroll
  for (int g = 0; g < 32 / G; ++g) {
    float m = v[g * G];
#pragma unroll
    for (int e = 1; e < G; ++e) m = fmaxf(m, v[g * G + e]);
    out[g] = m;
  }
}

template <int GL>
__device__ __forceinline__ void write_groups(const float* v, float* dst, int g_first, int g_lo,
                                             int g_hi) {
  float m[32 >> GL];
  group_max<GL>(v, m);
#pragma unroll
  for (int g = 0; g < (32 >> GL); ++g) {
    const int gg = g_first + g;  // global group index
    if (gg >= g_lo && gg <= g_hi) dst[gg - g_lo] = m[g];
  }
}

__global__ void __launch_bounds__(kTcThreads, 1) nn_scan_kernel(Staged st, NNCfg nn, NNScan sc,
                                                                int pass) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;               // [hi: 4 chunks][lo: 4 chunks] x 128 rows x 16 B
  uint8_t* Bs = sm + 2 * kAHalf;  // [kStages][bf16 image 8 chunks x 64 rows x 16 B]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[kAcc], tempty[kAcc];
  __shared__ uint32_t taddr_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const NNWork w = st.work[blockIdx.x];
  const NNTile tile = st.tiles[w.tile];
  const ReqInfo rq = st.req[tile.req];
  const int src = w.source;
  // global token ranges: the source's scanned range and this chunk
  const int s_lo = rq.tok_off[src] + (src == 1 ? nn.recent : 0);
  const int s_hi = rq.tok_off[src] + rq.len[src];
  const int g0 = rq.tok_off[src] + w.t0, g1 = rq.tok_off[src] + w.t1;
  const int tile0 = g0 / kNT;
  const int ntiles = (g1 + kNT - 1) / kNT - tile0;

  // ---- prologue: candidate hi/lo (A operand), barriers, TMEM ----
  if (warp < 4) {
    const int c = tid;
    const bool real = c < tile.n;
    const float4* cu = reinterpret_cast<const float4*>(st.cand_unit + (size_t)(tile.item0 + (real ? c : 0)) * kEmbed);
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {  // 8 elements per 16-byte chunk
      const float4 v0 = cu[2 * ch], v1 = cu[2 * ch + 1];
      const float f[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) split_pair(real ? f[2 * i] : 0.f, real ? f[2 * i + 1] : 0.f, hi[i], lo[i]);
      *reinterpret_cast<uint4*>(As + ch * kASlab + c * 16) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(As + kAHalf + ch * kASlab + c * 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  } else if (warp == kProdWarp) {
    if (lane == 0) {
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);  // the MMA commit frees the stage
      }
      for (int b = 0; b < kAcc; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], kEpiThreads);
      }
      mbar_fence_init();
    }
  } else if (warp == kMmaWarp) {
    tmem_alloc<256>(&taddr_s);
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t T = taddr_s;

  if (warp == kProdWarp) {
    // ---- producer: one bulk copy per pre-tiled 8 KB token tile ----
    if (lane == 0) {
      const uint8_t* img = reinterpret_cast<const uint8_t*>(st.tok_bf16);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], kBTile);
        bulk_g2s(Bs + s * kBTile, img + (size_t)(tile0 + i) * kBTile, kBTile, &full[s]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer: 2 k-steps x 3 terms per tile ----
    if (lane == 0) {
      const uint32_t id = idesc_bf16(128, kNT);
      const uint32_t a_hi = smem_u32(As), a_lo = a_hi + kAHalf;
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages, b = i % kAcc;
        mbar_wait(&full[s], (i / kStages) & 1);
        mbar_wait(&tempty[b], ((i / kAcc) & 1) ^ 1);
        fence_after();
        const uint32_t b_hi = smem_u32(Bs + s * kBTile), b_lo = b_hi + 4 * kNT * 16;
        const uint32_t d = T + b * kNT;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint64_t ah = sdesc(a_hi + 2 * j * kASlab, kASlab, 128);
          const uint64_t al = sdesc(a_lo + 2 * j * kASlab, kASlab, 128);
          const uint64_t bh = sdesc(b_hi + 2 * j * kNT * 16, kNT * 16, 128);
          const uint64_t bl = sdesc(b_lo + 2 * j * kNT * 16, kNT * 16, 128);
          mma_bf16_ss(d, ah, bh, id, j > 0);
          mma_bf16_ss(d, ah, bl, id, 1);
          mma_bf16_ss(d, al, bh, id, 1);
        }
        commit(&empty[s]);
        commit(&tfull[b]);
      }
    }
  } else {
    // ---- epilogue: thread = (candidate, column half) ----
    const int c = tid & 127;
    const int half = warp >> 2;
    const bool mine = c < tile.n;
    const int item = tile.item0 + (mine ? c : 0);
    const int glog = rq.glog[src];
    const int gl_lo = s_lo >> glog, gl_hi = (s_hi - 1) >> glog;  // the source's global groups
    float* gdst = sc.gmax + ((size_t)item * 3 + src) * sc.gcap;
    float gate = 0.0f;
    unsigned* cnt = sc.count + (size_t)item * 3 + src;
    uint16_t* sdst = sc.surv + (size_t)item * sc.surv_stride + (rq.tok_off[src] - rq.tok_off[0]);
    if (pass == 2) gate = sc.bound[(size_t)item * 3 + src] - 2.0f * kGateEps;
    const uint32_t lane_base = T + ((uint32_t)((warp & 3) * 32) << 16) + 32 * half;
    for (int i = 0; i < ntiles; ++i) {
      const int b = i % kAcc;
      const int col0 = (tile0 + i) * kNT + 32 * half;  // global token of column 0
      mbar_wait(&tfull[b], (i / kAcc) & 1);
      fence_after();
      float v[32];
      tmem_ld32(lane_base + b * kNT, reinterpret_cast<uint32_t*>(v));
      tmem_ld_wait();
      fence_before();
      mbar_arrive(&tempty[b]);
      if (col0 + 32 <= g0 || col0 >= g1) continue;  // warp-uniform: half outside the chunk
      const bool partial = col0 < g0 || col0 + 32 > g1;
      uint32_t valid = 0xffffffffu;
      if (partial) {
        const int a = max(g0 - col0, 0), z = min(g1 - col0, 32);
        valid = (z >= 32 ? 0xffffffffu : ((1u << z) - 1u)) & ~((1u << a) - 1u);
      }
      if (pass == 1) {
        if (partial) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = ((valid >> e) & 1u) ? v[e] : -INFINITY;
        }
        if (!mine) continue;
        const int gf = col0 >> glog;
        switch (glog) {
          case 0: write_groups<0>(v, gdst, gf, gl_lo, gl_hi); break;
          case 1: write_groups<1>(v, gdst, gf, gl_lo, gl_hi); break;
          case 2: write_groups<2>(v, gdst, gf, gl_lo, gl_hi); break;
          case 3: write_groups<3>(v, gdst, gf, gl_lo, gl_hi); break;
          case 4: write_groups<4>(v, gdst, gf, gl_lo, gl_hi); break;
          default: write_groups<5>(v, gdst, gf, gl_lo, gl_hi); break;
        }
      } else {
        uint32_t m = 0u;
#pragma unroll
        for (int e = 0; e < 32; ++e) m |= (v[e] >= gate ? 1u : 0u) << e;
        m &= valid;
        if (!mine || m == 0u) continue;
        unsigned pos = atomicAdd(cnt, (unsigned)__popc(m));
        const int base = col0 - rq.tok_off[src];  // source index of column 0
        while (m) {
          const int e = __ffs(m) - 1;
          m &= m - 1;
          sdst[pos++] = (uint16_t)(base + e);
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_free<256>(T);
}

// T = k-th largest group maximum of a (candidate, source): one warp per
// (candidate, source), MSB-first radix select over order-preserving u32
// images (8-bit digits, early exit once the k-th is isolated).  Also resets
// the pass-2 survivor counter.
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u >> 31) ? (u & 0x7fffffffu) : ~u);
}

constexpr int kBoundWarps = 4;

__global__ void __launch_bounds__(32 * kBoundWarps) nn_bound_kernel(Staged st, NNCfg nn, NNScan sc) {
  extern __shared__ uint32_t bvals[];  // [kBoundWarps][gcap]
  __shared__ unsigned hist_s[kBoundWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kBoundWarps + warp;
  const int s = blockIdx.y;
  if (item >= st.n_items) return;
  if (lane == 0) sc.count[(size_t)item * 3 + s] = 0u;
  const ReqInfo rq = st.req[st.item_req[item]];
  const int k = nn.k[s];
  const int lo = rq.tok_off[s] + (s == 1 ? nn.recent : 0), hi = rq.tok_off[s] + rq.len[s];
  if (k == 0 || hi - lo <= k) return;  // no scan: everything (or nothing) is selected
  const int glog = rq.glog[s];
  const int ng = ((hi - 1) >> glog) - (lo >> glog) + 1;
  float* out = sc.bound + (size_t)item * 3 + s;
  if (ng < k) {
    if (lane == 0) *out = -INFINITY;
    return;
  }
  const float* g = sc.gmax + ((size_t)item * 3 + s) * sc.gcap;
  uint32_t* a = bvals + warp * sc.gcap;
  for (int i = lane; i < ng; i += 32) a[i] = f2ord(g[i]);
  __syncwarp();
  uint32_t prefix = 0u, pmask = 0u;
  int want = k;
  unsigned* h = hist_s[warp];
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) h[i] = 0u;
    __syncwarp();
    for (int i = lane; i < ng; i += 32)
      if ((a[i] & pmask) == prefix) atomicAdd(&h[(a[i] >> shift) & 255], 1u);
    __syncwarp();
    unsigned c8[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c8[j] = h[255 - 8 * lane - j];
      tot += c8[j];
    }
    unsigned incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned excl = incl - tot;
    const unsigned sel = __ballot_sync(0xffffffffu, excl < (unsigned)want && (unsigned)want <= incl);
    const int srcl = __ffs(sel) - 1;
    int digit = 0, above = 0, inb = 0;
    if (lane == srcl) {
      unsigned run = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (run + c8[j] >= (unsigned)want) {
          digit = 255 - 8 * lane - j;
          above = (int)run;
          inb = (int)c8[j];
          break;
        }
        run += c8[j];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, srcl);
    above = __shfl_sync(0xffffffffu, above, srcl);
    inb = __shfl_sync(0xffffffffu, inb, srcl);
    want -= above;
    prefix |= (uint32_t)digit << shift;
    pmask |= 255u << shift;
    __syncwarp();
    if (inb == want) {  // the whole bucket is in the top k: its minimum is the k-th
      uint32_t mn = 0xffffffffu;
      for (int i = lane; i < ng; i += 32)
        if ((a[i] & pmask) == prefix) mn = min(mn, a[i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      prefix = mn;
      break;
    }
  }
  if (lane == 0) *out = ord2f(prefix);
}

cudaError_t set_debug_timeline(long long* dev, int block) {
  cudaError_t e = cudaMemcpyToSymbol(g_dbg_block, &block, sizeof(block));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_dbg_timeline, &dev, sizeof(dev));
}

cudaError_t launch_nn_scan(const Staged& st, const NNCfg& nn, const NNScan& sc, int pass,
                           cudaStream_t s) {
  if (st.n_work == 0) return cudaSuccess;
  const size_t smem = 2 * kAHalf + kStages * kBTile;
  cudaError_t e = cudaFuncSetAttribute(nn_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  nn_scan_kernel<<<st.n_work, kTcThreads, smem, s>>>(st, nn, sc, pass);
  return cudaGetLastError();
}

cudaError_t launch_nn_bound(const Staged& st, const NNCfg& nn, const NNScan& sc, cudaStream_t s) {
  if (st.n_items == 0) return cudaSuccess;
  const size_t smem = (size_t)kBoundWarps * sc.gcap * 4;
  cudaError_t e = cudaFuncSetAttribute(nn_bound_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((st.n_items + kBoundWarps - 1) / kBoundWarps, 3);
  nn_bound_kernel<<<grid, 32 * kBoundWarps, smem, s>>>(st, nn, sc);
  return cudaGetLastError();
}

}  // namespace tav2
