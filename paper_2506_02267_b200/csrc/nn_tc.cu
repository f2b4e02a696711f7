// K2 on the tensor cores: candidate-anchored NN scores of a 128-candidate
// tile against a token chunk, fused with an exact two-pass top-k.
//
// Reference semantics (nnsearch.py:274-286, :313-347): score(t, c) =
// f64(unit(dequantize(q_t))) . f64(unit(c)), top-k by (score desc, index asc).
//
// Tensor-core part: approximate scores for every (candidate, token) as a
// bf16x3 GEMM of the f32 unit vectors (x = hi + lo, a.b ~= ah.bh + ah.bl +
// al.bh), M = 128 candidates x N = 64 tokens x K = 32 per tile, f32
// accumulation in TMEM.  |approx - exact| <= 3*2^-18*sum|a_j b_j| + f32
// accumulation <= 2.3e-5 for unit vectors (measured max 5.7e-6,
// tools/measure_bf16x3_err.py); the gate margin is eps = 1e-4.
// Exact part: the survivors of the gate are re-scored on the SIMT cores with
// the reference formula (f64 dot of the f32 unit vectors), so the selected
// index sets follow the reference's f64 ranking.
//
//   pass 1: each (chunk, column half) keeps, in registers, its top-8
//           approximate scores (2*8*nw >= k by the planner) and publishes
//           them; nn_bound_kernel computes T = k-th largest of the union:
//           >= k tokens have approx >= T, hence the exact k-th best is
//           >= T - eps and every exact top-k token has approx >= T - 2 eps.
//   pass 2: each chunk re-scans, computes exact keys only for approx >=
//           T - 2 eps and keeps the best k (append, heapify when full).
// A single-chunk source (nw == 1) is done exactly in pass 1.  In every exact
// scan, once the heap is full the gate also rises to (k-th best exact score
// held) - 2 eps, evaluated per 64-token tile.
// The merge folds the per-chunk lists (nn_merge.cu).
//
// Roles (320 threads): warps 0-3 epilogue (thread = candidate = TMEM lane;
// in pass 1 warps 4-7 take the upper 32 columns of every tile), warp 8 producer (one 8 KB cp.async.bulk per 64-token tile: prep_kernel
// writes the bf16 hi/lo token image pre-tiled in the UMMA slab layout;
// 4-stage ring), warp 9 MMA issuer.  TMEM: 4 accumulator buffers x 64 cols.
// Tiles follow the global token index, so a chunk's first/last tiles are
// partial; columns outside the chunk are masked in the epilogue.
#include <cuda.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

constexpr int kNT = 64;          // tokens per MMA tile (N)
constexpr int kStages = 4;       // smem ring depth
constexpr int kAcc = 4;          // TMEM accumulator buffers
constexpr int kTcThreads = 320;
constexpr int kEpiWarps = 8;     // pass 1: two threads (column halves) per candidate
constexpr int kProdWarp = 8, kMmaWarp = 9;
constexpr int kTopM = 8;         // pass-1 register list per (chunk, column half)
constexpr float kGateEps = 1e-4f;

constexpr int kASlab = 128 * 16;            // one 16-byte K chunk of 128 candidate rows
constexpr int kAHalf = 4 * kASlab;          // 32 bf16 of 128 rows (8 KB)
constexpr int kBTile = 8 * kNT * 16;        // token tile: 8 chunks (hi 0-3, lo 4-7) x 64 rows (8 KB)
constexpr int kRTile = kNT * kEmbed * 4;    // the same 64 tokens' f32 unit rows (8 KB, exact re-scoring)
constexpr int kStage = kBTile + kRTile;

// Debug timeline (tav2_debug_timeline): %globaltimer stamps of CTA 0.
__device__ long long* g_dbg_timeline = nullptr;
__device__ int g_dbg_block = 0;
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DBG_STAMP(slot)                                                                \
  do {                                                                                 \
    long long* d_ = g_dbg_timeline;                                                    \
    if (d_ && blockIdx.x == g_dbg_block && blockIdx.y == 0) d_[(slot) + 160 * (pass - 1)] = gtime(); \
  } while (0)

template <int M>  // pass-1 register list size (compile time: branch-free bubble)
__global__ void __launch_bounds__(kTcThreads, 1) nn_tc_kernel(Staged st, NNCfg nn, uint64_t* part,
                                                              float* part1, const float* bound, int kmax,
                                                              int tile_size, int pass) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;                                   // [hi: 4 chunks][lo: 4 chunks] x 128 rows x 16 B
  uint8_t* Bs = sm + 2 * kAHalf;  // [kStages][bf16 image 8 chunks x 64 rows x 16 B | f32 rows 64 x 128 B]
  uint64_t* heap = reinterpret_cast<uint64_t*>(Bs + kStages * kStage);  // [k][cpb]
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[kAcc], tempty[kAcc];
  __shared__ uint32_t taddr_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) DBG_STAMP(0);
  const NNWork w = st.work[blockIdx.x];
  const NNTile tile = st.tiles[w.tile];
  const ReqInfo rq = st.req[tile.req];
  const int src = w.source;
  const int nw = tile.nwork[src];
  if (pass == 2 && nw == 1) return;  // pass 1 was already exact (block-uniform)
  const int k = nn.k[src];
  const bool exact = pass == 2 || nw == 1;  // exact keys + heap, else approximate top-M
  const int jchunk = blockIdx.x - tile.work0[src];
  const int cpb = tile_size / gridDim.y;  // candidates owned by this CTA
  const int c_lo = blockIdx.y * cpb;
  // global 64-token tiles covering rows [tok_off + t0, tok_off + t1)
  const int g0 = rq.tok_off[src] + w.t0, g1 = rq.tok_off[src] + w.t1;
  const int tile0 = g0 / kNT;
  const int ntiles = (g1 + kNT - 1) / kNT - tile0;

  // ---- prologue: candidate hi/lo (A operand), heaps, barriers, TMEM ----
  const int nepi = exact ? 128 : 256;  // epilogue threads that consume a stage
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
    if (exact && c >= c_lo && c < c_lo + cpb) {
      uint64_t* hh = heap + (c - c_lo);
      for (int i = 0; i < k; ++i) hh[i * cpb] = 0ull;
    }
  } else if (warp == kProdWarp) {
    if (lane == 0) {
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1 + nepi);  // MMA commit + the epilogue (reads the f32 rows)
      }
      for (int b = 0; b < kAcc; ++b) {
        mbar_init(&tfull[b], 1);
        mbar_init(&tempty[b], nepi);
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
  if (tid == 0) DBG_STAMP(1);

  if (warp == kProdWarp) {
    // ---- producer: one bulk copy per pre-tiled 8 KB token tile ----
    if (lane == 0) {
      const uint8_t* img = reinterpret_cast<const uint8_t*>(st.tok_bf16);
      const uint8_t* rows = reinterpret_cast<const uint8_t*>(st.tok_unit);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        if (i < 32) DBG_STAMP(8 + i);
        mbar_expect_tx(&full[s], kStage);
        bulk_g2s(Bs + s * kStage, img + (size_t)(tile0 + i) * kBTile, kBTile, &full[s]);
        bulk_g2s(Bs + s * kStage + kBTile, rows + (size_t)(tile0 + i) * kRTile, kRTile, &full[s]);
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
        if (i < 32) DBG_STAMP(40 + i);
        mbar_wait(&tempty[b], ((i / kAcc) & 1) ^ 1);
        if (i < 32) DBG_STAMP(72 + i);
        fence_after();
        const uint32_t b_hi = smem_u32(Bs + s * kStage), b_lo = b_hi + 4 * kNT * 16;
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
  } else if (warp < 4 || !exact) {
    // ---- epilogue: approx scores -> top-M (pass 1) / gated exact top-k ----
    const int c = tid & 127;
    const int half = warp >> 2;  // pass 1: column half of every tile
    const bool mine = c >= c_lo && c < c_lo + cpb && c < tile.n;
    uint64_t* h = heap + (c - c_lo);
    uint64_t root = 0ull;
    int hn = 0;  // heap fill (append mode until k, then heapify)
    float top[M];  // descending
#pragma unroll
    for (int i = 0; i < M; ++i) top[i] = -INFINITY;
    float thr = -FLT_MAX;  // exact-path gate (-inf marks columns past the chunk)
    if (pass == 2 && mine) thr = bound[(size_t)(tile.item0 + c) * 3 + src] - 2.0f * kGateEps;
    float uc[kEmbed];  // exact path: this candidate's f32 unit vector
    {
      const float* cu = st.cand_unit + (size_t)(tile.item0 + (mine ? c : 0)) * kEmbed;
#pragma unroll
      for (int j = 0; j < kEmbed; ++j) uc[j] = cu[j];
    }
    const uint32_t lane_base = T + ((uint32_t)((warp & 3) * 32) << 16);
    for (int i = 0; i < ntiles; ++i) {
      const int b = i % kAcc;
      const int tb = (tile0 + i) * kNT - rq.tok_off[src];  // source index of column 0
      mbar_wait(&tfull[b], (i / kAcc) & 1);
      if (tid == 0 && i < 32) DBG_STAMP(104 + i);
      fence_after();
      float sc[kNT];
      if (exact) {
        tmem_ld32(lane_base + b * kNT, reinterpret_cast<uint32_t*>(sc));
        tmem_ld32(lane_base + b * kNT + 32, reinterpret_cast<uint32_t*>(sc + 32));
      } else {
        tmem_ld32(lane_base + b * kNT + 32 * half, reinterpret_cast<uint32_t*>(sc));
      }
      tmem_ld_wait();
      fence_before();
      mbar_arrive(&tempty[b]);
      const int stg = i % kStages;
      const float* rowsm = reinterpret_cast<const float*>(Bs + stg * kStage + kBTile);
      if (!mine) {
        mbar_arrive(&empty[stg]);
        continue;
      }
      const int e_lo = w.t0 - tb, e_hi = w.t1 - tb;  // columns of this chunk: [e_lo, e_hi)
      if (!exact) {
#pragma unroll
        for (int e2 = 0; e2 < 32; ++e2) {
          const int e = 32 * half + e2;
          float x = (e >= e_lo && e < e_hi) ? sc[e2] : -INFINITY;
          if (x > top[M - 1]) {  // sorted insert, register bubble
#pragma unroll
            for (int j = 0; j < M; ++j) {
              const float hv = fmaxf(top[j], x);
              x = fminf(top[j], x);
              top[j] = hv;
            }
          }
        }
        mbar_arrive(&empty[stg]);
        continue;
      }
      // gate: the pass-2 bound, tightened by the k-th best exact score held
      // so far once the heap is full (a token beating it has approx >= it - eps)
      float gate = thr;
      if (hn == k) gate = fmaxf(gate, (float)key_score(root) - 2.0f * kGateEps - 1e-6f);
      uint64_t pass_mask = 0ull;  // gate survivors of this tile
#pragma unroll
      for (int e = 0; e < kNT; ++e)
        if (e >= e_lo && e < e_hi && sc[e] >= gate) pass_mask |= 1ull << e;
      while (pass_mask) {
        const int e = __ffsll((long long)pass_mask) - 1;
        pass_mask &= pass_mask - 1;
        const int t = tb + e;
        // reference formula: f64 dot of the f32 unit vectors (nnsearch.py:344-347)
        const float4* row = reinterpret_cast<const float4*>(rowsm + e * kEmbed);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // independent chains
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 v = row[q4];
          a0 = fma((double)v.x, (double)uc[4 * q4], a0);
          a1 = fma((double)v.y, (double)uc[4 * q4 + 1], a1);
          a2 = fma((double)v.z, (double)uc[4 * q4 + 2], a2);
          a3 = fma((double)v.w, (double)uc[4 * q4 + 3], a3);
        }
        const double s = (a0 + a1) + (a2 + a3);
        const uint64_t key = score_key(s, t);
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
      mbar_arrive(&empty[stg]);
      if (tid == 0 && i < 32) DBG_STAMP(136 + i);
    }
    if (mine) {
      if (!exact) {
        float* dst = part1 + part_offset(tile, src, c, jchunk, 2 * M, tile_size) + half * M;
#pragma unroll
        for (int j = 0; j < M; ++j) dst[j] = top[j];
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
  if (tid == 0) DBG_STAMP(2);
  fence_before();
  __syncthreads();
  if (tid == 0) DBG_STAMP(3);
  if (warp == kMmaWarp) tmem_free<256>(T);
}

// T = k-th largest of the union of a (candidate, source)'s pass-1 lists
// (nw chunks x 2 halves x M floats): one warp, MSB-first radix select over
// order-preserving u32 images, 8-bit digits.
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u >> 31) ? (u & 0x7fffffffu) : ~u);
}

__global__ void __launch_bounds__(128) nn_bound_kernel(Staged st, NNCfg nn, const float* part1,
                                                       float* bound, int tile_size, int M) {
  __shared__ unsigned hist[4][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const NNTile tile = st.tiles[blockIdx.x];
  const int s = blockIdx.y;
  const int c = blockIdx.z * 4 + warp;
  if (c >= tile.n) return;
  const int nw = tile.nwork[s];
  if (nw <= 1) return;  // single exact chunk: no pass-1 bound
  const int k = nn.k[s];
  const int n = nw * 2 * M;  // <= 2 * kMergeCap / k * ... bounded by the planner (<= 512)
  const float* p = part1 + part_offset(tile, s, c, 0, 2 * M, tile_size);
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = 32 * i + lane < n ? f2ord(p[32 * i + lane]) : 0u;
  uint32_t prefix = 0u, pmask = 0u;
  int want = k;
  unsigned* h = hist[warp];
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) h[i] = 0u;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (32 * i + lane < n && (v[i] & pmask) == prefix) atomicAdd(&h[(v[i] >> shift) & 255], 1u);
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
    if (sel == 0u) {  // fewer than k values: no bound
      prefix = 0u;
      break;
    }
    const int srcl = __ffs(sel) - 1;
    int digit = 0, above = 0;
    if (lane == srcl) {
      unsigned run = excl;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (run + c8[j] >= (unsigned)want) {
          digit = 255 - 8 * lane - j;
          above = (int)run;
          break;
        }
        run += c8[j];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, srcl);
    above = __shfl_sync(0xffffffffu, above, srcl);
    want -= above;
    prefix |= (uint32_t)digit << shift;
    pmask |= 255u << shift;
    __syncwarp();
  }
  if (lane == 0) bound[(size_t)(tile.item0 + c) * 3 + s] = prefix ? ord2f(prefix) : -INFINITY;
}

cudaError_t launch_nn_bound(const Staged& st, const NNCfg& nn, const float* part1, float* bound,
                            int tile_size, cudaStream_t s) {
  if (st.n_tiles == 0) return cudaSuccess;
  dim3 grid(st.n_tiles, 3, (tile_size + 3) / 4);
  nn_bound_kernel<<<grid, 128, 0, s>>>(st, nn, part1, bound, tile_size, kTopM);
  return cudaGetLastError();
}

cudaError_t set_debug_timeline(long long* dev, int block) {
  cudaError_t e = cudaMemcpyToSymbol(g_dbg_block, &block, sizeof(block));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_dbg_timeline, &dev, sizeof(dev));
}

cudaError_t launch_nn_tc(const Staged& st, const NNCfg& nn, uint64_t* part, float* part1,
                         const float* bound, int kmax, int tile_size, int pass, cudaStream_t s) {
  if (st.n_work == 0) return cudaSuccess;
  // heap of cpb x kmax u64 per CTA (pass 2 / exact single chunks): split the
  // 128-candidate tile over 2 CTAs when kmax > 128 so that it fits
  const int halves = kmax > 128 ? 2 : 1;
  const size_t smem = 2 * kAHalf + kStages * kStage + (size_t)kmax * (tile_size / halves) * 8;
  auto kern = nn_tc_kernel<kTopM>;  // the planner sizes chunks for 2 x top-8 lists per chunk
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(st.n_work, halves);
  kern<<<grid, kTcThreads, smem, s>>>(st, nn, part, part1, bound, kmax, tile_size, pass);
  return cudaGetLastError();
}

}  // namespace tav2
