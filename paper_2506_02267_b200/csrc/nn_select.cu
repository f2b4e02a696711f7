// Exact top-k selection over the NN scan survivors, written as the Eq. 2
// index layout.
//
// Reference: nnsearch.py:344-347 (f64 score of the f32 unit vectors), :361
// (stable top-k: larger score, then lower index), :364 (segment content in
// descending storage index), :153-180 (_layout), :144/:354 (the verbatim
// recent real-time segment RT[:r], reversed), :108 (k > n selects all).
//
// One warp per (candidate, source):
//   1. a source with n <= k tokens selects all of them (no scan ran);
//   2. otherwise every survivor of the scan's gate (nn_scan.cu) gets its
//      exact key (reference f64 score | inverted index); n <= 256 (the normal
//      case: about k + a few dozen survivors): the survivors' token rows are
//      staged in shared memory by cp.async (one memory round trip), scored by
//      the lanes in parallel, and every key ranked against all others (a
//      rolled broadcast loop); the k best win.  Larger n -- degenerate
//      sources with massive ties, e.g. a zero candidate -- uses a radix select
//      (keys recomputed per pass);
//   3. the winners are marked in a bitmap over source positions and emitted
//      in descending storage index (radix path: a shared bitonic sort).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dbg.cuh"
#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

constexpr int kSelWarps = 2;
constexpr int kSelCap = 256;    // shared-memory key array per warp (2 KB)
constexpr int kSelCache = 256;  // survivors sorted in registers
constexpr int kCaps0 = 16384;   // LIFELONG_CAP (core.py:31): source positions per bitmap

// (index + 1 | f32 score): sorts by storage index, never 0 (0 pads)
__device__ __forceinline__ uint64_t winner_key(uint64_t key) {
  return ((uint64_t)(key_index(key) + 1) << 32) | (uint64_t)__float_as_uint((float)key_score(key));
}

// reference score: f64 dot of the f32 unit vectors (nnsearch.py:344-347);
// four independent chains in a fixed order, so equal rows score equal
__device__ __forceinline__ double dot_exact(const float4* r, const float* uc) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    a0 = fma((double)r[q4].x, (double)uc[4 * q4], a0);
    a1 = fma((double)r[q4].y, (double)uc[4 * q4 + 1], a1);
    a2 = fma((double)r[q4].z, (double)uc[4 * q4 + 2], a2);
    a3 = fma((double)r[q4].w, (double)uc[4 * q4 + 3], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

struct KeySrc {  // survivors of one (candidate, source)
  const uint16_t* surv;
  const float* tok;  // the source's f32 unit rows
  float uc[kEmbed];
  __device__ __forceinline__ uint64_t key(int i) const {
    const int t = surv[i];
    float4 r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(tok + (size_t)t * kEmbed) + q);
    return score_key(dot_exact(r, uc), t);
  }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Keys of n <= kSelCache survivors into a[]: the warp stages kRowBatch token
// rows at a time in shared memory with cp.async (8 lanes x 16 B per row, all
// copies in flight at once; 16-byte chunk c of row r stored at chunk
// c ^ (r & 7) so the per-lane row reads below are bank-conflict free), then
// every lane scores its rows exactly.
constexpr int kRowBatch = 128;
__device__ __forceinline__ void keys_staged(const KeySrc& ks, int n, int lane, float4* rows, uint64_t* a) {
  for (int b0 = 0; b0 < n; b0 += kRowBatch) {
    const int nb = min(kRowBatch, n - b0);
    for (int rr = lane >> 3; rr < nb; rr += 4) {
      const int t = ks.surv[b0 + rr];
      const int c = lane & 7;
      cp_async16(rows + rr * 8 + (c ^ (rr & 7)), ks.tok + (size_t)t * kEmbed + 4 * c);
    }
    cp_async_wait_all();
    __syncwarp();
    for (int rr = lane; rr < nb; rr += 32) {
      float4 r[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) r[c] = rows[rr * 8 + (c ^ (rr & 7))];
      a[b0 + rr] = score_key(dot_exact(r, ks.uc), ks.surv[b0 + rr]);
    }
    __syncwarp();
  }
}

// Emit the winners marked in a per-warp bitmap over source positions in
// descending storage index (the segment order, nnsearch.py:364): lane l
// scans words [W - per(l+1), W - per l), high first; a warp prefix sum of the
// per-lane counts places its bits.
__device__ __forceinline__ void emit_bitmap(const uint32_t* bm, int words, int k, int lane, int32_t* orow,
                                            float* srow, const KeySrc& ks) {
  const int per = (words + 31) / 32;
  const int w_hi = words - per * lane;  // this lane's words: [w_hi - per, w_hi)
  int cnt = 0;
  for (int w = w_hi - 1; w >= max(w_hi - per, 0); --w) cnt += __popc(bm[w]);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int pos = incl - cnt;
  for (int w = w_hi - 1; w >= max(w_hi - per, 0); --w) {
    uint32_t m = bm[w];
    while (m) {
      const int b = 31 - __clz(m);
      m &= ~(1u << b);
      const int t = 32 * w + b;
      if (pos < k) {
        orow[pos] = t;
        if (srow) {
          float4 r[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(ks.tok + (size_t)t * kEmbed) + q);
          srow[pos] = (float)dot_exact(r, ks.uc);
        }
      }
      ++pos;
    }
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  for (int j = total + lane; j < k; j += 32) {
    orow[j] = -1;
    if (srow) srow[j] = 0.0f;
  }
}

// The k largest of n <= 32 R keys a[0..n) (shared) win: lane-owned key
// i = j*32 + lane has rank #{m : a[m] > key} (keys are unique), counted with a
// rolled loop of broadcast reads -- compact code (a fully unrolled sorting
// network runs once per SM and is bound by instruction fetch).
template <int R>
__device__ __forceinline__ void select_rank(const uint64_t* a, int n, int k, int lane, uint32_t* bm) {
  uint64_t v[R];
  int rank[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    v[j] = j * 32 + lane < n ? a[j * 32 + lane] : 0ull;
    rank[j] = 0;
  }
#pragma unroll 4
  for (int m = 0; m < n; ++m) {
    const uint64_t x = a[m];
#pragma unroll
    for (int j = 0; j < R; ++j) rank[j] += x > v[j] ? 1 : 0;
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (j * 32 + lane < n && rank[j] < k) {
      const int t = key_index(v[j]);
      atomicOr(bm + (t >> 5), 1u << (t & 31));
    }
  __syncwarp();
}

__device__ __forceinline__ void warp_bitonic_desc_smem(uint64_t* a, int n, int lane) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        const int lo = 2 * stride * (i / stride) + (i % stride);
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        uint64_t x = a[lo], y = a[hi];
        if ((x < y) == desc) {
          a[lo] = y;
          a[hi] = x;
        }
      }
      __syncwarp();
    }
  }
}

// Path for n > kSelCache: MSB-first radix select (8-bit digits,
// warp-aggregated histogram) isolates the top k, then a shared bitonic sort
// orders the winners by index.
__device__ __forceinline__ void select_radix(const KeySrc& ks, int n, int k, int lane, uint64_t* a,
                                             unsigned* hist, int32_t* orow, float* srow) {
  const bool cached = n <= kSelCap;
  if (cached) {
    for (int i = lane; i < n; i += 32) a[i] = ks.key(i);
    __syncwarp();
  }
  uint64_t prefix = 0ull, pmask = 0ull;
  int want = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t x = i < n ? (cached ? a[i] : ks.key(i)) : 0ull;
      const int dg = (i < n && (x & pmask) == prefix) ? (int)((x >> shift) & 255) : 256;
      const unsigned peers = __match_any_sync(0xffffffffu, dg);
      if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
    }
    __syncwarp();
    // lane l owns digits 255-8l .. 248-8l (descending); suffix sums from the top
    unsigned c8[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c8[j] = hist[255 - 8 * lane - j];
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
    prefix |= (uint64_t)digit << shift;
    pmask |= 255ull << shift;
    __syncwarp();
    if (inb == want) break;  // the k-th key's bucket is selected whole
  }
  // winners (exactly k: keys are unique), compacted in place (slot v <= i)
  int v = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t x = i < n ? (cached ? a[i] : ks.key(i)) : 0ull;
    const bool keep = i < n && (x & pmask) >= prefix;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) a[v + __popc(m & ((1u << lane) - 1))] = winner_key(x);
    v += __popc(m);
    __syncwarp();
  }
  int np2 = 32;
  while (np2 < v) np2 <<= 1;
  for (int i = v + lane; i < np2; i += 32) a[i] = 0ull;
  __syncwarp();
  warp_bitonic_desc_smem(a, np2, lane);
  for (int j = lane; j < k; j += 32) {
    const uint64_t e = j < v ? a[j] : 0ull;
    orow[j] = e ? (int32_t)(e >> 32) - 1 : -1;
    if (srow) srow[j] = e ? __uint_as_float((uint32_t)e) : 0.0f;
  }
}

__device__ __forceinline__ void nn_select_body(const Staged& st, const NNCfg& nn, const NNScan& sc,
                                               int32_t* idx, float* scores);

__global__ void __launch_bounds__(32 * kSelWarps) nn_select_kernel(Staged st, NNCfg nn, NNScan sc,
                                                                   int32_t* idx, float* scores) {
  nn_select_body(st, nn, sc, idx, scores);
  __syncthreads();
  cta_stamp(kDbgSelect, 1);
}

__device__ __forceinline__ void nn_select_body(const Staged& st, const NNCfg& nn, const NNScan& sc,
                                               int32_t* idx, float* scores) {
  __shared__ uint64_t buf[kSelWarps][kSelCap];  // radix path key cache; also the sort array
  __shared__ unsigned hist_s[kSelWarps][256];
  __shared__ float4 rows_s[kSelWarps][kRowBatch * 8];  // staged token rows (16 KB per warp)
  __shared__ uint32_t bm_s[kSelWarps][kCaps0 / 32];      // winner bitmap over source positions
  uint64_t (&keys_s)[kSelWarps][kSelCap] = buf;
  cta_stamp(kDbgSelect, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kSelWarps + warp;
  const int s = blockIdx.y;
  griddep_launch();
  griddep_wait();  // scan pass 2 complete
  cta_stamp(kDbgSelect, 2);
  if (item >= st.n_items) return;  // warp-uniform
  const ReqInfo& rq = st.req[st.item_req[item]];
  const int S = nn.seq_len;
  const int k = nn.k[s];

  if (s == 1) {  // verbatim recent real-time segment RT[:r] reversed
    const int n_recent = min(nn.recent, rq.len[1]);
    for (int j = lane; j < nn.recent; j += 32) {
      idx[(size_t)item * S + nn.seg_start[1] + j] = j < n_recent ? n_recent - 1 - j : -1;
      if (scores) scores[(size_t)item * S + nn.seg_start[1] + j] = 0.0f;
    }
  }
  if (k == 0) return;
  const int seg = s == 0 ? 0 : (s == 1 ? 2 : 3);
  int32_t* orow = idx + (size_t)item * S + nn.seg_start[seg];
  float* srow = scores ? scores + (size_t)item * S + nn.seg_start[seg] : nullptr;
  const int lo = s == 1 ? min(nn.recent, rq.len[1]) : 0, hi = rq.len[s];

  if (hi - lo <= k) {  // 1. everything selected, descending storage index
    const float* tok = st.tok_unit + (size_t)rq.tok_off[s] * kEmbed;
    const float* cu = st.cand_unit + (size_t)item * kEmbed;
    for (int j = lane; j < k; j += 32) {
      const int t = hi - 1 - j;
      orow[j] = t >= lo ? t : -1;
      if (srow) {  // reference score: f64 dot of the f32 unit vectors (nnsearch.py:344-347)
        double a = 0.0;
        if (t >= lo)
          for (int q = 0; q < kEmbed; ++q) a = fma((double)tok[(size_t)t * kEmbed + q], (double)cu[q], a);
        srow[j] = (float)a;
      }
    }
    return;
  }
  // 2./3. select over the survivors
  KeySrc ks;
  ks.surv = sc.surv + (size_t)item * sc.surv_stride + (rq.tok_off[s] - rq.tok_off[0]);
  ks.tok = st.tok_unit + (size_t)rq.tok_off[s] * kEmbed;
  {
    const float4* cu = reinterpret_cast<const float4*>(st.cand_unit + (size_t)item * kEmbed);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 q = __ldg(cu + j);
      ks.uc[4 * j] = q.x; ks.uc[4 * j + 1] = q.y; ks.uc[4 * j + 2] = q.z; ks.uc[4 * j + 3] = q.w;
    }
  }
  const int n = min((int)sc.count[(size_t)item * 3 + s], hi - lo);
  const long long t_start = kDebug ? gtimer() : 0;
  uint64_t* a = keys_s[warp];
  if (max(n, k) <= kSelCache) {
    uint32_t* bm = bm_s[warp];
    const int words = (hi + 31) >> 5;
    for (int w = lane; w < words; w += 32) bm[w] = 0u;
    keys_staged(ks, n, lane, rows_s[warp], a);
    const int np = max(n, k);
    if (np <= 64) select_rank<2>(a, n, k, lane, bm);
    else if (np <= 128) select_rank<4>(a, n, k, lane, bm);
    else select_rank<8>(a, n, k, lane, bm);
    emit_bitmap(bm, words, k, lane, orow, srow, ks);
  } else {
    select_radix(ks, n, k, lane, buf[warp], hist_s[warp], orow, srow);
  }
  if (kDebug && lane == 0) sel_record(item * 3 + s, gtimer() - t_start, n);
}

cudaError_t set_dbg_cta_select(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t launch_nn_select(const Staged& st, const NNCfg& nn, const NNScan& sc, int32_t* idx,
                             float* scores, cudaStream_t s) {
  if (st.n_items == 0) return cudaSuccess;
  dim3 grid((st.n_items + kSelWarps - 1) / kSelWarps, 3);
  return launch_pdl(nn_select_kernel, grid, dim3(32 * kSelWarps), 0, s, st, nn, sc, idx, scores);
}

}  // namespace tav2
