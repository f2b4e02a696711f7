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
//      exact key (reference f64 score | inverted index; lanes score
//      survivors in parallel, two token rows in flight per lane) and the
//      keys are sorted descending: the first k win.  n <= 256 (the normal
//      case: about k + a few survivors) sorts in registers with a shuffle
//      bitonic network (NP/32 keys per lane); larger n -- degenerate sources
//      with massive ties, e.g. a zero candidate -- uses a shared-memory radix
//      select (keys cached up to kSelCap, recomputed per pass beyond);
//   3. the winners are re-keyed (index | f32 score) and sorted by descending
//      storage index the same way.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dbg.cuh"
#include "tav2_common.cuh"

namespace tav2 {

constexpr int kSelWarps = 4;
constexpr int kSelCap = 1024;  // shared-memory key cache per warp (8 KB)

// Bitonic sort, descending, of NP keys held as v[j] = element j*32 + lane.
template <int NP>
__device__ __forceinline__ void warp_sort_desc(uint64_t* v, int lane) {
  constexpr int R = NP / 32;
#pragma unroll
  for (int size = 2; size <= NP; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {  // partner in the same lane: register j ^ (stride / 32)
        const int rs = stride / 32;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j & rs) continue;
          const int e = j * 32 + lane;
          const bool desc = (e & size) == 0;
          const uint64_t a = v[j], b = v[j | rs];
          const bool sw = desc ? a < b : a > b;
          v[j] = sw ? b : a;
          v[j | rs] = sw ? a : b;
        }
      } else {  // partner lane ^ stride, same register
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int e = j * 32 + lane;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[j], stride);
          const bool desc = (e & size) == 0;
          const bool lower = (lane & stride) == 0;  // element e < partner
          const bool take_max = desc == lower;
          v[j] = take_max ? (v[j] > o ? v[j] : o) : (v[j] < o ? v[j] : o);
        }
      }
    }
  }
}

// (index + 1 | f32 score): sorts by storage index, never 0 (0 pads)
__device__ __forceinline__ uint64_t winner_key(uint64_t key) {
  return ((uint64_t)(key_index(key) + 1) << 32) | (uint64_t)__float_as_uint((float)key_score(key));
}

// reference score: f64 dot of the f32 unit vectors (nnsearch.py:344-347);
// four independent chains in a fixed order, so equal rows score equal
__device__ __forceinline__ double dot_exact(const float4* r, const double* uc) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    a0 = fma((double)r[q4].x, uc[4 * q4], a0);
    a1 = fma((double)r[q4].y, uc[4 * q4 + 1], a1);
    a2 = fma((double)r[q4].z, uc[4 * q4 + 2], a2);
    a3 = fma((double)r[q4].w, uc[4 * q4 + 3], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

struct KeySrc {  // survivors of one (candidate, source)
  const uint16_t* surv;
  const float* tok;  // the source's f32 unit rows
  double uc[kEmbed];
  __device__ __forceinline__ uint64_t key(int i) const {
    const int t = surv[i];
    float4 r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(tok + (size_t)t * kEmbed) + q);
    return score_key(dot_exact(r, uc), t);
  }
};

// Register path: n <= NP survivors; writes the k winners sorted by index.
template <int NP>
__device__ __forceinline__ void select_regs(const KeySrc& ks, int n, int k, int lane, int32_t* orow,
                                            float* srow) {
  constexpr int R = NP / 32;
  uint64_t v[R];
  int t[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int i = j * 32 + lane;
    t[j] = i < n ? (int)ks.surv[i] : -1;
  }
#pragma unroll
  for (int j = 0; j < R; j += 2) {  // two rows in flight per lane
    float4 r0[8], r1[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      r0[q] = t[j] >= 0 ? __ldg(reinterpret_cast<const float4*>(ks.tok + (size_t)t[j] * kEmbed) + q)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      if (j + 1 < R)
        r1[q] = t[j + 1] >= 0 ? __ldg(reinterpret_cast<const float4*>(ks.tok + (size_t)t[j + 1] * kEmbed) + q)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    v[j] = t[j] >= 0 ? score_key(dot_exact(r0, ks.uc), t[j]) : 0ull;  // real keys are > 0
    if (j + 1 < R) v[j + 1] = t[j + 1] >= 0 ? score_key(dot_exact(r1, ks.uc), t[j + 1]) : 0ull;
  }
  warp_sort_desc<NP>(v, lane);
#pragma unroll
  for (int j = 0; j < R; ++j) v[j] = (j * 32 + lane < k && v[j]) ? winner_key(v[j]) : 0ull;
  warp_sort_desc<NP>(v, lane);
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int i = j * 32 + lane;
    if (i < k) {
      orow[i] = v[j] ? (int32_t)(v[j] >> 32) - 1 : -1;
      if (srow) srow[i] = v[j] ? __uint_as_float((uint32_t)v[j]) : 0.0f;
    }
  }
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

// Shared-memory path for n > 256: MSB-first radix select (8-bit digits,
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
  __shared__ uint64_t buf[kSelWarps][kSelCap];
  __shared__ unsigned hist_s[kSelWarps][256];
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
  const int np = max(n, k);
  if (np <= 32) select_regs<32>(ks, n, k, lane, orow, srow);
  else if (np <= 64) select_regs<64>(ks, n, k, lane, orow, srow);
  else if (np <= 128) select_regs<128>(ks, n, k, lane, orow, srow);
  else if (np <= 256) select_regs<256>(ks, n, k, lane, orow, srow);
  else select_radix(ks, n, k, lane, buf[warp], hist_s[warp], orow, srow);
}

cudaError_t set_dbg_cta_select(long long* dev) { return set_dbg_cta_tu(dev); }

cudaError_t launch_nn_select(const Staged& st, const NNCfg& nn, const NNScan& sc, int32_t* idx,
                             float* scores, cudaStream_t s) {
  if (st.n_items == 0) return cudaSuccess;
  dim3 grid((st.n_items + kSelWarps - 1) / kSelWarps, 3);
  return launch_pdl(nn_select_kernel, grid, dim3(32 * kSelWarps), 0, s, st, nn, sc, idx, scores);
}

}  // namespace tav2
