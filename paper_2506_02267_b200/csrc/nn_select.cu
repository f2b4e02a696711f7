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
//   2. otherwise every survivor of the threshold scan (nn_scan.cu) gets its
//      exact key (f64 score with the reference formula | inverted index):
//      lanes score survivors in parallel, keys cached in shared memory (or
//      recomputed per radix pass when a degenerate source -- all scores
//      tied, e.g. a zero candidate -- leaves more than kSelCap survivors);
//   3. MSB-first radix select (8-bit digits) isolates the top k; it stops as
//      soon as the bucket holding the k-th key is entirely selected;
//   4. the winners are sorted by descending storage index (bitonic).
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"

namespace tav2 {

constexpr int kSelWarps = 4;
constexpr int kSelCap = 1024;  // cached survivor keys per warp (8 KB)

__device__ __forceinline__ void warp_bitonic_desc(uint64_t* a, int n, int lane) {
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

// reference score: f64 dot of the f32 unit vectors (nnsearch.py:344-347)
__device__ __forceinline__ double exact_score(const float* tok_unit_row, const double* uc) {
  const float4* row = reinterpret_cast<const float4*>(tok_unit_row);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int q4 = 0; q4 < 8; ++q4) {
    const float4 v = __ldg(row + q4);
    a0 = fma((double)v.x, uc[4 * q4], a0);
    a1 = fma((double)v.y, uc[4 * q4 + 1], a1);
    a2 = fma((double)v.z, uc[4 * q4 + 2], a2);
    a3 = fma((double)v.w, uc[4 * q4 + 3], a3);
  }
  return (a0 + a1) + (a2 + a3);
}

__global__ void __launch_bounds__(32 * kSelWarps) nn_select_kernel(Staged st, NNCfg nn, NNScan sc,
                                                                   int32_t* idx, float* scores) {
  __shared__ uint64_t buf[kSelWarps][kSelCap];
  __shared__ unsigned hist_s[kSelWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kSelWarps + warp;
  const int s = blockIdx.y;
  if (item >= st.n_items) return;  // warp-uniform
  const ReqInfo rq = st.req[st.item_req[item]];
  const int S = nn.seq_len;
  const int k = nn.k[s];
  uint64_t* a = buf[warp];

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
  const float* tok = st.tok_unit + (size_t)rq.tok_off[s] * kEmbed;
  double uc[kEmbed];
  {
    const float4* cu = reinterpret_cast<const float4*>(st.cand_unit + (size_t)item * kEmbed);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 v = __ldg(cu + j);
      uc[4 * j] = v.x; uc[4 * j + 1] = v.y; uc[4 * j + 2] = v.z; uc[4 * j + 3] = v.w;
    }
  }

  if (hi - lo <= k) {  // 1. everything selected, descending storage index
    for (int j = lane; j < k; j += 32) {
      const int t = hi - 1 - j;
      orow[j] = t >= lo ? t : -1;
      if (srow) srow[j] = t >= lo ? (float)exact_score(tok + (size_t)t * kEmbed, uc) : 0.0f;
    }
    return;
  }

  // 2. survivor keys
  const uint16_t* surv = sc.surv + (size_t)item * sc.surv_stride + (rq.tok_off[s] - rq.tok_off[0]);
  const int n = min((int)sc.count[(size_t)item * 3 + s], hi - lo);
  const bool cached = n <= kSelCap;
  auto key_of = [&](int i) -> uint64_t {
    const int t = surv[i];
    return score_key(exact_score(tok + (size_t)t * kEmbed, uc), t);
  };
  if (cached) {
    for (int i = lane; i < n; i += 32) a[i] = key_of(i);
    __syncwarp();
  }
  // 3. radix select: winners are the keys whose masked prefix >= `prefix`
  uint64_t prefix = 0ull, pmask = 0ull;
  if (n > k) {
    unsigned* hist = hist_s[warp];
    int want = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = lane; i < 256; i += 32) hist[i] = 0u;
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        const uint64_t v = cached ? a[i] : key_of(i);
        if ((v & pmask) == prefix) atomicAdd(&hist[(v >> shift) & 255], 1u);
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
  }
  // winners (exactly min(n, k): keys are unique), re-keyed (index << 32 | f32 score)
  __syncwarp();
  int v = 0;
  uint64_t* w = a;  // compacted in place (winner slot v <= source slot i)
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t x = i < n ? (cached ? a[i] : key_of(i)) : 0ull;
    const bool keep = i < n && (x & pmask) >= prefix;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep)
      w[v + __popc(m & ((1u << lane) - 1))] =
          ((uint64_t)key_index(x) << 32) | (uint64_t)__float_as_uint((float)key_score(x));
    v += __popc(m);
    __syncwarp();
  }
  // 4. sort by descending storage index
  int np2 = 32;
  while (np2 < v) np2 <<= 1;
  for (int i = v + lane; i < np2; i += 32) w[i] = 0ull;
  __syncwarp();
  warp_bitonic_desc(w, np2, lane);
  for (int j = lane; j < k; j += 32) {
    if (j < v) {
      const uint64_t e = w[j];
      orow[j] = (int32_t)(e >> 32);
      if (srow) srow[j] = __uint_as_float((uint32_t)e);
    } else {
      orow[j] = -1;
      if (srow) srow[j] = 0.0f;
    }
  }
}

cudaError_t launch_nn_select(const Staged& st, const NNCfg& nn, const NNScan& sc, int32_t* idx,
                             float* scores, cudaStream_t s) {
  if (st.n_items == 0) return cudaSuccess;
  dim3 grid((st.n_items + kSelWarps - 1) / kSelWarps, 3);
  nn_select_kernel<<<grid, 32 * kSelWarps, 0, s>>>(st, nn, sc, idx, scores);
  return cudaGetLastError();
}

}  // namespace tav2
