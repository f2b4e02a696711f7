// Top-k merge: folds the per-chunk partial top-k lists of every (candidate,
// NN source) into the final selection and writes the Eq. 2 index layout.
//
// Reference: nnsearch.py:361 (stable top-k: larger score, then lower index),
// :364 (segment content in descending storage index), :153-180 (_layout),
// :144/:354 (verbatim recent real-time segment RT[:r], reversed).
//
// One warp per (candidate, source):
//   1. T0 = max over chunks of the chunk's heap root (its k-th best key when
//      its list is full, slot 0 = 0 otherwise).  The global k-th best is
//      >= T0, so keys < T0 cannot be selected.
//   2. survivors (key >= T0) are compacted into shared memory (ballot +
//      popc); at most nwork * k <= kMergeCap of them by construction of the
//      plan (tav2_stage caps chunks so that nwork * k <= kMergeCap).
//   3. the k-th largest survivor by an MSB-first radix select (8-bit digits,
//      warp-aggregated shared-memory histograms); winners = keys >= it.
//   4. bitonic sort of the winners by descending storage index.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"

namespace tav2 {

constexpr int kMergeWarps = 2;
constexpr int kMergeCap = 2048;  // survivors per warp (16 KB)

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

__global__ void __launch_bounds__(32 * kMergeWarps) nn_merge_kernel(Staged st, NNCfg nn,
                                                                    const uint64_t* part, int kmax,
                                                                    int tile_size, int32_t* idx,
                                                                    float* scores) {
  __shared__ uint64_t buf[kMergeWarps][kMergeCap];
  __shared__ unsigned hist_s[kMergeWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const NNTile tile = st.tiles[blockIdx.x];
  const int s = blockIdx.y;
  const int lc = blockIdx.z * kMergeWarps + warp;
  if (lc >= tile.n) return;  // warp-uniform
  const int item = tile.item0 + lc;
  const int S = nn.seq_len;
  const int k = nn.k[s];
  uint64_t* a = buf[warp];

  if (s == 1) {  // verbatim recent real-time segment RT[:r] reversed
    const int n_recent = min(nn.recent, st.req[tile.req].len[1]);
    for (int j = lane; j < nn.recent; j += 32) {
      idx[(size_t)item * S + nn.seg_start[1] + j] = j < n_recent ? n_recent - 1 - j : -1;
      if (scores) scores[(size_t)item * S + nn.seg_start[1] + j] = 0.0f;
    }
  }
  if (k == 0) return;
  const int seg = s == 0 ? 0 : (s == 1 ? 2 : 3);
  int32_t* orow = idx + (size_t)item * S + nn.seg_start[seg];
  float* srow = scores ? scores + (size_t)item * S + nn.seg_start[seg] : nullptr;
  const int nw = tile.nwork[s];
  const uint64_t* p = part + part_offset(tile, s, lc, 0, kmax, tile_size);

  // 1. pruning threshold from the chunk roots
  uint64_t t0 = 0ull;
  for (int j = lane; j < nw; j += 32) t0 = max(t0, p[(size_t)j * kmax]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t0 = max(t0, __shfl_xor_sync(0xffffffffu, t0, o));
  if (t0 == 0ull) t0 = 1ull;  // drop empty slots

  // 2. compact survivors
  int n = 0;
  for (int j = 0; j < nw; ++j) {
    const uint64_t* q = p + (size_t)j * kmax;
    for (int i0 = 0; i0 < k; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t v = i < k ? q[i] : 0ull;
      const bool keep = v >= t0;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) a[n + __popc(m & ((1u << lane) - 1))] = v;
      n += __popc(m);
    }
  }
  // 3. k-th largest survivor by MSB-first radix select (8-bit digits)
  __syncwarp();
  uint64_t kth = 1ull;  // n <= k: everything survives
  if (n > k) {
    unsigned* hist = hist_s[warp];
    uint64_t prefix = 0ull, pmask = 0ull;
    int want = k;  // rank (1-based, from the top) inside the current prefix
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = lane; i < 256; i += 32) hist[i] = 0u;
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        const uint64_t v = a[i];
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
      const unsigned excl = incl - tot;  // keys with a larger digit in lanes < l
      const bool here = excl < (unsigned)want && (unsigned)want <= incl;
      const unsigned sel = __ballot_sync(0xffffffffu, here);
      const int src = __ffs(sel) - 1;
      int digit = 0, above = 0;
      if (lane == src) {
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
      digit = __shfl_sync(0xffffffffu, digit, src);
      above = __shfl_sync(0xffffffffu, above, src);
      want -= above;
      prefix |= (uint64_t)digit << shift;
      pmask |= 255ull << shift;
      __syncwarp();
    }
    kth = prefix;
  }
  // winners = survivors >= kth (exactly min(n, k) of them: keys are unique)
  int v = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint64_t x = i < n ? a[i] : 0ull;
    const bool keep = i < n && x >= kth;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) a[v + __popc(m & ((1u << lane) - 1))] = x;  // in-place compaction (v <= i)
    v += __popc(m);
    __syncwarp();
  }
  // 4. winners re-keyed as (index << 32 | f32 score), sorted by index desc
  uint64_t* w = a;  // in place: every lane holds its winners in registers first
  int np3 = 32;
  while (np3 < v) np3 <<= 1;
  uint64_t mine[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = lane + 32 * r;
    mine[r] = 0ull;
    if (i < v) {
      const uint64_t key = a[i];
      mine[r] = ((uint64_t)key_index(key) << 32) | (uint64_t)__float_as_uint((float)key_score(key));
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = lane + 32 * r;
    if (i < np3) w[i] = mine[r];
  }
  __syncwarp();
  warp_bitonic_desc(w, np3, lane);
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

cudaError_t launch_nn_merge(const Staged& st, const NNCfg& nn, const uint64_t* part, int kmax,
                            int tile_size, int32_t* idx, float* scores, cudaStream_t s) {
  if (st.n_tiles == 0) return cudaSuccess;
  dim3 grid(st.n_tiles, 3, (tile_size + kMergeWarps - 1) / kMergeWarps);
  nn_merge_kernel<<<grid, 32 * kMergeWarps, 0, s>>>(st, nn, part, kmax, tile_size, idx, scores);
  return cudaGetLastError();
}

}  // namespace tav2
