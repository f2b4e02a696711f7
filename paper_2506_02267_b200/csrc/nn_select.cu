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
//      exact key (sources too small to scan: select_direct) (reference f64 score | inverted index); n <= 256 (the normal
//      case: about k + a few dozen survivors): the survivors' token rows are
//      staged in shared memory by cp.async (one memory round trip), scored by
//      the lanes in parallel, and the k-th largest key found by bisection
//      (warp-wide counts); the k best win.  Larger n -- degenerate
//      sources with massive ties, e.g. a zero candidate -- uses a radix select
//      (keys recomputed per pass);
//   3. the winners are marked in a bitmap over source positions and emitted
//      in descending storage index (radix path: a shared bitonic sort).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "dbg.cuh"
#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

constexpr int kSelWarps = 2;
constexpr int kSelCap = 512;    // shared-memory key array per warp (4 KB)
constexpr int kSelCache = 512;  // survivors whose keys are staged (k_ll = 256: ~k + a few dozen)
constexpr int kCaps0 = 16384;   // LIFELONG_CAP (core.py:31): source positions per bitmap

// (index + 1 | f32 score): sorts by storage index, never 0 (0 pads)
__device__ __forceinline__ uint64_t winner_key(uint64_t key) {
  return ((uint64_t)(key_index(key) + 1) << 32) | (uint64_t)__float_as_uint((float)key_score(key));
}

// reference score: f64 dot of the f32 unit vectors (nnsearch.py:344-347);
// four independent chains in a fixed order, so equal rows score equal
// (both operands converted on the fly: a register-resident f64 copy of the
// candidate costs 64 registers, i.e. select-kernel occupancy)
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
  const uint16_t* surv;  // scan survivor list, or null: every token from `first` on
  int first;
  const float* tok;  // the source's f32 unit rows
  float uc[kEmbed];  // the candidate's unit row
  __device__ __forceinline__ int token(int i) const { return surv ? (int)surv[i] : first + i; }
  __device__ __forceinline__ uint64_t key(int i) const {
    const int t = token(i);
    float4 r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(tok + (size_t)t * kEmbed) + q);
    return score_key(dot_exact(r, uc), t);
  }
};

// .ca: cached in L1 -- every candidate of a request reads the same token rows
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Keys of n <= kSelCache survivors into a[]: the warp stages kRowBatch token
// rows at a time in shared memory with cp.async (8 lanes x 16 B per row, all
// copies in flight at once; 16-byte chunk c of row r stored at chunk
// c ^ (r & 7) so the per-lane row reads below are bank-conflict free), then
// every lane scores its rows exactly.
constexpr int kRowBatch = 64;
// The survivor indices are first copied to sidx (all loads in flight at
// once; fetching them inside the copy loop serialised one L2 round trip per
// row group).
__device__ __forceinline__ void keys_staged(const KeySrc& ks, int n, int lane, float4* rows, uint64_t* a,
                                            uint16_t* sidx) {
#pragma unroll
  for (int j = 0; j < kSelCache / 32; ++j) {
    const int i = j * 32 + lane;
    if (i < n) sidx[i] = (uint16_t)ks.token(i);
  }
  __syncwarp();
  // 32-row batches double-buffered in the two halves of `rows`: batch b + 1
  // is in flight (cp.async group) while batch b is scored, so the L2 round
  // trips overlap instead of one per 64-row batch
  constexpr int kHalf = kRowBatch / 2;
  auto issue = [&](int b) {
    const int b0 = b * kHalf, nb = min(kHalf, n - b0);
    float4* dst = rows + (b & 1) * kHalf * 8;
    for (int rr = lane >> 3; rr < nb; rr += 4) {
      const int t = sidx[b0 + rr];
      const int c = lane & 7;
      cp_async16(dst + rr * 8 + (c ^ (rr & 7)), ks.tok + (size_t)t * kEmbed + 4 * c);
    }
    cp_async_commit();
  };
  const int nbat = (n + kHalf - 1) / kHalf;
  if (nbat > 0) issue(0);
  for (int b = 0; b < nbat; ++b) {
    if (b + 1 < nbat) {
      issue(b + 1);
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncwarp();
    const int rr = lane, b0 = b * kHalf;
    if (b0 + rr < n) {
      const float4* src = rows + (b & 1) * kHalf * 8;
      float4 r[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) r[c] = src[rr * 8 + (c ^ (rr & 7))];
      a[b0 + rr] = score_key(dot_exact(r, ks.uc), sidx[b0 + rr]);
    }
    __syncwarp();  // this half is refilled by issue(b + 2)
  }
}

// Winner bitmap over source positions, per warp.  Logical word w (positions
// 32w..32w+31) of a `words`-word bitmap lives at bm_phys(w): emitting lane l
// owns logical words words-1-per*l-j (j = 0..per-1, descending) at physical
// j*32 + l, so its reads are bank-conflict free.  (per*32 words.)
// (per = words per lane, rounded up to a power of two: the mapping's
// division and modulo become a shift and a mask -- an integer division by a
// runtime divisor was ~20 instructions in every winner mark)
__device__ __forceinline__ int bm_per_log(int words) {
  const int per = (words + 31) >> 5;  // 1 .. 16
  return 32 - __clz(per - 1);          // ceil(log2(per)) (0 for per = 1)
}
__device__ __forceinline__ int bm_phys(int w, int words) {
  const int lg = bm_per_log(words);
  const int r = words - 1 - w;
  return (r & ((1 << lg) - 1)) * 32 + (r >> lg);
}
__device__ __forceinline__ void bm_mark(uint32_t* bm, int words, int t) {
  atomicOr(bm + bm_phys(t >> 5, words), 1u << (t & 31));
}
__device__ __forceinline__ void bm_clear(uint32_t* bm, int words, int lane) {
  for (int w = lane; w < (32 << bm_per_log(words)); w += 32) bm[w] = 0u;
}

// Emit the winners marked in the bitmap in descending storage index (the
// segment order, nnsearch.py:364): lane l scans its words high first; a warp
// prefix sum of the per-lane counts places its bits.
__device__ __forceinline__ void emit_bitmap(const uint32_t* bm, int words, int k, int lane, int32_t* orow,
                                            double* srow, const KeySrc& ks, int dbg_slot = -1, long long t0 = 0) {
  const int per = 1 << bm_per_log(words);  // <= 16 (kCaps0 positions), as bm_phys
  const int w_hi = words - per * lane;  // this lane's logical words: [w_hi - per, w_hi)
  int cnt = 0;
  uint32_t nz = 0u;  // this lane's nonzero words (bit j: logical word w_hi - 1 - j)
  for (int j = 0; j < per && w_hi - 1 - j >= 0; ++j) {
    const int c = __popc(bm[j * 32 + lane]);
    cnt += c;
    nz |= (c != 0 ? 1u : 0u) << j;
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int pos = incl - cnt;
  if (kDebug && dbg_slot >= 0 && lane == 0) sel_record_phase(dbg_slot, 2, gtimer() - t0);
  // only the nonzero words, descending storage index (j ascending, bits high
  // to low); the reference scores in a second, lane-parallel pass
  while (nz) {
    const int j = __ffs(nz) - 1;
    nz &= nz - 1;
    const int w = w_hi - 1 - j;
    uint32_t m = bm[j * 32 + lane];
    while (m) {
      const int b = 31 - __clz(m);
      m &= ~(1u << b);
      if (pos < k) orow[pos] = 32 * w + b;
      ++pos;
    }
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  for (int j = total + lane; j < k; j += 32) orow[j] = -1;
  if (srow) {  // the exact f64 key of every winner (nnsearch.py:362-363)
    __syncwarp();
    for (int j = lane; j < k; j += 32) {
      const int t = j < total ? orow[j] : -1;
      double v = 0.0;
      if (t >= 0) {
        float4 r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(ks.tok + (size_t)t * kEmbed) + q);
        v = dot_exact(r, ks.uc);
      }
      srow[j] = v;
    }
  }
}

// The k largest of n <= 32 R keys a[0..n) (shared) win: lane-owned key
// i = j*32 + lane has rank #{m : a[m] > key} (keys are unique), counted with a
// rolled loop of broadcast reads (cheapest for small n).
template <int R>
__device__ __forceinline__ void select_rank(const uint64_t* a, int n, int k, int lane, uint32_t* bm, int words) {
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
    if (j * 32 + lane < n && rank[j] < k) bm_mark(bm, words, key_index(v[j]));
  __syncwarp();
}

// The k largest of n <= 32 R keys a[0..n) (shared) win, found by bisection
// on the keys: T_hi = the largest t
// with #{hi32(key) >= t} >= k (32-bit halving, early exit when the count is
// exactly k), then, among the keys tied at hi32 == T_hi, the same search on
// the low 32 bits.  Winners = keys >= (T_hi, T_lo): exactly k (keys are
// unique).  ~3 R instructions per halving (<= 64 halvings, usually one
// 32-bit search ending early) instead of ranking every key against all n.
// (keys in registers: key j * 32 + lane in kv[j])
template <int R>
__device__ __forceinline__ void select_bisect_regs(const uint64_t* kv, int n, int k, int lane, uint32_t* bm,
                                                   int words) {
  if (n <= 0) return;  // (warp-uniform)
  uint32_t vh[R], vl[R];
  bool in[R];
  uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    in[j] = j * 32 + lane < n;
    const uint64_t x = in[j] ? kv[j] : 0ull;
    vh[j] = (uint32_t)(x >> 32);
    vl[j] = (uint32_t)x;
    if (in[j]) {
      mn = min(mn, vh[j]);
      mx = max(mx, vh[j]);
    }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  auto cnt_hi = [&](uint32_t t) {
    unsigned c = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) c += (in[j] && vh[j] >= t) ? 1u : 0u;
    return (int)__reduce_add_sync(0xffffffffu, c);
  };
  // count(>= lo) >= k > count(>= hi); hi = mx + 1 may wrap only if mx = ~0
  uint64_t lo = mn, hi = (uint64_t)mx + 1;
  int c_lo = n;
  while (hi - lo > 1) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    const int c = cnt_hi((uint32_t)mid);
    if (c >= k) {
      lo = mid;
      c_lo = c;
      if (c == k) break;
    } else {
      hi = mid;
    }
  }
  const uint32_t th = (uint32_t)lo;
  uint32_t tl = 0u;
  if (c_lo > k) {  // ties at hi32 == th: pick the k - above largest low halves
    const int above = lo == 0xffffffffull ? 0 : cnt_hi(th + 1);
    const int want = k - above;
    auto cnt_lo = [&](uint32_t t) {
      unsigned c = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) c += (in[j] && vh[j] == th && vl[j] >= t) ? 1u : 0u;
      return (int)__reduce_add_sync(0xffffffffu, c);
    };
    uint64_t l2 = 0, h2 = 0x100000000ull;
    while (h2 - l2 > 1) {
      const uint64_t mid = l2 + ((h2 - l2) >> 1);
      const int c = cnt_lo((uint32_t)mid);
      if (c >= want) {
        l2 = mid;
        if (c == want) break;
      } else {
        h2 = mid;
      }
    }
    tl = (uint32_t)l2;
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (in[j] && (vh[j] > th || (vh[j] == th && vl[j] >= tl)))
      bm_mark(bm, words, key_index(((uint64_t)vh[j] << 32) | vl[j]));
  __syncwarp();
}

template <int R>
__device__ __forceinline__ void select_bisect(const uint64_t* a, int n, int k, int lane, uint32_t* bm, int words) {
  uint64_t kv[R];
#pragma unroll
  for (int j = 0; j < R; ++j) kv[j] = j * 32 + lane < n ? a[j * 32 + lane] : 0ull;
  select_bisect_regs<R>(kv, n, k, lane, bm, words);
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

// The k largest of 256 < n <= kSelCap keys a[0..n) (shared; the k_ll = 256
// sweep point: about k + a few dozen survivors): MSB-first radix select on
// the cached keys (8-bit digits, warp-aggregated histogram; usually done
// after the first one or two digits), winners marked in the bitmap.
__device__ __forceinline__ void select_radix_cached(const uint64_t* a, int n, int k, int lane, unsigned* hist,
                                                    uint32_t* bm, int words) {
  uint64_t prefix = 0ull, pmask = 0ull;
  int want = k;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t x = i < n ? a[i] : 0ull;
      const int dg = (i < n && (x & pmask) == prefix) ? (int)((x >> shift) & 255) : 256;
      const unsigned peers = __match_any_sync(0xffffffffu, dg);
      if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
    }
    __syncwarp();
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
  // winners: exactly k keys (unique) have (key & pmask) >= prefix
  for (int i = lane; i < n; i += 32) {
    const uint64_t x = a[i];
    if ((x & pmask) >= prefix) bm_mark(bm, words, key_index(x));
  }
  __syncwarp();
}

// Path for n > kSelCache: MSB-first radix select (8-bit digits,
// warp-aggregated histogram) isolates the top k, then a shared bitonic sort
// orders the winners by index.
__device__ __forceinline__ void select_radix(const KeySrc& ks, int n, int k, int lane, uint64_t* a,
                                             unsigned* hist, int32_t* orow, double* srow) {
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
    if (srow) {  // the exact f64 key of the winner (its f32 image only sorts)
      double v = 0.0;
      if (e) {
        float4 r[8];
        const int t = (int)(e >> 32) - 1;
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(ks.tok + (size_t)t * kEmbed) + q);
        v = dot_exact(r, ks.uc);
      }
      srow[j] = v;
    }
  }
}

// Sources too small to scan (n <= kDirectMax selectable tokens: the RT tail
// and IMP at their 256-token caps, short LL histories), two-level, so FP64
// (DFMA issues at 1/8 the FFMA rate here) runs only where the order is in
// doubt:
//   1. approximate scores in f32 for every token (rows staged by cp.async;
//      two FFMA chains of 16 products: |approx - exact| <= gamma_17 <
//      1.02e-6 <= kDirEps / 2 for unit vectors) and a 256-bin histogram over
//      [-1, 1]; bin b holds the k-th largest approximation;
//   2. approx >= upper edge of b + 2 eps: certainly in the exact top k (fewer
//      than k tokens have approx >= that edge, and any token scoring higher
//      exactly is among them); approx < lower edge of b - 2 eps: certainly
//      out (k tokens have approx >= the lower edge, hence exact >= edge -
//      eps); the rest (the bin and its 2 eps margins, a handful) get the
//      exact f64 key and the best k - (certain winners) of them win.
constexpr float kDirEps = 2.5e-6f;
constexpr int kDirBins = 256;
__device__ __forceinline__ void select_direct(const KeySrc& ks, const float* ucf, int n, int k, int lane,
                                              float4* rows, unsigned* hist, uint64_t* a, uint32_t* bm, int words) {
  const int lo = ks.first;
#pragma unroll
  for (int b = 0; b < kDirBins / 32; ++b) hist[b * 32 + lane] = 0u;
  float ap[kDirectMax / 32];
  // 32-row batches double-buffered (as keys_staged): batch b + 1 in flight
  // while batch b is scored; fully unrolled so ap[] stays in registers
  constexpr int kHalf = kRowBatch / 2;
  auto issue = [&](int b) {
    const int b0 = b * kHalf, nb = min(kHalf, n - b0);
    float4* dst = rows + (b & 1) * kHalf * 8;
    for (int i = lane; i < nb * 8; i += 32) {
      const int rr = i >> 3, c = i & 7;
      cp_async16(dst + rr * 8 + (c ^ (rr & 7)), ks.tok + (size_t)(lo + b0 + rr) * kEmbed + 4 * c);
    }
    cp_async_commit();
  };
  const int nbat = (n + kHalf - 1) / kHalf;
  if (nbat > 0) issue(0);
#pragma unroll
  for (int b = 0; b < kDirectMax / 32; ++b) {
    float v = -INFINITY;
    if (b < nbat) {  // (warp-uniform)
      if (b + 1 < nbat) {
        issue(b + 1);
        cp_async_wait_group<1>();
      } else {
        cp_async_wait_group<0>();
      }
      __syncwarp();
      const int rr = lane;
      if (b * kHalf + rr < n) {
        const float4* src = rows + (b & 1) * kHalf * 8;
        float e0 = 0.f, e1 = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 x = src[rr * 8 + (q ^ (rr & 7))];
          float& e = (q & 1) ? e1 : e0;
          e = fmaf(x.x, ucf[4 * q], e);
          e = fmaf(x.y, ucf[4 * q + 1], e);
          e = fmaf(x.z, ucf[4 * q + 2], e);
          e = fmaf(x.w, ucf[4 * q + 3], e);
        }
        v = e0 + e1;
        atomicAdd(hist + min(max((int)((v + 1.0f) * (kDirBins / 2)), 0), kDirBins - 1), 1u);
      }
      __syncwarp();  // this half is refilled by issue(b + 2)
    }
    ap[b] = v;
  }
  __syncwarp();
  // bin of the k-th largest approximation: lane l owns bins 255 - 8l .. 248 - 8l
  unsigned h8[8], tot = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    h8[q] = hist[kDirBins - 1 - 8 * lane - q];
    tot += h8[q];
  }
  unsigned incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned sel = __ballot_sync(0xffffffffu, incl >= (unsigned)k && incl - tot < (unsigned)k);
  const int src = __ffs(sel) - 1;
  int kbin = 0;
  if (lane == src) {
    unsigned run = incl - tot;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      run += h8[q];
      if (run >= (unsigned)k) { kbin = kDirBins - 1 - 8 * lane - q; break; }
    }
  }
  kbin = __shfl_sync(0xffffffffu, kbin, src);
  const float win_t = (float)(kbin + 1) / (kDirBins / 2) - 1.0f + 2.0f * kDirEps;
  const float amb_t = (float)kbin / (kDirBins / 2) - 1.0f - 2.0f * kDirEps;
  int c_w = 0, m = 0;
#pragma unroll
  for (int jj = 0; jj < kDirectMax / 32; ++jj) {
    const int rr = jj * 32 + lane;
    const bool win = ap[jj] >= win_t;  // (-inf for rr >= n)
    const bool amb = !win && ap[jj] >= amb_t;
    if (win) bm_mark(bm, words, lo + rr);
    c_w += __popc(__ballot_sync(0xffffffffu, win));
    const unsigned ma = __ballot_sync(0xffffffffu, amb);
    if (amb) {
      float4 r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(ks.tok + (size_t)(lo + rr) * kEmbed) + q);
      a[m + __popc(ma & ((1u << lane) - 1))] = score_key(dot_exact(r, ks.uc), lo + rr);
    }
    m += __popc(ma);
  }
  __syncwarp();
  const int want = k - c_w;
  if (m <= 64) select_rank<2>(a, m, want, lane, bm, words);
  else if (m <= 128) select_bisect<4>(a, m, want, lane, bm, words);
  else select_bisect<8>(a, m, want, lane, bm, words);
}

__device__ __forceinline__ void nn_select_body(const Staged& st, const NNCfg& nn, const NNScan& sc,
                                               int32_t* idx, double* scores);

// CTA -> (candidate pair, source): source-major, the slowest source (0,
// long-lifelong) first, so the second wave (6 CTAs per SM at C2: 888 of
// 1,500 CTAs in the first) holds only short source-1/2 warps.  (A
// candidate-major order measured 1% slower; an order that also moves the
// source-1/2 warps of the SKUT CTAs' first candidates into the first wave
// measured neutral: the SKUT's claimed last rounds absorb its start skew.)
__device__ __forceinline__ int sel_item(int warp) { return blockIdx.x * kSelWarps + warp; }
__device__ __forceinline__ int sel_source() { return blockIdx.y; }

__global__ void __launch_bounds__(32 * kSelWarps) nn_select_kernel(Staged st, NNCfg nn, NNScan sc,
                                                                   int32_t* idx, double* scores, SelFlags sel) {
  nn_select_body(st, nn, sc, idx, scores);
  if (sel.done) {  // this (candidate, source)'s idx / scores rows are written (release)
    const int item = sel_item(threadIdx.x >> 5);
    if (item < st.n_items && item < sel.n_first) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        st_release_gpu(sel.done + 3 * item + sel_source(), ld_acquire_gpu(sel.epoch));
      }
    }
  }
  __syncthreads();
  cta_stamp(kDbgSelect, 1);
}

__device__ __forceinline__ void nn_select_body(const Staged& st, const NNCfg& nn, const NNScan& sc,
                                               int32_t* idx, double* scores) {
  __shared__ uint64_t buf[kSelWarps][kSelCap];  // radix path key cache; also the sort array
  __shared__ unsigned hist_s[kSelWarps][256];
  __shared__ float4 rows_s[kSelWarps][kRowBatch * 8];  // staged token rows (8 KB per warp)
  __shared__ uint32_t bm_s[kSelWarps][kCaps0 / 32];      // winner bitmap over source positions
  __shared__ uint16_t sidx_s[kSelWarps][kSelCache];     // survivor indices
  uint64_t (&keys_s)[kSelWarps][kSelCap] = buf;
  cta_stamp(kDbgSelect, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = sel_item(warp);
  const int s = sel_source();
  // the request's source offsets / lengths come from the staged plan (copied
  // before the chain started): read before the wait, their round trips overlap it
  int q_len1 = 0, q_lens = 0, q_off0 = 0, q_offs = 0;
  if (item < st.n_items) {
    const ReqInfo& rq0 = st.req[st.item_req[item]];
    q_len1 = rq0.len[1];
    q_lens = rq0.len[s];
    q_off0 = rq0.tok_off[0];
    q_offs = rq0.tok_off[s];
  }
  griddep_wait();  // scan pass 2 complete
  // dependents launch only now: with SelFlags the SKUT kernel skips its
  // up-front griddep_wait, so it must not start before prep .. scan2 are
  // complete (measured: no cost against triggering at CTA start)
  griddep_launch();
  cta_stamp(kDbgSelect, 2);
  if (item >= st.n_items) return;  // warp-uniform
  const int S = nn.seq_len;
  const int k = nn.k[s];

  if (s == 1) {  // verbatim recent real-time segment RT[:r] reversed
    const int n_recent = min(nn.recent, q_len1);
    for (int j = lane; j < nn.recent; j += 32) {
      idx[(size_t)item * S + nn.seg_start[1] + j] = j < n_recent ? n_recent - 1 - j : -1;
      if (scores) scores[(size_t)item * S + nn.seg_start[1] + j] = 0.0;
    }
  }
  if (k == 0) return;
  const int seg = s == 0 ? 0 : (s == 1 ? 2 : 3);
  int32_t* orow = idx + (size_t)item * S + nn.seg_start[seg];
  double* srow = scores ? scores + (size_t)item * S + nn.seg_start[seg] : nullptr;
  const int lo = s == 1 ? min(nn.recent, q_len1) : 0, hi = q_lens;

  if (hi - lo <= k) {  // 1. everything selected, descending storage index
    const float* tok = st.tok_unit + (size_t)q_offs * kEmbed;
    const float* cu = st.cand_unit + (size_t)item * kEmbed;
    for (int j = lane; j < k; j += 32) {
      const int t = hi - 1 - j;
      orow[j] = t >= lo ? t : -1;
      if (srow) {  // reference score: f64 dot of the f32 unit vectors (nnsearch.py:344-347)
        double a = 0.0;
        if (t >= lo) {
          float4 r[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(tok + (size_t)t * kEmbed) + q);
          a = dot_exact(r, cu);
        }
        srow[j] = a;
      }
    }
    return;
  }
  // 2./3. select over the survivors (all tokens of a source too small to scan)
  const bool scanned = nn_scanned(hi - lo, k);
  KeySrc ks;
  ks.surv = scanned ? sc.surv + (size_t)item * sc.surv_stride + (q_offs - q_off0) : nullptr;
  ks.first = lo;
  ks.tok = st.tok_unit + (size_t)q_offs * kEmbed;
  {
    const float4* cu = reinterpret_cast<const float4*>(st.cand_unit + (size_t)item * kEmbed);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 q = __ldg(cu + j);
      ks.uc[4 * j] = q.x; ks.uc[4 * j + 1] = q.y; ks.uc[4 * j + 2] = q.z; ks.uc[4 * j + 3] = q.w;
    }
  }
  const float* ucf = ks.uc;
  const int n = scanned ? min((int)sc.count[(size_t)item * 3 + s], hi - lo) : hi - lo;
  const long long t_start = kDebug ? gtimer() : 0;
  uint64_t* a = keys_s[warp];
  if (!scanned) {
    uint32_t* bm = bm_s[warp];
    const int words = (hi + 31) >> 5;
    bm_clear(bm, words, lane);
    __syncwarp();
    select_direct(ks, ucf, n, k, lane, rows_s[warp], hist_s[warp], a, bm, words);
    if (kDebug && lane == 0) sel_record_phase(item * 3 + s, 1, gtimer() - t_start);
    emit_bitmap(bm, words, k, lane, orow, srow, ks);
  } else if (max(n, k) <= kSelCache) {
    uint32_t* bm = bm_s[warp];
    const int words = (hi + 31) >> 5;
    bm_clear(bm, words, lane);
    keys_staged(ks, n, lane, rows_s[warp], a, sidx_s[warp]);
    if (kDebug && lane == 0) sel_record_phase(item * 3 + s, 0, gtimer() - t_start);
    const int np = max(n, k);
    if (np <= 64) select_rank<2>(a, n, k, lane, bm, words);
    else if (np <= 128) select_bisect<4>(a, n, k, lane, bm, words);
    else if (np <= 256) select_bisect<8>(a, n, k, lane, bm, words);
    else select_radix_cached(a, n, k, lane, hist_s[warp], bm, words);
    if (kDebug && lane == 0) sel_record_phase(item * 3 + s, 1, gtimer() - t_start);
    emit_bitmap(bm, words, k, lane, orow, srow, ks, kDebug ? item * 3 + s : -1, t_start);
  } else {
    select_radix(ks, n, k, lane, buf[warp], hist_s[warp], orow, srow);
  }
  if (kDebug && lane == 0) sel_record(item * 3 + s, gtimer() - t_start, n);
}

cudaError_t set_dbg_cta_select(long long* dev) { return set_dbg_cta_tu(dev); }

// similarity_scores (nnsearch.py:83-90): the f64 dot of every token of one
// source of a staged request with one staged candidate -- the f32 unit rows
// prep_kernel derived (core.py:54-79 op order), widened to f64 exactly as
// the reference's unit64 @ cand64 (nnsearch.py:344-347).  Thread per token.
__global__ void __launch_bounds__(256) similarity_kernel(Staged st, int item, int source, double* out) {
  griddep_wait();
  const ReqInfo& rq = st.req[st.item_req[item]];
  const int n = rq.len[source];
  const float* tok = st.tok_unit + (size_t)rq.tok_off[source] * kEmbed;
  float uc[kEmbed];
#pragma unroll
  for (int q = 0; q < kEmbed; ++q) uc[q] = st.cand_unit[(size_t)item * kEmbed + q];
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    float4 r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __ldg(reinterpret_cast<const float4*>(tok + (size_t)t * kEmbed) + q);
    out[t] = dot_exact(r, uc);
  }
}

cudaError_t launch_similarity(const Staged& st, int item, int source, int n, double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (n + 255) / 256;
  return launch_pdl(similarity_kernel, dim3(blocks < 148 ? blocks : 148), dim3(256), 0, s, st, item, source, out);
}

cudaError_t launch_nn_select(const Staged& st, const NNCfg& nn, const NNScan& sc, int32_t* idx,
                             double* scores, SelFlags sel, cudaStream_t s) {
  if (st.n_items == 0) return cudaSuccess;
  const dim3 grid((st.n_items + kSelWarps - 1) / kSelWarps, 3);
  return launch_pdl(nn_select_kernel, grid, dim3(32 * kSelWarps), 0, s, st, nn, sc, idx, scores, sel);
}

}  // namespace tav2
