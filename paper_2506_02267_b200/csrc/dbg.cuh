// Debug: per-CTA %globaltimer stamps (start / end) of every kernel of the
// ranking path, for tools/cta_timeline.py.  Compiled in only for the debug
// library (-DTAV2_DEBUG, build.build(debug=True)): the production kernels
// carry no stamp code and no debug-pointer loads.  Each translation unit has its
// own copy of the pointer (no relocatable device code); tav2_debug_cta sets
// all of them.  Slot layout: [kernel id][start | end | inputs ready][4096 CTAs].
#pragma once

#include <cuda_runtime.h>

namespace tav2 {

enum DbgKernel { kDbgPrep = 0, kDbgScan1 = 1, kDbgBound = 2, kDbgScan2 = 3, kDbgSelect = 4, kDbgSkut = 5 };
constexpr int kDbgCtas = 4096;

static __device__ long long* g_dbg_cta = nullptr;

#ifdef TAV2_DEBUG
constexpr bool kDebug = true;
#else
constexpr bool kDebug = false;
#endif

__device__ __forceinline__ void cta_stamp(int kid, int which) {
  if constexpr (!kDebug) return;
  long long* d = g_dbg_cta;
  if (d != nullptr && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    const int b = blockIdx.x + gridDim.x * blockIdx.y;
    if (b < kDbgCtas) d[(kid * 3 + which) * kDbgCtas + b] = t;
  }
}

// debug: a per-(candidate, source) record of the select kernel at kernel
// id 6: [6][0][item*3+s] = warp time (ns), [6][1][item*3+s] = survivors
__device__ __forceinline__ void sel_record(int slot, long long dur, long long n) {
  if constexpr (!kDebug) return;
  long long* d = g_dbg_cta;
  if (d != nullptr && slot < kDbgCtas) {
    d[(6 * 3 + 0) * kDbgCtas + slot] = dur;
    d[(6 * 3 + 1) * kDbgCtas + slot] = n;
  }
}
// select phase end times (relative to the warp's start): 0 keys staged and
// scored, 1 threshold found (record 7; the debug buffer holds 8 x 3 x 4096)
__device__ __forceinline__ void sel_record_phase(int slot, int phase, long long dur) {
  if constexpr (!kDebug) return;
  long long* d = g_dbg_cta;
  if (d != nullptr && slot < kDbgCtas) d[(phase == 0 ? 6 * 3 + 2 : 7 * 3 + phase - 1) * kDbgCtas + slot] = dur;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

static inline cudaError_t set_dbg_cta_tu(long long* dev) {
  return cudaMemcpyToSymbol(g_dbg_cta, &dev, sizeof(dev));
}

}  // namespace tav2
