/*
 * tav2_internal.h -- diagnostics exported by libtav2.so that are not part of
 * the reference-facing interface (no reference equivalent).
 */
#ifndef TAV2_INTERNAL_H_
#define TAV2_INTERNAL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One 128 x N x K tcgen05 MMA through the operand layouts the kernels use
 * (which: 0 bf16 SS K-major, 1 bf16 A-in-TMEM, 2 bf16 B MN-major, 3 i8 with a
 * TMA-loaded B, 4 i8 manual B).  A: [128, K], B: [N, K] ([K, N] for case 2),
 * row-major device buffers; D: [128, N] f32 (s32 for i8).  Synchronous. */
int tav2_tc_selftest(int which, const void* A, const void* B, void* D, int N, int K, void* stream);

/* Debug (libtav2_debug.so only): device buffer (>= 704 int64) receiving
 * %globaltimer stamps of NN scan work unit `block`'s CTA (slots 0..319,
 * 520..583), the older SKUT kernels' stamps (320..511) and the per-segment
 * clock64 accounting of skut_tc3 CTA 0 (640..703).  NULL disables.  Not
 * thread-safe. */
int tav2_debug_timeline(long long* dev, int block);

/* Debug (libtav2_debug.so only): device buffer (>= 8 * 3 * 4096 int64)
 * receiving per-CTA %globaltimer stamps of every ranking-path kernel
 * ([kernel][start | end | inputs ready][CTA]; kernels: prep, nn_scan pass 1,
 * nn_bound, nn_scan pass 2, nn_select, skut) and, at kernel 6, per
 * (candidate, source) select time and survivor count.  NULL disables.  Not
 * thread-safe. */
int tav2_debug_cta(long long* dev);

/* CUDA-graph cache of the launch chain (run_chain): number of captured
 * graphs held and whether capture was abandoned (direct launches only). */
int tav2_graph_info(const void* ctx, int32_t* n_graphs, int32_t* broken);

#ifdef __cplusplus
}
#endif
#endif
