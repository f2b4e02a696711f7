// Shared device/host definitions for the tav2 kernels (sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/tav2.h"

namespace tav2 {

constexpr int kEmbed = 32;      // EMBED_DIM (core.py:10)
constexpr int kDModel = 64;     // 2 * embed (encoder.py:38)
constexpr int kFfn = 32;        // EncoderConfig.ffn_dim
constexpr int kCtx = 8;         // ModelConfig.ctx_dim
constexpr int kHidden = 64;     // ModelConfig.hidden_dim
constexpr int kHeads = 4;       // NUM_HEADS (dataset.py:36)
constexpr int kMaxSeq = 384;    // S = recent + k_ll + k_rt + k_imp
constexpr int kMaxLayers = 8;
constexpr int kMaxK = 256;      // per-segment k (SURVEY C5 sweep)
constexpr int kIdxBits = 14;    // LIFELONG_CAP = 16384 (core.py:31)
constexpr uint64_t kIdxMask = (1ull << kIdxBits) - 1;

// ---------------------------------------------------------------------------
// Per-batch staging plan.  The pinned host arena and the device staged
// region share this byte layout so staging is ONE contiguous H2D copy.
// ---------------------------------------------------------------------------
struct ReqInfo {          // one unique request (DedupBatch.users entry)
  int32_t tok_off[3];     // first token of LL / RT / IMP in the token arena
  int32_t len[3];         // source lengths
  int32_t item_off;       // first item (candidate) of this request
  int32_t n_items;
  int32_t glog[3];        // NN scan group size 2^glog per source (planner)
  int32_t pad_;
};

// Approximate-score gate margin of the threshold scan (nn_scan.cu): the
// scan scores fp16(unit(q)) . fp16(unit(c)) with f32 accumulation; fp16
// round-to-nearest has unit roundoff u = 2^-11, so for unit vectors
// |approx - exact| <= 2u + u^2 + 32 * 2^-24 (accumulation) < 9.8e-4.
constexpr float kGateEps = 1.1e-3f;
// The scan's token operand: 256-token tiles of the fp16 unit rows in the UMMA
// K-major no-swizzle layout, [4 chunks of 8 elements][256 rows][16 B].
constexpr int kScanTile = 256;
constexpr int kScanTileBytes = 4 * kScanTile * 16;
// Sources with at most kDirectMax selectable tokens skip the scan: nn_select
// scores all of them exactly (one staged batch per warp is cheaper than a
// scan CTA whose per-token group maxima and survivor lists cost more than the
// exact f64 dot products they prune).
constexpr int kDirectMax = 256;
// n_sel = selectable tokens of a source (RT: len - min(recent, len))
__host__ __device__ inline bool nn_scanned(int n_sel, int k) { return k > 0 && n_sel > k && n_sel > kDirectMax; }

struct NNWork {           // one (candidate tile, source, token chunk) unit
  int32_t tile;           // candidate tile id
  int32_t source;         // 0 = LL, 1 = RT tail (RT[r:]), 2 = IMP
  int32_t t0, t1;         // token range, source-relative (RT tail: RT index)
};

constexpr int kTile = 128;  // candidates per NN tile (tcgen05 M)
struct NNTile {           // up to kTile consecutive items of one request
  int32_t req;
  int32_t item0;
  int32_t n;
  int32_t work0[3];       // first work unit of each source for this tile
  int32_t nwork[3];       // number of chunks per source
};

// Device buffers of the threshold-scan NN (nn_scan.cu / nn_select.cu).
struct NNScan {
  float* gmax;            // [items][3][gcap] pass-1 group maxima
  float* bound;           // [items][3] k-th largest group maximum
  unsigned* count;        // [items][3] pass-2 survivor counts
  uint16_t* surv;         // [items][surv_stride] survivor source indices, per-source sub-lists
  int gcap, surv_stride;
};

struct Plan {
  int32_t n_req, n_items, n_tok;
  int32_t n_tiles, n_work, tile_size, n_scopy;
  // byte offsets inside the staged region
  int64_t off_req, off_tiles, off_work, off_item_req, off_ctx, off_cand, off_scopy, off_action,
      off_surface, off_emb, bytes;
};

// One HBM-store user's token run copied into the staged token columns
// (store_gather_kernel): tokens [src, src + n) of the store pool -> [dst, dst + n).
struct StoreCopy {
  int64_t src, dst;
  int32_t n, pad_;
};

// Device view of the model parameters (all f32, reference names in
// comments; layouts exactly as the reference arrays, row-major [in, out]).
struct Params {
  int32_t num_layers, seq_len, action_rows, surface_rows;
  const float* action_table;    // encoder.action_table   [A, 64]
  const float* surface_table;   // encoder.surface_table  [256, 64] (rows 0..3 used)
  const float* position_table;  // encoder.position_table [S, 64]
  const float* out_linear;      // encoder.out_linear     [64, 64]
  const float* wq[kMaxLayers];  // encoder.layerI.wq      [64, 64]
  const float* wk[kMaxLayers];
  const float* wv[kMaxLayers];
  const float* wo[kMaxLayers];
  const float* w1[kMaxLayers];  // [64, 32]
  const float* w2[kMaxLayers];  // [32, 64]
  const float* ln1_scale[kMaxLayers];
  const float* ln1_shift[kMaxLayers];
  const float* ln2_scale[kMaxLayers];
  const float* ln2_shift[kMaxLayers];
  const float* head_w1;  // head.w1 [104, 64]
  const float* head_b1;  // head.b1 [64]
  const float* head_w2;  // head.w2 [64, 4]
  const float* head_b2;  // head.b2 [4]
};

// bf16x3 weight images for the tensor-core SKUT (built once at load time).
// Every matrix W [in, out] is stored as the UMMA B operand W^T [N=out][K=in],
// K-major, 16-byte chunk slabs: element (n, k) at (k/8)*(N*16) + n*16 +
// (k%8)*2, hi image followed by lo image (hi = bf16(w), lo = bf16(w - hi)).
struct SkutImages {
  const uint8_t* wa[kMaxLayers];  // layer L: [Wq|Wk|Wv]^T  N=192 K=64   48 KB
  const uint8_t* wb[kMaxLayers];  // layer L: Wo^T (16 KB) | W1^T (8 KB) | W2^T (8 KB)
  const uint8_t* wout;            // out_linear^T N=64 K=64 16 KB
};
constexpr int kImgWA = 2 * 192 * 64 * 2;  // 49152
constexpr int kImgWB = 2 * (64 * 64 + 32 * 64 + 64 * 32) * 2;  // 32768
constexpr int kImgWO = 2 * 64 * 64 * 2;   // 16384

// Images of the folded tensor-core SKUT (skut_tc3.cu), same slab layout:
// per layer [ [Wqk|Wvo]^T N=128 K=64 (32 KB) | W1^T (8 KB) | W2^T (8 KB) ],
// Wqk = Wq Wk^T log2(e)/8 and Wvo = Wv Wo in f64 before the split.
struct SkutImages3 {
  const uint8_t* w[kMaxLayers];
  const uint8_t* wout;
  const uint8_t* w2out;  // W2 of the last layer times W_out (f64 product): the fused final FFN / pool GEMM
};
constexpr int kImg3WA = 2 * 128 * 64 * 2;  // 32768
constexpr int kImg3WB = kImgWB - kImgWO;   // 16384 (W1 | W2)
constexpr int kImg3WO = kImgWO;
constexpr int kImg3W2O = 2 * 64 * 32 * 2;  // 8192 (W2 W_out, K = 32, N = 64)

struct NNCfg {
  int32_t recent, k[3];       // k[0] = k_ll, k[1] = k_rt, k[2] = k_imp
  int32_t seg_start[4];       // layout starts: NN_LL, RT_recent, NN_RT_tail, NN_IMP
  int32_t seq_len;
};

// Staged batch, device side.
struct Staged {
  const ReqInfo* req;
  const NNTile* tiles;
  const NNWork* work;
  const int32_t* item_req;
  const float* ctx;        // [R, 8]
  const float* cand;       // [N, 32]
  const uint16_t* action;  // [T]
  const uint8_t* surface;  // [T]
  const int8_t* emb;       // [T, 32]
  float* tok_unit;         // [T, 32] derived: unit(dequantize(q)) (core.py:77-79)
  uint32_t* tok_img;       // derived: fp16 unit rows, kScanTile-token tiles (prep_kernel)
  float* cand_unit;        // [N, 32] derived: l2_normalize_rows(cand)
  float* tok_feat;         // [T, 64] derived: [unit(q) | 0] + action rows + surface row (Eq. 4 token part)
  int n_req, n_items, n_tok, n_tiles, n_work;
};

// ---------------------------------------------------------------------------
// Top-k keys: larger key == better.  High bits: order-preserving image of
// the f64 score truncated to 50 bits; low 14 bits: (2^14-1 - idx) so that on
// equal scores the lower storage index wins (argsort stable, nnsearch.py:361).
// ---------------------------------------------------------------------------
__host__ __device__ inline uint64_t score_key(double s, int idx) {
  s = s + 0.0;  // -0.0 -> +0.0 so zero scores tie exactly like the reference
  uint64_t u;
#ifdef __CUDA_ARCH__
  u = (uint64_t)__double_as_longlong(s);
#else
  memcpy(&u, &s, 8);
#endif
  u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  return (u & ~kIdxMask) | (kIdxMask - (uint64_t)idx);
}
__host__ __device__ inline int key_index(uint64_t key) { return (int)(kIdxMask - (key & kIdxMask)); }
__host__ __device__ inline double key_score(uint64_t key) {
  uint64_t u = key & ~kIdxMask;
  u = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  double s;
#ifdef __CUDA_ARCH__
  s = __longlong_as_double((long long)u);
#else
  memcpy(&s, &u, 8);
#endif
  return s;
}

}  // namespace tav2

// ---------------------------------------------------------------------------
// Programmatic dependent launch: every kernel of the path is launched with
// programmatic stream serialization, lets its dependents launch as soon as
// all of its CTAs started (griddep_launch) and runs its input-independent
// prologue (barrier init, TMEM alloc, plan / weight loads) before
// griddep_wait(), which returns once the preceding kernel completed and its
// writes are visible.  Outside a PDL chain both are no-ops.
// ---------------------------------------------------------------------------
namespace tav2 {
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Per-(candidate, source) completion flags of nn_select for the first
// candidate of every SKUT CTA (items < n_first = the SKUT grid size): a SKUT
// CTA starts its first candidate as soon as that candidate's three
// selections are written instead of waiting for the whole select grid, so
// the select kernel's tail overlaps the transformer; before its second
// candidate's idx reads it executes griddep_wait (by then select is
// normally long complete).  done[3 item + s] = epoch (a per-context counter,
// never 0, bumped per fused run) is stored with release semantics after the
// warp's idx writes; the reader spins with ld.acquire.  done == null:
// griddep_wait up front as for every other kernel.
struct SelFlags {
  uint32_t* done;
  const uint32_t* epoch;  // device word: the current run's epoch (prep_kernel bumps it)
  int n_first;
  // device word after the epoch: the SKUT's item counter from its third
  // round on (prep_kernel zeroes it; null -> static round-robin items)
  uint32_t* next_item = nullptr;
};
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) and the SM count cost a
// host round trip each; every launcher calls these instead (cached per
// kernel and device, defined in tav2_api.cu)
cudaError_t set_max_dyn_smem(const void* kern, int bytes);
int device_sms();
bool pdl_enabled();  // TAV2_NO_PDL=1 disables programmatic dependent launch (A/B timing)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace tav2

// Host-side launchers (defined in the kernel translation units).
namespace tav2 {
cudaError_t launch_prep(const Staged& st, const Params* p, cudaStream_t s, uint32_t* epoch_bump = nullptr);
bool skut_tc3_supported(const NNCfg& nn, const Params& p);
cudaError_t launch_skut_tc3(const Params& p, const SkutImages3& img, const NNCfg& nn, const Staged& st,
                            const int32_t* idx, int n, float* logits, float* pooled, SelFlags sel, bool f16,
                            cudaStream_t s);
bool skut_tc4_supported(const NNCfg& nn, const Params& p);
cudaError_t launch_skut_tc4(const Params& p, const SkutImages3& img, const NNCfg& nn, const Staged& st,
                            const int32_t* idx, int n, float* logits, float* pooled, bool f16, cudaStream_t s);
cudaError_t launch_nn_scan(const Staged& st, const NNCfg& nn, const NNScan& sc, int pass,
                           cudaStream_t s);
cudaError_t launch_nn_bound(const Staged& st, const NNCfg& nn, const NNScan& sc, cudaStream_t s);
cudaError_t launch_store_gather(const StoreCopy* d, int n, int max_tok, const int8_t* semb,
                                const uint16_t* sact, const uint8_t* ssurf, int8_t* demb, uint16_t* dact,
                                uint8_t* dsurf, cudaStream_t s);
cudaError_t launch_nn_select(const Staged& st, const NNCfg& nn, const NNScan& sc, int32_t* idx,
                             double* scores, SelFlags sel, cudaStream_t s);
cudaError_t set_debug_timeline(long long* dev, int block);
cudaError_t set_debug_skut(long long* dev);
cudaError_t set_debug_skut3(long long* dev);
cudaError_t set_dbg_cta_prep(long long* dev);
cudaError_t set_dbg_cta_scan(long long* dev);
cudaError_t set_dbg_cta_select(long long* dev);
cudaError_t set_dbg_cta_skut(long long* dev);
cudaError_t set_dbg_cta_skut3(long long* dev);
bool make_rows32_map(CUtensorMap* map, const void* base, int64_t rows, int box_rows);
cudaError_t launch_encode(const Staged& st, const NNCfg& nn, const Params& p, const int32_t* idx,
                          float* F, uint8_t* mask, cudaStream_t s);
cudaError_t launch_skut_simt(const Params& p, const NNCfg& nn, const Staged* st,
                             const int32_t* idx, const float* F, const uint8_t* fmask, int n,
                             float* scratch, float* U, float* logits, float* pooled, int cs_shift,
                             cudaStream_t s, const uint8_t* extra = nullptr, long long extra_stride = 0);
cudaError_t launch_skut_tc(const Params& p, const SkutImages& img, const NNCfg& nn,
                           const Staged* st, const int32_t* idx, const float* F,
                           const uint8_t* fmask, int n, float* U, float* logits, float* pooled,
                           cudaStream_t s);
cudaError_t launch_similarity(const Staged& st, int item, int source, int n, double* out, cudaStream_t s);
cudaError_t launch_head(const Params& p, const Staged& st, float* pooled, int n, float* logits, bool spin,
                        cudaStream_t s);
constexpr uint32_t kPooledEmpty = 0xffffffffu;  // a NaN no arithmetic produces: "not written yet"
cudaError_t launch_pool(const float* U, const uint8_t* mask, const float* out_linear, int n, int S, float* pooled,
                        cudaStream_t s);
int skut_simt_grid(int n);
size_t skut_simt_scratch_floats(int seq_len);
}  // namespace tav2
