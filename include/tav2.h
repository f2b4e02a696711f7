/*
 * tav2.h -- C ABI of the B200-native TransAct V2 serving-time ranking path.
 *
 * The reference (seqrank 0.1.0, /root/reference/pkg/src/seqrank) is pure
 * Python/numpy and has no FFI; its boundary is the Python module API.  Each
 * entry point below replaces one reference function on the hot path (cited
 * file:line), takes plain pointers + sizes (no torch types), returns an int
 * status (TAV2_OK == 0) and reports details through tav2_last_error().
 * Device pointers are CUDA global-memory pointers; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Ownership mirrors the reference arena contract (serving/arena.py:16-55):
 * a tav2_ctx owns one pinned host staging arena and one device workspace,
 * both sized once at creation from tav2_capacity; nothing is allocated on
 * the hot path.  One ctx per worker thread (arena.py:17); params are
 * immutable after tav2_load_params.
 */
#ifndef TAV2_H_
#define TAV2_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TAV2_OK 0
#define TAV2_EINVAL 1   /* maps to seqrank.core.ValidationError (core.py:36) */
#define TAV2_ECUDA 2    /* CUDA runtime / launch failure -> RuntimeError     */
#define TAV2_ECAP 3     /* request exceeds the ctx capacity                  */
#define TAV2_ESTATE 4   /* call order violated (e.g. run before stage)       */

/* Precision modes of the scoring path (north_star: fp32 parity mode and the
 * bf16 headline mode). */
#define TAV2_MODE_FP32 0  /* logits within 1e-5: fp16x3 split GEMMs on tcgen05 (S <= 384) */
#define TAV2_MODE_BF16 1  /* logits within 2e-3 (observed ~4e-5): bf16x3 split GEMMs  */
/* Both modes select the NN index sets identically: fp16 tcgen05 threshold
 * scan + exact f64 re-scoring of the survivors (the reference's formula). */

/* ModelConfig (trainer.py:42-70) + NNConfig (nnsearch.py:25-46) as ints. */
typedef struct {
  int32_t embed_dim;    /* EncoderConfig.embed_dim   (must be 32)  */
  int32_t seq_len;      /* EncoderConfig.seq_len     (<= 384)      */
  int32_t ffn_dim;      /* EncoderConfig.ffn_dim     (must be 32)  */
  int32_t num_layers;   /* EncoderConfig.num_layers  (1..8)        */
  int32_t action_rows;  /* EncoderConfig.action_rows (<= 16)       */
  int32_t surface_rows; /* EncoderConfig.surface_rows (>= 4)       */
  int32_t ctx_dim;      /* ModelConfig.ctx_dim       (must be 8)   */
  int32_t hidden_dim;   /* ModelConfig.hidden_dim    (must be 64)  */
  int32_t recent;       /* NNConfig.recent        */
  int32_t k_lifelong;   /* NNConfig.k_lifelong    */
  int32_t k_realtime;   /* NNConfig.k_realtime    */
  int32_t k_impression; /* NNConfig.k_impression  */
} tav2_config;

/* Workspace sizing (the Arena capacity, arena.py:20). */
typedef struct {
  int32_t max_requests;   /* unique requests per staged batch          */
  int32_t max_items;      /* candidates per staged batch (all requests) */
  int64_t max_tokens;     /* LL+RT+IMP tokens per staged batch          */
} tav2_capacity;

/* One request, host side, caller-owned (build_dedup_batch input,
 * nnsearch.py:214-244; TokenBlock columns core.py:102-126).  Sources are
 * 0 = lifelong, 1 = realtime, 2 = impression, each newest-first. */
typedef struct {
  const int8_t* emb[3];       /* [len[s], 32] int8 quantized embeddings */
  const uint16_t* action[3];  /* [len[s]] action bitmasks               */
  const uint8_t* surface[3];  /* [len[s]] surface ids                   */
  int32_t len[3];
  const float* candidates;    /* [n_cand, 32] f32 candidate embeddings  */
  int32_t n_cand;
  const float* ctx;           /* [ctx_dim] request context (dataset.py:282-289) */
  /* from_store != 0: the user's sequences are read from the HBM-resident
   * store (tav2_store_put) under store_user; emb/action/surface/len are
   * ignored and only the candidates, ctx and plan cross PCIe. */
  int32_t from_store;
  uint64_t store_user;
} tav2_request;

typedef struct tav2_ctx tav2_ctx;

/* Create / destroy a worker context.  device = CUDA ordinal. */
int tav2_create(const tav2_config* cfg, const tav2_capacity* cap, int device, tav2_ctx** out);
int tav2_destroy(tav2_ctx* ctx);

/* RankingModel.load / EncoderParams.from_tensors (trainer.py:145-161,
 * encoder.py:122-137): named f32 host tensors using the reference
 * checkpoint names ("encoder.layer0.wq", "head.w1", ...).  Copies them to
 * device once and derives the split-precision weight images. */
int tav2_load_params(tav2_ctx* ctx, int n, const char* const* names, const float* const* data,
                     const int64_t* numel);

/* build_dedup_batch + Arena.take (nnsearch.py:214-244, arena.py:32-47):
 * packs the requests into the pinned arena and issues ONE host->device copy
 * on `stream`.  Writes the staged item count to *n_items. */
int tav2_stage(tav2_ctx* ctx, const tav2_request* reqs, int n_req, void* stream, int32_t* n_items);

/* fused_assemble (nnsearch.py:289-369) on the staged batch: per item and
 * NN segment the top-k token indices (stable ties -> lower index), laid out
 * in Eq. 2 order (nnsearch.py:153-180).  idx_dev: [n_items, seq_len] int32,
 * source-relative indices (RT-tail offset by `recent`), -1 on padding.
 * scores_dev (nullable): [n_items, seq_len] f64 score of each NN slot -- the
 * reference's float64 dot of the f32 unit vectors (nnsearch.py:344-347,
 * returned by fused_assemble(return_scores=True) at :362-363); 0 elsewhere. */
int tav2_nn_select(tav2_ctx* ctx, int mode, int32_t* idx_dev, double* scores_dev, void* stream);

/* similarity_scores (nnsearch.py:83-90) on the staged batch: the f64 score
 * of every token of `source` (0 = LL, 1 = RT, 2 = IMP; all tokens, RT from
 * index 0) of item `item`'s request against that item's candidate.
 * scores_dev: [len(source)] f64. */
int tav2_similarity(tav2_ctx* ctx, int32_t item, int32_t source, double* scores_dev, void* stream);

/* pool (encoder.py:265-273) over caller encoder outputs: u_dev [n, seq_len,
 * 64] f32, mask_dev [n, seq_len] u8 -> pooled_dev [n, 64] f32 (max over the
 * valid rows of U out_linear; zeros for an item with no valid row). */
int tav2_pool(tav2_ctx* ctx, const float* u_dev, const uint8_t* mask_dev, int32_t n, float* pooled_dev,
              void* stream);

/* encode_batch (encoder.py:161-188) from staged tokens + idx_dev:
 * features_dev [n_items, seq_len, 64] f32, mask_dev [n_items, seq_len] u8. */
int tav2_encode(tav2_ctx* ctx, const int32_t* idx_dev, float* features_dev, uint8_t* mask_dev,
                void* stream);

/* forward_fused (encoder.py:314-462) over caller features:
 * features_dev/u_dev [n, seq_len, 64] f32, mask_dev [n, seq_len] u8. */
int tav2_forward(tav2_ctx* ctx, int mode, const float* features_dev, const uint8_t* mask_dev,
                 int32_t n, float* u_dev, void* stream);

/* forward_fused(..., extra_mask) (encoder.py:314-462, :366-377): as
 * tav2_forward, with a custom attention mask ANDed into causal & key-valid
 * (NAL training masks; not on the serving path).  extra_dev [seq_len,
 * seq_len] u8 shared by the batch (extra_batched = 0) or [n, seq_len,
 * seq_len] (extra_batched = 1); a row with no allowed key gets a zero
 * attention output.  extra_dev == NULL is tav2_forward. */
int tav2_forward_masked(tav2_ctx* ctx, int mode, const float* features_dev, const uint8_t* mask_dev,
                        const uint8_t* extra_dev, int32_t extra_batched, int32_t n, float* u_dev, void* stream);

/* Fused K3+K4+K5 on the staged batch: gather + Eq. 4 encode + SKUT + pool +
 * CTR head (trainer.py:345-366).  logits_dev [n_items, 4] f32 (pre-sigmoid);
 * pooled_dev (nullable) [n_items, 64] f32. */
int tav2_score(tav2_ctx* ctx, int mode, const int32_t* idx_dev, float* logits_dev,
               float* pooled_dev, void* stream);

/* The spec'd rank() host to host: stage -> nn_select ->
 * score -> one device->host copy.  logits_host [sum n_cand, 4] f32;
 * idx_host (nullable) [sum n_cand, seq_len] int32 for NN-feature logging.
 * Synchronises `stream` before returning. */
int tav2_rank(tav2_ctx* ctx, const tav2_request* reqs, int n_req, int mode, float* logits_host,
              int32_t* idx_host, void* stream);

/* Pipelined rank (the serving loop): stage + nn_select + score + result
 * copies are enqueued without waiting, into one of TAV2_STAGE_SLOTS staging slots, so the
 * host packing and H2D copy of the next request overlap the kernels of the
 * current one.  Returns the slot in *slot_out; at most TAV2_STAGE_SLOTS submits may be in
 * flight: collect a slot before submitting into it again (submit blocks until
 * the slot's previous rank finished).  want_idx: also copy the NN indices
 * (NN-feature logging).  The chain runs on the slot's own internal compute
 * stream, ordered after the work already enqueued on `stream`; the two
 * slots' kernels may overlap on the device (slot-private workspaces). */
int tav2_rank_submit(tav2_ctx* ctx, const tav2_request* reqs, int n_req, int mode, int want_idx,
                     void* stream, int32_t* slot_out);

/* Number of staging slots (submits that may be in flight at once). */
#define TAV2_STAGE_SLOTS 4
int tav2_stage_slots(void);

/* Block until a submitted rank's kernels and result copies finished, without
 * touching the context's staging state: a completion thread may wait here
 * while another thread submits into the other slot (the caller guarantees
 * the slot is not resubmitted before it is collected). */
int tav2_rank_wait(tav2_ctx* ctx, int slot);

/* Wait for a submitted rank and copy its results out: logits_host
 * [n_items, 4] f32, idx_host (nullable, requires want_idx) [n_items, seq_len]. */
int tav2_rank_collect(tav2_ctx* ctx, int slot, float* logits_host, int32_t* idx_host);

/* Device-resident variant used by the throughput benchmark: nn_select +
 * score on the currently staged batch, no host traffic. */
int tav2_run_staged(tav2_ctx* ctx, int mode, float* logits_dev, void* stream);

/* Per-kernel device time, measured with CUDA events recorded on the launch
 * stream around every kernel of the path.  on=1 resets the accumulators. */
int tav2_set_profiling(tav2_ctx* ctx, int on);

/* Accumulated per-kernel times since profiling was enabled: fills up to
 * `max` entries (kernel name, total ms, launch count); returns the number of
 * kernels seen.  Synchronises the pending events. */
int tav2_kernel_times(tav2_ctx* ctx, const char** names, double* ms, int32_t* launches, int max);

/* Number of kernel launches the last tav2_run_staged / tav2_rank issued. */
int tav2_last_launch_count(const tav2_ctx* ctx);

/* HBM-resident feature store (FeatureStore, serving/store.py:25-72; the
 * .tav2 bulk load of dataset.py:91-131 feeds tav2_store_put).  One slot of
 * LIFELONG+REALTIME+IMPRESSION cap tokens per user (35 B/token: emb i8[32],
 * action u16, surface u8) in one device pool; a request with from_store set
 * is staged by device-to-device copies from its user's slot instead of
 * host->device copies of its tokens.  Writes replace a user wholesale and
 * are ordered with staging on the context's copy stream, so a staged batch
 * always sees one consistent snapshot of each user.
 *
 * tav2_store_reserve: (re)allocate the pool for max_users users (drops all
 * users).  tav2_store_put: insert or replace user_id from seqs' token
 * columns (seqs->len within the caps: the Python mirror truncates to the
 * newest tokens first, store.py:19-22); returns TAV2_ECAP when the pool is
 * full.  tav2_store_remove: TAV2_EINVAL if absent.  tav2_store_count: the
 * number of resident users (-1 on a null context). */
int tav2_store_reserve(tav2_ctx* ctx, int32_t max_users);
int tav2_store_put(tav2_ctx* ctx, uint64_t user_id, const tav2_request* seqs);
int tav2_store_remove(tav2_ctx* ctx, uint64_t user_id);
int tav2_store_count(const tav2_ctx* ctx);

/* Thread-local message for the last non-zero status. */
const char* tav2_last_error(void);

/* Library / kernel build identification (arch, version). */
const char* tav2_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TAV2_H_ */
