// C ABI (include/tav2.h): worker context, pinned staging arena, parameter
// upload, batch planning and the launch sequence of the ranking path.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <string.h>

#include <string>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include <cuda_fp16.h>

#include "tav2_common.cuh"

using namespace tav2;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      return fail(TAV2_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                               \
  } while (0)


constexpr int kMinChunk = 256;    // minimum LL tokens per work unit
constexpr int kCaps[3] = {16384, 256, 256};  // LIFELONG/REALTIME/IMPRESSION_CAP (core.py:31-33)
constexpr int64_t kStoreSlotTok = 16384 + 256 + 256;

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }
inline int cdiv(int a, int b) { return (a + b - 1) / b; }

}  // namespace

cudaError_t tav2::set_max_dyn_smem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  int& v = done[{kern, dev}];
  if (v >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) v = bytes;
  return e;
}

int tav2::device_sms() {
  static std::mutex mu;
  static std::map<int, int> sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> g(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  sms[dev] = n;
  return n;
}

bool tav2::pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TAV2_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

// A/B switches read from the environment on every call (cheap; test-only)
static bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '1';
}

struct tav2_ctx {
  tav2_config cfg;
  tav2_capacity cap;
  int device = 0;
  NNCfg nn{};
  int kmax = 1;
  int max_tiles = 0, max_work = 0;
  int sms = 148;

  // Two staging slots (pinned host arena + device mirror of the staged
  // region each), so the host packing and H2D copy of the next batch overlap
  // the kernels of the current one (tav2_rank_submit).  H2D copies run on
  // copy_stream; ev_staged[s]: slot s's copy done (host arena reusable, the
  // compute stream may read it); ev_done[s]: the kernels (and result copies)
  // of slot s done (device region and pinned outputs reusable).
  static constexpr int kStageSlots = TAV2_STAGE_SLOTS;
  unsigned char* h_arena[kStageSlots] = {};
  unsigned char* d_staged[kStageSlots] = {};
  int64_t staged_cap = 0;
  cudaEvent_t ev_staged[kStageSlots] = {};
  cudaEvent_t ev_done[kStageSlots] = {};
  cudaStream_t copy_stream = nullptr;
  Plan plans[kStageSlots]{};
  int cur = 0;        // slot of the current staged batch
  int next_slot = 0;  // slot the next stage uses
  float* h_out[kStageSlots] = {};     // pinned logits of a submitted rank
  int32_t* h_idx[kStageSlots] = {};   // pinned NN indices (optional)
  int out_n[kStageSlots] = {};
  bool out_idx[kStageSlots] = {};
  // Derived device buffers, one set per staging slot: the launch chains of
  // two submitted requests (tav2_rank_submit, one compute stream per slot)
  // may then run concurrently -- request i+1's NN kernels on the SMs that
  // request i's SKUT tail frees.  A slot's buffers are reused only after
  // ev_done[slot] (tav2_stage orders the next use of the slot after it).
  struct Derived {
    float* tok_unit = nullptr;
    uint32_t* tok_img = nullptr;
    float* cand_unit = nullptr;
    float* tok_feat = nullptr;    // [T, 64] Eq. 4 token features (prep, bf16 SKUT gather)
    NNScan scan{};                // threshold-scan NN buffers (nn_scan.cu)
    uint32_t* sel_done = nullptr;   // per-(candidate, source) select flags (SelFlags)
    uint32_t* sel_epoch = nullptr;  // device word: the current run's flag epoch (prep bumps it)
    float* skut_scratch = nullptr;  // SIMT SKUT scratch
    float* pooled = nullptr;        // [N, 64] skut_tc3 pooled vectors -> head_kernel
  };
  Derived dv[kStageSlots];
  cudaStream_t slot_stream[kStageSlots] = {};  // tav2_rank_submit compute streams
  cudaEvent_t ev_caller[kStageSlots] = {};     // caller-stream order -> slot stream
  Derived& cur_dv() { return dv[cur]; }

  int32_t* idx = nullptr;
  float* logits = nullptr;
  // tav2_rank_submit: per-slot index / logit buffers, so the result copies
  // of one request (on d2h_stream, after ev_comp[slot]) overlap the next
  // request's kernels on the compute stream instead of sitting between them
  int32_t* idx_s[kStageSlots] = {};
  float* logits_s[kStageSlots] = {};
  cudaEvent_t ev_comp[kStageSlots] = {};
  cudaStream_t d2h_stream = nullptr;
  // CUDA graphs of the launch chain prep .. SKUT (run_chain): one per
  // (staging slot, mode, output buffer, batch plan), captured the second
  // time a shape is seen and replayed after; invalidated by tav2_load_params
  struct GraphEntry {
    int slot, mode;
    const float* logits;
    const int32_t* idx;
    Plan plan;
    cudaGraphExec_t exec;
    int launches;
    uint64_t last_use;
  };
  std::vector<GraphEntry> graphs;
  std::vector<std::pair<int, Plan>> graph_seen;  // shapes run once (candidates for capture)
  cudaStream_t cap_stream = nullptr;
  uint64_t graph_tick = 0;
  bool graph_broken = false;  // a capture failed: launch directly from then on
  // params
  float* d_params = nullptr;
  Params params{};
  uint8_t* d_images = nullptr;  // bf16x3 weight images (tensor-core SKUT)
  SkutImages images{};
  uint8_t* d_images3 = nullptr;  // folded images of skut_tc3 (Wqk, Wvo)
  SkutImages3 images3{};   // bf16x3 parts
  SkutImages3 images3h{};  // fp16x3 parts (fp32 mode)
  bool params_ok = false;
  // Cauchy-Schwarz softmax shift range (tensor-core SKUTs): exponents stay
  // >= -2 m' with m' <= cs_bound*; usable while 2 m' <= 120 (ex2 range)
  double cs_bound3 = 0.0, cs_bound = 0.0;
  // current batch: plans[cur]
  bool staged = false;
  int launches = 0;
  // per-kernel profiling (CUDA events on the launch stream)
  struct Slot {
    const char* name = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    bool pending = false;
    double ms = 0.0;
    int n = 0;
  };
  static constexpr int kSlots = 8;
  Slot slots[kSlots];
  bool profiling = false;
  // HBM-resident feature store (tav2_store_*): one slot of kStoreSlotTok
  // tokens per user, column pools [users][kStoreSlotTok][...]
  struct StoreEntry {
    int slot;
    int32_t len[3];
  };
  int8_t* st_emb = nullptr;
  uint16_t* st_act = nullptr;
  uint8_t* st_surf = nullptr;
  int st_users = 0;
  std::unordered_map<uint64_t, StoreEntry> st_map;
  std::vector<int> st_free;
};

namespace {

// largest singular value of a 64x64 row-major matrix (power iteration on MᵀM)
double spectral_norm64(const std::vector<double>& m) {
  std::vector<double> v(64, 1.0 / 8.0), u(64), w(64);
  double sig = 0.0;
  for (int it = 0; it < 200; ++it) {
    for (int i = 0; i < 64; ++i) {
      double a = 0.0;
      for (int j = 0; j < 64; ++j) a += m[i * 64 + j] * v[j];
      u[i] = a;
    }
    double nw = 0.0;
    for (int j = 0; j < 64; ++j) {
      double a = 0.0;
      for (int i = 0; i < 64; ++i) a += m[i * 64 + j] * u[i];
      w[j] = a;
      nw += a * a;
    }
    nw = std::sqrt(nw);
    if (nw == 0.0) return 0.0;
    for (int j = 0; j < 64; ++j) v[j] = w[j] / nw;
    sig = std::sqrt(nw);
  }
  return sig * 1.0001;  // power iteration approaches from below
}

Staged staged_view(tav2_ctx* c) {
  Staged s{};
  const Plan& p = c->plans[c->cur];
  unsigned char* b = c->d_staged[c->cur];
  s.req = reinterpret_cast<const ReqInfo*>(b + p.off_req);
  s.tiles = reinterpret_cast<const NNTile*>(b + p.off_tiles);
  s.work = reinterpret_cast<const NNWork*>(b + p.off_work);
  s.item_req = reinterpret_cast<const int32_t*>(b + p.off_item_req);
  s.ctx = reinterpret_cast<const float*>(b + p.off_ctx);
  s.cand = reinterpret_cast<const float*>(b + p.off_cand);
  s.action = reinterpret_cast<const uint16_t*>(b + p.off_action);
  s.surface = reinterpret_cast<const uint8_t*>(b + p.off_surface);
  s.emb = reinterpret_cast<const int8_t*>(b + p.off_emb);
  const tav2_ctx::Derived& d = c->dv[c->cur];
  s.tok_unit = d.tok_unit;
  s.tok_img = d.tok_img;
  s.cand_unit = d.cand_unit;
  s.tok_feat = d.tok_feat;
  s.n_req = p.n_req;
  s.n_items = p.n_items;
  s.n_tok = p.n_tok;
  s.n_tiles = p.n_tiles;
  s.n_work = p.n_work;
  return s;
}

int64_t staged_bytes(int R, int N, int64_t T, int tiles, int work) {
  int64_t o = 0;
  o = align256(o + (int64_t)R * sizeof(ReqInfo));
  o = align256(o + (int64_t)tiles * sizeof(NNTile));
  o = align256(o + (int64_t)work * sizeof(NNWork));
  o = align256(o + (int64_t)N * 4);
  o = align256(o + (int64_t)R * kCtx * 4);
  o = align256(o + (int64_t)N * kEmbed * 4);
  o = align256(o + T * 2);
  o = align256(o + T);
  o = align256(o + T * kEmbed);
  return o;
}

int free_all(tav2_ctx* c) {
  for (int k = 0; k < tav2_ctx::kStageSlots; ++k) {
    cudaFreeHost(c->h_arena[k]);
    cudaFree(c->d_staged[k]);
    cudaFreeHost(c->h_out[k]);
    cudaFreeHost(c->h_idx[k]);
    if (c->ev_staged[k]) cudaEventDestroy(c->ev_staged[k]);
    if (c->ev_done[k]) cudaEventDestroy(c->ev_done[k]);
    if (c->ev_comp[k]) cudaEventDestroy(c->ev_comp[k]);
    cudaFree(c->idx_s[k]);
    cudaFree(c->logits_s[k]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
  cudaFree(c->st_emb);
  cudaFree(c->st_act);
  cudaFree(c->st_surf);
  for (auto& d : c->dv) {
    cudaFree(d.tok_unit);
    cudaFree(d.tok_img);
    cudaFree(d.cand_unit);
    cudaFree(d.tok_feat);
    cudaFree(d.scan.gmax);
    cudaFree(d.scan.bound);
    cudaFree(d.scan.count);
    cudaFree(d.scan.surv);
    cudaFree(d.sel_done);
    cudaFree(d.sel_epoch);
    cudaFree(d.skut_scratch);
    cudaFree(d.pooled);
  }
  for (int k = 0; k < tav2_ctx::kStageSlots; ++k) {
    if (c->slot_stream[k]) cudaStreamDestroy(c->slot_stream[k]);
    if (c->ev_caller[k]) cudaEventDestroy(c->ev_caller[k]);
  }
  cudaFree(c->d_images3);
  cudaFree(c->idx);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  cudaFree(c->logits);
  cudaFree(c->d_params);
  cudaFree(c->d_images);
  for (auto& sl : c->slots) {
    if (sl.a) cudaEventDestroy(sl.a);
    if (sl.b) cudaEventDestroy(sl.b);
  }
  return 0;
}

void settle(tav2_ctx::Slot& sl) {
  if (!sl.pending) return;
  cudaEventSynchronize(sl.b);
  float t = 0.f;
  if (cudaEventElapsedTime(&t, sl.a, sl.b) == cudaSuccess) sl.ms += t;
  sl.n++;
  sl.pending = false;
}

// Launch `fn` (returning cudaError_t); when profiling, bracket it with events.
template <class F>
cudaError_t timed(tav2_ctx* c, const char* name, cudaStream_t s, F&& fn) {
  c->launches++;
  if (!c->profiling) return fn();
  tav2_ctx::Slot* sl = nullptr;
  for (auto& x : c->slots) {
    if (x.name == name || (x.name && strcmp(x.name, name) == 0)) { sl = &x; break; }
    if (!x.name) { x.name = name; sl = &x; break; }
  }
  if (!sl) return fn();
  if (!sl->a) {
    cudaEventCreate(&sl->a);
    cudaEventCreate(&sl->b);
  }
  settle(*sl);
  cudaEventRecord(sl->a, s);
  cudaError_t e = fn();
  cudaEventRecord(sl->b, s);
  sl->pending = true;
  return e;
}

}  // namespace

extern "C" {

const char* tav2_last_error(void) { return g_err.c_str(); }

const char* tav2_build_info(void) {
  return "tav2 0.1.0; kernels sm_100a (tcgen05/TMA) + SIMT fp32 parity mode; C ABI include/tav2.h";
}

int tav2_create(const tav2_config* cfg, const tav2_capacity* cap, int device, tav2_ctx** out) {
  if (!cfg || !cap || !out) return fail(TAV2_EINVAL, "null argument");
  *out = nullptr;
  const tav2_config& m = *cfg;
  if (m.embed_dim != kEmbed || m.ffn_dim != kFfn || m.ctx_dim != kCtx || m.hidden_dim != kHidden)
    return fail(TAV2_EINVAL,
                "unsupported model shape on the B200 path: embed_dim=%d ffn_dim=%d ctx_dim=%d "
                "hidden_dim=%d (need 32/32/8/64)",
                m.embed_dim, m.ffn_dim, m.ctx_dim, m.hidden_dim);
  if (m.num_layers < 1 || m.num_layers > kMaxLayers)
    return fail(TAV2_EINVAL, "num_layers %d outside [1, %d]", m.num_layers, kMaxLayers);
  if (m.action_rows < 1 || m.action_rows > 16 || m.surface_rows < 4)
    return fail(TAV2_EINVAL, "action_rows must be 1..16 and surface_rows >= 4");
  if (m.recent < 0 || m.k_lifelong < 0 || m.k_realtime < 0 || m.k_impression < 0)
    return fail(TAV2_EINVAL, "segment lengths must be non-negative");  // nnsearch.py:42-44
  int S = m.recent + m.k_lifelong + m.k_realtime + m.k_impression;
  if (S == 0) return fail(TAV2_EINVAL, "assembled sequence length must be positive");
  if (S != m.seq_len)
    return fail(TAV2_EINVAL, "encoder seq_len %d must equal the assembly length %d", m.seq_len, S);
  if (S > kMaxSeq) return fail(TAV2_EINVAL, "seq_len %d exceeds %d", S, kMaxSeq);
  if (m.k_lifelong > kMaxK || m.k_realtime > kMaxK || m.k_impression > kMaxK)
    return fail(TAV2_EINVAL, "per-segment k exceeds %d", kMaxK);
  if (cap->max_requests < 1 || cap->max_items < 1 || cap->max_tokens < 0)
    return fail(TAV2_EINVAL, "invalid capacity");

  tav2_ctx* c = new tav2_ctx();
  c->cfg = m;
  c->cap = *cap;
  c->device = device;
  c->nn.recent = m.recent;
  c->nn.k[0] = m.k_lifelong;
  c->nn.k[1] = m.k_realtime;
  c->nn.k[2] = m.k_impression;
  c->nn.seg_start[0] = 0;
  c->nn.seg_start[1] = m.k_lifelong;
  c->nn.seg_start[2] = m.k_lifelong + m.recent;
  c->nn.seg_start[3] = m.k_lifelong + m.recent + m.k_realtime;
  c->nn.seq_len = S;
  c->kmax = std::max(1, std::max(m.k_lifelong, std::max(m.k_realtime, m.k_impression)));
  const int R = cap->max_requests, N = cap->max_items;
  const int64_t T = cap->max_tokens;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (c->sms <= 0) c->sms = 148;
  c->max_tiles = R + cdiv(N, kTile);
  c->max_work = 3 * c->max_tiles + c->sms;
  c->staged_cap = staged_bytes(R, N, T, c->max_tiles, c->max_work);

  auto bad = [&](cudaError_t e, const char* what) {
    fail(TAV2_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    free_all(c);
    delete c;
    return TAV2_ECUDA;
  };
  cudaError_t e;
  if ((e = cudaSetDevice(device)) != cudaSuccess) return bad(e, "cudaSetDevice");
  for (int k = 0; k < tav2_ctx::kStageSlots; ++k) {
    if ((e = cudaMallocHost(&c->h_arena[k], c->staged_cap)) != cudaSuccess) return bad(e, "pinned arena");
    if ((e = cudaMalloc(&c->d_staged[k], c->staged_cap)) != cudaSuccess) return bad(e, "staged region");
    if ((e = cudaMallocHost(&c->h_out[k], (size_t)N * kHeads * 4)) != cudaSuccess) return bad(e, "pinned logits");
    if ((e = cudaMallocHost(&c->h_idx[k], (size_t)N * S * 4)) != cudaSuccess) return bad(e, "pinned indices");
    if ((e = cudaEventCreateWithFlags(&c->ev_staged[k], cudaEventDisableTiming)) != cudaSuccess) return bad(e, "event");
    if ((e = cudaEventCreateWithFlags(&c->ev_done[k], cudaEventDisableTiming)) != cudaSuccess) return bad(e, "event");
    if ((e = cudaEventCreateWithFlags(&c->ev_comp[k], cudaEventDisableTiming)) != cudaSuccess) return bad(e, "event");
  }
  if ((e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bad(e, "copy stream");

  for (int k = 0; k < tav2_ctx::kStageSlots; ++k) {
    tav2_ctx::Derived& d = c->dv[k];
    // padded to whole 64-token tiles (+1): the NN kernel bulk-copies full tiles
    if ((e = cudaMalloc(&d.tok_unit, (size_t)(cdiv((int)std::max<int64_t>(T, 1), 64) + 1) * 64 * kEmbed * 4)) !=
        cudaSuccess)
      return bad(e, "tok_unit");
    if ((e = cudaMalloc(&d.tok_img, (size_t)(cdiv((int)std::max<int64_t>(T, 1), kScanTile) + 1) * kScanTileBytes)) !=
        cudaSuccess)
      return bad(e, "token image");
    if ((e = cudaMalloc(&d.cand_unit, (size_t)N * kEmbed * 4)) != cudaSuccess) return bad(e, "cand_unit");
    if ((e = cudaMalloc(&d.tok_feat, (size_t)std::max<int64_t>(T, 1) * kDModel * 4)) != cudaSuccess)
      return bad(e, "token features");
    // scan buffers: a source has at most max(8k + 2, 16384/32 + 2) groups
    // (planner), a (candidate, source) at most its source length of survivors
    d.scan.gcap = (std::max(8 * c->kmax + 2, kCaps[0] / 32 + 2) + 8 + 7) & ~7;  // + 8: aligned rows
    d.scan.surv_stride =
        (int)((std::min<int64_t>(std::max<int64_t>(T, 8), kCaps[0] + kCaps[1] + kCaps[2]) + 7) & ~int64_t(7));
    if ((e = cudaMalloc(&d.scan.gmax, (size_t)N * 3 * d.scan.gcap * 4)) != cudaSuccess)
      return bad(e, "scan group maxima");
    if ((e = cudaMalloc(&d.scan.bound, (size_t)N * 3 * 4)) != cudaSuccess) return bad(e, "scan bounds");
    if ((e = cudaMalloc(&d.scan.count, (size_t)N * 3 * 4)) != cudaSuccess) return bad(e, "scan counts");
    if ((e = cudaMalloc(&d.scan.surv, (size_t)N * d.scan.surv_stride * 2)) != cudaSuccess)
      return bad(e, "scan survivors");
    if ((e = cudaMalloc(&d.sel_done, (size_t)N * 3 * 4)) != cudaSuccess) return bad(e, "select flags");
    if ((e = cudaMemset(d.sel_done, 0, (size_t)N * 3 * 4)) != cudaSuccess) return bad(e, "select flags");
    if ((e = cudaMalloc(&d.sel_epoch, 8)) != cudaSuccess) return bad(e, "select epoch");  // + SKUT item counter
    if ((e = cudaMemset(d.sel_epoch, 0, 8)) != cudaSuccess) return bad(e, "select epoch");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if ((e = cudaMalloc(&d.skut_scratch, (size_t)sms * skut_simt_scratch_floats(S) * 4)) != cudaSuccess)
      return bad(e, "skut scratch");
    if ((e = cudaMalloc(&d.pooled, (size_t)N * kDModel * 4)) != cudaSuccess) return bad(e, "pooled");
    // every entry kPooledEmpty between runs (head_kernel restores it)
    if ((e = cudaMemset(d.pooled, 0xff, (size_t)N * kDModel * 4)) != cudaSuccess) return bad(e, "pooled");
    if ((e = cudaStreamCreateWithFlags(&c->slot_stream[k], cudaStreamNonBlocking)) != cudaSuccess)
      return bad(e, "slot stream");
    if ((e = cudaEventCreateWithFlags(&c->ev_caller[k], cudaEventDisableTiming)) != cudaSuccess)
      return bad(e, "event");
  }
  if ((e = cudaMalloc(&c->idx, (size_t)N * S * 4)) != cudaSuccess) return bad(e, "idx");
  if ((e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bad(e, "capture stream");
  if ((e = cudaMalloc(&c->logits, (size_t)N * kHeads * 4)) != cudaSuccess) return bad(e, "logits");
  for (int k = 0; k < tav2_ctx::kStageSlots; ++k) {
    if ((e = cudaMalloc(&c->idx_s[k], (size_t)N * S * 4)) != cudaSuccess) return bad(e, "slot idx");
    if ((e = cudaMalloc(&c->logits_s[k], (size_t)N * kHeads * 4)) != cudaSuccess) return bad(e, "slot logits");
  }
  if ((e = cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return bad(e, "d2h stream");
  *out = c;
  return TAV2_OK;
}

int tav2_destroy(tav2_ctx* c) {
  if (!c) return TAV2_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  free_all(c);
  delete c;
  return TAV2_OK;
}

int tav2_load_params(tav2_ctx* c, int n, const char* const* names, const float* const* data,
                     const int64_t* numel) {
  if (!c || (n > 0 && (!names || !data || !numel))) return fail(TAV2_EINVAL, "null argument");
  const tav2_config& m = c->cfg;
  const int d = kDModel;
  struct Want {
    std::string name;
    int64_t numel;
    const float** slot;
  };
  Params P{};
  P.num_layers = m.num_layers;
  P.seq_len = m.seq_len;
  P.action_rows = m.action_rows;
  P.surface_rows = m.surface_rows;
  std::vector<Want> want = {
      {"encoder.action_table", (int64_t)m.action_rows * d, &P.action_table},
      {"encoder.surface_table", (int64_t)m.surface_rows * d, &P.surface_table},
      {"encoder.position_table", (int64_t)m.seq_len * d, &P.position_table},
      {"encoder.out_linear", (int64_t)d * d, &P.out_linear},
      {"head.w1", (int64_t)(d + kEmbed + kCtx) * kHidden, &P.head_w1},
      {"head.b1", kHidden, &P.head_b1},
      {"head.w2", (int64_t)kHidden * kHeads, &P.head_w2},
      {"head.b2", kHeads, &P.head_b2},
  };
  for (int L = 0; L < m.num_layers; ++L) {
    std::string p = "encoder.layer" + std::to_string(L) + ".";
    want.push_back({p + "wq", d * d, &P.wq[L]});
    want.push_back({p + "wk", d * d, &P.wk[L]});
    want.push_back({p + "wv", d * d, &P.wv[L]});
    want.push_back({p + "wo", d * d, &P.wo[L]});
    want.push_back({p + "w1", d * kFfn, &P.w1[L]});
    want.push_back({p + "w2", kFfn * d, &P.w2[L]});
    want.push_back({p + "ln1_scale", d, &P.ln1_scale[L]});
    want.push_back({p + "ln1_shift", d, &P.ln1_shift[L]});
    want.push_back({p + "ln2_scale", d, &P.ln2_scale[L]});
    want.push_back({p + "ln2_shift", d, &P.ln2_shift[L]});
  }
  int64_t total = 0;
  std::vector<int> src(want.size(), -1);
  std::vector<int64_t> off(want.size());
  for (size_t w = 0; w < want.size(); ++w) {
    for (int i = 0; i < n; ++i)
      if (names[i] && want[w].name == names[i]) src[w] = i;
    if (src[w] < 0) return fail(TAV2_EINVAL, "missing parameter tensor '%s'", want[w].name.c_str());
    if (numel[src[w]] != want[w].numel)
      return fail(TAV2_EINVAL, "parameter '%s' has %lld elements, expected %lld",
                  want[w].name.c_str(), (long long)numel[src[w]], (long long)want[w].numel);
    off[w] = total;
    total += (want[w].numel + 63) & ~int64_t(63);  // 256-byte aligned tensors
  }
  CU(cudaSetDevice(c->device));
  if (c->d_params) {
    CU(cudaDeviceSynchronize());
    cudaFree(c->d_params);
  cudaFree(c->d_images);
    c->d_params = nullptr;
  }
  CU(cudaMalloc(&c->d_params, total * 4));
  std::vector<float> host(total, 0.0f);
  for (size_t w = 0; w < want.size(); ++w) {
    memcpy(host.data() + off[w], data[src[w]], want[w].numel * 4);
    *want[w].slot = c->d_params + off[w];
  }
  CU(cudaMemcpy(c->d_params, host.data(), total * 4, cudaMemcpyHostToDevice));
  c->params = P;

  // ---- bf16 hi/lo weight images, UMMA B-operand layout (tav2_common.cuh) ----
  auto host_of = [&](const float* dev) { return host.data() + (dev - c->d_params); };
  const int L = m.num_layers;
  const size_t img_bytes = (size_t)L * (kImgWA + kImgWB) + kImgWO;
  std::vector<uint8_t> img(img_bytes, 0);
  auto bf16 = [](float x) -> uint16_t {  // round-to-nearest-even
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
  };
  auto bf16f = [](uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
  };
  // fp16 (IEEE binary16, round-to-nearest-even, subnormals kept) parts of
  // the fp16x3 images (skut_tc3 in fp32 mode)
  auto f16 = [](float x) -> uint16_t { return __half_as_ushort(__float2half_rn(x)); };
  auto f16f = [](uint16_t h) { return __half2float(__ushort_as_half(h)); };
  bool put_f16 = false;  // the format `put` writes
  // write W^T of an [in, out] matrix into a (N = n_total, K) slab image at row offset n0
  auto put = [&](uint8_t* base, int n_total, int K, int n0, const float* W, int in, int out) {
    uint8_t* lo_base = base + (size_t)n_total * K * 2;
    for (int k = 0; k < in; ++k)
      for (int n = 0; n < out; ++n) {
        const float w = W[k * out + n];
        const uint16_t hi = put_f16 ? f16(w) : bf16(w);
        const uint16_t lo = put_f16 ? f16(w - f16f(hi)) : bf16(w - bf16f(hi));
        const size_t off = (size_t)(k / 8) * (n_total * 16) + (size_t)(n0 + n) * 16 + (k % 8) * 2;
        memcpy(base + off, &hi, 2);
        memcpy(lo_base + off, &lo, 2);
      }
  };
  for (int l = 0; l < L; ++l) {
    uint8_t* wa = img.data() + (size_t)l * (kImgWA + kImgWB);
    uint8_t* wb = wa + kImgWA;
    put(wa, 192, 64, 0, host_of(P.wq[l]), 64, 64);
    put(wa, 192, 64, 64, host_of(P.wk[l]), 64, 64);
    put(wa, 192, 64, 128, host_of(P.wv[l]), 64, 64);
    put(wb, 64, 64, 0, host_of(P.wo[l]), 64, 64);                   // 16 KB
    put(wb + 16384, 32, 64, 0, host_of(P.w1[l]), 64, 32);           //  8 KB
    put(wb + 16384 + 8192, 64, 32, 0, host_of(P.w2[l]), 32, 64);    //  8 KB
  }
  put(img.data() + (size_t)L * (kImgWA + kImgWB), 64, 64, 0, host_of(P.out_linear), 64, 64);
  if (c->d_images) cudaFree(c->d_images);
  c->d_images = nullptr;
  CU(cudaMalloc(&c->d_images, img_bytes));
  CU(cudaMemcpy(c->d_images, img.data(), img_bytes, cudaMemcpyHostToDevice));
  for (int l = 0; l < L; ++l) {
    c->images.wa[l] = c->d_images + (size_t)l * (kImgWA + kImgWB);
    c->images.wb[l] = c->images.wa[l] + kImgWA;
  }
  c->images.wout = c->d_images + (size_t)L * (kImgWA + kImgWB);

  // ---- folded images of skut_tc3: per layer [ [Wqk|Wvo]^T | W1^T | W2^T ] ----
  // Wqk = Wq Wk^T * log2(e)/8 (scores in the exp2 domain), Wvo = Wv Wo; f64
  // products rounded once to f32 before the bf16 hi/lo split.
  c->cs_bound3 = c->cs_bound = 0.0;
  {
    const size_t lay = (size_t)kImg3WA + kImg3WB;
    const size_t bytes3 = (size_t)L * lay + kImg3WO + kImg3W2O;
    std::vector<uint8_t> img3(bytes3, 0), img3h(bytes3, 0);
    std::vector<float> wqk(64 * 64), wvo(64 * 64);
    const double sc = 1.4426950408889634 / 8.0;
    for (int l = 0; l < L; ++l) {
      const float *wq = host_of(P.wq[l]), *wk = host_of(P.wk[l]), *wv = host_of(P.wv[l]), *wo = host_of(P.wo[l]);
      for (int i = 0; i < 64; ++i)
        for (int j = 0; j < 64; ++j) {
          double a = 0.0, b = 0.0;
          for (int m2 = 0; m2 < 64; ++m2) {
            a += (double)wq[i * 64 + m2] * (double)wk[j * 64 + m2];
            b += (double)wv[i * 64 + m2] * (double)wo[m2 * 64 + j];
          }
          wqk[i * 64 + j] = (float)(a * sc);
          wvo[i * 64 + j] = (float)b;
        }
      // softmax-shift range of this layer: m' = ||q'_r|| max_j ||a_j|| <=
      // ||Wqk||_2 A^2 (folded, skut_tc3) or ||Wq||_2 ||Wk||_2 A^2 log2e/8
      // (skut_tc), with A = max|ln1_scale| sqrt(d) + ||ln1_shift||_2 >= ||a||
      {
        const float *g = host_of(P.ln1_scale[l]), *bt = host_of(P.ln1_shift[l]);
        double gm = 0.0, bn = 0.0;
        for (int i = 0; i < 64; ++i) {
          gm = std::max(gm, std::fabs((double)g[i]));
          bn += (double)bt[i] * bt[i];
        }
        const double A = gm * 8.0 + std::sqrt(bn);
        std::vector<double> m1(64 * 64), m2(64 * 64), m3(64 * 64);
        for (int i = 0; i < 64 * 64; ++i) {
          m1[i] = wqk[i];
          m2[i] = wq[i];
          m3[i] = wk[i];
        }
        c->cs_bound3 = std::max(c->cs_bound3, spectral_norm64(m1) * A * A);
        c->cs_bound = std::max(c->cs_bound, spectral_norm64(m2) * spectral_norm64(m3) * sc * A * A);
      }
      for (int h16 = 0; h16 < 2; ++h16) {  // bf16x3 (bf16 mode) and fp16x3 (fp32 mode) images
        put_f16 = h16 != 0;
        uint8_t* base = (h16 ? img3h : img3).data() + (size_t)l * lay;
        put(base, 128, 64, 0, wqk.data(), 64, 64);
        put(base, 128, 64, 64, wvo.data(), 64, 64);
        put(base + kImg3WA, 32, 64, 0, host_of(P.w1[l]), 64, 32);
        put(base + kImg3WA + 8192, 64, 32, 0, host_of(P.w2[l]), 32, 64);
      }
    }
    // W2' = W2 W_out of the last layer (f64): skut_tc3 computes the pooled
    // projection y = x W_out of the last layer's output x = x_mid + ReLU(H) W2
    // as x_mid W_out + ReLU(H) W2' -- one GEMM round trip instead of two
    std::vector<float> w2o(32 * 64);
    {
      const float *w2 = host_of(P.w2[L - 1]), *wo = host_of(P.out_linear);
      for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 64; ++j) {
          double a = 0.0;
          for (int m2 = 0; m2 < 64; ++m2) a += (double)w2[i * 64 + m2] * (double)wo[m2 * 64 + j];
          w2o[i * 64 + j] = (float)a;
        }
    }
    for (int h16 = 0; h16 < 2; ++h16) {
      put_f16 = h16 != 0;
      put((h16 ? img3h : img3).data() + (size_t)L * lay, 64, 64, 0, host_of(P.out_linear), 64, 64);
      put((h16 ? img3h : img3).data() + (size_t)L * lay + kImg3WO, 64, 32, 0, w2o.data(), 32, 64);
    }
    put_f16 = false;
    if (c->d_images3) cudaFree(c->d_images3);
    c->d_images3 = nullptr;
    CU(cudaMalloc(&c->d_images3, 2 * bytes3));
    CU(cudaMemcpy(c->d_images3, img3.data(), bytes3, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_images3 + bytes3, img3h.data(), bytes3, cudaMemcpyHostToDevice));
    for (int l = 0; l < L; ++l) {
      c->images3.w[l] = c->d_images3 + (size_t)l * lay;
      c->images3h.w[l] = c->d_images3 + bytes3 + (size_t)l * lay;
    }
    c->images3.wout = c->d_images3 + (size_t)L * lay;
    c->images3h.wout = c->d_images3 + bytes3 + (size_t)L * lay;
    c->images3.w2out = c->images3.wout + kImg3WO;
    c->images3h.w2out = c->images3h.wout + kImg3WO;
  }
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);  // captured with the old parameters
  c->graphs.clear();
  c->graph_seen.clear();
  c->params_ok = true;
  return TAV2_OK;
}

int tav2_store_reserve(tav2_ctx* c, int32_t max_users) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  if (max_users < 0) return fail(TAV2_EINVAL, "max_users must be >= 0");
  CU(cudaSetDevice(c->device));
  CU(cudaStreamSynchronize(c->copy_stream));  // pending staging copies may read the old pool
  cudaFree(c->st_emb);
  cudaFree(c->st_act);
  cudaFree(c->st_surf);
  c->st_emb = nullptr;
  c->st_act = nullptr;
  c->st_surf = nullptr;
  c->st_users = 0;
  c->st_map.clear();
  c->st_free.clear();
  if (max_users == 0) return TAV2_OK;
  const int64_t n = (int64_t)max_users * kStoreSlotTok;
  cudaError_t e;
  if ((e = cudaMalloc(&c->st_emb, n * kEmbed)) != cudaSuccess || (e = cudaMalloc(&c->st_act, n * 2)) != cudaSuccess ||
      (e = cudaMalloc(&c->st_surf, n)) != cudaSuccess)
    return fail(TAV2_ECUDA, "store pool of %d users: %s", max_users, cudaGetErrorString(e));
  c->st_users = max_users;
  for (int i = max_users - 1; i >= 0; --i) c->st_free.push_back(i);
  return TAV2_OK;
}

int tav2_store_put(tav2_ctx* c, uint64_t user_id, const tav2_request* q) {
  if (!c || !q) return fail(TAV2_EINVAL, "null argument");
  for (int k = 0; k < 3; ++k) {
    if (q->len[k] < 0 || q->len[k] > kCaps[k])
      return fail(TAV2_EINVAL, "source %d length %d outside [0, %d]", k, q->len[k], kCaps[k]);
    if (q->len[k] > 0 && (!q->emb[k] || !q->action[k] || !q->surface[k]))
      return fail(TAV2_EINVAL, "source %d has null columns", k);
  }
  auto it = c->st_map.find(user_id);
  int slot;
  if (it != c->st_map.end()) {
    slot = it->second.slot;  // replace wholesale (ordered after earlier staging on copy_stream)
  } else {
    if (c->st_free.empty())
      return fail(TAV2_ECAP, "HBM store full (%d users; tav2_store_reserve)", c->st_users);
    slot = c->st_free.back();
  }
  CU(cudaSetDevice(c->device));
  int64_t o = (int64_t)slot * kStoreSlotTok;
  for (int k = 0; k < 3; ++k) {
    const int64_t n = q->len[k];
    if (!n) continue;
    // pageable sources: each copy has consumed the caller's buffer on return
    CU(cudaMemcpyAsync(c->st_emb + o * kEmbed, q->emb[k], n * kEmbed, cudaMemcpyHostToDevice, c->copy_stream));
    CU(cudaMemcpyAsync(c->st_act + o, q->action[k], n * 2, cudaMemcpyHostToDevice, c->copy_stream));
    CU(cudaMemcpyAsync(c->st_surf + o, q->surface[k], n, cudaMemcpyHostToDevice, c->copy_stream));
    o += n;
  }
  if (it == c->st_map.end()) {
    c->st_free.pop_back();
    it = c->st_map.emplace(user_id, tav2_ctx::StoreEntry{slot, {0, 0, 0}}).first;
  }
  for (int k = 0; k < 3; ++k) it->second.len[k] = q->len[k];
  return TAV2_OK;
}

int tav2_store_remove(tav2_ctx* c, uint64_t user_id) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  auto it = c->st_map.find(user_id);
  if (it == c->st_map.end()) return fail(TAV2_EINVAL, "user %llu is not in the HBM store", (unsigned long long)user_id);
  c->st_free.push_back(it->second.slot);  // reuse is ordered after pending staging copies (copy_stream)
  c->st_map.erase(it);
  return TAV2_OK;
}

int tav2_store_count(const tav2_ctx* c) {
  if (!c) {
    fail(TAV2_EINVAL, "null context");
    return -1;
  }
  return (int)c->st_map.size();
}

int tav2_stage(tav2_ctx* c, const tav2_request* reqs, int n_req, void* stream, int32_t* n_items) {
  if (!c || !reqs) return fail(TAV2_EINVAL, "null argument");
  if (n_req < 1) return fail(TAV2_EINVAL, "at least one request required");  // nnsearch.py:221
  if (n_req > c->cap.max_requests)
    return fail(TAV2_ECAP, "%d requests exceed capacity %d", n_req, c->cap.max_requests);
  cudaStream_t s = (cudaStream_t)stream;
  const NNCfg& nn = c->nn;
  int N = 0;
  int64_t T = 0;
  int tiles = 0;
  // requests served from the HBM store: their lengths come from the store,
  // their token columns are copied device-to-device at staging time
  std::vector<tav2_request> rq_store;
  const tav2_ctx::StoreEntry* const no_entry = nullptr;
  std::vector<const tav2_ctx::StoreEntry*> ent((size_t)n_req, no_entry);
  for (int r = 0; r < n_req; ++r) {
    if (!reqs[r].from_store) continue;
    auto it = c->st_map.find(reqs[r].store_user);
    if (it == c->st_map.end())
      return fail(TAV2_EINVAL, "request %d: user %llu is not in the HBM store", r,
                  (unsigned long long)reqs[r].store_user);
    ent[r] = &it->second;
  }
  if (std::any_of(ent.begin(), ent.end(), [](const tav2_ctx::StoreEntry* e) { return e != nullptr; })) {
    rq_store.assign(reqs, reqs + n_req);
    for (int r = 0; r < n_req; ++r)
      if (ent[r])
        for (int k = 0; k < 3; ++k) {
          rq_store[r].len[k] = ent[r]->len[k];
          rq_store[r].emb[k] = nullptr;
          rq_store[r].action[k] = nullptr;
          rq_store[r].surface[k] = nullptr;
        }
    reqs = rq_store.data();
  }
  for (int r = 0; r < n_req; ++r) {
    const tav2_request& q = reqs[r];
    if (q.n_cand < 1 || !q.candidates)
      return fail(TAV2_EINVAL, "each request needs a non-empty (M, E) candidate array");
    if (ent[r]) {
      N += q.n_cand;
      T += (int64_t)q.len[0] + q.len[1] + q.len[2];
      tiles += cdiv(q.n_cand, kTile);
      continue;
    }
    for (int k = 0; k < 3; ++k) {
      if (q.len[k] < 0 || q.len[k] > kCaps[k])
        return fail(TAV2_EINVAL, "request %d source %d length %d outside [0, %d]", r, k, q.len[k],
                    kCaps[k]);
      if (q.len[k] > 0 && (!q.emb[k] || !q.action[k] || !q.surface[k]))
        return fail(TAV2_EINVAL, "request %d source %d has null columns", r, k);
    }
    N += q.n_cand;
    T += (int64_t)q.len[0] + q.len[1] + q.len[2];
    tiles += cdiv(q.n_cand, kTile);
  }
  if (N > c->cap.max_items) return fail(TAV2_ECAP, "%d items exceed capacity %d", N, c->cap.max_items);
  if (T > c->cap.max_tokens)
    return fail(TAV2_ECAP, "%lld tokens exceed capacity %lld", (long long)T, (long long)c->cap.max_tokens);

  // ---- NN work decomposition: one CTA per (candidate tile, source, chunk).
  // A source with n <= k tokens needs no scan (all selected), nor one with
  // n <= kDirectMax (nn_select scores every token exactly).  Otherwise the
  // threshold scan (nn_scan.cu) groups its tokens in G = 2^glog (about 4k to
  // 8k groups, G <= 32); chunk boundaries are kScanTile-aligned in the global
  // token index so every group and tile lies in one chunk.  RT tail and IMP take one
  // chunk per tile; LL chunks (>= kMinChunk tokens) fill the SMs. ----
  auto scanned = [&](const tav2_request& q, int s) {
    const int lo = s == 1 ? std::min(nn.recent, q.len[1]) : 0;
    return nn_scanned(q.len[s] - lo, nn.k[s]);
  };
  auto group_log = [&](int n, int k) {
    int g = 0;
    while (g < 5 && (n >> (g + 1)) >= 4 * k) ++g;
    return g;
  };
  int other = 0;
  for (int r = 0; r < n_req; ++r) {
    const int t = cdiv(reqs[r].n_cand, kTile);
    other += t * ((int)scanned(reqs[r], 1) + (int)scanned(reqs[r], 2));
  }
  const int ll_chunks_target = std::max(1, (c->sms - other) / std::max(tiles, 1));
  // token placement: the host requests' tokens first (one contiguous prefix
  // per column section, so the H2D copies skip the store requests' ranges),
  // then the store requests'
  std::vector<int64_t> tok_base((size_t)n_req);
  int64_t T_host = 0;
  {
    int64_t o = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int r = 0; r < n_req; ++r)
        if ((ent[r] != nullptr) == (pass == 1)) {
          tok_base[r] = o;
          o += (int64_t)reqs[r].len[0] + reqs[r].len[1] + reqs[r].len[2];
          if (pass == 0) T_host = o;
        }
  }
  std::vector<NNTile> vt;
  std::vector<NNWork> vw;
  std::vector<int> glogs((size_t)n_req * 3, 0);
  vt.reserve(tiles);
  {
    int item = 0;
    for (int r = 0; r < n_req; ++r) {
      const tav2_request& q = reqs[r];
      const int64_t tok_req = tok_base[r];
      int64_t tok_off[3];
      for (int s = 0, o = 0; s < 3; ++s) {
        tok_off[s] = tok_req + o;
        o += q.len[s];
        if (scanned(q, s)) glogs[r * 3 + s] = group_log(q.len[s] - (s == 1 ? nn.recent : 0), nn.k[s]);
      }
      for (int i0 = 0; i0 < q.n_cand; i0 += kTile) {
        NNTile t{};
        t.req = r;
        t.item0 = item + i0;
        t.n = std::min(kTile, q.n_cand - i0);
        const int tid = (int)vt.size();
        for (int s = 0; s < 3; ++s) {
          const int lo = s == 1 ? nn.recent : 0, hi = q.len[s];
          t.work0[s] = (int)vw.size();
          t.nwork[s] = 0;
          if (!scanned(q, s)) continue;
          int nch = 1;
          if (s == 0) nch = std::max(1, std::min(ll_chunks_target, (hi - lo) / kMinChunk));
          const int64_t step = std::max<int64_t>(kScanTile, ((int64_t)cdiv(hi - lo, nch) + kScanTile - 1) &
                                                                   ~int64_t(kScanTile - 1));
          for (int64_t a = tok_off[s] + lo, end = tok_off[s] + hi; a < end;) {
            const int64_t b = std::min(end, (a & ~int64_t(kScanTile - 1)) + step);
            vw.push_back(NNWork{tid, s, (int32_t)(a - tok_off[s]), (int32_t)(b - tok_off[s])});
            t.nwork[s]++;
            a = b;
          }
        }
        vt.push_back(t);
      }
      item += q.n_cand;
    }
  }
  if ((int)vt.size() > c->max_tiles || (int)vw.size() > c->max_work)
    return fail(TAV2_ECAP, "NN plan (%zu tiles, %zu work) exceeds capacity", vt.size(), vw.size());

  Plan p{};
  p.n_req = n_req;
  p.n_items = N;
  p.n_tok = (int32_t)T;
  p.n_tiles = (int)vt.size();
  p.n_work = (int)vw.size();
  p.tile_size = kTile;
  int64_t o = 0;
  p.off_req = o; o = align256(o + (int64_t)n_req * sizeof(ReqInfo));
  p.off_tiles = o; o = align256(o + (int64_t)p.n_tiles * sizeof(NNTile));
  p.off_work = o; o = align256(o + (int64_t)p.n_work * sizeof(NNWork));
  p.off_item_req = o; o = align256(o + (int64_t)N * 4);
  p.off_ctx = o; o = align256(o + (int64_t)n_req * kCtx * 4);
  p.off_cand = o; o = align256(o + (int64_t)N * kEmbed * 4);
  p.n_scopy = (int)std::count_if(ent.begin(), ent.end(), [](const tav2_ctx::StoreEntry* e) { return e != nullptr; });
  p.off_scopy = o; o = align256(o + (int64_t)p.n_scopy * sizeof(StoreCopy));
  p.off_action = o; o = align256(o + T * 2);
  p.off_surface = o; o = align256(o + T);
  p.off_emb = o; o = align256(o + T * kEmbed);
  p.bytes = o;

  // The slot's arena is reused: its previous H2D copy must have drained
  // before we overwrite it (arena reset contract, arena.py:49-55).
  const int slot = c->next_slot;
  CU(cudaEventSynchronize(c->ev_staged[slot]));
  unsigned char* h = c->h_arena[slot];
  ReqInfo* ri = reinterpret_cast<ReqInfo*>(h + p.off_req);
  int32_t* item_req = reinterpret_cast<int32_t*>(h + p.off_item_req);
  float* ctx = reinterpret_cast<float*>(h + p.off_ctx);
  float* cand = reinterpret_cast<float*>(h + p.off_cand);
  uint16_t* act = reinterpret_cast<uint16_t*>(h + p.off_action);
  uint8_t* surf = h + p.off_surface;
  int8_t* emb = reinterpret_cast<int8_t*>(h + p.off_emb);
  StoreCopy* scopy = reinterpret_cast<StoreCopy*>(h + p.off_scopy);
  int max_store_tok = 0;
  for (int r = 0, j = 0; r < n_req; ++r)
    if (ent[r]) {
      const int n = reqs[r].len[0] + reqs[r].len[1] + reqs[r].len[2];
      scopy[j++] = StoreCopy{(int64_t)ent[r]->slot * kStoreSlotTok, tok_base[r], n, 0};
      max_store_tok = std::max(max_store_tok, n);
    }
  int item = 0;
  for (int r = 0; r < n_req; ++r) {
    const tav2_request& q = reqs[r];
    int64_t tok = tok_base[r];
    ri[r].item_off = item;
    ri[r].n_items = q.n_cand;
    ri[r].pad_ = 0;
    for (int s = 0; s < 3; ++s) {
      ri[r].tok_off[s] = (int32_t)tok;
      ri[r].len[s] = q.len[s];
      ri[r].glog[s] = glogs[r * 3 + s];
      if (q.len[s] && !ent[r]) {
        memcpy(emb + tok * kEmbed, q.emb[s], (size_t)q.len[s] * kEmbed);
        memcpy(act + tok, q.action[s], (size_t)q.len[s] * 2);
        memcpy(surf + tok, q.surface[s], (size_t)q.len[s]);
      }
      tok += q.len[s];
    }
    memcpy(cand + (int64_t)item * kEmbed, q.candidates, (size_t)q.n_cand * kEmbed * 4);
    for (int i = 0; i < q.n_cand; ++i) item_req[item + i] = r;
    if (q.ctx)
      memcpy(ctx + r * kCtx, q.ctx, kCtx * 4);
    else
      memset(ctx + r * kCtx, 0, kCtx * 4);
    item += q.n_cand;
  }
  if (!vt.empty()) memcpy(h + p.off_tiles, vt.data(), vt.size() * sizeof(NNTile));
  if (!vw.empty()) memcpy(h + p.off_work, vw.data(), vw.size() * sizeof(NNWork));

  CU(cudaSetDevice(c->device));
  // the device region is rewritten once the kernels that read it last finished
  CU(cudaStreamWaitEvent(c->copy_stream, c->ev_done[slot], 0));
  unsigned char* d = c->d_staged[slot];
  if (T_host == T) {
    CU(cudaMemcpyAsync(d, h, p.bytes, cudaMemcpyHostToDevice, c->copy_stream));
  } else {  // header + the host tokens' prefix of each column section
    CU(cudaMemcpyAsync(d, h, p.off_action, cudaMemcpyHostToDevice, c->copy_stream));
    if (T_host > 0) {
      CU(cudaMemcpyAsync(d + p.off_action, h + p.off_action, T_host * 2, cudaMemcpyHostToDevice, c->copy_stream));
      CU(cudaMemcpyAsync(d + p.off_surface, h + p.off_surface, T_host, cudaMemcpyHostToDevice, c->copy_stream));
      CU(cudaMemcpyAsync(d + p.off_emb, h + p.off_emb, T_host * kEmbed, cudaMemcpyHostToDevice, c->copy_stream));
    }
    // the store users' tokens, device to device: one gather launch over the
    // copy descriptors (staged with the header)
    CU(launch_store_gather(reinterpret_cast<const StoreCopy*>(d + p.off_scopy), p.n_scopy, max_store_tok,
                           c->st_emb, c->st_act, c->st_surf, reinterpret_cast<int8_t*>(d + p.off_emb),
                           reinterpret_cast<uint16_t*>(d + p.off_action), d + p.off_surface, c->copy_stream));
    c->launches++;
  }
  CU(cudaEventRecord(c->ev_staged[slot], c->copy_stream));
  CU(cudaStreamWaitEvent(s, c->ev_staged[slot], 0));
  c->plans[slot] = p;
  c->cur = slot;
  c->next_slot = (slot + 1) % tav2_ctx::kStageSlots;
  c->staged = true;
  if (n_items) *n_items = N;
  return TAV2_OK;
}

}  // extern "C"

namespace {

// the staged slot's kernels are enqueued: its device region may be rewritten
// (by a later stage of the same slot) once they finish
int mark_used(tav2_ctx* c, cudaStream_t s) {
  CU(cudaEventRecord(c->ev_done[c->cur], s));
  return TAV2_OK;
}

int check_ready(tav2_ctx* c, int mode) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  if (!c->staged) return fail(TAV2_ESTATE, "no staged batch: call tav2_stage first");
  if (mode != TAV2_MODE_FP32 && mode != TAV2_MODE_BF16)
    return fail(TAV2_EINVAL, "unknown precision mode %d", mode);
  return TAV2_OK;
}

// Fused select -> SKUT runs hand over per candidate (SelFlags): a fresh
// epoch per run, so flags left by any earlier run never match.
SelFlags next_sel(tav2_ctx* c) {
#ifdef TAV2_NO_SELFLAGS
  return SelFlags{nullptr, nullptr, 0};
#endif
  return SelFlags{c->cur_dv().sel_done, c->cur_dv().sel_epoch, device_sms(), c->cur_dv().sel_epoch + 1};
}

// NN selection (both precision modes: the scan's survivors are re-scored with
// the reference's f64 formula, so the index sets are the reference's).
int run_nn(tav2_ctx* c, int32_t* idx, double* scores, cudaStream_t s, SelFlags sel = {nullptr, 0, 0}) {
  Staged st = staged_view(c);
  CU(timed(c, "prep", s, [&] {
    return launch_prep(st, c->params_ok ? &c->params : nullptr, s, sel.done ? c->cur_dv().sel_epoch : nullptr);
  }));
  CU(timed(c, "nn_scan1", s, [&] { return launch_nn_scan(st, c->nn, c->cur_dv().scan, 1, s); }));
  CU(timed(c, "nn_bound", s, [&] { return launch_nn_bound(st, c->nn, c->cur_dv().scan, s); }));
  CU(timed(c, "nn_scan2", s, [&] { return launch_nn_scan(st, c->nn, c->cur_dv().scan, 2, s); }));
  CU(timed(c, "nn_select", s, [&] { return launch_nn_select(st, c->nn, c->cur_dv().scan, idx, scores, sel, s); }));
  return TAV2_OK;
}

int run_score(tav2_ctx* c, int mode, const int32_t* idx, float* logits, float* pooled,
              cudaStream_t s, SelFlags sel = {nullptr, 0, 0}) {
  if (!c->params_ok) return fail(TAV2_ESTATE, "parameters not loaded");
  Staged st = staged_view(c);
  // The 2-row-tile tensor-core SKUT holds K/V of <= 256 keys in shared
  // memory; longer sequences (the k_ll = 256 sweep point, S = 352) run the
  // SIMT kernel, which is f32 throughout and so also meets the bf16 budget.
  // tensor-core SKUTs only while their single-pass softmax shift provably
  // stays in the exp2 range (2 m' <= 120); the SIMT kernel keeps a running max
  const bool tc3_ok = c->cs_bound3 <= 60.0, tc_ok = c->cs_bound <= 60.0;
  // S <= 192: the folded tensor-core SKUT -- bf16x3 parts in bf16 mode;
  // fp16x3 parts with a true-max softmax in fp32 mode (logits within 1e-5)
  if (tc3_ok && skut_tc3_supported(c->nn, c->params)) {
    const bool f16 = mode == TAV2_MODE_FP32;
    // the CTR head runs as its own kernel over the pooled vectors (head_kernel);
    // into the workspace (kPooledEmpty between runs) it starts per candidate as
    // soon as the candidate's pooled vector has landed
    float* pw = pooled ? pooled : c->cur_dv().pooled;
    CU(timed(c, f16 ? "skut_tc3_f16" : "skut_tc3", s, [&] {
      return launch_skut_tc3(c->params, f16 ? c->images3h : c->images3, c->nn, st, idx, st.n_items, logits, pw,
                             sel, f16, s);
    }));
    CU(timed(c, "head", s, [&] { return launch_head(c->params, st, pw, st.n_items, logits, pooled == nullptr, s); }));
    return TAV2_OK;
  }
  // 192 < S <= 384 (the k_ll = 128 / 256 sweep points): the same folded
  // bf16x3 / fp16x3 transformer on 2-CTA clusters, keys shared over DSMEM
  if (tc3_ok && skut_tc4_supported(c->nn, c->params) && !getenv_flag("TAV2_NO_TC4")) {
    const bool f16 = mode == TAV2_MODE_FP32;
    CU(timed(c, f16 ? "skut_tc4_f16" : "skut_tc4", s, [&] {
      return launch_skut_tc4(c->params, f16 ? c->images3h : c->images3, c->nn, st, idx, st.n_items, logits, pooled,
                             f16, s);
    }));
    return TAV2_OK;
  }
  if (mode == TAV2_MODE_BF16 && tc_ok && c->nn.seq_len <= 256) {
    CU(timed(c, "skut_tc", s, [&] {
      return launch_skut_tc(c->params, c->images, c->nn, &st, idx, nullptr, nullptr, st.n_items,
                            nullptr, logits, pooled, s);
    }));
    return TAV2_OK;
  }
  CU(timed(c, "skut_simt", s, [&] {
    return launch_skut_simt(c->params, c->nn, &st, idx, nullptr, nullptr, st.n_items,
                            c->cur_dv().skut_scratch, nullptr, logits, pooled, (int)tc_ok, s);
  }));
  return TAV2_OK;
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("TAV2_NO_GRAPH");
    return !(e && e[0] == '1');
  }();
  return on;
}

bool same_plan(const Plan& a, const Plan& b) {  // field by field (no padding bytes)
  return a.n_req == b.n_req && a.n_items == b.n_items && a.n_tok == b.n_tok && a.n_tiles == b.n_tiles &&
         a.n_work == b.n_work && a.tile_size == b.tile_size && a.n_scopy == b.n_scopy && a.off_req == b.off_req &&
         a.off_tiles == b.off_tiles && a.off_work == b.off_work && a.off_item_req == b.off_item_req &&
         a.off_ctx == b.off_ctx && a.off_cand == b.off_cand && a.off_scopy == b.off_scopy &&
         a.off_action == b.off_action && a.off_surface == b.off_surface && a.off_emb == b.off_emb &&
         a.bytes == b.bytes;
}

// The whole launch chain of a rank on the staged batch: prep -> scan1 ->
// bound -> scan2 -> select -> SKUT (programmatic dependent launches, the
// select -> SKUT per-candidate flag handover).  A batch shape seen before
// runs as one CUDA graph (captured on the ctx's capture stream the second
// time the shape occurs; every kernel argument is a function of the slot,
// the plan, the mode and the output buffer -- the flag epoch lives in
// device memory), so a repeated shape costs one cudaGraphLaunch instead of
// six launches.  Profiling (per-kernel events) launches directly.
int run_chain(tav2_ctx* c, int mode, float* logits, int32_t* idx, cudaStream_t s) {
  const SelFlags sel = next_sel(c);
  const Plan& pl = c->plans[c->cur];
  if (!c->profiling && graphs_enabled() && !c->graph_broken) {
    for (auto& g : c->graphs) {
      if (g.slot == c->cur && g.mode == mode && g.logits == logits && g.idx == idx && same_plan(g.plan, pl)) {
        g.last_use = ++c->graph_tick;
        c->launches = g.launches;
        CU(cudaGraphLaunch(g.exec, s));
        return TAV2_OK;
      }
    }
    bool seen = false;
    for (auto& x : c->graph_seen) seen = seen || (x.first == c->cur && same_plan(x.second, pl));
    if (seen) {  // second occurrence: capture
      cudaGraph_t graph = nullptr;
      cudaGraphExec_t exec = nullptr;
      c->launches = 0;
      int rc = TAV2_OK;
      if (cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        rc = run_nn(c, idx, nullptr, c->cap_stream, sel);
        if (!rc) rc = run_score(c, mode, idx, logits, nullptr, c->cap_stream, sel);
        const cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
        if (!rc && e == cudaSuccess && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
          if (c->graphs.size() >= 8) {  // evict the least recently used
            auto lru = c->graphs.begin();
            for (auto it = c->graphs.begin(); it != c->graphs.end(); ++it)
              if (it->last_use < lru->last_use) lru = it;
            cudaGraphExecDestroy(lru->exec);
            c->graphs.erase(lru);
          }
          c->graphs.push_back({c->cur, mode, logits, idx, pl, exec, c->launches, ++c->graph_tick});
          if (graph) cudaGraphDestroy(graph);
          CU(cudaGraphLaunch(exec, s));
          return TAV2_OK;
        }
        if (graph) cudaGraphDestroy(graph);
      }
      cudaGetLastError();  // clear a capture error; launch directly from now on
      c->graph_broken = true;
    } else {
      if (c->graph_seen.size() >= 32) c->graph_seen.erase(c->graph_seen.begin());
      c->graph_seen.push_back({c->cur, pl});
    }
  }
  c->launches = 0;
  int rc = run_nn(c, idx, nullptr, s, sel);
  if (!rc) rc = run_score(c, mode, idx, logits, nullptr, s, sel);
  return rc;
}


}  // namespace

extern "C" {

int tav2_nn_select(tav2_ctx* c, int mode, int32_t* idx_dev, double* scores_dev, void* stream) {
  int rc = check_ready(c, mode);
  if (rc) return rc;
  if (!idx_dev) return fail(TAV2_EINVAL, "idx_dev is null");
  CU(cudaSetDevice(c->device));
  c->launches = 0;
  int rc2 = run_nn(c, idx_dev, scores_dev, (cudaStream_t)stream);
  return rc2 ? rc2 : mark_used(c, (cudaStream_t)stream);
}

int tav2_similarity(tav2_ctx* c, int32_t item, int32_t source, double* scores_dev, void* stream) {
  int rc = check_ready(c, TAV2_MODE_FP32);
  if (rc) return rc;
  if (!scores_dev) return fail(TAV2_EINVAL, "scores_dev is null");
  if (source < 0 || source > 2) return fail(TAV2_EINVAL, "source must be 0 (LL), 1 (RT) or 2 (IMP)");
  const Plan& pl = c->plans[c->cur];
  if (item < 0 || item >= pl.n_items) return fail(TAV2_EINVAL, "item %d out of range", item);
  const ReqInfo* rq = reinterpret_cast<const ReqInfo*>(c->h_arena[c->cur] + pl.off_req);
  const int32_t* item_req = reinterpret_cast<const int32_t*>(c->h_arena[c->cur] + pl.off_item_req);
  const int n = rq[item_req[item]].len[source];
  CU(cudaSetDevice(c->device));
  Staged st = staged_view(c);
  CU(launch_prep(st, nullptr, (cudaStream_t)stream));
  CU(launch_similarity(st, item, source, n, scores_dev, (cudaStream_t)stream));
  return mark_used(c, (cudaStream_t)stream);
}

int tav2_pool(tav2_ctx* c, const float* u_dev, const uint8_t* mask_dev, int32_t n, float* pooled_dev,
              void* stream) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  if (!c->params_ok) return fail(TAV2_ESTATE, "parameters not loaded");
  if (n < 0) return fail(TAV2_EINVAL, "negative batch");
  if (n == 0) return TAV2_OK;
  if (!u_dev || !mask_dev || !pooled_dev) return fail(TAV2_EINVAL, "null device pointer");
  CU(cudaSetDevice(c->device));
  CU(launch_pool(u_dev, mask_dev, c->params.out_linear, n, c->nn.seq_len, pooled_dev, (cudaStream_t)stream));
  return TAV2_OK;
}

int tav2_encode(tav2_ctx* c, const int32_t* idx_dev, float* features_dev, uint8_t* mask_dev,
                void* stream) {
  int rc = check_ready(c, TAV2_MODE_FP32);
  if (rc) return rc;
  if (!c->params_ok) return fail(TAV2_ESTATE, "parameters not loaded");
  if (!idx_dev || !features_dev || !mask_dev) return fail(TAV2_EINVAL, "null device pointer");
  CU(cudaSetDevice(c->device));
  Staged st = staged_view(c);
  CU(launch_prep(st, nullptr, (cudaStream_t)stream));
  CU(launch_encode(st, c->nn, c->params, idx_dev, features_dev, mask_dev, (cudaStream_t)stream));
  return mark_used(c, (cudaStream_t)stream);
}

int tav2_forward(tav2_ctx* c, int mode, const float* features_dev, const uint8_t* mask_dev,
                 int32_t n, float* u_dev, void* stream) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  if (!c->params_ok) return fail(TAV2_ESTATE, "parameters not loaded");
  if (mode != TAV2_MODE_FP32 && mode != TAV2_MODE_BF16)
    return fail(TAV2_EINVAL, "unknown precision mode %d", mode);
  if (n < 0) return fail(TAV2_EINVAL, "negative batch");
  if (n == 0) return TAV2_OK;
  if (!features_dev || !mask_dev || !u_dev) return fail(TAV2_EINVAL, "null device pointer");
  CU(cudaSetDevice(c->device));
  if (mode == TAV2_MODE_BF16 && c->cs_bound <= 60.0 && c->nn.seq_len <= 256) {
    CU(launch_skut_tc(c->params, c->images, c->nn, nullptr, nullptr, features_dev, mask_dev, n,
                      u_dev, nullptr, nullptr, (cudaStream_t)stream));
    return TAV2_OK;
  }
  CU(launch_skut_simt(c->params, c->nn, nullptr, nullptr, features_dev, mask_dev, n,
                      c->cur_dv().skut_scratch, u_dev, nullptr, nullptr, (int)(c->cs_bound <= 60.0),
                      (cudaStream_t)stream));
  return TAV2_OK;
}

int tav2_forward_masked(tav2_ctx* c, int mode, const float* features_dev, const uint8_t* mask_dev,
                        const uint8_t* extra_dev, int32_t extra_batched, int32_t n, float* u_dev, void* stream) {
  if (!extra_dev) return tav2_forward(c, mode, features_dev, mask_dev, n, u_dev, stream);
  if (!c) return fail(TAV2_EINVAL, "null context");
  if (!c->params_ok) return fail(TAV2_ESTATE, "parameters not loaded");
  if (mode != TAV2_MODE_FP32 && mode != TAV2_MODE_BF16)
    return fail(TAV2_EINVAL, "unknown precision mode %d", mode);
  if (n < 0) return fail(TAV2_EINVAL, "negative batch");
  if (n == 0) return TAV2_OK;
  if (!features_dev || !mask_dev || !u_dev) return fail(TAV2_EINVAL, "null device pointer");
  CU(cudaSetDevice(c->device));
  // f32 SIMT transformer with the running-max softmax (the custom mask may
  // drop a row's own key, so the diagonal-based shifts do not apply); it
  // meets both modes' tolerances
  const long long S = c->nn.seq_len;
  CU(launch_skut_simt(c->params, c->nn, nullptr, nullptr, features_dev, mask_dev, n, c->cur_dv().skut_scratch, u_dev,
                      nullptr, nullptr, 0, (cudaStream_t)stream, extra_dev, extra_batched ? S * S : 0));
  return TAV2_OK;
}

int tav2_score(tav2_ctx* c, int mode, const int32_t* idx_dev, float* logits_dev, float* pooled_dev,
               void* stream) {
  int rc = check_ready(c, mode);
  if (rc) return rc;
  if (!idx_dev || !logits_dev) return fail(TAV2_EINVAL, "null device pointer");
  CU(cudaSetDevice(c->device));
  c->launches = 0;
  Staged st = staged_view(c);
  CU(timed(c, "prep", (cudaStream_t)stream, [&] { return launch_prep(st, &c->params, (cudaStream_t)stream); }));
  rc = run_score(c, mode, idx_dev, logits_dev, pooled_dev, (cudaStream_t)stream);
  return rc ? rc : mark_used(c, (cudaStream_t)stream);
}

int tav2_run_staged(tav2_ctx* c, int mode, float* logits_dev, void* stream) {
  int rc = check_ready(c, mode);
  if (rc) return rc;
  CU(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if ((rc = run_chain(c, mode, logits_dev ? logits_dev : c->logits, c->idx, s))) return rc;
  return mark_used(c, s);
}

int tav2_rank_submit(tav2_ctx* c, const tav2_request* reqs, int n_req, int mode, int want_idx, void* stream,
                     int32_t* slot_out) {
  if (!c || !slot_out) return fail(TAV2_EINVAL, "null argument");
  const int slot = c->next_slot;
  // the slot's pinned outputs are free once its previous rank finished
  CU(cudaEventSynchronize(c->ev_done[slot]));
  // Each slot's chain runs on the slot's own compute stream (after the
  // caller's stream: work the caller enqueued first stays first), so two
  // submitted requests' kernels can overlap: request i+1's NN chain fills
  // the SMs request i's SKUT tail frees (slot-private derived buffers).
  cudaStream_t s = c->slot_stream[slot];
  CU(cudaEventRecord(c->ev_caller[slot], (cudaStream_t)stream));
  CU(cudaStreamWaitEvent(s, c->ev_caller[slot], 0));
  int32_t n = 0;
  int rc = tav2_stage(c, reqs, n_req, s, &n);
  if (rc) return rc;
  if ((rc = run_chain(c, mode, c->logits_s[slot], c->idx_s[slot], s))) return rc;
  // result copies on the d2h stream: the compute stream goes straight on to
  // the next request's kernels
  CU(cudaEventRecord(c->ev_comp[slot], s));
  CU(cudaStreamWaitEvent(c->d2h_stream, c->ev_comp[slot], 0));
  CU(cudaMemcpyAsync(c->h_out[slot], c->logits_s[slot], (size_t)n * kHeads * 4, cudaMemcpyDeviceToHost,
                     c->d2h_stream));
  if (want_idx)
    CU(cudaMemcpyAsync(c->h_idx[slot], c->idx_s[slot], (size_t)n * c->nn.seq_len * 4, cudaMemcpyDeviceToHost,
                       c->d2h_stream));
  c->out_n[slot] = n;
  c->out_idx[slot] = want_idx != 0;
  CU(cudaEventRecord(c->ev_done[slot], c->d2h_stream));  // kernels + result copies of this slot
  *slot_out = slot;
  return TAV2_OK;
}

int tav2_rank_wait(tav2_ctx* c, int slot) {
  if (!c || slot < 0 || slot >= tav2_ctx::kStageSlots) return fail(TAV2_EINVAL, "bad slot");
  CU(cudaEventSynchronize(c->ev_done[slot]));
  return TAV2_OK;
}

int tav2_rank_collect(tav2_ctx* c, int slot, float* logits_host, int32_t* idx_host) {
  if (!c || slot < 0 || slot >= tav2_ctx::kStageSlots) return fail(TAV2_EINVAL, "bad slot");
  if (!logits_host) return fail(TAV2_EINVAL, "logits_host is null");
  CU(cudaEventSynchronize(c->ev_done[slot]));
  memcpy(logits_host, c->h_out[slot], (size_t)c->out_n[slot] * kHeads * 4);
  if (idx_host) {
    if (!c->out_idx[slot]) return fail(TAV2_ESTATE, "indices were not requested at submit");
    memcpy(idx_host, c->h_idx[slot], (size_t)c->out_n[slot] * c->nn.seq_len * 4);
  }
  return TAV2_OK;
}

int tav2_rank(tav2_ctx* c, const tav2_request* reqs, int n_req, int mode, float* logits_host,
              int32_t* idx_host, void* stream) {
  if (!logits_host) return fail(TAV2_EINVAL, "logits_host is null");
  int32_t n = 0;
  int rc = tav2_stage(c, reqs, n_req, stream, &n);
  if (rc) return rc;
  if ((rc = tav2_run_staged(c, mode, c->logits, stream))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(logits_host, c->logits, (size_t)n * kHeads * 4, cudaMemcpyDeviceToHost, s));
  if (idx_host)
    CU(cudaMemcpyAsync(idx_host, c->idx, (size_t)n * c->nn.seq_len * 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return TAV2_OK;
}

int tav2_last_launch_count(const tav2_ctx* c) { return c ? c->launches : 0; }

int tav2_stage_slots(void) { return TAV2_STAGE_SLOTS; }

int tav2_graph_info(const void* ctx, int32_t* n_graphs, int32_t* broken) {
  const tav2_ctx* c = static_cast<const tav2_ctx*>(ctx);
  if (!c) return fail(TAV2_EINVAL, "null context");
  if (n_graphs) *n_graphs = (int32_t)c->graphs.size();
  if (broken) *broken = c->graph_broken ? 1 : 0;
  return TAV2_OK;
}

int tav2_debug_timeline(long long* dev, int block) {
  return set_debug_timeline(dev, block) == cudaSuccess && set_debug_skut(dev ? dev + 320 : nullptr) == cudaSuccess &&
                 set_debug_skut3(dev ? dev + 640 : nullptr) == cudaSuccess
             ? TAV2_OK
             : fail(TAV2_ECUDA, "debug timeline");
}

int tav2_debug_cta(long long* dev) {
  if (set_dbg_cta_prep(dev) != cudaSuccess || set_dbg_cta_scan(dev) != cudaSuccess ||
      set_dbg_cta_select(dev) != cudaSuccess || set_dbg_cta_skut(dev) != cudaSuccess ||
      set_dbg_cta_skut3(dev) != cudaSuccess)
    return fail(TAV2_ECUDA, "debug cta stamps");
  return TAV2_OK;
}

int tav2_set_profiling(tav2_ctx* c, int on) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  for (auto& sl : c->slots) {
    settle(sl);
    sl.ms = 0.0;
    sl.n = 0;
  }
  c->profiling = on != 0;
  return TAV2_OK;
}

int tav2_kernel_times(tav2_ctx* c, const char** names, double* ms, int32_t* launches, int max) {
  if (!c) return fail(TAV2_EINVAL, "null context");
  int k = 0;
  for (auto& sl : c->slots) {
    if (!sl.name) continue;
    settle(sl);
    if (k < max) {
      if (names) names[k] = sl.name;
      if (ms) ms[k] = sl.ms;
      if (launches) launches[k] = sl.n;
    }
    ++k;
  }
  return k;
}

}  // extern "C"
