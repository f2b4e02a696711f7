"""Per-worker engine: one native tav2 context (pinned staging arena + device
workspace, the B200 analogue of ``serving/arena.py``'s per-worker Arena)
holding one immutable model.

PyTorch is used only as plumbing: device buffers and the CUDA stream.  All
compute runs in ``libtav2.so``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import functools
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .core import EMBED_DIM, UserSequences, ValidationError
from .model import ModelConfig, RankingModel
from .nnsearch import AssembledSequence, DedupBatch, NNConfig


@dataclass(frozen=True)
class Capacity:
    max_requests: int = 64
    max_items: int = 4096
    max_tokens: int = 64 * (16384 + 512)


def _cfg_struct(mc: ModelConfig) -> N.Config:
    e, nn = mc.encoder, mc.nn
    return N.Config(e.embed_dim, e.seq_len, e.ffn_dim, e.num_layers, e.action_rows, e.surface_rows,
                    mc.ctx_dim, mc.hidden_dim, nn.recent, nn.k_lifelong, nn.k_realtime,
                    nn.k_impression)


@dataclass(frozen=True)
class StoreUser:
    """A request's user read from the engine's HBM-resident store
    (``Engine.store_put``) instead of host token columns."""

    user_id: int


def _columns(user: UserSequences, r, keep) -> None:
    for s, blk in enumerate(user.blocks()):
        emb = np.ascontiguousarray(blk.embeddings, np.int8)
        act = np.ascontiguousarray(blk.actions, np.uint16)
        surf = np.ascontiguousarray(blk.surfaces, np.uint8)
        if emb.ndim != 2 or emb.shape[1] != EMBED_DIM:
            raise ValidationError(f"token embeddings must be (n, {EMBED_DIM}) int8")
        keep += [emb, act, surf]
        r.emb[s], r.action[s], r.surface[s] = emb.ctypes.data, act.ctypes.data, surf.ctypes.data
        r.len[s] = len(blk)


def _locked(fn):
    """Serialise a method on the engine's lock: one native context is never
    driven by two threads at once (arena.py:17), whoever calls it."""

    @functools.wraps(fn)
    def wrapper(self, *a, **kw):
        with self._lock:
            return fn(self, *a, **kw)

    return wrapper


class _Pack:
    """Keeps the numpy columns of a request list alive across a native call.
    A request's user is a UserSequences (host columns) or a StoreUser."""

    def __init__(self, requests):
        self.keep = []
        self.arr = (N.Request * len(requests))()
        for i, (user, cands, ctx) in enumerate(requests):
            r = self.arr[i]
            if isinstance(user, StoreUser):
                r.from_store, r.store_user = 1, int(user.user_id)
            else:
                _columns(user, r, self.keep)
            c = np.ascontiguousarray(cands, np.float32)
            if c.ndim != 2 or c.shape[1] != EMBED_DIM:
                raise ValidationError(f"candidates must be (n, {EMBED_DIM}) float32")
            x = np.ascontiguousarray(ctx if ctx is not None else np.zeros(8), np.float32)
            self.keep += [c, x]
            r.candidates, r.n_cand, r.ctx = c.ctypes.data, len(c), x.ctypes.data


class Engine:
    """One native worker context (arena.py:16-55): a pinned staging arena and
    a device workspace sized once from ``capacity``.  Every native call runs
    under the engine's lock, so a shared engine serialises its callers
    (give each worker thread its own engine for parallelism).

    Capacity overflow follows the reference arena (arena.py:40-44): a batch
    that does not fit is split into fitting sub-batches, and a single request
    larger than the whole capacity runs on a fallback context sized for it;
    both count in ``overflow_count`` instead of failing the batch."""

    def __init__(self, model: RankingModel | None = None, config: ModelConfig | None = None,
                 capacity: Capacity = Capacity(), device: int = 0):
        if model is None and config is None:
            raise ValidationError("need a model or a ModelConfig")
        self.config = model.config if model is not None else config
        self.config.validate()
        self.capacity = capacity
        self.device = device
        self.torch_device = torch.device("cuda", device)
        self._lib = N.lib()
        self._ctx = ctypes.c_void_p()
        cap = N.Capacity(capacity.max_requests, capacity.max_items, capacity.max_tokens)
        N.check(self._lib.tav2_create(ctypes.byref(_cfg_struct(self.config)), ctypes.byref(cap),
                                      device, ctypes.byref(self._ctx)))
        self.model = None
        self.n_items = 0
        self.overflow_count = 0
        self._perm = None          # staged item order -> batch item order (DedupBatch)
        self._store_tokens = {}    # user id -> resident token count (capacity planning)
        self._fallback = None      # context for requests larger than `capacity`
        self._lock = threading.RLock()
        if model is not None:
            self.load_model(model)

    @classmethod
    def for_batch(cls, cfg: NNConfig, batch: DedupBatch, device: int = 0) -> "Engine":
        toks = sum(u.total_tokens() for u in batch.users)
        cap = Capacity(len(batch.users), len(batch), max(toks, 1))
        return cls(config=ModelConfig.for_nn(cfg), capacity=cap, device=device)

    @property
    def nn_cfg(self) -> NNConfig:
        return self.config.nn

    def close(self) -> None:
        if getattr(self, "_fallback", None) is not None:
            self._fallback.close()
            self._fallback = None
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.tav2_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------
    @_locked
    def load_model(self, model: RankingModel) -> None:
        """RankingModel.load equivalent: upload the named tensors once."""
        if model.config != self.config:
            raise ValidationError("model config differs from the engine config")
        tensors = {k: np.ascontiguousarray(v, np.float32) for k, v in model.named_tensors().items()}
        names = (ctypes.c_char_p * len(tensors))(*[k.encode() for k in tensors])
        data = (ctypes.c_void_p * len(tensors))(*[v.ctypes.data for v in tensors.values()])
        numel = (ctypes.c_int64 * len(tensors))(*[v.size for v in tensors.values()])
        N.check(self._lib.tav2_load_params(self._ctx, len(tensors), names, data, numel))
        self.model = model

    def stream(self) -> int:
        return torch.cuda.current_stream(self.torch_device).cuda_stream

    # ------------------------------------------------------------------
    # HBM-resident feature store (tav2_store_*; serving.DeviceFeatureStore
    # is the FeatureStore-shaped front end)
    @_locked
    def store_reserve(self, max_users: int) -> None:
        """(Re)allocate the device pool for max_users users (drops all)."""
        N.check(self._lib.tav2_store_reserve(self._ctx, int(max_users)))
        self._store_tokens.clear()

    @_locked
    def store_put(self, user_id: int, user: UserSequences) -> None:
        """Insert or replace a user's sequences in HBM (lengths within the caps)."""
        r, keep = N.Request(), []
        _columns(user, r, keep)
        N.check(self._lib.tav2_store_put(self._ctx, int(user_id), ctypes.byref(r)))
        self._store_tokens[int(user_id)] = user.total_tokens()

    @_locked
    def store_remove(self, user_id: int) -> None:
        N.check(self._lib.tav2_store_remove(self._ctx, int(user_id)))
        self._store_tokens.pop(int(user_id), None)

    def store_count(self) -> int:
        return int(self._lib.tav2_store_count(self._ctx))

    # ------------------------------------------------------------------
    # capacity planning (the arena contract, arena.py:32-47)
    def _size(self, req) -> tuple[int, int]:
        user, cands, _ = req
        if isinstance(user, StoreUser):
            toks = self._store_tokens.get(int(user.user_id), 0)
        else:
            toks = user.total_tokens()
        return len(cands), toks

    def _fits(self, n_req, items, toks) -> bool:
        c = self.capacity
        return n_req <= c.max_requests and items <= c.max_items and toks <= c.max_tokens

    def _chunks(self, requests):
        """Greedy split into sub-batches that fit the capacity, in order;
        yields (chunk, oversized) with oversized=True for a single request
        larger than the whole capacity."""
        cur, items, toks = [], 0, 0
        for req in requests:
            i, t = self._size(req)
            if not self._fits(1, i, t):
                if cur:
                    yield cur, False
                    cur, items, toks = [], 0, 0
                yield [req], True
                continue
            if cur and not self._fits(len(cur) + 1, items + i, toks + t):
                yield cur, False
                cur, items, toks = [], 0, 0
            cur.append(req)
            items += i
            toks += t
        if cur:
            yield cur, False

    def _fallback_engine(self, req) -> "Engine":
        """The counted fallback allocation (arena.py:40-44): a context sized
        for one request that exceeds ``capacity``; kept for reuse."""
        i, t = self._size(req)
        if isinstance(req[0], StoreUser):
            raise ValidationError("a stored user's request exceeds the engine capacity")
        fb = self._fallback
        if fb is None or not fb._fits(1, i, t):
            if fb is not None:
                fb.close()
            cap = Capacity(1, max(i, self.capacity.max_items), max(t, self.capacity.max_tokens, 1))
            fb = Engine(self.model, config=self.config, capacity=cap, device=self.device)
            self._fallback = fb
        return fb

    @_locked
    def stage(self, requests) -> int:
        """requests: list of (UserSequences | StoreUser, candidates[M,32], ctx[8] | None)."""
        pack = _Pack(requests)
        n = ctypes.c_int32()
        N.check(self._lib.tav2_stage(self._ctx, pack.arr, len(requests), self.stream(),
                                     ctypes.byref(n)))
        self.n_items = n.value
        self._perm = None
        return n.value

    @_locked
    def stage_batch(self, batch: DedupBatch, contexts=None) -> int:
        """Stage a DedupBatch (items grouped by request on the device; see
        ``DedupBatch.grouped_order``)."""
        batch.validate()
        perm = batch.grouped_order()
        cands = batch.candidates[perm]
        reqs = []
        for r, sl in enumerate(batch.request_slices()):
            ctx = None if contexts is None else contexts[r]
            reqs.append((batch.users[r], cands[sl], ctx))
        n = self.stage(reqs)
        self._perm = None if np.array_equal(perm, np.arange(len(perm))) else perm
        return n

    def _unpermute(self, a: np.ndarray) -> np.ndarray:
        if self._perm is None:
            return a
        out = np.empty_like(a)
        out[self._perm] = a
        return out

    def _mode(self, mode: str) -> int:
        try:
            return N.MODES[mode]
        except KeyError:
            raise ValidationError(f"unknown precision mode {mode!r} (fp32 | bf16)") from None

    # ------------------------------------------------------------------
    @_locked
    def nn_select(self, batch: DedupBatch, mode: str = "bf16", return_scores: bool = False):
        """Device NN selection over a DedupBatch -> idx [N, S] int32 (-1 pad)
        in batch item order (and the f64 score of every NN slot)."""
        toks = sum(u.total_tokens() for u in batch.users)
        if not self._fits(len(batch.users), len(batch), toks):
            raise ValidationError("batch exceeds the engine capacity (use fused_assemble without an "
                                  "engine, or a larger Capacity)")
        n = self.stage_batch(batch)
        S = self.config.nn.seq_len
        idx = torch.empty((n, S), dtype=torch.int32, device=self.torch_device)
        sc = torch.empty((n, S), dtype=torch.float64, device=self.torch_device) if return_scores else None
        N.check(self._lib.tav2_nn_select(self._ctx, self._mode(mode), N.ptr(idx), N.ptr(sc),
                                         self.stream()))
        idx_h = self._unpermute(idx.cpu().numpy())
        if return_scores:
            return idx_h, self._unpermute(sc.cpu().numpy())
        return idx_h

    @_locked
    def similarity(self, user: UserSequences, candidates: np.ndarray, source: int = 0, item: int = 0):
        """similarity_scores of every token of one source (0 LL, 1 RT, 2 IMP)
        against candidate `item` (tav2_similarity) -> f64 [len(source)]."""
        n = len(user.blocks()[source])
        self.stage([(user, candidates, None)])
        out = torch.empty((max(n, 1),), dtype=torch.float64, device=self.torch_device)
        N.check(self._lib.tav2_similarity(self._ctx, int(item), int(source), N.ptr(out), self.stream()))
        return out.cpu().numpy()[:n]

    def _stage_assembled(self, seqs: list[AssembledSequence], candidates: np.ndarray, contexts=None):
        """Stage already-assembled sequences: each becomes a one-item request
        whose sources hold exactly its valid tokens, with the index layout
        that gathers them back in place -> device idx [B, S]."""
        if self.model is None:
            raise ValidationError("no model loaded")
        cfg = self.config.nn
        S = cfg.seq_len
        if any(len(s) != S for s in seqs):
            raise ValidationError("assembled length must match the positional table")
        starts, lens = cfg.segment_starts(), cfg.segment_lengths()
        reqs, idx = [], np.full((len(seqs), S), -1, np.int32)
        for i, s in enumerate(seqs):
            parts = []
            for g in range(4):
                v = int(np.count_nonzero(s.mask[starts[g]:starts[g] + lens[g]]))
                parts.append(np.arange(starts[g], starts[g] + v))
            ll, rt, imp = parts[0], np.concatenate([parts[1], parts[2]]), parts[3]
            idx[i, parts[0]] = np.arange(len(ll))
            idx[i, parts[1]] = np.arange(len(parts[1]))
            idx[i, parts[2]] = len(parts[1]) + np.arange(len(parts[2]))
            idx[i, parts[3]] = np.arange(len(imp))
            user = UserSequences(s.block.take(ll), s.block.take(rt), s.block.take(imp))
            ctx = None if contexts is None else contexts[i]
            reqs.append((user, np.asarray(candidates[i:i + 1], np.float32), ctx))
        if not self._fits(len(reqs), len(reqs), sum(u.total_tokens() for u, _, _ in reqs)):
            raise ValidationError("batch exceeds the engine capacity")
        self.stage(reqs)
        return torch.from_numpy(idx).to(self.torch_device)

    @_locked
    def encode(self, seqs: list[AssembledSequence], candidates: np.ndarray):
        """encode_batch (encoder.py:161-188) on the GPU -> (F [B,S,64], mask [B,S])."""
        idx_d = self._stage_assembled(seqs, candidates)
        n, S = idx_d.shape
        F = torch.empty((n, S, 2 * EMBED_DIM), dtype=torch.float32, device=self.torch_device)
        m = torch.empty((n, S), dtype=torch.uint8, device=self.torch_device)
        N.check(self._lib.tav2_encode(self._ctx, N.ptr(idx_d), N.ptr(F), N.ptr(m), self.stream()))
        return F.cpu().numpy(), m.cpu().numpy().astype(bool)

    @_locked
    def score_assembled(self, seqs: list[AssembledSequence], candidates: np.ndarray, contexts,
                        mode: str = "fp32"):
        """The fused gather + encode + SKUT + pool + head (tav2_score) over
        assembled sequences -> (logits [B, 4], pooled [B, 64])."""
        idx_d = self._stage_assembled(seqs, candidates, contexts)
        logits, pooled = self.score_staged(idx_d, mode=mode, pooled=True)
        return logits.cpu().numpy(), pooled.cpu().numpy()

    @_locked
    def pool(self, u: np.ndarray, mask: np.ndarray) -> np.ndarray:
        """pool (encoder.py:265-273) over encoder outputs U [B, S, 64] -> [B, 64]."""
        if self.model is None:
            raise ValidationError("no model loaded")
        u = np.asarray(u, np.float32)
        B, S, d = u.shape
        if S != self.config.nn.seq_len or d != 2 * EMBED_DIM:
            raise ValidationError("encoder output shape does not match the model")
        U = torch.from_numpy(np.ascontiguousarray(u)).to(self.torch_device)
        m = torch.from_numpy(np.ascontiguousarray(mask, np.uint8)).to(self.torch_device)
        out = torch.empty((B, d), dtype=torch.float32, device=self.torch_device)
        N.check(self._lib.tav2_pool(self._ctx, N.ptr(U), N.ptr(m), B, N.ptr(out), self.stream()))
        return out.cpu().numpy()

    @_locked
    def forward(self, features: np.ndarray, mask: np.ndarray, mode: str = "fp32", extra_mask=None) -> np.ndarray:
        """forward_fused over caller features (B, S, 64) -> U (valid rows);
        extra_mask [S, S] or [B, S, S] (encoder.py:366-377) -> tav2_forward_masked."""
        if self.model is None:
            raise ValidationError("no model loaded")
        B, S, d = features.shape
        if S != self.config.nn.seq_len or d != 2 * EMBED_DIM:
            raise ValidationError("feature shape does not match the model")
        F = torch.from_numpy(np.ascontiguousarray(features, np.float32)).to(self.torch_device)
        m = torch.from_numpy(np.ascontiguousarray(mask, np.uint8)).to(self.torch_device)
        U = torch.empty_like(F)
        if extra_mask is None:
            N.check(self._lib.tav2_forward(self._ctx, self._mode(mode), N.ptr(F), N.ptr(m), B, N.ptr(U),
                                           self.stream()))
        else:
            em = np.asarray(extra_mask, bool)
            if em.shape not in ((S, S), (B, S, S)):
                raise ValidationError("extra_mask must be (L, L) or (B, L, L)")
            X = torch.from_numpy(np.ascontiguousarray(em, np.uint8)).to(self.torch_device)
            N.check(self._lib.tav2_forward_masked(self._ctx, self._mode(mode), N.ptr(F), N.ptr(m), N.ptr(X),
                                                  int(em.ndim == 3), B, N.ptr(U), self.stream()))
        return U.cpu().numpy()

    @_locked
    def rank_requests(self, requests, mode: str = "bf16", return_indices: bool = False):
        """Host-to-host rank over (user, candidates, ctx) requests -> logits [N, 4]
        (request order kept).  A batch beyond the capacity is split / run on
        the fallback context and counted in ``overflow_count``."""
        if self.model is None:
            raise ValidationError("no model loaded")
        requests = list(requests)
        chunks = list(self._chunks(requests))
        if len(chunks) > 1 or (chunks and chunks[0][1]):
            self.overflow_count += 1
            outs = []
            for chunk, big in chunks:
                eng = self._fallback_engine(chunk[0]) if big else self
                outs.append(eng._rank_native(chunk, mode, return_indices))
            if return_indices:
                return (np.concatenate([o[0] for o in outs]), np.concatenate([o[1] for o in outs]))
            return np.concatenate(outs)
        return self._rank_native(requests, mode, return_indices)

    def _rank_native(self, requests, mode, return_indices):
        pack = _Pack(requests)
        n = sum(len(c) for _, c, _ in requests)
        logits = np.empty((n, 4), np.float32)
        idx = np.empty((n, self.config.nn.seq_len), np.int32) if return_indices else None
        N.check(self._lib.tav2_rank(self._ctx, pack.arr, len(requests), self._mode(mode),
                                    logits.ctypes.data, N.ptr(idx), self.stream()))
        return (logits, idx) if return_indices else logits

    @_locked
    def rank_pipelined(self, batches, mode: str = "bf16", return_indices: bool = False,
                       latencies: list | None = None):
        """Serving loop (tav2_rank_submit / tav2_rank_collect): every batch of
        (user, candidates, ctx) requests is submitted -- host packing into one
        of the pinned staging slots (tav2_stage_slots), H2D copy, kernels and
        result copies all enqueued -- while up to slots - 1 earlier batches are
        still in flight, so the host work, H2D and NN kernels of batch i+1
        overlap the kernels of batch i.  Returns the list
        of logits arrays (with indices if requested) in batch order;
        `latencies` (optional list) receives each batch's submit-to-collect
        wall time in seconds."""
        if self.model is None:
            raise ValidationError("no model loaded")
        mode_i = self._mode(mode)
        out, pending = [], []
        depth = self._lib.tav2_stage_slots() - 1  # submits kept in flight beyond the newest

        def collect(p):
            slot, n, _pack, t0 = p
            logits = np.empty((n, 4), np.float32)
            idx = np.empty((n, self.config.nn.seq_len), np.int32) if return_indices else None
            N.check(self._lib.tav2_rank_collect(self._ctx, slot, logits.ctypes.data, N.ptr(idx)))
            if latencies is not None:
                latencies.append(time.perf_counter() - t0)
            out.append((logits, idx) if return_indices else logits)

        for reqs in batches:
            t0 = time.perf_counter()
            reqs = list(reqs)
            ch = list(self._chunks(reqs))
            if len(ch) > 1 or (ch and ch[0][1]):  # overflow: drain, then the counted slow path
                while pending:
                    collect(pending.pop(0))
                out.append(self.rank_requests(reqs, mode=mode, return_indices=return_indices))
                if latencies is not None:
                    latencies.append(time.perf_counter() - t0)
                continue
            pack = _Pack(reqs)
            n = sum(len(c) for _, c, _ in reqs)
            slot = ctypes.c_int32()
            N.check(self._lib.tav2_rank_submit(self._ctx, pack.arr, len(reqs), mode_i, int(return_indices),
                                               self.stream(), ctypes.byref(slot)))
            pending.append((slot.value, n, pack, t0))
            if len(pending) > depth:
                collect(pending.pop(0))
        while pending:
            collect(pending.pop(0))
        return out

    # ---- the serving loop's primitives (serving.PipelinedHandler) ----
    def fits(self, requests) -> bool:
        """True when the request list stages as one batch (no overflow path)."""
        ch = list(self._chunks(list(requests)))
        return len(ch) == 1 and not ch[0][1]

    @_locked
    def submit(self, requests, mode: str = "bf16", want_idx: bool = False) -> tuple[int, int, object]:
        """tav2_rank_submit: stage into the next free slot and enqueue the
        whole rank; returns (slot, items, keep-alive).  At most
        tav2_stage_slots() submits may be outstanding: ``wait`` + ``collect``
        a slot before it is reused."""
        if self.model is None:
            raise ValidationError("no model loaded")
        pack = _Pack(requests)
        slot = ctypes.c_int32()
        N.check(self._lib.tav2_rank_submit(self._ctx, pack.arr, len(requests), self._mode(mode), int(want_idx),
                                           self.stream(), ctypes.byref(slot)))
        return slot.value, sum(len(c) for _, c, _ in requests), pack

    def wait(self, slot: int) -> None:
        """tav2_rank_wait: block until a submitted rank finished.  Deliberately
        not under the engine lock, so another thread can submit meanwhile."""
        N.check(self._lib.tav2_rank_wait(self._ctx, int(slot)))

    @_locked
    def collect(self, slot: int, n: int, want_idx: bool = False):
        logits = np.empty((n, 4), np.float32)
        idx = np.empty((n, self.config.nn.seq_len), np.int32) if want_idx else None
        N.check(self._lib.tav2_rank_collect(self._ctx, int(slot), logits.ctypes.data, N.ptr(idx)))
        return (logits, idx) if want_idx else logits

    @_locked
    def run_staged(self, mode: str, logits: torch.Tensor | None = None) -> None:
        """Device-resident path (bench ``value``): NN + score on the staged batch."""
        N.check(self._lib.tav2_run_staged(self._ctx, self._mode(mode), N.ptr(logits), self.stream()))

    @_locked
    def score_staged(self, idx: torch.Tensor, mode: str = "bf16", pooled: bool = False):
        logits = torch.empty((self.n_items, 4), dtype=torch.float32, device=self.torch_device)
        pl = torch.empty((self.n_items, 64), dtype=torch.float32, device=self.torch_device) if pooled else None
        N.check(self._lib.tav2_score(self._ctx, self._mode(mode), N.ptr(idx), N.ptr(logits), N.ptr(pl),
                                     self.stream()))
        return (logits, pl) if pooled else logits

    def graph_info(self) -> tuple[int, bool]:
        """(captured launch-chain graphs held, capture abandoned)."""
        n, b = ctypes.c_int32(), ctypes.c_int32()
        N.check(self._lib.tav2_graph_info(self._ctx, ctypes.byref(n), ctypes.byref(b)))
        return n.value, bool(b.value)

    def last_launch_count(self) -> int:
        return int(self._lib.tav2_last_launch_count(self._ctx))

    def set_profiling(self, on: bool) -> None:
        N.check(self._lib.tav2_set_profiling(self._ctx, int(on)))

    def kernel_times(self) -> dict[str, tuple[float, int]]:
        """{kernel: (total ms, launches)} accumulated since set_profiling(True)."""
        n = 16
        names = (ctypes.c_char_p * n)()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int32 * n)()
        k = self._lib.tav2_kernel_times(self._ctx, names, ms, cnt, n)
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(min(k, n))}


# ---------------------------------------------------------------------------
# Implicit per-thread engines for the module-level functions the reference
# calls without an engine (fused_assemble(arena=None), similarity_scores,
# top_k_nn, assemble, encode_batch / forward_fused / pool(params)).  One
# engine per (thread, NNConfig, parameter object), created on first use and
# grown when a call needs more capacity -- never per call.
# ---------------------------------------------------------------------------

_TLS = threading.local()


def implicit_engine(nn: NNConfig, requests: int = 1, items: int = 1, tokens: int = 1,
                    model: RankingModel | None = None) -> Engine:
    cache = getattr(_TLS, "engines", None)
    if cache is None:
        cache = _TLS.engines = {}
    key = (nn, id(model) if model is not None else None)
    eng, ref = cache.get(key, (None, None))
    if eng is not None and model is not None and ref is not model:
        eng = None  # the id was recycled by another object
    if eng is None or not eng._fits(requests, items, tokens):
        old = eng.capacity if eng is not None else Capacity(1, 1, 1)
        cap = Capacity(max(requests, old.max_requests), max(items, old.max_items, 64),
                       max(tokens, old.max_tokens, 16896))
        if eng is not None:
            eng.close()
        cfg = model.config if model is not None else ModelConfig.for_nn(nn)
        eng = Engine(model, config=cfg, capacity=cap, device=torch.cuda.current_device())
        cache[key] = (eng, model)
    return eng
