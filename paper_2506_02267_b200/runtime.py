"""Per-worker engine: one native tav2 context (pinned staging arena + device
workspace, the B200 analogue of ``serving/arena.py``'s per-worker Arena)
holding one immutable model.

PyTorch is used only as plumbing: device buffers and the CUDA stream.  All
compute runs in ``libtav2.so``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
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
    """One native worker context (never share across threads, arena.py:17)."""

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
    def store_reserve(self, max_users: int) -> None:
        """(Re)allocate the device pool for max_users users (drops all)."""
        N.check(self._lib.tav2_store_reserve(self._ctx, int(max_users)))

    def store_put(self, user_id: int, user: UserSequences) -> None:
        """Insert or replace a user's sequences in HBM (lengths within the caps)."""
        r, keep = N.Request(), []
        _columns(user, r, keep)
        N.check(self._lib.tav2_store_put(self._ctx, int(user_id), ctypes.byref(r)))

    def store_remove(self, user_id: int) -> None:
        N.check(self._lib.tav2_store_remove(self._ctx, int(user_id)))

    def store_count(self) -> int:
        return int(self._lib.tav2_store_count(self._ctx))

    def stage(self, requests) -> int:
        """requests: list of (UserSequences | StoreUser, candidates[M,32], ctx[8] | None)."""
        pack = _Pack(requests)
        n = ctypes.c_int32()
        N.check(self._lib.tav2_stage(self._ctx, pack.arr, len(requests), self.stream(),
                                     ctypes.byref(n)))
        self.n_items = n.value
        return n.value

    def stage_batch(self, batch: DedupBatch, contexts=None) -> int:
        batch.validate()
        reqs = []
        for r, sl in enumerate(batch.request_slices()):
            ctx = None if contexts is None else contexts[r]
            reqs.append((batch.users[r], batch.candidates[sl], ctx))
        return self.stage(reqs)

    def _mode(self, mode: str) -> int:
        try:
            return N.MODES[mode]
        except KeyError:
            raise ValidationError(f"unknown precision mode {mode!r} (fp32 | bf16)") from None

    # ------------------------------------------------------------------
    def nn_select(self, batch: DedupBatch, mode: str = "bf16", return_scores: bool = False):
        """Device NN selection over a DedupBatch -> idx [N, S] int32 (-1 pad)."""
        n = self.stage_batch(batch)
        S = self.config.nn.seq_len
        idx = torch.empty((n, S), dtype=torch.int32, device=self.torch_device)
        sc = torch.empty((n, S), dtype=torch.float32, device=self.torch_device) if return_scores else None
        N.check(self._lib.tav2_nn_select(self._ctx, self._mode(mode), N.ptr(idx), N.ptr(sc),
                                         self.stream()))
        idx_h = idx.cpu().numpy()
        if return_scores:
            return idx_h, sc.cpu().numpy()
        return idx_h

    def encode(self, seqs: list[AssembledSequence], candidates: np.ndarray):
        """encode_batch (encoder.py:161-188) on the GPU -> (F [B,S,64], mask [B,S])."""
        if self.model is None:
            raise ValidationError("no model loaded")
        cfg = self.config.nn
        S = cfg.seq_len
        if any(len(s) != S for s in seqs):
            raise ValidationError("assembled length must match the positional table")
        starts, lens = cfg.segment_starts(), cfg.segment_lengths()
        reqs, idx = [], np.full((len(seqs), S), -1, np.int32)
        from .core import TokenBlock

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
            reqs.append((user, np.asarray(candidates[i:i + 1], np.float32), None))
        n = self.stage(reqs)
        idx_d = torch.from_numpy(idx).to(self.torch_device)
        F = torch.empty((n, S, 2 * EMBED_DIM), dtype=torch.float32, device=self.torch_device)
        m = torch.empty((n, S), dtype=torch.uint8, device=self.torch_device)
        N.check(self._lib.tav2_encode(self._ctx, N.ptr(idx_d), N.ptr(F), N.ptr(m), self.stream()))
        return F.cpu().numpy(), m.cpu().numpy().astype(bool)

    def forward(self, features: np.ndarray, mask: np.ndarray, mode: str = "fp32") -> np.ndarray:
        """forward_fused over caller features (B, S, 64) -> U (valid rows)."""
        if self.model is None:
            raise ValidationError("no model loaded")
        B, S, d = features.shape
        if S != self.config.nn.seq_len or d != 2 * EMBED_DIM:
            raise ValidationError("feature shape does not match the model")
        F = torch.from_numpy(np.ascontiguousarray(features, np.float32)).to(self.torch_device)
        m = torch.from_numpy(np.ascontiguousarray(mask, np.uint8)).to(self.torch_device)
        U = torch.empty_like(F)
        N.check(self._lib.tav2_forward(self._ctx, self._mode(mode), N.ptr(F), N.ptr(m), B, N.ptr(U),
                                       self.stream()))
        return U.cpu().numpy()

    def rank_requests(self, requests, mode: str = "bf16", return_indices: bool = False):
        """Host-to-host rank over (user, candidates, ctx) requests -> logits [N, 4]."""
        if self.model is None:
            raise ValidationError("no model loaded")
        pack = _Pack(requests)
        n = sum(len(c) for _, c, _ in requests)
        logits = np.empty((n, 4), np.float32)
        idx = np.empty((n, self.config.nn.seq_len), np.int32) if return_indices else None
        N.check(self._lib.tav2_rank(self._ctx, pack.arr, len(requests), self._mode(mode),
                                    logits.ctypes.data, N.ptr(idx), self.stream()))
        return (logits, idx) if return_indices else logits

    def rank_pipelined(self, batches, mode: str = "bf16", return_indices: bool = False,
                       latencies: list | None = None):
        """Serving loop (tav2_rank_submit / tav2_rank_collect): every batch of
        (user, candidates, ctx) requests is submitted -- host packing into one
        of two pinned staging slots, H2D copy, kernels and result copies all
        enqueued -- before the previous batch is collected, so the host work
        and H2D of batch i+1 overlap the kernels of batch i.  Returns the list
        of logits arrays (with indices if requested) in batch order;
        `latencies` (optional list) receives each batch's submit-to-collect
        wall time in seconds."""
        if self.model is None:
            raise ValidationError("no model loaded")
        mode_i = self._mode(mode)
        out, pending = [], None

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
            pack = _Pack(reqs)
            n = sum(len(c) for _, c, _ in reqs)
            slot = ctypes.c_int32()
            N.check(self._lib.tav2_rank_submit(self._ctx, pack.arr, len(reqs), mode_i, int(return_indices),
                                               self.stream(), ctypes.byref(slot)))
            if pending is not None:
                collect(pending)
            pending = (slot.value, n, pack, t0)
        if pending is not None:
            collect(pending)
        return out

    def run_staged(self, mode: str, logits: torch.Tensor | None = None) -> None:
        """Device-resident path (bench ``value``): NN + score on the staged batch."""
        N.check(self._lib.tav2_run_staged(self._ctx, self._mode(mode), N.ptr(logits), self.stream()))

    def score_staged(self, idx: torch.Tensor, mode: str = "bf16", pooled: bool = False):
        logits = torch.empty((self.n_items, 4), dtype=torch.float32, device=self.torch_device)
        pl = torch.empty((self.n_items, 64), dtype=torch.float32, device=self.torch_device) if pooled else None
        N.check(self._lib.tav2_score(self._ctx, self._mode(mode), N.ptr(idx), N.ptr(logits), N.ptr(pl),
                                     self.stream()))
        return (logits, pl) if pooled else logits

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
