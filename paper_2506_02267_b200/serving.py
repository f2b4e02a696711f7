"""The serving entry point: ``rank()``, which the reference
specifies but never ships, composed as the reference's serving-optimised
path build_dedup_batch -> fused_assemble -> encode_batch -> forward_fused ->
pool -> head (trainer.py:354-366), executed on the B200.

Also the nearest-rank percentile of ``serving/stats.py:36-45`` used for the
p50/p99 request latencies, and a ``DynamicBatcher`` handler adapter
(batcher.py:87, :140) so the GPU rank plugs into the reference batcher.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

import threading

from .core import IMPRESSION_CAP, LIFELONG_CAP, REALTIME_CAP, TokenBlock, UserSequences
from .dataset import HEAD_NAMES, context_features, read_store
from .model import HeadConfig
from .runtime import Engine, StoreUser


@dataclass
class RankResponse:
    """Per-candidate head probabilities + final score, candidate order kept."""

    item_ids: np.ndarray
    logits: np.ndarray      # (n, 4) f32 pre-sigmoid
    probs: np.ndarray       # (n, 4) f32
    final: np.ndarray       # (n,) f64 utility-weighted score (evaluation.py:35-37)
    cold_start: bool = False
    nn_indices: np.ndarray | None = field(default=None, repr=False)

    def heads(self, i: int) -> dict[str, float]:
        return {h: float(self.probs[i, j]) for j, h in enumerate(HEAD_NAMES)}


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Stable split-form sigmoid (trainer.py:230-236)."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def _response(ids, logits, heads: HeadConfig, cold, idx=None) -> RankResponse:
    probs = sigmoid(logits)
    final = probs.astype(np.float64) @ np.asarray(heads.utility_weights, np.float64)
    return RankResponse(np.asarray(ids), logits, probs, final, cold, idx)


def rank(engine: Engine, user_id: int, user: UserSequences | None, candidates: np.ndarray,
         item_ids=None, mode: str = "bf16", log_nn_features: bool = False) -> RankResponse:
    """Score one request.  An unknown user (``user is None``) is served with
    empty sequences and flagged cold-start."""
    cold = user is None
    user = UserSequences() if cold else user
    cands = np.asarray(candidates, np.float32)
    ids = np.arange(len(cands), dtype=np.uint64) if item_ids is None else item_ids
    ctx = context_features(user_id, engine.config.ctx_dim)
    out = engine.rank_requests([(user, cands, ctx)], mode=mode, return_indices=log_nn_features)
    logits, idx = out if log_nn_features else (out, None)
    return _response(ids, logits, engine.config.heads, cold, idx)


def rank_many(engine: Engine, requests, mode: str = "bf16") -> list[RankResponse]:
    """Co-batched rank of several (user_id, user|None|StoreUser, candidates)
    requests; results are independent of co-batching."""
    packed = []
    for uid, user, cands in requests:
        packed.append((UserSequences() if user is None else user, np.asarray(cands, np.float32),
                       context_features(uid, engine.config.ctx_dim)))
    logits = engine.rank_requests(packed, mode=mode)
    out, o = [], 0
    for (uid, user, cands) in requests:
        n = len(cands)
        out.append(_response(np.arange(n, dtype=np.uint64), logits[o:o + n], engine.config.heads,
                             user is None))
        o += n
    return out


def _truncate(block: TokenBlock, cap: int) -> TokenBlock:
    """Keep the newest `cap` tokens (store.py:19-22; blocks are newest-first)."""
    return block if len(block) <= cap else block.take(np.arange(cap))


class DeviceFeatureStore:
    """FeatureStore (serving/store.py:25-72) whose users also live in HBM:
    ``put`` uploads the (cap-truncated) sequences once into the engine's
    resident pool (tav2_store_put), and requests for a stored user stage only
    their candidates -- the user's tokens are copied device to device.
    Writes replace a user wholesale; staging and writes are ordered on the
    engine's copy stream, so a ranked batch sees one consistent snapshot."""

    def __init__(self, engine: Engine, max_users: int, ll_cap: int = LIFELONG_CAP,
                 rt_cap: int = REALTIME_CAP, imp_cap: int = IMPRESSION_CAP):
        self.engine = engine
        self._users: dict[int, UserSequences] = {}
        self._lock = threading.Lock()
        self._caps = (ll_cap, rt_cap, imp_cap)
        self.generation = 0
        engine.store_reserve(max_users)

    def put(self, user_id: int, seqs: UserSequences) -> None:
        """Insert or replace a user; sequences beyond the caps keep only their
        most recent tokens (store.py:41-53)."""
        ll_cap, rt_cap, imp_cap = self._caps
        seqs = UserSequences(_truncate(seqs.lifelong, ll_cap), _truncate(seqs.realtime, rt_cap),
                             _truncate(seqs.impression, imp_cap))
        seqs.validate(ll_cap, rt_cap, imp_cap)
        with self._lock:
            self.engine.store_put(user_id, seqs)
            self._users[user_id] = seqs
            self.generation += 1

    def remove(self, user_id: int) -> None:
        with self._lock:
            self.engine.store_remove(user_id)
            del self._users[user_id]
            self.generation += 1

    def get(self, user_id: int) -> UserSequences | None:
        return self._users.get(user_id)

    def ref(self, user_id: int) -> StoreUser | None:
        """The request-side handle of a stored user (None if absent)."""
        return StoreUser(user_id) if user_id in self._users else None

    def __contains__(self, user_id: int) -> bool:
        return user_id in self._users

    def __len__(self) -> int:
        return len(self._users)

    def load(self, path) -> int:
        """Bulk-load a `.tav2` store file; returns the user count (store.py:59-64)."""
        users = read_store(path)
        for user_id, seqs in users:
            self.put(user_id, seqs)
        return len(users)

    @classmethod
    def from_pairs(cls, engine: Engine, max_users: int, pairs, **kwargs) -> "DeviceFeatureStore":
        store = cls(engine, max_users, **kwargs)
        for user_id, seqs in pairs:
            store.put(user_id, seqs)
        return store


def batcher_handler(engine: Engine, store, mode: str = "bf16"):
    """Adapter for ``DynamicBatcher(cfg, handler)``: each Pending payload is
    ``(user_id, candidates)``; users come from ``store.get`` (store.py:54) --
    or, for a DeviceFeatureStore, straight from HBM."""

    def user_of(uid):
        if isinstance(store, DeviceFeatureStore):
            return store.ref(uid)
        return store.get(uid)

    def handler(batch, worker_index):  # noqa: ARG001 - batcher contract
        reqs = [(uid, user_of(uid), cands) for uid, cands in (p.payload for p in batch)]
        for p, r in zip(batch, rank_many(engine, reqs, mode=mode)):
            p.set_result(r)

    return handler


def nearest_rank(values, p: float) -> float | None:
    """Nearest-rank percentile, rank = ceil(p/100 * n) (stats.py:36-45)."""
    v = sorted(values)
    if not v:
        return None
    r = max(1, int(math.ceil(p * len(v) / 100.0)))
    return v[min(r, len(v)) - 1]
