"""``seqrank.trainer`` names on the serving side: the model types and the
forward pass over a batch (trainer.py:42-161, :170-176, :338-374).

``model_forward`` runs on the B200: the fused gather + Eq. 4 encode + SKUT +
pool + CTR head kernel (tav2_score, the ranking path) gives the logits and
pooled vectors, and the encoder outputs ``u`` come from tav2_encode +
tav2_forward.  Training (loss, backward, optimisers, NAL) is not on the
serving path: ``ForwardState.cache`` holds the forward values a caller can
inspect, not the reference's backward caches.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import UserSequences, ValidationError
from .model import HeadConfig, HeadParams, ModelConfig, RankingModel  # noqa: F401
from .serving import sigmoid


@dataclass
class TrainBatch:
    """trainer.py:170-175."""

    assembled: list
    candidates: np.ndarray  # (B, E) float32
    labels: np.ndarray      # (B, H) uint8
    contexts: np.ndarray    # (B, ctx_dim) float32
    users: list[UserSequences]


@dataclass
class ForwardState:
    """trainer.py:338-342."""

    probs: np.ndarray  # (B, H)
    u: np.ndarray      # (B, L, d)
    mask: np.ndarray
    cache: dict | None


def model_forward(model: RankingModel, batch: TrainBatch, want_cache: bool = True, engine=None,
                  mode: str = "fp32") -> ForwardState:
    """Encode -> transformer -> masked max-pool -> CTR head -> sigmoid
    (trainer.py:345-374) on the GPU.  ``mode`` "fp32" (default, within 1e-5 of
    the reference's logits) or "bf16"."""
    from .encoder import _engine, _nn_of

    if not batch.assembled:
        raise ValidationError("empty batch")
    if engine is None:
        toks = int(sum(np.count_nonzero(s.mask) for s in batch.assembled))
        nn = _nn_of(batch.assembled)
        if nn != model.config.nn:
            raise ValidationError("assembled layout differs from the model's NNConfig")
        from .runtime import implicit_engine

        B = len(batch.assembled)
        engine = implicit_engine(nn, requests=B, items=B, tokens=max(toks, 1), model=model)
    cands = np.asarray(batch.candidates, np.float32)
    ctx = np.asarray(batch.contexts, np.float32)
    logits, pooled = engine.score_assembled(batch.assembled, cands, ctx, mode=mode)
    features, mask = engine.encode(batch.assembled, cands)
    u = engine.forward(features, mask, mode=mode)
    probs = sigmoid(logits)
    cache = dict(u=u, features=features, pooled=pooled, logits=logits) if want_cache else None
    return ForwardState(probs, u, mask, cache)
