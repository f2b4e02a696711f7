"""Candidate-anchored NN selection: configuration, the assembled-sequence
types, the de-duplicated request batch and the GPU ``fused_assemble``.

Public names follow ``seqrank.nnsearch`` (nnsearch.py:22-369).  The
selection itself runs on the B200 (``tav2_nn_select``; the per-item helpers
``similarity_scores`` / ``top_k_nn`` / ``assemble`` too, through
``tav2_similarity`` and the same selection kernels); this module builds the
request batch and turns the device index layout back into
``AssembledSequence`` objects when a caller asks for them.  Functions that
the reference calls without an engine (its ``arena=None``) use a per-thread
implicit engine (``runtime.implicit_engine``), created once and reused.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import EMBED_DIM, TokenBlock, UserSequences, ValidationError

SEGMENT_NAMES = ("nn_lifelong", "recent_realtime", "nn_realtime_tail", "nn_impression")
MAX_SEGMENT_K = 256  # per-segment k of the device selection (kMaxK, tav2_common.cuh)


@dataclass(frozen=True)
class NNConfig:
    """Segment budget (nnsearch.py:25-46)."""

    recent: int = 32
    k_lifelong: int = 96
    k_realtime: int = 32
    k_impression: int = 32

    @property
    def seq_len(self) -> int:
        return self.recent + self.k_lifelong + self.k_realtime + self.k_impression

    def segment_lengths(self) -> tuple[int, int, int, int]:
        return (self.k_lifelong, self.recent, self.k_realtime, self.k_impression)

    def segment_starts(self) -> tuple[int, int, int, int]:
        lens = self.segment_lengths()
        return (0, lens[0], lens[0] + lens[1], lens[0] + lens[1] + lens[2])

    def validate(self) -> None:
        if min(self.recent, self.k_lifelong, self.k_realtime, self.k_impression) < 0:
            raise ValidationError("segment lengths must be non-negative")
        if self.seq_len == 0:
            raise ValidationError("assembled sequence length must be positive")


@dataclass(frozen=True)
class Segment:
    name: str
    start: int
    stop: int
    valid: int


@dataclass
class AssembledSequence:
    """Padded model input (nnsearch.py:58-80)."""

    block: TokenBlock
    mask: np.ndarray
    segments: tuple[Segment, ...]

    def __len__(self) -> int:
        return len(self.block)

    def segment(self, name: str) -> Segment:
        for seg in self.segments:
            if seg.name == name:
                return seg
        raise KeyError(name)

    def equals(self, other: "AssembledSequence") -> bool:
        return (self.block.equals(other.block) and np.array_equal(self.mask, other.mask)
                and self.segments == other.segments)


@dataclass
class DedupBatch:
    """Request-level features stored once + per-item offsets (nnsearch.py:188-211)."""

    users: list[UserSequences]
    offsets: np.ndarray       # (n_items,) int32
    candidates: np.ndarray    # (n_items, E) float32
    item_ids: np.ndarray      # (n_items,) uint64

    def __len__(self) -> int:
        return len(self.offsets)

    def validate(self) -> None:
        n = len(self.offsets)
        if not (len(self.candidates) == len(self.item_ids) == n):
            raise ValidationError("item columns disagree on length")
        if n and (self.offsets.min() < 0 or self.offsets.max() >= len(self.users)):
            raise ValidationError("offset out of range")
        if len(np.unique(self.offsets)) != len(self.users):
            raise ValidationError("every unique request must be referenced")

    def grouped_order(self) -> np.ndarray:
        """Item permutation that groups items by request, keeping their
        order within a request (identity for a build_dedup_batch batch).
        The device stages requests contiguously; results are scattered back
        through this permutation, so interleaved offsets -- which the
        reference accepts (nnsearch.py:307-308) -- give the same per-item
        results."""
        return np.argsort(self.offsets, kind="stable")

    def request_slices(self) -> list[slice]:
        """Slices of the grouped item order (``grouped_order``) per request."""
        bounds = np.searchsorted(np.sort(self.offsets, kind="stable"), np.arange(len(self.users) + 1))
        return [slice(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]


def build_dedup_batch(requests) -> DedupBatch:
    """(user, candidates[M,E], item_ids|None) requests -> DedupBatch
    (nnsearch.py:214-244); item order is preserved."""
    if not requests:
        raise ValidationError("at least one request required")
    users, offsets, cands, ids = [], [], [], []
    for user, candidates, item_ids in requests:
        candidates = np.asarray(candidates, dtype=np.float32)
        if candidates.ndim != 2 or len(candidates) == 0:
            raise ValidationError("each request needs a non-empty (M, E) candidate array")
        if item_ids is None:
            item_ids = np.arange(len(candidates), dtype=np.uint64)
        users.append(user)
        offsets.append(np.full(len(candidates), len(users) - 1, np.int32))
        cands.append(candidates)
        ids.append(np.asarray(item_ids, dtype=np.uint64))
    batch = DedupBatch(users, np.concatenate(offsets), np.ascontiguousarray(np.concatenate(cands)),
                       np.concatenate(ids))
    batch.validate()
    return batch


def sequence_feature_bytes(user: UserSequences, embed_dim: int = EMBED_DIM) -> int:
    """Wire bytes of one request's sequences (nnsearch.py:247-249)."""
    return user.total_tokens() * (7 + embed_dim)


def dedup_sequence_bytes(batch: DedupBatch) -> int:
    return sum(sequence_feature_bytes(u) for u in batch.users)


def broadcast_sequence_bytes(batch: DedupBatch) -> int:
    per = [sequence_feature_bytes(u) for u in batch.users]
    return int(sum(per[o] for o in batch.offsets))


def assembled_from_indices(user: UserSequences, idx_row: np.ndarray, cfg: NNConfig) -> AssembledSequence:
    """Materialise one ``AssembledSequence`` from a device index row
    (source-relative indices, -1 padding; layout of nnsearch.py:153-180)."""
    S = cfg.seq_len
    ts = np.zeros(S, np.uint32)
    act = np.zeros(S, np.uint16)
    surf = np.zeros(S, np.uint8)
    emb = np.zeros((S, EMBED_DIM), np.int8)
    mask = idx_row >= 0
    segments = []
    sources = (user.lifelong, user.realtime, user.realtime, user.impression)
    for name, start, length, blk in zip(SEGMENT_NAMES, cfg.segment_starts(), cfg.segment_lengths(),
                                        sources):
        sl = slice(start, start + length)
        sel = idx_row[sl]
        valid = int(np.count_nonzero(sel >= 0))
        if valid:
            ii = sel[:valid]
            ts[start:start + valid] = blk.timestamps[ii]
            act[start:start + valid] = blk.actions[ii]
            surf[start:start + valid] = blk.surfaces[ii]
            emb[start:start + valid] = blk.embeddings[ii]
        segments.append(Segment(name, start, start + length, valid))
    return AssembledSequence(TokenBlock(ts, act, surf, emb), mask, tuple(segments))


def _engine_for(cfg: NNConfig, batch: DedupBatch, engine=None, arena=None):
    from .runtime import Engine, implicit_engine

    eng = engine if engine is not None else arena if isinstance(arena, Engine) else None
    if eng is None:
        toks = sum(u.total_tokens() for u in batch.users)
        return implicit_engine(cfg, requests=len(batch.users), items=len(batch), tokens=max(toks, 1))
    if eng.nn_cfg != cfg:
        raise ValidationError("engine NNConfig differs from the requested one")
    return eng


def fused_assemble(batch: DedupBatch, cfg: NNConfig, arena=None, return_scores: bool = False,
                   engine=None, mode: str = "bf16"):
    """GPU ``fused_assemble`` (nnsearch.py:289-369).

    ``engine`` is a :class:`paper_2506_02267_b200.runtime.Engine` (the
    per-worker native context, standing in for the reference's ``arena``);
    without one the calling thread's implicit engine for ``cfg`` is used.
    Returns one AssembledSequence per item (item order kept, interleaved
    offsets allowed) and, when asked, per item ``{segment: f64 scores best
    first}`` -- the reference's float64 dots (nnsearch.py:362-363).
    """
    cfg.validate()
    batch.validate()
    eng = _engine_for(cfg, batch, engine, arena)
    idx, scores = eng.nn_select(batch, mode=mode, return_scores=True)
    out = [assembled_from_indices(batch.users[o], idx[i], cfg) for i, o in enumerate(batch.offsets)]
    if not return_scores:
        return out
    per_item = []
    for i in range(len(batch)):
        d = {}
        for name, start, length in zip(SEGMENT_NAMES, cfg.segment_starts(), cfg.segment_lengths()):
            if name == "recent_realtime" or length == 0:
                continue
            sel = idx[i, start:start + length]
            v = int(np.count_nonzero(sel >= 0))
            if v == 0:
                continue
            sc = scores[i, start:start + v]
            order = np.lexsort((sel[:v], -sc))  # best first, ties -> lower index (stable argsort)
            d[name] = sc[order]
        per_item.append(d)
    return out, per_item


def similarity_scores(block: TokenBlock, candidate: np.ndarray, engine=None) -> np.ndarray:
    """f64 score of every token of `block` against `candidate` (nnsearch.py:83-90),
    computed on the GPU (tav2_similarity)."""
    from .runtime import implicit_engine

    if len(block) == 0:
        return np.zeros(0, dtype=np.float64)
    user = UserSequences(block, TokenBlock.empty(), TokenBlock.empty())
    cand = np.asarray(candidate, np.float32).reshape(1, -1)
    eng = engine if engine is not None else implicit_engine(
        NNConfig(recent=0, k_lifelong=1, k_realtime=0, k_impression=0), requests=1, items=1, tokens=len(block))
    return eng.similarity(user, cand, source=0)


def top_k_nn(block: TokenBlock, candidate: np.ndarray, k: int, return_scores: bool = False, engine=None):
    """Indices of the k highest-similarity tokens, best first, ties to the
    smaller index (nnsearch.py:93-112): the GPU selection (tav2_nn_select)
    over a one-source request; all indices when the block is shorter."""
    from .runtime import implicit_engine

    if k < 0:
        raise ValidationError("k must be non-negative")
    if k == 0 or len(block) == 0:
        z = np.zeros(0, np.intp)
        return (z, np.zeros(0, np.float64)) if return_scores else z
    kk = min(k, len(block))
    if kk > MAX_SEGMENT_K:  # beyond the selection kernels' segment budget: order the GPU scores
        s = similarity_scores(block, candidate, engine=engine)
        picked = np.argsort(-s, kind="stable")[:kk]
        return (picked, s[picked]) if return_scores else picked
    cfg = NNConfig(recent=0, k_lifelong=kk, k_realtime=0, k_impression=0)
    user = UserSequences(block, TokenBlock.empty(), TokenBlock.empty())
    batch = build_dedup_batch([(user, np.asarray(candidate, np.float32).reshape(1, -1), None)])
    eng = engine if engine is not None else implicit_engine(cfg, requests=1, items=1, tokens=len(block))
    idx, sc = eng.nn_select(batch, return_scores=True)
    sel, s = idx[0, :kk], sc[0, :kk]
    order = np.lexsort((sel, -s))
    picked = sel[order].astype(np.intp)
    return (picked, s[order]) if return_scores else picked


def assemble(user: UserSequences, candidate: np.ndarray, cfg: NNConfig, engine=None) -> AssembledSequence:
    """One (user, candidate) model input (nnsearch.py:121-150): the fused GPU
    selection on a one-item batch (identical to the reference's per-item
    path, which fused_assemble matches token for token)."""
    cfg.validate()
    batch = build_dedup_batch([(user, np.asarray(candidate, np.float32).reshape(1, -1), None)])
    return fused_assemble(batch, cfg, engine=engine)[0]
