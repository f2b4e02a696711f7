"""Head names, request context features and a vectorised synthetic request
generator with the structure of ``seqrank.dataset.generate_synthetic``
(dataset.py:297-427): per-user interest clusters, 15% HIDE tokens from
foreign clusters, 10% multi-hot positives, impressions 75% foreign, unit
f32 candidates half near / half far.  Values differ from the reference's
per-token Python loop (this one is ~1000x faster); the distribution is the
same, which is all the benchmark needs.
"""

from __future__ import annotations

from dataclasses import dataclass

import functools

import numpy as np

from .core import (CLICK, CLOSEUP, EMBED_DIM, HIDE, IMPRESSION, REPIN, TokenBlock, UserSequences,
                   ValidationError, quantize)

HEAD_NAMES = ("repin", "click", "closeup", "hide")
NUM_HEADS = len(HEAD_NAMES)

_LL_BASE_TS = 1_700_000_000
_RT_BASE_TS = 1_750_000_000


def context_features(user_id: int, dim: int = 8) -> np.ndarray:
    """Deterministic request context in [-1, 1] (dataset.py:282-289).  A pure
    function of (user_id, dim): memoised, because seeding a Generator costs
    ~25 us -- the largest piece of a serving batch's per-request host work."""
    return _context_features(int(user_id), int(dim)).copy()


@functools.lru_cache(maxsize=1 << 16)
def _context_features(user_id: int, dim: int) -> np.ndarray:
    rng = np.random.default_rng([user_id, 96321])
    return rng.uniform(-1.0, 1.0, dim).astype(np.float32)


@dataclass
class SyntheticRequest:
    user_id: int
    user: UserSequences
    candidates: np.ndarray  # (n, 32) f32 unit rows
    ctx: np.ndarray         # (8,) f32


def _unit(x: np.ndarray) -> np.ndarray:
    n = np.linalg.norm(x, axis=-1, keepdims=True).astype(np.float32)
    return (x / np.where(n == 0, 1, n)).astype(np.float32)


def _noisy(rng, centroids, which, sigma=0.08):
    return _unit(centroids[which] + rng.normal(0.0, sigma, (len(which), EMBED_DIM)).astype(np.float32))


def _engagement(rng, n, near, far, base_ts, step) -> TokenBlock:
    ts = (base_ts - np.arange(n, dtype=np.int64) * step).astype(np.uint32)
    surf = rng.integers(0, 4, n).astype(np.uint8)
    hide = rng.random(n) < 0.15
    pos = rng.choice(np.array([REPIN, CLICK, CLOSEUP], np.uint16), n)
    extra = np.where(rng.random(n) < 0.1, rng.choice(np.array([REPIN, CLOSEUP], np.uint16), n), 0)
    act = np.where(hide, HIDE, pos | extra).astype(np.uint16)
    emb = np.where(hide[:, None], far(n), near(n))
    return TokenBlock(ts, act, surf, quantize(emb))


def _impressions(rng, n, near, far) -> TokenBlock:
    ts = (_RT_BASE_TS + 30 - np.arange(n, dtype=np.int64) * 60).astype(np.uint32)
    surf = rng.integers(0, 4, n).astype(np.uint8)
    emb = np.where((rng.random(n) < 0.75)[:, None], far(n), near(n))
    return TokenBlock(ts, np.full(n, IMPRESSION, np.uint16), surf, quantize(emb))


def generate_requests(num_requests: int, n_candidates: int, ll_tokens: int = 16384,
                      rt_tokens: int = 256, imp_tokens: int = 256, num_clusters: int = 8,
                      seed: int = 0) -> list[SyntheticRequest]:
    """Synthetic serving requests: one user + N candidates each."""
    rng = np.random.default_rng(seed)
    centroids = _unit(rng.normal(0.0, 1.0, (num_clusters, EMBED_DIM)).astype(np.float32))
    out = []
    for r in range(num_requests):
        uid = r + 1
        k = int(rng.integers(1, min(3, num_clusters) + 1))
        interests = rng.choice(num_clusters, k, replace=False)
        foreign = np.setdiff1d(np.arange(num_clusters), interests)

        def near(n, _i=interests):
            return _noisy(rng, centroids, rng.choice(_i, n))

        def far(n, _f=foreign):
            if len(_f) == 0:
                return _unit(rng.normal(0, 1, (n, EMBED_DIM)).astype(np.float32))
            return _noisy(rng, centroids, rng.choice(_f, n))

        user = UserSequences(_engagement(rng, ll_tokens, near, far, _LL_BASE_TS, 3600),
                             _engagement(rng, rt_tokens, near, far, _RT_BASE_TS, 60),
                             _impressions(rng, imp_tokens, near, far))
        is_near = rng.random(n_candidates) < 0.5
        cands = np.where(is_near[:, None], near(n_candidates), far(n_candidates)).astype(np.float32)
        out.append(SyntheticRequest(uid, user, np.ascontiguousarray(cands), context_features(uid)))
    return out


# ---------------------------------------------------------------------------
# The reference generator itself (dataset.py:297-427), draw for draw: the
# same Generator calls in the same order, so a seed gives bit-identical
# users and candidates (pinned against the live reference by
# oracle/gen_c2_golden.py -> tests/golden/c2_seed0.npz).  It is a per-token
# Python loop like the reference (~1 s per 16k-token user); the benchmark and
# the shape tests use it so their inputs are the reference's.
# ---------------------------------------------------------------------------


@dataclass
class SyntheticConfig:
    """dataset.py:296-321."""

    num_users: int = 100
    num_clusters: int = 8
    ll_tokens: int = 128
    rt_tokens: int = 48
    imp_tokens: int = 48
    positive_rate: float = 0.9
    hide_rate: float = 0.9
    chunks_per_user: int = 2
    chunk_size: int = 8
    seed: int = 0

    def validate(self) -> None:
        if min(self.num_users, self.num_clusters, self.ll_tokens, self.rt_tokens, self.imp_tokens,
               self.chunks_per_user, self.chunk_size) < 1:
            raise ValidationError("all synthetic counts must be >= 1")
        if not (0.0 <= self.positive_rate <= 1.0 and 0.0 <= self.hide_rate <= 1.0):
            raise ValidationError("rates must lie in [0, 1]")


@dataclass
class TrainingExample:
    """One labelled (user, candidate) pair (dataset.py:179-203)."""

    user_id: int
    chunk_id: int
    candidate: np.ndarray
    labels: np.ndarray
    nn_features: object = None


@dataclass
class SyntheticData:
    users: list
    examples: list
    centroids: np.ndarray


def _unit_vec(e: np.ndarray) -> np.ndarray:
    """The reference's per-vector l2_normalize (core.py:60-66): f32 dot,
    float sqrt, one f32 division (bit-for-bit, unlike the row-wise form)."""
    e = np.asarray(e, dtype=np.float32)
    nrm = float(np.sqrt(np.dot(e, e)))
    return e.copy() if nrm == 0.0 else e / np.float32(nrm)


def generate_synthetic(cfg: SyntheticConfig) -> SyntheticData:
    """Users with 1-3 interest clusters, engagement / impression blocks and
    labelled candidate chunks, drawn exactly as dataset.py:335-427 does."""
    cfg.validate()
    rng = np.random.default_rng(cfg.seed)
    normal, random, choice, integers = rng.normal, rng.random, rng.choice, rng.integers
    centroids = normal(0.0, 1.0, (cfg.num_clusters, EMBED_DIM)).astype(np.float32)
    centroids = np.stack([_unit_vec(c) for c in centroids])
    pos3 = (REPIN, CLICK, CLOSEUP)
    pos2 = (REPIN, CLOSEUP)
    users, examples, chunk_id = [], [], 0
    for uid in range(1, cfg.num_users + 1):
        k = int(integers(1, min(3, cfg.num_clusters) + 1))
        interests = choice(cfg.num_clusters, k, replace=False)
        foreign = np.setdiff1d(np.arange(cfg.num_clusters), interests)

        def near(_i=interests):
            c = centroids[int(choice(_i))]
            return _unit_vec(c + normal(0.0, 0.08, EMBED_DIM).astype(np.float32))

        def far(_f=foreign):
            if len(_f) == 0:
                return _unit_vec(normal(0.0, 1.0, EMBED_DIM).astype(np.float32))
            c = centroids[int(choice(_f))]
            return _unit_vec(c + normal(0.0, 0.08, EMBED_DIM).astype(np.float32))

        def engagement(n, base_ts, step):
            ts = base_ts - np.arange(n, dtype=np.int64) * step
            act = np.zeros(n, np.uint16)
            surf = integers(0, 4, n).astype(np.uint8)
            emb = np.zeros((n, EMBED_DIM), np.int8)
            for i in range(n):
                if random() < 0.15:
                    act[i] = HIDE
                    emb[i] = quantize(far())
                else:
                    a = int(choice(pos3))
                    if random() < 0.1:  # multi-hot pair
                        a |= int(choice(pos2))
                    act[i] = a
                    emb[i] = quantize(near())
            return TokenBlock(ts, act, surf, emb)

        def impressions(n):
            ts = _RT_BASE_TS + 30 - np.arange(n, dtype=np.int64) * 60
            surf = integers(0, 4, n).astype(np.uint8)
            emb = np.zeros((n, EMBED_DIM), np.int8)
            for i in range(n):
                emb[i] = quantize(far() if random() < 0.75 else near())
            return TokenBlock(ts, np.full(n, IMPRESSION, np.uint16), surf, emb)

        seqs = UserSequences(engagement(cfg.ll_tokens, _LL_BASE_TS, 3600),
                             engagement(cfg.rt_tokens, _RT_BASE_TS, 60), impressions(cfg.imp_tokens))
        seqs.validate()
        users.append((uid, seqs))
        for _ in range(cfg.chunks_per_user):
            chunk_id += 1
            for _ in range(cfg.chunk_size):
                labels = np.zeros(NUM_HEADS, np.uint8)
                if random() < 0.5:
                    emb = near()
                    labels[0] = random() < cfg.positive_rate
                    labels[1] = random() < cfg.positive_rate * 0.7
                    labels[2] = random() < cfg.positive_rate * 0.5
                else:
                    emb = far()
                    labels[3] = random() < cfg.hide_rate
                examples.append(TrainingExample(uid, chunk_id, emb, labels))
    return SyntheticData(users, examples, centroids)


def synthetic_requests(num_requests: int, n_candidates: int, ll_tokens: int = 16384,
                       rt_tokens: int = 256, imp_tokens: int = 256, seed: int = 0) -> list[SyntheticRequest]:
    """Serving requests from the reference generator: request
    i is ``generate_synthetic(num_users=1, num_clusters=8, L, 256, 256,
    chunks_per_user=1, chunk_size=N, seed=seed + i)``'s user and its N
    candidate embeddings; ctx = context_features(user id)."""
    out = []
    for i in range(num_requests):
        d = generate_synthetic(SyntheticConfig(num_users=1, num_clusters=8, ll_tokens=ll_tokens,
                                               rt_tokens=rt_tokens, imp_tokens=imp_tokens, chunks_per_user=1,
                                               chunk_size=n_candidates, seed=seed + i))
        uid, user = d.users[0]
        cands = np.ascontiguousarray(np.stack([e.candidate for e in d.examples]), np.float32)
        out.append(SyntheticRequest(uid, user, cands, context_features(uid)))
    return out


# ---------------------------------------------------------------------------
# NN-feature logging (training-serving alignment): the
# assembled sequence a request was scored with, serialised in the reference's
# record format (dataset.py:49-66 token records, :138-149 assembled block) so
# the logged bytes equal what the reference's own logger would write.
# ---------------------------------------------------------------------------

def token_record_dtype(embed_dim: int = 32) -> np.dtype:
    """One token on the wire: u32 ts, u16 action, u8 surface, embed_dim x i8."""
    return np.dtype([("ts", "<u4"), ("action", "<u2"), ("surface", "u1"), ("emb", "i1", (embed_dim,))])


def pack_token_block(block) -> bytes:
    rec = np.empty(len(block), dtype=token_record_dtype(block.embeddings.shape[1]))
    rec["ts"], rec["action"], rec["surface"], rec["emb"] = (block.timestamps, block.actions, block.surfaces,
                                                            block.embeddings)
    return rec.tobytes()


def pack_assembled(seq) -> bytes:
    """<HBB> (sequence length, embed dim, segment count), one <HH> (configured
    length, valid count) per segment, then the padded token records."""
    import struct

    head = struct.pack("<HBB", len(seq), seq.block.embeddings.shape[1], len(seq.segments))
    segs = b"".join(struct.pack("<HH", g.stop - g.start, g.valid) for g in seq.segments)
    return head + segs + pack_token_block(seq.block)


def log_nn_features(users, idx: np.ndarray, offsets, cfg) -> list[bytes]:
    """Logged records of a ranked batch: `idx` [n_items, seq_len] from
    Engine.rank_requests(..., return_indices=True) / tav2_rank(idx_host),
    `offsets[i]` the request index of item i."""
    from .nnsearch import assembled_from_indices

    return [pack_assembled(assembled_from_indices(users[o], idx[i], cfg)) for i, o in enumerate(offsets)]


# ---------------------------------------------------------------------------
# Sequence store (.tav2): bulk source of the HBM-resident feature store
# (serving.DeviceFeatureStore.load).  Byte format of dataset.py:85-131:
# <4sHQ> (magic, version, user count), then per user <QHHH> (user id,
# ll/rt/imp lengths) followed by the three packed token blocks.
# ---------------------------------------------------------------------------

STORE_MAGIC = b"TAV2"
FORMAT_VERSION = 1


class FormatError(ValueError):
    """Malformed store file; the message carries the byte offset (dataset.py:44-46)."""


def unpack_token_block(buf: bytes, offset: int, count: int, embed_dim: int = EMBED_DIM):
    dt = token_record_dtype(embed_dim)
    end = offset + count * dt.itemsize
    if end > len(buf):
        raise FormatError(f"token block truncated at byte {offset}")
    rec = np.frombuffer(buf, dtype=dt, count=count, offset=offset)
    return TokenBlock(rec["ts"], rec["action"], rec["surface"], rec["emb"]), end


def write_store(path, users) -> None:
    """Write (user_id, UserSequences) pairs; validates every record (dataset.py:90-103)."""
    import struct

    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sHQ", STORE_MAGIC, FORMAT_VERSION, len(users)))
        for user_id, seqs in users:
            seqs.validate()
            fh.write(struct.pack("<QHHH", user_id, len(seqs.lifelong), len(seqs.realtime), len(seqs.impression)))
            for blk in seqs.blocks():
                fh.write(pack_token_block(blk))


def read_store(path) -> list:
    """Read a .tav2 store back into (user_id, UserSequences) pairs (dataset.py:106-131)."""
    import struct
    from pathlib import Path

    buf = Path(path).read_bytes()
    fh, uh = struct.Struct("<4sHQ"), struct.Struct("<QHHH")
    if len(buf) < fh.size:
        raise FormatError(f"store header truncated at byte {len(buf)}")
    magic, version, count = fh.unpack_from(buf, 0)
    if magic != STORE_MAGIC:
        raise FormatError(f"bad store magic {magic!r} at byte 0")
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported store version {version} at byte 4")
    users, pos = [], fh.size
    for _ in range(count):
        if pos + uh.size > len(buf):
            raise FormatError(f"user record truncated at byte {pos}")
        user_id, n_ll, n_rt, n_imp = uh.unpack_from(buf, pos)
        pos += uh.size
        ll, pos = unpack_token_block(buf, pos, n_ll)
        rt, pos = unpack_token_block(buf, pos, n_rt)
        imp, pos = unpack_token_block(buf, pos, n_imp)
        users.append((user_id, UserSequences(ll, rt, imp)))
    if pos != len(buf):
        raise FormatError(f"{len(buf) - pos} trailing bytes at byte {pos}")
    return users
