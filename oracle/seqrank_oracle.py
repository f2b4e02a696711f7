"""CPU oracle for the TransAct V2 serving-time ranking path.

TEST INFRASTRUCTURE ONLY.  This module is a numpy restatement of the
reference package ``seqrank`` 0.1.0 (``/root/reference/pkg/src/seqrank``)
for the hot path named in BASELINE.json ``north_star``:

    request dedup -> fused NN selection (dequantize + normalize + f64 dot +
    stable top-k) -> Eq. 2 layout -> Eq. 4 encode -> 2-layer SKUT forward
    -> linear + masked max-pool -> CTR head.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import it, and only as the checker / the timed CPU baseline.  The
product package (``paper_2506_02267_b200``) never imports it.

Parity pin: every function below is checked against the live reference (run
in the build container) by ``oracle/gen_golden.py``, which also writes the
golden fixtures in ``tests/golden/`` that the CPU test-suite replays.

Every function cites the reference ``file:line`` it restates.  The oracle
works on plain arrays (token columns per source, candidate matrix, a
``name -> ndarray`` parameter dict using the reference checkpoint names) so
it is independent of both the reference and the product package.
"""

from __future__ import annotations

import numpy as np

EMBED_DIM = 32
QUANT_SCALE = 0.65
QUANT_MAX = 127
SURFACE_OTHER = 3
LN_EPS = 1e-5
SEGMENT_NAMES = ("nn_lifelong", "recent_realtime", "nn_realtime_tail", "nn_impression")
NUM_HEADS = 4
UTILITY_WEIGHTS = (1.0, 0.5, 0.25, -2.0)  # losses.py:29


# ---------------------------------------------------------------------------
# codec (core.py)
# ---------------------------------------------------------------------------


def quantize(e):
    """core.py:40-51 -- round-half-away, clamp to +-127."""
    e = np.asarray(e, dtype=np.float64)
    if not np.all(np.isfinite(e)):
        raise ValueError("embedding components must be finite")
    s = e / QUANT_SCALE * QUANT_MAX
    r = np.copysign(np.floor(np.abs(s) + 0.5), s)
    return np.clip(r, -QUANT_MAX, QUANT_MAX).astype(np.int8)


def dequantize(q):
    """core.py:54-57 -- (q.f32 / 127) * 0.65 in float32."""
    return (np.asarray(q).astype(np.float32) / np.float32(QUANT_MAX)) * np.float32(QUANT_SCALE)


def unit_rows(m):
    """core.py:69-74 -- row L2 normalize in f32, zero rows stay zero."""
    m = np.asarray(m, dtype=np.float32)
    n = np.sqrt(np.einsum("ij,ij->i", m, m, dtype=np.float32))
    n = np.where(n == 0.0, np.float32(1.0), n)
    return m / n[:, None]


def unit_tokens(q):
    """core.py:77-79 / nnsearch.py:274-286 (bit-identical fused form)."""
    q = np.asarray(q, np.int8).reshape(-1, EMBED_DIM)
    return unit_rows(dequantize(q))


# ---------------------------------------------------------------------------
# NN selection (nnsearch.py)
# ---------------------------------------------------------------------------


def seq_len(cfg):
    """nnsearch.py:35-37; cfg = (recent, k_ll, k_rt, k_imp)."""
    return int(sum(cfg))


def segment_lengths(cfg):
    """nnsearch.py:39-40 -- layout order (k_ll, recent, k_rt, k_imp)."""
    r, kl, kr, ki = cfg
    return (kl, r, kr, ki)


def _topk_desc_storage(dots, k):
    """nnsearch.py:114-118, :361-364 -- stable top-k, then descending index."""
    picked = np.argsort(-dots, kind="stable")[:k]
    return picked, np.sort(picked)[::-1]


def nn_select_request(ll, rt, imp, cands, cfg, return_scores=False):
    """fused_assemble for one request (nnsearch.py:289-369).

    ll/rt/imp: int8 [n, 32] token embeddings of each source (newest first).
    cands: f32 [m, 32].  Returns, per candidate, the four per-segment index
    arrays (indices into the segment's *source block*: LL, RT, RT (already
    offset by r, :133/:327) and IMP) in layout order, plus best-first f64
    scores per NN segment when asked.
    """
    r, k_ll, k_rt, k_imp = cfg
    cands = np.asarray(cands, np.float32)
    m = len(cands)
    unit_c = unit_rows(cands)  # :313-320 (same f32 ops)
    cand64 = unit_c.T.astype(np.float64)  # :321-323
    n_rt = len(rt)
    n_recent = min(r, n_rt)
    sources = {
        "nn_lifelong": (np.asarray(ll, np.int8).reshape(-1, EMBED_DIM), k_ll, 0),
        "nn_realtime_tail": (np.asarray(rt, np.int8).reshape(-1, EMBED_DIM)[r:], k_rt, r),
        "nn_impression": (np.asarray(imp, np.int8).reshape(-1, EMBED_DIM), k_imp, 0),
    }
    dots = {}
    for name, (emb, k, _) in sources.items():  # :335-348
        if len(emb) == 0 or k == 0:
            dots[name] = None
        else:
            dots[name] = unit_tokens(emb).astype(np.float64) @ cand64
    out, scores = [], []
    recent = np.arange(n_recent - 1, -1, -1)  # :144, :354
    for col in range(m):  # :350-366
        segs, sc = [], {}
        for name in SEGMENT_NAMES:
            if name == "recent_realtime":
                segs.append(recent)
                continue
            d = dots[name]
            if d is None:
                segs.append(np.zeros(0, np.intp))
                continue
            k, off = sources[name][1], sources[name][2]
            picked, seg = _topk_desc_storage(d[:, col], k)
            sc[name] = d[picked, col].copy()
            segs.append(seg + off)  # RT-tail indices are relative to r (:133)
        out.append(segs)
        scores.append(sc)
    if return_scores:
        return out, scores
    return out


def similarity_scores(emb, cand):
    """nnsearch.py:83-90 -- naive path f64 scores for one candidate."""
    emb = np.asarray(emb, np.int8).reshape(-1, EMBED_DIM)
    if len(emb) == 0:
        return np.zeros(0, np.float64)
    uc = unit_rows(np.asarray(cand, np.float32)[None, :])[0]
    return unit_tokens(emb).astype(np.float64) @ uc.astype(np.float64)


def layout(segs, cols, cfg):
    """nnsearch.py:153-180 -- fixed padded layout of the per-segment picks.

    segs: 4 index arrays (layout order) into the per-segment source columns
    ``cols = [(emb, action, surface, ts) for LL, RT, RT, IMP]``.
    Returns dict(emb i8 [S,32], action u16 [S], surface u8 [S], ts u32 [S],
    mask bool [S], valid [4]).
    """
    S = seq_len(cfg)
    out = dict(
        emb=np.zeros((S, EMBED_DIM), np.int8),
        action=np.zeros(S, np.uint16),
        surface=np.zeros(S, np.uint8),
        ts=np.zeros(S, np.uint32),
        mask=np.zeros(S, bool),
        valid=np.zeros(4, np.int32),
    )
    start = 0
    for s, (idx, seg_len) in enumerate(zip(segs, segment_lengths(cfg))):
        v = len(idx)
        if v:
            emb, act, surf, ts = cols[s]
            out["emb"][start : start + v] = emb[idx]
            out["action"][start : start + v] = act[idx]
            out["surface"][start : start + v] = surf[idx]
            out["ts"][start : start + v] = ts[idx]
            out["mask"][start : start + v] = True
        out["valid"][s] = v
        start += seg_len
    return out


# ---------------------------------------------------------------------------
# encode + transformer + pool + head (encoder.py, trainer.py)
# ---------------------------------------------------------------------------


def encode_batch(emb, action, surface, mask, cands, P, num_layers=2):
    """encoder.py:161-188 -- Eq. 4 early fusion.

    emb [B,S,32] i8, action [B,S] u16, surface [B,S] u8, mask [B,S] bool,
    cands [B,32] f32 -> features [B,S,64] f32.
    """
    at = P["encoder.action_table"]
    st = P["encoder.surface_table"]
    pt = P["encoder.position_table"]
    dtype = at.dtype
    B, S = mask.shape
    E = emb.shape[-1]
    unit = unit_rows(dequantize(emb.reshape(B * S, E))).reshape(B, S, E)
    unit_c = unit_rows(np.asarray(cands, np.float32))
    bits = (action.astype(np.int64)[..., None] >> np.arange(at.shape[0])) & 1
    surf = surface.astype(np.intp)
    surf[surf > SURFACE_OTHER] = SURFACE_OTHER  # :178
    F = np.zeros((B, S, 2 * E), dtype)
    F[:, :, :E] = unit
    F[:, :, E:] = unit_c[:, None, :]
    F += bits.astype(dtype) @ at
    F += st[surf]
    F += pt[None, :, :]
    F *= mask[:, :, None].astype(dtype)
    return F


def layer_norm(x, scale, shift):
    """encoder.py:196-200."""
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    return xc / np.sqrt(var + np.asarray(LN_EPS, x.dtype)) * scale + shift


def masked_softmax(logits, allowed):
    """encoder.py:203-211 -- fully masked rows give 0."""
    neg = np.array(-np.inf, logits.dtype)
    z = np.where(allowed, logits, neg)
    mx = z.max(-1, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, logits.dtype.type(0))
    w = np.exp(z - mx)
    den = w.sum(-1, keepdims=True)
    return w / np.where(den == 0, logits.dtype.type(1), den)


def _layers(P):
    n = 0
    while f"encoder.layer{n}.wq" in P:
        n += 1
    return [
        {k: P[f"encoder.layer{i}.{k}"] for k in
         ("wq", "wk", "wv", "wo", "w1", "w2", "ln1_scale", "ln1_shift", "ln2_scale", "ln2_shift")}
        for i in range(n)
    ]


def forward_layered(F, mask, P):
    """encoder.py:221-246 / trainer.py:261-291 -- batched layered forward."""
    x = np.array(F)
    B, S, d = x.shape
    scale = x.dtype.type(1.0 / np.sqrt(d))
    allowed = np.tril(np.ones((S, S), bool))[None] & mask[:, None, :]
    for L in _layers(P):
        a = layer_norm(x, L["ln1_scale"], L["ln1_shift"])
        q, k, v = a @ L["wq"], a @ L["wk"], a @ L["wv"]
        p = masked_softmax((q @ k.transpose(0, 2, 1)) * scale, allowed)
        x = x + (p @ v) @ L["wo"]
        f = layer_norm(x, L["ln2_scale"], L["ln2_shift"])
        x = x + np.maximum(f @ L["w1"], 0) @ L["w2"]
    return x


def forward_fused(F, mask, P, tile=64, extra_mask=None):
    """encoder.py:314-462 -- tiled online-softmax single-pass forward.  Same
    operation order as the reference so CPU timing is representative.
    extra_mask ([S, S] or [B, S, S] bool, encoder.py:366-377): key j allowed
    for row i only where set, on top of causal & key-valid; a row with no
    allowed key gets a zero attention output (row_any)."""
    B, S, d = F.shape
    dtype = F.dtype
    neg = np.float32(-1e30) if dtype == np.float32 else np.float64(-1e300)
    tile = max(1, min(tile, S))
    scale = dtype.type(1.0 / np.sqrt(d))
    x = np.array(F)
    a_in = np.empty_like(x)
    invalid = ~mask
    bad = None
    if extra_mask is not None:  # :366-377
        em = np.broadcast_to(np.asarray(extra_mask, bool), (B, S, S))
        bad = ~em | np.triu(np.ones((S, S), bool), 1)[None] | invalid[:, None, :]
        row_any = (~bad.all(-1)).astype(dtype)
    else:
        row_any = np.maximum.accumulate(mask.astype(dtype), axis=1)  # :379-381
    triu = np.triu(np.ones((tile, tile), bool), 1)
    nt = (S + tile - 1) // tile
    for L in _layers(P):
        for ti in range(nt):
            s0, s1 = ti * tile, min((ti + 1) * tile, S)
            a_in[:, s0:s1] = layer_norm(x[:, s0:s1], L["ln1_scale"], L["ln1_shift"])
        for qi in range(nt):
            qs, qe = qi * tile, min((qi + 1) * tile, S)
            tq = qe - qs
            q = a_in[:, qs:qe] @ L["wq"]
            m = np.full((B, tq), neg, dtype)
            l = np.zeros((B, tq), dtype)
            acc = np.zeros((B, tq, d), dtype)
            for kj in range(qi + 1):  # :407-443
                ks, ke = kj * tile, min((kj + 1) * tile, S)
                tk = ke - ks
                k = a_in[:, ks:ke] @ L["wk"]
                v = a_in[:, ks:ke] @ L["wv"]
                s = (q @ k.transpose(0, 2, 1)) * scale
                if bad is not None:  # :418-419
                    s = np.where(bad[:, qs:qe, ks:ke], neg, s)
                else:
                    s = np.where(invalid[:, None, ks:ke], neg, s)
                    if kj == qi:
                        s = np.where(triu[:tq, :tk], neg, s)
                mn = np.maximum(s.max(-1), m)
                al = np.exp(m - mn)
                m = mn
                s = np.exp(s - mn[:, :, None])
                l = l * al + s.sum(-1)
                acc = acc * al[:, :, None] + s @ v
            l = np.maximum(l, dtype.type(1e-30))  # :445-447
            att = acc / l[:, :, None] * row_any[:, qs:qe, None]
            x[:, qs:qe] += att @ L["wo"]  # :449-450
            f = layer_norm(x[:, qs:qe], L["ln2_scale"], L["ln2_shift"])
            x[:, qs:qe] += np.maximum(f @ L["w1"], 0) @ L["w2"]  # :455-460
    return x


def pool_head(U, mask, cands, ctx, P):
    """trainer.py:354-366 (pool = encoder.py:265-273 batched).

    Returns (pooled [B,64], logits [B,4]) in f32.
    """
    dtype = U.dtype
    y = U @ P["encoder.out_linear"]
    ym = np.where(mask[:, :, None], y, np.array(-np.inf, dtype))
    pooled = ym.max(1)
    pooled[~mask.any(1)] = 0
    unit_c = unit_rows(np.asarray(cands, np.float32)).astype(dtype)
    z = np.concatenate([pooled, unit_c, np.asarray(ctx, dtype)], axis=1)
    h = np.maximum(z @ P["head.w1"] + P["head.b1"], 0)
    logits = h @ P["head.w2"] + P["head.b2"]
    return pooled, logits


def sigmoid(x):
    """trainer.py:230-236 -- split form."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def final_score(probs):
    """evaluation.py:35-37 with HeadConfig.utility_weights (losses.py:29)."""
    return np.asarray(probs, np.float64) @ np.asarray(UTILITY_WEIGHTS, np.float64)


def context_features(user_id, dim=8):
    """dataset.py:282-289."""
    rng = np.random.default_rng([int(user_id), 96321])
    return rng.uniform(-1.0, 1.0, dim).astype(np.float32)


# ---------------------------------------------------------------------------
# parameters (trainer.py:88-102, encoder.py:75-108)
# ---------------------------------------------------------------------------


def model_init(seed=0, embed_dim=32, seq_len=192, ffn_dim=32, num_layers=2,
               action_rows=16, surface_rows=256, ctx_dim=8, hidden_dim=64):
    """RankingModel.init draw order: per layer wq,wk,wv,wo,w1,w2; then the
    action, surface, position tables; out_linear; head w1, w2; nal.proj."""
    rng = np.random.default_rng([seed, 0])
    d, f = 2 * embed_dim, ffn_dim
    ws = 1.0 / np.sqrt(d)

    def w(*shape, scale=ws):
        return rng.normal(0.0, scale, shape).astype(np.float32)

    P = {}
    layers = []
    for _ in range(num_layers):
        layers.append(dict(wq=w(d, d), wk=w(d, d), wv=w(d, d), wo=w(d, d),
                           w1=w(d, f), w2=w(f, d, scale=1.0 / np.sqrt(f))))
    P["encoder.action_table"] = w(action_rows, d, scale=0.1)
    P["encoder.surface_table"] = w(surface_rows, d, scale=0.1)
    P["encoder.position_table"] = w(seq_len, d, scale=0.1)
    P["encoder.out_linear"] = w(d, d)
    for i, L in enumerate(layers):
        for k, v in L.items():
            P[f"encoder.layer{i}.{k}"] = v
        P[f"encoder.layer{i}.ln1_scale"] = np.ones(d, np.float32)
        P[f"encoder.layer{i}.ln1_shift"] = np.zeros(d, np.float32)
        P[f"encoder.layer{i}.ln2_scale"] = np.ones(d, np.float32)
        P[f"encoder.layer{i}.ln2_shift"] = np.zeros(d, np.float32)
    in_dim = d + embed_dim + ctx_dim
    P["head.w1"] = rng.normal(0, 1 / np.sqrt(in_dim), (in_dim, hidden_dim)).astype(np.float32)
    P["head.b1"] = np.zeros(hidden_dim, np.float32)
    P["head.w2"] = rng.normal(0, 1 / np.sqrt(hidden_dim), (hidden_dim, NUM_HEADS)).astype(np.float32)
    P["head.b2"] = np.zeros(NUM_HEADS, np.float32)
    P["nal.proj"] = rng.normal(0, 1 / np.sqrt(d), (d, embed_dim)).astype(np.float32)
    return P


# ---------------------------------------------------------------------------
# full request (the spec'd rank(), composed as BASELINE.md §3)
# ---------------------------------------------------------------------------


def rank_request(user, cands, ctx, P, cfg, return_detail=False, forward="fused"):
    """One request end to end.

    user: dict with per-source columns ``{ll,rt,imp}_{emb,action,surface,ts}``.
    Returns logits [m,4] f32 (and the per-item segment indices, scores and
    assembled layouts when ``return_detail``).
    """
    segs, scores = nn_select_request(user["ll_emb"], user["rt_emb"], user["imp_emb"],
                                     cands, cfg, return_scores=True)
    cols = []
    for src in ("ll", "rt", "rt", "imp"):
        cols.append((user[f"{src}_emb"], user[f"{src}_action"], user[f"{src}_surface"],
                     user[f"{src}_ts"]))
    lay = [layout(s, cols, cfg) for s in segs]
    emb = np.stack([x["emb"] for x in lay])
    act = np.stack([x["action"] for x in lay])
    surf = np.stack([x["surface"] for x in lay])
    mask = np.stack([x["mask"] for x in lay])
    F = encode_batch(emb, act, surf, mask, cands, P)
    U = forward_fused(F, mask, P) if forward == "fused" else forward_layered(F, mask, P)
    ctxb = np.broadcast_to(np.asarray(ctx, np.float32), (len(cands), len(ctx)))
    _, logits = pool_head(U, mask, cands, ctxb, P)
    if return_detail:
        return logits, dict(segs=segs, scores=scores, layout=lay, features=F, mask=mask)
    return logits
