"""Generate the golden fixtures in tests/golden/ from the LIVE reference.

TEST INFRASTRUCTURE ONLY.  Runs in the build container, where the reference
package is importable from /root/reference/pkg/src (it does not exist on the
GPU box, so the fixtures are committed).  For every case it

  1. builds a request batch (the reference's own generate_synthetic for the
     realistic cases, hand-built token blocks for the edge cases listed in
     SURVEY.md §8c),
  2. runs the reference path build_dedup_batch -> fused_assemble(
     return_scores=True) -> encode_batch -> forward_fused -> pool + head
     (trainer.py:354-366), and the naive per-item indices
     (_nn_segment_indices over similarity_scores, nnsearch.py:83-118),
  3. runs oracle/seqrank_oracle.py on the same inputs and asserts that it
     reproduces the reference (indices / layouts bit-exact, floats <= 1e-6),
  4. writes inputs + reference outputs to tests/golden/<case>.npz.

Usage:  python oracle/gen_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from seqrank import core as rcore  # noqa: E402
from seqrank import dataset as rdata  # noqa: E402
from seqrank import encoder as renc  # noqa: E402
from seqrank import nnsearch as rnn  # noqa: E402
from seqrank import trainer as rtr  # noqa: E402

from oracle import seqrank_oracle as orc  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def params_digest(P: dict) -> str:
    h = hashlib.sha256()
    for k in sorted(P):
        h.update(k.encode())
        h.update(np.ascontiguousarray(P[k], "<f4").tobytes())
    return h.hexdigest()


def ref_model(seed, nn_cfg):
    cfg = rtr.ModelConfig(
        encoder=renc.EncoderConfig(seq_len=nn_cfg.seq_len), nn=nn_cfg
    )
    return rtr.RankingModel.init(cfg, seed=seed)


def ref_forward(model, batch, seqs, ctx):
    """trainer.py:354-366 over forward_fused output (BASELINE.md §3 path)."""
    F, mask = renc.encode_batch(seqs, batch.candidates, model.encoder)
    U = renc.forward_fused(F, mask, model.encoder)
    y = U @ model.encoder.out_linear
    ym = np.where(mask[:, :, None], y, np.array(-np.inf, y.dtype))
    pooled = ym.max(1)
    pooled[~mask.any(1)] = 0
    unit_c = rcore.l2_normalize_rows(batch.candidates).astype(np.float32)
    z = np.concatenate([pooled, unit_c, ctx], axis=1)
    h = np.maximum(z @ model.head.w1 + model.head.b1, 0)
    logits = h @ model.head.w2 + model.head.b2
    return F, mask, U, pooled, logits


def block(n, rng, base_ts, step, impression=False, dup=0):
    ts = (base_ts - np.arange(n, dtype=np.int64) * step).astype(np.uint32)
    if impression:
        act = np.full(n, rcore.IMPRESSION, np.uint16)
    else:
        act = rng.choice([1, 2, 4, 8, 1 | 4, 2 | 4, 1 | 2 | 4], n).astype(np.uint16)
    surf = rng.integers(0, 256, n).astype(np.uint8)  # includes ids > 3
    e = rng.normal(0, 0.2, (n, 32))
    emb = rcore.quantize(e)
    if dup and n > 1:  # plant exact duplicate embeddings -> score ties
        src = rng.integers(0, n, dup)
        dst = rng.integers(0, n, dup)
        emb[dst] = emb[src]
    return rcore.TokenBlock(ts, act, surf, emb)


def edge_users(rng):
    empty = rcore.UserSequences()
    tiny = rcore.UserSequences(  # L < k, RT <= r, IMP < k
        block(10, rng, 1_700_000_000, 3600, dup=3),
        block(20, rng, 1_750_000_000, 60),
        block(5, rng, 1_750_000_030, 60, impression=True),
    )
    dups = rcore.UserSequences(  # many exact ties in every source
        block(400, rng, 1_700_000_000, 3600, dup=200),
        block(90, rng, 1_750_000_000, 60, dup=40),
        block(70, rng, 1_750_000_030, 60, impression=True, dup=30),
    )
    ll_only = rcore.UserSequences(block(150, rng, 1_700_000_000, 3600), rcore.TokenBlock.empty(),
                                  rcore.TokenBlock.empty())
    for u in (tiny, dups, ll_only):
        u.validate()
    return [empty, tiny, dups, ll_only]


def synthetic_users(n_users, ll, rt, imp, chunk, seed):
    data = rdata.generate_synthetic(rdata.SyntheticConfig(
        num_users=n_users, num_clusters=8, ll_tokens=ll, rt_tokens=rt, imp_tokens=imp,
        chunks_per_user=1, chunk_size=chunk, seed=seed))
    reqs = []
    for uid, seqs in data.users:
        cands = np.stack([ex.candidate for ex in data.examples if ex.user_id == uid])
        reqs.append((uid, seqs, cands.astype(np.float32)))
    return reqs


def run_case(name, reqs, nn_cfg, seed=0):
    """reqs: list of (user_id, UserSequences, cands[m,32])."""
    model = ref_model(seed, nn_cfg)
    batch = rnn.build_dedup_batch([(u, c, None) for _, u, c in reqs])
    seqs, scores = rnn.fused_assemble(batch, nn_cfg, return_scores=True)
    ctx = np.stack([rdata.context_features(reqs[o][0]) for o in batch.offsets])
    F, mask, U, pooled, logits = ref_forward(model, batch, seqs, ctx)

    # naive per-item indices (source-relative; RT tail offset by r)
    S = nn_cfg.seq_len
    idx = np.full((len(batch), S), -1, np.int32)
    ref_scores = np.full((len(batch), S), np.nan, np.float64)
    kth = np.full((len(batch), 4), np.nan, np.float64)
    for i, o in enumerate(batch.offsets):
        user, cand = batch.users[o], batch.candidates[i]
        rt = user.realtime
        r = nn_cfg.recent
        start = 0
        for s, (seg, seg_len) in enumerate(zip(rnn.SEGMENT_NAMES, nn_cfg.segment_lengths())):
            if seg == "recent_realtime":
                n_recent = min(r, len(rt))
                sel = np.arange(n_recent - 1, -1, -1)
            else:
                src = {"nn_lifelong": user.lifelong,
                       "nn_realtime_tail": rt.take(np.arange(r, len(rt))) if len(rt) > r else None,
                       "nn_impression": user.impression}[seg]
                k = {"nn_lifelong": nn_cfg.k_lifelong, "nn_realtime_tail": nn_cfg.k_realtime,
                     "nn_impression": nn_cfg.k_impression}[seg]
                if src is None or len(src) == 0 or k == 0:
                    sel = np.zeros(0, np.intp)
                else:
                    d = rnn.similarity_scores(src, cand)
                    sel = rnn._nn_segment_indices(d, k)
                    ref_scores[i, start:start + len(sel)] = d[sel]
                    kth[i, s] = np.sort(d)[::-1][min(k, len(d)) - 1]
                    if seg == "nn_realtime_tail":
                        sel = sel + r
            idx[i, start:start + len(sel)] = sel
            start += seg_len

    # ---- oracle must reproduce the reference ------------------------------
    P = orc.model_init(seed, seq_len=S)
    assert params_digest(P) == params_digest(model.named_tensors()), "model_init drift"
    cfg = (nn_cfg.recent, nn_cfg.k_lifelong, nn_cfg.k_realtime, nn_cfg.k_impression)
    row = 0
    for (uid, user, cands) in reqs:
        ud = user_dict(user)
        lg, det = orc.rank_request(ud, cands, orc.context_features(uid), P, cfg, return_detail=True)
        m = len(cands)
        for j in range(m):
            flat = np.concatenate(det["segs"][j]) if det["segs"][j] else np.zeros(0)
            ref_flat = idx[row + j][idx[row + j] >= 0]
            assert np.array_equal(flat, ref_flat), f"{name}: index mismatch item {row + j}"
            lay = det["layout"][j]
            sq = seqs[row + j]
            assert np.array_equal(lay["emb"], sq.block.embeddings)
            assert np.array_equal(lay["ts"], sq.block.timestamps)
            assert np.array_equal(lay["action"], sq.block.actions)
            assert np.array_equal(lay["surface"], sq.block.surfaces)
            assert np.array_equal(lay["mask"], sq.mask)
            for seg, sc in det["scores"][j].items():
                # f64 BLAS blocking differs with operand layout: ~1e-16
                assert np.abs(sc - scores[row + j][seg]).max() <= 1e-12
        err = np.abs(lg - logits[row:row + m]).max()
        assert err <= 1e-6, f"{name}: oracle logits off by {err}"
        row += m

    # ---- serialise ---------------------------------------------------------
    arrays = dict(
        cfg=np.array(cfg, np.int32), seed=np.array(seed), offsets=batch.offsets,
        candidates=batch.candidates, ctx=ctx.astype(np.float32),
        user_ids=np.array([u for u, _, _ in reqs], np.int64),
        idx=idx, ref_scores=ref_scores, kth=kth,
        mask=mask, logits=logits.astype(np.float32), pooled=pooled.astype(np.float32),
        layout_emb=np.stack([s.block.embeddings for s in seqs]),
        layout_action=np.stack([s.block.actions for s in seqs]),
        layout_surface=np.stack([s.block.surfaces for s in seqs]),
        layout_ts=np.stack([s.block.timestamps for s in seqs]),
        seg_valid=np.array([[g.valid for g in s.segments] for s in seqs], np.int32),
        features_head=F[:4].astype(np.float32), U_head=U[:4].astype(np.float32),
    )
    # NN-feature logging records: the reference's own
    # pack_assembled bytes of every assembled sequence (dataset.py:138-149)
    packed = [rdata.pack_assembled(sq) for sq in seqs]
    arrays["packed_assembled"] = np.frombuffer(b"".join(packed), np.uint8)
    arrays["packed_offsets"] = np.cumsum([0] + [len(b) for b in packed]).astype(np.int64)
    for r_i, (_, user, _) in enumerate(reqs):
        for src, blk in (("ll", user.lifelong), ("rt", user.realtime), ("imp", user.impression)):
            arrays[f"r{r_i}_{src}_emb"] = blk.embeddings
            arrays[f"r{r_i}_{src}_action"] = blk.actions
            arrays[f"r{r_i}_{src}_surface"] = blk.surfaces
            arrays[f"r{r_i}_{src}_ts"] = blk.timestamps
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
    return dict(items=len(batch), requests=len(reqs), S=S,
                params_sha256=params_digest(P))


def user_dict(user):
    d = {}
    for src, blk in (("ll", user.lifelong), ("rt", user.realtime), ("imp", user.impression)):
        d[f"{src}_emb"] = blk.embeddings
        d[f"{src}_action"] = blk.actions
        d[f"{src}_surface"] = blk.surfaces
        d[f"{src}_ts"] = blk.timestamps
    return d


def kat():
    """SPEC.md KATs checked in SURVEY §4, recorded with their reference values."""
    return dict(
        quantize_in=[0.65, 0.0, -1.0, 0.325],
        quantize_out=rcore.quantize(np.array([0.65, 0.0, -1.0, 0.325])).tolist(),
        dequantize_64=float(rcore.dequantize(np.array([64], np.int8))[0]),
        context_7=rdata.context_features(7).tolist(),
        build_dedup_offsets=rnn.build_dedup_batch([
            (rcore.UserSequences(), np.zeros((2, 32), np.float32), None),
            (rcore.UserSequences(), np.zeros((3, 32), np.float32), None),
        ]).offsets.tolist(),
    )


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(1234)
    manifest = {}
    default = rnn.NNConfig()
    c1 = rnn.NNConfig(recent=32, k_lifelong=32, k_realtime=0, k_impression=0)

    # C1: CPU reference default (1 x 64 candidates, L=1024, S=64)
    manifest["c1_cpu_default"] = run_case("c1_cpu_default", synthetic_users(1, 1024, 256, 256, 64, 0), c1)
    # default NNConfig (S=192), co-batched requests of different sizes
    reqs = synthetic_users(3, 600, 80, 60, 6, 1)
    reqs[1] = (reqs[1][0], reqs[1][1], reqs[1][2][:3])  # ragged candidate counts
    manifest["cobatch_s192"] = run_case("cobatch_s192", reqs, default)
    # the same middle request alone (co-batched == solo)
    manifest["solo_s192"] = run_case("solo_s192", [reqs[1]], default)
    # edge cases: empty user, L<k, RT<=r, ties, LL-only; zero candidate; N=1
    users = edge_users(rng)
    erq = []
    for i, u in enumerate(users):
        m = 1 if i == 0 else 4
        c = rng.normal(0, 1, (m, 32)).astype(np.float32)
        if i == 1:
            c[0] = 0.0  # zero candidate -> all scores 0 -> ties to lowest index
        if i == 2:  # candidate equal to a duplicated token direction
            c[1] = rcore.dequantize(u.lifelong.embeddings[3])
        erq.append((100 + i, u, c))
    manifest["edge_s192"] = run_case("edge_s192", erq, default)
    manifest["edge_k0"] = run_case("edge_k0", erq[1:3], rnn.NNConfig(recent=8, k_lifelong=16,
                                                                     k_realtime=0, k_impression=8))
    # larger k (sweep shape), S = 96 + 256 = 352
    manifest["k256_s352"] = run_case("k256_s352", synthetic_users(1, 2048, 256, 256, 8, 3),
                                     rnn.NNConfig(k_lifelong=256))
    manifest["kat"] = kat()
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
