"""The reference module API served by the B200 path (drop-in names of
seqrank.nnsearch / encoder / trainer), replayed
against the live reference's golden vectors:

* nnsearch: similarity_scores, top_k_nn, assemble, fused_assemble without an
  engine (implicit per-thread engine) and with interleaved offsets;
* encoder: encode / encode_batch / forward_fused / forward_reference / pool
  taking the reference's EncoderParams;
* trainer: model_forward -> ForwardState;
* the arena contract: batches beyond the capacity are split or run on the
  counted fallback context, never failed (arena.py:40-44).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402
from conftest import load_case  # noqa: E402
from helpers import to_user  # noqa: E402
from oracle import seqrank_oracle as orc  # noqa: E402


def _case(name):
    z, reqs = load_case(name)
    return z, reqs, P.NNConfig(*[int(v) for v in z["cfg"]])


def _golden_seqs(z, nn):
    """AssembledSequences of the reference (golden layout arrays)."""
    out = []
    for i in range(len(z["offsets"])):
        blk = P.TokenBlock(z["layout_ts"][i], z["layout_action"][i], z["layout_surface"][i], z["layout_emb"][i])
        segs = tuple(P.Segment(n, s, s + ln, int(v)) for n, s, ln, v in zip(
            P.nnsearch.SEGMENT_NAMES, nn.segment_starts(), nn.segment_lengths(), z["seg_valid"][i]))
        out.append(P.AssembledSequence(blk, z["mask"][i].astype(bool), segs))
    return out


def test_similarity_scores_and_top_k_nn():
    z, reqs, nn = _case("cobatch_s192")
    u = to_user(reqs[0]["user"])
    for c in z["candidates"][:3]:
        for blk, key in ((u.lifelong, "ll_emb"), (u.realtime, "rt_emb"), (u.impression, "imp_emb")):
            got = P.similarity_scores(blk, c)
            ref = orc.similarity_scores(reqs[0]["user"][key], c)
            assert got.dtype == np.float64 and got.shape == ref.shape
            assert np.abs(got - ref).max() <= 1e-12
            for k in (1, 7, 40, len(blk) + 3):
                picked, sc = P.top_k_nn(blk, c, k, return_scores=True)
                order = np.argsort(-ref, kind="stable")[:k]
                assert np.array_equal(picked, order), (key, k)
                assert np.abs(sc - ref[order]).max() <= 1e-12
    assert len(P.similarity_scores(P.TokenBlock.empty(), z["candidates"][0])) == 0
    assert len(P.top_k_nn(u.lifelong, z["candidates"][0], 0)) == 0
    with pytest.raises(P.ValidationError):
        P.top_k_nn(u.lifelong, z["candidates"][0], -1)


@pytest.mark.parametrize("case", ["cobatch_s192", "edge_s192"])
def test_assemble_and_implicit_fused_assemble(case):
    z, reqs, nn = _case(case)
    ref = _golden_seqs(z, nn)
    users = [to_user(r["user"]) for r in reqs]
    for i, o in enumerate(z["offsets"]):
        assert P.assemble(users[o], z["candidates"][i], nn).equals(ref[i]), f"item {i}"
    batch = P.build_dedup_batch([(u, r["cands"], None) for u, r in zip(users, reqs)])
    seqs, scores = P.fused_assemble(batch, nn, return_scores=True)  # no engine: implicit one
    for i in range(len(batch)):
        assert seqs[i].equals(ref[i])
        for g, name in enumerate(P.nnsearch.SEGMENT_NAMES):
            if name in scores[i]:
                a = nn.segment_starts()[g]
                v = scores[i][name]
                refv = np.sort(z["ref_scores"][i, a:a + len(v)])[::-1]
                assert np.abs(v - refv).max() <= 1e-12


def test_interleaved_offsets_match_grouped():
    """The reference accepts items interleaved across requests
    (nnsearch.py:307-308); per-item results must not depend on it."""
    z, reqs, nn = _case("cobatch_s192")
    users = [to_user(r["user"]) for r in reqs]
    grouped = P.build_dedup_batch([(u, r["cands"], None) for u, r in zip(users, reqs)])
    perm = np.random.default_rng(3).permutation(len(grouped))
    inter = P.DedupBatch(users, grouped.offsets[perm], grouped.candidates[perm], grouped.item_ids[perm])
    a = P.fused_assemble(grouped, nn)
    b = P.fused_assemble(inter, nn)
    for j, i in enumerate(perm):
        assert b[j].equals(a[i])


def test_encoder_api_with_reference_params():
    z, reqs, nn = _case("cobatch_s192")
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=int(z["seed"]))
    params = model.encoder
    seqs = _golden_seqs(z, nn)
    F, mask = P.encode_batch(seqs[:4], z["candidates"][:4], params)
    assert np.abs(F - z["features_head"]).max() <= 1e-6
    assert np.array_equal(mask, z["mask"][:4])
    one = P.encode(seqs[0], z["candidates"][0], params)
    assert np.array_equal(one.features, F[0])
    U = P.forward_fused(F, mask, params)
    m = mask[:, :, None]
    assert np.abs((U - z["U_head"]) * m).max() <= 2e-5
    u0 = P.forward_reference(one, params)
    assert np.abs((u0 - z["U_head"][0]) * m[0]).max() <= 2e-5
    pooled = P.pool(z["U_head"], z["mask"][:4], params)
    assert np.abs(pooled - z["pooled"][:4]).max() <= 1e-5
    p0 = P.pool(z["U_head"][0], z["mask"][0], params)
    assert p0.shape == (64,) and np.abs(p0 - z["pooled"][0]).max() <= 1e-5
    assert np.array_equal(P.pool(z["U_head"][0], np.zeros(nn.seq_len, bool), params), np.zeros(64, np.float32))


def test_model_forward_matches_reference_logits():
    z, reqs, nn = _case("cobatch_s192")
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=int(z["seed"]))
    seqs = _golden_seqs(z, nn)
    batch = P.TrainBatch(seqs, z["candidates"], np.zeros((len(seqs), 4), np.uint8), z["ctx"],
                         [to_user(reqs[o]["user"]) for o in z["offsets"]])
    st = P.model_forward(model, batch)
    ref_probs = orc.sigmoid(z["logits"].astype(np.float64))
    assert np.abs(st.probs - ref_probs).max() <= 1e-5
    assert np.abs(st.cache["logits"] - z["logits"]).max() <= 1e-5
    assert np.abs(st.cache["pooled"] - z["pooled"]).max() <= 5e-5
    assert np.abs((st.u[:4] - z["U_head"]) * st.mask[:4, :, None]).max() <= 2e-5


def test_capacity_overflow_splits_and_falls_back():
    """arena.py:40-44 / SPEC.md:509: overflow is counted, never a failure."""
    nn = P.NNConfig()
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    reqs = P.generate_requests(3, 24, ll_tokens=1500, seed=11)
    packed = [(r.user, r.candidates, r.ctx) for r in reqs]
    big = Engine(model, capacity=Capacity(8, 256, 8 * 2100))
    ref = big.rank_requests(packed)
    small = Engine(model, capacity=Capacity(2, 30, 4000))  # one request of 24 items / 2012 tokens fits
    got = small.rank_requests(packed)
    assert np.array_equal(got, ref) and small.overflow_count == 1
    tiny = Engine(model, capacity=Capacity(1, 10, 1000))  # every request is larger: fallback context
    got = tiny.rank_requests(packed)
    assert np.array_equal(got, ref) and tiny.overflow_count == 1
    out = tiny.rank_pipelined([packed[:1], packed[1:]])
    assert np.array_equal(np.concatenate(out), ref) and tiny.overflow_count == 3


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_forward_fused_extra_mask(mode):
    """forward_fused(..., extra_mask) (encoder.py:366-377) on
    the GPU vs the live reference, shared [L, L] and per-item [B, L, L]
    masks, including rows with no allowed key and rows without their own key."""
    import os

    from conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, "shapes", "extra_mask.npz"))
    nn = P.NNConfig()
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=int(z["seed"]))
    m = z["mask"][:, :, None]
    for em, U in ((z["extra2"], z["U2"]), (z["extra3"], z["U3"])):
        got = P.forward_fused(z["F"], z["mask"], model.encoder, extra_mask=em, mode=mode)
        assert np.abs((got - U) * m).max() <= 2e-5
