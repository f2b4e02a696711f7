"""GPU parity at the benchmarked shapes (BASELINE configs), on
inputs from the reference's own generator (``dataset.synthetic_requests``, the
draw-for-draw port of ``generate_synthetic`` pinned by request digests in
tests/golden/shapes/c2_generator.json):

* C2 (1 x 1000, L = 16,384): every candidate against the live reference's
  outputs (tests/golden/shapes/c2_seed0.npz: index layout, k-th scores,
  logits, pooled), and the benchmark's other pool requests against the
  oracle, in both precision modes;
* C3 (32 x 500): the full index contract on every request, logits on a
  candidate sample of each;
* C4 (1 x 8192 split over g = 2, 4, 8): slices scored separately equal the
  unsplit run bit for bit;
* ``fused_assemble(return_scores=True)``: the reference's f64 scores.
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.parallel import split_bounds  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402
from conftest import GOLDEN  # noqa: E402
from helpers import check_nn_contract, from_user, oracle_layout, ref_scores_fn  # noqa: E402
from oracle import seqrank_oracle as orc  # noqa: E402

TOL = {"fp32": 1e-5, "bf16": 2e-3}
POOLED_TOL = {"fp32": 5e-5, "bf16": 5e-3}
NN = P.NNConfig()
CFG = (NN.recent, NN.k_lifelong, NN.k_realtime, NN.k_impression)
SHAPES = os.path.join(GOLDEN, "shapes")


def _digest(r):
    h = hashlib.sha256()
    for blk in r.user.blocks():
        for a in (blk.timestamps, blk.actions, blk.surfaces, blk.embeddings):
            h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.ascontiguousarray(r.candidates, np.float32).tobytes())
    h.update(np.ascontiguousarray(r.ctx, np.float32).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def c2_requests():
    with open(os.path.join(SHAPES, "c2_generator.json")) as fh:
        meta = json.load(fh)
    reqs = P.synthetic_requests(4, 1000, 16384, 256, 256, seed=0)
    for s, r in enumerate(reqs):  # the port reproduces the reference generator here too
        assert _digest(r) == meta["request_sha256_by_seed"][str(s)], f"generator drift, seed {s}"
    return reqs


@pytest.fixture(scope="module")
def engine():
    model = P.RankingModel.init(P.ModelConfig.for_nn(NN), seed=0)
    return Engine(model, capacity=Capacity(32, 16384, 32 * 16896))


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_c2_all_candidates_vs_reference(c2_requests, engine, mode):
    z = np.load(os.path.join(SHAPES, "c2_seed0.npz"))
    r = c2_requests[0]
    logits, idx = engine.rank_requests([(r.user, r.candidates, r.ctx)], mode=mode, return_indices=True)
    user = from_user(r.user)
    swaps = check_nn_contract(idx, z["idx"].astype(np.int32), ref_scores_fn(lambda i: user, r.candidates),
                              z["kth"], NN.segment_starts(), NN.segment_lengths())
    a, b = NN.segment_starts()[1], NN.segment_starts()[1] + NN.recent
    assert np.array_equal(idx[:, a:b], z["idx"][:, a:b])
    if swaps == 0:
        assert np.array_equal(idx, z["idx"])
    err = float(np.abs(logits - z["logits"]).max())
    assert err <= TOL[mode], f"C2 {mode}: max |dlogit| = {err}"
    # the pooled vectors of the fused kernel (trainer.py:354-359) vs the reference's
    engine.stage([(r.user, r.candidates, r.ctx)])
    idx_d = torch.from_numpy(idx).cuda()
    lg2, pooled = engine.score_staged(idx_d, mode=mode, pooled=True)
    assert np.array_equal(lg2.cpu().numpy(), logits)
    perr = float(np.abs(pooled.cpu().numpy() - z["pooled"]).max())
    assert perr <= POOLED_TOL[mode], f"C2 {mode}: max |dpooled| = {perr}"


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c2_bench_pool_vs_oracle(c2_requests, engine, seed):
    """The benchmark's request pool (rank 0: seeds 0..3), every candidate."""
    r = c2_requests[seed]
    user = from_user(r.user)
    ref_idx, kth = oracle_layout(user, r.candidates, CFG)
    Pd = orc.model_init(0, seq_len=NN.seq_len)
    ref = orc.rank_request(user, r.candidates, r.ctx, Pd, CFG)
    for mode in ("bf16", "fp32"):
        logits, idx = engine.rank_requests([(r.user, r.candidates, r.ctx)], mode=mode, return_indices=True)
        check_nn_contract(idx, ref_idx, ref_scores_fn(lambda i: user, r.candidates), kth,
                          NN.segment_starts(), NN.segment_lengths())
        err = float(np.abs(logits - ref).max())
        assert err <= TOL[mode], f"seed {seed} {mode}: max |dlogit| = {err}"


def test_c3_batch_vs_oracle(engine):
    """C3's per-GPU batch: 32 requests x 500 candidates co-batched in one run."""
    reqs = P.synthetic_requests(32, 500, 16384, 256, 256, seed=100)
    batch = [(r.user, r.candidates, r.ctx) for r in reqs]
    Pd = orc.model_init(0, seq_len=NN.seq_len)
    rng = np.random.default_rng(0)
    for mode in ("bf16", "fp32"):
        logits, idx = engine.rank_requests(batch, mode=mode, return_indices=True)
        assert logits.shape == (32 * 500, 4)
        for q, r in enumerate(reqs):
            sl = slice(500 * q, 500 * (q + 1))
            user = from_user(r.user)
            if mode == "bf16":  # the selection is mode-independent; check it once
                ref_idx, kth = oracle_layout(user, r.candidates, CFG)
                check_nn_contract(idx[sl], ref_idx, ref_scores_fn(lambda i, u=user: u, r.candidates), kth,
                                  NN.segment_starts(), NN.segment_lengths())
            pick = rng.choice(500, 6, replace=False)
            ref = orc.rank_request(user, r.candidates[pick], r.ctx, Pd, CFG)
            err = float(np.abs(logits[sl][pick] - ref).max())
            assert err <= TOL[mode], f"C3 request {q} {mode}: max |dlogit| = {err}"


def test_c4_split_equals_unsplit(engine):
    """One 8,192-candidate request scored whole vs as g contiguous slices
    (parallel.rank_split's layout): identical bits (per-candidate math is
    independent of the batch it runs in)."""
    r = P.synthetic_requests(1, 8192, 16384, 256, 256, seed=7)[0]
    for mode in ("bf16", "fp32"):
        whole, idx = engine.rank_requests([(r.user, r.candidates, r.ctx)], mode=mode, return_indices=True)
        for g in (2, 4, 8):
            parts, pidx = [], []
            for lo, hi in split_bounds(len(r.candidates), g):
                lg, ix = engine.rank_requests([(r.user, r.candidates[lo:hi], r.ctx)], mode=mode,
                                              return_indices=True)
                parts.append(lg)
                pidx.append(ix)
            assert np.array_equal(np.concatenate(parts), whole), f"{mode} g={g}"
            assert np.array_equal(np.concatenate(pidx), idx), f"{mode} g={g}"


def test_fused_assemble_return_scores_are_reference_f64(c2_requests):
    """P.fused_assemble(..., return_scores=True) on the C2 request: the
    AssembledSequences equal the reference's layouts and the scores are the
    reference's float64 dots (nnsearch.py:362-363) -- not an f32 image."""
    z = np.load(os.path.join(SHAPES, "c2_seed0.npz"))
    r = c2_requests[0]
    n = len(z["scores_head"])
    batch = P.build_dedup_batch([(r.user, r.candidates[:n], None)])
    seqs, scores = P.fused_assemble(batch, NN, return_scores=True)
    for i in range(n):
        ref_seq = P.nnsearch.assembled_from_indices(r.user, z["idx"][i].astype(np.int32), NN)
        assert seqs[i].equals(ref_seq), f"item {i}"
        for name, start, length in zip(P.nnsearch.SEGMENT_NAMES, NN.segment_starts(), NN.segment_lengths()):
            ref = z["scores_head"][i, start:start + length]
            ref = ref[~np.isnan(ref)]
            if name == "recent_realtime":
                assert name not in scores[i]
                continue
            got = scores[i][name]
            assert got.dtype == np.float64 and len(got) == len(ref)
            assert np.abs(got - ref).max() <= 1e-12, f"item {i} {name}"
