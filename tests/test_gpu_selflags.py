"""The per-candidate select -> SKUT handover (SelFlags, tav2_common.cuh): a
fused run's SKUT CTAs start their first candidate on its three select
flags (epoch-tagged, one epoch per fused run) instead of the whole select
grid.  Flags left by earlier runs must never release a later one: the batch
size goes up and down across runs (items that a smaller run does not
rewrite keep an older epoch), the unfused entry points (tav2_nn_select /
tav2_score) run in between, and every fused result must equal the unfused
result of the same batch bit for bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import _native as N  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402


def _batch(n_cand, seed):
    r = P.generate_requests(1, n_cand, ll_tokens=16384, seed=seed)[0]
    return [(r.user, r.candidates, r.ctx)]


def _unfused(eng, batch, nn):
    """tav2_nn_select into a user buffer, then tav2_score on it (no flags)."""
    n = eng.stage(batch)
    idx = torch.empty((n, nn.seq_len), dtype=torch.int32, device=eng.torch_device)
    N.check(eng._lib.tav2_nn_select(eng._ctx, eng._mode("bf16"), N.ptr(idx), N.ptr(None), eng.stream()))
    lg = eng.score_staged(idx, mode="bf16")
    torch.cuda.synchronize()
    return lg.cpu().numpy(), idx.cpu().numpy()


def test_fused_equals_unfused_across_epochs():
    nn = P.NNConfig()
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    eng = Engine(model, capacity=Capacity(1, 1000, 16896))
    ref = Engine(model, capacity=Capacity(1, 1000, 16896))
    for step, n_cand in enumerate([1000, 120, 700, 148, 149, 1000, 3, 1000]):
        batch = _batch(n_cand, seed=100 + step)
        lg, idx = eng.rank_requests(batch, mode="bf16", return_indices=True)
        rl, ri = _unfused(ref, batch, nn)
        assert np.array_equal(idx, ri), f"step {step}: indices differ"
        assert np.array_equal(lg, rl), f"step {step}: logits differ (n={n_cand})"


def test_unfused_between_fused_runs():
    nn = P.NNConfig()
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=1)
    eng = Engine(model, capacity=Capacity(1, 1000, 16896))
    b1, b2 = _batch(1000, 7), _batch(400, 8)
    first, _ = eng.rank_requests(b1, mode="bf16", return_indices=True)
    lg2, _ = _unfused(eng, b2, nn)
    fused2, _ = eng.rank_requests(b2, mode="bf16", return_indices=True)
    assert np.array_equal(lg2, fused2)
    again, _ = eng.rank_requests(b1, mode="bf16", return_indices=True)
    assert np.array_equal(first, again)


def test_multi_request_batch_fused_equals_unfused():
    """Several requests co-batched (600 items > 148 flagged first candidates):
    the items past the first SKUT wave go through griddepcontrol.wait."""
    nn = P.NNConfig()
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=2)
    eng = Engine(model, capacity=Capacity(6, 600, 6 * 16896))
    ref = Engine(model, capacity=Capacity(6, 600, 6 * 16896))
    reqs = P.generate_requests(6, 100, ll_tokens=8192, seed=11)
    batch = [(r.user, r.candidates, r.ctx) for r in reqs]
    for _ in range(2):
        lg, idx = eng.rank_requests(batch, mode="bf16", return_indices=True)
        rl, ri = _unfused(ref, batch, nn)
        assert np.array_equal(idx, ri)
        assert np.array_equal(lg, rl)
