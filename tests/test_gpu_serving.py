"""The serving loop on the GPU: batcher handlers give the
same results as ranking each request alone (co-batching independence,
SPEC.md:512), one engine per worker or a shared one; the pipelined handler
under the DynamicBatcher (this package's, and the reference's own
serving/batcher.py when the reference is installed in baseline/_ref)."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import serving as S  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402
from conftest import REPO  # noqa: E402

NN = P.NNConfig()


@pytest.fixture(scope="module")
def model():
    return P.RankingModel.init(P.ModelConfig.for_nn(NN), seed=0)


@pytest.fixture(scope="module")
def users():
    reqs = P.generate_requests(6, 8, ll_tokens=3000, seed=21)
    return {100 + i: r.user for i, r in enumerate(reqs)}


def _payloads(n, seed=4):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        uid = 100 + int(rng.integers(0, 7))  # 106 is unknown -> cold start
        out.append((uid, rng.normal(size=(int(rng.integers(1, 40)), 32)).astype(np.float32)))
    return out


def _expected(eng, users, payloads):
    exp = []
    for uid, c in payloads:
        exp.append(S.rank(eng, uid, users.get(uid), c).logits)
    return exp


def _run(batcher_cls, cfg_cls, handler, payloads):
    b = batcher_cls(cfg_cls(max_batch=64, max_wait=0.002, workers=2), handler)
    b.start()
    try:
        ps = [b.submit(p, len(p[1])) for p in payloads]
        for p in ps:
            assert p.done.wait(30), "request timed out"
    finally:
        b.stop()
    for p in ps:
        assert p.error is None, p.error
    return [p.result for p in ps]


def test_sync_handler_engine_per_worker(model, users):
    engines = [Engine(model, capacity=Capacity(16, 512, 16 * 3600)) for _ in range(2)]
    payloads = _payloads(30)
    exp = _expected(engines[0], users, payloads)
    stats = S.LatencyStats()
    res = _run(S.DynamicBatcher, S.BatcherConfig, S.batcher_handler(engines, users, stats=stats), payloads)
    for r, e, (uid, _) in zip(res, exp, payloads):
        assert np.array_equal(r.logits, e)
        assert r.cold_start == (uid not in users)
    for stage in ("queueing", "batch_prep", "forward", "e2e"):
        assert stats.percentile(stage, 50) is not None


def _batchers():
    yield S.DynamicBatcher, S.BatcherConfig
    ref = os.path.join(REPO, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "seqrank")):
        sys.path.insert(0, ref)
        from seqrank.serving import batcher as rb

        yield rb.DynamicBatcher, rb.BatcherConfig


def test_pipelined_handler_under_both_batchers(model, users):
    eng = Engine(model, capacity=Capacity(16, 512, 16 * 3600))
    payloads = _payloads(40, seed=9)
    exp = _expected(eng, users, payloads)
    for bcls, ccls in _batchers():
        stats = S.LatencyStats()
        h = S.PipelinedHandler(eng, users, stats=stats)
        try:
            res = _run(bcls, ccls, h, payloads)
        finally:
            h.close()
        for r, e in zip(res, exp):
            assert np.array_equal(r.logits, e), bcls.__module__
        s = stats.summary()
        assert all(s[k]["p50"] is not None for k in S.STAGES), s


def test_pipelined_handler_overflow_path(model, users):
    eng = Engine(model, capacity=Capacity(2, 48, 2 * 3600))  # most batches exceed it
    payloads = _payloads(12, seed=2)
    exp = _expected(Engine(model, capacity=Capacity(16, 512, 16 * 3600)), users, payloads)
    h = S.PipelinedHandler(eng, users)
    try:
        res = _run(S.DynamicBatcher, S.BatcherConfig, h, payloads)
    finally:
        h.close()
    for r, e in zip(res, exp):
        assert np.array_equal(r.logits, e)


def test_graph_replay_equals_direct_launches(model):
    """run_chain: a batch shape runs directly the first time, is captured
    as a CUDA graph the second time and replayed after -- identical logits,
    including with shapes alternating between the two staging slots and a
    fresh select-flag epoch (device word) per run."""
    eng = Engine(model, capacity=Capacity(4, 2048, 4 * 17000))
    a = P.generate_requests(1, 300, ll_tokens=16384, seed=31)
    b = P.generate_requests(2, 120, ll_tokens=5000, seed=32)
    pa = [(r.user, r.candidates, r.ctx) for r in a]
    pb = [(r.user, r.candidates, r.ctx) for r in b]
    ref_a = eng.rank_requests(pa)  # direct
    ref_b = eng.rank_requests(pb)
    for _ in range(4):  # capture, then replays; alternating shapes and slots
        assert np.array_equal(eng.rank_requests(pa), ref_a)
        assert np.array_equal(eng.rank_requests(pb), ref_b)
        assert eng.last_launch_count() == 7  # prep, scan1, bound, scan2, select, skut_tc3, head
    n_graphs, broken = eng.graph_info()
    assert not broken and n_graphs >= 2, (n_graphs, broken)
    outs = eng.rank_pipelined([pa, pb, pa, pb, pa])
    for o, r in zip(outs, [ref_a, ref_b, ref_a, ref_b, ref_a]):
        assert np.array_equal(o, r)
    # device-resident runs on one staged batch: replay == direct bit for bit
    eng.stage(pa)
    lg = torch.empty((300, 4), dtype=torch.float32, device="cuda")
    res = []
    for _ in range(4):
        eng.run_staged("bf16", lg)
        res.append(lg.cpu().numpy().copy())
    for r in res[1:]:
        assert np.array_equal(r, res[0])
    assert np.array_equal(res[0], ref_a)
