"""Host-side logic of the package (no GPU): codec, batch building, byte
accounting, model construction/checkpoints, layout materialisation."""
import hashlib
import os

import numpy as np
import pytest

import paper_2506_02267_b200 as P
from paper_2506_02267_b200 import checkpoint, nnsearch, serving
from conftest import REPO, golden_cases, load_case
from helpers import to_user
from oracle import seqrank_oracle as orc


def test_quantize_kats():
    assert P.quantize(np.array([0.65, 0.0, -1.0, 0.325])).tolist() == [127, 0, -127, 64]
    assert float(P.dequantize(np.array([64], np.int8))[0]) == pytest.approx(0.327559, abs=1e-6)
    x = np.random.default_rng(0).uniform(-0.65, 0.65, 100000)
    assert np.abs(P.dequantize(P.quantize(x)) - x).max() <= 0.65 / 254 + 1e-7
    assert np.array_equal(P.quantize(x), orc.quantize(x))
    with pytest.raises(P.ValidationError):
        P.quantize(np.array([np.nan]))


def test_build_dedup_batch_offsets_and_bytes():
    u = P.UserSequences()
    b = P.build_dedup_batch([(u, np.zeros((2, 32)), None), (u, np.zeros((3, 32)), None)])
    assert b.offsets.tolist() == [0, 0, 1, 1, 1]
    assert [s.stop - s.start for s in b.request_slices()] == [2, 3]
    r = P.generate_requests(1, 128, 300, 40, 40)[0]
    b = P.build_dedup_batch([(r.user, r.candidates, None)])
    assert nnsearch.broadcast_sequence_bytes(b) == 128 * nnsearch.dedup_sequence_bytes(b)
    with pytest.raises(P.ValidationError):
        P.build_dedup_batch([])
    with pytest.raises(P.ValidationError):
        P.build_dedup_batch([(u, np.zeros((0, 32)), None)])


def _digest(t):
    h = hashlib.sha256()
    for k in sorted(t):
        h.update(k.encode())
        h.update(np.ascontiguousarray(t[k], "<f4").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("nn", [P.NNConfig(), P.NNConfig(32, 32, 0, 0), P.NNConfig(k_lifelong=256)])
def test_model_init_matches_reference_draw_order(nn, golden_manifest):
    m = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    assert _digest(m.named_tensors()) == _digest(orc.model_init(0, seq_len=nn.seq_len))


def test_checkpoint_roundtrip(tmp_path):
    m = P.RankingModel.init(P.ModelConfig(), seed=3)
    path = tmp_path / "m.srck"
    m.save(path)
    m2 = P.RankingModel.load(path)
    assert m2.config == m.config
    assert _digest(m2.named_tensors()) == _digest(m.named_tensors())
    raw = path.read_bytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(checkpoint.CheckpointError):
        checkpoint.load_tensors(tmp_path / "bad")


@pytest.mark.parametrize("case", golden_cases())
def test_layout_from_reference_indices(case):
    """assembled_from_indices(reference idx) == reference AssembledSequence."""
    z, reqs = load_case(case)
    cfg = P.NNConfig(*[int(v) for v in z["cfg"]])
    for i, o in enumerate(z["offsets"]):
        seq = nnsearch.assembled_from_indices(to_user(reqs[o]["user"]), z["idx"][i], cfg)
        assert np.array_equal(seq.block.embeddings, z["layout_emb"][i])
        assert np.array_equal(seq.block.timestamps, z["layout_ts"][i])
        assert np.array_equal(seq.block.actions, z["layout_action"][i])
        assert np.array_equal(seq.block.surfaces, z["layout_surface"][i])
        assert np.array_equal(seq.mask, z["mask"][i])
        assert [s.valid for s in seq.segments] == z["seg_valid"][i].tolist()


def test_nearest_rank_percentiles():
    v = list(range(1, 101))
    assert serving.nearest_rank(v, 50) == 50 and serving.nearest_rank(v, 99) == 99
    assert serving.nearest_rank([7], 99) == 7 and serving.nearest_rank([], 50) is None


def test_sigmoid_and_final_score():
    x = np.array([[-50.0, 0.0, 3.0, 50.0]], np.float32)
    np.testing.assert_allclose(serving.sigmoid(x), orc.sigmoid(x))
    r = serving._response(np.arange(1), x, P.HeadConfig(), False)
    np.testing.assert_allclose(r.final, orc.final_score(r.probs))


def test_sigmoid_bit_identical_to_the_split_form():
    """serving.sigmoid computes both branches from one exp(-|x|); the
    reference's split form (trainer.py:230-236, oracle.sigmoid) must come out
    bit for bit, in f32 and f64, at every array length (SIMD tails)."""
    rng = np.random.default_rng(11)
    for dt in (np.float32, np.float64):
        for shape in [(), (1,), (3, 4), (17, 4), (1000, 4), (8192, 4)]:
            x = (rng.standard_normal(shape) * 12).astype(dt)
            if x.size >= 4:
                x.flat[:4] = [0.0, -0.0, -110.0, 110.0]
            a, b = serving.sigmoid(x), orc.sigmoid(x)
            assert a.dtype == b.dtype and a.shape == b.shape
            assert a.tobytes() == b.tobytes(), (dt, shape)
    nan = serving.sigmoid(np.array([np.nan, 1.0], np.float32))
    assert np.isnan(nan[0]) and nan[1] == orc.sigmoid(np.array([1.0], np.float32))[0]


def test_synthetic_requests_are_valid():
    for r in P.generate_requests(3, 50, 2000, 256, 256, seed=5):
        r.user.validate()
        assert r.candidates.shape == (50, 32)
        np.testing.assert_allclose(np.linalg.norm(r.candidates, axis=1), 1, atol=1e-5)
        np.testing.assert_array_equal(r.ctx, P.context_features(r.user_id))


def test_einsum_row_norm_order_restated():
    """prep_kernel's quad_sumsq reproduces numpy's f32 einsum row norm order
    bit for bit (the reference's unit vectors, core.py:72, nnsearch.py:282)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("einsum_order", os.path.join(REPO, "tools", "einsum_order.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    q = np.random.default_rng(5).integers(-127, 128, (20000, 32)).astype(np.int8)
    x = (q.astype(np.float32) / np.float32(127)) * np.float32(0.65)
    assert np.array_equal(mod.restated(x), np.einsum("ij,ij->i", x, x, dtype=np.float32))
    c = np.random.default_rng(6).normal(size=(20000, 32)).astype(np.float32)
    assert np.array_equal(mod.restated(c), np.einsum("ij,ij->i", c, c, dtype=np.float32))
