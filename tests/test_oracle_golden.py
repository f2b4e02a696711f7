"""The CPU oracle (oracle/seqrank_oracle.py) against the golden vectors the
live reference produced (oracle/gen_golden.py).  Pins the oracle before any
GPU result is compared with it."""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case
from helpers import to_user
from oracle import seqrank_oracle as orc

CASES = golden_cases()


def digest(P):
    h = hashlib.sha256()
    for k in sorted(P):
        h.update(k.encode())
        h.update(np.ascontiguousarray(P[k], "<f4").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("case", CASES)
def test_oracle_reproduces_reference(case, golden_manifest):
    z, reqs = load_case(case)
    cfg = tuple(int(v) for v in z["cfg"])
    P = orc.model_init(int(z["seed"]), seq_len=orc.seq_len(cfg))
    assert digest(P) == golden_manifest[case]["params_sha256"]
    row = 0
    for rq in reqs:
        lg, det = orc.rank_request(rq["user"], rq["cands"], rq["ctx"], P, cfg, return_detail=True)
        m = len(rq["cands"])
        for j in range(m):
            got = np.concatenate(det["segs"][j])
            exp = z["idx"][row + j][z["idx"][row + j] >= 0]
            assert np.array_equal(got, exp)
            lay = det["layout"][j]
            assert np.array_equal(lay["emb"], z["layout_emb"][row + j])
            assert np.array_equal(lay["mask"], z["mask"][row + j])
            assert np.array_equal(lay["valid"], z["seg_valid"][row + j])
        np.testing.assert_allclose(lg, z["logits"][row:row + m], atol=1e-6, rtol=0)
        row += m


@pytest.mark.parametrize("case", CASES)
def test_oracle_layered_matches_fused(case):
    """encoder.py:298-300 self-check: forward_fused == forward_reference."""
    z, _ = load_case(case)
    cfg = tuple(int(v) for v in z["cfg"])
    P = orc.model_init(int(z["seed"]), seq_len=orc.seq_len(cfg))
    F, mask = z["features_head"], z["mask"][:4]
    Uf = orc.forward_fused(F, mask, P)
    Ul = orc.forward_layered(F, mask, P)
    m = mask[:, :, None]
    assert np.abs((Uf - Ul) * m).max() <= 1e-5
    assert np.abs((Uf - z["U_head"]) * m).max() <= 1e-6


def test_kats(golden_manifest):
    k = golden_manifest["kat"]
    assert orc.quantize(np.array(k["quantize_in"])).tolist() == k["quantize_out"]
    assert float(orc.dequantize(np.array([64], np.int8))[0]) == k["dequantize_64"]
    np.testing.assert_array_equal(orc.context_features(7), np.array(k["context_7"], np.float32))


def test_topk_spec_examples():
    """dots (0.9, 0.1, 0.5), k=2 -> {0, 2}; ties -> index 0."""
    picked, seg = orc._topk_desc_storage(np.array([0.9, 0.1, 0.5]), 2)
    assert picked.tolist() == [0, 2] and seg.tolist() == [2, 0]
    picked, _ = orc._topk_desc_storage(np.array([0.9, 0.1, 0.5]), 5)
    assert picked.tolist() == [0, 2, 1]
    picked, _ = orc._topk_desc_storage(np.array([0.3, 0.3]), 1)
    assert picked.tolist() == [0]


@pytest.mark.parametrize("case", golden_cases())
def test_nn_feature_log_bytes_match_reference(case):
    """The package's record packer over the reference layout reproduces the
    reference's own pack_assembled bytes (dataset.py:138-149)."""
    import paper_2506_02267_b200 as P
    from paper_2506_02267_b200.dataset import log_nn_features

    z, reqs = load_case(case)
    nn = P.NNConfig(*[int(v) for v in z["cfg"]])
    users = [to_user(r["user"]) for r in reqs]
    recs = log_nn_features(users, z["idx"], z["offsets"], nn)
    blob, off = z["packed_assembled"].tobytes(), z["packed_offsets"]
    assert len(recs) == len(off) - 1
    for i, rec in enumerate(recs):
        assert rec == blob[off[i]:off[i + 1]], f"{case}: record {i} differs"


def test_oracle_extra_mask_matches_reference():
    """forward_fused(extra_mask) restated in the oracle == the live reference's
    output (tests/golden/shapes/extra_mask.npz, oracle/gen_extra_mask_golden.py)."""
    z = np.load(os.path.join(GOLDEN, "shapes", "extra_mask.npz"))
    P = orc.model_init(int(z["seed"]), seq_len=z["mask"].shape[1])
    m = z["mask"][:, :, None]
    for em, U in ((z["extra2"], z["U2"]), (z["extra3"], z["U3"])):
        O = orc.forward_fused(z["F"], z["mask"], P, extra_mask=em)
        assert np.abs((O - U) * m).max() <= 1e-6
