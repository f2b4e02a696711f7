"""Golden vectors for forward_fused(..., extra_mask) (encoder.py:314-462,
:366-377) from the LIVE reference.

TEST INFRASTRUCTURE ONLY (build container; the reference is not on the GPU
box).  Features and mask come from the reference's own encode_batch over a
co-batched synthetic request (default NNConfig, S = 192); two custom masks:
a shared [S, S] mask and a per-item [B, S, S] mask, each random with some
rows fully disallowed and the diagonal sometimes dropped.  The oracle must
reproduce the reference (<= 1e-6); writes tests/golden/shapes/extra_mask.npz.

Usage:  python oracle/gen_extra_mask_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from seqrank import encoder as renc  # noqa: E402
from seqrank import nnsearch as rnn  # noqa: E402

from oracle import seqrank_oracle as orc  # noqa: E402
from oracle.gen_golden import params_digest, ref_model, synthetic_users  # noqa: E402


def main():
    cfg = rnn.NNConfig()
    model = ref_model(0, cfg)
    reqs = synthetic_users(2, 700, 80, 60, 3, 5)
    batch = rnn.build_dedup_batch([(u, c, None) for _, u, c in reqs])
    seqs = rnn.fused_assemble(batch, cfg)
    F, mask = renc.encode_batch(seqs, batch.candidates, model.encoder)
    B, S = mask.shape
    rng = np.random.default_rng(17)
    e2 = rng.random((S, S)) < 0.7
    e2[5] = False  # a row with no allowed key
    e2[np.arange(0, S, 7), np.arange(0, S, 7)] = False  # some rows lose their own key
    e3 = rng.random((B, S, S)) < 0.5
    e3[0, 40] = False
    U2 = renc.forward_fused(F, mask, model.encoder, extra_mask=e2)
    U3 = renc.forward_fused(F, mask, model.encoder, extra_mask=e3)
    P = orc.model_init(0, seq_len=S)
    assert params_digest(P) == params_digest(model.named_tensors())
    m = mask[:, :, None]
    for em, U in ((e2, U2), (e3, U3)):
        O = orc.forward_fused(F, mask, P, extra_mask=em)
        err = float(np.abs((O - U) * m).max())
        assert err <= 1e-6, err
        print(f"oracle == reference forward_fused(extra_mask {em.shape}): {err:.2e}")
    out = os.path.join(REPO, "tests", "golden", "shapes", "extra_mask.npz")
    np.savez_compressed(out, F=F.astype(np.float32), mask=mask, extra2=e2, extra3=e3, U2=U2.astype(np.float32),
                        U3=U3.astype(np.float32), seed=np.array(0))
    print("wrote", out)


if __name__ == "__main__":
    main()
