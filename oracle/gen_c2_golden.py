"""Golden fixture at the benchmarked shape (BASELINE configs[1], C2) from the
LIVE reference.

TEST INFRASTRUCTURE ONLY.  Runs in the build container, where the reference
package is importable from /root/reference/pkg/src (it does not exist on the
GPU box, so the outputs are committed as tests/golden/shapes/c2_seed0.npz).

  1. The reference generator ``generate_synthetic(SyntheticConfig(num_users=1,
     num_clusters=8, ll_tokens=16384, rt_tokens=256, imp_tokens=256,
     chunks_per_user=1, chunk_size=1000, seed=s))`` (dataset.py:335-427) is
     run for the benchmark's request seeds s = 0..3 and the package's port
     ``paper_2506_02267_b200.dataset.synthetic_requests`` must reproduce it
     bit for bit (users, candidates); the input digests are recorded, so the
     GPU box regenerates the identical requests without the reference.
  2. For seed 0 the reference path build_dedup_batch -> fused_assemble(
     return_scores=True) -> encode_batch -> forward_fused -> pool + head
     (trainer.py:354-366) runs on all 1,000 candidates; the per-item index
     layout (source-relative, RT tail offset by r, -1 padding), the k-th
     score of every NN segment, the logits and the pooled vectors are saved,
     plus the f64 scores the reference returns for the first 64 items.
  3. The oracle (oracle/seqrank_oracle.py) must reproduce the reference on
     the same request (indices exact, logits <= 1e-6).

Usage:  python oracle/gen_c2_golden.py
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

from seqrank import dataset as rdata  # noqa: E402
from seqrank import nnsearch as rnn  # noqa: E402

from oracle import seqrank_oracle as orc  # noqa: E402
from oracle.gen_golden import params_digest, ref_forward, ref_model, user_dict  # noqa: E402
from paper_2506_02267_b200 import dataset as pdata  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden", "shapes")
N_CAND, LL, RT, IMP = 1000, 16384, 256, 256
SEEDS = (0, 1, 2, 3)
N_SCORES = 64


def request_digest(user, cands, ctx) -> str:
    h = hashlib.sha256()
    for blk in (user.lifelong, user.realtime, user.impression):
        for a in (blk.timestamps, blk.actions, blk.surfaces, blk.embeddings):
            h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.ascontiguousarray(cands, np.float32).tobytes())
    h.update(np.ascontiguousarray(ctx, np.float32).tobytes())
    return h.hexdigest()


def reference_request(seed):
    d = rdata.generate_synthetic(rdata.SyntheticConfig(
        num_users=1, num_clusters=8, ll_tokens=LL, rt_tokens=RT, imp_tokens=IMP, chunks_per_user=1,
        chunk_size=N_CAND, seed=seed))
    uid, user = d.users[0]
    cands = np.stack([e.candidate for e in d.examples]).astype(np.float32)
    return uid, user, cands, rdata.context_features(uid)


def main():
    digests = {}
    reqs = {}
    for s in SEEDS:
        uid, user, cands, ctx = reference_request(s)
        port = pdata.synthetic_requests(1, N_CAND, LL, RT, IMP, seed=s)[0]
        assert port.user_id == uid
        dg = request_digest(user, cands, ctx)
        assert request_digest(port.user, port.candidates, port.ctx) == dg, f"generator port drift, seed {s}"
        digests[str(s)] = dg
        reqs[s] = (uid, user, cands, ctx)
        print(f"seed {s}: port == reference generator ({dg[:16]})")

    uid, user, cands, ctx1 = reqs[0]
    cfg = rnn.NNConfig()
    model = ref_model(0, cfg)
    batch = rnn.build_dedup_batch([(user, cands, None)])
    seqs, scores = rnn.fused_assemble(batch, cfg, return_scores=True)
    ctx = np.repeat(ctx1[None], len(batch), 0).astype(np.float32)
    F, mask, U, pooled, logits = ref_forward(model, batch, seqs, ctx)

    S = cfg.seq_len
    r = cfg.recent
    idx = np.full((N_CAND, S), -1, np.int16)
    kth = np.full((N_CAND, 4), np.nan, np.float64)
    src = {"nn_lifelong": user.lifelong, "nn_realtime_tail": user.realtime.take(np.arange(r, len(user.realtime))),
           "nn_impression": user.impression}
    kk = {"nn_lifelong": cfg.k_lifelong, "nn_realtime_tail": cfg.k_realtime, "nn_impression": cfg.k_impression}
    for i in range(N_CAND):
        start = 0
        for g, (seg, seg_len) in enumerate(zip(rnn.SEGMENT_NAMES, cfg.segment_lengths())):
            if seg == "recent_realtime":
                sel = np.arange(min(r, len(user.realtime)) - 1, -1, -1)
            else:
                d = rnn.similarity_scores(src[seg], cands[i])
                sel = rnn._nn_segment_indices(d, kk[seg])
                kth[i, g] = np.sort(d)[::-1][min(kk[seg], len(d)) - 1]
                if seg == "nn_realtime_tail":
                    sel = sel + r
            idx[i, start:start + len(sel)] = sel
            start += seg_len
    # fused_assemble's token layout == the naive per-item indices (spot check)
    for i in (0, 1, 499, 999):
        assert np.array_equal(seqs[i].block.embeddings[seqs[i].mask],
                              np.concatenate([src_blk.embeddings[ii] for src_blk, ii in (
                                  (user.lifelong, idx[i, :96][idx[i, :96] >= 0]),
                                  (user.realtime, idx[i, 96:160][idx[i, 96:160] >= 0]),
                                  (user.impression, idx[i, 160:][idx[i, 160:] >= 0]))]))

    # the oracle reproduces the reference on this request
    P = orc.model_init(0, seq_len=S)
    assert params_digest(P) == params_digest(model.named_tensors())
    lg, det = orc.rank_request(user_dict(user), cands, ctx1, P, (32, 96, 32, 32), return_detail=True)
    for i in range(N_CAND):
        flat = np.concatenate(det["segs"][i])
        assert np.array_equal(flat, idx[i][idx[i] >= 0]), f"oracle index mismatch item {i}"
    err = float(np.abs(lg - logits).max())
    assert err <= 1e-6, err
    print(f"oracle == reference at C2: indices exact, logits {err:.2e}")

    sc = np.full((N_SCORES, S), np.nan, np.float64)  # reference f64 scores, best first per segment
    for i in range(N_SCORES):
        start = 0
        for seg, seg_len in zip(rnn.SEGMENT_NAMES, cfg.segment_lengths()):
            if seg in scores[i]:
                v = scores[i][seg]
                sc[i, start:start + len(v)] = v
            start += seg_len
    np.savez_compressed(os.path.join(OUT, "c2_seed0.npz"), idx=idx, kth=kth, logits=logits.astype(np.float32),
                        pooled=pooled.astype(np.float32), scores_head=sc,
                        seg_valid=np.array([[g.valid for g in s_.segments] for s_ in seqs[:N_SCORES]], np.int32))
    with open(os.path.join(OUT, "c2_generator.json"), "w") as fh:
        json.dump({"config": dict(num_users=1, num_clusters=8, ll_tokens=LL, rt_tokens=RT, imp_tokens=IMP,
                                  chunks_per_user=1, chunk_size=N_CAND),
                   "request_sha256_by_seed": digests, "params_sha256": params_digest(P),
                   "oracle_vs_reference_logits": err}, fh, indent=1)
    print("wrote tests/golden/shapes/c2_seed0.npz, c2_generator.json")


if __name__ == "__main__":
    main()
