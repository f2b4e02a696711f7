"""Golden fixture for the HBM feature store front end.

TEST INFRASTRUCTURE ONLY.  Runs in the build container with the LIVE
reference importable from /root/reference/pkg/src: builds a few users with
the reference's own generate_synthetic (plus an over-cap real-time block and
an empty user), pushes them through the reference FeatureStore.put (cap
truncation, store.py:41-53) and write_store (dataset.py:90-103), and commits

  tests/golden/store/ref.tav2    the reference's .tav2 bytes of the stored users
  tests/golden/store/ref.npz     per user: the raw input columns and caps

so tests/test_store.py can check paper_2506_02267_b200.dataset.read_store /
write_store and serving.DeviceFeatureStore truncation against them without
the reference present.

Usage:  python oracle/gen_store_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from seqrank import core as rcore  # noqa: E402
from seqrank import dataset as rdata  # noqa: E402
from seqrank.serving import store as rstore  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden", "store")
CAPS = (3000, 200, 256)  # small lifelong / real-time caps so truncation is exercised


def main() -> None:
    cfg = rdata.SyntheticConfig(num_users=3, num_clusters=8, ll_tokens=3500, rt_tokens=256, imp_tokens=100,
                                chunks_per_user=1, chunk_size=4, seed=5)
    ds = rdata.generate_synthetic(cfg)
    users = [(int(uid), seqs) for uid, seqs in ds.users]
    users.append((424242, rcore.UserSequences(rcore.TokenBlock.empty(), rcore.TokenBlock.empty(),
                                               rcore.TokenBlock.empty())))
    st = rstore.FeatureStore(*CAPS)
    for uid, seqs in users:
        st.put(uid, seqs)
    stored = [(uid, st.get(uid)) for uid, _ in users]
    rdata.write_store(os.path.join(OUT, "ref.tav2"), stored)
    arrs = {"caps": np.array(CAPS, np.int64), "user_ids": np.array([u for u, _ in users], np.uint64)}
    for i, (uid, seqs) in enumerate(users):
        for name, blk in zip(("ll", "rt", "imp"), (seqs.lifelong, seqs.realtime, seqs.impression)):
            arrs[f"u{i}_{name}_ts"] = blk.timestamps
            arrs[f"u{i}_{name}_action"] = blk.actions
            arrs[f"u{i}_{name}_surface"] = blk.surfaces
            arrs[f"u{i}_{name}_emb"] = blk.embeddings
    np.savez_compressed(os.path.join(OUT, "ref.npz"), **arrs)
    print("users", [(u, len(s.lifelong), len(s.realtime), len(s.impression)) for u, s in stored])


if __name__ == "__main__":
    main()
