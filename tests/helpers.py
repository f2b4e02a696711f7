"""Shared conversions between golden fixtures / oracle dicts and the package."""
import numpy as np

from paper_2506_02267_b200.core import TokenBlock, UserSequences


def to_user(d):
    return UserSequences(*[TokenBlock(d[f"{s}_ts"], d[f"{s}_action"], d[f"{s}_surface"], d[f"{s}_emb"])
                           for s in ("ll", "rt", "imp")])


def from_user(u):
    d = {}
    for s, b in zip(("ll", "rt", "imp"), u.blocks()):
        d[f"{s}_emb"], d[f"{s}_action"], d[f"{s}_surface"], d[f"{s}_ts"] = (
            b.embeddings, b.actions, b.surfaces, b.timestamps)
    return d


def check_nn_contract(idx_gpu, idx_ref, ref_scores_fn, kth, seg_starts, seg_lens, tol=1e-6):
    """North-star index contract: per NN segment the selected sets may differ
    only in tokens whose reference score lies within `tol` of the k-th score;
    the order within a segment must then be descending storage index.
    Returns the number of tolerated tie swaps."""
    swaps = 0
    for i in range(len(idx_ref)):
        for g in (0, 2, 3):
            a, b = seg_starts[g], seg_starts[g] + seg_lens[g]
            ga, ra = idx_gpu[i, a:b], idx_ref[i, a:b]
            gv, rv = ga[ga >= 0], ra[ra >= 0]
            assert len(gv) == len(rv), f"item {i} seg {g}: {len(gv)} picks vs {len(rv)}"
            assert np.all(ga[len(gv):] == -1)
            assert np.all(np.diff(gv) < 0), f"item {i} seg {g}: not descending"
            diff = np.setxor1d(gv, rv)
            if len(diff):
                s = ref_scores_fn(i, g, diff)
                assert np.all(np.abs(s - kth[i, g]) <= tol), (
                    f"item {i} seg {g}: set differs beyond ties: {diff} {s} kth={kth[i, g]}")
                swaps += len(diff) // 2
    return swaps
