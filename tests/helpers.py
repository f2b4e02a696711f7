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


def oracle_layout(user, cands, cfg):
    """The oracle's selection of one request in the device index layout:
    idx [m, S] (source-relative, RT tail offset by r, -1 padding) and the
    k-th best score of every NN segment kth [m, 4] (NaN where empty)."""
    from oracle import seqrank_oracle as orc

    segs, scores = orc.nn_select_request(user["ll_emb"], user["rt_emb"], user["imp_emb"], cands, cfg,
                                         return_scores=True)
    r, k_ll, k_rt, k_imp = cfg
    lens = (k_ll, r, k_rt, k_imp)
    starts = np.cumsum((0,) + lens[:-1])
    idx = np.full((len(cands), sum(lens)), -1, np.int32)
    kth = np.full((len(cands), 4), np.nan)
    names = ("nn_lifelong", "recent_realtime", "nn_realtime_tail", "nn_impression")
    for i, (sg, sc) in enumerate(zip(segs, scores)):
        for g in range(4):
            idx[i, starts[g]:starts[g] + len(sg[g])] = sg[g]
            if names[g] in sc and len(sc[names[g]]):
                kth[i, g] = sc[names[g]][-1]
    return idx, kth


def ref_scores_fn(user_of_item, cands):
    """Reference f64 scores of given source-relative tokens (tie windows)."""
    from oracle import seqrank_oracle as orc

    def fn(i, g, idx):
        u = user_of_item(i)
        src = {0: "ll", 2: "rt", 3: "imp"}[g]
        return orc.similarity_scores(u[f"{src}_emb"], cands[i])[idx]
    return fn
