"""Logit error of the folded tensor-core SKUT (skut_tc3's algorithm) under
split-precision operand formats, emulated in numpy against the oracle's f32
forward on C2 inputs (reference generator, seed 0):

  bf16x3 : a.b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi, bf16 parts (bf16 mode)
  fp16x3 : the same with fp16 parts (11-bit significands: ~2^-22 per product)
  ... with the softmax shift = the single-pass Cauchy-Schwarz bound m_cs
  (bf16 mode), the true row max (two-pass), or max(s_rr, m_cs - 15) (the
  row's diagonal score: skut_tc3's fp32 mode) -- fp16 P underflows under a
  loose shift.

Usage: python tools/split_precision_err.py [n_candidates]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from oracle import seqrank_oracle as orc  # noqa: E402

LOG2E = 1.4426950408889634


def rnd_bf16(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def rnd_fp16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


def split(x, rnd):
    hi = rnd(x)
    lo = rnd(np.asarray(x, np.float32) - hi)
    return hi, lo


def mm3(a, b, rnd):
    ah, al = split(a, rnd)
    bh, bl = split(b, rnd)
    f = lambda u, v: (u.astype(np.float64) @ v.astype(np.float64))  # noqa: E731
    return (f(ah, bh) + f(ah, bl) + f(al, bh)).astype(np.float32)


def ln(x, g, b):
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    return (xc / np.sqrt(var + np.float32(1e-5)) * g + b).astype(np.float32)


def forward(F, mask, Pd, rnd, true_max, stats=None):
    x = F.astype(np.float32).copy()
    B, S, d = x.shape
    allowed = np.tril(np.ones((S, S), bool))[None] & mask[:, None, :]
    for L in orc._layers(Pd):
        wqk = (L["wq"].astype(np.float64) @ L["wk"].T.astype(np.float64) * LOG2E / 8).astype(np.float32)
        wvo = (L["wv"].astype(np.float64) @ L["wo"].astype(np.float64)).astype(np.float32)
        a = ln(x, L["ln1_scale"], L["ln1_shift"]) * mask[:, :, None]
        q = mm3(a, wqk, rnd)
        v = mm3(a, wvo, rnd)
        s = np.stack([mm3(q[i], a[i].T, rnd) for i in range(B)])
        an = np.sqrt((a * a).sum(-1).max(-1))[:, None, None]
        m_cs = np.sqrt((q * q).sum(-1, keepdims=True)) * an
        if true_max == "max":
            m = np.where(allowed, s, -np.inf).max(-1, keepdims=True)
            m = np.where(np.isfinite(m), m, 0)
        elif true_max == "diag":  # skut_tc3 fp32 mode: m' = max(s_rr, m_cs - 15)
            srr = np.einsum("bsd,bsd->bs", q, a)[:, :, None]
            m = np.maximum(srr, m_cs - 15)
            if stats is not None:
                stats.append(float(np.mean((m_cs - 15 > srr)[mask])))
        else:
            m = m_cs
        p = np.where(allowed, np.exp2(s - m), 0).astype(np.float32)
        lsum = p.sum(-1, keepdims=True)
        o = np.stack([mm3(p[i], v[i], rnd) for i in range(B)])
        x = x + np.where(lsum > 0, o / np.where(lsum > 0, lsum, 1), 0)
        f = ln(x, L["ln2_scale"], L["ln2_shift"]) * mask[:, :, None]
        h = np.maximum(mm3(f, L["w1"], rnd), 0)
        x = x + mm3(h, L["w2"], rnd)
    return x * mask[:, :, None]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    r = P.synthetic_requests(1, n, 16384, 256, 256, seed=0)[0]
    user = {f"{s}_{c}": getattr(b, a) for s, b in zip(("ll", "rt", "imp"), r.user.blocks())
            for c, a in (("emb", "embeddings"), ("action", "actions"), ("surface", "surfaces"), ("ts", "timestamps"))}
    Pd = orc.model_init(0, seq_len=192)
    ref, det = orc.rank_request(user, r.candidates, r.ctx, Pd, (32, 96, 32, 32), return_detail=True)
    F, mask = det["features"], det["mask"]
    ctx = np.broadcast_to(r.ctx, (n, 8))
    for name, rnd in (("bf16x3", rnd_bf16), ("fp16x3", rnd_fp16)):
        for tm in ("cs", "max", "diag"):
            st = []
            U = forward(F, mask, Pd, rnd, tm, st)
            # pool GEMM in the same split format, head in f32
            y = np.stack([mm3(U[i], Pd["encoder.out_linear"], rnd) for i in range(n)])
            ym = np.where(mask[:, :, None], y, -np.inf)
            pooled = ym.max(1)
            pooled[~mask.any(1)] = 0
            z = np.concatenate([pooled, orc.unit_rows(r.candidates), ctx], 1)
            h = np.maximum(z @ Pd["head.w1"] + Pd["head.b1"], 0)
            lg = h @ Pd["head.w2"] + Pd["head.b2"]
            err = np.abs(lg - ref)
            extra = f"  (rows shifted by m_cs - 15: {max(st):.2%})" if st else ""
            print(f"{name:7s} shift={tm:4s}: max |dlogit| {err.max():.3g}  p99 {np.quantile(err, 0.99):.3g}{extra}")


if __name__ == "__main__":
    main()
