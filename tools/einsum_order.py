"""Probe numpy's float32 einsum("ij,ij->i") summation order (the reference's
row norms, core.py:72 / nnsearch.py:282 / :317) so prep_kernel can reproduce
it bit for bit.

Rows holding 1.0 at position p and 2^-12 at two positions k1, k2 reveal the
association tree: the two 2^-24 squares survive only if they are added to
each other before either meets 1.0 (ties-to-even drops a lone 2^-24).
Prints each position's pre-combining partners, then checks the inferred
order (4 lanes of stride 4, unrolled-by-4 reverse order, (l0+l1)+(l2+l3))
against np.einsum on random dequantized rows.
"""
import sys

import numpy as np


def restated(x):
    """The inferred order (mirrors quad_sumsq in csrc/prep.cu)."""
    s = (x * x).astype(np.float32)
    lanes = []
    for ln in range(4):
        a = s[:, 12 + ln]
        for m in (8, 4, 0, 28, 24, 20, 16):
            a = (s[:, m + ln] + a).astype(np.float32)
        lanes.append(a)
    return ((lanes[0] + lanes[1]).astype(np.float32) + (lanes[2] + lanes[3]).astype(np.float32)).astype(np.float32)


def main():
    es = lambda x: np.einsum("ij,ij->i", x, x, dtype=np.float32)  # noqa: E731
    for p in (0, 5, 31):
        rows, pairs = [], []
        for k1 in range(32):
            for k2 in range(k1 + 1, 32):
                if p in (k1, k2):
                    continue
                r = np.zeros(32, np.float32)
                r[p], r[k1], r[k2] = 1.0, 2.0 ** -12, 2.0 ** -12
                rows.append(r)
                pairs.append((k1, k2))
        out = es(np.array(rows))
        comb = [pr for pr, o in zip(pairs, out) if o > 1.0]
        q = 1 if p == 0 else 0
        print(f"1.0 at {p}: partners of {q}:", sorted({b for a, b in comb if a == q} | {a for a, b in comb if b == q}))
    q = np.random.default_rng(0).integers(-127, 128, (100000, 32)).astype(np.int8)
    x = (q.astype(np.float32) / np.float32(127)) * np.float32(0.65)
    match = float(np.mean(restated(x) == es(x)))
    print(f"restated order == np.einsum on {len(x)} rows: {match:.6f}")
    return 0 if match == 1.0 else 1


if __name__ == "__main__":
    sys.exit(main())
