"""Measure |bf16x3 tensor-core dot - f64 dot| for unit vectors (K=32) using
the tcgen05 self-test MMA (three hi/lo terms summed on the host)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2506_02267_b200 import _native as N

def mma(A, B):
    D = torch.empty((128, B.shape[0]), dtype=torch.float32, device="cuda")
    rc = N.lib().tav2_tc_selftest(0, A.data_ptr(), B.data_ptr(), D.data_ptr(), B.shape[0], 32, 0)
    assert rc == 0
    return D.double().cpu().numpy()

rng = np.random.default_rng(0)
worst = 0.0
for it in range(20):
    a = rng.normal(size=(128, 32)).astype(np.float32); a /= np.linalg.norm(a, axis=1, keepdims=True)
    b = rng.normal(size=(256, 32)).astype(np.float32); b /= np.linalg.norm(b, axis=1, keepdims=True)
    if it % 2: b[:128] = a + rng.normal(scale=1e-3, size=a.shape).astype(np.float32)  # near-parallel
    ta, tb = torch.from_numpy(a), torch.from_numpy(b)
    ah = ta.bfloat16(); al = (ta - ah.float()).bfloat16()
    bh = tb.bfloat16(); bl = (tb - bh.float()).bfloat16()
    approx = mma(ah.cuda(), bh.cuda()) + mma(ah.cuda(), bl.cuda()) + mma(al.cuda(), bh.cuda())
    exact = a.astype(np.float64) @ b.astype(np.float64).T
    worst = max(worst, np.abs(approx - exact).max())
print(f"max |bf16x3 - f64| over unit vectors: {worst:.3e}")
