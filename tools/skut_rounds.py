"""SKUT launch time against the number of candidate rounds (n = k x SMs):
the slope is the time per round (one candidate per CTA), the intercept the
kernel's fixed cost (launch, weight staging, first encode, tail).  Uses the
profiled pass (CUDA events around every kernel, L2 flushed before each run)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

sms = torch.cuda.get_device_properties(0).multi_processor_count
nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
rows = []
for k in [1, 2, 3, 4, 5, 6, 7, 8]:
    n_cand = k * sms
    eng = Engine(model, capacity=Capacity(1, n_cand, 16896))
    r = P.synthetic_requests(1, n_cand, 16384, 256, 256, seed=0)[0]
    eng.stage([(r.user, r.candidates, r.ctx)])
    logits = torch.empty((n_cand, 4), device="cuda")
    for _ in range(5):
        eng.run_staged("bf16", logits)
    eng.set_profiling(True)
    for i in range(50):
        flush.fill_(float(i))
        eng.run_staged("bf16", logits)
    torch.cuda.synchronize()
    kt = eng.kernel_times()
    eng.set_profiling(False)
    sk = {name: v[0] / max(v[1], 1) for name, v in kt.items()}
    rows.append((k, sk.get("skut_tc3", float("nan")), sk.get("head", float("nan"))))
    print(f"rounds {k} n {n_cand}: skut_tc3 {rows[-1][1]:.4f} ms head {rows[-1][2]:.4f} ms", flush=True)
ks = torch.tensor([r[0] for r in rows], dtype=torch.float64)
ts = torch.tensor([r[1] for r in rows], dtype=torch.float64)
A = torch.stack([ks, torch.ones_like(ks)], 1)
sol = torch.linalg.lstsq(A, ts[:, None]).solution.flatten()
print(f"fit: {sol[0] * 1e3:.2f} us per round + {sol[1] * 1e3:.2f} us fixed")
