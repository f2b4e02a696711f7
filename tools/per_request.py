"""Device time per step of each of the benchmark's pool requests (C2,
reference generator seeds 0..3), CUDA events, L2 flushed between steps."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
reqs = P.synthetic_requests(4, 1000, 16384, 256, 256, seed=0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
lg = torch.empty((1000, 4), device="cuda")
out = []
for i, r in enumerate(reqs):
    eng.stage([(r.user, r.candidates, r.ctx)])
    for _ in range(10):
        eng.run_staged("bf16", lg)
    ts = []
    for _ in range(50):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run_staged("bf16", lg)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out.append(f"req{i} {np.median(ts):.4f}")
print(" ".join(out))
