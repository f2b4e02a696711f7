"""One device-resident C5 point for profiling (ncu): 1 x 1000 candidates,
L = 16,384, NNConfig(32, k_ll, 32, 32); argv: k_ll [mode] [steps]."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mode = sys.argv[2] if len(sys.argv) > 2 else "bf16"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
nn = P.NNConfig(32, k, 32, 32)
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.synthetic_requests(1, 1000, 16384, 256, 256, seed=3)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((1000, 4), device="cuda")
for _ in range(steps):
    eng.run_staged(mode, logits)
torch.cuda.synchronize()
print("ok", float(logits.abs().sum()))
