"""C2-sized run for compute-sanitizer: one 1000-candidate L=16384 request,
fused twice (the select-flag handover covers the first 148 candidates, the
rest go through griddepcontrol.wait), checked against the unfused path."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.generate_requests(1, 1000, 16384, seed=1)[0]
a = eng.rank_requests([(r.user, r.candidates, r.ctx)], mode="bf16")
b = eng.rank_requests([(r.user, r.candidates, r.ctx)], mode="bf16")
assert np.array_equal(a, b)
torch.cuda.synchronize()
print("C2 sanitizer run ok", a.shape, float(np.abs(a).max()))
