"""Host-side cost of the synchronous rank path at C2: _Pack (Python), tav2_stage
(C++ packing into the pinned arena + H2D enqueue) and the whole tav2_rank."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import runtime as R  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.synthetic_requests(1, 1000, 16384, 256, 256, seed=0)[0]
reqs = [(r.user, r.candidates, r.ctx)]
for _ in range(20):
    eng.rank_requests(reqs)
torch.cuda.synchronize()


def med(f, n=200):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts))


print(f"_Pack            {med(lambda: R._Pack(reqs)):8.1f} us")
print(f"stage            {med(lambda: (eng.stage(reqs), torch.cuda.synchronize())):8.1f} us (incl. H2D + sync)")
print(f"rank_requests    {med(lambda: eng.rank_requests(reqs)):8.1f} us")
