"""Max |logit - oracle| of the bf16 mode at C2 shape on a candidate sample
(the precision margin against the north-star 2e-3 budget)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2506_02267_b200 as P  # noqa: E402
from helpers import from_user  # noqa: E402
from oracle import seqrank_oracle as orc  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
Pd = orc.model_init(0, seq_len=nn.seq_len)
worst = 0.0
for seed in (7, 8):
    r = P.generate_requests(1, 1000, ll_tokens=16384, seed=seed)[0]
    logits = eng.rank_requests([(r.user, r.candidates, r.ctx)], mode="bf16")
    sample = np.arange(0, 1000, 25)
    lg = orc.rank_request(from_user(r.user), r.candidates[sample], r.ctx, Pd, (32, 96, 32, 32))
    err = np.abs(logits[sample] - lg)
    worst = max(worst, float(err.max()))
    print(f"seed {seed}: max |dlogit| {err.max():.3g}  p99 {np.percentile(err, 99):.3g}  mean {err.mean():.3g}")
print(f"worst {worst:.3g} (budget 2e-3)")
