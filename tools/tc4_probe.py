"""skut_tc4 (2-CTA cluster SKUT, 192 < S <= 384) probe: logits vs the SIMT /
unfolded path (TAV2_NO_TC4=1) on reference-generator requests, and the
device-resident rate at k_ll = 128 / 256 (1 x 1000 candidates, L = 16,384)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from sweep import point  # noqa: E402

import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

for k in (128, 256):
    cfg = (32, k, 32, 32)
    nn = P.NNConfig(*cfg)
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    reqs = P.synthetic_requests(2, 300, 16384, 256, 256, seed=5)
    eng = Engine(model, capacity=Capacity(2, 600, 2 * (16384 + 512)))
    rq = [(r.user, r.candidates, r.ctx) for r in reqs]
    for mode in ("bf16", "fp32"):
        a = eng.rank_requests(rq, mode=mode)
        os.environ["TAV2_NO_TC4"] = "1"
        b = eng.rank_requests(rq, mode=mode)
        del os.environ["TAV2_NO_TC4"]
        print(json.dumps({"k_ll": k, "mode": mode, "max_dlogit_vs_fallback": float(np.abs(a - b).max()),
                          "finite": bool(np.isfinite(a).all())}), flush=True)
for k in (128, 256):
    for mode in ("bf16", "fp32"):
        print(json.dumps(dict(sweep="k_ll", **point(1, 1000, 16384, (32, k, 32, 32), mode=mode))), flush=True)
