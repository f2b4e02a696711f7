"""Where the SKUT's fixed cost goes (debug library, globaltimer stamps per
CTA): launch -> select flags seen (ready) -> weights landed -> first item
pooled -> last item pooled -> CTA end, for n candidates (default one round).

    python tools/skut_first_item.py [n_candidates] [--flush]
"""
import os
import sys

os.environ["TAV2_DEBUG"] = "1"

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import _native as N  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

sms = torch.cuda.get_device_properties(0).multi_processor_count
n_cand = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else sms
nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, n_cand, 16896))
r = P.synthetic_requests(1, n_cand, 16384, 256, 256, seed=0)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((n_cand, 4), device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    eng.run_staged("bf16", logits)
torch.cuda.synchronize()
buf = torch.zeros(10 * 3 * 4096, dtype=torch.int64, device="cuda")
N.lib().tav2_debug_cta(buf.data_ptr())
if "--flush" in sys.argv:
    flush.zero_()
torch.cuda.synchronize()
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
N.lib().tav2_debug_cta(None)
t = buf.cpu().numpy().reshape(10, 3, 4096)
g = min(n_cand, sms)
launch, end, ready = t[5, 0, :g], t[5, 1, :g], t[5, 2, :g]
wts, first, last = t[8, 2, :g], t[8, 0, :g], t[8, 1, :g]
lastl, gdw = t[9, 1, :g], t[9, 0, :g]
sel_end = t[4, 1][t[4, 1] > 0].max()
t0 = launch.min()
us = lambda x: (x - t0) / 1e3  # noqa: E731
q = lambda x: f"med {np.median(x):7.2f} min {x.min():7.2f} max {x.max():7.2f}"  # noqa: E731
print(f"n {n_cand}, {g} CTAs (us from the first SKUT CTA start; last select CTA ended at {us(sel_end):.2f})")
print("launch            ", q(us(launch)))
print("ready (flags)     ", q(us(ready)))
print("weights landed    ", q(us(wts)))
print("1st last layer    ", q(us(lastl)))
print("griddep_wait done ", q(us(gdw)))
print("first item pooled ", q(us(first)))
print("last item pooled  ", q(us(last)))
print("end               ", q(us(end)))
print("ready->first      ", q((first - ready) / 1e3))
print("first->last       ", q((last - first) / 1e3))
print("last->end         ", q((end - last) / 1e3))
