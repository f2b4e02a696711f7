"""Per-tile %globaltimer timeline of one NN scan work unit (both passes) at C2.

    python tools/nn_timeline.py [work_unit]
"""
import os
import sys

os.environ["TAV2_DEBUG"] = "1"  # the timeline-instrumented library

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import _native as N  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.generate_requests(1, 1000, 16384, seed=1)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((1000, 4), device="cuda")
for _ in range(3):
    eng.run_staged("bf16", logits)
torch.cuda.synchronize()
buf = torch.zeros(2048, dtype=torch.int64, device="cuda")
blk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
N.lib().tav2_debug_timeline(buf.data_ptr(), blk)
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
N.lib().tav2_debug_timeline(None, 0)
t = buf.cpu().numpy()
for p in (1, 2):
    b = 160 * (p - 1)
    t0 = t[b]
    f = lambda x: (x - t0) / 1e3 if x else float("nan")  # noqa: E731
    print(f"pass {p}: end {f(t[b + 150]):.2f} us after inputs ready")
    for i in range(32):
        if not t[b + 8 + i]:
            break
        extra = f"  mma complete {f(t[520 + 40 * (p - 1) + i]):6.2f}"
        print(f"  tile {i:2d}: copy {f(t[b + 8 + i]):6.2f}  mma {f(t[b + 40 + i]):6.2f}{extra}  "
              f"epi sees {f(t[b + 72 + i]):6.2f}  done {f(t[b + 104 + i]):6.2f}")

b = 0
t0 = t[0]
print("pass 1 per-warp: r1 ld / r1 proc / r2 ld / r2 proc / barrier / write-out, us")
for i in range(4):
    for w in range(16):
        row = [(t[1100 + (i * 16 + w) * 6 + j] - t0) / 1e3 if t[1100 + (i * 16 + w) * 6 + j] else float("nan")
               for j in range(6)]
        print(f"  tile {i} w{w}: " + " ".join(f"{x:6.2f}" for x in row))
