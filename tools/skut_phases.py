"""Per-segment clock64 accounting of the tensor-core SKUT (skut_tc3, CTA 0,
the two tile leaders = row thread + MMA issuer), averaged over the
candidates CTA 0 scores at C2.  Uses the debug library (TAV2_DEBUG=1)."""
import os
import sys

os.environ["TAV2_DEBUG"] = "1"

import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import _native as N  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

NAMES = ["encode", "encode barrier", "kvfree wait", "P1 LN1->A,K", "issue M1 QV'", "wait M1",
         "P2 Q'->A,V'->smem", "kvready+issue M2 S", "wait M2", "P3 softmax", "issue M3 PV",
         "wait M3", "P4 x+=O'/l,LN2", "issue M4 W1", "wait M4", "P5 ReLU", "issue M5 W2", "wait M5",
         "P6 x+=", "pool x->A", "issue pool", "wait pool", "max-pool+barriers", "head",
         "P3a kvready wait", "P3b exp loop", "P3c zero fill", "(M3 issue alone, in 10)",
         "M1 simt wait", "M3 simt wait", "M4 simt wait"]

n_cand = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, n_cand, 16896))
r = P.synthetic_requests(1, n_cand, 16384, 256, 256, seed=0)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((n_cand, 4), device="cuda")
for _ in range(3):
    eng.run_staged("bf16", logits)
torch.cuda.synchronize()
buf = torch.zeros(1024, dtype=torch.int64, device="cuda")
N.lib().tav2_debug_timeline(buf.data_ptr(), 0)
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
N.lib().tav2_debug_timeline(None, 0)
t = buf.cpu().numpy()[640:704]
for tile in (0, 1):
    s = t[32 * tile: 32 * tile + 32]
    items = max(int(s[31]), 1)
    tot = sum(int(v) for v in s[:27]) + sum(int(v) for v in s[28:31])
    print(f"tile {tile}: {items} items, {tot / items:.0f} cycles/item")
    for i, nm in enumerate(NAMES):
        print(f"  {i:2d} {nm:20s} {s[i] / items:8.0f} cyc/item  {100 * s[i] / max(tot, 1):5.1f}%")
