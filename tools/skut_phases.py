"""Per-segment clock64 accounting of the tensor-core SKUT (CTA 0, thread 0 =
tile-0 row thread + issuer), averaged over the candidates CTA 0 scores at C2."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import _native as N  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

NAMES = {0: "encode", 1: "encode barrier", 2: "LN1->A", 3: "issue QKV", 4: "wait QKV mma",
         5: "QKV epilogue", 6: "kvready+issue S", 7: "wait S mma", 8: "softmax", 9: "issue PV",
         10: "wait PV mma", 11: "O/l->A", 12: "issue Wo", 13: "wait Wo mma", 14: "x+=, LN2->A",
         15: "issue W1", 16: "wait W1 mma", 17: "ReLU->A2", 18: "issue W2", 19: "wait W2 mma",
         20: "x+=", 21: "x->A (pool)", 22: "issue pool", 23: "wait pool mma", 24: "max-pool",
         25: "pool barrier", 26: "head", 27: "item barrier"}

n_cand = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, n_cand, 16896))
r = P.generate_requests(1, n_cand, 16384, seed=1)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((n_cand, 4), device="cuda")
for _ in range(3):
    eng.run_staged("bf16", logits)
torch.cuda.synchronize()
buf = torch.zeros(640, dtype=torch.int64, device="cuda")
N.lib().tav2_debug_timeline(buf.data_ptr(), 0)
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
N.lib().tav2_debug_timeline(None, 0)
t = buf.cpu().numpy()[320:]
items = max(int(t[63]), 1)
tot = sum(int(t[i]) for i in NAMES)
print(f"CTA 0: {items} items, {tot / items:.0f} cycles/item")
for i, nm in NAMES.items():
    print(f"  {i:2d} {nm:18s} {t[i] / items:8.0f} cyc/item  {100 * t[i] / max(tot, 1):5.1f}%")
