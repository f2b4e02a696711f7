"""Phase timeline of the tensor-core SKUT (CTA 0, first candidate) at C2."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2506_02267_b200 as P
from paper_2506_02267_b200 import _native as N
from paper_2506_02267_b200.runtime import Capacity, Engine

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.generate_requests(1, 1000, 16384, seed=1)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((1000, 4), device="cuda")
for _ in range(3):
    eng.run_staged("bf16", logits)
torch.cuda.synchronize()
buf = torch.zeros(640, dtype=torch.int64, device="cuda")
N.lib().tav2_debug_timeline(buf.data_ptr(), 0)
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
N.lib().tav2_debug_timeline(None, 0)
t = buf.cpu().numpy()[320:]
names = ["LN1->QKV", "QKVepi->S", "softmax->PV", "O/l->Wo", "LN2->W1", "relu->W2"] * 2 + ["pool"]
t0 = t[0]
prev = t0
for p in range(13):
    simt, mma, done, allin = t[2 * p], t[2 * p + 1], t[64 + p], t[160 + p]
    print(f"{names[p]:12s} w0 simt {(simt - prev)/1e3:5.2f} us | all warps in +{(allin - simt)/1e3:5.2f} | issue {(mma - allin)/1e3:5.2f} | mma {(done - mma)/1e3:5.2f}")
    prev = done
