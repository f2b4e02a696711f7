"""Print the %globaltimer timeline of NN CTA 0 (pass 1 and pass 2) at C2."""
import sys
import numpy as np
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
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
blk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
N.lib().tav2_debug_timeline(buf.data_ptr(), blk)
eng.set_profiling(True)
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
print(eng.kernel_times())
N.lib().tav2_debug_timeline(None, 0)
allt = buf.cpu().numpy()
for ps in (0, 1):
    t = allt[160 * ps:]
    t0 = t[0]
    rel = lambda x: (x - t0) / 1000.0 if x else float("nan")
    print(f"pass {ps+1}: prologue done {rel(t[1]):.2f} us, epilogue done {rel(t[2]):.2f}, exit {rel(t[3]):.2f}")
    for i in range(0, 17, 1 if blk else 4):
        print(f"  tile {i:2d}: copy issue {rel(t[8+i]):8.2f}  full {rel(t[40+i]):8.2f}  mma {rel(t[72+i]):8.2f}  epi {rel(t[104+i]):8.2f} done {rel(t[136+i]):8.2f}")
