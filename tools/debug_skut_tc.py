"""Debug driver: forward_fused in bf16 (tcgen05) vs fp32 (SIMT) for one
NNConfig given on the command line; run each config in its own process with
a timeout so a hang is isolated."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P
from paper_2506_02267_b200.runtime import Capacity, Engine

cfg = P.NNConfig(*[int(v) for v in sys.argv[1].split(",")])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dens = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
model = P.RankingModel.init(P.ModelConfig.for_nn(cfg), seed=0)
eng = Engine(model, capacity=Capacity(1, max(n, 1), 1024))
rng = np.random.default_rng(0)
S = cfg.seq_len
F = rng.normal(0, 0.5, (n, S, 64)).astype(np.float32)
mask = rng.random((n, S)) < dens
F *= mask[:, :, None]
U32 = eng.forward(F, mask, mode="fp32")
torch.cuda.synchronize()
U16 = eng.forward(F, mask, mode="bf16")
torch.cuda.synchronize()
err = np.abs((U16 - U32) * mask[:, :, None]).max()
print(f"S={S} n={n} dens={dens}: max|U_bf16 - U_fp32| = {err:.3g}", flush=True)
