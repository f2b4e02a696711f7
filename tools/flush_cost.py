"""Per-kernel cost of a cold L2 (the bench flushes L2 between timed steps,
which also evicts every kernel's code): profiled C2 runs with and without a
256 MB write between them, and the whole chain's step time both ways."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.synthetic_requests(1, 1000, 16384, 256, 256, seed=0)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((1000, 4), device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(10):
    eng.run_staged("bf16", logits)
for fl in (True, False):
    eng.set_profiling(True)
    for i in range(100):
        if fl:
            flush.fill_(float(i))
        eng.run_staged("bf16", logits)
    torch.cuda.synchronize()
    kt = eng.kernel_times()
    eng.set_profiling(False)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
    for i in range(100):
        if fl:
            flush.fill_(float(i))
        ev[i][0].record()
        eng.run_staged("bf16", logits)
        ev[i][1].record()
    torch.cuda.synchronize()
    step = sum(a.elapsed_time(b) for a, b in ev) / 100
    print(("flushed  " if fl else "warm L2  ") + f"step {step * 1e3:7.1f} us | " +
          " ".join(f"{k} {v[0] / v[1] * 1e3:6.1f}" for k, v in kt.items()), flush=True)
