"""Where the pipelined serving loop's time goes: per request, host time in
submit (pack + H2D enqueue + launch) and collect (wait + copy out), and the
GPU-side spacing of consecutive requests (a CUDA event recorded on the
compute stream right after each submit)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
reqs = [[(r.user, r.candidates, r.ctx)] for r in P.synthetic_requests(4, 1000, 16384, 256, 256, seed=0)]
n = 200
prof = "--profile" in sys.argv
for rep in range(2):
    if prof and rep == 1:
        eng.set_profiling(True)
    evs, t_sub, t_col = [], [], []
    pending = None
    t0 = time.perf_counter()
    for i in range(n + 1):
        if i < n:
            a = time.perf_counter()
            slot, m, keep = eng.submit(reqs[i % 4])
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            evs.append(ev)
            t_sub.append(time.perf_counter() - a)
        if pending is not None:
            a = time.perf_counter()
            eng.wait(pending[0])
            eng.collect(pending[0], pending[1])
            t_col.append(time.perf_counter() - a)
        pending = (slot, m, keep) if i < n else None
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    gaps = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]
    print(f"rep {rep}: {n * 1000 / wall:.0f} cand/s; submit med {1e6 * np.median(t_sub):.0f} us, collect med "
          f"{1e6 * np.median(t_col):.0f} us; GPU spacing med {1e3 * np.median(gaps):.1f} us p90 {1e3 * np.quantile(gaps, 0.9):.1f}")
    if prof and rep == 1:
        kt = eng.kernel_times()
        print("  per-kernel us (pipelined, events around each):",
              {k: round(1e3 * v[0] / max(v[1], 1), 1) for k, v in kt.items()})
