"""Open-loop latency at fixed arrival rates through DynamicBatcher +
PipelinedHandler (bench.py's open_loop leg), repeated, with the slowest
requests' arrival times -- are tail latencies steady-state or one-off
stalls?"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(4, 4000, 4 * 16896))
pool = [[r] for r in P.synthetic_requests(4, 1000, 16384, 256, 256, seed=0)]
sw0 = sys.getswitchinterval()
runs = [(sw0, 0.5, 1), (2e-4, 0.5, 1), (sw0, 0.7, 1), (2e-4, 0.7, 1), (2e-4, 0.85, 1)]
if "--batch" in sys.argv:  # up to 2 / 4 requests per batch (max_batch in items)
    runs = [(2e-4, f, b) for f in (0.5, 0.7, 0.85, 0.95) for b in (1, 2, 4)]
for sw, frac, per_batch in runs:
    rate = frac * 5.5e6 / 1000
    sys.setswitchinterval(sw)
    r = bench._open_loop(eng, pool, "bf16", rate, seconds=2.0, per_batch=per_batch)
    sys.setswitchinterval(sw0)
    print(f"switch {sw * 1e3:.1f} ms rate {rate:.0f} req/s, <= {per_batch} req/batch: p50 {r['p50_request_ms']} p99 {r['p99_request_ms']} ms, achieved "
          f"{r['achieved_cand_s'] / 1e6:.2f}M cand/s; queueing p99 {r['stages_ms']['queueing']['p99']} "
          f"forward p99 {r['stages_ms']['forward']['p99']}", flush=True)
