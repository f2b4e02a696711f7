"""Would two requests' launch chains overlap usefully?  Pipelined serving
throughput at C2 with (a) one Engine (its two staging slots on one compute
stream: request i+1's chain starts after request i's SKUT), (b) two Engines
on two compute streams, requests alternating (request i+1's NN chain can run
on the SMs request i's SKUT tail frees), (c) device-only: run_staged
alternating on the two engines' streams with no host work."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
reqs = P.synthetic_requests(4, 1000, 16384, 256, 256, seed=0)
packed = [[(r.user, r.candidates, r.ctx)] for r in reqs]
cap = Capacity(1, 1000, 16896)
e = [Engine(model, capacity=cap), Engine(model, capacity=cap)]
st = [torch.cuda.Stream(), torch.cuda.Stream()]
STEPS = 400

# (a) one engine, the library's own two-slot pipeline
e[0].rank_pipelined([packed[i % 4] for i in range(20)])
t0 = time.perf_counter()
e[0].rank_pipelined([packed[i % 4] for i in range(STEPS)])
ta = time.perf_counter() - t0
print(f"(a) one engine pipelined: {STEPS * 1000 / ta / 1e6:.3f} M cand/s")


def two(steps):
    pend = []
    for i in range(steps):
        k = i % 2
        with torch.cuda.stream(st[k]):
            slot, n, pack = e[k].submit(packed[i % 4])
        pend.append((k, slot, n, pack))
        if len(pend) > 2:
            k0, s0, n0, _ = pend.pop(0)
            e[k0].collect(s0, n0)
    for k0, s0, n0, _ in pend:
        e[k0].collect(s0, n0)


two(20)
torch.cuda.synchronize()
t0 = time.perf_counter()
two(STEPS)
tb = time.perf_counter() - t0
print(f"(b) two engines, two streams: {STEPS * 1000 / tb / 1e6:.3f} M cand/s")

# (c) device only
for k in range(2):
    e[k].stage(packed[k])
lg = [torch.empty((1000, 4), device="cuda") for _ in range(2)]
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(STEPS):
        k = i % 2
        with torch.cuda.stream(st[k]):
            e[k].run_staged("bf16", lg[k])
    torch.cuda.synchronize()
    tc = time.perf_counter() - t0
print(f"(c) device-only, two streams alternating: {STEPS * 1000 / tc / 1e6:.3f} M cand/s")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(STEPS):
    with torch.cuda.stream(st[0]):
        e[0].run_staged("bf16", lg[0])
torch.cuda.synchronize()
td = time.perf_counter() - t0
print(f"(d) device-only, one engine back to back: {STEPS * 1000 / td / 1e6:.3f} M cand/s")
