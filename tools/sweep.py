"""C5 sweeps: device-resident candidates/s at 1,000 candidates
for lifelong length L in {1k, 2k, 4k, 8k, 16k} (NNConfig(32, 96, 32, 32),
S = 192) and for k_ll in {32, 64, 128, 256} at L = 16,384 (S = 96 + k_ll),
plus the C3 batched shape (32 requests x 500 candidates per GPU), and fp32
mode at k_ll in {96, 128, 256}.  Inputs from the reference generator.  Writes
one JSON object per point (stdout), L2 flushed between steps."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402


def point(n_req, n_cand, L, cfg, steps=50, warmup=5, mode="bf16"):
    nn = P.NNConfig(*cfg)
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    eng = Engine(model, capacity=Capacity(n_req, n_req * n_cand, n_req * (L + 512)))
    reqs = P.synthetic_requests(n_req, n_cand, L, 256, 256, seed=3)  # the reference generator
    eng.stage([(r.user, r.candidates, r.ctx) for r in reqs])
    logits = torch.empty((n_req * n_cand, 4), device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(warmup):
        eng.run_staged(mode, logits)
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))
        st[i].record()
        eng.run_staged(mode, logits)
        en[i].record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(st, en)) / steps
    eng.set_profiling(True)
    for i in range(10):
        eng.run_staged(mode, logits)
    torch.cuda.synchronize()
    kt = {k: round(v[0] / max(v[1], 1), 4) for k, v in eng.kernel_times().items()}
    return {"mode": mode, "requests": n_req, "candidates_per_request": n_cand, "L": L, "nn": list(cfg), "S": nn.seq_len,
            "ms_per_step": round(ms, 4), "candidates_per_s": round(n_req * n_cand / (ms / 1e3), 1),
            "kernel_ms": kt}


if __name__ == "__main__":
    for L in (1024, 2048, 4096, 8192, 16384):
        print(json.dumps(dict(sweep="L", **point(1, 1000, L, (32, 96, 32, 32)))), flush=True)
    for k in (32, 64, 128, 256):
        print(json.dumps(dict(sweep="k_ll", **point(1, 1000, 16384, (32, k, 32, 32)))), flush=True)
    for k in (96, 128, 256):
        print(json.dumps(dict(sweep="k_ll fp32", **point(1, 1000, 16384, (32, k, 32, 32), mode="fp32"))), flush=True)
    print(json.dumps(dict(sweep="C3", **point(32, 500, 16384, (32, 96, 32, 32), steps=20, warmup=3))), flush=True)
