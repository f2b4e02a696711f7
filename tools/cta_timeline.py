"""Per-kernel CTA timeline of one C2 step (globaltimer stamps at CTA start /
end, tav2_debug_cta): when each kernel's first CTA starts, how long CTAs run,
when the last ends -- shows launch gaps, ramp and tails of the path.

    python tools/cta_timeline.py [n_candidates] [--flush]
"""
import os
import sys

os.environ["TAV2_DEBUG"] = "1"  # the timeline-instrumented library

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import _native as N  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine  # noqa: E402

KERNELS = ["prep", "nn_scan1", "nn_bound", "nn_scan2", "nn_select", "skut"]
n_cand = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1000
nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, n_cand, 16896))
r = P.synthetic_requests(1, n_cand, 16384, 256, 256, seed=0)[0]
eng.stage([(r.user, r.candidates, r.ctx)])
logits = torch.empty((n_cand, 4), device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    eng.run_staged("bf16", logits)
torch.cuda.synchronize()
buf = torch.zeros(10 * 3 * 4096, dtype=torch.int64, device="cuda")  # kernel ids 0-8 (8: SKUT item stamps)
N.lib().tav2_debug_cta(buf.data_ptr())
if "--flush" in sys.argv:
    flush.zero_()
torch.cuda.synchronize()
eng.run_staged("bf16", logits)
torch.cuda.synchronize()
N.lib().tav2_debug_cta(None)
t = buf.cpu().numpy().reshape(10, 3, 4096)
t0 = min(int(t[k, 0][t[k, 0] > 0].min()) for k in range(6) if (t[k, 0] > 0).any())
for k, name in enumerate(KERNELS):
    n = int((t[k, 0] > 0).sum())
    if not n:
        continue
    st, en, rd = t[k, 0, :n], t[k, 1, :n], t[k, 2, :n]
    us = lambda x: (x - t0) / 1e3  # noqa: E731
    line = f"{name:10s} ctas {n:5d}  launch {us(st.min()):7.2f}..{us(st.max()):7.2f}"
    if (rd > 0).all():
        line += f"  ready {us(rd.min()):7.2f}..{us(rd.max()):7.2f}"
    if (en > 0).all():
        line += f"  end {us(en.min()):7.2f}..{us(en.max()):7.2f}"
        if (rd > 0).all():
            d = (en - rd) / 1e3
            line += f"  run med {np.median(d):6.2f} max {d.max():6.2f} (argmax {int(d.argmax())})"
    print(line)

rec_t, rec_n = t[6, 0], t[6, 1]
sel = rec_t > 0
if sel.any():
    d = rec_t[sel] / 1e3
    print(f"select warps: {sel.sum()}  time med {np.median(d):.2f} p99 {np.percentile(d, 99):.2f} max {d.max():.2f} us;"
          f" survivors med {np.median(rec_n[sel]):.0f} max {rec_n[sel].max()}; slowest (item, src, n):",
          [(int(i) // 3, int(i) % 3, int(rec_n[i])) for i in np.argsort(-rec_t)[:5]])
    st_t, bi_t = t[6, 2], t[7, 0]
    for src in range(3):
        m = sel & (np.arange(len(rec_t)) % 3 == src)
        if m.any():
            print(f"  source {src}: survivors med {np.median(rec_n[m]):.0f} p90 {np.percentile(rec_n[m], 90):.0f} "
                  f"max {rec_n[m].max()}, warp time med {np.median(rec_t[m]) / 1e3:.2f} max {rec_t[m].max() / 1e3:.2f} us")
    for src in range(3):
        m = sel & (np.arange(len(rec_t)) % 3 == src) & (st_t > 0)
        if m.any():
            em_t = t[7, 1]
            print(f"  source {src}: warps {m.sum()} total med {np.median(rec_t[m]) / 1e3:.2f} us, keys staged+scored "
                  f"med {np.median(st_t[m]) / 1e3:.2f} us, threshold found med {np.median(bi_t[m]) / 1e3:.2f} us, "
                  f"emit counted med {np.median(em_t[m]) / 1e3:.2f} us, n med {np.median(rec_n[m]):.0f}")


if "--detail" in sys.argv:  # the slowest CTAs of every kernel
    for k, name in enumerate(KERNELS):
        n = int((t[k, 0] > 0).sum())
        if not n:
            continue
        st, en, rd = t[k, 0, :n], t[k, 1, :n], t[k, 2, :n]
        if not ((rd > 0).all() and (en > 0).all()):
            continue
        d = (en - rd) / 1e3
        top = np.argsort(-d)[:6]
        print(f"{name}: run > 2 us: {(d > 2).sum()} CTAs; slowest (cta, launch, ready, end, run):",
              [(int(i), round((st[i] - t0) / 1e3, 2), round((rd[i] - t0) / 1e3, 2), round((en[i] - t0) / 1e3, 2),
                round(float(d[i]), 2)) for i in top])
