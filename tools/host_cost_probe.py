"""Per-request host cost of the serving path's pieces (C2 request), each
timed in a loop on the GPU box: where the batcher thread's time goes."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2506_02267_b200 as P  # noqa: E402
from paper_2506_02267_b200 import serving as S  # noqa: E402
from paper_2506_02267_b200.dataset import context_features  # noqa: E402
from paper_2506_02267_b200.runtime import Capacity, Engine, _Pack  # noqa: E402

nn = P.NNConfig()
model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
eng = Engine(model, capacity=Capacity(1, 1000, 16896))
r = P.synthetic_requests(1, 1000, 16384, 256, 256, seed=0)[0]
req = [(r.user, r.candidates, r.ctx)]


def t(name, fn, n=300):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:28s} {(time.perf_counter() - t0) / n * 1e6:8.1f} us", flush=True)


t("context_features", lambda: context_features(7, 8))
t("np.asarray cands", lambda: np.asarray(r.candidates, np.float32))
t("engine.fits", lambda: eng.fits(req))
t("_Pack", lambda: _Pack(req))
t("engine.stream()", eng.stream)


def sub_wait_collect():
    slot, n, keep = eng.submit(req)
    eng.wait(slot)
    eng.collect(slot, n)


def sub_only():
    slot, n, keep = eng.submit(req)
    return slot, n, keep


t("submit+wait+collect", sub_wait_collect, 100)
t0 = time.perf_counter()
ts = []
for _ in range(50):
    a = time.perf_counter()
    slot, n, keep = eng.submit(req)
    ts.append(time.perf_counter() - a)
    eng.wait(slot)
print(f"{'submit alone':28s} {np.median(ts) * 1e6:8.1f} us (median)")
logits = np.random.default_rng(0).standard_normal((1000, 4)).astype(np.float32)
t("_response", lambda: S._response(np.arange(1000, dtype=np.uint64), logits, model.config.heads, False))
st = S.LatencyStats(window=3600.0)
t("stats.record", lambda: st.record("forward", 1e-4))
t("time.monotonic", time.monotonic)

# the copy tav2_stage does: the request's columns into a pinned arena
import torch  # noqa: E402

cols = [b.embeddings for b in (r.user.lifelong, r.user.realtime, r.user.impression)] + [r.candidates]
cols += [b.actions for b in (r.user.lifelong, r.user.realtime, r.user.impression)]
cols += [b.surfaces for b in (r.user.lifelong, r.user.realtime, r.user.impression)]
nbytes = sum(c.nbytes for c in cols)
pinned = torch.empty(nbytes + 4096, dtype=torch.uint8, pin_memory=True).numpy()
plain = np.empty_like(pinned)


def copy_into(dst):
    o = 0
    for c in cols:
        b = c.reshape(-1).view(np.uint8)
        dst[o:o + b.size] = b
        o += b.size


t(f"numpy copy {nbytes >> 10} KB -> pinned", lambda: copy_into(pinned))
t(f"numpy copy {nbytes >> 10} KB -> pageable", lambda: copy_into(plain))
t("eng.stage (tav2_stage)", lambda: eng.stage(req))

import ctypes  # noqa: E402

pk = _Pack(req)
nn_ = ctypes.c_int32()
sid = eng.stream()
t("raw tav2_stage (ctypes)", lambda: eng._lib.tav2_stage(eng._ctx, pk.arr, 1, sid, ctypes.byref(nn_)))
t("eng.stage again", lambda: eng.stage(req))
