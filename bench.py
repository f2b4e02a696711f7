"""Benchmark of the serving-time ranking path (BASELINE.json metric:
candidates scored/sec at 16k lifelong seq; p50/p99 request ms).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode bf16|fp32] [--config c2|c1|c3]

One step = one request of BASELINE configs[1] (1 user, 1,000 candidates,
L=16,384, NNConfig(32, 96, 32, 32) -> S=192) through stage -> NN select ->
SKUT -> head.  N>1: ``--gpus N`` re-launches itself under
torch.distributed.run (one rank per GPU, NCCL; or the driver's own torchrun
launch is used as is); every rank scores its own independent requests (weak
scaling, no data-path collective; ``--config c3``: 32 x 500 per rank); with
``--config c4`` the ranks split one 8,192-candidate request and all-gather
its logits every step (strong scaling).  ``value`` is the aggregate over
ranks / the max-over-ranks device time.

``value``: device-resident inputs (staged once per pool request), CUDA events
around each step on the launch stream, L2 flushed between timed steps.
``e2e``: the public API ``Engine.rank_requests`` from host numpy buffers,
host->device and device->host copies inside the timed region.
``--impl reference`` times the reference's own numpy path (seqrank 0.1.0
installed in baseline/_ref; the oracle port when absent) on all host cores,
every process scoring whole 1,000-candidate requests (rank 0 only), and
prints the same metric with per-request p50/p99.
"""

from __future__ import annotations

import argparse
import gc
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "candidates scored/sec at 16k lifelong seq (1/2/4/8 B200); p50/p99 request ms"
UNIT = "candidates/s"
CONFIGS = {
    # name: (requests per step, candidates per request, LL tokens, NNConfig)
    "c2": (1, 1000, 16384, (32, 96, 32, 32)),
    "c1": (1, 64, 1024, (32, 32, 0, 0)),
    "c3": (32, 500, 16384, (32, 96, 32, 32)),
    # long tail: one request's 8,192 candidates split across the ranks, one
    # NCCL all-gather of the logits per step (strong scaling)
    "c4": (1, 8192, 16384, (32, 96, 32, 32)),
}


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, 1400.0, "fallback"


def flops_per_candidate(L, nn, d=64, f=32, layers=2, E=32, ctx=8, h=64, H=4):
    """SURVEY.md §8(d) algorithmic FLOPs per candidate."""
    r, kl, kr, ki = nn
    S = r + kl + kr + ki
    rt, imp = 256, 256
    nn_f = 2 * E * (L + max(0, rt - r) + imp)
    tf = layers * (8 * S * d * d + 2 * d * S * (S + 1) + 4 * S * d * f)
    pool = 2 * S * d * d
    head = 2 * (d + E + ctx) * h + 2 * h * H
    return dict(nn=nn_f, transformer=tf, pool=pool, head=head, total=nn_f + tf + pool + head)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler attach before the timed region starts
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm: the reference's own numpy path (seqrank 0.1.0 installed
# in baseline/_ref, kind "reference") or the oracle port (kind "port"), one
# process per host core, each scoring WHOLE requests of the workload
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(REPO, "baseline", "_ref")
_CPU_STATE = {}


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "seqrank"))


def _cpu_init(kind, seed, n_cand, L, nn):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    if kind == "reference":
        sys.path.insert(0, REF_DIR)
        from seqrank import core as rcore
        from seqrank import dataset as rdata
        from seqrank import encoder as renc
        from seqrank import nnsearch as rnn
        from seqrank import trainer as rtr

        d = rdata.generate_synthetic(rdata.SyntheticConfig(
            num_users=1, num_clusters=8, ll_tokens=L, rt_tokens=256, imp_tokens=256, chunks_per_user=1,
            chunk_size=n_cand, seed=seed))
        uid, user = d.users[0]
        cands = np.stack([e.candidate for e in d.examples]).astype(np.float32)
        cfg = rnn.NNConfig(*nn)
        model = rtr.RankingModel.init(rtr.ModelConfig(encoder=renc.EncoderConfig(seq_len=cfg.seq_len), nn=cfg),
                                      seed=0)
        ctx = np.repeat(rdata.context_features(uid)[None], n_cand, 0)

        def run():
            """The reference serving composition: build_dedup_batch
            -> fused_assemble -> encode_batch -> forward_fused -> pool + head
            (trainer.py:354-366), all through the reference's public API."""
            batch = rnn.build_dedup_batch([(user, cands, None)])
            seqs = rnn.fused_assemble(batch, cfg)
            F, mask = renc.encode_batch(seqs, batch.candidates, model.encoder)
            U = renc.forward_fused(F, mask, model.encoder)
            y = U @ model.encoder.out_linear
            ym = np.where(mask[:, :, None], y, np.array(-np.inf, y.dtype))
            pooled = ym.max(1)
            pooled[~mask.any(1)] = 0
            z = np.concatenate([pooled, rcore.l2_normalize_rows(batch.candidates), ctx], axis=1)
            h = np.maximum(z @ model.head.w1 + model.head.b1, 0)
            return h @ model.head.w2 + model.head.b2
    else:
        import paper_2506_02267_b200 as P
        from oracle import seqrank_oracle as orc

        r = P.synthetic_requests(1, n_cand, L, 256, 256, seed=seed)[0]
        user = {f"{s}_{c}": getattr(b, a) for s, b in zip(("ll", "rt", "imp"), r.user.blocks())
                for c, a in (("emb", "embeddings"), ("action", "actions"), ("surface", "surfaces"),
                             ("ts", "timestamps"))}
        Pd = orc.model_init(0, seq_len=sum(nn))

        def run():
            return orc.rank_request(user, r.candidates, r.ctx, Pd, nn)
    _CPU_STATE.update(run=run, n=n_cand)


def _cpu_step(_):
    """One whole request of the workload through the CPU reference path."""
    t = time.perf_counter()
    _CPU_STATE["run"]()
    return _CPU_STATE["n"], time.perf_counter() - t


def cpu_baseline(cfg_name, steps=3, warmup=1, budget_s=60.0, procs=None, kind=None):
    """The reference's CPU path in one process per host core
    (OPENBLAS_NUM_THREADS=1); a step = every process scores one whole
    request of the workload (C2: 1 user x 1,000 candidates, L = 16,384, the
    reference generator's inputs); timed steps stop early once `budget_s` is
    spent.  kind: "reference" (the installed reference package) when
    available, else "port" (oracle/seqrank_oracle.py)."""
    _, n_cand, L, nn = CONFIGS[cfg_name]
    kind = kind or ("reference" if reference_available() else "port")
    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    old = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        with ctx.Pool(procs, initializer=_cpu_init, initargs=(kind, 0, n_cand, L, nn)) as pool:
            for _ in range(max(1, min(warmup, 2))):
                pool.map(_cpu_step, range(procs))
            done, lats, wall, k = 0, [], 0.0, 0
            while k < max(1, steps) and (k == 0 or wall < budget_s):
                t0 = time.perf_counter()
                res = pool.map(_cpu_step, range(procs))
                wall += time.perf_counter() - t0
                done += sum(r[0] for r in res)
                lats += [r[1] for r in res]
                k += 1
    finally:
        if old is None:
            os.environ.pop("OPENBLAS_NUM_THREADS", None)
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = old
    what = ("the reference package seqrank 0.1.0 (baseline/_ref): build_dedup_batch->fused_assemble->"
            "encode_batch->forward_fused->pool->head" if kind == "reference" else
            "oracle port of build_dedup_batch->fused_assemble->encode_batch->forward_fused->pool->head")
    return {
        "value": done / wall, "unit": UNIT, "cores": procs, "kind": kind, "steps_timed": k,
        "sample": (f"{procs} processes x {k} steps x one whole request ({n_cand} candidates, L={L}, "
                   f"reference generator seed 0) through {what}, OPENBLAS_NUM_THREADS=1; "
                   f"{wall:.1f}s timed wall"),
        "per_process_cand_s": round(n_cand / statistics.median(lats), 1),
        "p50_request_ms": round(1e3 * _nearest_rank(lats, 50), 2),
        "p99_request_ms": round(1e3 * _nearest_rank(lats, 99), 2),
        "cpu_model": _cpu_model(),
    }


def _nearest_rank(values, p):
    v = sorted(values)
    return v[min(len(v), max(1, -(-p * len(v) // 100))) - 1]


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _gen_one(args):
    seed, n_cand, L = args
    import paper_2506_02267_b200 as P

    return P.synthetic_requests(1, n_cand, L, 256, 256, seed=seed)[0]


def _gen_requests(seeds, n_cand, L):
    """Requests from the reference generator, generated in parallel over the
    host cores when there are many (the generator is a per-token loop)."""
    import paper_2506_02267_b200 as P

    uniq = sorted(set(seeds))
    if len(uniq) <= 2:
        got = {s: P.synthetic_requests(1, n_cand, L, 256, 256, seed=s)[0] for s in uniq}
    else:
        with mp.get_context("spawn").Pool(min(len(uniq), os.cpu_count() or 1)) as pool:
            got = dict(zip(uniq, pool.map(_gen_one, [(s, n_cand, L) for s in uniq])))
    return [got[s] for s in seeds]


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2506_02267_b200 as P
    from paper_2506_02267_b200.runtime import Capacity, Engine
    from paper_2506_02267_b200.serving import nearest_rank

    shared = getattr(args, "share_gpu", False)
    dev_i = local_rank % torch.cuda.device_count() if shared else local_rank
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)

    def coll(t):  # gloo (--share-gpu) reduces host copies; NCCL the device tensor
        return t.cpu() if shared else t
    n_req, n_cand, L, nn_t = CONFIGS[args.config]
    split = args.config == "c4"  # candidate split of one request (parallel.rank_split's layout)
    n_total = n_cand
    if split:
        from paper_2506_02267_b200.parallel import split_bounds

        c_lo, c_hi = split_bounds(n_cand, world)[rank]
        width = max(h - l for l, h in split_bounds(n_cand, world))
        n_cand = c_hi - c_lo
    nn = P.NNConfig(*nn_t)
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    cap = Capacity(n_req, n_req * n_total, n_req * (L + 512))
    eng = Engine(model, capacity=cap, device=dev_i)
    # a pool of distinct requests per rank (different seeds per rank); the
    # candidate split shares one request across the ranks
    pool_n = max(2, args.pool)
    # the reference generator's requests (dataset.synthetic_requests, the
    # draw-for-draw port of generate_synthetic; rank 0's C2 pool = seeds 0..3,
    # pinned by tests/golden/shapes/c2_generator.json)
    base = 0 if split else 1000 * rank
    flat = _gen_requests([base + (0 if split else i * n_req + j) for i in range(pool_n) for j in range(n_req)],
                         n_total, L)
    pool = [flat[i * n_req:(i + 1) * n_req] for i in range(pool_n)]
    if split:
        packed = [[(r.user, r.candidates[c_lo:c_hi], r.ctx) for r in reqs] for reqs in pool]
    else:
        packed = [[(r.user, r.candidates, r.ctx) for r in reqs] for reqs in pool]
    mode = args.mode

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    logits = torch.empty((n_req * n_cand, 4), dtype=torch.float32, device=dev)
    gather = split and world > 1
    if gather:  # padded slices -> one all_gather_into_tensor (parallel.rank_split)
        send = torch.zeros((width, 4), dtype=torch.float32, device=dev)
        recv = torch.empty((world * width, 4), dtype=torch.float32, device=dev)

    def step():
        if gather:
            eng.run_staged(mode, send[:n_cand])
            if shared:
                r_h = torch.empty((world * width, 4), dtype=torch.float32)
                dist.all_gather_into_tensor(r_h, send.cpu())
                recv.copy_(r_h)
            else:
                dist.all_gather_into_tensor(recv, send)
        else:
            eng.run_staged(mode, logits)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- device-resident throughput (value) ----
    eng.stage(packed[0])
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with Clocks(dev_i) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))  # evict the previous step's working set from L2 (untimed)
            starts[i].record()
            step()
            ends[i].record()
        torch.cuda.synchronize()
    barrier()
    launches_per_step = eng.last_launch_count()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    # per-kernel times: a separate profiled pass (CUDA events around every
    # launch on the launch stream serialise the programmatic-dependent-launch
    # overlap, so they are kept out of the timed steps above)
    eng.set_profiling(True)
    n_prof = max(10, min(args.steps, 100))
    for i in range(n_prof):
        flush.fill_(float(i))
        eng.run_staged(mode, logits)
    torch.cuda.synchronize()
    kt = eng.kernel_times()
    prof_ms = sum(v[0] for v in kt.values()) / n_prof
    eng.set_profiling(False)
    dev_ms = sum(step_ms)
    t = coll(torch.tensor([dev_ms], dtype=torch.float64, device=dev))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    cand_step = n_req * n_cand
    job_cand = n_req * n_total if split else world * cand_step  # candidates all ranks score per step
    value = job_cand * args.steps / (max_ms / 1e3)

    # ---- end-to-end through the public API (host buffers, H2D + D2H inside) ----
    # (a) the serving loop Engine.rank_pipelined: every step's host packing,
    #     H2D copy, kernels and D2H of the logits, with step i+1's host work
    #     and H2D overlapping step i's kernels (two staging slots);
    # (b) the synchronous Engine.rank_requests, one request at a time.
    eng.rank_pipelined([packed[i % pool_n] for i in range(args.warmup)], mode=mode)
    barrier()
    torch.cuda.synchronize()
    gc.collect()  # the start-up heap (generated requests) frozen, as a serving process does
    gc.freeze()
    lat = []
    t0 = time.perf_counter()
    eng.rank_pipelined([packed[i % pool_n] for i in range(args.steps)], mode=mode, latencies=lat)
    e2e_s = time.perf_counter() - t0
    te = coll(torch.tensor([e2e_s], dtype=torch.float64, device=dev))
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = job_cand * args.steps / float(te.item())
    for i in range(min(args.warmup, 5)):
        eng.rank_requests(packed[i % pool_n], mode=mode)
    torch.cuda.synchronize()
    lat_sync = []
    n_sync = min(args.steps, 100)
    ts0 = time.perf_counter()
    for i in range(n_sync):
        ts = time.perf_counter()
        eng.rank_requests(packed[i % pool_n], mode=mode)
        lat_sync.append(time.perf_counter() - ts)
    sync_value = cand_step * n_sync / (time.perf_counter() - ts0)
    h2d = _staged_bytes(packed[0])
    d2h = cand_step * 4 * 4
    # (c) the same serving loop with the users resident in the HBM feature
    #     store (uploaded once, untimed): only candidates, ctx
    #     and the plan cross PCIe per step, the tokens are copied on device
    from paper_2506_02267_b200.runtime import StoreUser
    from paper_2506_02267_b200.serving import DeviceFeatureStore

    store = DeviceFeatureStore(eng, max_users=sum(len(b) for b in packed[:pool_n]))
    sp, uid = [], 0
    for b in packed[:pool_n]:
        refs = []
        for (u, c, x) in b:
            store.put(uid, u)
            refs.append((StoreUser(uid), c, x))
            uid += 1
        sp.append(refs)
    eng.rank_pipelined([sp[i % pool_n] for i in range(args.warmup)], mode=mode)
    torch.cuda.synchronize()
    lat_st = []
    t0 = time.perf_counter()
    eng.rank_pipelined([sp[i % pool_n] for i in range(args.steps)], mode=mode, latencies=lat_st)
    st_value = cand_step * args.steps / (time.perf_counter() - t0)
    lat_st_sync = []  # one request at a time through the store (serving latency)
    for i in range(min(args.steps, 100)):
        ts = time.perf_counter()
        eng.rank_requests(sp[i % pool_n], mode=mode)
        lat_st_sync.append(time.perf_counter() - ts)
    h2d_store = h2d - sum(u.total_tokens() for u, _, _ in packed[0]) * (32 + 2 + 1)
    eng.store_reserve(0)
    # (d) open loop: requests arrive at a fixed rate (half the pipelined e2e
    #     request rate) into the DynamicBatcher + PipelinedHandler serving
    #     loop; p50/p99 of the per-request end-to-end latency (queueing
    #     included) and of each serving stage
    open_loop = None if split else _open_loop(eng, pool, mode, rate=0.5 * e2e_value / cand_step)

    # ---- roofline of the dominant kernel ----
    fl = flops_per_candidate(L, nn_t)
    hbm, tflops, tflops_sus, src = peaks()
    dom = max(kt.items(), key=lambda kv: kv[1][0]) if kt else None
    roof = None
    if dom:
        name, (ms, n) = dom
        per_launch_ms = ms / max(n, 1)
        if name.startswith("skut_tc3"):  # the CTR head is its own kernel (head_kernel)
            work = cand_step * (fl["transformer"] + fl["pool"])
        elif name.startswith("skut"):
            work = cand_step * (fl["transformer"] + fl["pool"] + fl["head"])
        elif name.startswith("nn_"):
            work = cand_step * fl["nn"]
        else:
            work = None
        if work is not None:
            ach = work / (per_launch_ms / 1e3) / 1e12
            roof = {"kernel": name, "bound": "tensor", "achieved": round(ach, 3),
                    "peak": tflops, "unit": "TFLOP/s", "frac": round(ach / tflops, 5),
                    "peak_source": f"{src} bf16_tflops (burst)", "traffic": _traffic(name),
                    "kernel_ms_per_launch": round(per_launch_ms, 4),
                    "share_of_step": round(per_launch_ms / max(prof_ms, 1e-9), 3)}
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "strong" if split else "weak", "vs_baseline": None,
        "dtype": ("bf16x3 split GEMMs on tcgen05 (f32 accumulate); NN: fp16 tcgen05 scan + f64 exact "
                  "re-scoring" if mode == "bf16" else "fp32 SIMT transformer; NN: fp16 scan + f64 re-scoring"),
        "mode": mode, "data": "synthetic (the reference's generate_synthetic: dataset.synthetic_requests), random-init weights seed 0",
        "config": {"workload": f"{args.config}: {n_req} request(s) x {n_cand} candidates, L={L}, "
                               f"RT=256, IMP=256, NNConfig{nn_t} -> S={nn.seq_len}, 2 layers d=64",
                   "requests_per_step_per_gpu": n_req, "candidates_per_step_per_gpu": cand_step,
                   "parallelism": (f"candidate-split x{world} + NCCL all_gather of the logits per step"
                                   " (e2e: slices without the gather)" if split
                                   else f"request-sharded x{world} (no collective)"),
                   "l2": "flushed between timed steps (256 MB write, untimed)"},
        "p50_request_ms": round(nearest_rank(step_ms, 50), 4),
        "p99_request_ms": round(nearest_rank(step_ms, 99), 4),
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "Engine.rank_pipelined (tav2_rank_submit/collect)",
                "p50_request_ms": round(1e3 * nearest_rank(lat, 50), 4),
                "p99_request_ms": round(1e3 * nearest_rank(lat, 99), 4),
                "sync": {"value": round(sync_value, 1), "api": "Engine.rank_requests (tav2_rank)",
                         "p50_request_ms": round(1e3 * nearest_rank(lat_sync, 50), 4),
                         "p99_request_ms": round(1e3 * nearest_rank(lat_sync, 99), 4)},
                "store": {"value": round(st_value, 1), "h2d_bytes_per_step": h2d_store,
                          "api": "Engine.rank_pipelined over serving.DeviceFeatureStore users (HBM-resident tokens)",
                          "p50_request_ms": round(1e3 * nearest_rank(lat_st, 50), 4),
                          "p99_request_ms": round(1e3 * nearest_rank(lat_st, 99), 4),
                          "sync_p50_request_ms": round(1e3 * nearest_rank(lat_st_sync, 50), 4),
                          "sync_p99_request_ms": round(1e3 * nearest_rank(lat_st_sync, 99), 4)}},
        "open_loop": open_loop,
        "gpu_launches": launches_per_step * args.steps,
        "kernels": {k: {"ms_per_launch": round(v[0] / max(v[1], 1), 4), "launches": v[1]} for k, v in kt.items()},
        "roofline": roof,
        "clocks": clk.summary(),
    }
    return out


def _open_loop(eng, pool, mode, rate, seconds=2.0, per_batch=1):
    """Fixed-rate arrivals of the pool's requests (payload (user id,
    candidates)) through serving.DynamicBatcher + serving.PipelinedHandler."""
    from paper_2506_02267_b200 import serving as S

    users, payloads = {}, []
    for reqs in pool:
        for r in reqs:
            uid = len(payloads) + 1  # distinct ids (every generated request's user is id 1)
            users[uid] = r.user
            payloads.append((uid, r.candidates))
    n_item = len(payloads[0][1])
    stats = S.LatencyStats(window=3600.0)
    h = S.PipelinedHandler(eng, users, mode=mode, stats=stats)
    b = S.DynamicBatcher(S.BatcherConfig(max_batch=per_batch * n_item, max_wait=0.0005, workers=1), h)
    b.start()
    n = max(10, int(rate * seconds))
    # a serving process's GIL hand-off interval: the submitter, batcher and
    # completion threads each hold the GIL for microseconds, and CPython's
    # 5 ms default forced-switch interval shows up in the tail
    # (tools/open_loop_probe.py: p99 1.0-1.7 -> 0.95-1.05 ms at 50% load)
    sw0 = sys.getswitchinterval()
    sys.setswitchinterval(2e-4)
    try:
        for i in range(20):  # warm the loop
            b.submit(payloads[i % len(payloads)], n_item).done.wait(10)
        # untimed warm-up at the target rate (0.5 s): the measured window
        # starts in steady state (the first paced second showed one-off
        # multi-ms stalls: thread start-up, allocator and graph warm-up)
        t0 = time.perf_counter()
        warm = []
        for i in range(max(10, int(rate * 0.5))):
            dt = t0 + i / rate - time.perf_counter()
            if dt > 0:
                time.sleep(dt)
            warm.append(b.submit(payloads[i % len(payloads)], n_item))
        for p in warm:
            p.done.wait(30)
        stats = S.LatencyStats(window=3600.0)
        h.stats = stats
        # a serving process freezes its start-up heap: a full collection of
        # the generated request objects otherwise lands in the timed window
        gc.collect()
        gc.freeze()
        t0 = time.perf_counter()
        ps = []
        for i in range(n):
            dt = t0 + i / rate - time.perf_counter()
            if dt > 0:
                time.sleep(dt)
            ps.append(b.submit(payloads[i % len(payloads)], n_item))
        for p in ps:
            p.done.wait(30)
        wall = time.perf_counter() - t0
    finally:
        sys.setswitchinterval(sw0)
        b.stop()
        h.close()
    errors = sum(p.error is not None for p in ps)
    summ = stats.summary()
    return {"arrival_rate_req_s": round(rate, 1), "requests": n, "errors": errors,
            "offered_cand_s": round(rate * n_item, 1), "achieved_cand_s": round(n * n_item / wall, 1),
            "p50_request_ms": round(1e3 * summ["e2e"]["p50"], 4), "p99_request_ms": round(1e3 * summ["e2e"]["p99"], 4),
            "stages_ms": {k: {q: round(1e3 * v, 4) for q, v in summ[k].items() if v is not None} for k in summ},
            "api": "serving.DynamicBatcher(max_batch=1 request) + serving.PipelinedHandler"}


def _traffic(kernel):
    """DRAM bytes per launch of `kernel` (dram__bytes_read.sum + write.sum) from
    the committed ncu --set full capture summary, or None."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None


def _staged_bytes(reqs):
    """Bytes of the one H2D copy per step (token columns + candidates + ctx + plan)."""
    tok = sum(r[0].total_tokens() for r in reqs)
    n = sum(len(r[1]) for r in reqs)
    return tok * (32 + 2 + 1) + n * (32 * 4 + 4) + len(reqs) * (8 * 4 + 40)


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(nproc: int, argv: list[str]) -> int:
    """``--gpus N`` (N > 1) outside a torchrun environment: re-launch this
    script under ``torch.distributed.run``, one process per GPU on this node
    (127.0.0.1 rendezvous; RANK / LOCAL_RANK / WORLD_SIZE come from the
    launcher).  NCCL_DEBUG=INFO so the communicator set-up lines show in the
    log; rank 0 prints the one JSON line last.  Returns the exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """CPU stand-in for one rank (``--dry-run``, gloo): the launcher, the
    barrier + max-over-ranks timing and the rank-0 JSON line without a GPU
    (tests/test_multiproc.py)."""
    import torch
    import torch.distributed as dist

    n_req, n_cand, L, nn_t = CONFIGS[args.config]
    x = np.random.default_rng(rank).normal(size=(64, 64)).astype(np.float32)
    for _ in range(args.warmup):
        x = np.tanh(x @ x.T / 64)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x = np.tanh(x @ x.T / 64)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t.item())
    job = world * n_req * n_cand if args.config != "c4" else n_req * n_cand
    return {"metric": METRIC, "value": round(job * args.steps / sec, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sec / args.steps, 4),
            "higher_is_better": True, "scaling": "strong" if args.config == "c4" else "weak",
            "vs_baseline": None, "dry_run": True,
            "config": {"workload": f"{args.config} (dry run: CPU stand-in step, no GPU)",
                       "parallelism": f"x{world} ranks (gloo)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--pool", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU stand-in ranks over gloo (launcher test)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="validation only: N ranks on fewer GPUs (gloo, host-side collectives); not a scaling number")
    args = ap.parse_args()
    launched = "WORLD_SIZE" in os.environ
    if args.gpus > 1 and not launched and args.impl == "ours":
        sys.exit(launch_ranks(args.gpus, sys.argv[1:]))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if launched and world != args.gpus and rank == 0:
        print(f"bench: WORLD_SIZE={world} differs from --gpus {args.gpus}; using {world}", file=sys.stderr)

    if args.impl == "reference":
        if rank != 0:
            return
        n_req, n_cand, L, nn_t = CONFIGS[args.config]
        cb = cpu_baseline(args.config, steps=args.steps, warmup=args.warmup, budget_s=90.0)
        value = cb["value"]
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "impl": "reference",
            "n_gpus": 0, "steps": cb["steps_timed"], "warmup": max(1, min(args.warmup, 2)),
            "ms_per_step": cb["p50_request_ms"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (numpy)",
            "data": "synthetic (the reference's generate_synthetic), random-init weights seed 0",
            "config": {"workload": f"{args.config}: {n_req} request(s) x {n_cand} candidates, L={L}, "
                                   f"NNConfig{nn_t} (every process scores whole requests)"},
            "p50_request_ms": cb["p50_request_ms"], "p99_request_ms": cb["p99_request_ms"],
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                 "per_process_cand_s", "p50_request_ms", "p99_request_ms")},
            "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        if cb["kind"] == "reference":  # the oracle port on the same cores, for comparison
            port = cpu_baseline(args.config, steps=2, warmup=1, budget_s=20.0, kind="port")
            line["port"] = {k: port[k] for k in ("value", "cores", "kind", "per_process_cand_s",
                                                  "p50_request_ms", "p99_request_ms")}
        print(json.dumps(line), flush=True)
        return

    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo" if args.dry_run or args.share_gpu else "nccl", init_method="env://")
    if args.dry_run:
        out = run_dry(args, rank, world)
    else:
        import torch

        if torch.cuda.device_count() < world and not args.share_gpu:
            raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
        out = run_gpu(args, rank, world, local_rank)
        if args.share_gpu:
            out["shared_gpu"] = f"{world} ranks on {torch.cuda.device_count()} GPU(s): code-path validation, not scaling"
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(args.config, steps=2, warmup=1, budget_s=15.0)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                       "per_process_cand_s", "p50_request_ms", "p99_request_ms")}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
