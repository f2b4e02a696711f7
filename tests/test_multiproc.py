"""N>1 host logic on CPU with gloo, world_size 2: request sharding is a
partition, the candidate-split all-gather reassembles a request exactly
(bit-for-bit equal to scoring it unsplit), and ``bench.py --gpus 2`` launches
two ranks itself.  The slice scorer is the reference path (the CPU oracle's
rank_request: NN selection -> encode -> fused forward -> pool -> head) so the
test needs no GPU; the same split on the B200 engine is
tests/test_gpu_shapes.py::test_c4_split_equals_unsplit."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_02267_b200.parallel import rank_split, shard_requests, split_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


_STATE = {}


def _request():
    """A small request of the reference generator's shape (oracle user dict)."""
    if "req" not in _STATE:
        from paper_2506_02267_b200.dataset import generate_requests

        r = generate_requests(1, 8, ll_tokens=300, rt_tokens=40, imp_tokens=40, seed=3)[0]
        user = {f"{s}_{c}": getattr(b, a) for s, b in zip(("ll", "rt", "imp"), r.user.blocks())
                for c, a in (("emb", "embeddings"), ("action", "actions"), ("surface", "surfaces"),
                             ("ts", "timestamps"))}
        from oracle import seqrank_oracle as orc

        _STATE["req"] = (user, r.ctx, orc.model_init(0, seq_len=64), orc)
    return _STATE["req"]


def _scorer(cands):
    """The reference path per candidate slice: logits [m, 4] (per-candidate
    work is independent, so slicing cannot change a candidate's result)."""
    user, ctx, P, orc = _request()
    return np.asarray(orc.rank_request(user, cands, ctx, P, (16, 16, 16, 16)), np.float32)


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cands = np.random.default_rng(9).normal(size=(n, 32)).astype(np.float32)
        out = rank_split(_scorer, cands)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 33])
def test_candidate_split_allgather_equals_unsplit(n):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cands = np.random.default_rng(9).normal(size=(n, 32)).astype(np.float32)
    ref = _scorer(cands)
    for r in range(world):
        assert np.array_equal(res[r], ref)


def test_shard_requests_partition_and_bounds():
    reqs = list(range(11))
    parts = [shard_requests(reqs, r, 4) for r in range(4)]
    assert sorted(x for p in parts for x in p) == reqs
    b = split_bounds(10, 4)
    assert b == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert split_bounds(1, 3) == [(0, 1), (1, 1), (1, 1)]
    with pytest.raises(ValueError):
        shard_requests(reqs, 4, 4)


def test_bench_launches_ranks_itself():
    """``python bench.py --gpus 2`` (no torchrun around it) re-launches itself
    as two ranks; rank 0 prints one JSON line with n_gpus = 2."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, NCCL_DEBUG="WARN")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "3",
                          "--warmup", "3", "--dry-run"], capture_output=True, text=True, timeout=300,
                         env=env, cwd=repo)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
