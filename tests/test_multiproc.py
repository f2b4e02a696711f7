"""N>1 host logic on CPU with gloo, world_size 2: request sharding is a
partition, and the candidate-split all-gather reassembles a request exactly
(bit-for-bit equal to scoring it unsplit).  The scorer here is the CPU
oracle's pool+head over fixed sequences so the test needs no GPU."""
import os
import socket

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


def _scorer(cands):
    """Deterministic per-candidate scorer (independent rows, like the path)."""
    w = np.random.default_rng(5).normal(size=(32, 4)).astype(np.float32)
    # explicit per-row reduction: bit-identical however the rows are sliced
    return np.tanh((cands[:, :, None] * w[None]).sum(1)).astype(np.float32)


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


@pytest.mark.parametrize("n", [7, 8192])
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
