"""Multi-GPU serving: one process per GPU (torch.distributed, NCCL over
NVLink/NVSwitch for the single collective, gloo in CPU tests).

* ``shard_requests``: requests are independent (fused_assemble loops over
  requests, nnsearch.py:307; scores do not depend on co-batching,
  SPEC.md:512), so a batch is split across ranks with no collective on the
  hot path.
* ``rank_split``: one oversized request (C4, e.g. 8,192 candidates) is split
  by candidates.  Every rank stages the same user sequences, scores a
  contiguous candidate slice, and one all-gather of the (n/g, 4) f32 logits
  reassembles the request in candidate order.  Per-candidate math is
  independent, so the gathered logits equal a single-GPU run bit for bit.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist


def shard_requests(requests: Sequence, rank: int, world: int) -> list:
    """Round-robin request sharding (request i -> rank i % world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    return [r for i, r in enumerate(requests) if i % world == rank]


def split_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced candidate slices [lo, hi) per rank (ragged ok)."""
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def rank_split(score_slice: Callable[[np.ndarray], np.ndarray], candidates: np.ndarray,
               group=None, device: torch.device | None = None) -> np.ndarray:
    """Score `candidates` split across the ranks of `group`.

    ``score_slice(cands_slice) -> logits [m, 4] f32`` scores this rank's
    slice (on the GPU: ``lambda c: engine.rank_requests([(user, c, ctx)])``).
    Slices are padded to a common length so a single ``all_gather_into_tensor``
    (NCCL) moves them; padding rows are dropped on reassembly.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(candidates)
    bounds = split_bounds(n, world)
    lo, hi = bounds[rank]
    width = max(h - l for l, h in bounds)
    local = np.zeros((width, 4), np.float32)
    if hi > lo:
        local[: hi - lo] = score_slice(np.ascontiguousarray(candidates[lo:hi]))
    dev = device if device is not None else torch.device("cpu")
    send = torch.from_numpy(local).to(dev)
    recv = torch.empty((world * width, 4), dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    full = recv.cpu().numpy().reshape(world, width, 4)
    return np.concatenate([full[r, : h - l] for r, (l, h) in enumerate(bounds)])
