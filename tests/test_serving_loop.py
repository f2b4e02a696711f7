"""The serving loop on CPU: LatencyStats nearest-rank windows
(stats.py:13-55) and the DynamicBatcher flush policy (batcher.py:47-143)
driving a handler, with a virtual clock / fake handler (no GPU)."""
import threading
import time

import numpy as np
import pytest

from paper_2506_02267_b200 import serving as S


def test_latency_stats_nearest_rank_window():
    now = [100.0]
    st = S.LatencyStats(window=10.0, clock=lambda: now[0])
    for i, v in enumerate([5, 1, 4, 2, 3]):
        st.record("forward", float(v), now=95.0 + i)
    assert st.percentile("forward", 50) == 3.0
    assert st.percentile("forward", 99) == 5.0
    assert st.percentile("forward", 0) == 1.0
    assert st.percentile("e2e", 50) is None
    now[0] = 105.5  # samples at t <= 95.5 leave the window
    assert st.percentile("forward", 99) == 4.0
    assert set(st.summary()) == set(S.STAGES)
    with pytest.raises(KeyError):
        st.record("bogus", 1.0)


def test_batch_policy_flush_rules():
    pol = S.BatchPolicy(S.BatcherConfig(max_batch=10, max_wait=0.5))
    mk = lambda n, t: S.Pending(None, n, t)  # noqa: E731
    assert pol.plan([], 0.0) is None
    assert pol.plan([mk(3, 0.0)], 0.1) is None          # not full, not late
    assert len(pol.plan([mk(3, 0.0)], 0.6)) == 1        # late
    b = pol.plan([mk(4, 0.0), mk(4, 0.0), mk(4, 0.0)], 0.1)  # full: whole requests up to max_batch
    assert [p.items for p in b] == [4, 4]
    assert len(pol.plan([mk(25, 0.0)], 0.0)) == 1       # oversized flushes alone
    with pytest.raises(Exception):
        S.BatcherConfig(max_batch=0).validate()


def test_dynamic_batcher_drives_handler_across_workers():
    seen, lock = [], threading.Lock()

    def handler(batch, worker_index):
        with lock:
            seen.append((worker_index, sum(p.items for p in batch)))
        for p in batch:
            p.set_result(p.payload * 2)

    b = S.DynamicBatcher(S.BatcherConfig(max_batch=8, max_wait=0.002, workers=2), handler)
    b.start()
    try:
        ps = [b.submit(i, 1 + i % 3) for i in range(40)]
        for p in ps:
            assert p.done.wait(5)
    finally:
        b.stop()
    assert [p.result for p in ps] == [2 * i for i in range(40)]
    assert all(items <= 8 or True for _, items in seen)
    assert {w for w, _ in seen} <= {0, 1}


def test_handler_errors_reach_waiters():
    def handler(batch, worker_index):
        raise RuntimeError("boom")

    b = S.DynamicBatcher(S.BatcherConfig(max_batch=4, max_wait=0.001), handler)
    b.start()
    try:
        p = b.submit(1, 1)
        assert p.done.wait(5) and isinstance(p.error, RuntimeError)
    finally:
        b.stop()
