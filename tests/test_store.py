"""HBM-resident feature store: the FeatureStore front end
(serving.DeviceFeatureStore, store.py:25-72), the .tav2 reader/writer it
bulk-loads from (dataset.py:85-131), and -- on the GPU -- ranking a stored
user is identical to ranking the same user from host columns.

Golden: tests/golden/store/ref.tav2 is the reference's own write_store output
after its FeatureStore.put truncation (oracle/gen_store_golden.py).
"""
import os

import numpy as np
import pytest

import paper_2506_02267_b200 as P
from paper_2506_02267_b200 import dataset as D
from paper_2506_02267_b200.core import TokenBlock, UserSequences

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "store")


def _golden_users():
    z = dict(np.load(os.path.join(GOLD, "ref.npz")))
    users = []
    for i, uid in enumerate(z["user_ids"]):
        blks = [TokenBlock(z[f"u{i}_{n}_ts"], z[f"u{i}_{n}_action"], z[f"u{i}_{n}_surface"], z[f"u{i}_{n}_emb"])
                for n in ("ll", "rt", "imp")]
        users.append((int(uid), UserSequences(*blks)))
    return tuple(int(c) for c in z["caps"]), users


def _truncated(users, caps):
    from paper_2506_02267_b200.serving import _truncate

    return [(u, UserSequences(*[_truncate(b, c) for b, c in zip(s.blocks(), caps)])) for u, s in users]


def test_read_store_reads_reference_bytes():
    caps, users = _golden_users()
    got = D.read_store(os.path.join(GOLD, "ref.tav2"))
    want = _truncated(users, caps)  # the reference stored the cap-truncated users
    assert [u for u, _ in got] == [u for u, _ in want]
    for (_, a), (_, b) in zip(got, want):
        assert a.equals(b)


def test_write_store_bytes_equal_reference(tmp_path):
    caps, users = _golden_users()
    path = tmp_path / "x.tav2"
    D.write_store(path, _truncated(users, caps))
    assert path.read_bytes() == open(os.path.join(GOLD, "ref.tav2"), "rb").read()


def test_truncation_keeps_newest_tokens():
    caps, users = _golden_users()
    _, u = users[0]
    assert len(u.lifelong) > caps[0] and len(u.realtime) > caps[1]
    (_, t), = _truncated([users[0]], caps)
    assert np.array_equal(t.lifelong.embeddings, u.lifelong.embeddings[:caps[0]])
    assert np.array_equal(t.realtime.timestamps, u.realtime.timestamps[:caps[1]])


@pytest.mark.parametrize("bad", [b"XXXX", b"TAV2\x02\x00"])
def test_read_store_format_errors(tmp_path, bad):
    path = tmp_path / "bad.tav2"
    src = open(os.path.join(GOLD, "ref.tav2"), "rb").read()
    path.write_bytes(bad + src[len(bad):])
    with pytest.raises(D.FormatError):
        D.read_store(path)
    path.write_bytes(src + b"\x00")
    with pytest.raises(D.FormatError, match="trailing"):
        D.read_store(path)


# ---------------------------------------------------------------------------
# GPU: the resident path through the C ABI
# ---------------------------------------------------------------------------

def _engine(nn=None, max_users=8):
    from paper_2506_02267_b200.runtime import Capacity, Engine

    nn = nn or P.NNConfig()
    model = P.RankingModel.init(P.ModelConfig.for_nn(nn), seed=0)
    return Engine(model, capacity=Capacity(8, 4096, 8 * 16896))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_gpu_store_rank_equals_host_rank(mode):
    from paper_2506_02267_b200.serving import DeviceFeatureStore

    eng = _engine()
    reqs = P.generate_requests(3, 150, ll_tokens=5000, seed=21)
    store = DeviceFeatureStore(eng, max_users=4)
    for i, r in enumerate(reqs):
        store.put(100 + i, r.user)
    assert len(store) == 3 and eng.store_count() == 3
    host = [(r.user, r.candidates, r.ctx) for r in reqs]
    want, widx = eng.rank_requests(host, mode=mode, return_indices=True)
    # all from the store, and mixed (store, host, store) in one staged batch
    res = [(store.ref(100 + i), r.candidates, r.ctx) for i, r in enumerate(reqs)]
    got, gidx = eng.rank_requests(res, mode=mode, return_indices=True)
    assert np.array_equal(got, want) and np.array_equal(gidx, widx)
    mixed = [res[0], host[1], res[2]]
    got2, gidx2 = eng.rank_requests(mixed, mode=mode, return_indices=True)
    assert np.array_equal(got2, want) and np.array_equal(gidx2, widx)
    # the pipelined serving loop reads the store the same way
    out = eng.rank_pipelined([[res[0]], [res[1], res[2]]], mode=mode)
    assert np.array_equal(np.concatenate(out), want)


@pytest.mark.gpu
def test_gpu_store_replace_remove_and_capacity():
    from paper_2506_02267_b200.runtime import StoreUser
    from paper_2506_02267_b200.serving import DeviceFeatureStore

    eng = _engine()
    a, b = P.generate_requests(2, 64, ll_tokens=3000, seed=5)
    store = DeviceFeatureStore(eng, max_users=2)
    store.put(7, a.user)
    g0 = store.generation
    store.put(7, b.user)  # replaced wholesale
    assert store.generation == g0 + 1 and len(store) == 1
    got = eng.rank_requests([(store.ref(7), b.candidates, b.ctx)])
    want = eng.rank_requests([(b.user, b.candidates, b.ctx)])
    assert np.array_equal(got, want)
    store.put(8, a.user)
    with pytest.raises(P.ValidationError, match="full"):
        store.put(9, a.user)
    store.remove(8)
    store.put(9, a.user)  # the freed slot is reused
    with pytest.raises(P.ValidationError, match="not in the HBM store"):
        eng.rank_requests([(StoreUser(8), a.candidates, a.ctx)])


@pytest.mark.gpu
def test_gpu_store_load_truncates_like_reference(tmp_path):
    """Bulk load of the reference-written .tav2 (over-cap users truncated by
    the reference's FeatureStore.put) ranks like the truncated host users."""
    from paper_2506_02267_b200.serving import DeviceFeatureStore, rank_many

    caps, users = _golden_users()
    eng = _engine()
    store = DeviceFeatureStore(eng, max_users=8, ll_cap=caps[0], rt_cap=caps[1], imp_cap=caps[2])
    assert store.load(os.path.join(GOLD, "ref.tav2")) == len(users)
    cands = P.generate_requests(1, 40, ll_tokens=100, seed=3)[0].candidates
    trunc = dict(_truncated(users, caps))
    for uid, _ in users:
        got = rank_many(eng, [(uid, store.ref(uid), cands)])[0].logits
        want = rank_many(eng, [(uid, trunc[uid], cands)])[0].logits
        assert np.array_equal(got, want)
    # put() applies the same truncation to raw over-cap users
    uid, raw = users[0]
    store.put(uid, raw)
    assert store.get(uid).equals(trunc[uid])


@pytest.mark.gpu
def test_gpu_store_abi_errors():
    """tav2_store_* argument checks surface as ValidationError (the Python
    mirror truncates first; the C ABI itself rejects over-cap columns)."""
    eng = _engine()
    eng.store_reserve(2)
    r = P.generate_requests(1, 8, ll_tokens=300, seed=2)[0]
    blk = r.user.realtime
    over = UserSequences(r.user.lifelong, TokenBlock(np.concatenate([blk.timestamps] * 2),
                                                     np.concatenate([blk.actions] * 2),
                                                     np.concatenate([blk.surfaces] * 2),
                                                     np.concatenate([blk.embeddings] * 2)),
                         r.user.impression)
    with pytest.raises(P.ValidationError, match="outside"):
        eng.store_put(1, over)  # 512 real-time tokens > REALTIME_CAP
    with pytest.raises(P.ValidationError, match="not in the HBM store"):
        eng.store_remove(12345)
    eng.store_put(1, r.user)
    assert eng.store_count() == 1
    eng.store_reserve(0)  # drops every user
    assert eng.store_count() == 0
    from paper_2506_02267_b200.runtime import StoreUser

    with pytest.raises(P.ValidationError, match="not in the HBM store"):
        eng.rank_requests([(StoreUser(1), r.candidates, r.ctx)])
