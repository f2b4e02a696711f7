import glob
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the native CUDA path)")


def golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_case(name):
    """Golden fixture -> (arrays, requests) with requests as oracle user dicts."""
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    reqs = []
    r = 0
    offs = z["offsets"]
    while f"r{r}_ll_emb" in z:
        user = {}
        for src in ("ll", "rt", "imp"):
            for col in ("emb", "action", "surface", "ts"):
                user[f"{src}_{col}"] = z[f"r{r}_{src}_{col}"]
        sel = offs == r
        reqs.append(dict(user=user, uid=int(z["user_ids"][r]), cands=z["candidates"][sel],
                         ctx=z["ctx"][sel][0]))
        r += 1
    return z, reqs


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_manifest():
    return manifest()
