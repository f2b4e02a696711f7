"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; argument validation happens before any CUDA call."""
import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_2506_02267_b200 import _native as N
from paper_2506_02267_b200 import build

HEADERS = [os.path.join(REPO, "include", h) for h in ("tav2.h", "tav2_internal.h")]


def declared():
    src = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tav2_\w+)\s*\(", src, re.M)))


def test_library_builds_and_exports_header_symbols():
    build.build()
    lib = N.lib()
    names = declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(N.EXPORTS)
    assert b"sm_100a" in lib.tav2_build_info()


def test_create_validates_config_without_gpu():
    lib = N.lib()
    bad = N.Config(16, 192, 32, 2, 16, 256, 8, 64, 32, 96, 32, 32)  # embed_dim 16
    cap = N.Capacity(1, 16, 1024)
    ctx = ctypes.c_void_p()
    rc = lib.tav2_create(ctypes.byref(bad), ctypes.byref(cap), 0, ctypes.byref(ctx))
    assert rc == N.TAV2_EINVAL and b"embed_dim" in lib.tav2_last_error()
    bad = N.Config(32, 100, 32, 2, 16, 256, 8, 64, 32, 96, 32, 32)  # seq_len != sum
    assert lib.tav2_create(ctypes.byref(bad), ctypes.byref(cap), 0, ctypes.byref(ctx)) == N.TAV2_EINVAL
    with pytest.raises(Exception):
        N.check(N.TAV2_EINVAL)


def test_no_cpu_fallback_in_product_path():
    """The package must not import the oracle (test infrastructure only)."""
    pkg = os.path.join(REPO, "paper_2506_02267_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, f)).read().replace("oracle/", ""), f
