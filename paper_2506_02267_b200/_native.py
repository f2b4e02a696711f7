"""ctypes binding of the C ABI in include/tav2.h.

The library is the only compute path: if it cannot be loaded the package
raises instead of falling back to anything else.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .core import ValidationError

HERE = os.path.dirname(os.path.abspath(__file__))
# TAV2_DEBUG=1 selects the timeline-instrumented build (tools/*_timeline.py)
# TAV2_LIB=x selects an A/B experiment build libtav2_x.so (build.build(variant=...))
LIB_PATH = os.path.join(HERE, "_lib", f"libtav2_{os.environ['TAV2_LIB']}.so" if os.environ.get("TAV2_LIB")
                        else "libtav2_debug.so" if os.environ.get("TAV2_DEBUG") == "1"
                        else "libtav2.so")

TAV2_OK, TAV2_EINVAL, TAV2_ECUDA, TAV2_ECAP, TAV2_ESTATE = 0, 1, 2, 3, 4
MODE_FP32, MODE_BF16 = 0, 1
MODES = {"fp32": MODE_FP32, "bf16": MODE_BF16}

EXPORTS = (
    "tav2_create", "tav2_destroy", "tav2_load_params", "tav2_stage", "tav2_nn_select",
    "tav2_encode", "tav2_forward", "tav2_score", "tav2_rank", "tav2_run_staged",
    "tav2_last_launch_count", "tav2_last_error", "tav2_build_info", "tav2_set_profiling",
    "tav2_kernel_times", "tav2_tc_selftest", "tav2_debug_timeline", "tav2_debug_cta",
    "tav2_rank_submit", "tav2_rank_collect",
    "tav2_store_reserve", "tav2_store_put", "tav2_store_remove", "tav2_store_count",
    "tav2_similarity", "tav2_pool", "tav2_rank_wait", "tav2_graph_info", "tav2_forward_masked",
    "tav2_stage_slots",
)


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "embed_dim", "seq_len", "ffn_dim", "num_layers", "action_rows", "surface_rows",
        "ctx_dim", "hidden_dim", "recent", "k_lifelong", "k_realtime", "k_impression")]


class Capacity(ctypes.Structure):
    _fields_ = [("max_requests", ctypes.c_int32), ("max_items", ctypes.c_int32),
                ("max_tokens", ctypes.c_int64)]


class Request(ctypes.Structure):
    _fields_ = [
        ("emb", ctypes.c_void_p * 3),
        ("action", ctypes.c_void_p * 3),
        ("surface", ctypes.c_void_p * 3),
        ("len", ctypes.c_int32 * 3),
        ("candidates", ctypes.c_void_p),
        ("n_cand", ctypes.c_int32),
        ("ctx", ctypes.c_void_p),
        ("from_store", ctypes.c_int32),
        ("store_user", ctypes.c_uint64),
    ]


class NativeError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libtav2.so once; fail loudly if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} not found: build it with `python -m paper_2506_02267_b200.build` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
            L.tav2_create.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(Capacity), ctypes.c_int,
                                      ctypes.POINTER(vp)]
            L.tav2_destroy.argtypes = [vp]
            L.tav2_load_params.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_char_p),
                                           ctypes.POINTER(vp), ctypes.POINTER(i64)]
            L.tav2_stage.argtypes = [vp, ctypes.POINTER(Request), ctypes.c_int, vp,
                                     ctypes.POINTER(i32)]
            L.tav2_nn_select.argtypes = [vp, ctypes.c_int, vp, vp, vp]
            L.tav2_encode.argtypes = [vp, vp, vp, vp, vp]
            L.tav2_similarity.argtypes = [vp, i32, i32, vp, vp]
            L.tav2_pool.argtypes = [vp, vp, vp, i32, vp, vp]
            L.tav2_forward.argtypes = [vp, ctypes.c_int, vp, vp, i32, vp, vp]
            L.tav2_forward_masked.argtypes = [vp, ctypes.c_int, vp, vp, vp, i32, i32, vp, vp]
            L.tav2_score.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp]
            L.tav2_rank.argtypes = [vp, ctypes.POINTER(Request), ctypes.c_int, ctypes.c_int, vp, vp,
                                    vp]
            L.tav2_run_staged.argtypes = [vp, ctypes.c_int, vp, vp]
            L.tav2_rank_submit.argtypes = [vp, ctypes.POINTER(Request), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           vp, ctypes.POINTER(i32)]
            L.tav2_rank_collect.argtypes = [vp, ctypes.c_int, vp, vp]
            L.tav2_rank_wait.argtypes = [vp, ctypes.c_int]
            L.tav2_graph_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
            L.tav2_store_reserve.argtypes = [vp, i32]
            L.tav2_store_put.argtypes = [vp, ctypes.c_uint64, ctypes.POINTER(Request)]
            L.tav2_store_remove.argtypes = [vp, ctypes.c_uint64]
            L.tav2_store_count.argtypes = [vp]
            L.tav2_last_launch_count.argtypes = [vp]
            L.tav2_set_profiling.argtypes = [vp, ctypes.c_int]
            L.tav2_kernel_times.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p),
                                            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32),
                                            ctypes.c_int]
            L.tav2_debug_timeline.argtypes = [vp, ctypes.c_int]
            L.tav2_debug_cta.argtypes = [vp]
            L.tav2_tc_selftest.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
            L.tav2_stage_slots.argtypes = []
            L.tav2_last_error.restype = ctypes.c_char_p
            L.tav2_build_info.restype = ctypes.c_char_p
            for name in EXPORTS:
                getattr(L, name)  # every declared symbol must resolve
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == TAV2_OK:
        return
    msg = lib().tav2_last_error().decode()
    if rc == TAV2_EINVAL:
        raise ValidationError(msg)
    if rc == TAV2_ECAP:
        raise ValidationError(f"capacity exceeded: {msg}")
    raise NativeError(f"tav2 error {rc}: {msg}")


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()
