"""Build the native library ``_lib/libtav2.so`` (sm_100a) in-tree.

nvcc cross-compiles without a GPU, so this runs in the build container; the
resulting .so travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libtav2.so")
LIB_DEBUG = os.path.join(LIBDIR, "libtav2_debug.so")  # + per-CTA / per-phase timeline stamps
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _digest(extra: list[str]) -> str:
    h = hashlib.sha256()
    for p in sources() + sorted(
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))
    ) + [os.path.join(INCLUDE, "tav2.h")]:
        h.update(open(p, "rb").read())
    h.update(" ".join(ARCH + FLAGS + extra).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, debug: bool = False,
          variant: str | None = None, defines: tuple[str, ...] = ()) -> str:
    """Compile every .cu under csrc/ into one shared library (parallel).
    debug=True builds libtav2_debug.so with the timeline stamps compiled in
    (tools/*_timeline.py; select it with TAV2_DEBUG=1).  variant="x" with
    defines=("-DFOO",) builds libtav2_x.so for A/B experiments (select it
    with TAV2_LIB=x)."""
    os.makedirs(LIBDIR, exist_ok=True)
    lib = LIB_DEBUG if debug else LIB
    extra = (["-DTAV2_DEBUG=1"] + os.environ.get("TAV2_EXTRA_FLAGS", "").split()) if debug else []
    if variant:
        lib = os.path.join(LIBDIR, f"libtav2_{variant}.so")
        extra = extra + list(defines)
    stamp = lib + ".sha256"
    dig = _digest(extra)
    if not force and os.path.exists(lib) and os.path.exists(stamp):
        if open(stamp).read().strip() == dig:
            return lib
    objs, procs = [], []
    for src in sources():
        obj = os.path.join(LIBDIR, os.path.basename(src) + f".{os.path.basename(lib)}.o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", INCLUDE, "-Xptxas", "-v", "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
        if verbose:
            print(out)
    cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcuda"]
    out = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if out.returncode != 0:
        raise RuntimeError(f"link failed:\n{out.stdout.decode()}")
    for o in objs:
        os.remove(o)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
