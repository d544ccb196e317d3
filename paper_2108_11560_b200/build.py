"""Build the sm_100a shared library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_2108_11560_b200.build [--force]

Produces ``paper_2108_11560_b200/libbessel_logk.so`` from ``csrc/*.cu`` with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and a static CUDA
runtime (no libcudart/libcuda link-time dependency, so the library also
loads on a CPU-only host for ABI checks).  FP64 code is compiled without
fast-math; the FP32 fast paths use explicit ``*.approx`` PTX.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbessel_logk.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-diag-suppress", "177",
    "-I", os.path.join(ROOT, "include"),
    "--shared", "-cudart", "static",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return (sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")))
            + [os.path.join(ROOT, "include", "bessel_logk.h")])


def kernel_source_sha256() -> str:
    """sha256 of everything that determines the kernels' instruction stream
    (csrc sources, the header, the build flags in this file): bench.py marks a
    roofline whose ncu counts were captured from other sources as stale."""
    import hashlib
    files = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                   + glob.glob(os.path.join(CSRC, "*.inc")))
    files += [os.path.join(ROOT, "include", "bessel_logk.h"), os.path.abspath(__file__)]
    h = hashlib.sha256()
    for f in files:
        h.update(os.path.relpath(f, ROOT).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines=()) -> str:
    """Build the library (``out``/``defines`` only for tuning variants)."""
    target = out or LIB
    if out is None and not force and not is_stale():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-o", tmp] + sources()
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


def build_diag() -> str:
    """The diagnostics variant (tools/ only; -DBLK_DIAG adds the two-kernel
    split blk_debug_split_f64, not part of the public ABI):
    paper_2108_11560_b200/variants/diag.so."""
    out = os.path.join(HERE, "variants", "diag.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in _deps()):
        return out
    return build(out=out, defines=["BLK_DIAG"])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
