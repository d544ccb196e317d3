"""CPU-side checks of the C ABI boundary: the library loads without a GPU,
exports every function include/bessel_logk.h declares, and rejects invalid
arguments with BLK_EINVAL before making any CUDA call."""
import ctypes
import os
import subprocess

import pytest

import paper_2108_11560_b200 as blk
from paper_2108_11560_b200 import build as _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    _build.build()
    return blk.lib()


def test_exports_every_header_function(L):
    names = blk.header_functions()
    assert len(names) == 16, names
    for nm in names:
        assert hasattr(L, nm), nm
    out = subprocess.run(["nm", "-D", "--defined-only", blk.library_path],
                         capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= exported
    # nothing but the C ABI is exported (hidden visibility for the rest)
    assert exported == set(names), sorted(exported - set(names))


def test_header_is_plain_c():
    """The header compiles as C99 with no CUDA or torch headers."""
    src = '#include "bessel_logk.h"\nint main(void){return (int)sizeof(blk_options);}\n'
    p = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c",
                        "-I", os.path.join(ROOT, "include"), "-"], input=src, text=True,
                       capture_output=True)
    assert p.returncode == 0, p.stderr


def test_kernel_is_sm100a_sass(L):
    """The fatbin carries sm_100a SASS (cuobjdump) for the fused kernels."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", blk.library_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _f64(L, v, x, n, a, b, c, nbins, opts=None):
    if opts is None:
        return L.bessel_logk_f64(v, x, n, a, b, c, nbins, None)
    return L.bessel_logk_f64_ex(v, x, n, a, b, c, nbins, ctypes.byref(opts), None)


FAKE = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first


def test_invalid_arguments(L):
    assert _f64(L, FAKE, FAKE, 10, FAKE, None, None, 1) == blk.BLK_EINVAL
    assert _f64(L, FAKE, FAKE, 10, FAKE, None, None, 65537) == blk.BLK_EINVAL
    assert _f64(L, FAKE, FAKE, 10, None, None, None, 128) == blk.BLK_EINVAL
    assert _f64(L, None, FAKE, 10, FAKE, None, None, 128) == blk.BLK_EINVAL
    assert _f64(L, FAKE, None, 10, FAKE, None, None, 128) == blk.BLK_EINVAL
    assert b"nbins" in L.bessel_logk_last_error() or L.bessel_logk_last_error()
    bad = [blk._Options(3, 0, 0), blk._Options(64, 0, 0), blk._Options(0, 2, 0),
           blk._Options(0, 0, 48), blk._Options(0, 0, 256), blk._Options(-1, 0, 0),
           blk._Options(0, 0, 0, 3), blk._Options(0, 0, 0, -1),
           blk._Options(2, 0, 0, blk.BLK_KERNEL_VEC128)]   # 128-bit I/O: one lane per element
    for o in bad:
        assert _f64(L, FAKE, FAKE, 10, FAKE, None, None, 128, o) == blk.BLK_EINVAL
    assert L.bessel_logk_f32(FAKE, FAKE, 10, None, None, None, 128, None) == blk.BLK_EINVAL
    assert L.bessel_logk_f64_host(FAKE, FAKE, 10, FAKE, None, None, 1, None, 0, 0,
                                  None) == blk.BLK_EINVAL


def test_empty_batch_is_noop(L):
    # n == 0 returns OK without touching CUDA (works on a CPU-only host)
    assert _f64(L, None, None, 0, FAKE, None, None, 128) == blk.BLK_OK
    assert L.bessel_logk_f32(None, None, 0, None, None, FAKE, 2, None) == blk.BLK_OK


def test_workspace_size(L):
    assert L.bessel_logk_host_workspace_bytes(1 << 20, 8) >= 3 * 5 * (1 << 20) * 8
    assert blk.host_workspace_bytes(0) == L.bessel_logk_host_workspace_bytes(1 << 20, 8)
    assert L.bessel_logk_version().startswith(b"bessel_logk")


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2108_11560_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "oracle.c" not in txt, f


def test_oracle_used_only_where_allowed():
    """oracle/ is test infrastructure: only tests/, __graft_entry__.py (smoke)
    and bench.py (cpu_baseline / --impl reference) may import it."""
    allowed = {os.path.join(ROOT, "__graft_entry__.py"), os.path.join(ROOT, "bench.py")}
    skip = {os.path.join(ROOT, d) for d in ("tests", "oracle", ".git", "gpurun_out", "baseline")}
    for dp, dirs, files in os.walk(ROOT):
        dirs[:] = [d for d in dirs if os.path.join(dp, d) not in skip]
        for f in files:
            path = os.path.join(dp, f)
            if f.endswith(".py") and path not in allowed:
                txt = open(path).read()
                assert "import oracle" not in txt and "from oracle" not in txt, path
