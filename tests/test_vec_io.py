"""BLK_KERNEL_VEC128: the kernels' 128-bit warp-cooperative I/O variant
(BASELINE.json north_star (3); paper_2108_11560_b200/csrc/logk_io.cuh).

The arithmetic is the SIMPLE kernel's, so the outputs must equal its outputs
bit for bit (with one lane per element) for every output subset, for batch
sizes that end inside a warp, and when a stream is not 16-byte aligned (the
host then launches the scalar-I/O kernel).  Parity against the oracle on one
config closes the loop; guard regions check that the 16-byte stores write
exactly the n outputs."""
import numpy as np
import pytest
import torch

import oracle
import paper_2108_11560_b200 as blk
import workloads
from parity import assert_parity

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
KINDS = ("logk", "dv", "dx")
SUBSETS = [("logk", "dv", "dx"), ("logk",), ("dv",), ("dx",), ("logk", "dv"), ("logk", "dx"),
           ("dv", "dx")]


def _inputs(cfg, n, dt):
    v, x = workloads.generate(cfg, 11, n)
    return (torch.from_numpy(np.asarray(v, np.float64)).to(DEV, dt),
            torch.from_numpy(np.asarray(x, np.float64)).to(DEV, dt))


def _same(a, b):
    return torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0))


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("n", [1, 31, 32, 33, 127, 4096 + 17, 70001])
def test_vec128_bitwise_equals_simple(prec, n):
    dt = torch.float64 if prec == 64 else torch.float32
    v, x = _inputs("c2" if prec == 64 else "c4", n, dt)
    if n >= 8:   # special values and invalid inputs inside a vectorised warp
        v[:4] = torch.tensor([-3.5, 0.0, float("nan"), 2.0], dtype=dt)
        x[:4] = torch.tensor([1.0, 0.5, 1.0, -1.0], dtype=dt)
    for outs in SUBSETS if n in (33, 4096 + 17) else SUBSETS[:1]:
        ref = blk.log_bessel_k(v, x, outputs=outs, lanes_per_element=1)
        got = blk.log_bessel_k(v, x, outputs=outs, kernel=blk.BLK_KERNEL_VEC128)
        torch.cuda.synchronize()
        for a, b in zip(got, ref):
            assert _same(a, b), (prec, n, outs)


@pytest.mark.parametrize("prec", [64, 32])
def test_vec128_misaligned_falls_back(prec):
    """Views starting one element in (8-/4-byte aligned, not 16): the scalar
    kernel runs; same bits."""
    dt = torch.float64 if prec == 64 else torch.float32
    v, x = _inputs("c2" if prec == 64 else "c4", 5001, dt)
    vv, xv = v[1:], x[1:]
    outs = [torch.empty(5001, dtype=dt, device=DEV)[1:] for _ in range(3)]
    f = blk.bessel_logk_f64 if prec == 64 else blk.bessel_logk_f32
    f(vv, xv, *outs, kernel=blk.BLK_KERNEL_VEC128)
    ref = blk.log_bessel_k(vv, xv, lanes_per_element=1)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert _same(a, b)


def test_vec128_parity_vs_oracle():
    c = workloads.CONFIGS["c3"]
    v, x = workloads.generate("c3", 5, 3 * 4096 + 45)
    vt = torch.from_numpy(np.asarray(v)).to(DEV)
    xt = torch.from_numpy(np.asarray(x)).to(DEV)
    got = blk.log_bessel_k(vt, xt, kernel=blk.BLK_KERNEL_VEC128)
    got = {k: t.cpu().numpy() for k, t in zip(KINDS, got)}
    ref = dict(zip(KINDS, oracle.logk(np.asarray(v, np.float64), np.asarray(x, np.float64), 128,
                                      threads=8)))
    assert_parity(got, ref, c.precision, "c3 VEC128")


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("n", [32, 45, 1037])
def test_vec128_guards(prec, n):
    """16-byte-aligned windows inside sentinel-filled buffers: the vector
    stores write exactly the n outputs, nothing before or after."""
    dt = torch.float64 if prec == 64 else torch.float32
    G = 4096   # guard elements: keeps the windows 16-byte aligned
    sent = -2.5e300 if prec == 64 else -3.1e38
    v, x = _inputs("c2" if prec == 64 else "c4", n, dt)
    bufs = [torch.full((n + 2 * G,), sent, dtype=dt, device=DEV) for _ in range(3)]
    outs = [b[G:G + n] for b in bufs]
    f = blk.bessel_logk_f64 if prec == 64 else blk.bessel_logk_f32
    f(v, x, *outs, kernel=blk.BLK_KERNEL_VEC128)
    ref = blk.log_bessel_k(v, x, lanes_per_element=1)
    torch.cuda.synchronize()
    for b, o, r in zip(bufs, outs, ref):
        assert bool((b[:G] == sent).all()) and bool((b[G + n:] == sent).all())
        assert _same(o, r)
