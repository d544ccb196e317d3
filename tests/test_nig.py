"""NIG log-likelihood: oracle pins on CPU, GPU parity,
and the cross-rank sum over gloo."""
import math
import os
import socket

import numpy as np
import pytest
import scipy.stats
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import nig as onig

PARAMS = [(2.0, 0.5, 1.5, 0.3), (0.7, -0.3, 0.2, -1.0), (15.0, 10.0, 3.0, 2.0)]


def _sample(n, seed):
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, 3.0, n)


@pytest.mark.parametrize("a,b,d,m", PARAMS)
def test_oracle_logpdf_vs_scipy(a, b, d, m):
    """log p of the oracle (paper's method for log K_1) vs scipy.stats.norminvgauss."""
    y = _sample(300, 1)
    t = onig.nig_terms(y, a, b, d, m)
    ref = scipy.stats.norminvgauss(a * d, b * d, loc=m, scale=d).logpdf(y)
    assert np.max(np.abs(t[0] - ref) / np.maximum(1, np.abs(ref))) < 1e-13


@pytest.mark.parametrize("a,b,d,m", PARAMS)
def test_oracle_gradient_vs_finite_differences(a, b, d, m):
    """The chain-rule gradient vs central differences of the summed log p."""
    y = _sample(200, 2)
    g, _ = onig.nig_loglik(y, a, b, d, m)
    th = np.array([a, b, d, m])
    for k in range(4):
        hk = 1e-5 * max(1.0, abs(th[k]))
        tp, tm = th.copy(), th.copy()
        tp[k] += hk
        tm[k] -= hk
        fd = (onig.nig_loglik(y, *tp)[0][0] - onig.nig_loglik(y, *tm)[0][0]) / (2 * hk)
        assert abs(fd - g[k + 1]) <= 1e-6 * max(1.0, abs(g[k + 1])), (k, fd, g[k + 1])


def test_oracle_density_normalised():
    """The NIG density integrates to 1 and has mean m + d b/g (closed form)."""
    a, b, d, m = 2.0, 0.5, 1.5, 0.3
    y = np.linspace(-60, 60, 120001)
    p = np.exp(onig.nig_terms(y, a, b, d, m)[0])
    dy = y[1] - y[0]
    assert abs(np.sum(p) * dy - 1.0) < 1e-10
    mean = np.sum(p * y) * dy
    assert abs(mean - (m + d * b / math.sqrt(a * a - b * b))) < 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("a,b,d,m", PARAMS)
@pytest.mark.parametrize("n", [1, 127, 128, 129, 50_000])
def test_gpu_nig_vs_oracle(a, b, d, m, n):
    import paper_2108_11560_b200 as blk
    y = _sample(n, 3)
    out = blk.nig_loglik(torch.from_numpy(y).cuda(), a, b, d, m).cpu().numpy()
    ref, mag = onig.nig_loglik(y, a, b, d, m)
    # per-term errors ~1e-13 relative; the sums can cancel (gradient ~0 near
    # the optimum), so the tolerance is relative to the sum of |terms|
    assert np.all(np.abs(out - ref) <= 1e-12 * np.maximum(1.0, mag)), (out, ref)


@pytest.mark.gpu
def test_gpu_nig_deterministic_and_empty():
    import paper_2108_11560_b200 as blk
    y = torch.from_numpy(_sample(100_000, 4)).cuda()
    a1 = blk.nig_loglik(y, 2.0, 0.5, 1.5, 0.3)
    a2 = blk.nig_loglik(y, 2.0, 0.5, 1.5, 0.3)
    assert torch.equal(a1, a2)
    z = blk.nig_loglik(torch.empty(0, dtype=torch.float64, device="cuda"), 2.0, 0.5, 1.5, 0.3)
    assert torch.equal(z.cpu(), torch.zeros(5, dtype=torch.float64))
    with pytest.raises(blk.BesselLogKError):
        blk.nig_loglik(y, 1.0, 2.0, 1.0, 0.0)    # |beta| >= alpha


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_sums(y, a, b, d, m, nbins):
    """CPU stand-in for the kernels' per-rank sums (test only): the oracle."""
    return torch.from_numpy(onig.nig_terms(y, a, b, d, m, nbins).sum(axis=1))


def _worker(rank, world, port, q):
    from paper_2108_11560_b200 import dist as bdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        y = _sample(1000, 5)
        lo, hi = bdist.shard_range(y.size, world, rank)
        tot = bdist.nig_loglik_sharded(y[lo:hi], 2.0, 0.5, 1.5, 0.3, compute=_cpu_sums)
        q.put((rank, tot.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_nig_loglik_sharded():
    """dist.nig_loglik_sharded at world size 2 over gloo: each rank's shard
    sums, one all-reduce, the same 5-vector on both ranks equal to the
    single-process sums."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = _sample(1000, 5)
    ref = onig.nig_terms(y, 2.0, 0.5, 1.5, 0.3).sum(axis=1)
    for r in (0, 1):
        assert np.allclose(res[r], ref, rtol=1e-13, atol=1e-10)
    assert np.array_equal(res[0], res[1])


@pytest.mark.gpu
def test_nig_sharded_torchrun():
    """dist.nig_loglik_sharded end to end under torchrun over every GPU of the
    box (NCCL; world 1 on the one-GPU pool, 8 on a full node): per-rank CUDA
    kernels on contiguous shards, the all-reduce on the kernels' stream, the
    result against the oracle on the whole sample (tests/mgpu_nig_driver.py).
    NCCL_DEBUG=INFO shows the communicator's ranks in the log."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    g = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr",
           "127.0.0.1", f"--nproc-per-node={g}", os.path.join(here, "mgpu_nig_driver.py")]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", NCCL_DEBUG="INFO")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"NIG OK world={g}" in r.stdout
