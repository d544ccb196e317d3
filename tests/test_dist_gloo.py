"""Host-side logic of the multi-GPU driver, world_size 2 over gloo on CPU:
contiguous shards cover the batch exactly once, sampled outputs gathered
from the shards equal the single-process result, and the elapsed-time
reduction takes the max over ranks.  The per-element compute here is the
CPU oracle standing in for the CUDA kernel (test only; the product driver
passes the CUDA entry point)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_11560_b200 import dist as bdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import oracle
    import workloads
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def gen(lo, cnt):
            return workloads.generate("c2", lo, cnt, n=n)

        def compute(v, x):
            lk, dv, dx = oracle.logk(v, x, 64)
            return {"logk": torch.from_numpy(lk), "dv": torch.from_numpy(dv),
                    "dx": torch.from_numpy(dx)}

        lo, hi, out = bdist.run_sharded(compute, gen, n, world, rank)
        idx = np.array([0, 1, n // 2 - 1, n // 2, n // 2 + 1, n - 1, 17, 333])
        got = bdist.gather_samples(out, lo, hi, idx)
        tmax = bdist.max_over_ranks(1.0 + rank)
        if rank == 0:
            q.put(({k: t.numpy() for k, t in got.items()}, tmax, (lo, hi)))
        else:
            q.put((None, tmax, (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_shard_range_cover():
    for n in (0, 1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            parts = [bdist.shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1
    with pytest.raises(ValueError):
        bdist.shard_range(10, 2, 2)


def test_gloo_two_ranks_gather_and_max():
    import oracle
    import workloads
    n = 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = next(r[0] for r in res if r[0] is not None)
    assert all(r[1] == 2.0 for r in res)
    bounds = sorted(r[2] for r in res)
    assert bounds == [(0, 500), (500, 1000)]
    idx = np.array([0, 1, n // 2 - 1, n // 2, n // 2 + 1, n - 1, 17, 333])
    v, x = workloads.generate("c2", 0, n)
    ref = oracle.logk(v[idx], x[idx], 64)
    for k, r in zip(("logk", "dv", "dx"), ref):
        assert np.array_equal(got[k], r), k
