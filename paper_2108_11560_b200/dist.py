"""Multi-GPU driver: contiguous sharding of the element batch, one process per
GPU (torchrun), no collective on the data path (elements are independent,
P:58).  torch.distributed (NCCL over NVLink/NVSwitch on B200, gloo in
the CPU tests) is used only after the timed region:

  * ``max_over_ranks``   all_reduce(MAX) of a per-rank elapsed time;
  * ``gather_samples``   collects the outputs at a set of GLOBAL element
    indices on every rank (each index is owned by exactly one shard, so a SUM
    all-reduce of the zero-padded per-rank pieces assembles them exactly).

``run_sharded`` evaluates one rank's shard with a caller-supplied compute
function (the CUDA entry point in production).
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int):
    """Contiguous, balanced [lo, hi) of rank ``rank`` among ``world``."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard arguments")
    return n * rank // world, n * (rank + 1) // world


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(t):
    """Sum a small tensor (e.g. the 5 NIG log-likelihood sums) over all ranks in
    place -- the one collective of the NIG path (NCCL over NVLink on B200)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def nig_loglik_sharded(y_local, alpha, beta, delta, mu, nbins=128):
    """Per-rank NIG sums on this rank's shard (CUDA kernels), then all_reduce."""
    import paper_2108_11560_b200 as blk
    out = blk.nig_loglik(y_local, alpha, beta, delta, mu, nbins=nbins)
    return allreduce_sum(out)


def gather_samples(local: dict, lo: int, hi: int, global_idx, device=None) -> dict:
    """local: kind -> 1-D tensor holding this rank's shard [lo, hi).
    Returns kind -> tensor of len(global_idx) (identical on every rank)."""
    import torch
    import torch.distributed as dist
    idx = np.asarray(global_idx, dtype=np.int64)
    mine = (idx >= lo) & (idx < hi)
    pos = torch.from_numpy(np.nonzero(mine)[0]).to(device)
    loc = torch.from_numpy(idx[mine] - lo).to(device)
    out = {}
    for k, t in local.items():
        buf = torch.zeros(idx.size, dtype=torch.float64, device=device)
        if loc.numel():
            buf[pos] = t[loc.to(t.device)].to(device=device, dtype=torch.float64)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        out[k] = buf
    return out


def run_sharded(compute, v_global_fn, n: int, world: int, rank: int):
    """Evaluate shard ``rank``: v_global_fn(lo, count) -> (v, x) host arrays;
    compute(v, x) -> dict kind -> tensor.  Returns (lo, hi, outputs)."""
    lo, hi = shard_range(n, world, rank)
    v, x = v_global_fn(lo, hi - lo)
    return lo, hi, compute(v, x)
