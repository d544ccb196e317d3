"""Multi-GPU driver: contiguous sharding of the element batch, one process per
GPU (torchrun), no collective on the data path of log K (elements are
independent).  torch.distributed (NCCL over NVLink/NVSwitch on
B200, gloo in the CPU tests) is used only:

  * ``max_over_ranks``     all_reduce(MAX) of a per-rank elapsed time (bench);
  * ``gather_samples``     all_gather of each rank's own outputs at a set of
    GLOBAL element indices (for checking against the oracle);
  * ``nig_loglik_sharded`` the one real exchange of any path: the five NIG
    log-likelihood sums (40 bytes) all-reduced across ranks, enqueued on the
    stream the kernels ran on, with no host synchronisation.

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


def _multi():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if _multi():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(t, stream=None):
    """Sum a small tensor over all ranks in place.  For a CUDA tensor the
    collective is enqueued on ``stream`` (default: the current stream) after
    the work already there -- the kernels that produced ``t`` -- and the call
    returns without synchronising the host (NCCL collectives are
    asynchronous to the host; the next op on ``stream`` sees the sum)."""
    import torch
    import torch.distributed as dist
    if not _multi():
        return t
    if t.is_cuda:
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(t.device)):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def nig_loglik_sharded(y_local, alpha, beta, delta, mu, nbins=128, stream=None, compute=None):
    """NIG log-likelihood sums (sum log p, d/d(alpha, beta, delta, mu)) of the
    sample whose contiguous shard ``y_local`` this rank holds: per-rank sums by
    the CUDA kernels (``compute`` overrides them -- tests only), then one
    all-reduce of the five numbers on the same stream (no host sync).
    Returns the summed 5-vector (device tensor for the CUDA path)."""
    if compute is None:
        import paper_2108_11560_b200 as blk
        out = blk.nig_loglik(y_local, alpha, beta, delta, mu, nbins=nbins, stream=stream)
    else:
        out = compute(y_local, alpha, beta, delta, mu, nbins)
    return allreduce_sum(out, stream=stream)


def gather_samples(local: dict, lo: int, hi: int, global_idx, device=None) -> dict:
    """local: kind -> 1-D tensor holding this rank's shard [lo, hi).
    Returns kind -> float64 tensor of len(global_idx) on ``device``, the same
    on every rank: each rank contributes the samples its shard owns
    (all_gather of (count-padded) positions and values), no rank sends
    anything it does not own."""
    import torch
    import torch.distributed as dist
    idx = np.asarray(global_idx, dtype=np.int64)
    mine = np.nonzero((idx >= lo) & (idx < hi))[0]
    pos = torch.from_numpy(mine).to(device)
    loc = torch.from_numpy(idx[mine] - lo)
    kinds = sorted(local)
    vals = torch.stack([local[k][loc.to(local[k].device)].to(device=device, dtype=torch.float64)
                        for k in kinds]) if kinds else torch.empty(0, device=device)
    if not _multi():
        out = {k: torch.zeros(idx.size, dtype=torch.float64, device=device) for k in kinds}
        for r, k in enumerate(kinds):
            out[k][pos] = vals[r]
        return out
    world = dist.get_world_size()
    cnt = torch.tensor([mine.size], dtype=torch.int64, device=device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    cmax = int(max(int(c.item()) for c in cnts))
    ppos = torch.full((cmax,), -1, dtype=torch.int64, device=device)
    ppos[:mine.size] = pos
    pval = torch.zeros((len(kinds), cmax), dtype=torch.float64, device=device)
    pval[:, :mine.size] = vals
    all_pos = [torch.empty_like(ppos) for _ in range(world)]
    all_val = [torch.empty_like(pval) for _ in range(world)]
    dist.all_gather(all_pos, ppos)
    dist.all_gather(all_val, pval)
    out = {k: torch.zeros(idx.size, dtype=torch.float64, device=device) for k in kinds}
    for p, v, c in zip(all_pos, all_val, cnts):
        c = int(c.item())
        for r, k in enumerate(kinds):
            out[k][p[:c]] = v[r, :c]
    return out


def run_sharded(compute, v_global_fn, n: int, world: int, rank: int):
    """Evaluate shard ``rank``: v_global_fn(lo, count) -> (v, x) host arrays;
    compute(v, x) -> dict kind -> tensor.  Returns (lo, hi, outputs)."""
    lo, hi = shard_range(n, world, rank)
    v, x = v_global_fn(lo, hi - lo)
    return lo, hi, compute(v, x)
