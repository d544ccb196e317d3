"""NIG log-likelihood sharded over all GPUs, launched by
tests/test_nig.py::test_nig_sharded_torchrun as
    python -m torch.distributed.run --standalone --nproc-per-node=G tests/mgpu_nig_driver.py
Rank r holds the contiguous shard [r N/G, (r+1) N/G) of one seeded sample;
dist.nig_loglik_sharded runs the CUDA kernels on it and all-reduces the five
sums on the same stream; rank 0 compares them with the oracle (oracle/nig.py)
on the whole sample, and every rank checks it holds the same 5-vector."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import nig as onig  # noqa: E402
from paper_2108_11560_b200 import dist as bdist  # noqa: E402

N = 200_003
PARAMS = (2.0, 0.5, 1.5, 0.3)


def main():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    y = np.random.default_rng(9).normal(0.0, 3.0, N)
    lo, hi = bdist.shard_range(N, world, rank)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        yl = torch.from_numpy(y[lo:hi]).to(dev, non_blocking=False)
    s.synchronize()
    out = bdist.nig_loglik_sharded(yl, *PARAMS, nbins=128, stream=s)
    s.synchronize()
    got = out.cpu().numpy()
    allv = [torch.empty(5, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(allv, out)
    for t in allv:
        assert np.array_equal(t.cpu().numpy(), got)
    if rank == 0:
        ref, mag = onig.nig_loglik(y, *PARAMS)
        assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, mag)), (got, ref)
        print(f"NIG OK world={world} n={N} sum_logp={got[0]:.6f}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
