"""Multi-GPU driver check (north_star (4)), launched by
tests/test_multigpu.py as
    python -m torch.distributed.run --standalone --nproc-per-node=G tests/mgpu_driver.py CFG N
One process per GPU; rank r evaluates the contiguous shard [r N/G, (r+1) N/G)
of config CFG with the CUDA entry point -- no collective on the data path --
then NCCL gathers the inputs and outputs at 4096 global sample indices to
every rank, and rank 0 checks them element by element against the CPU oracle
and checks that the max-over-ranks timing reduction is consistent."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402
from paper_2108_11560_b200 import dist as bdist  # noqa: E402
from parity import assert_parity  # noqa: E402


def main():
    cfg, n = sys.argv[1], int(sys.argv[2])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = workloads.CONFIGS[cfg]
    lo, hi = bdist.shard_range(n, world, rank)
    v, x = workloads.generate(cfg, lo, hi - lo, n=n)
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = blk.log_bessel_k(vt, xt, outputs=c.outputs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ms_max = bdist.max_over_ranks(ms, device=dev)
    assert ms_max >= ms
    idx = np.unique(np.concatenate([np.linspace(0, n - 1, 4000).astype(np.int64),
                                    np.arange(world) * (n // world)]))   # every shard start
    local_out = dict(zip(c.outputs, res))
    local_out["v"], local_out["x"] = vt, xt
    g = bdist.gather_samples(local_out, lo, hi, idx, device=dev)
    if rank == 0:
        vs, xs = g["v"].cpu().numpy(), g["x"].cpu().numpy()
        # the gathered inputs are the global stream's elements (shards tile the batch)
        vr, xr = workloads.generate(cfg, 0, n, n=n) if n <= (1 << 22) else (None, None)
        if vr is not None:
            assert np.array_equal(vs, vr[idx].astype(np.float64))
            assert np.array_equal(xs, xr[idx].astype(np.float64))
        ref = oracle.logk(vs, xs, 128, threads=8)
        ref = dict(zip(("logk", "dv", "dx"), ref))
        got = {k: g[k].cpu().numpy() for k in c.outputs}
        assert_parity(got, {k: ref[k] for k in c.outputs}, c.precision, f"{cfg} world={world}")
        print(f"MGPU OK cfg={cfg} n={n} world={world} samples={idx.size} max_ms={ms_max:.3f}",
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
