"""Small invocations of every kernel for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): the FP64 kernel at 1/2/8/32 lanes per
element with ragged tails and empty lanes, the FP32 kernel, the Hessian and
plan kernels, both NIG kernels, the zero-copy and the staged host paths, and
the microbenchmarks.  Run as
    compute-sanitizer --tool memcheck python tests/tools/sanitize_run.py
(tools/gpu_sanitize.sh).  Prints SANITIZE RUN OK at the end."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    v, x = workloads.generate("c2", 0, 1000 + 37)
    v[:5] = [-3.0, 0.0, np.nan, 1.0, 2.0]
    x[:5] = [1.0, 2.0, 1.0, -1.0, 1e-30]
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    for lanes in (1, 2, 8, 32):
        for nb in (2, 16, 128):
            blk.log_bessel_k(vt, xt, nbins=nb, lanes_per_element=lanes)
            blk.log_bessel_k(vt, xt, nbins=nb, lanes_per_element=lanes, outputs=("dx",))
    blk.log_bessel_k(vt, xt, nbins=128, range_mode=blk.BLK_RANGE_F64)
    blk.log_bessel_k(vt[:1], xt[:1])
    v4, x4 = workloads.generate("c4", 0, 1000 + 37)
    v4t, x4t = torch.from_numpy(v4).to(dev), torch.from_numpy(x4).to(dev)
    for lanes in (1, 4, 32):
        for nb in (2, 128):
            blk.log_bessel_k(v4t, x4t, nbins=nb, lanes_per_element=lanes)
    for lanes in (1, 8):
        blk.log_bessel_k_hess(vt, xt, lanes_per_element=lanes)
    blk.bessel_logk_plan_f64(vt, xt, nbins=16)
    blk.bessel_logk_plan_f64(vt, xt, nbins=128)
    y = torch.from_numpy(np.random.default_rng(1).normal(0, 3, 1000 + 37)).to(dev)
    blk.nig_loglik(y, 2.0, 0.5, 1.5, 0.3)
    blk.nig_loglik(y[:0], 2.0, 0.5, 1.5, 0.3)
    # host entry points: zero-copy (pinned) and staged (pageable) transports
    hv, hx = torch.from_numpy(v).pin_memory(), torch.from_numpy(x).pin_memory()
    ho = [torch.empty(v.size, dtype=torch.float64).pin_memory() for _ in range(3)]
    blk.bessel_logk_f64_host(hv, hx, *ho, nbins=128)
    pv, px = torch.from_numpy(v.copy()), torch.from_numpy(x.copy())
    po = [torch.empty(v.size, dtype=torch.float64) for _ in range(3)]
    chunk = 256
    ws = torch.empty(blk.host_workspace_bytes(chunk), dtype=torch.uint8, device=dev)
    blk.bessel_logk_f64_host(pv, px, *po, nbins=128, workspace=ws, chunk=chunk)
    h4v, h4x = torch.from_numpy(v4).pin_memory(), torch.from_numpy(x4).pin_memory()
    h4o = [torch.empty(v4.size, dtype=torch.float32).pin_memory() for _ in range(3)]
    blk.bessel_logk_f32_host(h4v, h4x, *h4o, nbins=128)
    out = torch.empty(4 * 128, dtype=torch.float64, device=dev)
    out32 = torch.empty(4 * 128, dtype=torch.float32, device=dev)
    blk.microbench("fp64", 4, 128, 4, out)
    blk.microbench("fp32", 4, 128, 4, out32)
    blk.microbench("mufu", 4, 128, 4, out32)
    torch.cuda.synchronize()
    for a, b in zip(ho, po):
        assert torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0))
    print("SANITIZE RUN OK", flush=True)


if __name__ == "__main__":
    main()
