"""Throughput of the fused NIG log-likelihood + gradient (one GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402

for n in (1 << 20, 1 << 24):
    y = torch.from_numpy(np.random.default_rng(0).normal(0, 3, n)).cuda()
    ws = torch.empty(blk.lib().bessel_nig_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    out = torch.empty(5, dtype=torch.float64, device="cuda")
    for _ in range(3):
        blk.nig_loglik(y, 2.0, 0.5, 1.5, 0.3, out=out, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        blk.nig_loglik(y, 2.0, 0.5, 1.5, 0.3, out=out, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"nig n={n} {ts[5]:.3f} ms  {n / ts[5] * 1e3:.3e} samples/s  out={out.cpu().numpy()}")
