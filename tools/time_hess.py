"""Throughput of the second-derivative (Hessian) entry point vs the first-order one (one GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _timing import device_time  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402



def timeit(fn, reps=10):
    return device_time(fn, reps)


for cfg in ("c2", "c3"):
    n = 1 << 20
    v, x = workloads.generate(cfg, 0, n)
    vt, xt = torch.from_numpy(v).cuda(), torch.from_numpy(x).cuda()
    t1 = timeit(lambda: blk.log_bessel_k(vt, xt))
    t2 = timeit(lambda: blk.log_bessel_k_hess(vt, xt))
    print(f"{cfg} n={n} first-order {t1:.3f} ms {n / t1 * 1e3:.3e}/s | with Hessian {t2:.3f} ms "
          f"{n / t2 * 1e3:.3e}/s", flush=True)
