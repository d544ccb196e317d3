"""evals/s of the fused FP64 kernel vs block size (block retirement granularity).
usage: python tools/blocksize.py CFG N"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402
from _timing import device_time  # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
v, x = workloads.generate(cfg, 0, n)
vt, xt = torch.from_numpy(v).cuda(), torch.from_numpy(x).cuda()
o = [torch.empty_like(vt) for _ in range(3)]
ref = None
for bt in (128, 96, 64, 32):
    ms = device_time(lambda: blk.bessel_logk_f64(vt, xt, *o, block_threads=bt, lanes_per_element=1), 20)
    same = ref is None or all(torch.equal(a, b) for a, b in zip(o, ref))
    if ref is None:
        ref = [t.clone() for t in o]
    print(f"{cfg} n={n} block_threads={bt:3d} {ms:.4f} ms {n / ms * 1e3:.3e} evals/s bitwise-same={same}",
          flush=True)
