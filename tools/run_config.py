"""Launch one config a few times (for ncu captures).  usage: python tools/run_config.py CFG N NBINS"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402

cfg, n, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = workloads.CONFIGS[cfg]
v, x = workloads.generate(cfg, 0, n)
vt, xt = torch.from_numpy(v).cuda(), torch.from_numpy(x).cuda()
for _ in range(3):
    blk.log_bessel_k(vt, xt, nbins=nb, outputs=c.outputs)
torch.cuda.synchronize()
print("ok")
