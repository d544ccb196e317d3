"""Run the wide-domain FP64 fuzz inputs (tests/test_gpu_parity.py::test_wide_domain_fuzz)
through the FP64 entry point and save inputs + outputs for offline analysis.
    python tools/dump_fuzz.py OUT.npz"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402

out = {}
for seed in (1, 2, 3):
    rng = np.random.default_rng(seed)
    n = 20000
    v = 10.0 ** rng.uniform(-6, np.log10(2e4), n)
    v[rng.random(n) < 0.02] = 0.0
    v *= np.where(rng.random(n) < 0.1, -1.0, 1.0)
    x = 10.0 ** rng.uniform(-12, 7, n)
    vt, xt = torch.from_numpy(v).cuda(), torch.from_numpy(x).cuda()
    r = blk.log_bessel_k(vt, xt)
    p = blk.bessel_logk_plan_f64(vt, xt, nbins=128)
    torch.cuda.synchronize()
    out[f"v{seed}"], out[f"x{seed}"] = v, x
    out[f"o{seed}"] = np.stack([t.cpu().numpy() for t in r], 1)
    out[f"p{seed}"] = np.stack([t.cpu().numpy() for t in p], 1)
np.savez_compressed(sys.argv[1], **out)
print("ok")
