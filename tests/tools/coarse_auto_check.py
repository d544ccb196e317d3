"""Element-wise parity against the oracle and throughput of the FP64 entry
point at bin counts near the FP32/FP64 range-finder switch (AUTO mode), for a
library build given on the command line (default: the in-tree one).
usage: python tests/tools/coarse_auto_check.py [--lib X.so] [--nbins 40,48,56,63,64]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from parity import TOL, max_errors  # noqa: E402
from _timing import device_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2108_11560_b200", "libbessel_logk.so"))
    ap.add_argument("--nbins", default="40,48,56,63,64")
    ap.add_argument("--n", type=int, default=20000)
    a = ap.parse_args()
    L = ctypes.CDLL(a.lib)
    vp, sz, ci = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    L.bessel_logk_f64.argtypes = [vp, vp, sz, vp, vp, vp, ci, vp]
    dev = torch.device("cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for nb in [int(t) for t in a.nbins.split(",")]:
        worst = {}
        for cfg in ("c1", "c2", "c3", "c4", "c5"):
            v, x = workloads.generate(cfg, 0, min(a.n, workloads.CONFIGS[cfg].n))
            v = np.asarray(v, np.float64)
            x = np.asarray(x, np.float64)
            vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
            o = [torch.empty_like(vt) for _ in range(3)]
            P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o)]
            assert L.bessel_logk_f64(P[0], P[1], len(v), P[2], P[3], P[4], nb, s) == 0
            torch.cuda.synchronize()
            got = dict(zip(("logk", "dv", "dx"), (t.cpu().numpy() for t in o)))
            ref = dict(zip(("logk", "dv", "dx"), oracle.logk(v, x, nb, threads=16)))
            e = max_errors(got, ref)
            worst[cfg] = {k: e[k] / TOL["f64"][k] for k in e}
        v, x = workloads.generate("c3", 0, 1 << 22)
        vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
        o = [torch.empty_like(vt) for _ in range(3)]
        P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o)]
        ms = device_time(lambda: L.bessel_logk_f64(P[0], P[1], len(v), P[2], P[3], P[4], nb, s), 10)
        w = " ".join(f"{c}:" + "/".join(f"{worst[c][k]:.2g}" for k in ("logk", "dv", "dx")) for c in worst)
        print(f"nbins={nb:3d} c3 2^22 {ms:.3f} ms {len(v) / ms * 1e3:.3e} evals/s | max err / tol (logK/dv/dx) {w}",
              flush=True)


if __name__ == "__main__":
    main()
