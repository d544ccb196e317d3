"""Time the public entry point of several library builds on one config and
check them against the oracle on a sample.
usage: python tests/tools/variant_time.py CFG N lib1.so lib2.so ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, 'tools'))
from _timing import device_time  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from parity import max_errors  # noqa: E402



def timeit(fn, reps=10):
    return device_time(fn, reps)


def main():
    cfg, n = sys.argv[1], int(sys.argv[2])
    c = workloads.CONFIGS[cfg]
    f32 = c.precision == "f32"
    v, x = workloads.generate(cfg, 0, n)
    dev = torch.device("cuda")
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    o = [torch.empty_like(vt) for _ in range(3)]
    vp = ctypes.c_void_p
    P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o)]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    idx = np.linspace(0, n - 1, 2048).astype(np.int64)
    ref = oracle.logk(v[idx].astype(np.float64), x[idx].astype(np.float64), 128, threads=8)
    ref = dict(zip(("logk", "dv", "dx"), ref))
    for path in sys.argv[3:]:
        L = ctypes.CDLL(os.path.abspath(path))
        f = L.bessel_logk_f32 if f32 else L.bessel_logk_f64
        f.restype = ctypes.c_int
        f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp]
        ms = timeit(lambda: f(P[0], P[1], n, P[2], P[3], P[4], 128, s))
        got = {k: t.cpu().numpy()[idx].astype(np.float64) for k, t in zip(("logk", "dv", "dx"), o)}
        err = max_errors(got, ref)
        print(f"{os.path.basename(path):18s} {cfg} n={n} {ms:.3f} ms {n / ms * 1e3:.3e} evals/s  "
              + " ".join(f"{k}={e:.1e}" for k, e in err.items()), flush=True)


if __name__ == "__main__":
    main()
