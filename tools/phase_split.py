"""Time the two phases of the FP64 hot path separately (blk_debug_split_f64)
and the fused kernel variants, on one config.  usage: python tools/phase_split.py CFG [NBINS]"""
import ctypes
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


def main():
    cfg = sys.argv[1]
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    c = workloads.CONFIGS[cfg]
    v, x = workloads.generate(cfg, 0, min(c.n, 1 << 22))
    dev = torch.device("cuda")
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    n = vt.numel()
    o = [torch.empty_like(vt) for _ in range(3)]
    scratch = torch.empty(n * 32, dtype=torch.uint8, device=dev)
    from paper_2108_11560_b200 import build as _b
    L = ctypes.CDLL(_b.build_diag())   # the split exists only in the diagnostics build
    f = L.blk_debug_split_f64
    f.restype = ctypes.c_int
    vp = ctypes.c_void_p
    f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int, vp]
    P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o, scratch)]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def split(ph):
        return lambda: f(P[0], P[1], n, P[2], P[3], P[4], nb, P[5], ph, s)

    split(1)()
    res = {}
    for name, fn in [("plan", split(1)), ("quad", split(2)), ("plan+quad", split(3)),
                     ("fused simple", lambda: blk.bessel_logk_f64(vt, xt, *o, nbins=nb, kernel=1))]:
        ms = timeit(fn)
        res[name] = ms
        print(f"{cfg} n={n} nbins={nb} {name:14s} {ms:.3f} ms  {n / ms * 1e3:.3e} evals/s", flush=True)


if __name__ == "__main__":
    main()
