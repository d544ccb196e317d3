"""Time tuning variants (separately built .so files): quadrature-only (split
phase 2), plan-only (phase 1), fused simple kernel.
usage: python tools/variant_sweep.py CFG NBINS lib1.so lib2.so ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _timing import device_time  # noqa: E402

import workloads  # noqa: E402


class Opt(ctypes.Structure):
    _fields_ = [("lanes_per_element", ctypes.c_int), ("range_mode", ctypes.c_int),
                ("block_threads", ctypes.c_int), ("kernel", ctypes.c_int)]



def timeit(fn, reps=10):
    return device_time(fn, reps)


def main():
    cfg, nb = sys.argv[1], int(sys.argv[2])
    c = workloads.CONFIGS[cfg]
    v, x = workloads.generate(cfg, 0, min(c.n, 1 << 22))
    dev = torch.device("cuda")
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    n = vt.numel()
    o = [torch.empty_like(vt) for _ in range(3)]
    scratch = torch.empty(n * 32, dtype=torch.uint8, device=dev)
    vp = ctypes.c_void_p
    P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o, scratch)]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ref = None
    for path in sys.argv[3:]:
        L = ctypes.CDLL(os.path.abspath(path))
        sp = L.blk_debug_split_f64
        sp.restype = ctypes.c_int
        sp.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int, vp]
        fx = L.bessel_logk_f64_ex
        fx.restype = ctypes.c_int
        fx.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, ctypes.POINTER(Opt), vp]
        o1 = Opt(1, 0, 0, 1)
        sp(P[0], P[1], n, P[2], P[3], P[4], nb, P[5], 1, s)
        r = {}
        r["plan"] = timeit(lambda: sp(P[0], P[1], n, P[2], P[3], P[4], nb, P[5], 1, s))
        r["quad"] = timeit(lambda: sp(P[0], P[1], n, P[2], P[3], P[4], nb, P[5], 2, s))
        r["simple"] = timeit(lambda: fx(P[0], P[1], n, P[2], P[3], P[4], nb, ctypes.byref(o1), s))
        res = [t.clone() for t in o]
        if ref is None:
            ref = res
        err = max(float(((a - b).abs() / b.abs().clamp_min(1)).max()) for a, b in zip(res, ref))
        print(f"{os.path.basename(path):16s} {cfg} n={n} " +
              " ".join(f"{k}={ms:.3f}ms({n / ms * 1e3 / 1e9:.2f}G/s)" for k, ms in r.items()) +
              f"  maxdiff_vs_first:{err:.1e}", flush=True)


if __name__ == "__main__":
    main()
