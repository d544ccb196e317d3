"""A/B timing of library builds (tools/build_variants.py outputs and the
in-tree library) on the full-size configs, interleaved round by round so
clock drift hits every build alike; also checks the builds agree bit for bit.
usage: python tools/ab_libs.py [--rounds R] [--nbins N] CFG[,CFG..] lib1.so lib2.so ...
FP64 entry point for c1-c3/c5, FP32 for c4; c5 sized 2^26 here."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from _timing import device_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--nbins", type=int, default=128)
    ap.add_argument("--e2e", action="store_true",
                    help="also time the host entry points on pinned (zero-copy) buffers")
    ap.add_argument("cfgs")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    vp, sz, ci = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    libs = []
    for p in a.libs:
        L = ctypes.CDLL(os.path.abspath(p))
        for name in ("bessel_logk_f64", "bessel_logk_f32"):
            getattr(L, name).argtypes = [vp, vp, sz, vp, vp, vp, ci, vp]
            getattr(L, name).restype = ci
            getattr(L, name + "_host").argtypes = [vp, vp, sz, vp, vp, vp, ci, vp, sz, sz, vp]
            getattr(L, name + "_host").restype = ci
        libs.append((os.path.basename(p), L))
    dev = torch.device("cuda")
    for cfg in a.cfgs.split(","):
        c = workloads.CONFIGS[cfg]
        n = min(c.n, 1 << 26)
        v, x = workloads.generate(cfg, 0, n)
        dt = torch.float32 if cfg == "c4" else torch.float64
        vt = torch.from_numpy(np.asarray(v)).to(dev, dt)
        xt = torch.from_numpy(np.asarray(x)).to(dev, dt)
        outs = {nm: [torch.empty_like(vt) for _ in range(3)] for nm, _ in libs}
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        fns = {}
        for nm, L in libs:
            f = L.bessel_logk_f32 if dt == torch.float32 else L.bessel_logk_f64
            P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *outs[nm])]
            fns[nm] = (lambda f=f, P=P: f(P[0], P[1], n, P[2], P[3], P[4], a.nbins, s))
            assert fns[nm]() == 0
            if a.e2e:
                hv, hx = vt.cpu().pin_memory(), xt.cpu().pin_memory()
                ho = [torch.empty(n, dtype=dt).pin_memory() for _ in range(3)]
                fh = L.bessel_logk_f32_host if dt == torch.float32 else L.bessel_logk_f64_host
                H = [ctypes.c_void_p(t.data_ptr()) for t in (hv, hx, *ho)]
                fns[nm + ":e2e"] = (lambda fh=fh, H=H, keep=(hv, hx, ho):
                                    fh(H[0], H[1], n, H[2], H[3], H[4], a.nbins, None, 0, 0, s))
                assert fns[nm + ":e2e"]() == 0
        torch.cuda.synchronize()
        ref = outs[libs[0][0]]
        for nm, _ in libs[1:]:
            same = all(torch.equal(p.nan_to_num(7.0), q.nan_to_num(7.0)) for p, q in zip(outs[nm], ref))
            print(f"{cfg} {nm}: bitwise equal to {libs[0][0]}: {same}")
        times = {nm: [] for nm in fns}
        for _ in range(a.rounds):
            for nm in fns:
                times[nm].append(device_time(fns[nm], reps=5))
        for nm in fns:
            ms = float(np.median(times[nm]))
            print(f"{cfg} n={n} nbins={a.nbins} {nm:24s} {ms:.4f} ms  {n / ms * 1e3:.4e} evals/s  "
                  f"rounds {' '.join(f'{t:.4f}' for t in times[nm])}", flush=True)


if __name__ == "__main__":
    main()
