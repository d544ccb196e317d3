"""Time kernel variants (separately built .so files) on one config.
usage: python tools/sweep_ws.py CONFIG NBINS lib1.so[:kernel] lib2.so[:kernel] ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402


class Opt(ctypes.Structure):
    _fields_ = [("lanes_per_element", ctypes.c_int), ("range_mode", ctypes.c_int),
                ("block_threads", ctypes.c_int), ("kernel", ctypes.c_int)]


def main():
    cfg, nb = sys.argv[1], int(sys.argv[2])
    c = workloads.CONFIGS[cfg]
    v, x = workloads.generate(cfg, 0, min(c.n, 1 << 22))
    dev = torch.device("cuda")
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    n = vt.numel()
    outs = [torch.empty_like(vt) for _ in range(3)]
    ref = None
    for spec in sys.argv[3:]:
        path, _, kern = spec.partition(":")
        L = ctypes.CDLL(os.path.abspath(path))
        f = L.bessel_logk_f64_ex if c.precision == "f64" else L.bessel_logk_f32_ex
        f.restype = ctypes.c_int
        vp = ctypes.c_void_p
        f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, ctypes.POINTER(Opt), vp]
        o = Opt(0, 0, 0, int(kern or 0))
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        ptr = [ctypes.c_void_p(t.data_ptr()) if k in c.outputs else None
               for t, k in zip(outs, ("logk", "dv", "dx"))]

        def call():
            rc = f(ctypes.c_void_p(vt.data_ptr()), ctypes.c_void_p(xt.data_ptr()), n,
                   ptr[0], ptr[1], ptr[2], nb, ctypes.byref(o), s)
            assert rc == 0, rc
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res = [t.clone() for t in outs]
        same = "" if ref is None else " bitwise-same-as-first=" + str(all(
            torch.equal(a, b) for a, b, k in zip(res, ref, ("logk", "dv", "dx")) if k in c.outputs))
        if ref is None:
            ref = res
        print(f"{spec:50s} n={n} median {ts[5]:.3f} ms  best {ts[0]:.3f} ms  "
              f"{n / ts[5] * 1e3:.3e} evals/s{same}", flush=True)


if __name__ == "__main__":
    main()
