"""Latency of small batches: 200 back-to-back launches on one stream between two
events (resolution well below a microsecond per launch); several library builds.
usage: python tools/small_batch.py CFG lib1.so lib2.so ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402

cfg = sys.argv[1]
vp = ctypes.c_void_p
for path in sys.argv[2:]:
    L = ctypes.CDLL(os.path.abspath(path))
    f = L.bessel_logk_f64
    f.restype = ctypes.c_int
    f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp]
    line = []
    for n in (1000, 3000, 10000, 20000):
        v, x = workloads.generate(cfg, 0, min(n, workloads.CONFIGS[cfg].n))
        vt, xt = torch.from_numpy(v).cuda(), torch.from_numpy(x).cuda()
        o = [torch.empty_like(vt) for _ in range(3)]
        P = [vp(t.data_ptr()) for t in (vt, xt, *o)]
        s = vp(torch.cuda.current_stream().cuda_stream)
        for _ in range(10):
            f(P[0], P[1], vt.numel(), P[2], P[3], P[4], 128, s)
        torch.cuda.synchronize()
        torch.cuda._sleep(200000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            f(P[0], P[1], vt.numel(), P[2], P[3], P[4], 128, s)
        e1.record()
        torch.cuda.synchronize()
        line.append(f"n={vt.numel()}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us")
    print(f"{os.path.basename(path):12s} " + "  ".join(line), flush=True)
