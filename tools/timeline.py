"""Per-warp timeline of the fused FP64 kernel (diagnostic build with BLK_TIMELINE):
when warps start, finish their plan and finish, relative to the first start.
usage: python tools/timeline.py LIB.so CFG N"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402


def main():
    lib, cfg, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
    L = ctypes.CDLL(os.path.abspath(lib))
    vp = ctypes.c_void_p
    f = L.bessel_logk_f64
    f.restype = ctypes.c_int
    f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp]
    v, x = workloads.generate(cfg, 0, n)
    dev = torch.device("cuda")
    vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
    o = [torch.empty_like(vt) for _ in range(3)]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o)]
    for _ in range(5):
        f(P[0], P[1], n, P[2], P[3], P[4], 128, s)
    torch.cuda.synchronize()
    W = (n + 31) // 32
    buf = (ctypes.c_ulonglong * (W * 4))()
    L.blk_debug_timeline(buf, ctypes.c_size_t(W))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(W, 4).astype(np.float64)
    t0 = a[:, 0].min()
    st, pl, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
    T = en.max()
    print(f"{cfg} n={n} warps={W} kernel span {T:.1f} us")
    print(f"  warp duration: plan mean {np.mean(pl - st):.1f} us max {np.max(pl - st):.1f}; "
          f"quad mean {np.mean(en - pl):.1f} max {np.max(en - pl):.1f}; total mean {np.mean(en - st):.1f}")
    print(f"  last warp start {st.max():.1f} us; first warp end {en.min():.1f} us")
    # active warps over time (per-SM average) in 20 bins
    edges = np.linspace(0, T, 41)
    mid = 0.5 * (edges[1:] + edges[:-1])
    act = [np.sum((st <= m) & (en > m)) / 148 for m in mid]
    inplan = [np.sum((st <= m) & (pl > m)) / 148 for m in mid]
    for m, ac, ip in zip(mid, act, inplan):
        print(f"  t={m:7.1f} us  warps/SM {ac:5.1f}  in plan {ip:5.1f}")


if __name__ == "__main__":
    main()
