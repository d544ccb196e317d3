"""evals/s of the fused FP64 kernel vs batch size (wave quantisation / tail).
usage: python tools/time_sizes.py CFG N1 N2 ...   (sizes may be 'w9' = 9 full waves of 6x148 blocks of 128)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _timing import device_time  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402



def timeit(fn, reps=20):
    return device_time(fn, reps)


def main():
    cfg = sys.argv[1]
    c = workloads.CONFIGS[cfg]
    sizes = []
    for s in sys.argv[2:]:
        sizes.append(int(float(s[1:]) * 6 * 148 * 128) if s.startswith("w") else int(s))
    nmax = max(sizes)
    v, x = workloads.generate(cfg, 0, min(nmax, c.n))
    reps = (nmax + len(v) - 1) // len(v)
    dev = torch.device("cuda")
    vt = torch.from_numpy(v).to(dev).repeat(reps)[:nmax]
    xt = torch.from_numpy(x).to(dev).repeat(reps)[:nmax]
    o = [torch.empty_like(vt) for _ in range(3)]
    import ctypes
    from paper_2108_11560_b200 import build as _b
    L = ctypes.CDLL(_b.build_diag())   # the split exists only in the diagnostics build
    f = L.blk_debug_split_f64
    f.restype = ctypes.c_int
    vp = ctypes.c_void_p
    f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int, vp]
    scratch = torch.empty(nmax * 32, dtype=torch.uint8, device=dev)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = [ctypes.c_void_p(t.data_ptr()) for t in (vt, xt, *o, scratch)]
    split = "--split" in os.environ.get("TS_OPTS", "")
    lanes_list = [int(a) for a in os.environ.get("TS_LANES", "0").split(",")]
    for n in sizes:
      for lanes in lanes_list:
        ms = timeit(lambda: blk.bessel_logk_f64(vt[:n], xt[:n], o[0][:n], o[1][:n], o[2][:n], nbins=128,
                                                lanes_per_element=lanes))
        line = (f"{cfg} n={n:9d} waves={n / (6 * 148 * 128):6.2f} lanes={lanes} fused {ms:.4f} ms  "
                f"{n / ms * 1e3:.3e} evals/s")
        if split and lanes == lanes_list[0]:
            f(P[0], P[1], n, P[2], P[3], P[4], 128, P[5], 1, s)
            mp = timeit(lambda: f(P[0], P[1], n, P[2], P[3], P[4], 128, P[5], 1, s))
            mq = timeit(lambda: f(P[0], P[1], n, P[2], P[3], P[4], 128, P[5], 2, s))
            line += f" | plan {mp:.4f} ms quad {mq:.4f} ms"
        print(line, flush=True)


if __name__ == "__main__":
    main()
