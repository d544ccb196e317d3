"""evals/s of the fused FP64 kernel vs batch size (wave quantisation / tail).
usage: python tools/time_sizes.py CFG N1 N2 ...   (sizes may be 'w9' = 9 full waves of 6x148 blocks of 128)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


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
    for n in sizes:
        ms = timeit(lambda: blk.bessel_logk_f64(vt[:n], xt[:n], o[0][:n], o[1][:n], o[2][:n], nbins=128))
        print(f"{cfg} n={n:9d} waves={n / (6 * 148 * 128):6.2f} {ms:.4f} ms  {n / ms * 1e3:.3e} evals/s",
              flush=True)


if __name__ == "__main__":
    main()
