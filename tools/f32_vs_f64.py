"""FP32 vs FP64 entry point on the SAME inputs (BASELINE.json config c4's
distribution, drawn in float32 and widened exactly to float64 for the FP64
kernel), all three outputs, n = 128 bins; device time per launch (CUDA events
around single launches, L2 flushed in between) and evals/s of each.

    python tools/f32_vs_f64.py [--n 16777216] [--nbins 128] [--cfg c4]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402


def timed(fn, reps, flush):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=1 << 24)
    p.add_argument("--nbins", type=int, nargs="+", default=[128])
    p.add_argument("--cfg", default="c4")
    p.add_argument("--reps", type=int, default=10)
    a = p.parse_args()
    dev = torch.device("cuda:0")
    v, x = workloads.generate(a.cfg, 0, a.n)
    v32 = torch.from_numpy(v.astype("float32")).to(dev)
    x32 = torch.from_numpy(x.astype("float32")).to(dev)
    v64, x64 = v32.double(), x32.double()
    o32 = [torch.empty_like(v32) for _ in range(3)]
    o64 = [torch.empty_like(v64) for _ in range(3)]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for nb in a.nbins:
        t64 = timed(lambda: blk.bessel_logk_f64(v64, x64, *o64, nbins=nb), a.reps, flush)
        t32 = timed(lambda: blk.bessel_logk_f32(v32, x32, *o32, nbins=nb), a.reps, flush)
        print(json.dumps({"cfg": a.cfg, "n": a.n, "nbins": nb, "f64_ms": t64, "f32_ms": t32,
                          "f64_evals_s": a.n / (t64 * 1e-3), "f32_evals_s": a.n / (t32 * 1e-3),
                          "f32_speedup": t64 / t32}), flush=True)


if __name__ == "__main__":
    main()
