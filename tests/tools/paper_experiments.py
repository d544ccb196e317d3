"""The paper's experiments, run on the B200 path.

(a) Accuracy grid of Sec. 3.1 (Fig. 2): v = 0..99 (100 values) x
    x = 10^-1 .. 10^2.1 (33 values, log-spaced), error metric
    log10(|Delta|/eps + 1) with Delta relative to max(1, |ref|) for
    log K and relative for the derivatives (reading R19), reference = the
    long-double brute force of the plain definition (oracle/brute.c) -- the
    paper used Mathematica, which is not available.  The FP64 kernel, the
    FP32 entry point (eps = 2^-23) and the CPU oracle are all scored.
(b) Batch-size sweep of Sec. 3.4 (Fig. 5): v = 10^(2r)-1,
    x = 10^(3r-1), sizes 10 .. 2^28; time per call (CUDA events, one launch
    each, inputs resident) -- flat until the GPU is filled, then linear.

usage: python tests/tools/paper_experiments.py [--out profiles/r01_paper_experiments.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402

EPS64 = 2.0 ** -52
EPS32 = 2.0 ** -23


def metric(got, ref, kind, eps):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.maximum(1.0, np.abs(ref)) if kind == "logk" else np.where(ref == 0, 1.0, np.abs(ref))
    return np.log10(np.abs(got - ref) / den / eps + 1.0)


def accuracy_grid(nbins=128):
    vv, xx = np.meshgrid(np.linspace(0.0, 99.0, 100), np.logspace(-1.0, 2.1, 33), indexing="ij")
    v, x = vv.ravel(), xx.ravel()
    bl, bv, bx = oracle.brute(v, x, 1 << 14, threads=16)
    ref = {"logk": bl, "dv": bv, "dx": bx}
    dev = torch.device("cuda")
    out = {}
    for name, dt, eps in (("gpu_f64", torch.float64, EPS64), ("gpu_f32", torch.float32, EPS32)):
        vt = torch.from_numpy(v).to(dev, dt)
        xt = torch.from_numpy(x).to(dev, dt)
        res = blk.log_bessel_k(vt, xt, nbins=nbins)
        torch.cuda.synchronize()
        got = dict(zip(("logk", "dv", "dx"), (r.double().cpu().numpy() for r in res)))
        out[name] = summarize(got, ref, eps)
    ol, ov, ox = oracle.logk(v, x, nbins, threads=16)
    out["oracle_f64"] = summarize({"logk": ol, "dv": ov, "dx": ox}, ref, EPS64)
    return out


def summarize(got, ref, eps):
    s = {}
    for k in ("logk", "dv", "dx"):
        m = metric(got[k], ref[k], k, eps)
        m = m[np.isfinite(m)]
        s[k] = {"mean": float(m.mean()), "max": float(m.max()),
                "cells_ge_1": int((m >= 1).sum()), "cells_ge_4": int((m >= 4).sum())}
    return s


def batch_sweep(nbins=128, max_log2=28):
    dev = torch.device("cuda")
    sizes = [10, 100, 1000, 10_000, 100_000] + [1 << k for k in range(17, max_log2 + 1)]
    v, x = workloads.generate("fig5", 0, sizes[-1], n=sizes[-1])
    vt_all = torch.from_numpy(v).to(dev)
    xt_all = torch.from_numpy(x).to(dev)
    rows = []
    for n in sizes:
        vt, xt = vt_all[:n], xt_all[:n]
        outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(3)]
        for _ in range(3):
            blk.bessel_logk_f64(vt, xt, *outs, nbins=nbins)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            blk.bessel_logk_f64(vt, xt, *outs, nbins=nbins)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        rows.append({"n": n, "ms": ts[3], "evals_per_s": n / ts[3] * 1e3})
        print(json.dumps(rows[-1]), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--max-log2", type=int, default=28)
    args = ap.parse_args()
    res = {"accuracy_grid_n128": accuracy_grid(128), "accuracy_grid_n64": accuracy_grid(64)}
    print(json.dumps(res, indent=1), flush=True)
    res["batch_sweep"] = batch_sweep(128, args.max_log2)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
