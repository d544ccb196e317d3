"""Throughput + sampled parity on every BASELINE.json config (one GPU).
usage: python tests/tools/report_configs.py [--nbins 128] [--out profiles/x.json]
Prints one line per (config, nbins, kernel variant)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402
from parity import max_errors  # noqa: E402


def gen_device(cfg, n, dev):
    c = workloads.CONFIGS[cfg]
    dt = torch.float32 if c.precision == "f32" else torch.float64
    vt = torch.empty(n, dtype=dt, device=dev)
    xt = torch.empty(n, dtype=dt, device=dev)
    step = 1 << 24
    for s in range(0, n, step):
        v, x = workloads.generate(cfg, s, min(step, n - s), n=n)
        vt[s:s + v.size] = torch.from_numpy(v).to(dev)
        xt[s:s + v.size] = torch.from_numpy(x).to(dev)
    return vt, xt


def time_launch(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in range(reps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nbins", type=int, nargs="+", default=[128])
    ap.add_argument("--configs", nargs="+", default=list(workloads.CONFIGS))
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    dev = torch.device("cuda")
    rows = []
    for cfg in args.configs:
        c = workloads.CONFIGS[cfg]
        vt, xt = gen_device(cfg, c.n, dev)
        outs = [torch.empty_like(vt) if k in c.outputs else None for k in ("logk", "dv", "dx")]
        fn64 = blk.bessel_logk_f64 if c.precision == "f64" else blk.bessel_logk_f32
        idx = np.unique(np.concatenate([workloads.sample_indices(cfg, 2048, seed=21),
                                        np.arange(256), np.arange(c.n - 256, c.n)]))
        vs, xs = workloads.gather(cfg, idx)
        for nb in args.nbins:
            ref = dict(zip(("logk", "dv", "dx"),
                           oracle.logk(vs.astype(np.float64), xs.astype(np.float64), nb, threads=16)))
            reps = 20 if c.n <= (1 << 24) else 5
            med, best = time_launch(lambda: fn64(vt, xt, *outs, nbins=nb), reps)
            it = torch.from_numpy(idx).to(dev)
            got = {k: o[it].double().cpu().numpy() for k, o in zip(("logk", "dv", "dx"), outs)
                   if o is not None}
            err = max_errors(got, ref)
            row = {"config": cfg, "n": c.n, "precision": c.precision, "nbins": nb,
                   "outputs": list(c.outputs), "ms_median": med, "ms_best": best,
                   "evals_per_s": c.n / (med * 1e-3), "max_rel_err_vs_oracle": err,
                   "sample": int(idx.size)}
            rows.append(row)
            print(json.dumps(row), flush=True)
        del vt, xt, outs
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
