"""Computation time per (v, x) -- the paper's Sec. 3.2 experiment (P:308-322,
Fig. 3) for the proposed method on the GPU: on the accuracy grid of Sec. 3.1
(v = 0..99, x = 10^(-1..2.1), 100 x 33 cells) a batch of 2^20 copies of each
(v, x) pair is timed (FP64 entry point, n = 128 bins, one element per lane,
device time of the launch).  A batch of identical elements is the worst case
for a data-parallel kernel (every warp in the same phase at the same time),
and "the computation time in this case is the worst computation time for the
included v and x": the paper asks for a uniform map.
usage: python tools/time_map.py [--out profiles/x.json] [--copies 20] [--f32]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
from _timing import device_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--copies", type=int, default=20, help="log2 of the batch of identical pairs")
    ap.add_argument("--nbins", type=int, default=128)
    ap.add_argument("--f32", action="store_true")
    a = ap.parse_args()
    dt = torch.float32 if a.f32 else torch.float64
    n = 1 << a.copies
    vs = np.linspace(0.0, 99.0, 100)
    xs = np.logspace(-1.0, 2.1, 33)
    dev = torch.device("cuda")
    v = torch.empty(n, dtype=dt, device=dev)
    x = torch.empty(n, dtype=dt, device=dev)
    outs = [torch.empty(n, dtype=dt, device=dev) for _ in range(3)]
    fn = blk.bessel_logk_f32 if a.f32 else blk.bessel_logk_f64
    ns = np.zeros((vs.size, xs.size))
    for i, vi in enumerate(vs):
        v.fill_(float(vi))
        for j, xj in enumerate(xs):
            x.fill_(float(xj))
            ms = device_time(lambda: fn(v, x, *outs, nbins=a.nbins, lanes_per_element=1), reps=3, warm=1)
            ns[i, j] = ms * 1e6 / n
    # mixed batch of the same cells for reference (every cell's pair, shuffled)
    vv, xx = np.meshgrid(vs, xs, indexing="ij")
    rng = np.random.default_rng(0)
    idx = rng.integers(0, vv.size, n)
    vm = torch.from_numpy(vv.ravel()[idx]).to(dev, dt)
    xm = torch.from_numpy(xx.ravel()[idx]).to(dev, dt)
    mixed = device_time(lambda: fn(vm, xm, *outs, nbins=a.nbins, lanes_per_element=1), reps=5) * 1e6 / n
    flat = ns.ravel()
    worst = np.argsort(flat)[::-1][:5]
    res = {
        "what": f"ns per element of a batch of 2^{a.copies} identical (v, x), "
                f"{'FP32' if a.f32 else 'FP64'} entry point, nbins={a.nbins}",
        "min": float(flat.min()), "median": float(np.median(flat)), "max": float(flat.max()),
        "max_over_min": float(flat.max() / flat.min()),
        "max_over_median": float(flat.max() / np.median(flat)),
        "mixed_batch_ns_per_element": float(mixed),
        "worst_cells": [{"v": float(vv.ravel()[k]), "x": float(xx.ravel()[k]), "ns": float(flat[k])}
                        for k in worst],
        "by_v_max": [float(r.max()) for r in ns], "by_x_max": [float(c.max()) for c in ns.T],
        "grid_ns": ns.round(4).tolist(),
    }
    print(json.dumps({k: res[k] for k in ("what", "min", "median", "max", "max_over_min",
                                          "max_over_median", "mixed_batch_ns_per_element",
                                          "worst_cells")}, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
