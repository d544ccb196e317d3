"""Large seeded fuzz of the FP64 / FP32 entry points against the oracle (AUTO
mode, one element per lane and automatic lanes), over the five configs'
distributions and random bin counts from 48 up (where parity is asserted
element by element): prints the worst error of each output in units of the
north_star tolerance.  usage: python tests/tools/fuzz_parity.py [--n 200000] [--seed 1]"""
import argparse
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
from parity import TOL, max_errors  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    worst = {}
    for trial in range(12):
        cfg = ("c1", "c2", "c3", "c4", "c5")[trial % 5]
        nb = int(rng.choice([48, 49, 55, 63, 64, 65, 100, 127, 128, 129, 200, 256]))
        c = workloads.CONFIGS[cfg]
        m = min(a.n, c.n)
        start = int(rng.integers(0, max(1, c.n - m)))
        v, x = workloads.generate(cfg, start, m)
        prec = "f32" if c.precision == "f32" else "f64"
        dt = torch.float32 if prec == "f32" else torch.float64
        vt = torch.from_numpy(np.asarray(v)).to("cuda", dt)
        xt = torch.from_numpy(np.asarray(x)).to("cuda", dt)
        for lanes in (1, 0):
            got = dict(zip(("logk", "dv", "dx"),
                           (t.cpu().numpy() for t in blk.log_bessel_k(vt, xt, nbins=nb, lanes_per_element=lanes))))
            vv, xx = np.asarray(v, np.float64), np.asarray(x, np.float64)
            le = oracle.log_eps_f32() if prec == "f32" else None
            ref = oracle.logk(vv, xx, nb, threads=16, **({"log_eps": le} if le is not None else {}))
            e = max_errors(got, dict(zip(("logk", "dv", "dx"), ref)))
            key = f"{cfg} {prec}"
            r = {k: e[k] / TOL[prec][k] for k in e}
            w = worst.setdefault(key, {k: 0.0 for k in r})
            for k in r:
                w[k] = max(w[k], r[k])
            print(f"{cfg} start={start} n={m} nbins={nb} lanes={lanes or 'auto'}: max err / tol "
                  + " ".join(f"{k} {r[k]:.3g}" for k in r), flush=True)
    print("worst:", {k: {kk: round(vv, 4) for kk, vv in w.items()} for k, w in worst.items()})
    bad = [k for k, w in worst.items() if any(vv > 1.0 for vv in w.values())]
    print("FAIL" if bad else "PASS", bad)


if __name__ == "__main__":
    main()
