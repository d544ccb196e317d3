"""Dump the kernels' plans and outputs for offline analysis (no oracle here).
    python tools/dump_plans.py OUT.npz"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402


def wide(seed, n=6000):
    rng = np.random.default_rng(seed)
    v = 10.0 ** rng.uniform(-6, 4, n)
    v[rng.random(n) < 0.02] = 0.0
    x = 10.0 ** rng.uniform(-12, 6, n)
    return v, x


def main():
    dev = torch.device("cuda:0")
    sets = {"c1": workloads.generate("c1", 0, 1500)}
    for nb in (64, 96, 127, 2, 8):
        sets[f"wide{nb}"] = wide((5151 if nb >= 48 else 4242) + nb)
    out = {}
    for name, (v, x) in sets.items():
        vt = torch.from_numpy(np.asarray(v, np.float64)).to(dev)
        xt = torch.from_numpy(np.asarray(x, np.float64)).to(dev)
        out[f"{name}_v"], out[f"{name}_x"] = np.asarray(v, np.float64), np.asarray(x, np.float64)
        for nb in ((2, 3, 8, 16, 64, 128) if name == "c1" else (int(name[4:]),)):
            for mode in (0, 1):
                plan = blk.bessel_logk_plan_f64(vt, xt, nbins=nb, range_mode=mode)
                res = blk.log_bessel_k(vt, xt, nbins=nb, range_mode=mode, lanes_per_element=1)
                torch.cuda.synchronize()
                out[f"{name}_n{nb}_m{mode}_plan"] = np.stack([p.cpu().numpy() for p in plan], 1)
                out[f"{name}_n{nb}_m{mode}_out"] = np.stack([r.cpu().numpy() for r in res], 1)
    np.savez_compressed(sys.argv[1], **out)
    print("saved", len(out))


if __name__ == "__main__":
    main()
