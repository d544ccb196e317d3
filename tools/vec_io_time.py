"""BLK_KERNEL_SIMPLE vs BLK_KERNEL_VEC128 (128-bit warp-cooperative I/O) on the
full-size configs through the in-tree library, interleaved rounds, CUDA-event
time of one launch (tools/_timing.py).
usage: python tools/vec_io_time.py [CFG ...]   (default c3 c4 c2)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402
from _timing import device_time  # noqa: E402


def main():
    dev = torch.device("cuda")
    for cfg in sys.argv[1:] or ["c3", "c4", "c2"]:
        c = workloads.CONFIGS[cfg]
        n = min(c.n, 1 << 26)
        dt = torch.float32 if c.precision == "f32" else torch.float64
        v, x = workloads.generate(cfg, 0, n)
        vt = torch.from_numpy(np.asarray(v)).to(dev, dt)
        xt = torch.from_numpy(np.asarray(x)).to(dev, dt)
        f = blk.bessel_logk_f32 if dt == torch.float32 else blk.bessel_logk_f64
        res = {}
        for name, kern in (("simple", blk.BLK_KERNEL_SIMPLE), ("vec128", blk.BLK_KERNEL_VEC128)):
            o = [torch.empty_like(vt) for _ in range(3)]
            res[name] = (o, (lambda o=o, kern=kern: f(vt, xt, *o, kernel=kern, lanes_per_element=1)))
            res[name][1]()
        torch.cuda.synchronize()
        same = all(torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0))
                   for a, b in zip(res["simple"][0], res["vec128"][0]))
        ts = {k: [] for k in res}
        for _ in range(5):
            for k, (_, fn) in res.items():
                ts[k].append(device_time(fn, reps=5))
        ms = {k: float(np.median(t)) for k, t in ts.items()}
        print(f"{cfg} n={n} {c.precision}: simple {ms['simple']:.4f} ms ({n / ms['simple'] * 1e3:.4e}/s), "
              f"vec128 {ms['vec128']:.4f} ms ({n / ms['vec128'] * 1e3:.4e}/s), "
              f"vec128/simple time {ms['vec128'] / ms['simple']:.4f}, bitwise equal {same}", flush=True)


if __name__ == "__main__":
    main()
