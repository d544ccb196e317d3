"""Time the fused FP64 kernel with the FP32 (auto) and the FP64 range finder
(range_mode 0 / 1) on the bench configs; reports ms per call and evals/s."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_2108_11560_b200 as blk
from tools._timing import device_time


def main():
    n = 1 << 20
    for cfg in ("c2", "c3", "c4"):
        v, x = workloads.generate(cfg, 0, n)
        v = torch.as_tensor(v, dtype=torch.float64, device="cuda")
        x = torch.as_tensor(x, dtype=torch.float64, device="cuda")
        outs = [torch.empty_like(v) for _ in range(3)]
        for mode in (0, 1):
            fn = lambda: blk.bessel_logk_f64(v, x, *outs, nbins=128, range_mode=mode)
            ms = device_time(fn)
            print(f"{cfg} range_mode {mode} {ms:.3f} ms {n / ms * 1e3:.3e} evals/s", flush=True)


if __name__ == "__main__":
    main()
