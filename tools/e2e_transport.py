"""Host-buffer entry point on pinned buffers: zero-copy transport (default) vs the
staged chunk pipeline (BLK_HOST_PIPELINE=1), 2^20 elements of c2 and c3, wall-clock
per call (the call synchronizes), median of 15; checks both give identical outputs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402


def main():
    n = 1 << 20
    for cfg in ("c2", "c3"):
        v, x = workloads.generate(cfg, 0, n)
        hv = torch.from_numpy(v).pin_memory()
        hx = torch.from_numpy(x).pin_memory()
        res = {}
        for mode in ("staged", "zero_copy", "staged", "zero_copy"):
            if mode == "staged":
                os.environ["BLK_HOST_PIPELINE"] = "1"
            else:
                os.environ.pop("BLK_HOST_PIPELINE", None)
            outs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
            ws = torch.empty(blk.host_workspace_bytes(1 << 18), dtype=torch.uint8, device="cuda")
            for _ in range(3):
                blk.bessel_logk_f64_host(hv, hx, *outs, nbins=128, workspace=ws, chunk=1 << 18)
            ts = []
            for _ in range(15):
                t = time.perf_counter()
                blk.bessel_logk_f64_host(hv, hx, *outs, nbins=128, workspace=ws, chunk=1 << 18)
                ts.append(time.perf_counter() - t)
            ms = sorted(ts)[len(ts) // 2] * 1e3
            res[mode] = [o.numpy().copy() for o in outs]
            print(f"{cfg} {mode:9s} {ms:.3f} ms {n / ms * 1e3:.3e} evals/s", flush=True)
        same = all(np.array_equal(a, b) for a, b in zip(res["staged"], res["zero_copy"]))
        print(f"{cfg} zero-copy outputs identical to the staged pipeline: {same}", flush=True)


if __name__ == "__main__":
    main()
