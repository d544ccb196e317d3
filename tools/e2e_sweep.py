"""End-to-end (host buffers, H2D + kernel + D2H) throughput vs chunk size.
usage: python tools/e2e_sweep.py CFG N chunk1 chunk2 ..."""
import os
import sys

# chunked (staged) transport: pinned buffers would otherwise take the zero-copy one
os.environ["BLK_HOST_PIPELINE"] = "1"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2108_11560_b200 as blk  # noqa: E402
import workloads  # noqa: E402


def main():
    cfg, n = sys.argv[1], int(sys.argv[2])
    v, x = workloads.generate(cfg, 0, n)
    hv = torch.from_numpy(v).pin_memory()
    hx = torch.from_numpy(x).pin_memory()
    ho = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
    for ch in [int(c) for c in sys.argv[3:]]:
        ws = torch.empty(blk.host_workspace_bytes(ch), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream()

        def step():
            blk.bessel_logk_f64_host(hv, hx, *ho, nbins=128, workspace=ws, chunk=ch, stream=st)

        for _ in range(3):
            step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(10):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{cfg} n={n} chunk={ch:8d} {ms:.3f} ms/step {n / ms * 1e3:.3e} evals/s", flush=True)


if __name__ == "__main__":
    main()
