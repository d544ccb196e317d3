#!/usr/bin/env python
"""Benchmark of the fused sm_100a log K_v(x) + d/dv + d/dx kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--nbins 128]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle on host cores

A step is one pass of the whole hot path (range finding + fixed-bin quadrature
+ the three outputs) over one batch.  The default workload
is config c3 of BASELINE.json -- 2^24 FP64 pairs, v~logU[10,1000],
x~logU[1e-3,10], all three outputs: the largest single-GPU FP64 config that
asks for log K, d/dv and d/dx, which is what the metric names.  With N GPUs
the one batch is split into N contiguous shards, one per rank (north_star
(4)): strong scaling, no collective on the data path; NCCL only reduces the
timings (max over ranks).  `--weak` gives every rank its own full batch.

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events
on the launching stream; between steps a 512 MiB buffer is written to flush
L2 (outside the events).  Inputs are resident in HBM.  `e2e` repeats the
metric through the C-ABI host-buffer entry point (pinned host arrays, which it
reads and writes over PCIe from the kernel -- zero-copy; v, x and the outputs
cross PCIe inside the timed region).

Roofline: the FP64 (or FP32) work per element of the kernel comes from an
ncu capture of the current kernel sources (profiles/roofline_counts.json,
written by tools/roofline_counts.py and stamped with the sha256 of the
sources it was captured from); when the sources differ the line says
"stale": true.  Peaks are measured in the same run (DFMA / FFMA / MUFU.EX2
microbenchmarks: MEASURED_PEAKS.json has no FP64 figure).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

COUNTS = os.path.join(ROOT, "profiles", "roofline_counts.json")
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2


def roofline_counts(cfg, nbins):
    """(entry, stale, sha) for this workload from profiles/roofline_counts.json."""
    from paper_2108_11560_b200.build import kernel_source_sha256
    sha = kernel_source_sha256()
    try:
        data = json.load(open(COUNTS))
    except (OSError, ValueError):
        return None, True, sha
    entry = data.get("captures", {}).get(f"{cfg}/{nbins}")
    return entry, data.get("kernel_source_sha256") != sha, data.get("kernel_source_sha256")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c3", choices=list(workloads.CONFIGS))
    p.add_argument("--nbins", type=int, default=128)
    p.add_argument("--n", type=int, default=0, help="override elements per GPU")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=None,
                   help="oracle seconds: the GPU arm's cpu_baseline (default 10), or per "
                        "step of --impl reference (default: the run fits in ~2 minutes)")
    p.add_argument("--out", default="")
    p.add_argument("--weak", action="store_true",
                   help="every rank its own full batch (default: the one batch in N shards)")
    return p.parse_args()


def _generate_chunked(cfg, start, count, total):
    """Inputs [start, start+count) in 2^24-element pieces (bounded host memory)."""
    import numpy as _np
    parts_v, parts_x = [], []
    step = 1 << 24
    for s0 in range(start, start + count, step):
        m = min(step, start + count - s0)
        v, x = workloads.generate(cfg, s0, m, n=total)
        parts_v.append(v)
        parts_x.append(x)
    if not parts_v:
        return workloads.generate(cfg, 0, 0, n=max(total, 1))
    return _np.concatenate(parts_v), _np.concatenate(parts_x)


def cpu_info():
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        aff = os.cpu_count()
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return aff, model


def oracle_rate(cfg, nbins, seconds, threads):
    """Time the oracle (as it stands) on a bounded prefix sample of the workload.
    Returns (evals/s, evaluations, seconds, sample elements)."""
    import oracle
    v, x = workloads.generate(cfg, 0, 2048)
    t = time.perf_counter()
    oracle.logk(v.astype(np.float64), x.astype(np.float64), nbins, threads=threads)
    probe = time.perf_counter() - t
    per = probe / 2048
    want = max(4096, int(seconds / per * threads * 0.9))
    n = int(min(workloads.CONFIGS[cfg].n, want, 1 << 22))
    v, x = workloads.generate(cfg, 0, n)
    v = v.astype(np.float64)
    x = x.astype(np.float64)
    # repeat passes over the prefix sample until ~`seconds` of CPU work
    passes, t = 0, time.perf_counter()
    while True:
        oracle.logk(v, x, nbins, threads=threads)
        passes += 1
        dt = time.perf_counter() - t
        if dt >= seconds * 0.9 or passes * n >= want:
            break
    return passes * n / dt, passes * n, dt, n


class ClockSampler:
    """SM clock + clock-event reasons sampled DURING the timed region.

    NVML (pynvml) polled from a thread every ~1 ms (the timed region of a
    default run is only a few ms long, below nvidia-smi's 100 ms sampling);
    only samples taken between mark_begin() and mark_end() count.  Falls back
    to `nvidia-smi -lms 100` when NVML is unavailable."""
    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80))
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []          # (t, sm_mhz, max_mhz, reasons_mask)
        self.begin = self.end = None
        self.stop_flag = threading.Event()
        self.nvml = None
        self.proc = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll_nvml, daemon=True)
        except Exception:  # pragma: no cover - no NVML
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.thread = threading.Thread(target=self._read_smi, daemon=True)
            except OSError:
                return
        self.thread.start()

    def _poll_nvml(self):
        pynvml, h = self.nvml
        while not self.stop_flag.is_set():
            try:
                mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:  # pragma: no cover
                break
            self.samples.append((time.perf_counter(), float(mhz), float(self.max_mhz), int(rs)))
            time.sleep(0.001)

    def _read_smi(self):
        for ln in self.proc.stdout:
            f = [c.strip() for c in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                mask = 0
                for (nm, bit), val in zip((("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
                                           ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4)),
                                          f[4:8]):
                    if val.lower() == "active":
                        mask |= bit
                self.samples.append((time.perf_counter(), float(f[0]), float(f[1]), mask))
            except ValueError:
                continue

    def mark_begin(self):
        self.begin = time.perf_counter()

    def mark_end(self):
        self.end = time.perf_counter()

    def stop(self):
        self.stop_flag.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if getattr(self, "thread", None) is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        lo = self.begin if self.begin is not None else -1e30
        hi = self.end if self.end is not None else 1e30
        inside = [smp for smp in self.samples if lo <= smp[0] <= hi] or self.samples
        mask = 0
        for smp in inside:
            mask |= smp[3]
        return {"sm_mhz": statistics.median(smp[1] for smp in inside),
                "sm_max_mhz": max(smp[2] for smp in inside),
                "samples": len(inside),
                "source": "nvml 1 ms" if self.nvml else "nvidia-smi 100 ms",
                "window": "timed region" if len(inside) < len(self.samples) or self.begin else "run",
                "reasons": sorted(nm for nm, bit in self.REASONS if mask & bit)}


def workload_config(args, c, total, world):
    """The `config` object: the same keys and values for both arms."""
    return {"workload": args.config, "describe": c.describe, "elements_total": total,
            "nbins": args.nbins, "outputs": list(c.outputs),
            "l2": "flushed between timed steps (512 MiB write, outside events)",
            "parallelism": f"dp{world} (contiguous element shards, no collective)"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on host cores (rank 0 only)."""
    if rank != 0:
        return
    cores, model = cpu_info()
    c = workloads.CONFIGS[args.config]
    per_step = args.cpu_seconds or max(1.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    rates = []
    n_used = n_el = 0
    for i in range(args.warmup + args.steps):
        r, n_used, _, n_el = oracle_rate(args.config, args.nbins, per_step, cores)
        if i >= args.warmup:
            rates.append(r)
    value = statistics.median(rates)
    total = (args.n or c.n) * (args.gpus if args.weak else 1)
    sample = (f"{n_used} evaluations per step: the first {n_el} elements of {args.config}, "
              f"{n_used // max(1, n_el)} pass(es), {cores} threads, CPU {model}")
    line = {
        "impl": "reference", "metric": "logK+dv+dx evals/sec FP64" if c.precision == "f64"
        else "logK+dv+dx evals/sec FP32", "value": value,
        "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_used / value * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64" if c.precision == "f64" else "f32",
        "data": "synthetic (seeded numpy PCG64 blocks, BASELINE.json config distribution)",
        "config": workload_config(args, c, total, args.gpus),
        "sample": sample,
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2108_11560_b200 as blk
    from paper_2108_11560_b200.dist import shard_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = workloads.CONFIGS[args.config]
    dt = torch.float64 if c.precision == "f64" else torch.float32
    if args.weak:
        # weak scaling: every rank its own batch of the config's size
        scaling = "weak"
        per = args.n or c.n
        total = per * world
        lo, hi = rank * per, (rank + 1) * per
    else:
        # strong scaling: the config's one batch in contiguous shards (north_star (4))
        scaling = "strong"
        total = args.n or c.n
        lo, hi = shard_range(total, world, rank)
    n = hi - lo
    v_np, x_np = _generate_chunked(args.config, lo, n, total)
    v = torch.from_numpy(v_np).to(dev)
    x = torch.from_numpy(x_np).to(dev)
    outs = {k: (torch.empty(n, dtype=dt, device=dev) if k in c.outputs else None)
            for k in ("logk", "dv", "dx")}
    fn = blk.bessel_logk_f64 if dt == torch.float64 else blk.bessel_logk_f32
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        fn(v, x, outs["logk"], outs["dv"], outs["dx"], nbins=args.nbins, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # peak-rate microbenchmarks (roofline denominators), same process and clocks
    mb_out = torch.empty(148 * 4 * 256, dtype=torch.float64, device=dev)
    mb_out32 = torch.empty(148 * 4 * 256, dtype=torch.float32, device=dev)

    def mb(kind, out, iters):
        blk.microbench(kind, 148 * 4, 256, 64, out, stream=stream)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ops = blk.microbench(kind, 148 * 4, 256, iters, out, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return ops / (e0.elapsed_time(e1) * 1e-3)

    fp64_ops = mb("fp64", mb_out, 20000)
    fp32_ops = mb("fp32", mb_out32, 20000)
    mufu_ops = mb("mufu", mb_out32, 5000)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark_begin()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        starts[i].record(stream)
        step()
        ends[i].record(stream)
    torch.cuda.synchronize()
    sampler.mark_end()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    ms_per_step = total_ms / args.steps
    value = total * args.steps / (total_ms * 1e-3)
    local_ms = sum(step_ms) / args.steps        # this rank's kernel time per launch

    # end to end through the host-buffer C-ABI entry point (pinned host
    # buffers: zero-copy, no device workspace needed)
    e2e = None
    e2e_launches = 0
    if not args.no_e2e:
        hv = torch.from_numpy(v_np).pin_memory()
        hx = torch.from_numpy(x_np).pin_memory()
        hout = {k: (torch.empty(n, dtype=dt).pin_memory() if k in c.outputs else None)
                for k in ("logk", "dv", "dx")}
        hfn = blk.bessel_logk_f64_host if dt == torch.float64 else blk.bessel_logk_f32_host

        def hstep():
            hfn(hv, hx, hout["logk"], hout["dv"], hout["dx"], nbins=args.nbins, stream=stream)

        for _ in range(2):
            hstep()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            hstep()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e_launches = args.steps   # zero-copy: one kernel launch per call
        esz = 8 if dt == torch.float64 else 4
        e2e = {"value": total * args.steps / (float(e2e_ms.item()) * 1e-3), "unit": "evals/s",
               "h2d_bytes_per_step": 2 * n * esz * world,
               "d2h_bytes_per_step": len(c.outputs) * n * esz * world,
               "path": f"{hfn.__name__} (pinned host buffers: zero-copy, the kernel reads and "
                       "writes them over PCIe)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    counts, stale, counts_sha = roofline_counts(args.config, args.nbins)
    rate = n / (local_ms * 1e-3)                # this rank's kernel, elements per second
    esz = 8 if dt == torch.float64 else 4
    alg_bytes = n * esz * (2 + len(c.outputs))
    common = {"stale": stale, "counts": "profiles/roofline_counts.json" if counts else None,
              "counts_source_sha256": counts_sha,
              "kernel_time": "CUDA events around each launch on its stream (one launch per step)",
              "algorithmic_bytes": alg_bytes,
              "hbm_gbs": alg_bytes / (local_ms * 1e-3) / 1e9,
              "traffic": counts["dram_bytes_per_element"] * n if counts else None,
              "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)"}
    if dt == torch.float64:
        peak = fp64_ops * 2 / 1e12
        ach = counts["fp64_flops_per_element"] * rate / 1e12 if counts else None
        iss = counts["fp64_inst_per_element"] * rate if counts else None
        roof = {"bound": "alu", "pipe": "fp64", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak if ach else None,
                "fp64_issue": {"achieved_inst_per_s": iss, "peak_inst_per_s": fp64_ops,
                               "frac": iss / fp64_ops if iss else None,
                               "inst_per_element": counts["fp64_inst_per_element"] if counts else None},
                "flops_per_element": counts["fp64_flops_per_element"] if counts else None,
                "fp32_frac": (counts["fp32_flops_per_element"] * rate / 1e12) / (fp32_ops * 2 / 1e12)
                if counts else None,
                "mufu_frac": counts["mufu_per_element"] * rate / mufu_ops if counts else None,
                "peak_source": "in-run DFMA microbenchmark (blk_microbench_fp64; 2 flops per DFMA); "
                               f"nominal {NOMINAL_FP64_TFLOPS:.1f} TF/s = 148 SM x 64 DFMA/clk x 1.965 GHz"}
    else:
        peak32 = fp32_ops * 2 / 1e12
        ach = counts["fp32_flops_per_element"] * rate / 1e12 if counts else None
        roof = {"bound": "alu", "pipe": "fp32 (+ fp64 exponent, MUFU)", "achieved": ach,
                "peak": peak32, "unit": "TFLOP/s", "frac": ach / peak32 if ach else None,
                "fp64_frac": (counts["fp64_flops_per_element"] * rate / 1e12) / (fp64_ops * 2 / 1e12)
                if counts else None,
                "mufu_frac": counts["mufu_per_element"] * rate / mufu_ops if counts else None,
                "peak_source": "in-run FFMA/DFMA/MUFU.EX2 microbenchmarks"}
    roof.update(common)
    # issue slots: warp instructions per element (ncu) against 4 per clock per SM at the
    # SM clock sampled during the timed region -- the resource the FP32 kernel is bound by
    # (no single pipe saturates there), and a cross-check of ncu's issue-active figure
    sm_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
    if counts and counts.get("warp_inst_per_32_elements"):
        wi = counts["warp_inst_per_32_elements"] / 32.0 * rate
        roof["issue"] = {"warp_inst_per_32_elements": counts["warp_inst_per_32_elements"],
                         "achieved_warp_inst_per_s": wi, "peak_warp_inst_per_s": 148 * 4 * sm_hz,
                         "frac": wi / (148 * 4 * sm_hz)}
        if dt != torch.float64:
            # the FP32 kernel mixes FP32 FMA-pipe work, one FP64 exponent per 4 nodes and
            # one MUFU.EX2 per node; no pipe saturates (ncu: issue ~64%, XU ~52%, FMA ~33%)
            # and issue slots are what it is bound by: that is the headline fraction, the
            # FFMA-flop fraction stays beside it
            roof["fp32_flops"] = {"achieved": roof["achieved"], "peak": roof["peak"],
                                  "unit": "TFLOP/s", "frac": roof["frac"]}
            roof.update({"pipe": "issue slots (FP32 FMA + FP64 exponent + MUFU mix)",
                         "achieved": wi, "peak": 148 * 4 * sm_hz, "unit": "warp-inst/s",
                         "frac": roof["issue"]["frac"],
                         "peak_source": "4 warp instructions per clock per SM x 148 SMs x the SM "
                                        "clock sampled in the timed region; flop peaks from the "
                                        "in-run FFMA/DFMA/MUFU.EX2 microbenchmarks"})

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cores, model = cpu_info()
        r, ns, secs, nel = oracle_rate(args.config, args.nbins, args.cpu_seconds or 10.0, cores)
        cpu = {"value": r, "unit": "evals/s", "cores": cores, "kind": "oracle",
               "sample": f"{ns} evaluations: the first {nel} elements of {args.config}, "
                         f"{ns // max(1, nel)} pass(es) ({secs:.1f} s, {cores} threads, {model})"}

    line = {
        "metric": "logK+dv+dx evals/sec FP64" if dt == torch.float64 else "logK+dv+dx evals/sec FP32",
        "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64" if dt == torch.float64 else "f32",
        "data": "synthetic (seeded numpy PCG64 blocks, BASELINE.json config distribution)",
        "config": workload_config(args, c, total, world),
        "elements_per_gpu": n,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "gpu_launches_e2e": e2e_launches,
        "clocks": clocks,
        "peaks_measured": {"fp64_tflops": fp64_ops * 2 / 1e12, "fp32_tflops": fp32_ops * 2 / 1e12,
                           "mufu_ex2_gops": mufu_ops / 1e9},
        "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
    }
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(line, f, indent=1)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
