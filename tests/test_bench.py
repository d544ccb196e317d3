"""bench.py's output contract: one JSON line with the keys the driver reads.
The reference arm (the CPU oracle) runs here; the GPU arm on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline",
        "e2e")


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    """--impl reference: the oracle on host cores, same config object as the
    GPU arm, a bounded sample described in cpu_baseline, e2e with no copies."""
    line = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0",
                 "--cpu-seconds", "1"])
    for k in KEYS:
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["workload"] == "c1" and line["config"]["nbins"] == 128
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_contract():
    """The default workload (c3), the roofline from the current sources' ncu
    counts (not stale), e2e through the host-buffer entry point, clocks."""
    line = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    for k in KEYS:
        assert k in line, k
    assert line["config"]["workload"] == "c3" and line["scaling"] == "strong"
    assert line["dtype"] == "f64" and line["gpu_launches"] == 2
    roof = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    assert roof["stale"] is False, "profiles/roofline_counts.json is not from the current sources"
    assert 0.2 < roof["frac"] < 1.0 and 0.2 < roof["fp64_issue"]["frac"] < 1.0
    assert 0.2 < roof["issue"]["frac"] < 1.0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 2 * 8 * (1 << 24)
    assert "sm_mhz" in line["clocks"]
