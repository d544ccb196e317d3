"""The multi-GPU driver end to end on every GPU of the box (1 on the
development pool, 8 on a full node): torchrun, contiguous shards, NCCL
gather of sampled inputs/outputs, oracle check on rank 0 (tests/mgpu_driver.py)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("cfg,n", [("c3", 1 << 22), ("c2", 1 << 20), ("c5", 1 << 22), ("c4", 1 << 21)])
def test_sharded_driver(cfg, n):
    g = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1",
           f"--nproc-per-node={g}", os.path.join(HERE, "mgpu_driver.py"), cfg, str(n)]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", NCCL_DEBUG="INFO")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"MGPU OK cfg={cfg} n={n} world={g}" in r.stdout
