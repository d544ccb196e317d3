"""Seeded synthetic (v, x) workloads -- shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: it only draws inputs.  It
implements the five BASELINE.json configs (recipe in DESIGN.md §4):

  c1  10^4  FP64  v ~ U[0,10],          x ~ logU[1e-2, 1e2]   all 3 outputs
  c2  2^20  FP64  v ~ U[0,100],         x ~ logU[1e-1, 1e3]   all 3 outputs
  c3  2^24  FP64  v ~ logU[10,1000],    x ~ logU[1e-3, 1e1]   all 3 outputs
  c4  2^26  FP32  v ~ U[0,50],          x ~ logU[1e-2, 1e2]   all 3 outputs
  c5  2^28  FP64  v ~ {1,.5,2.5,5},     x = a*sqrt(d^2+y^2),  log K, dlogK/dx
                  a ~ logU[0.5,20], d ~ logU[0.1,5], y ~ N(0, 3^2)  (NIG batch)

"log-uniform in [a,b]" is x = 10**U(log10 a, log10 b).  Generation is in
fixed blocks of 2^20 elements; block b of config k is drawn from
numpy PCG64(SeedSequence(seed, spawn_key=(k, b))), arrays in the order v, x
(c5: v, a, d, y).  Element i of a config is therefore the same no matter
how the batch is sharded across ranks or sampled for the oracle, and of the
total size requested (blocks are always drawn at full length and sliced).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BLOCK = 1 << 20


@dataclass(frozen=True)
class Config:
    name: str
    index: int
    n: int
    precision: str          # "f64" | "f32"
    outputs: tuple          # subset of ("logk", "dv", "dx")
    describe: str


CONFIGS = {
    "c1": Config("c1", 1, 10_000, "f64", ("logk", "dv", "dx"),
                 "1e4 pairs FP64, v~U[0,10], x~logU[1e-2,1e2], seed 0"),
    "c2": Config("c2", 2, 1 << 20, "f64", ("logk", "dv", "dx"),
                 "2^20 pairs FP64, v~U[0,100], x~logU[1e-1,1e3]"),
    "c3": Config("c3", 3, 1 << 24, "f64", ("logk", "dv", "dx"),
                 "2^24 pairs FP64, v~logU[10,1000], x~logU[1e-3,1e1] (peaked)"),
    "c4": Config("c4", 4, 1 << 26, "f32", ("logk", "dv", "dx"),
                 "2^26 pairs FP32, v~U[0,50], x~logU[1e-2,1e2]"),
    "c5": Config("c5", 5, 1 << 28, "f64", ("logk", "dx"),
                 "2^28 pairs FP64 NIG batch, v~{1,.5,2.5,5}, x=a*sqrt(d^2+y^2)"),
    # the paper's own batch-size experiment (Sec. 3.4, Fig. 5):
    # v = 10^(2r) - 1 in [0, 99], x = 10^(3r - 1) in [0.1, 100], r ~ U(0,1)
    "fig5": Config("fig5", 6, 1 << 28, "f64", ("logk", "dv", "dx"),
                   "paper Fig. 5 distribution: v=10^(2r)-1, x=10^(3r-1), r~U(0,1)"),
}


def _logu(rng, lo, hi, n):
    return 10.0 ** rng.uniform(np.log10(lo), np.log10(hi), n)


def _block(cfg: Config, b: int, count: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(seed, spawn_key=(cfg.index, b))))
    k = cfg.name
    if k == "c1":
        v = rng.uniform(0.0, 10.0, count)
        x = _logu(rng, 1e-2, 1e2, count)
    elif k == "c2":
        v = rng.uniform(0.0, 100.0, count)
        x = _logu(rng, 1e-1, 1e3, count)
    elif k == "c3":
        v = _logu(rng, 10.0, 1000.0, count)
        x = _logu(rng, 1e-3, 1e1, count)
    elif k == "c4":
        v = rng.uniform(0.0, 50.0, count)
        x = _logu(rng, 1e-2, 1e2, count)
    elif k == "fig5":
        r = rng.uniform(0.0, 1.0, count)
        v = 10.0 ** (2.0 * r) - 1.0
        x = 10.0 ** (3.0 * r - 1.0)
    elif k == "c5":
        v = rng.choice(np.array([1.0, 0.5, 2.5, 5.0]), count)
        a = _logu(rng, 0.5, 20.0, count)
        d = _logu(rng, 0.1, 5.0, count)
        y = rng.normal(0.0, 3.0, count)
        x = a * np.sqrt(d * d + y * y)
    else:  # pragma: no cover
        raise KeyError(k)
    return v, x


def generate(name: str, start: int = 0, count: int | None = None, seed: int = 0,
             n: int | None = None):
    """Elements [start, start+count) of config ``name`` as numpy arrays.

    Returns float64 arrays for FP64 configs and float32 for c4.  ``n``
    overrides the config's total size (the block layout, hence element i,
    does not depend on it).
    """
    cfg = CONFIGS[name]
    total = cfg.n if n is None else int(n)
    if count is None:
        count = total - start
    if start < 0 or count < 0 or start + count > total:
        raise ValueError("range outside the config")
    vs, xs = [], []
    b0, b1 = start // BLOCK, (start + count + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        blk_len = min(BLOCK, total - b * BLOCK)
        v, x = _block(cfg, b, BLOCK, seed)
        lo = max(start, b * BLOCK) - b * BLOCK
        hi = min(start + count, b * BLOCK + blk_len) - b * BLOCK
        vs.append(v[lo:hi])
        xs.append(x[lo:hi])
    v = np.concatenate(vs) if vs else np.empty(0)
    x = np.concatenate(xs) if xs else np.empty(0)
    dt = np.float32 if cfg.precision == "f32" else np.float64
    return v.astype(dt), x.astype(dt)


def sample_indices(name: str, count: int, seed: int = 1, n: int | None = None):
    """Sorted, seeded sample of element indices (for oracle checks at full size)."""
    total = CONFIGS[name].n if n is None else int(n)
    count = min(count, total)
    rng = np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(seed, spawn_key=(CONFIGS[name].index, 1 << 30))))
    return np.sort(rng.choice(total, size=count, replace=False))


def gather(name: str, idx, seed: int = 0, n: int | None = None):
    """Inputs at arbitrary indices (block-wise, without generating everything)."""
    idx = np.asarray(idx, dtype=np.int64)
    cfg = CONFIGS[name]
    total = cfg.n if n is None else int(n)
    v = np.empty(idx.size)
    x = np.empty(idx.size)
    blocks = idx // BLOCK
    for b in np.unique(blocks):
        sel = np.nonzero(blocks == b)[0]
        vb, xb = _block(cfg, int(b), BLOCK, seed)
        v[sel] = vb[idx[sel] - b * BLOCK]
        x[sel] = xb[idx[sel] - b * BLOCK]
    dt = np.float32 if cfg.precision == "f32" else np.float64
    return v.astype(dt), x.astype(dt)
