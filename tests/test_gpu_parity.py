"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle,
element by element on the same seeded inputs (BASELINE.json configs c1-c5),
plus edge cases, invariances and full-size sampled checks in the launch
configuration bench.py times."""
import numpy as np
import pytest
import torch

import oracle
import paper_2108_11560_b200 as blk
import workloads
from parity import assert_parity, max_errors

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
NB = 128
KINDS = ("logk", "dv", "dx")


def run_gpu(v, x, nbins=NB, outputs=KINDS, **kw):
    dt = torch.float32 if v.dtype == np.float32 else torch.float64
    vt = torch.from_numpy(np.ascontiguousarray(v)).to(DEV, dt)
    xt = torch.from_numpy(np.ascontiguousarray(x)).to(DEV, dt)
    res = blk.log_bessel_k(vt, xt, nbins=nbins, outputs=outputs, **kw)
    torch.cuda.synchronize()
    return {k: r.cpu().numpy() for k, r in zip(outputs, res)}


def run_oracle(v, x, nbins=NB, threads=8):
    r = oracle.logk(np.asarray(v, np.float64), np.asarray(x, np.float64), nbins, threads=threads)
    return dict(zip(KINDS, r))


# --------------------------------------------------------------- per config
MID_N = 3 * 8192 + 77   # many blocks of 128 threads and a ragged tail


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_parity_config(cfg):
    c = workloads.CONFIGS[cfg]
    n = min(c.n, MID_N)
    v, x = workloads.generate(cfg, 0, n)
    outs = c.outputs
    got = run_gpu(v, x, outputs=outs)
    ref = run_oracle(v, x)
    assert_parity(got, ref, c.precision, cfg)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_parity_config_f64_range(cfg):
    """range_mode=BLK_RANGE_F64: the paper's working-precision range finder."""
    c = workloads.CONFIGS[cfg]
    v, x = workloads.generate(cfg, 0, 4099)
    got = run_gpu(v, x, outputs=c.outputs, range_mode=blk.BLK_RANGE_F64)
    assert_parity(got, run_oracle(v, x), c.precision, cfg)


@pytest.mark.parametrize("lanes", [1, 2, 4, 8, 16, 32])
def test_parity_lanes_per_element(lanes):
    """K3: bins split across lanes + shuffle reduction, same tolerance."""
    v, x = workloads.generate("c2", 0, 3001)
    got = run_gpu(v, x, lanes_per_element=lanes)
    assert_parity(got, run_oracle(v, x), "f64", f"lanes={lanes}")
    got32 = run_gpu(v.astype(np.float32), x.astype(np.float32), lanes_per_element=lanes)
    assert_parity(got32, run_oracle(v.astype(np.float32), x.astype(np.float32)), "f32",
                  f"f32 lanes={lanes}")


NBINS_ALL = [2, 3, 8, 16, 17, 32, 47, 48, 56, 63, 64, 96, 127, 256, 1000]
# BLK_RANGE_AUTO's switch to the FP32 range finder (logk_range.cuh kF32PlanMinBins)
F32_PLAN_MIN_BINS = 48


def gpu_plan(v, x, nbins, range_mode=0):
    """(t_p, g(t_p), t0, t1) per element as the FP64 entry point finds it
    (bessel_logk_plan_f64), as an (n, 4) array."""
    vt = torch.from_numpy(np.ascontiguousarray(v, np.float64)).to(DEV)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(DEV)
    res = blk.bessel_logk_plan_f64(vt, xt, nbins=nbins, range_mode=range_mode)
    torch.cuda.synchronize()
    return np.stack([r.cpu().numpy() for r in res], axis=1)


def check_on_plan(got, v, x, nbins, ctx, range_mode=0, pin=60, tol_d=None):
    """Several plans are correct (R20): the result of Eq. (int) is unique only
    given the range.  So: (1) the kernel's outputs equal the oracle's
    quadrature on the kernel's own plan, element by element, at the FP64
    tolerance; (2) where the kernel's plan equals the oracle's (to 1e-12) they
    equal the oracle's outputs too (the same range ends, the same shift to
    1e-14); (3) the kernel's plan is valid -- for the
    FP64 range finder the pin of the oracle's plan (outer side of the exact
    30-digit roots, within the 10-iteration bracket bound), for the FP32 one
    its stopping rule plus FP32 resolution (plan_pins.plan_check_f32) -- on
    the elements whose plan differs from the oracle's and a seeded sample.
    Returns the fraction of elements whose plan differs."""
    from parity import errors
    from plan_pins import mp_plan, plan_check_f32, plan_violations
    plan = gpu_plan(v, x, nbins, range_mode)
    ref = dict(zip(KINDS, oracle.quad_on_plan(v, x, plan[:, 1], plan[:, 2], plan[:, 3], nbins,
                                              threads=8)))
    if tol_d is None:
        assert_parity(got, ref, "f64", ctx + " (oracle quadrature on the kernel's plan)")
    else:
        assert np.array_equal(np.isnan(got["logk"]), np.isnan(ref["logk"]))
        ok = ~np.isnan(ref["logk"])
        assert errors(got["logk"][ok], ref["logk"][ok], "logk").max() <= 1e-12, ctx
        for k in ("dv", "dx"):
            assert np.all(errors(got[k][ok], ref[k][ok], k) <= tol_d[ok]), (ctx, k)
    lk, dv, dx, oplan = oracle.logk(v, x, nbins, with_plan=True, threads=8)
    fin = np.isfinite(oplan).all(axis=1) & np.isfinite(plan).all(axis=1)
    same = (fin & (plan[:, 2] == oplan[:, 2]) & (plan[:, 3] == oplan[:, 3])
            & (np.abs(plan[:, 1] - oplan[:, 1]) <= 1e-14 * np.maximum(1, np.abs(oplan[:, 1]))))
    if tol_d is None:
        assert_parity({k: g[same] for k, g in got.items()},
                      {k: r[same] for k, r in zip(KINDS, (lk, dv, dx))}, "f64", ctx + " (same plan)")
    diff = np.nonzero(fin & ~same)[0]
    rng = np.random.default_rng(nbins)
    idx = np.unique(np.concatenate([diff[:pin], rng.choice(np.nonzero(fin)[0], min(pin, fin.sum()),
                                                           replace=False)]))
    exact = [mp_plan(v[i], x[i]) for i in idx]
    f32 = range_mode == 0 and nbins >= F32_PLAN_MIN_BINS
    if f32:   # the FP32 finder's tolerances (logk_range.cuh fz_tol_for)
        end_nats, peak_gap = (8.0, 4.0) if nbins >= 128 else (0.1, 1.0 / 64)
        bad = plan_check_f32(np.abs(v[idx]), x[idx], plan[idx], exact, end_nats, peak_gap)
    else:
        bad = plan_violations(np.abs(v[idx]), x[idx], plan[idx], exact)
    assert not bad.any(), (ctx, idx[bad][:5], v[idx][bad][:3], x[idx][bad][:3], plan[idx][bad][:2])
    return diff.size / max(1, fin.sum())


@pytest.mark.parametrize("nbins", NBINS_ALL)
def test_parity_nbins(nbins):
    """Every bin count, coarse ones included, in the default (AUTO) mode.
    From 48 bins the trapezoid error is at rounding level and any
    conservative range gives the oracle's values: element-by-element parity
    at the north_star tolerance.  Coarser grids' discretisation error depends
    on where the nodes fall, i.e. on the range, and the paper's 10-iteration
    FindZero is not always converged (the oracle's t0 moves by up to 5e-3
    between 10 and 30 iterations, test_oracle_pins), so a rounding-level tie
    in one sign test (F(t_newton) < 0) can pick another, equally valid,
    range (measured: ~12% of c1's elements end up with t_p or t1 ~1e-9
    apart, where Newton lands on the root to rounding and F(t_newton) is
    +-0): there AUTO runs the FP64 range finder and check_on_plan compares
    what is unique (Eq. (int) on the kernel's range) and checks the range."""
    v, x = workloads.generate("c1", 0, 1500)
    got = run_gpu(v, x, nbins=nbins)
    if nbins >= F32_PLAN_MIN_BINS:
        assert_parity(got, run_oracle(v, x, nbins=nbins), "f64", f"nbins={nbins}")
    frac = check_on_plan(got, v, x, nbins, f"nbins={nbins}")
    print(f"nbins={nbins}: plans differing from the oracle's on {frac:.2%} of elements")


def run_oracle_f32(v, x, nbins=NB):
    """The FP32 entry point's method is Alg. 1-3 with eps = 2^-23 (R9): the
    oracle in double on the float inputs widened exactly, log eps = log 2^-23."""
    r = oracle.logk(np.asarray(v, np.float64), np.asarray(x, np.float64), nbins,
                    log_eps=oracle.log_eps_f32(), threads=8)
    return dict(zip(KINDS, r))


@pytest.mark.parametrize("nbins", NBINS_ALL)
def test_parity_nbins_f32(nbins):
    """The FP32 entry point at every bin count against the oracle run with the
    FP32 threshold eps = 2^-23, at the FP32 north_star tolerance."""
    v, x = workloads.generate("c4", 0, 1500)
    got = run_gpu(v, x, nbins=nbins)
    assert_parity(got, run_oracle_f32(v, x, nbins), "f32", f"f32 nbins={nbins}")
    if nbins >= 64:   # converged: the eps = 2^-52 oracle agrees as well
        assert_parity(got, run_oracle(v, x, nbins), "f32", f"f32 nbins={nbins} (eps 2^-52)")


@pytest.mark.parametrize("nbins", [2, 3, 16, 33, 128])
@pytest.mark.parametrize("lanes", [8, 32])
def test_empty_lanes(nbins, lanes):
    """lanes_per_element larger than the nodes per lane allow leaves lanes with
    no node (n + 1 < lanes x ceil((n + 1)/lanes)); they must not take back the
    end node's half weight (found by review: at nbins = 2, 32 lanes, 30 lanes
    did).  North_star tolerance, FP64 and FP32."""
    v, x = workloads.generate("c1", 0, 700)
    got = run_gpu(v, x, nbins=nbins, lanes_per_element=lanes)
    check_on_plan(got, v, x, nbins, f"nbins={nbins} lanes={lanes}", pin=20)
    v4, x4 = workloads.generate("c4", 0, 700)
    got4 = run_gpu(v4, x4, nbins=nbins, lanes_per_element=lanes)
    assert_parity(got4, run_oracle_f32(v4, x4, nbins), "f32", f"f32 nbins={nbins} lanes={lanes}")


def test_max_nbins():
    v, x = workloads.generate("c3", 0, 300)
    got = run_gpu(v, x, nbins=65536)
    ref = run_oracle(v, x, nbins=65536)
    assert_parity(got, ref, "f64", "nbins=65536")


# ------------------------------------------------------------------ edges
@pytest.mark.parametrize("kernel", [0, 1])
def test_empty_and_tiny_batches(kernel):
    for n in (0, 1, 2, 31, 32, 33, 127, 129, 4097):
        v, x = workloads.generate("c2", 5, n)
        got = run_gpu(v, x, kernel=kernel)
        if n:
            assert_parity(got, run_oracle(v, x), "f64", f"n={n}")
        else:
            assert all(g.size == 0 for g in got.values())


def test_special_values():
    v = np.array([0.0, -0.0, 0.5, -0.5, -3.7, 2.5, 1.0, 1.0, 1.0, np.nan, np.inf, 1.0, 1.0, 0.1])
    x = np.array([1.0, 2.0, 1.0, 1.0, 0.3, 3.0, 0.0, -1.0, np.nan, 1.0, 1.0, np.inf, 1e-3, 0.01])
    got = run_gpu(v, x)
    ref = run_oracle(v, x)
    assert_parity(got, ref, "f64", "special")
    assert got["dv"][0] == 0.0 and got["dv"][1] == 0.0
    # exact closed form at v=1/2 (DLMF 10.39.2)
    assert abs(got["logk"][2] - (0.5 * np.log(np.pi / 2) - 1)) < 1e-13
    assert abs(got["dx"][2] + 1.5) < 1e-13
    # odd/even in v
    assert got["logk"][2] == got["logk"][3] and got["dv"][2] == -got["dv"][3]


@pytest.mark.parametrize("kernel", [0, 1])
def test_extreme_domain(kernel):
    """Beyond the paper's grid (R22), incl. the FP64 range-finder fallback domain.

    The exponent g(t) - g(t_p) is a difference of terms as large as x cosh t
    and v t, so in double both the oracle and the kernel carry an absolute
    error ~eps * (x + v t_p) in every weight (tolerance note).
    For the five configs that is < 3e-12 and the north_star tolerances apply
    unchanged; beyond them kappa = eps (x + v t_p + 40) is the floor of any
    double evaluation -- at x = 1e8 the oracle's dv is 1.4e-9 from the exact
    value, and test_oracle_pins.py::test_large_x_dv_vs_brute_force pins it
    within 0.5 kappa of the long-double brute force -- so the derivative
    tolerance here is max(1e-10, 5 kappa).  Measured against the oracle: <= 0.05
    kappa here, <= 1.96 kappa on the wide-domain fuzz (profiles/r02zh_kappa.log)."""
    v = np.array([0, 0, 5, 0, 10, 2000, 5000, 1e4, 0.5, 5, 0, 30.0, 2e4, 3.0])
    x = np.array([1e3, 1e4, 1e5, 1e6, 1e8, 1e-3, 1e-4, 1e-2, 1e-6, 1e-10, 1e-8, 1e-30, 1.0, 1e-40])
    got = run_gpu(v, x, kernel=kernel)
    lk, dv, dx, plan = oracle.logk(v, x, NB, with_plan=True)
    kappa = np.finfo(float).eps * (x + v * plan[:, 0] + 40.0)
    tol_d = np.maximum(1e-10, 5 * kappa)
    from parity import errors
    assert np.all(errors(got["logk"], lk, "logk") <= 1e-12)
    assert np.all(errors(got["dx"], dx, "dx") <= tol_d)
    assert np.all(errors(got["dv"], dv, "dv") <= tol_d)
    _report_kappa("extreme", got, dv, dx, kappa)


def _report_kappa(ctx, got, dv, dx, kappa):
    """Print the derivative errors against the bound max(1e-10, 5 kappa): in
    units of kappa where the kappa term is the larger one, as relative errors
    elsewhere (evidence for the bound)."""
    from parity import errors
    ok = np.isfinite(dv) & np.isfinite(dx) & (dv != 0)
    big = ok & (5 * kappa > 1e-10)
    small = ok & ~big
    out = []
    for k, r in (("dv", dv), ("dx", dx)):
        e = errors(got[k], r, k)
        kb = (e[big] / kappa[big]).max() if big.any() else 0.0
        sr = e[small].max() if small.any() else 0.0
        out.append(f"{k}: {kb:.3f} kappa where 5 kappa > 1e-10 ({big.sum()}), {sr:.1e} rel. elsewhere")
    print(f"{ctx}: " + "; ".join(out))


def test_large_x_dv_vs_brute_force_gpu():
    """d log K/dv for x in [1e5, 1e8] (the inputs of test_oracle_pins::
    test_large_x_dv_vs_brute_force): the exponent's own rounding kappa =
    eps (x + v t_p + 40) is the floor of any double evaluation there (the
    oracle sits within 0.5 kappa of the long-double brute force).  The kernel
    is held to 2 kappa against the brute force and 2.5 kappa against the
    oracle; log K and dx to the north_star tolerances."""
    rng = np.random.default_rng(3)
    n = 300
    x = 10 ** rng.uniform(5, 8, n)
    v = np.where(rng.random(n) < 0.5, rng.uniform(0, 30, n), 10 ** rng.uniform(-3, 3.5, n))
    got = run_gpu(v, x)
    lk, dv, dx, plan = oracle.logk(v, x, NB, with_plan=True)
    b = oracle.brute(v, x, threads=8)
    kappa = np.finfo(float).eps * (x + v * plan[:, 0] + 40.0)
    rb = np.abs(got["dv"] - b[1]) / (kappa * np.abs(b[1]))
    ro = np.abs(got["dv"] - dv) / (kappa * np.abs(dv))
    print(f"large-x dv: max {rb.max():.3f} kappa vs brute, {ro.max():.3f} kappa vs oracle")
    assert rb.max() <= 2.0 and ro.max() <= 2.5, (rb.max(), ro.max())
    assert_parity({"logk": got["logk"], "dx": got["dx"]}, {"logk": lk, "dx": dx}, "f64", "large x")


def test_misaligned_pointers():
    """torch storage offsets can leave 8-B (not 16-B) alignment."""
    v, x = workloads.generate("c2", 0, 1001)
    vt = torch.from_numpy(v).to(DEV)
    xt = torch.from_numpy(x).to(DEV)
    base = torch.empty(3 * 1001 + 3, dtype=torch.float64, device=DEV)
    out = [base[1:1002], base[1002:2003], base[2003:3004]]
    blk.bessel_logk_f64(vt[1:], xt[1:], out[0][1:], out[1][1:], out[2][1:], nbins=NB)
    torch.cuda.synchronize()
    got = {k: o[1:].cpu().numpy() for k, o in zip(KINDS, out)}
    assert_parity(got, run_oracle(v[1:], x[1:]), "f64", "misaligned")


# ------------------------------------------------------------ invariances
def test_bitwise_determinism_and_output_subsets():
    v, x = workloads.generate("c2", 0, 5000)
    a = run_gpu(v, x)
    b = run_gpu(v, x)
    for k in KINDS:
        assert np.array_equal(a[k], b[k])
    for subset in (("logk",), ("dv",), ("dx",), ("logk", "dx"), ("dv", "dx")):
        s = run_gpu(v, x, outputs=subset)
        for k in subset:
            assert np.array_equal(s[k], a[k]), (subset, k)


def test_permutation_and_shard_invariance():
    v, x = workloads.generate("c3", 0, 4096)
    a = run_gpu(v, x, lanes_per_element=1)
    perm = np.random.default_rng(0).permutation(v.size)
    b = run_gpu(v[perm], x[perm], lanes_per_element=1)
    for k in KINDS:
        assert np.array_equal(a[k][perm], b[k])
    for p in (2, 4, 8):
        bounds = np.linspace(0, v.size, p + 1).astype(int)
        parts = [run_gpu(v[lo:hi], x[lo:hi], lanes_per_element=1) for lo, hi in zip(bounds[:-1], bounds[1:])]
        for k in KINDS:
            assert np.array_equal(np.concatenate([q[k] for q in parts]), a[k])


def _host_buffers(a, dtype, transport):
    """CPU tensors for the host entry point: pinned (zero-copy transport),
    pageable (staged), or pinned inputs with pageable outputs (staged)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.pin_memory() if transport in ("zero_copy", "forced_staged") else t


@pytest.mark.parametrize("transport", ["zero_copy", "staged_pageable", "staged_mixed", "forced_staged"])
def test_host_entry_point_matches_device_path(transport, monkeypatch):
    """Both transports of bessel_logk_f64_host (zero-copy for mapped pinned
    buffers, staged chunks otherwise) equal the device path bit for bit, with
    a ragged last chunk; one output NULL on the zero-copy transport too."""
    if transport == "forced_staged":
        monkeypatch.setenv("BLK_HOST_PIPELINE", "1")
    v, x = workloads.generate("c2", 0, 70001)
    dev = run_gpu(v, x, lanes_per_element=1)
    vt = _host_buffers(v, torch.float64, "zero_copy" if transport == "staged_mixed" else transport)
    xt = _host_buffers(x, torch.float64, "zero_copy" if transport == "staged_mixed" else transport)
    outs = [_host_buffers(np.full(v.size, np.nan), torch.float64, transport) for _ in range(3)]
    chunk = 16384
    ws = torch.empty(blk.host_workspace_bytes(chunk), dtype=torch.uint8, device=DEV)
    blk.bessel_logk_f64_host(vt, xt, *outs, nbins=NB, workspace=ws, chunk=chunk)
    for k, o in zip(KINDS, outs):
        assert np.array_equal(o.numpy(), dev[k]), k
    # dlogk_dv NULL: the other two outputs unchanged, nothing written for dv
    outs2 = [_host_buffers(np.full(v.size, np.nan), torch.float64, transport) for _ in range(3)]
    blk.bessel_logk_f64_host(vt, xt, outs2[0], None, outs2[2], nbins=NB, workspace=ws, chunk=chunk)
    assert np.array_equal(outs2[0].numpy(), dev["logk"])
    assert np.array_equal(outs2[2].numpy(), dev["dx"])
    assert np.all(np.isnan(outs2[1].numpy()))


@pytest.mark.parametrize("transport", ["zero_copy", "staged_pageable"])
def test_host_entry_point_f32_matches_device_path(transport):
    v, x = workloads.generate("c4", 0, 50003)
    dev = run_gpu(v, x, lanes_per_element=1)
    vt = _host_buffers(v, torch.float32, transport)
    xt = _host_buffers(x, torch.float32, transport)
    outs = [_host_buffers(np.zeros(v.size, np.float32), torch.float32, transport) for _ in range(3)]
    chunk = 8192
    ws = torch.empty(blk.host_workspace_bytes(chunk, 4), dtype=torch.uint8, device=DEV)
    blk.bessel_logk_f32_host(vt, xt, *outs, nbins=NB, workspace=ws, chunk=chunk)
    for k, o in zip(KINDS, outs):
        assert np.array_equal(o.numpy(), dev[k]), k


def test_mathematical_properties_gpu():
    """Symmetry, recurrence and Eq. (deriv) hold on the GPU outputs directly."""
    rng = np.random.default_rng(2)
    v = rng.uniform(1.0, 60.0, 3000)
    x = 10 ** rng.uniform(-2, 2.5, 3000)
    lm = run_gpu(v - 1, x)["logk"]
    a = run_gpu(v, x)
    lp = run_gpu(v + 1, x)["logk"]
    rec_l = np.exp(lp - a["logk"])
    rec_r = np.exp(lm - a["logk"]) + 2 * v / x
    assert np.max(np.abs(rec_l - rec_r) / rec_r) < 1e-11
    ref_dx = -(np.exp(lm - a["logk"]) + np.exp(lp - a["logk"])) / 2
    assert np.max(np.abs(a["dx"] - ref_dx) / np.abs(ref_dx)) < 1e-11
    neg = run_gpu(-v, x)
    assert np.array_equal(neg["logk"], a["logk"]) and np.array_equal(neg["dv"], -a["dv"])


# ----------------------------------------------- full sizes, bench launch cfg
def _full_check(cfg, n_sample=2048, edge=512, chunked=False):
    c = workloads.CONFIGS[cfg]
    n = c.n
    dt = torch.float32 if c.precision == "f32" else torch.float64
    vt = torch.empty(n, dtype=dt, device=DEV)
    xt = torch.empty(n, dtype=dt, device=DEV)
    step = 1 << 24
    for s in range(0, n, step):
        v, x = workloads.generate(cfg, s, min(step, n - s))
        vt[s:s + v.size] = torch.from_numpy(v).to(DEV)
        xt[s:s + v.size] = torch.from_numpy(x).to(DEV)
    res = blk.log_bessel_k(vt, xt, nbins=NB, outputs=c.outputs)
    torch.cuda.synchronize()
    idx = np.unique(np.concatenate([workloads.sample_indices(cfg, n_sample, seed=11),
                                    np.arange(edge), np.arange(n - edge, n)]))
    it = torch.from_numpy(idx).to(DEV)
    got = {k: r[it].cpu().numpy() for k, r in zip(c.outputs, res)}
    vs, xs = workloads.gather(cfg, idx)
    ref = run_oracle(vs, xs)
    assert_parity(got, ref, c.precision, f"{cfg} full")
    # properties at every element: finite, dlogK/dx <= -1, dlogK/dv >= 0 (v >= 0)
    for k, r in zip(c.outputs, res):
        assert bool(torch.isfinite(r).all()), k
        if k == "dx":
            assert float(r.max()) <= -1.0 + (1e-5 if dt == torch.float32 else 1e-12)
        if k == "dv":
            assert float(r.min()) >= 0.0


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_full_size_sampled(cfg):
    _full_check(cfg)


def test_full_size_c5_sampled():
    _full_check("c5", n_sample=1024, edge=256)


def test_microbenchmarks_run():
    out = torch.empty(148 * 256, dtype=torch.float64, device=DEV)
    ops = blk.microbench("fp64", 148, 256, 10, out)
    out32 = torch.empty(148 * 256, dtype=torch.float32, device=DEV)
    blk.microbench("fp32", 148, 256, 10, out32)
    blk.microbench("mufu", 148, 256, 10, out32)
    torch.cuda.synchronize()
    assert ops == 148 * 256 * 10 * 16
    assert bool(torch.isfinite(out).all())


# --------------------------------------------- the paper's own experiments
def test_paper_accuracy_grid():
    """Sec. 3.1: on v = 0..99 x x = 10^-1..10^2.1 (100 x 33) the
    error metric log10(|Delta|/eps + 1) against the plain definition
    (long-double brute force) has no region >= 4 (the paper's cut for an
    inaccurate region) and a mean below 1 for log K and dx; FP32
    (eps = 2^-23) likewise ('less than 1 eps in most regions')."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "paper_experiments", os.path.join(os.path.dirname(__file__), "tools",
                                          "paper_experiments.py"))
    pe = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(pe)
    res = pe.accuracy_grid(128)
    for name in ("gpu_f64", "gpu_f32"):
        for k in ("logk", "dx", "dv"):
            assert res[name][k]["cells_ge_4"] == 0, (name, k, res[name][k])
        assert res[name]["logk"]["mean"] < 1.0, res[name]
        assert res[name]["dx"]["mean"] < 1.0, res[name]


# ------------------------------------------------ second derivatives (§8(f) 1)
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c5"])
@pytest.mark.parametrize("lanes", [1, 4])
def test_parity_hessian(cfg, lanes):
    """d2/dv2, d2/dx2, d2/dvdx in the same pass vs the oracle.  The outputs are
    differences of moments (S11/S0 - (S1/S0)^2 ...), so both sides lose
    |moment|/|result| in relative precision; the bound is 1e-10 of the result
    plus 1e-12 of the moment it is formed from (north_star's 1e-10 for the
    first derivatives)."""
    v, x = workloads.generate(cfg, 0, 6001)
    v = v.astype(np.float64)
    x = x.astype(np.float64)
    dev = torch.device("cuda")
    out = blk.log_bessel_k_hess(torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev),
                                lanes_per_element=lanes)
    torch.cuda.synchronize()
    got = [o.cpu().numpy() for o in out]
    lk, dv, dx, dvv, dxx, dvx = oracle.logk_hess(v, x, NB, threads=8)
    assert_parity({"logk": got[0], "dv": got[1], "dx": got[2]},
                  {"logk": lk, "dv": dv, "dx": dx}, "f64", f"hess {cfg}")
    for g, r, mom in ((got[3], dvv, np.abs(dvv) + dv * dv), (got[4], dxx, np.abs(dxx) + dx * dx),
                      (got[5], dvx, np.abs(dvx) + np.abs(dv * dx))):
        bad = np.abs(g - r) > 1e-10 * np.abs(r) + 1e-12 * mom
        assert not bad.any(), (np.nonzero(bad)[0][:5], g[bad][:3], r[bad][:3])
    # the Bessel ODE on the GPU outputs directly
    ode = 1 + v * v / (x * x) - got[2] / x - got[2] ** 2
    assert np.all(np.abs(got[4] - ode) <= 1e-11 * (np.abs(ode) + got[2] ** 2 + v * v / (x * x) + 1))


def test_loop_switch_small_order():
    """The FP64 quadrature takes the v2 loop (S1 from 2E - w) for v = 0 and
    v t1 >= 1e-3 and the general loop (additive p = 1 - q) below (DESIGN.md
    §5): both sides of the switch, incl. large x (short ranges, small t1),
    stay within the FP64 tolerance."""
    v = np.repeat([0.0, 1e-12, 1e-8, 9.99e-6, 1.0e-5, 1.01e-5, 1e-4, 1e-3, 1e-2], 7)
    x = np.tile([1e-2, 0.1, 1.0, 3.0, 10.0, 100.0, 1000.0], 9)
    for dt in (np.float64,):
        got = run_gpu(v.astype(dt), x.astype(dt))
        ref = run_oracle(v, x)
        assert_parity(got, ref, "f64", "small order")
        assert np.all(got["dv"][v == 0] == 0.0)
        # d/dv log K -> 0 like v: the relative error must not blow up as v -> 0
        nz = v > 0
        rel = np.abs(got["dv"][nz] - ref["dv"][nz]) / np.abs(ref["dv"][nz])
        assert rel.max() <= 1e-10


def test_f32_fixed_point_exponent_edges():
    """FP32 entry point: the fixed-point exponent path (dmin > -60) and its
    fallback give FP32-tolerance results across the whole c4 domain corner
    set, incl. tiny/huge x and v = 0."""
    v = np.repeat(np.array([0.0, 1e-6, 0.5, 5.0, 25.0, 50.0], np.float32), 6)
    x = np.tile(np.array([1e-2, 0.05, 1.0, 10.0, 60.0, 100.0], np.float32), 6)
    got = run_gpu(v, x)
    ref = run_oracle(v.astype(np.float64), x.astype(np.float64))
    assert_parity(got, ref, "f32", "f32 edges")
    assert np.all(got["dv"][v == 0] == 0.0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_wide_domain_fuzz(seed):
    """Seeded fuzz far beyond the five configs (R22): v in {0} U logU[1e-6, 2e4],
    x in logU[1e-12, 1e7], both range finders (FP32 for x in [1e-30, 1e4],
    v <= 1e4; FP64 otherwise) and both quadrature loops.  Tolerance as in
    test_extreme_domain: the north_star bounds, widened for the derivatives by
    the exponent's own rounding eps*(x + v t_p) that the oracle also carries."""
    rng = np.random.default_rng(seed)
    n = 20000
    v = 10.0 ** rng.uniform(-6, np.log10(2e4), n)
    v[rng.random(n) < 0.02] = 0.0
    v *= np.where(rng.random(n) < 0.1, -1.0, 1.0)
    x = 10.0 ** rng.uniform(-12, 7, n)
    got = run_gpu(v, x)
    lk, dv, dx, plan = oracle.logk(v, x, NB, with_plan=True, threads=8)
    from parity import errors
    kappa = np.finfo(float).eps * (x + np.abs(v) * plan[:, 0] + 40.0)
    tol_d = np.maximum(1e-10, 5 * kappa)
    assert np.array_equal(np.isnan(got["logk"]), np.isnan(lk))
    ok = ~np.isnan(lk)
    tol_l = np.maximum(1e-12, kappa[ok] / np.maximum(1.0, np.abs(lk[ok])))
    e0 = errors(got["logk"][ok], lk[ok], "logk")
    assert np.all(e0 <= tol_l), (e0.max(), v[ok][np.argmax(e0)], x[ok][np.argmax(e0)])
    e2 = errors(got["dx"][ok], dx[ok], "dx")
    assert np.all(e2 <= tol_d[ok]), (v[ok][np.argmax(e2 / tol_d[ok])], x[ok][np.argmax(e2 / tol_d[ok])])
    e1 = errors(got["dv"][ok], dv[ok], "dv")
    assert np.all(e1 <= tol_d[ok]), (v[ok][np.argmax(e1 / tol_d[ok])], x[ok][np.argmax(e1 / tol_d[ok])])
    assert np.all(got["dv"][v == 0] == 0.0)
    _report_kappa(f"wide fuzz {seed}", got, dv, dx, kappa)


@pytest.mark.parametrize("seed", [1, 2])
def test_wide_domain_fuzz_f32(seed):
    """FP32 entry point on a domain wider than config 4: v in {0} U U[0, 200],
    x in logU[1e-4, 1e3]; FP32 tolerances against the FP64 oracle on the
    widened float inputs."""
    rng = np.random.default_rng(100 + seed)
    n = 20000
    v = rng.uniform(0.0, 200.0, n).astype(np.float32)
    v[rng.random(n) < 0.02] = 0.0
    x = (10.0 ** rng.uniform(-4, 3, n)).astype(np.float32)
    got = run_gpu(v, x)
    ref = run_oracle(v.astype(np.float64), x.astype(np.float64))
    assert_parity(got, ref, "f32", "f32 fuzz")
    assert np.all(got["dv"][v == 0] == 0.0)


def test_f32_extreme_peaks():
    """FP32 entry point where the peak sits far out (t_p up to ~80) and g is
    sharply curved there (|g''| ~ 1e3-1e4): the peak search must bound the
    gap g(max) - g(t_p) (the log-sum-exp shift), not the position of t_p,
    or the fixed-point FP32 weights overflow (R4)."""
    v = np.array([1e4, 1e4, 5e3, 2e3, 1e4, 8e3, 300.0, 1e4], np.float32)
    x = np.array([1e-30, 1e-25, 1e-20, 1e-30, 1e-10, 1e-3, 1e-30, 1.0], np.float32)
    got = run_gpu(v, x)
    ref = run_oracle(v.astype(np.float64), x.astype(np.float64))
    assert_parity(got, ref, "f32", "f32 extreme peaks")


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_wide_domain_fuzz_f32_full(seed):
    """FP32 entry point over its whole range-finder domain and beyond:
    v in {0} U logU[1e-4, 2e4], x in logU[1e-36, 1e6] (the FP32 range finder
    for x in [1e-30, 1e4], v <= 1e4, the FP64 one elsewhere), FP32
    tolerances against the FP64 oracle on the widened float inputs."""
    rng = np.random.default_rng(200 + seed)
    n = 20000
    v = (10.0 ** rng.uniform(-4, np.log10(2e4), n)).astype(np.float32)
    v[rng.random(n) < 0.02] = 0.0
    x = (10.0 ** rng.uniform(-36, 6, n)).astype(np.float32)
    got = run_gpu(v, x)
    ref = run_oracle(v.astype(np.float64), x.astype(np.float64))
    # where the exact output is beyond FLT_MAX (d log K/dx ~ -cosh t_p for
    # t_p > 88.7), the FP32 result is the correctly signed infinity
    big = {k: np.abs(r) > np.finfo(np.float32).max for k, r in ref.items()}
    fmax = float(np.finfo(np.float32).max)
    for k in ref:
        g, r = got[k][big[k]].astype(np.float64), ref[k][big[k]]
        # +-inf, or FLT_MAX itself when the exact value is within rounding of it
        assert np.all((np.sign(g) == np.sign(r)) & (np.abs(g) >= fmax * (1 - 1e-4))), k
    keep = ~(big["logk"] | big["dv"] | big["dx"])
    assert keep.mean() > 0.95
    assert_parity({k: g[keep] for k, g in got.items()}, {k: r[keep] for k, r in ref.items()},
                  "f32", "f32 full-domain fuzz")


def test_f64_far_out_extremes():
    """FP64 ranges as far out as double allows: t_p up to ~700 (x down to
    1e-300, where e^t_p is near DBL_MAX), orders up to 1e6; x = 1e-305 puts
    t_p past 709, where the oracle's own cosh overflows and both sides must
    return NaN.  Tolerances as in test_extreme_domain."""
    v = np.array([1e4, 1e4, 1.0, 100.0, 1e4, 1e6, 1e5, 2.5, 0.0])
    x = np.array([1e-305, 1e-300, 1e-300, 1e-250, 1e-200, 1.0, 1e-10, 1e-280, 1e-300])
    got = run_gpu(v, x)
    lk, dv, dx, plan = oracle.logk(v, x, NB, with_plan=True)
    from parity import errors
    for g, r in ((got["logk"], lk), (got["dv"], dv), (got["dx"], dx)):
        assert np.array_equal(np.isnan(g), np.isnan(r))
    ok = ~np.isnan(lk)
    kappa = np.finfo(float).eps * (x + v * np.nan_to_num(plan[:, 0]) + 40.0)
    tol_d = np.maximum(1e-10, 5 * kappa)
    assert np.all(errors(got["logk"][ok], lk[ok], "logk") <= 1e-12)
    assert np.all(errors(got["dx"][ok], dx[ok], "dx") <= tol_d[ok])
    assert np.all(errors(got["dv"][ok], dv[ok], "dv") <= tol_d[ok])


def test_ranges_past_double_overflow_are_nan():
    """R23: an eps-support that reaches t = 709 (e^t overflows double at 709.78,
    cosh t at 710.48 -- x near or below DBL_MIN for small orders, where the
    integrand is still O(1) there) has no result in double, on the GPU as in
    the oracle: NaN on both sides, at every bin count and in both range modes;
    x = 1e-300 (ranges ending at ~695) stays finite and in parity."""
    xs = [5e-324, 1e-320, 1e-310, 2.2e-308, 1e-306, 1e-303, 1e-300]
    vs = [0.0, 0.5, 1.0, 3.0]
    v = np.array([a for a in vs for _ in xs])
    x = np.array([b for _ in vs for b in xs])
    for nb in (3, 48, 128):
        for mode in (blk.BLK_RANGE_AUTO, blk.BLK_RANGE_F64):
            got = run_gpu(v, x, nbins=nb, range_mode=mode)
            lk, dv, dx, plan = oracle.logk(v, x, nb, with_plan=True)
            for k, r in zip(KINDS, (lk, dv, dx)):
                assert np.array_equal(np.isnan(got[k]), np.isnan(r)), (nb, mode, k)
            fin = ~np.isnan(lk)
            assert np.all(plan[fin, 3] < 709.0) and fin[x == 1e-300].all()
            if nb >= F32_PLAN_MIN_BINS:
                assert_parity({k: g[fin] for k, g in got.items()},
                              {k: r[fin] for k, r in zip(KINDS, (lk, dv, dx))}, "f64",
                              f"nbins={nb} mode={mode}")


def test_hessian_wide_fuzz():
    """Second derivatives beyond the configs: v in {0} U logU[1e-3, 1e3], x in
    logU[1e-6, 1e4]; bound as in test_parity_hessian, widened by the
    exponent's own rounding eps*(x + v t_p) that both sides carry."""
    rng = np.random.default_rng(7)
    n = 6000
    v = 10.0 ** rng.uniform(-3, 3, n)
    v[rng.random(n) < 0.03] = 0.0
    x = 10.0 ** rng.uniform(-6, 4, n)
    dev = torch.device("cuda")
    out = blk.log_bessel_k_hess(torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev))
    torch.cuda.synchronize()
    got = [o.cpu().numpy() for o in out]
    lk, dv, dx, dvv, dxx, dvx = oracle.logk_hess(v, x, NB, threads=8)
    _, _, _, plan = oracle.logk(v, x, NB, with_plan=True, threads=8)
    kap = np.maximum(1.0, 10 * np.finfo(float).eps * (x + v * plan[:, 0] + 40.0) / 1e-10)
    for g, r, mom in ((got[3], dvv, np.abs(dvv) + dv * dv), (got[4], dxx, np.abs(dxx) + dx * dx),
                      (got[5], dvx, np.abs(dvx) + np.abs(dv * dx))):
        bad = np.abs(g - r) > kap * (1e-10 * np.abs(r) + 1e-12 * mom)
        assert not bad.any(), (v[bad][:4], x[bad][:4], g[bad][:3], r[bad][:3])


def _wide_inputs(seed, n=6000):
    rng = np.random.default_rng(seed)
    v = 10.0 ** rng.uniform(-6, 4, n)
    v[rng.random(n) < 0.02] = 0.0
    x = 10.0 ** rng.uniform(-12, 6, n)
    return v, x


def _wide_tol_d(v, x, nbins):
    _, _, _, plan = oracle.logk(v, x, nbins, with_plan=True, threads=8)
    kappa = np.finfo(float).eps * (x + np.abs(v) * np.nan_to_num(plan[:, 0]) + 40.0)
    return np.maximum(1e-10, 5 * kappa)


def _assert_wide(got, v, x, nbins):
    lk, dv, dx, plan = oracle.logk(v, x, nbins, with_plan=True, threads=8)
    from parity import errors
    kappa = np.finfo(float).eps * (x + np.abs(v) * plan[:, 0] + 40.0)
    tol_d = np.maximum(1e-10, 5 * kappa)
    ok = ~np.isnan(lk)
    assert np.array_equal(np.isnan(got["logk"]), ~ok)
    assert errors(got["logk"][ok], lk[ok], "logk").max() <= 1e-12
    assert np.all(errors(got["dx"][ok], dx[ok], "dx") <= tol_d[ok])
    assert np.all(errors(got["dv"][ok], dv[ok], "dv") <= tol_d[ok])


@pytest.mark.parametrize("lanes,kernel,nbins", [(2, 0, 128), (8, 0, 128), (32, 0, 200), (1, 1, 128),
                                                (4, 0, 160), (1, 0, 2048)])
def test_wide_domain_fuzz_variants(lanes, kernel, nbins):
    """The wide-domain FP64 fuzz through the other launch variants (lanes per
    element, other converged bin counts)."""
    v, x = _wide_inputs(lanes * 1000 + kernel * 10 + nbins)
    _assert_wide(run_gpu(v, x, nbins=nbins, lanes_per_element=lanes, kernel=kernel), v, x, nbins)


@pytest.mark.parametrize("lanes,nbins", [(1, 48), (8, 56), (1, 64), (4, 96), (1, 127)])
def test_wide_domain_auto_48_127(lanes, nbins):
    """AUTO at 48-127 bins (the FP32 range finder, 0.1-nat tolerance tier) on
    the wide domain: small v with tiny x puts t_p ~ 25 with ranges ~30 wide,
    where 48-127 nodes still leave a discretisation error that depends on the
    range, so the outputs are checked on the kernel's own (valid) plan."""
    v, x = _wide_inputs(5151 + nbins)
    got = run_gpu(v, x, nbins=nbins, lanes_per_element=lanes)
    frac = check_on_plan(got, v, x, nbins, f"wide auto nbins={nbins}", tol_d=_wide_tol_d(v, x, nbins))
    print(f"wide auto nbins={nbins}: plans differing on {frac:.2%}")


@pytest.mark.parametrize("lanes,nbins", [(8, 64), (4, 33), (1, 48), (1, 8), (2, 2)])
def test_wide_domain_coarse_bins_f64_range(lanes, nbins):
    """Coarse grids on the wide domain with the FP64 range finder (the
    paper's working precision, BLK_RANGE_F64; AUTO below 64 bins): the
    outputs on the kernel's own plan, and that plan's validity, as in
    test_parity_nbins."""
    v, x = _wide_inputs(4242 + nbins)
    got = run_gpu(v, x, nbins=nbins, lanes_per_element=lanes, range_mode=blk.BLK_RANGE_F64)
    frac = check_on_plan(got, v, x, nbins, f"wide f64 nbins={nbins}", range_mode=blk.BLK_RANGE_F64,
                         tol_d=_wide_tol_d(v, x, nbins))
    print(f"wide f64-range nbins={nbins}: plans differing on {frac:.2%}")


def test_cuda_graph_capture():
    """The device entry points only enqueue (no allocation, no sync), so they
    can be captured in a CUDA graph and replayed; results equal a direct call."""
    v, x = workloads.generate("c2", 0, 20000)
    vt = torch.from_numpy(v).to(DEV)
    xt = torch.from_numpy(x).to(DEV)
    outs = [torch.empty_like(vt) for _ in range(3)]
    ref = [torch.empty_like(vt) for _ in range(3)]
    blk.bessel_logk_f64(vt, xt, *ref, nbins=NB, lanes_per_element=1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        blk.bessel_logk_f64(vt, xt, *outs, nbins=NB, lanes_per_element=1, stream=s)  # warm-up
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        blk.bessel_logk_f64(vt, xt, *outs, nbins=NB, lanes_per_element=1,
                            stream=torch.cuda.current_stream())
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("lanes", [1, 2, 0])
def test_large_order_cancellation(lanes):
    """log K where x cosh t ~ 1e4 cancels against v t (found by the wide-domain
    fuzz at v = 18140, x = 12025): the v2 loop steps the cosh factors with
    accurate e^{+-h} - 1 (fma(X, u, X)) instead of a rounded e^{+-h}, whose
    rounding drifted the exponent by (n/G) ulp of x cosh t -- 2.2e-11 at one
    lane per element, 7x the floor eps (x + v t_p); the build before that
    change fails this test at lanes 1 and 2."""
    from parity import cancellation_band
    v, x = cancellation_band(256, 7)
    got = run_gpu(v, x, lanes_per_element=lanes)
    lk, dv, dx, plan = oracle.logk(v, x, NB, with_plan=True, threads=8)
    from parity import errors
    assert np.all(np.abs(lk) <= 25.0)
    # kappa = eps (x + v t_p), one rounding of the exponent's ~1e4 terms, is
    # the floor of any double evaluation (DESIGN.md §3 tolerance note).  The
    # oracle's independent per-node roundings average to <= 0.45 kappa
    # (test_oracle_pins); the kernel's B_c = v t_c - s and start state are
    # shared by a group / a lane, and a peak this narrow spans ~2 groups, so
    # they average less: log K is held to 2 kappa against the long-double
    # brute force and 2.5 kappa against the oracle.
    kappa = np.finfo(float).eps * (x + v * plan[:, 0] + 40.0)
    tol_l = np.maximum(1e-12, kappa / np.maximum(1.0, np.abs(lk)))
    lk_b = oracle.brute(v, x, threads=8)[0]
    eb = errors(got["logk"], lk_b, "logk")
    assert np.all(eb <= 2 * tol_l), ((eb / tol_l).max(), v[np.argmax(eb / tol_l)], x[np.argmax(eb / tol_l)])
    e0 = errors(got["logk"], lk, "logk")
    assert np.all(e0 <= 2.5 * tol_l), ((e0 / tol_l).max(), v[np.argmax(e0 / tol_l)])
    tol_d = np.maximum(1e-10, 5 * kappa)
    assert np.all(errors(got["dv"], dv, "dv") <= tol_d)
    assert np.all(errors(got["dx"], dx, "dx") <= tol_d)


@pytest.mark.parametrize("seed", [1, 2])
def test_regime_boundary_fuzz(seed):
    """Orders next to the regime boundary v^2 = x, where the peak
    t_p -> 0, g''(t_p) -> 0 and the range brackets built from the curvature
    (R5b) degenerate and must fall back to Alg. 1: v = sqrt(x) (1 +- delta),
    delta in logU[1e-8, 0.3], x in logU[1e-6, 1e4]; FP64 and FP32 entry points
    at the north_star tolerances."""
    rng = np.random.default_rng(300 + seed)
    n = 8000
    x = 10.0 ** rng.uniform(-6, 4, n)
    delta = 10.0 ** rng.uniform(-8, np.log10(0.3), n) * np.where(rng.random(n) < 0.5, -1.0, 1.0)
    v = np.sqrt(x) * (1.0 + delta)
    got = run_gpu(v, x)
    assert_parity(got, run_oracle(v, x), "f64", "regime boundary")
    v32, x32 = v.astype(np.float32), x.astype(np.float32)
    got32 = run_gpu(v32, x32)
    assert_parity(got32, run_oracle(v32, x32), "f32", "regime boundary f32")


def test_peak_bracket_extremes():
    """The analytic peak bracket asinh(v/x) (R5b) at its extremes: v/x up to
    1e34 (the FP32 range finder's domain edge x = 1e-30, v = 1e4) and down to
    v/x ~ 1/v (v^2 just above x), against the oracle."""
    v = np.array([1e4, 1e4, 5e3, 1.0, 1e-3, 0.5, 30.0, 99.0, 1e4, 2.0])
    x = np.array([1e-30, 1e-20, 1e-10, 0.999, 0.99e-6, 0.2499, 1e-30, 9800.0, 9.9e3, 3.99])
    got = run_gpu(v, x)
    lk, dv, dx, plan = oracle.logk(v, x, NB, with_plan=True)
    from parity import errors
    kappa = np.finfo(float).eps * (x + v * plan[:, 0] + 40.0)   # tolerance note, DESIGN §3
    tol_d = np.maximum(1e-10, 5 * kappa)
    assert np.all(errors(got["logk"], lk, "logk") <= 1e-12)
    assert np.all(errors(got["dv"], dv, "dv") <= tol_d)
    assert np.all(errors(got["dx"], dx, "dx") <= tol_d)
