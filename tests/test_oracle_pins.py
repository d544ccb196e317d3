"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names what fixes the expected value: a closed form (DLMF), an
identity printed in the paper, a library (mpmath arbitrary precision), the
independent long-double brute force of the plain definition (oracle/brute.c,
itself pinned to mpmath here), or a constant printed in the paper
(tests/golden/paper_constants.txt).  Plausible oracle mistakes (a dropped
term, a sign, a swapped bracket end, c_m in the wrong place, the literal
early exit) each fail at least one of these.
"""
import math
import os

import mpmath
import numpy as np
import pytest

import oracle
import workloads

HERE = os.path.dirname(os.path.abspath(__file__))
mpmath.mp.dps = 34

# Oracle acceptance vs exact values.  The method at n=128 with fixed-iteration
# ranges is converged to rounding; the measured worst cases over
# 1000 config samples are 1.3e-15 (log K, relative to max(1,|ref|)), 9.4e-15
# (dv) and 4.9e-15 (dx).  These bounds are ~5-10x above that and far below
# any structural mistake (>= 1e-3).
TOL_LOGK = 1e-14
TOL_DV = 5e-14
TOL_DX = 5e-14


def rel_logk(a, ref):
    return np.abs(a - ref) / np.maximum(1.0, np.abs(ref))


def rel(a, ref):
    return np.abs(a - ref) / np.abs(ref)


XGRID = np.logspace(-3, 3, 61)


# ---------------------------------------------------------------- paper facts
def _golden():
    out = {}
    with open(os.path.join(HERE, "golden", "paper_constants.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, val, cite = line.split()
                out[k] = (val, cite)
    return out


def test_paper_printed_constants():
    """tol=1, max_iter=10; g(0)=-x, g'(0)=0; g''(0)=v^2-x."""
    gold = _golden()
    assert int(gold["max_iter"][0]) == oracle.MAX_ITER
    assert float(gold["tol"][0]) == 1.0
    assert float(gold["c_end"][0]) == 0.5
    rng = np.random.default_rng(7)
    for v, x in zip(rng.uniform(0, 100, 50), 10 ** rng.uniform(-3, 3, 50)):
        assert oracle.g(v, x, 0.0) == -x
        assert oracle.g1(v, x, 0.0) == 0.0
        assert oracle.g2(v, x, 0.0) == pytest.approx(v * v - x, rel=1e-15, abs=1e-300)


def test_log_integrand_matches_definition_mpmath():
    """g, g', g'' of Eq. (3)-(5) against mpmath differentiation of log f."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        v, x, t = rng.uniform(0, 50), 10 ** rng.uniform(-2, 2), rng.uniform(0, 6)
        f = lambda tt: mpmath.log(mpmath.cosh(v * tt)) - x * mpmath.cosh(tt)
        for k, fn in enumerate((oracle.g, oracle.g1, oracle.g2)):
            ref = float(mpmath.diff(f, mpmath.mpf(t), k))
            assert fn(v, x, t) == pytest.approx(ref, rel=1e-12, abs=1e-12 * max(1, x))


# -------------------------------------------------------------- closed forms
def test_half_integer_closed_forms_logk_dx():
    """DLMF 10.39.2 / 10.49.12: K_{1/2}=sqrt(pi/2x)e^{-x}, K_{3/2}=K_{1/2}(1+1/x),
    K_{5/2}=K_{1/2}(1+3/x+3/x^2) and their exact log-derivatives in x."""
    x = XGRID
    base = 0.5 * np.log(np.pi / (2 * x)) - x
    cases = {
        0.5: (base, -1 - 1 / (2 * x)),
        1.5: (base + np.log1p(1 / x), -1 - 1 / (2 * x) - 1 / (x * (x + 1))),
        2.5: (base + np.log(1 + 3 / x + 3 / x ** 2),
              -1 - 1 / (2 * x) - (3 * x + 6) / (x * (x * x + 3 * x + 3))),
    }
    for v, (lk_ref, dx_ref) in cases.items():
        lk, dv, dx = oracle.logk(np.full_like(x, v), x)
        assert rel_logk(lk, lk_ref).max() < TOL_LOGK, v
        assert rel(dx, dx_ref).max() < TOL_DX, v


def test_half_order_dv_closed_form():
    """DLMF 10.38.7: dK_nu/dnu at nu=1/2 is sqrt(pi/2x) E_1(2x) e^{x}, hence
    dlogK/dv = e^{2x} E_1(2x) -- the only closed-form d/dv pin."""
    x = np.logspace(-3, 2.5, 23)
    _, dv, _ = oracle.logk(np.full_like(x, 0.5), x)
    ref = np.array([float(mpmath.exp(2 * mpmath.mpf(xx)) * mpmath.e1(2 * mpmath.mpf(xx)))
                    for xx in x])
    assert rel(dv, ref).max() < TOL_DV


def test_dv_zero_at_order_zero():
    """t tanh(0 t) = 0: dlogK/dv is exactly 0 at v = 0 (K even in v)."""
    x = XGRID
    _, dv, _ = oracle.logk(np.zeros_like(x), x)
    assert np.all(dv == 0.0)


def test_order_symmetry():
    """K_{-v} = K_v (v in R): log K and dx even, dv odd -- bitwise."""
    rng = np.random.default_rng(11)
    v = rng.uniform(0, 200, 300)
    x = 10 ** rng.uniform(-3, 3, 300)
    a = oracle.logk(v, x)
    b = oracle.logk(-v, x)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], -b[1])
    assert np.array_equal(a[2], b[2])


def test_recurrence():
    """Eq. (recu): K_{v+1} = K_{v-1} + (2v/x) K_v, checked overflow-free
    as exp(l(v+1)-l(v)) = exp(l(v-1)-l(v)) + 2v/x."""
    rng = np.random.default_rng(5)
    v = rng.uniform(0.0, 60.0, 400)
    x = 10 ** rng.uniform(-2, 2.5, 400)
    lm, _, _ = oracle.logk(v - 1, x)
    l0, _, _ = oracle.logk(v, x)
    lp, _, _ = oracle.logk(v + 1, x)
    lhs = np.exp(lp - l0)
    rhs = np.exp(lm - l0) + 2 * v / x
    assert rel(lhs, rhs).max() < 2e-13


def test_dx_identity():
    """Eq. (deriv) (it is d log K / dx): -(K_{v-1}+K_{v+1})/(2K_v).
    Ties the S2 accumulator to log K at neighbouring orders."""
    rng = np.random.default_rng(6)
    v = rng.uniform(0.0, 60.0, 400)
    x = 10 ** rng.uniform(-2, 2.5, 400)
    lm, _, _ = oracle.logk(v - 1, x)
    l0, _, dx = oracle.logk(v, x)
    lp, _, _ = oracle.logk(v + 1, x)
    ref = -(np.exp(lm - l0) + np.exp(lp - l0)) / 2
    assert rel(dx, ref).max() < 2e-13
    # and the paper's printed form -v/x - K_{v-1}/K_v
    ref2 = -v / x - np.exp(lm - l0)
    assert rel(dx, ref2).max() < 1e-12


# --------------------------------------------------------------- libraries
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_oracle_vs_mpmath(cfg):
    """mpmath.besselk (34 digits) on seeded samples of every config domain:
    log K; dlogK/dx through K_{v+-1}; dlogK/dv by mpmath numerical differentiation."""
    idx = workloads.sample_indices(cfg, 40, seed=3)
    v, x = workloads.gather(cfg, idx)
    v = v.astype(np.float64)
    x = x.astype(np.float64)
    lk, dv, dx = oracle.logk(v, x)
    for i in range(v.size):
        vv, xx = mpmath.mpf(v[i]), mpmath.mpf(x[i])
        k0 = mpmath.besselk(vv, xx)
        ref = float(mpmath.log(k0))
        assert abs(lk[i] - ref) <= TOL_LOGK * max(1, abs(ref)), (v[i], x[i])
        refx = float(-(mpmath.besselk(vv - 1, xx) + mpmath.besselk(vv + 1, xx)) / (2 * k0))
        assert abs(dx[i] - refx) <= TOL_DX * abs(refx), (v[i], x[i])
        if i < 8:
            refv = float(mpmath.diff(lambda s: mpmath.log(mpmath.besselk(s, xx)), vv))
            assert abs(dv[i] - refv) <= TOL_DV * abs(refv), (v[i], x[i])


def test_brute_force_vs_mpmath():
    """Pin the brute force itself (plain definition, long double) to mpmath."""
    rng = np.random.default_rng(9)
    v = np.concatenate([rng.uniform(0, 100, 30), 10 ** rng.uniform(1, 3, 10)])
    x = np.concatenate([10 ** rng.uniform(-2, 3, 30), 10 ** rng.uniform(-3, 1, 10)])
    lk, dv, dx = oracle.brute(v, x, threads=8)
    for i in range(v.size):
        vv, xx = mpmath.mpf(v[i]), mpmath.mpf(x[i])
        k0 = mpmath.besselk(vv, xx)
        ref = float(mpmath.log(k0))
        assert abs(lk[i] - ref) <= 2e-16 * max(1, abs(ref)) + 1e-300
        refx = float(-(mpmath.besselk(vv - 1, xx) + mpmath.besselk(vv + 1, xx)) / (2 * k0))
        assert abs(dx[i] - refx) <= 1e-15 * abs(refx)


def test_brute_force_converged():
    """2^14 vs 2^15 bins: the brute force is converged (its own consistency)."""
    rng = np.random.default_rng(10)
    v = rng.uniform(0, 300, 40)
    x = 10 ** rng.uniform(-3, 3, 40)
    a = oracle.brute(v, x, 1 << 14, threads=8)
    b = oracle.brute(v, x, 1 << 15, threads=8)
    for k in range(3):
        assert np.allclose(a[k], b[k], rtol=4e-16, atol=0)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_oracle_vs_brute_force(cfg):
    """Oracle (Alg. 1-3, n=128) against the plain definition on 300 samples/config."""
    idx = workloads.sample_indices(cfg, 300, seed=4)
    v, x = workloads.gather(cfg, idx)
    v = v.astype(np.float64)
    x = x.astype(np.float64)
    o = oracle.logk(v, x)
    b = oracle.brute(v, x, threads=8)
    assert rel_logk(o[0], b[0]).max() < TOL_LOGK
    nz = b[1] != 0
    assert rel(o[1][nz], b[1][nz]).max() < TOL_DV
    assert rel(o[2], b[2]).max() < TOL_DX


def test_extreme_domain_vs_brute_force():
    """Beyond the paper's grid (R22): huge/small x and large v stay accurate."""
    v = np.array([0, 0, 5, 0, 10, 2000, 5000, 1e4, 0.5, 5, 0, 30.0])
    x = np.array([1e3, 1e4, 1e5, 1e6, 1e8, 1e-3, 1e-4, 1e-2, 1e-6, 1e-10, 1e-8, 1e-30])
    o = oracle.logk(v, x)
    b = oracle.brute(v, x)
    assert rel_logk(o[0], b[0]).max() < TOL_LOGK
    assert rel(o[2], b[2]).max() < 1e-12


def test_large_x_dv_vs_brute_force():
    """d log K/dv for x in [1e5, 1e8] (beyond the configs, R22) against the
    plain definition.  There every double evaluation of the exponent
    vt - x cosh t - g(t_p) carries an absolute error ~kappa = eps (x + v t_p
    + 40) (DESIGN.md §3 tolerance note), which a weighted mean such as
    S1/S0 turns into a relative error of order kappa; the long double brute
    force does not (eps_ld x <= 1e-11).  Measured: the oracle within 0.2 kappa
    (median 0.04 kappa); pinned at 0.5 kappa, the bound the GPU derivative
    parity tests at large x are stated in."""
    rng = np.random.default_rng(3)
    n = 300
    x = 10 ** rng.uniform(5, 8, n)
    v = np.where(rng.random(n) < 0.5, rng.uniform(0, 30, n), 10 ** rng.uniform(-3, 3.5, n))
    lk, dv, dx, plan = oracle.logk(v, x, 128, with_plan=True)
    b = oracle.brute(v, x, threads=8)
    kappa = np.finfo(float).eps * (x + v * plan[:, 0] + 40.0)
    assert np.all(np.abs(dv - b[1]) <= 0.5 * kappa * np.abs(b[1]))
    assert rel(dx, b[2]).max() < 1e-12
    assert rel_logk(lk, b[0]).max() < TOL_LOGK


# ------------------------------------------------------------ plan invariants
def test_plan_sign_invariants():
    """The sign invariants that define the plan: g'(t_p) <= 0 (peak approached
    from outside, R1), d(t0) <= 0 when t0 > 0, d(t1) < 0, t0 <= t_p <= t1
    (the plan's values themselves are pinned by test_plan_vs_mpmath_roots)."""
    le = oracle.log_eps_f64()
    for cfg in ["c1", "c2", "c3", "c5"]:
        idx = workloads.sample_indices(cfg, 200, seed=5)
        v, x = workloads.gather(cfg, idx)
        *_, plan = oracle.logk(v, x, with_plan=True)
        for i in range(v.size):
            tp, gp, t0, t1 = plan[i]
            assert 0 <= t0 <= tp <= t1
            assert gp == oracle.g(v[i], x[i], tp)
            if v[i] * v[i] > x[i]:
                assert tp > 0 and oracle.g1(v[i], x[i], tp) <= 0
            else:
                assert tp == 0
            if t0 > 0:
                assert oracle.g(v[i], x[i], t0) - gp - le <= 0
            assert oracle.g(v[i], x[i], t1) - gp - le < 0


def test_nbins_convergence():
    """Fixed n: doubling n from 128 to 256 changes nothing beyond rounding."""
    v, x = workloads.generate("c2", 0, 500)
    a = oracle.logk(v, x, 128)
    b = oracle.logk(v, x, 256)
    assert rel_logk(a[0], b[0]).max() < 1e-14
    assert rel(a[2], b[2]).max() < 5e-14


# --------------------------------------------------- readings
def test_reading_R7_cm_outside_exp():
    """Eq. (int) prints c_m INSIDE the exponential; that literal form is
    off by ~1e-2 on K_{1/2}(1), so the weights must multiply exp."""
    ref = 0.5 * math.log(math.pi / 2) - 1.0
    lit = oracle.logk_literal_cm([0.5], [1.0])[0]
    ours = oracle.logk([0.5], [1.0])[0][0]
    assert abs(lit - ref) > 1e-3
    assert abs(ours - ref) < 1e-15


def test_reading_R4_literal_early_exit_fails_on_c3():
    """The literal 'until |dt|<tol' with tol=1 leaves t_p far from
    the peak on config 3 (exp overflow / large error); fixed 10 iterations do not."""
    idx = workloads.sample_indices("c3", 400, seed=6)
    v, x = workloads.gather("c3", idx)
    lit = oracle.logk(v, x, tol=1.0)[0]
    fix = oracle.logk(v, x)[0]
    b = oracle.brute(v, x, threads=8)[0]
    bad_lit = ~np.isfinite(lit) | (rel_logk(np.nan_to_num(lit), b) > 1e-10)
    assert bad_lit.sum() > 0
    assert rel_logk(fix, b).max() < TOL_LOGK


def test_invalid_inputs_give_nan():
    """x <= 0 or non-finite inputs -> NaN outputs, no batch failure (R16)."""
    v = np.array([1.0, 1.0, 1.0, np.nan, np.inf, 1.0, 1.0])
    x = np.array([0.0, -1.0, np.nan, 1.0, 1.0, np.inf, 2.0])
    lk, dv, dx = oracle.logk(v, x)
    assert np.all(np.isnan(lk[:6])) and np.all(np.isnan(dv[:6])) and np.all(np.isnan(dx[:6]))
    assert np.isfinite(lk[6])


# ------------------------------------------------ second derivatives (§8(f) 1)
def test_hess_closed_forms_dxx():
    """d2/dx2 log K: 1/(2x^2) at v=1/2 and 1/(2x^2) + (2x+1)/(x^2 (x+1)^2) at v=3/2
    (differentiating the DLMF 10.39.2 closed forms)."""
    x = XGRID
    for v, ref in ((0.5, 1 / (2 * x * x)),
                   (1.5, 1 / (2 * x * x) + (2 * x + 1) / (x * x * (x + 1) ** 2))):
        _, _, dx, dvv, dxx, dvx = oracle.logk_hess(np.full_like(x, v), x)
        # S22/S0 - (S2/S0)^2 cancels by (dx^2)/|dxx| (5e5 at x=1e3): the error
        # bound is relative to the moment S22/S0 = dxx + dx^2
        assert np.all(np.abs(dxx - ref) <= 1e-14 * (np.abs(ref) + dx * dx)), v


def test_hess_bessel_ode():
    """K_v solves x^2 K'' + x K' - (x^2 + v^2) K = 0, i.e. with L = log K:
    L'' = 1 + v^2/x^2 - L'/x - L'^2 -- ties the S22 sum to the S2 sum."""
    rng = np.random.default_rng(12)
    v = rng.uniform(0.0, 80.0, 400)
    x = 10 ** rng.uniform(-2, 2.5, 400)
    lk, dv, dx, dvv, dxx, dvx = oracle.logk_hess(v, x)
    ref = 1 + v * v / (x * x) - dx / x - dx * dx
    # conditioning: the right side is a difference of terms ~ dx^2
    assert np.all(np.abs(dxx - ref) <= 1e-12 * (np.abs(ref) + dx * dx + v * v / (x * x) + 1))


def test_hess_symmetry_and_order_zero():
    """d2/dv2 and d2/dx2 even in v, d2/dvdx odd; d2/dvdx = 0 at v = 0."""
    rng = np.random.default_rng(13)
    v = rng.uniform(0, 50, 200)
    x = 10 ** rng.uniform(-2, 2, 200)
    a = oracle.logk_hess(v, x)
    b = oracle.logk_hess(-v, x)
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
    assert np.array_equal(a[5], -b[5])
    z = oracle.logk_hess(np.zeros(20), x[:20])
    assert np.all(z[5] == 0.0)


def test_hess_vs_mpmath():
    """Second derivatives against mpmath numerical differentiation of besselk."""
    pts = [(0.5, 1.0), (3.0, 2.0), (40.0, 5.0), (0.0, 0.5), (12.0, 0.3), (80.0, 200.0)]
    v = np.array([p[0] for p in pts])
    x = np.array([p[1] for p in pts])
    _, dv, dx, dvv, dxx, dvx = oracle.logk_hess(v, x)
    for i, (vi, xi) in enumerate(pts):
        f = lambda s, y: mpmath.log(mpmath.besselk(s, y))
        rvv = float(mpmath.diff(lambda s: f(s, xi), vi, 2))
        rxx = float(mpmath.diff(lambda y: f(vi, y), xi, 2))
        rvx = float(mpmath.diff(f, (vi, xi), (1, 1)))
        k_vv = abs(dvv[i]) + dv[i] ** 2
        k_xx = abs(dxx[i]) + dx[i] ** 2
        k_vx = abs(dvx[i]) + abs(dv[i] * dx[i])
        assert abs(dvv[i] - rvv) <= 1e-13 * k_vv + 1e-14, (vi, xi, dvv[i], rvv)
        assert abs(dxx[i] - rxx) <= 1e-13 * k_xx + 1e-14, (vi, xi, dxx[i], rxx)
        assert abs(dvx[i] - rvx) <= 1e-13 * k_vx + 1e-14, (vi, xi, dvx[i], rvx)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_hess_vs_brute_force(cfg):
    idx = workloads.sample_indices(cfg, 150, seed=14)
    v, x = workloads.gather(cfg, idx)
    _, dv, dx, dvv, dxx, dvx = oracle.logk_hess(v, x)
    bvv, bxx, bvx = oracle.brute_hess(v, x, threads=8)
    assert np.all(np.abs(dvv - bvv) <= 1e-13 * (np.abs(bvv) + dv * dv) + 1e-15)
    assert np.all(np.abs(dxx - bxx) <= 1e-13 * (np.abs(bxx) + dx * dx) + 1e-15)
    assert np.all(np.abs(dvx - bvx) <= 1e-13 * (np.abs(bvx) + np.abs(dv * dx)) + 1e-15)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_reading_R14_own_range_derivatives(cfg):
    """R14: the paper integrates each derivative integrand f^{(n,m)} over its OWN
    range (Sec. 4.1); the hot path shares f's range and nodes.  The
    oracle implements both; they agree to rounding (relative 2e-14 of max(1,|log K|):
    exp(log I - log K) carries eps*|log K|), and the own-range result is itself
    pinned to the long-double brute force."""
    v, x = workloads.generate(cfg, 0, 1500)
    v = v.astype(np.float64)
    x = x.astype(np.float64)
    lk, dv, dx = oracle.logk(v, x, 128)
    lk2, dv2, dx2 = oracle.logk_own_range(v, x, 128)
    assert np.array_equal(lk, lk2)
    sc = np.maximum(1.0, np.abs(lk))
    nz = dv != 0
    assert np.all(dv2[~nz] == 0.0)
    assert np.all(np.abs(dv2[nz] - dv[nz]) <= 2e-14 * sc[nz] * np.abs(dv[nz]))
    assert np.all(np.abs(dx2 - dx) <= 2e-14 * sc * np.abs(dx))
    bl, bv, bx = oracle.brute(v[:120], x[:120], threads=os.cpu_count() or 1)
    nzb = bv != 0
    assert np.all(np.abs(dv2[:120][nzb] - bv[nzb]) <= 5e-14 * sc[:120][nzb] * np.abs(bv[nzb]))
    assert np.all(np.abs(dx2[:120] - bx) <= 5e-14 * sc[:120] * np.abs(bx))


def test_cancellation_band_vs_brute_force():
    """Where v t and x cosh t (~1e4) cancel to |log K| < 20, the oracle's log K
    is within the exponent's rounding floor eps (x + v t_p) of the long-double
    plain-definition value (DESIGN.md §3 tolerance note): double arithmetic
    cannot do better there, and this is the floor the GPU test holds the
    kernels to."""
    from parity import cancellation_band, errors
    v, x = cancellation_band(128, 11)
    lk, _, _, plan = oracle.logk(v, x, 128, with_plan=True, threads=8)
    lk_b = oracle.brute(v, x, threads=8)[0]
    kappa = np.finfo(float).eps * (x + v * plan[:, 0] + 40.0)
    tol = np.maximum(1e-12, kappa / np.maximum(1.0, np.abs(lk_b)))
    e = errors(lk, lk_b, "logk")
    assert np.all(e <= tol), ((e / tol).max(), v[np.argmax(e / tol)], x[np.argmax(e / tol)])
    # and the floor is not vacuous: the oracle's error there is not far below it
    assert (e / tol).max() > 0.05


# ------------------------------------------------- the plan vs mpmath roots
from plan_pins import mp_plan, plan_violations  # noqa: E402


@pytest.fixture(scope="module")
def plan_samples():
    """200 seeded samples per config with their exact plans (elements whose
    d(0) sits within 1e-9 of the threshold are skipped: there the t0 search
    is taken or not by rounding)."""
    out = {}
    for cfg in ["c1", "c2", "c3", "c4", "c5"]:
        idx = workloads.sample_indices(cfg, 200, seed=21)
        v, x = workloads.gather(cfg, idx)
        v = v.astype(np.float64)
        x = x.astype(np.float64)
        ex = [mp_plan(a, b) for a, b in zip(v, x)]
        keep = np.array([abs(e[2]) > 1e-9 for e in ex])
        out[cfg] = (v[keep], x[keep], [e for e, k in zip(ex, keep) if k])
    return out


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_plan_vs_mpmath_roots(plan_samples, cfg):
    """Alg. 1-3's plan against 30-digit roots of g' = 0 and
    d(t) = 0: every t_p, t0, t1 lies on the outer side of its root within the
    bracket bound of 10 FindZero iterations (see plan_violations); g(t_p) is
    at most the exact peak value and within |g''| (W0 2^-10)^2 / 2 of it."""
    v, x, ex = plan_samples[cfg]
    assert v.size >= 190
    *_, plan = oracle.logk(v, x, with_plan=True)
    bad = plan_violations(v, x, plan, ex)
    assert not bad.any(), (np.nonzero(bad)[0][:5], v[bad][:3], x[bad][:3])
    for i in range(v.size):
        with mpmath.workdps(30):
            vv, xx, tps = mpmath.mpf(v[i]), mpmath.mpf(x[i]), mpmath.mpf(ex[i][0][0])
            gstar = float(mpmath.log(mpmath.cosh(vv * tps)) - xx * mpmath.cosh(tps))
        assert plan[i, 1] <= gstar + 1e-13 * max(1.0, abs(gstar))


@pytest.mark.parametrize("max_iter", [0, 1, 3])
def test_plan_pin_rejects_stalled_findzero(plan_samples, max_iter):
    """Negative pin: a FindZero that stalls -- returns Alg. 1's bracket end
    (0 iterations) or stops after 1 or 3 -- fails test_plan_vs_mpmath_roots on
    every config.  The value pins cannot see it: with 3 iterations the n = 128
    outputs agree with the converged ones to <= 2.3e-14 on c1/c2/c3/c5 (the
    range is only wider); with 0 or 1 they still do on c1 and c5
    (c2/c3 overflow: g(t_p) then lies too far below the peak)."""
    for cfg, (v, x, ex) in plan_samples.items():
        *_, plan = oracle.logk(v, x, with_plan=True, max_iter=max_iter)
        assert plan_violations(v, x, plan, ex).any(), (cfg, max_iter)


def test_reading_R23_ranges_past_double_overflow():
    """R23: where the eps-support reaches t = 709 the method cannot evaluate its
    integrand in double (cosh t overflows at 710.48 while x cosh t is still
    O(1)): the oracle returns NaN (like an invalid input, R16) instead of a
    silently truncated integral.  Closed form K_{1/2}(x) = sqrt(pi/(2x)) e^{-x}:
    at x = 1e-300 (support ending near t = 695) the oracle is finite and
    matches it; at x = 1e-310 it would need t up to ~717."""
    v = np.array([0.5, 0.5, 0.0, 1.0])
    x = np.array([1e-300, 1e-310, 5e-324, 2.2e-308])
    lk, dv, dx, plan = oracle.logk(v, x, 512, with_plan=True)
    assert np.isfinite(lk[0]) and plan[0, 3] < 709.0
    ref = 0.5 * np.log(np.pi / (2.0 * x[0])) - x[0]
    assert abs(lk[0] - ref) <= 1e-12 * abs(ref)
    assert np.isnan(lk[1:]).all() and np.isnan(dv[1:]).all() and np.isnan(dx[1:]).all()
