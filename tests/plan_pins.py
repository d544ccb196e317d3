"""Exact integration plans (30-digit mpmath) and the plan pins, shared by
tests/test_oracle_pins.py (the oracle's plan) and tests/test_gpu_parity.py
(the plan the kernels integrate over, bessel_logk_plan_f64).  Depends on
the definitions only (Alg. 1's doubling P:156-168), not
on oracle/ or the CUDA path."""
import mpmath
import numpy as np


def _mp_root(f, a, b):
    """Bisection to ~1e-26 relative on a sign change of f over (a, b)."""
    fa = f(a)
    assert fa * f(b) < 0
    tol = mpmath.mpf(10) ** -26
    while b - a > tol * max(1, abs(a)):
        m = (a + b) / 2
        fm = f(m)
        if fm == 0:
            return m
        if (fm > 0) == (fa > 0):
            a, fa = m, fm
        else:
            b = m
    return (a + b) / 2


def _mp_doubling(F, ts):
    """Alg. 1's bracket width from t_s (reading R5), with the exact
    F: m = min{m >= 0 : F(t_s + 2^(m+1)) < 0}; width 2 when m = 0, else 2^m."""
    m = 0
    while F(ts + mpmath.mpf(2) ** (m + 1)) >= 0:
        m += 1
    return 2.0 if m == 0 else float(2 ** m)


def mp_plan(v, x, log_eps=None):
    """The exact plan at 30 digits, from the definitions only (P:91-96,
    P:121-133): t_p* the root of g' = v tanh(vt) - x sinh t (0 when
    v^2 <= x), t0*, t1* the roots of d(t) = g(t) - g(t_p*) - log eps left and
    right of it (t0* = 0 when d(0) <= 0 has no root), plus Alg. 1's initial
    bracket widths W0 of the three searches (2^m, the t0 search: t_p)."""
    with mpmath.workdps(30):
        v, x = mpmath.mpf(float(v)), mpmath.mpf(float(x))
        L = mpmath.log(mpmath.mpf(2) ** -52) if log_eps is None else mpmath.mpf(log_eps)

        def g(t):
            return mpmath.log(mpmath.cosh(v * t)) - x * mpmath.cosh(t)

        def g1(t):
            return v * mpmath.tanh(v * t) - x * mpmath.sinh(t)

        tp, w_tp = mpmath.mpf(0), 0.0
        if v * v - x > 0:
            w_tp = _mp_doubling(g1, mpmath.mpf(0))
            hi = mpmath.mpf(2)
            while g1(hi) > 0:
                hi *= 2
            tp = _mp_root(g1, hi * mpmath.mpf(10) ** -30, hi)
        gp = g(tp)

        def d(t):
            return g(t) - gp - L

        t0 = mpmath.mpf(0)
        d0 = float(d(mpmath.mpf(0)))
        if d0 <= 0:
            t0 = _mp_root(d, mpmath.mpf(0), tp)
        w_t1 = _mp_doubling(d, tp)
        hi = tp + 2
        while d(hi) >= 0:
            hi = tp + 2 * (hi - tp)
        t1 = _mp_root(d, tp, hi)
        return (float(tp), float(t0), float(t1)), (w_tp, float(tp), w_t1), d0


def plan_violations(v, x, plan, exact):
    """Per element, whether the oracle's (t_p, t0, t1) break the pin:
      * orientation (R1, Alg. 2 keeps F(a) < 0 and returns a): t_p >= t_p*,
        t0 <= t0*, t1 >= t1* -- the range is conservative;
      * the 10-iteration bound: every iteration of Alg. 2 at least halves the
        bracket (t_shrink, and the Newton point clipped to [a, t_shrink]), so
        |t - t*| <= W0 2^-10 with W0 Alg. 1's bracket (t_p for the t0 search).
    Slack 1e-12 max(1, t*) for double rounding of F near its zero."""
    bad = []
    for i in range(len(v)):
        (tp_s, t0_s, t1_s), (w_tp, w_t0, w_t1), _ = exact[i]
        tp, _, t0, t1 = plan[i]
        out = False
        for t, ts, w, side in ((tp, tp_s, w_tp, +1), (t0, t0_s, w_t0, -1), (t1, t1_s, w_t1, +1)):
            slack = 1e-12 * max(1.0, abs(ts))
            if side * (t - ts) < -slack or abs(t - ts) > w * 2.0 ** -10 + slack:
                out = True
        bad.append(out)
    return np.array(bad)


def plan_check_f32(v, x, plan, exact, end_nats, peak_gap):
    """The FP32 range finder's plan (BLK_RANGE_AUTO from 48 bins): Alg. 1-2 in
    FP32, FindZero ending on the paper's "until" clause at working
    tolerances in log units (R4) -- an end once F(a) >= -end_nats, the peak
    once Newton's estimate of the gap below the maximum F^2/(2|F'|) is below
    peak_gap -- all capped at 10 iterations.  Valid when
      * the shift is at or below the exact peak value, by at most
        max(2 peak_gap, |g''(t_p*)| (W0 2^-10)^2 / 2) (the stopping rule with
        2x slack on Newton's estimate, or the 10-iteration bracket) plus e_d;
      * each range end lies on the outer side of the root of its OWN
        threshold g(t) = g_p + log eps (so also of the exact eps-support,
        g_p <= g(t_p*)), where d = g - g_p - log eps >= -end_nats - e_d (the
        stopping rule) or within W0 2^-10 + e_d / |g'| of it (the
        10-iteration bracket when Alg. 2's
        preference for the bisection point keeps Newton from converging --
        e.g. t1 for large x: bisection steps 2 -> 1 -> ... -> 0.0317 against
        the root 0.03125 after 10 iterations);
    e_d = 2^-20 (|g_p| + x cosh t + v t + 40) is the FP32 resolution of d.
    Returns the per-element violation mask."""
    bad = []
    with mpmath.workdps(30):
        L = mpmath.log(mpmath.mpf(2) ** -52)
        for i in range(len(v)):
            (tp_s, t0_s, t1_s), (w_tp, w_t0, w_t1), _ = exact[i]
            _, gp, t0, t1 = plan[i]
            vv, xx = mpmath.mpf(float(v[i])), mpmath.mpf(float(x[i]))

            def g(t):
                return mpmath.log(mpmath.cosh(vv * t)) - xx * mpmath.cosh(t)

            def g1(t):
                return vv * mpmath.tanh(vv * t) - xx * mpmath.sinh(t)

            tps = mpmath.mpf(tp_s)
            gstar = g(tps)
            g2 = abs(float(vv * vv / mpmath.cosh(vv * tps) ** 2 - xx * mpmath.cosh(tps)))
            e_p = 2.0 ** -20 * (abs(gp) + float(x[i]) * float(mpmath.cosh(tps)) + float(v[i]) * tp_s + 40.0)
            gap = float(gstar) - gp
            out = gap < -e_p or gap > max(2 * peak_gap, g2 * (w_tp * 2.0 ** -10) ** 2 / 2) + e_p

            def d(t):
                return g(t) - mpmath.mpf(gp) - L

            for t, side, w0 in ((t0, -1, w_t0), (t1, +1, w_t1)):
                if side < 0 and d(mpmath.mpf(0)) > 0:
                    out |= t != 0.0
                    continue
                if side < 0:
                    ts = _mp_root(d, mpmath.mpf(0), tps)
                else:
                    hi = tps + 2
                    while d(hi) >= 0:
                        hi = tps + 2 * (hi - tps)
                    ts = _mp_root(d, tps, hi)
                slope = abs(float(g1(ts)))
                ed = 2.0 ** -20 * (abs(gp) + float(x[i]) * float(mpmath.cosh(ts)) + float(v[i]) * float(ts) + 40.0)
                res = ed / max(slope, 1e-300)
                tsf = float(ts)
                dt = float(d(mpmath.mpf(float(t))))         # own threshold function at the end
                outer = side * (t - tsf) >= -res
                near = dt >= -end_nats - ed or abs(t - tsf) <= w0 * 2.0 ** -10 + res
                if not (outer and near):
                    out = True
            bad.append(out)
    return np.array(bad)
