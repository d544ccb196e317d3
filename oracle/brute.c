/*
 * oracle/brute.c -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.c header).
 *
 * Brute-force evaluation of the PLAIN DEFINITION, independent of the paper's
 * range-finding algorithm:
 *   K_v(x) = int_0^inf cosh(vt) exp(-x cosh t) dt           (Eq. 1-2)
 *   dK/dv  = int_0^inf t sinh(vt) exp(-x cosh t) dt
 *   dK/dx  = -int_0^inf cosh t cosh(vt) exp(-x cosh t) dt
 * in long double (x87 80-bit, eps_ld = 2^-63), by a dense trapezoid on a
 * generously padded range found by its own code (full-precision bisection
 * for the peak, then fixed steps out until the log-integrand has dropped by
 * 60 below its maximum, well past -log(eps_ld) = 43.7).  Shares nothing with
 * oracle.c except being C.
 *
 * Used to pin oracle.c (tests/test_oracle_pins.py); ~2-3 ms per element at
 * 2^14 bins, so tests use a few hundred elements.
 */
#include <math.h>
#include <stddef.h>

typedef long double ld;

static ld b_logcosh(ld z)
{
    z = fabsl(z);
    return z + log1pl(expl(-2.0L * z)) - logl(2.0L);
}

/* log f(t) = log cosh(vt) - x cosh t */
static ld b_logf(ld v, ld x, ld t) { return b_logcosh(v * t) - x * coshl(t); }
/* d/dt log f */
static ld b_dlogf(ld v, ld x, ld t) { return v * tanhl(v * t) - x * sinhl(t); }
static ld b_d2logf(ld v, ld x, ld t)
{
    ld ch = coshl(v * t);
    return v * v / (ch * ch) - x * coshl(t);
}

/*
 * nbins: trapezoid intervals (tests use 2^14 and 2^15 for the convergence
 * check).  Outputs: log K, dlogK/dv (odd in v), dlogK/dx; written as double.
 * Returns 0 or -1 on bad arguments.  Elements with x <= 0 / non-finite
 * inputs get NaN.
 */
static int brute_core(const double *v_in, const double *x_in, size_t n,
                      double *logk, double *dlogk_dv, double *dlogk_dx, double *hess,
                      int nbins);

int brute_logk(const double *v_in, const double *x_in, size_t n,
               double *logk, double *dlogk_dv, double *dlogk_dx, int nbins)
{
    return brute_core(v_in, x_in, n, logk, dlogk_dv, dlogk_dx, NULL, nbins);
}

/* Second derivatives of log K (d2/dv2, d2/dx2, d2/dvdx; 3 per element) from
 * the second-order differentiated integrands, plain definition. */
int brute_logk_hess(const double *v_in, const double *x_in, size_t n, double *hess, int nbins)
{
    return brute_core(v_in, x_in, n, NULL, NULL, NULL, hess, nbins);
}

static int brute_core(const double *v_in, const double *x_in, size_t n,
                      double *logk, double *dlogk_dv, double *dlogk_dx, double *hess,
                      int nbins)
{
    if (nbins < 2)
        return -1;
    for (size_t i = 0; i < n; ++i) {
        ld x = x_in[i], vs = v_in[i];
        if (!(x > 0) || !isfinite(x_in[i]) || !isfinite(v_in[i])) {
            if (logk) logk[i] = NAN;
            if (dlogk_dv) dlogk_dv[i] = NAN;
            if (dlogk_dx) dlogk_dx[i] = NAN;
            if (hess) hess[3 * i] = hess[3 * i + 1] = hess[3 * i + 2] = NAN;
            continue;
        }
        ld sgn = vs < 0 ? -1.0L : 1.0L;
        ld v = fabsl(vs);
        /* peak by plain bisection on the derivative (no Newton) */
        ld tp = 0.0L;
        if (b_dlogf(v, x, 1e-30L) > 0) {
            ld lo = 0.0L, hi = 1.0L;
            while (b_dlogf(v, x, hi) > 0)
                hi *= 2.0L;
            for (int it = 0; it < 400 && hi - lo > 0; ++it) {
                ld mid = 0.5L * (lo + hi);
                if (mid <= lo || mid >= hi)
                    break;
                if (b_dlogf(v, x, mid) > 0) lo = mid; else hi = mid;
            }
            tp = 0.5L * (lo + hi);
        }
        ld gp = b_logf(v, x, tp);
        ld curv = fabsl(b_d2logf(v, x, tp));
        ld sigma = curv > 0 ? 1.0L / sqrtl(curv) : 1.0L / sqrtl(x);
        ld step = fminl(0.05L, sigma / 4.0L);
        ld ta = tp, tb = tp;
        while (ta > 0 && b_logf(v, x, ta) > gp - 60.0L)
            ta = fmaxl(0.0L, ta - step);
        while (b_logf(v, x, tb) > gp - 60.0L)
            tb += step;
        ld h = (tb - ta) / nbins;
        ld S0 = 0, S1 = 0, S2 = 0, S11 = 0, S22 = 0, S12 = 0;
        for (int m = 0; m <= nbins; ++m) {
            ld t = ta + m * h;
            ld c = (m == 0 || m == nbins) ? 0.5L : 1.0L;
            ld w = c * expl(b_logf(v, x, t) - gp);
            ld ch = coshl(t), th = tanhl(v * t);
            S0 += w;
            S1 += w * t * th;
            S2 += w * ch;
            S11 += w * t * t;
            S22 += w * ch * ch;
            S12 += w * t * th * ch;
        }
        if (logk) logk[i] = (double)(gp + logl(h) + logl(S0));
        if (dlogk_dv) dlogk_dv[i] = (double)(sgn * S1 / S0);
        if (dlogk_dx) dlogk_dx[i] = (double)(-S2 / S0);
        if (hess) {
            ld m1 = S1 / S0, m2 = S2 / S0;
            hess[3 * i] = (double)(S11 / S0 - m1 * m1);
            hess[3 * i + 1] = (double)(S22 / S0 - m2 * m2);
            hess[3 * i + 2] = (double)(sgn * (-S12 / S0 + m1 * m2));
        }
    }
    return 0;
}
