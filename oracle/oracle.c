/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU implementation (C99, IEEE double) of
 * Takekawa's fixed-bin integration method for log K_v(x) and its derivatives
 * (arXiv 2108.11560, /root/reference/PAPER.md, cited below as P:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this.  The product path
 * (paper_2108_11560_b200/) never links, imports or executes it; the two share
 * no code, headers, helpers or constants.
 *
 * The algorithm is written out step by step in the paper's order and
 * notation (Alg. 1 FindRange, Alg. 2 FindZero, Alg. 3 LogBesselK, Eq. (int)),
 * with the readings of garbled / ambiguous passages listed in DESIGN.md §3
 * (tags R1..R22, the same numbering as SURVEY.md §8(c)).  No blocking,
 * fusion, recurrences or reordering: every point evaluation calls the libm
 * routines directly.
 *
 * Pins (tests/test_oracle_pins.py): closed forms K_{1/2}, K_{3/2}, K_{5/2}
 * (log K, d/dx, and d/dv at v=1/2 via e^{2x}E_1(2x)), the recurrence
 * K_{v+1}=K_{v-1}+(2v/x)K_v, symmetry in v, the identity
 * Eq. (deriv), d/dv = 0 at v = 0, mpmath besselk, and the
 * independent long-double brute force in oracle/brute.c.  The plan internals
 * (t_p, t0, t1) are pinned to 30-digit roots of g' = 0 and d(t) = 0
 * (tests/test_oracle_pins.py::test_plan_vs_mpmath_roots): each lies on the
 * outer side of its root (R1) within the 10-iteration bracket bound W0 2^-10,
 * and a FindZero that stalls (0, 1 or 3 iterations) fails that pin.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

#ifndef M_LN2
#define M_LN2 0.69314718055994530942
#endif

/* FindRange doubling cap (SURVEY 8(b) constants): t <= t_s + 2^11 */
#define ORACLE_RANGE_CAP 11

typedef struct {
    double v;   /* order, canonicalised to |v| (R15) */
    double x;   /* argument, x > 0 */
    double gp;  /* g(t_p), set once t_p is known */
    double L;   /* log(eps) (R8/R9) */
    int dn, dm; /* derivative integrand f^{(n,m)} of Sec. 4.1 (oracle_logk_own_range) */
} oracle_ctx;

/* log cosh(z), z >= 0, in the overflow-free form z + log1p(e^{-2z}) - log 2
 * (a plain identity; P:91 uses log cosh). */
static double log_cosh(double z)
{
    z = fabs(z);
    return z + log1p(exp(-2.0 * z)) - M_LN2;
}

/* P:91 Eq.(3): g(t) = log cosh(vt) - x cosh t */
static double g0(const oracle_ctx *c, double t)
{
    return log_cosh(c->v * t) - c->x * cosh(t);
}

/* P:95 Eq.(4): g'(t) = v tanh(vt) - x sinh t */
static double g1(const oracle_ctx *c, double t)
{
    return c->v * tanh(c->v * t) - c->x * sinh(t);
}

/* P:96 Eq.(5): g''(t) = v^2 sech^2(vt) - x cosh t */
static double g2(const oracle_ctx *c, double t)
{
    double ch = cosh(c->v * t);
    return c->v * c->v / (ch * ch) - c->x * cosh(t);
}

/* threshold function of P:205: d(t) = g(t) - g(t_p) - log eps */
static double dfun(const oracle_ctx *c, double t)
{
    return g0(c, t) - c->gp - c->L;
}

typedef double (*ofun)(const oracle_ctx *, double);

/*
 * Alg. 1 FindRange.  Requires F(ts) >= 0.  Finds the smallest
 * m >= 0 with F(ts + 2^{m+1}) < 0 and returns (ts + 2^m, ts + 2^{m+1}),
 * except that the lower end is ts itself when m = 0 (R5: t_s + 2^0 was never
 * tested, the zero may lie in (ts, ts+1)).  Returns 0 on success, -1 when the
 * doubling cap is exceeded.
 */
static int find_range(const oracle_ctx *c, ofun F, double ts, double *lo, double *hi)
{
    int m = 0;
    while (F(c, ts + ldexp(1.0, m + 1)) >= 0.0) {
        m = m + 1;
        if (m > ORACLE_RANGE_CAP)
            return -1;
    }
    *lo = (m == 0) ? ts : ts + ldexp(1.0, m);
    *hi = ts + ldexp(1.0, m + 1);
    return 0;
}

/*
 * Alg. 2 FindZero, "modified Newton method", with the readings
 * R1 (F(a) < 0 <= F(b), a is the end Alg. 3 passes first, return a),
 * R2 (Newton from the current a), R3 (clip to the segment [a, mid]),
 * R4 (max_iter = 10 fixed iterations when tol <= 0; tol > 0 reproduces the
 *     literal early exit "until |a_i - a_{i-1}| < tol"; max_iter = 0 returns
 *     the start a -- only for the negative pin of the plan test),
 * R18 (F'(a) == 0 or non-finite Newton step -> use the bisection point).
 */
static double find_zero(const oracle_ctx *c, ofun F, ofun dF, double a, double b,
                        int max_iter, double tol)
{
    for (int i = 1; i <= max_iter; ++i) {
        double a_prev = a;
        double mid = a + (b - a) / 2.0;                 /* t_shrink */
        double fa = F(c, a);
        double dfa = dF(c, a);
        double tn = mid;                                 /* t_newton */
        if (dfa != 0.0) {
            double s = a - fa / dfa;
            if (isfinite(s))
                tn = s;
        }
        double lo = fmin(a, mid), hi = fmax(a, mid);     /* Clip, R3 */
        if (tn < lo) tn = lo;
        if (tn > hi) tn = hi;
        if (F(c, mid) < 0.0) {
            a = mid;
        } else if (F(c, tn) < 0.0) {
            b = mid;
            a = tn;
        } else {
            b = tn;
        }
        if (tol > 0.0 && fabs(a - a_prev) < tol)         /* literal P:197 */
            break;
    }
    return a;
}

/* DESIGN.md R23: ranges must end below t = 709 (e^t overflows double at
 * 709.78, cosh t at 710.48). */
static const double kTMax = 709.0;

/* Integration plan of Alg. 3 for one canonical (v >= 0, x > 0). */
static int oracle_plan(oracle_ctx *c, int max_iter, double tol,
                       double *tp_out, double *t0_out, double *t1_out)
{
    double lo, hi;
    double tp = 0.0;
    if (c->v * c->v - c->x > 0.0) {                      /* g''(0) > 0; R17 */
        if (find_range(c, g1, 0.0, &lo, &hi) != 0)
            return -1;
        tp = find_zero(c, g1, g2, hi, lo, max_iter, tol); /* P:259 (t_e, t_s) */
    }
    c->gp = g0(c, tp);
    double t0 = 0.0;
    if (-c->x - c->gp <= c->L)                           /* g(0)-g(t_p) <= log eps */
        t0 = find_zero(c, dfun, g1, 0.0, tp, max_iter, tol);
    if (find_range(c, dfun, tp, &lo, &hi) != 0)
        return -1;
    double t1 = find_zero(c, dfun, g1, hi, lo, max_iter, tol);
    /* DESIGN.md R23: an eps-support that reaches t ~ 709, where e^t and
     * cosh t overflow in double, cannot be integrated by the method in double
     * (g is -inf there although the integrand is not small: x below ~1e-306
     * for small orders) -- no result, like an invalid input (R16). */
    if (!(t1 < kTMax))
        return -1;
    *tp_out = tp;
    *t0_out = t0;
    *t1_out = t1;
    return 0;
}

/*
 * Eq. (int) on the range [t0, t1] with shift c->gp = g(t_p):
 * n = nbins trapezoid intervals, nodes t_m = t0 + m h, h = (t1 - t0)/n,
 * weights c_0 = c_n = 1/2, else 1, multiplying the exponential (R7):
 *   S0 = sum c_m e^{g(t_m) - g_p},  log K = g_p + log h + log S0
 * and the derivative integrands of Sec. 4.1 on the same nodes (R14):
 *   S1 = sum c_m e^{g - g_p} t tanh(vt)  -> dlogK/dv = sign(v) S1/S0
 *   S2 = sum c_m e^{g - g_p} cosh t      -> dlogK/dx = -S2/S0
 * (+ the second-order sums when hess != NULL, see oracle_one_h).
 */
static void oracle_quadrature(const oracle_ctx *c, double s, double t0, double t1, int nbins,
                              double *logk, double *dv, double *dx, double *hess)
{
    double h = (t1 - t0) / nbins;
    double S0 = 0.0, S1 = 0.0, S2 = 0.0, S11 = 0.0, S22 = 0.0, S12 = 0.0;
    for (int m = 0; m <= nbins; ++m) {
        double t = t0 + m * h;
        double cm = (m == 0 || m == nbins) ? 0.5 : 1.0;
        double w = cm * exp(g0(c, t) - c->gp);
        S0 += w;
        S1 += w * t * tanh(c->v * t);
        S2 += w * cosh(t);
        S11 += w * t * t;
        S22 += w * cosh(t) * cosh(t);
        S12 += w * t * tanh(c->v * t) * cosh(t);
    }
    *logk = c->gp + log(h) + log(S0);
    *dv = s * S1 / S0;
    *dx = -S2 / S0;
    if (hess) {
        hess[0] = S11 / S0 - (S1 / S0) * (S1 / S0);
        hess[1] = S22 / S0 - (S2 / S0) * (S2 / S0);
        hess[2] = s * (-S12 / S0 + (S1 / S0) * (S2 / S0));
    }
}

/*
 * One element.  Eq. (int) with the weights c_m multiplying the
 * exponential (R7), the derivative integrands of Sec. 4.1
 * d/dv f = t sinh(vt) e^{-x cosh t} = f t tanh(vt),  d/dx f = -cosh t f,
 * accumulated over f's own range and nodes (R14).
 *   log K = g_p + log h + log S0,  dlogK/dv = sign(v) S1/S0,  dlogK/dx = -S2/S0
 */
static void oracle_one_h(double v_in, double x, int nbins, int max_iter, double tol,
                         double log_eps, double *logk, double *dv, double *dx,
                         double *plan, double *hess);

static void oracle_one(double v_in, double x, int nbins, int max_iter, double tol,
                       double log_eps, double *logk, double *dv, double *dx,
                       double *plan)
{
    oracle_one_h(v_in, x, nbins, max_iter, tol, log_eps, logk, dv, dx, plan, NULL);
}

/*
 * Same, plus (when hess != NULL) the second derivatives from the second-order
 * differentiated integrands of Sec. 4.1 (f^{(n,m)} with n+m = 2),
 * accumulated over f's range and nodes like the first-order ones (R14):
 *   d2K/dv2   = int t^2 cosh(vt) e^{-x cosh t}          -> S11 = sum w t^2
 *   d2K/dx2   = int cosh^2 t cosh(vt) e^{-x cosh t}     -> S22 = sum w cosh^2 t
 *   d2K/dvdx  = -int t cosh t sinh(vt) e^{-x cosh t}    -> S12 = sum w t tanh(vt) cosh t
 *   hess[0] = d2logK/dv2  = S11/S0 - (S1/S0)^2
 *   hess[1] = d2logK/dx2  = S22/S0 - (S2/S0)^2
 *   hess[2] = d2logK/dvdx = -S12/S0 + (S1/S0)(S2/S0)     (odd in v, like dv)
 */
static void oracle_one_h(double v_in, double x, int nbins, int max_iter, double tol,
                         double log_eps, double *logk, double *dv, double *dx,
                         double *plan, double *hess)
{
    double nanv = NAN;
    if (plan) { plan[0] = plan[1] = plan[2] = plan[3] = nanv; }
    if (hess) { hess[0] = hess[1] = hess[2] = nanv; }
    if (!(x > 0.0) || !isfinite(x) || !isfinite(v_in)) { /* R16 */
        *logk = *dv = *dx = nanv;
        return;
    }
    double s = (v_in < 0.0) ? -1.0 : 1.0;                /* R15 */
    oracle_ctx c = { fabs(v_in), x, 0.0, log_eps };
    double tp, t0, t1;
    if (oracle_plan(&c, max_iter, tol, &tp, &t0, &t1) != 0) {
        *logk = *dv = *dx = nanv;
        return;
    }
    if (plan) { plan[0] = tp; plan[1] = c.gp; plan[2] = t0; plan[3] = t1; }
    oracle_quadrature(&c, s, t0, t1, nbins, logk, dv, dx, hess);
}

/*
 * Sec. 4.1: the derivative integrands, each with ITS OWN range.
 * log (-1)^m f^{(n,m)}(t) = n log t + m log cosh t + log cosh(vt)  (n even)
 *                                                  + log sinh(vt)  (n odd)
 *                           - x cosh t                               (R13)
 * "and these also have the single range that should be integrated as the
 * f case": the same Alg. 1-3 on this log-integrand.  Used only as
 * the cross-check of R14 (the hot path shares f's range and nodes).
 */
static double gn0(const oracle_ctx *c, double t)
{
    double r = (c->dn ? c->dn * log(t) : 0.0) + c->dm * log_cosh(t) - c->x * cosh(t);
    if (c->dn % 2 == 0) return r + log_cosh(c->v * t);
    double z = c->v * t;                     /* log sinh z, overflow-free (z > 0) */
    return r + z + log(-expm1(-2.0 * z)) - M_LN2;
}
static double gn1(const oracle_ctx *c, double t)
{
    double r = (c->dn ? c->dn / t : 0.0) + c->dm * tanh(t) - c->x * sinh(t);
    if (c->dn % 2 == 0) return r + c->v * tanh(c->v * t);
    return r + c->v / tanh(c->v * t);
}
static double gn2(const oracle_ctx *c, double t)
{
    double ch = cosh(t), cv = cosh(c->v * t), sv = sinh(c->v * t);
    double r = (c->dn ? -c->dn / (t * t) : 0.0) + c->dm / (ch * ch) - c->x * ch;
    if (c->dn % 2 == 0) return r + c->v * c->v / (cv * cv);
    return r - c->v * c->v / (sv * sv);
}
static double dnfun(const oracle_ctx *c, double t)
{
    return gn0(c, t) - c->gp - c->L;
}

/* log of int_0^inf |f^{(n,m)}(t)| dt by Alg. 3 + Eq. (int) on its own range.
 * The peak test of P:257 generalises to "g' > 0 just right of 0": for n >= 1
 * g -> -inf at 0+ (always an interior peak); for n = 0 it is g''(0) > 0,
 * i.e. m + v^2 - x > 0.  Returns NaN when the plan fails. */
static double oracle_log_int_nm(double v, double x, int dn, int dm, int nbins, double log_eps)
{
    oracle_ctx c = { v, x, 0.0, log_eps, dn, dm };
    double lo, hi, tp = 0.0;
    int peaked = (dn > 0) ? 1 : (dm + v * v - x > 0.0);
    if (peaked) {
        if (find_range(&c, gn1, 0.0, &lo, &hi) != 0) return NAN;
        tp = find_zero(&c, gn1, gn2, hi, lo, 10, 0.0);
    }
    c.gp = gn0(&c, tp);
    double t0 = 0.0;
    if (!(gn0(&c, 0.0) - c.gp > c.L))            /* d(0) <= 0 (or -inf for n >= 1) */
        t0 = find_zero(&c, dnfun, gn1, 0.0, tp, 10, 0.0);
    if (find_range(&c, dnfun, tp, &lo, &hi) != 0) return NAN;
    double t1 = find_zero(&c, dnfun, gn1, hi, lo, 10, 0.0);
    double h = (t1 - t0) / nbins, S = 0.0;
    for (int k = 0; k <= nbins; ++k) {
        double t = t0 + k * h;
        double cm = (k == 0 || k == nbins) ? 0.5 : 1.0;
        double e = gn0(&c, t) - c.gp;
        if (isfinite(e)) S += cm * exp(e);       /* the t = 0 node of n >= 1 is 0 */
    }
    return c.gp + log(h) + log(S);
}

/* ---------------- exported (C ABI, loaded by tests via ctypes) ------------- */

/* log(2^-52): eps = DBL_EPSILON, R9 */
double oracle_log_eps_f64(void) { return log(ldexp(1.0, -52)); }
/* log(2^-23): eps = FLT_EPSILON, R9 */
double oracle_log_eps_f32(void) { return log(ldexp(1.0, -23)); }

/*
 * Batched oracle.  v, x, logk, dlogk_dv, dlogk_dx: host arrays of n doubles
 * (outputs may be NULL).  nbins >= 1 trapezoid intervals.  max_iter: FindZero
 * iterations (paper: 10).  tol <= 0: fixed iterations (R4); tol > 0: the
 * literal early exit.  log_eps: log of the threshold (oracle_log_eps_f64()).
 * plan (may be NULL): 4 doubles per element (t_p, g(t_p), t0, t1).
 * Returns 0, or -1 on invalid arguments.
 */
int oracle_logk(const double *v, const double *x, size_t n,
                double *logk, double *dlogk_dv, double *dlogk_dx,
                int nbins, int max_iter, double tol, double log_eps,
                double *plan)
{
    if (nbins < 1 || max_iter < 0)   /* max_iter = 0: FindZero returns its start (negative pin) */
        return -1;
    for (size_t i = 0; i < n; ++i) {
        double a, b, d;
        oracle_one(v[i], x[i], nbins, max_iter, tol, log_eps, &a, &b, &d,
                   plan ? plan + 4 * i : NULL);
        if (logk) logk[i] = a;
        if (dlogk_dv) dlogk_dv[i] = b;
        if (dlogk_dx) dlogk_dx[i] = d;
    }
    return 0;
}

/*
 * Eq. (int) on a GIVEN plan (gp, t0, t1 per element; host arrays of n
 * doubles), for checking a quadrature on another implementation's range
 * (several plans are correct, R20): the outputs are then unique.  NaN plan
 * entries or invalid inputs give NaN outputs.
 */
int oracle_quad_on_plan(const double *v, const double *x, size_t n, const double *gp,
                        const double *t0, const double *t1, double *logk, double *dlogk_dv,
                        double *dlogk_dx, int nbins)
{
    if (nbins < 1)
        return -1;
    for (size_t i = 0; i < n; ++i) {
        double a = NAN, b = NAN, d = NAN;
        if (x[i] > 0.0 && isfinite(x[i]) && isfinite(v[i]) && isfinite(gp[i]) &&
            isfinite(t0[i]) && isfinite(t1[i])) {
            oracle_ctx c = { fabs(v[i]), x[i], gp[i], 0.0 };
            oracle_quadrature(&c, (v[i] < 0.0) ? -1.0 : 1.0, t0[i], t1[i], nbins, &a, &b, &d, NULL);
        }
        if (logk) logk[i] = a;
        if (dlogk_dv) dlogk_dv[i] = b;
        if (dlogk_dx) dlogk_dx[i] = d;
    }
    return 0;
}

/*
 * Second derivatives (see oracle_one_h): hess has 3 doubles per element
 * (d2/dv2, d2/dx2, d2/dvdx); logk/dv/dx as in oracle_logk (may be NULL).
 */
int oracle_logk_hess(const double *v, const double *x, size_t n,
                     double *logk, double *dlogk_dv, double *dlogk_dx, double *hess,
                     int nbins, double log_eps)
{
    if (nbins < 1 || !hess)
        return -1;
    for (size_t i = 0; i < n; ++i) {
        double a, b, d;
        oracle_one_h(v[i], x[i], nbins, 10, 0.0, log_eps, &a, &b, &d, NULL, hess + 3 * i);
        if (logk) logk[i] = a;
        if (dlogk_dv) dlogk_dv[i] = b;
        if (dlogk_dx) dlogk_dx[i] = d;
    }
    return 0;
}

/* Point evaluations, exported so tests can check plan invariants
 * (d(t0) <= 0, d(t1) < 0, g'(t_p) sign) without re-deriving g. */
double oracle_g(double v, double x, double t)  { oracle_ctx c = { fabs(v), x, 0, 0 }; return g0(&c, t); }
double oracle_g1(double v, double x, double t) { oracle_ctx c = { fabs(v), x, 0, 0 }; return g1(&c, t); }
double oracle_g2(double v, double x, double t) { oracle_ctx c = { fabs(v), x, 0, 0 }; return g2(&c, t); }

/*
 * The LITERAL reading of Eq. (int), c_m inside the exponential:
 *   log K ~ g_p + log sum_m h exp(c_m (g(t_m) - g_p)).
 * Exported only so a test can show it is not the method (R7): it is off by
 * ~1e-2 on K_{1/2}(1).
 */
int oracle_logk_literal_cm(const double *v, const double *x, size_t n,
                           double *logk, int nbins, double log_eps)
{
    for (size_t i = 0; i < n; ++i) {
        double plan[4], a, b, d;
        oracle_one(v[i], x[i], nbins, 10, 0.0, log_eps, &a, &b, &d, plan);
        if (!isfinite(a)) { logk[i] = a; continue; }
        oracle_ctx c = { fabs(v[i]), x[i], plan[1], log_eps };
        double t0 = plan[2], t1 = plan[3], h = (t1 - t0) / nbins, S = 0.0;
        for (int m = 0; m <= nbins; ++m) {
            double t = t0 + m * h;
            double cm = (m == 0 || m == nbins) ? 0.5 : 1.0;
            S += h * exp(cm * (g0(&c, t) - c.gp));
        }
        logk[i] = c.gp + log(S);
    }
    return 0;
}

/*
 * Cross-check of R14: d log K/dv and d log K/dx from the derivative
 * integrands f^{(1,0)}, f^{(0,1)} integrated over their OWN ranges:
 *   dlogK/dv = sign(v) exp(log I10 - log K),  dlogK/dx = -exp(log I01 - log K),
 * log K from f's own plan as in oracle_logk.  v = 0 gives dv = 0 (f^{(1,0)} = 0).
 */
int oracle_logk_own_range(const double *v, const double *x, size_t n, double *logk,
                          double *dlogk_dv, double *dlogk_dx, int nbins, double log_eps)
{
    if (nbins < 1)
        return -1;
    for (size_t i = 0; i < n; ++i) {
        double lk, b, d;
        oracle_one(v[i], x[i], nbins, 10, 0.0, log_eps, &lk, &b, &d, NULL);
        if (logk) logk[i] = lk;
        double av = fabs(v[i]), s = (v[i] < 0.0) ? -1.0 : 1.0;
        if (!isfinite(lk)) {
            if (dlogk_dv) dlogk_dv[i] = NAN;
            if (dlogk_dx) dlogk_dx[i] = NAN;
            continue;
        }
        if (dlogk_dv)
            dlogk_dv[i] = (av == 0.0) ? 0.0
                          : s * exp(oracle_log_int_nm(av, x[i], 1, 0, nbins, log_eps) - lk);
        if (dlogk_dx)
            dlogk_dx[i] = -exp(oracle_log_int_nm(av, x[i], 0, 1, nbins, log_eps) - lk);
    }
    return 0;
}
