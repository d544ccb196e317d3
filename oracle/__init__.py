"""CPU oracle for the fixed-bin log K_v(x) method -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product package ``paper_2108_11560_b200`` never imports it and shares no code
with it.

Thin ctypes wrapper over ``oracle/oracle.c`` (Alg. 1-3 and Eq. (int) of
arXiv 2108.11560, step by step, in double) and ``oracle/brute.c`` (the plain
integral definition by dense long-double quadrature).  The shared library is
compiled with gcc by ``build()`` (also on first use).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "brute.c")]
_lock = threading.Lock()
_lib = None

# FindZero iteration count printed in Alg. 2
MAX_ITER = 10


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no -ffast-math: IEEE semantics)."""
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", "-o", tmp] + _SRCS + ["-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            dp = ctypes.c_void_p
            lib.oracle_logk.restype = ctypes.c_int
            lib.oracle_logk.argtypes = [dp, dp, ctypes.c_size_t, dp, dp, dp,
                                        ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_double, dp]
            lib.oracle_logk_literal_cm.restype = ctypes.c_int
            lib.oracle_logk_literal_cm.argtypes = [dp, dp, ctypes.c_size_t, dp,
                                                   ctypes.c_int, ctypes.c_double]
            lib.oracle_logk_hess.restype = ctypes.c_int
            lib.oracle_logk_hess.argtypes = [dp, dp, ctypes.c_size_t, dp, dp, dp, dp,
                                             ctypes.c_int, ctypes.c_double]
            lib.brute_logk_hess.restype = ctypes.c_int
            lib.brute_logk_hess.argtypes = [dp, dp, ctypes.c_size_t, dp, ctypes.c_int]
            lib.brute_logk.restype = ctypes.c_int
            lib.brute_logk.argtypes = [dp, dp, ctypes.c_size_t, dp, dp, dp,
                                       ctypes.c_int]
            for name in ("oracle_g", "oracle_g1", "oracle_g2"):
                f = getattr(lib, name)
                f.restype = ctypes.c_double
                f.argtypes = [ctypes.c_double] * 3
            lib.oracle_logk_own_range.restype = ctypes.c_int
            lib.oracle_logk_own_range.argtypes = [dp, dp, ctypes.c_size_t, dp, dp, dp,
                                                  ctypes.c_int, ctypes.c_double]
            lib.oracle_quad_on_plan.restype = ctypes.c_int
            lib.oracle_quad_on_plan.argtypes = [dp, dp, ctypes.c_size_t, dp, dp, dp, dp, dp, dp,
                                                ctypes.c_int]
            lib.oracle_log_eps_f64.restype = ctypes.c_double
            lib.oracle_log_eps_f32.restype = ctypes.c_double
            _lib = lib
    return _lib


def log_eps_f64() -> float:
    return _load().oracle_log_eps_f64()


def log_eps_f32() -> float:
    return _load().oracle_log_eps_f32()


def _ptr(a):
    return None if a is None else a.ctypes.data


def _as_f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def logk(v, x, nbins: int = 128, *, max_iter: int = MAX_ITER, tol: float = 0.0,
         log_eps: float | None = None, threads: int = 1, with_plan: bool = False):
    """Oracle log K_v(x), dlogK/dv, dlogK/dx (float64 arrays).

    ``tol <= 0`` -> fixed ``max_iter`` FindZero iterations (reading R4);
    ``tol > 0`` -> the literal early exit of Alg. 2.  ``threads > 1`` fans
    contiguous chunks out over host threads (ctypes releases the GIL); each
    element is still the same single-threaded code.  With ``with_plan`` also
    returns an (n, 4) array of (t_p, g(t_p), t0, t1).
    """
    lib = _load()
    v = _as_f64(v).ravel()
    x = _as_f64(x).ravel()
    if v.shape != x.shape:
        raise ValueError("v and x must have the same length")
    n = v.size
    le = log_eps_f64() if log_eps is None else float(log_eps)
    out = [np.empty(n), np.empty(n), np.empty(n)]
    plan = np.empty((n, 4)) if with_plan else None

    def run(lo, hi):
        if hi <= lo:
            return
        rc = lib.oracle_logk(
            v.ctypes.data + 8 * lo, x.ctypes.data + 8 * lo, hi - lo,
            out[0].ctypes.data + 8 * lo, out[1].ctypes.data + 8 * lo,
            out[2].ctypes.data + 8 * lo, int(nbins), int(max_iter), float(tol),
            le, None if plan is None else plan.ctypes.data + 32 * lo)
        if rc != 0:
            raise ValueError("oracle_logk: invalid arguments")

    if threads <= 1 or n < 1024:
        run(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda k: run(int(bounds[k]), int(bounds[k + 1])),
                        range(threads)))
    if with_plan:
        return out[0], out[1], out[2], plan
    return out[0], out[1], out[2]


def quad_on_plan(v, x, gp, t0, t1, nbins: int = 128, threads: int = 1):
    """Eq. (int) on a given plan (g(t_p), t0, t1 per element): log K, dlogK/dv,
    dlogK/dx.  Used to check another implementation's quadrature on ITS range
    (several plans are correct, R20; the outputs on a given plan are unique)."""
    lib = _load()
    arrs = [_as_f64(a).ravel() for a in (v, x, gp, t0, t1)]
    n = arrs[0].size
    out = [np.empty(n), np.empty(n), np.empty(n)]

    def run(lo, hi):
        if hi > lo:
            p = [a.ctypes.data + 8 * lo for a in arrs]
            rc = lib.oracle_quad_on_plan(p[0], p[1], hi - lo, p[2], p[3], p[4],
                                         *[o.ctypes.data + 8 * lo for o in out], int(nbins))
            if rc != 0:
                raise ValueError("oracle_quad_on_plan: invalid arguments")

    if threads <= 1 or n < 1024:
        run(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda k: run(int(bounds[k]), int(bounds[k + 1])), range(threads)))
    return out[0], out[1], out[2]


def logk_own_range(v, x, nbins: int = 128, threads: int = 1):
    """log K, dlogK/dv, dlogK/dx with each derivative integrand f^{(1,0)},
    f^{(0,1)} integrated over ITS OWN range (Sec. 4.1) --
    the cross-check of reading R14 (the hot path shares f's range)."""
    lib = _load()
    v = _as_f64(v).ravel()
    x = _as_f64(x).ravel()
    n = v.size
    out = [np.empty(n), np.empty(n), np.empty(n)]

    def run(lo, hi):
        if hi > lo:
            lib.oracle_logk_own_range(v.ctypes.data + 8 * lo, x.ctypes.data + 8 * lo, hi - lo,
                                      out[0].ctypes.data + 8 * lo, out[1].ctypes.data + 8 * lo,
                                      out[2].ctypes.data + 8 * lo, int(nbins), log_eps_f64())

    if threads <= 1 or n < 1024:
        run(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda k: run(int(bounds[k]), int(bounds[k + 1])), range(threads)))
    return out[0], out[1], out[2]


def logk_literal_cm(v, x, nbins: int = 128):
    """The literal Eq. (int) with c_m inside exp (R7) -- for the negative test."""
    lib = _load()
    v = _as_f64(v).ravel()
    x = _as_f64(x).ravel()
    out = np.empty(v.size)
    lib.oracle_logk_literal_cm(v.ctypes.data, x.ctypes.data, v.size,
                               out.ctypes.data, int(nbins), log_eps_f64())
    return out


def brute(v, x, nbins: int = 1 << 14, threads: int = 1):
    """Plain-definition long-double quadrature: (log K, dlogK/dv, dlogK/dx)."""
    lib = _load()
    v = _as_f64(v).ravel()
    x = _as_f64(x).ravel()
    n = v.size
    out = [np.empty(n), np.empty(n), np.empty(n)]

    def run(lo, hi):
        if hi <= lo:
            return
        lib.brute_logk(v.ctypes.data + 8 * lo, x.ctypes.data + 8 * lo, hi - lo,
                       out[0].ctypes.data + 8 * lo, out[1].ctypes.data + 8 * lo,
                       out[2].ctypes.data + 8 * lo, int(nbins))

    if threads <= 1:
        run(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda k: run(int(bounds[k]), int(bounds[k + 1])),
                        range(threads)))
    return out[0], out[1], out[2]


def g(v, x, t):
    return _load().oracle_g(float(v), float(x), float(t))


def g1(v, x, t):
    return _load().oracle_g1(float(v), float(x), float(t))


def g2(v, x, t):
    return _load().oracle_g2(float(v), float(x), float(t))


def logk_hess(v, x, nbins: int = 128, threads: int = 1):
    """Oracle second derivatives: (log K, dv, dx, dvv, dxx, dvx) as float64 arrays."""
    lib = _load()
    v = _as_f64(v).ravel()
    x = _as_f64(x).ravel()
    n = v.size
    lk, dv, dx = np.empty(n), np.empty(n), np.empty(n)
    hs = np.empty((n, 3))

    def run(lo, hi):
        if hi > lo:
            lib.oracle_logk_hess(v.ctypes.data + 8 * lo, x.ctypes.data + 8 * lo, hi - lo,
                                 lk.ctypes.data + 8 * lo, dv.ctypes.data + 8 * lo,
                                 dx.ctypes.data + 8 * lo, hs.ctypes.data + 24 * lo,
                                 int(nbins), log_eps_f64())

    if threads <= 1 or n < 1024:
        run(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda k: run(int(bounds[k]), int(bounds[k + 1])), range(threads)))
    return lk, dv, dx, hs[:, 0].copy(), hs[:, 1].copy(), hs[:, 2].copy()


def brute_hess(v, x, nbins: int = 1 << 14, threads: int = 1):
    """Plain-definition long-double second derivatives (dvv, dxx, dvx)."""
    lib = _load()
    v = _as_f64(v).ravel()
    x = _as_f64(x).ravel()
    n = v.size
    hs = np.empty((n, 3))

    def run(lo, hi):
        if hi > lo:
            lib.brute_logk_hess(v.ctypes.data + 8 * lo, x.ctypes.data + 8 * lo, hi - lo,
                                hs.ctypes.data + 24 * lo, int(nbins))

    if threads <= 1:
        run(0, n)
    else:
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda k: run(int(bounds[k]), int(bounds[k + 1])), range(threads)))
    return hs[:, 0].copy(), hs[:, 1].copy(), hs[:, 2].copy()
