"""NIG log-likelihood oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Textbook normal-inverse-Gaussian density (Barndorff-Nielsen 1997; the
application PAPER.md P:45-50 motivates), with log K_1 and dlogK_1/dz from the
oracle's step-by-step implementation of the paper's method:

  log p(y) = log a + log d - log pi + d g + b (y - m) - log q + log K_1(a q),
  q = sqrt(d^2 + (y-m)^2), g = sqrt(a^2 - b^2).

Gradient by the chain rule (D = dlogK_1/dz at z = a q):
  d/da = 1/a + d a/g + q D;  d/db = (y-m) - d b/g;
  d/dd = 1/d + g - d/q^2 + a D d/q;  d/dm = -b + (y-m)/q^2 - a D (y-m)/q.
Sums by math.fsum (exactly rounded).  Pinned in tests/test_nig.py against
scipy.stats.norminvgauss (log p) and central finite differences (gradient).
"""
from __future__ import annotations

import math

import numpy as np

from . import logk as _logk


def nig_terms(y, a, b, d, m, nbins: int = 128, threads: int = 8):
    """Per-element log p and its 4 partial derivatives: array (5, n)."""
    y = np.asarray(y, dtype=np.float64)
    r = y - m
    q = np.sqrt(d * d + r * r)
    g = math.sqrt(a * a - b * b)
    lk, _, D = _logk(np.ones_like(q), a * q, nbins, threads=threads)
    out = np.empty((5, y.size))
    out[0] = math.log(a) + math.log(d) - math.log(math.pi) + d * g + b * r - np.log(q) + lk
    out[1] = 1.0 / a + d * a / g + q * D
    out[2] = r - d * b / g
    out[3] = 1.0 / d + g - d / (q * q) + a * D * d / q
    out[4] = -b + r / (q * q) - a * D * r / q
    return out


def nig_loglik(y, a, b, d, m, nbins: int = 128, threads: int = 8):
    """(sum log p, d/da, d/db, d/dd, d/dm) and the sums of |terms| (for tolerances)."""
    t = nig_terms(y, a, b, d, m, nbins, threads)
    return (np.array([math.fsum(row) for row in t]),
            np.array([math.fsum(np.abs(row)) for row in t]))
