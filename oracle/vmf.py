"""oracle.vmf -- TEST INFRASTRUCTURE ONLY.

Plain von Mises-Fisher estimators of PAPER.md §6.3 (lines 663-693), float64
numpy / math.fsum, with the Bessel values from the binary128 oracle
(``oracle.log_iv``).  Nothing here is shared with the CUDA path.

* mean_direction   -- Eq. (mean direction estimate), lines 671-673:
                      mu = xbar / Rbar, xbar = mean of rows, Rbar = ||xbar||_2.
* a_p              -- A_p(kappa) = I_{p/2}(kappa) / I_{p/2-1}(kappa), line 677.
* kappa_estimates  -- Eq. (kappa estimates), lines 676-680 (Sra 2012):
                      kappa0 = Rbar (p - Rbar^2) / (1 - Rbar^2),
                      F(k) = k - (A_p(k) - Rbar) / (1 - A_p(k)^2 - (p-1)/k A_p(k)),
                      kappa1 = F(kappa0), kappa2 = F(kappa1).
* log_likelihood   -- lines 685-689, per-sample mean; with mu the estimate
                      above, mean(mu^T x_i) = Rbar.
* kappa_mle        -- the maximiser of log_likelihood over kappa >= 0
                      (lines 684, 691).  d logLik / d kappa = Rbar - A_p(kappa)
                      (from I_nu' = I_{nu+1} + (nu/kappa) I_nu), A_p is strictly
                      increasing, so the maximiser is the unique root; the
                      oracle finds it by plain bisection to machine precision.

Pinned by tests/test_oracle_pins.py against the paper's Table 7 (lines
695-711) and by analytic identities (Langevin function for p=3).
"""
from __future__ import annotations

import math

import numpy as np

from . import log_iv


def mean_direction(X):
    """Eq. (mean direction estimate). Column sums with math.fsum (exact-rounded)."""
    X = np.asarray(X, dtype=np.float64)
    n, p = X.shape
    xbar = np.array([math.fsum(X[:, j]) for j in range(p)]) / n
    rbar = math.sqrt(math.fsum(xbar * xbar))
    if rbar == 0.0:
        raise ValueError("mean resultant is zero: mean direction undefined")
    return xbar / rbar, rbar, xbar


def mean_resultant_rows(X):
    """Rbar for a large sample: column sums in float64 by numpy's pairwise summation
    (a library primitive; used where math.fsum over every column is too slow)."""
    X = np.asarray(X)
    xbar = np.sum(X, axis=0, dtype=np.float64) / X.shape[0]
    return math.sqrt(math.fsum((xbar * xbar).tolist()))


def a_p(p, kappa):
    """A_p(kappa) = I_{p/2}(kappa)/I_{p/2-1}(kappa) (line 677), from binary128 logs."""
    kappa = float(kappa)
    if kappa == 0.0:
        return 0.0
    h1, l1 = log_iv(p / 2.0, kappa, with_lo=True)
    h0, l0 = log_iv(p / 2.0 - 1.0, kappa, with_lo=True)
    d = (_scalar(h1) - _scalar(h0)) + (_scalar(l1) - _scalar(l0))
    return math.exp(d)


def _scalar(a):
    """The one element of a length-1 result array (marshalling only)."""
    return float(np.asarray(a).reshape(-1)[0])


def newton_F(p, rbar, kappa):
    """F(kappa) of Eq. (kappa estimates)."""
    A = a_p(p, kappa)
    return kappa - (A - rbar) / (1.0 - A * A - (p - 1.0) / kappa * A)


def kappa_estimates(p, rbar):
    """(kappa0, kappa1, kappa2) of Eq. (kappa estimates)."""
    if not (0.0 < rbar < 1.0):
        raise ValueError("Rbar must lie in (0, 1)")
    k0 = rbar * (p - rbar * rbar) / (1.0 - rbar * rbar)
    k1 = newton_F(p, rbar, k0)
    k2 = newton_F(p, rbar, k1)
    return k0, k1, k2


def log_likelihood(p, rbar, kappa):
    """Mean log-likelihood (lines 685-689) with mean(mu^T x_i) = Rbar."""
    lI = _scalar(log_iv(p / 2.0 - 1.0, kappa))
    return (p / 2.0 - 1.0) * math.log(kappa) - (p / 2.0) * math.log(2.0 * math.pi) - lI + kappa * rbar


def kappa_mle(p, rbar):
    """Root of Rbar - A_p(kappa) by bisection (maximiser of the log-likelihood)."""
    k0 = rbar * (p - rbar * rbar) / (1.0 - rbar * rbar)
    lo, hi = 0.0, max(1.0, 2.0 * k0)
    while a_p(p, hi) < rbar:
        lo, hi = hi, 2.0 * hi
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mid == lo or mid == hi:
            break
        if a_p(p, mid) < rbar:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def fit(X):
    """Full fit of a sample: mu, Rbar, (kappa0, kappa1, kappa2), kappa_mle, logLik(kappa_mle)."""
    X = np.asarray(X, dtype=np.float64)
    p = X.shape[1]
    mu, rbar, xbar = mean_direction(X)
    k0, k1, k2 = kappa_estimates(p, rbar)
    km = kappa_mle(p, rbar)
    return dict(mu=mu, rbar=rbar, xbar=xbar, kappa0=k0, kappa1=k1, kappa2=k2,
                kappa_mle=km, loglik=log_likelihood(p, rbar, km))
