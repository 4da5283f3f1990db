"""Pins for the oracle (-m "not gpu").

The oracle (oracle/) is checked against things other than itself: closed
forms, the Wronskian, the three-term recurrences, independent library routines
(mpmath at 40 digits, scipy's exponentially scaled ive/kve), and the paper's
Table 7.  Each check is chosen so that a plausible slip in the oracle (dropped
term, wrong sign, off-by-one in the order, transposed v/x) fails at least one.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import scipy.special as sps

import oracle
from oracle import vmf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
mpmath.mp.dps = 50


def _mp(h, l):
    return mpmath.mpf(float(np.asarray(h).reshape(-1)[0])) + mpmath.mpf(float(np.asarray(l).reshape(-1)[0]))


# ---------------------------------------------------------------- closed forms
def _closed_forms():
    cf = json.load(open(os.path.join(GOLDEN, "closed_forms.json")))
    return cf["x_grid"]


@pytest.mark.parametrize("x", _closed_forms())
def test_half_integer_closed_forms(x):
    X = mpmath.mpf(x)
    pref_i = mpmath.sqrt(2 / (mpmath.pi * X))
    k12 = mpmath.sqrt(mpmath.pi / (2 * X)) * mpmath.exp(-X)
    ref = {
        ("i", 0.5): mpmath.log(pref_i * mpmath.sinh(X)),
        ("i", 1.5): mpmath.log(pref_i * (mpmath.cosh(X) - mpmath.sinh(X) / X)),
        ("k", 0.5): mpmath.log(k12),
        ("k", 1.5): mpmath.log(k12 * (1 + 1 / X)),
        ("k", 2.5): mpmath.log(k12 * (1 + 3 / X + 3 / X ** 2)),
        ("k", -1.5): mpmath.log(k12 * (1 + 1 / X)),     # evenness K_{-v} = K_v
    }
    for (fn, v), r in ref.items():
        f = oracle.log_iv if fn == "i" else oracle.log_kv
        h, l = f(v, x, with_lo=True)
        got = _mp(h, l)
        err = abs(got - r) / max(abs(r), 1)
        assert err < 1e-25, (fn, v, x, float(got), float(r), float(err))


def test_special_values():
    assert oracle.log_iv(0.0, 0.0) == 0.0                       # I_0(0) = 1
    assert oracle.log_iv(2.0, 0.0) == -np.inf                   # I_v(0) = 0, v > 0
    assert oracle.log_kv(1.0, 0.0) == np.inf                    # pole of K at 0
    # small-argument limit I_v(x) ~ (x/2)^v / Gamma(v+1)
    v, x = 3.7, 1e-8
    assert abs(oracle.log_iv(v, x) - (v * math.log(x / 2) - math.lgamma(v + 1))) < 1e-14


# -------------------------------------------------------- independent library
def _rand_points(n, vmax, xmin, xmax, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, vmax, n), rng.uniform(xmin, xmax, n)


def test_against_mpmath_small_region():
    v, x = _rand_points(40, 150.0, 0.05, 150.0, 1)
    hi = oracle.log_iv(v, x)
    hk = oracle.log_kv(v, x)
    for vi, xi, a, b in zip(v, x, hi, hk):
        ri = mpmath.log(mpmath.besseli(vi, xi))
        rk = mpmath.log(mpmath.besselk(vi, xi))
        assert float(abs(a - ri) / max(abs(ri), 1)) < 4e-16
        assert float(abs(b - rk) / max(abs(rk), 1)) < 4e-16


def test_against_mpmath_large_points():
    pts = [(0.0, 700.0), (1.0, 1500.0), (200.0, 10.0), (1000.0, 1000.0),
           (150.0, 4000.0), (4000.0, 150.0), (12.6, 0.001), (99.5, 0.1)]
    for v, x in pts:
        ri = mpmath.log(mpmath.besseli(v, x))
        rk = mpmath.log(mpmath.besselk(v, x))
        a, b = oracle.log_iv(v, x)[0], oracle.log_kv(v, x)[0]
        assert float(abs(a - ri) / max(abs(ri), 1)) < 4e-16, (v, x)
        assert float(abs(b - rk) / max(abs(rk), 1)) < 4e-16, (v, x)


def test_against_scipy_scaled():
    # scipy's ive(v,x)=I_v(x) e^{-x}, kve(v,x)=K_v(x) e^{x} (Amos); ~1e-15 accurate here
    v, x = _rand_points(400, 50.0, 0.5, 500.0, 2)
    li = oracle.log_iv(v, x)
    lk = oracle.log_kv(v, x)
    si = np.log(sps.ive(v, x)) + x
    sk = np.log(sps.kve(v, x)) - x
    assert np.max(oracle.rel_err(si, li)) < 5e-14
    assert np.max(oracle.rel_err(sk, lk)) < 5e-14


# ----------------------------------------------------------------- identities
def _exact_order(v):
    """Round v to a multiple of 2^-30 so that v-1 and v+1 are exact in float64."""
    return float(np.round(v * 2.0 ** 30) / 2.0 ** 30)


def _wronskian_err(v, x):
    """|log(I_v K_{v+1} + I_{v+1} K_v) - (-log x)| evaluated at 50 digits."""
    v = _exact_order(v)
    a = _mp(*oracle.log_iv(v, x, with_lo=True)) + _mp(*oracle.log_kv(v + 1, x, with_lo=True))
    b = _mp(*oracle.log_iv(v + 1, x, with_lo=True)) + _mp(*oracle.log_kv(v, x, with_lo=True))
    m = max(a, b)
    s = m + mpmath.log(mpmath.exp(a - m) + mpmath.exp(b - m))
    ref = -mpmath.log(mpmath.mpf(x))
    return float(abs(s - ref) / max(abs(ref), 1))


def test_wronskian_wide_domain():
    rng = np.random.default_rng(3)
    lv = rng.uniform(math.log(1e-3), math.log(1e5), 60)
    lx = rng.uniform(math.log(1e-3), math.log(1e5), 60)
    for v, x in zip(np.exp(lv), np.exp(lx)):
        assert _wronskian_err(v, x) < 1e-24, (v, x)
    for v, x in [(0.0, 1e-3), (0.0, 1e5), (1e5, 1e5), (1e5, 1e-3), (10.0, 30.0)]:
        assert _wronskian_err(v, x) < 1e-24, (v, x)


def test_three_term_recurrences():
    # I_{v-1} - I_{v+1} = (2v/x) I_v ;  K_{v+1} - K_{v-1} = (2v/x) K_v   (DLMF 10.29.1)
    rng = np.random.default_rng(4)
    for v, x in zip(rng.uniform(1, 300, 30), np.exp(rng.uniform(math.log(0.01), math.log(3e4), 30))):
        v = _exact_order(v)
        Im = _mp(*oracle.log_iv(v - 1, x, with_lo=True))
        I0 = _mp(*oracle.log_iv(v, x, with_lo=True))
        Ip = _mp(*oracle.log_iv(v + 1, x, with_lo=True))
        lhs = mpmath.exp(Im - I0) - mpmath.exp(Ip - I0)
        assert abs(lhs - 2 * mpmath.mpf(v) / mpmath.mpf(x)) <= 1e-24 * max(mpmath.exp(Im - I0), 1), (v, x)
        Km = _mp(*oracle.log_kv(v - 1, x, with_lo=True))
        K0 = _mp(*oracle.log_kv(v, x, with_lo=True))
        Kp = _mp(*oracle.log_kv(v + 1, x, with_lo=True))
        lhs = mpmath.exp(Kp - K0) - mpmath.exp(Km - K0)
        assert abs(lhs - 2 * mpmath.mpf(v) / mpmath.mpf(x)) <= 1e-24 * max(mpmath.exp(Kp - K0), 1), (v, x)


def test_monotone_in_x():
    x = np.linspace(0.01, 150, 1000)
    for v in (0.0, 0.3, 7.0, 120.0):
        li = oracle.log_iv(np.full_like(x, v), x)
        lk = oracle.log_kv(np.full_like(x, v), x)
        assert np.all(np.diff(li) > 0)
        assert np.all(np.diff(lk) < 0)


# ---------------------------------------------------------------- vMF oracle
def test_vmf_table7():
    rows = json.load(open(os.path.join(GOLDEN, "vmf_table7.json")))["rows"]
    for r in rows:
        p = r["p"]
        rbar = vmf.a_p(p, r["kappa2"])
        k0, k1, k2 = vmf.kappa_estimates(p, rbar)
        tol = 1.5 * 10.0 ** (-r["digits"])      # two printed roundings
        assert abs(k0 - r["kappa0"]) <= tol, (p, k0)
        assert abs(k1 - r["kappa1"]) <= tol, (p, k1)
        assert abs(k2 - r["kappa2"]) <= tol, (p, k2)
        km = vmf.kappa_mle(p, rbar)
        assert abs(km - r["kappa2"]) / r["kappa2"] < 1e-10   # Table 7 caption: <= 3.87e-11


def test_vmf_langevin_p3():
    # A_3(k) = coth k - 1/k (I_{3/2}/I_{1/2})
    for k in (0.1, 2.0, 30.0, 700.0):
        assert abs(vmf.a_p(3, k) - (1 / math.tanh(k) - 1 / k)) < 1e-15
    # kappa0 closed form at p=3, Rbar=0.5 -> 11/6
    assert abs(vmf.kappa_estimates(3, 0.5)[0] - 11 / 6) < 1e-15


def test_vmf_mean_direction_and_gradient():
    mu, rbar, _ = vmf.mean_direction(np.array([[1.0, 0.0], [0.0, 1.0]]))
    assert abs(rbar - 1 / math.sqrt(2)) < 3e-16 and np.allclose(mu, [1 / math.sqrt(2)] * 2)
    with pytest.raises(ValueError):
        vmf.mean_direction(np.array([[1.0, 0.0], [-1.0, 0.0]]))
    # d logLik/dk = Rbar - A_p(k): central differences
    for p, rbar, k in [(64, 0.7, 50.0), (2048, 0.2, 400.0), (32768, 0.3, 1e4)]:
        h = k * 1e-6
        fd = (vmf.log_likelihood(p, rbar, k + h) - vmf.log_likelihood(p, rbar, k - h)) / (2 * h)
        an = rbar - vmf.a_p(p, k)
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)) + 1e-7


def test_vmf_loglik_p3_closed_form():
    """p = 3: I_{1/2}(k) = sqrt(2/(pi k)) sinh k, so C_3(k) = k / (4 pi sinh k) and the mean
    log-likelihood of PAPER.md §6.3 (lines 685-689, density normaliser lines 666-668) is
    log k - log(4 pi sinh k) + k Rbar.  Evaluated here at 50 digits with mpmath, independently
    of the oracle's series: a slip in the (p/2 - 1) log k, the (p/2) log 2 pi or the
    log I_{p/2-1} term fails it."""
    for rbar in (0.05, 0.5, 0.93):
        for k in (1e-3, 0.7, 3.0, 45.0, 600.0):
            K = mpmath.mpf(k)
            ref = mpmath.log(K) - mpmath.log(4 * mpmath.pi * mpmath.sinh(K)) + K * mpmath.mpf(rbar)
            got = vmf.log_likelihood(3, rbar, k)
            assert abs(got - float(ref)) <= 4e-15 * max(1.0, abs(float(ref))), (rbar, k, got, float(ref))


@pytest.mark.parametrize("p", [3, 64, 2048, 32768])
def test_vmf_loglik_uniform_limit(p):
    """kappa -> 0: f_p -> the uniform density on S^{p-1}, 1 / |S^{p-1}| = Gamma(p/2) / (2 pi^{p/2})
    (PAPER.md lines 666-668 with I_{p/2-1}(k) ~ (k/2)^{p/2-1} / Gamma(p/2)); p = 3 gives -log 4 pi."""
    k = 1e-9
    ref = math.lgamma(p / 2.0) - math.log(2.0) - (p / 2.0) * math.log(math.pi)
    got = vmf.log_likelihood(p, 0.3, k)          # k Rbar = 3e-10 and O(k^2) terms: below 1e-9
    assert abs(got - ref) <= 1e-9 * max(1.0, abs(ref)), (p, got, ref)
    if p == 3:
        assert abs(ref + math.log(4 * math.pi)) < 1e-15


# ------------------------------------------------------------- the parity yardstick
def test_rel_err_definition():
    """oracle.rel_err (R1): |got - ref| / max(|ref|, 1); NaN anywhere -> inf;
    infinities must match in sign; finite vs infinite -> inf."""
    inf, nan = np.inf, np.nan
    got = np.array([1.0, 0.0, 0.5 + 1e-14, 100.0 + 1e-11, -3.0, inf, -inf, inf, 2.0, nan, 1.0, inf, 0.0])
    ref = np.array([1.0, 0.0, 0.5, 100.0, 3.0, inf, -inf, -inf, inf, 1.0, nan, 7.0, 1e-300])
    e = oracle.rel_err(got, ref)
    assert e[0] == 0.0 and e[1] == 0.0                             # exact
    assert abs(e[2] - 1e-14) < 1e-17                               # |ref| < 1: absolute (the floor)
    assert abs(e[3] - 1e-13) < 1e-16                               # |ref| >= 1: relative
    assert e[4] == 2.0                                             # sign error
    assert e[5] == 0.0 and e[6] == 0.0                             # same infinities
    assert np.all(np.isinf(e[7:12]))                               # opposite infinities, inf vs finite, NaN
    assert e[12] == 1e-300
    assert oracle.rel_err(np.array([]), np.array([])).size == 0
    assert np.all(e >= 0)


def test_mean_resultant_rows_matches_fsum():
    """mean_resultant_rows (numpy pairwise column sums, used for the full-size GPU test) against
    mean_direction's math.fsum column sums (exact rounding), to 1e-15."""
    rng = np.random.default_rng(7)
    for n, d, c in ((500, 33, 0.4), (20000, 64, 0.05), (3, 2048, 1.0)):
        X = rng.normal(size=(n, d)) / math.sqrt(d)
        X[:, 0] += c
        X /= np.linalg.norm(X, axis=1, keepdims=True)
        _, rbar, _ = vmf.mean_direction(X)
        assert abs(vmf.mean_resultant_rows(X) - rbar) <= 1e-15, (n, d)
        assert abs(vmf.mean_resultant_rows(X.astype(np.float32)) -
                   vmf.mean_direction(X.astype(np.float32).astype(np.float64))[1]) <= 1e-15
