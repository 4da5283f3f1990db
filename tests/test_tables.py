"""Host logic of the CUDA path: the generated u_k(t) / 1/Gamma tables."""
from fractions import Fraction

import mpmath

from paper_2409_08729_b200 import gen_tables


def test_uk_hand_values():
    u = gen_tables.uk_polynomials()
    assert u[0] == {0: Fraction(1)}                                          # Eq. (u0)
    assert u[1] == {1: Fraction(3, 24), 3: Fraction(-5, 24)}                 # (3t - 5t^3)/24
    assert u[2] == {2: Fraction(81, 1152), 4: Fraction(-462, 1152), 6: Fraction(385, 1152)}
    # DLMF 10.41.10: u_3 = (30375 t^3 - 369603 t^5 + 765765 t^7 - 425425 t^9)/414720
    assert u[3] == {3: Fraction(30375, 414720), 5: Fraction(-369603, 414720),
                    7: Fraction(765765, 414720), 9: Fraction(-425425, 414720)}
    assert len(u) == 14 and max(u[13]) == 39 and min(u[13]) == 13


def test_uk_recurrence_identity():
    """u_{k+1} = (t^2 - t^4)/2 u_k' + 1/8 int_0^t (1 - 5 s^2) u_k -- checked numerically at t=0.37."""
    mpmath.mp.dps = 40
    u = gen_tables.uk_polynomials()
    t = mpmath.mpf("0.37")
    ev = lambda p, t: sum(mpmath.mpf(c.numerator) / c.denominator * t ** e for e, c in p.items())
    for k in range(13):
        d = mpmath.diff(lambda s: ev(u[k], s), t)
        integ = mpmath.quad(lambda s: (1 - 5 * s * s) * ev(u[k], s), [0, t])
        assert abs(ev(u[k + 1], t) - ((t ** 2 - t ** 4) / 2 * d + integ / 8)) < mpmath.mpf(10) ** -25


def test_uk_t1_stirling():
    """At t = 1, sum_k (-1)^k u_k(1)/v^k is the Stirling series of Gamma (DLMF 10.41.11 / 5.11.3):
    u_1(1) = -1/12, u_2(1) = 1/288."""
    u = gen_tables.uk_polynomials()
    assert sum(u[1].values()) == Fraction(-1, 12)
    assert sum(u[2].values()) == Fraction(1, 288)


def test_rgamma_taylor():
    c = gen_tables.rgamma_taylor()
    assert c[0] == 1.0 and abs(c[1] - 0.5772156649015329) < 1e-16
    z = 0.37
    assert abs(sum(cj * z ** j for j, cj in enumerate(c)) - float(mpmath.rgamma(1 + z))) < 1e-16


def test_generated_header_is_current():
    import os
    path = os.path.join(os.path.dirname(gen_tables.__file__), "csrc", "tables.h")
    assert open(path).read() == gen_tables.render()


def test_u_term_thresholds_are_the_tightest_integers_of_the_bound():
    # R12: rho_K is the smallest integer with M_{K+1} rho^-(K+1) <= 2^-56, where
    # M_{K+1} = max |P_{K+1}| on [0, 1] attained at t^2 = 0 (checked here in exact arithmetic)
    P = gen_tables.uk_P_coeffs(13)
    th = gen_tables.u_term_thresholds()
    for K, r in th.items():
        c = P[K + 1]
        M = abs(c[0])
        grid = [sum(cj * Fraction(i, 64) ** j for j, cj in enumerate(c)) for i in range(65)]
        assert max(abs(g) for g in grid) == M
        assert M * Fraction(2) ** 56 <= Fraction(r) ** (K + 1)
        assert M * Fraction(2) ** 56 > Fraction(r - 1) ** (K + 1)
    assert (th[4], th[6], th[8], th[9], th[10]) == (1749, 277, 107, 78, 61)


def test_miller_step_counts_in_kernel_source():
    """The fused fallback's Miller start M(x) (bessel_math.cuh, log_ivkv_trap),
    read from the kernel source, keeps the truncation error of r = I_{v+1}/I_v below
    2^-60 (f64) / 2^-30 (f32) on the band 1e-6 <= x <= 30, v <= 12.7.  Reference r: the
    same recurrence from M = 120 in long double, cross-checked against scipy's ive
    ratio (an independent routine) to 1e-13."""
    import os
    import re

    import numpy as np
    import scipy.special as sps

    src = open(os.path.join(os.path.dirname(gen_tables.__file__), "csrc", "bessel_math.cuh")).read()
    num = r"T\(([\d.]+)\)"
    # M(x) = the step count rounded up to a multiple of 4 (four steps per loop trip)
    m = re.search(r"const int M = \(\(sizeof\(T\) == 8 \? int\(fmin\(" + num + r" \+ x, fma\(" + num + r", x, "
                  + num + r"\)\)\) \+ 1\s*: int\(fmin\(" + num + r" \+ x, fma\(" + num + r", x, " + num
                  + r"\)\)\) \+ 1\) \+ 3\) & ~3;", src)
    assert m, "M(x) expression not found in log_ivkv_trap"
    a64, b64, c64, a32, b32, c32 = (float(g) for g in m.groups())
    L = np.longdouble

    def ratio(v, x, M):
        y1, y0 = L(0), L(1)
        for k in range(M, 0, -1):
            y1, y0 = y0, (2 * (L(v) + k) / L(x)) * y0 + y1
            if y0 > 1e300:
                y0, y1 = y0 * L(1e-300), y1 * L(1e-300)
        return y1 / y0

    xs = [1e-6, 1e-3, 0.3, 1.0, 2.0, 2.5, 4.9, 8.9, 13.0, 19.7, 25.0, 30.0]
    for x in xs:
        m64 = (int(min(a64 + x, b64 * x + c64)) + 1 + 3) & ~3
        m32 = (int(min(a32 + x, b32 * x + c32)) + 1 + 3) & ~3
        for v in (0.0, 0.5, 1.0, 4.2, 8.0, 12.69):
            ref = ratio(v, x, 120)
            if x >= 1e-3:
                assert abs(float(ref) - sps.ive(v + 1, x) / sps.ive(v, x)) <= 1e-13 * float(ref)
            assert float(abs(ratio(v, x, m64) - ref) / ref) < 2.0 ** -60, (x, v, m64)
            if x > 2:
                assert float(abs(ratio(v, x, m32) - ref) / ref) < 2.0 ** -30, (x, v, m32)
