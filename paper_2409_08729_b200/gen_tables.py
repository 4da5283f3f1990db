"""Generate the constant tables the CUDA kernels need (product code, host side).

Run as ``python -m paper_2409_08729_b200.gen_tables`` (``build()`` does it);
writes ``csrc/tables.h``.  Deterministic: regenerating yields identical bytes
(tests/test_tables.py checks that the committed header is current).

* u_k(t), k = 0..13 -- Debye polynomials of PAPER.md Eqs. (u0)/(uk)
  (lines 218-222): u_0 = 1,
      u_{k+1}(t) = (t^2 - t^4)/2 * u_k'(t) + 1/8 * int_0^t (1 - 5 s^2) u_k(s) ds,
  computed in exact rational arithmetic (fractions.Fraction).  u_k(t) has the
  monomials t^k, t^{k+2}, ..., t^{3k}; we store P_k with u_k(t) = t^k P_k(t^2).
  The paper found u_1..u_6 in DLMF 10.41(ii) and computed u_7..u_13 itself
  (line 223); the recurrence produces all of them.

* 1/Gamma(1+z) Taylor coefficients -- used by the K fallback (Temme's series,
  DESIGN.md §K-fallback), computed with mpmath at 60 digits.

* f64 log / exp tables of csrc/fastmath.cuh and the IEEE high words of the
  dispatch thresholds.
"""
from __future__ import annotations

import os
from fractions import Fraction

KMAX = 13


def uk_polynomials(kmax: int = KMAX):
    """Exact u_k(t) as dicts {power: Fraction} for k = 0..kmax."""
    polys = [{0: Fraction(1)}]
    for k in range(kmax):
        u = polys[-1]
        nxt: dict[int, Fraction] = {}
        # (t^2 - t^4)/2 * u'(t)
        for pw, c in u.items():
            if pw == 0:
                continue
            d = c * pw                      # coefficient of t^(pw-1)
            nxt[pw + 1] = nxt.get(pw + 1, Fraction(0)) + d / 2
            nxt[pw + 3] = nxt.get(pw + 3, Fraction(0)) - d / 2
        # 1/8 * int_0^t (1 - 5 s^2) u(s) ds
        for pw, c in u.items():
            nxt[pw + 1] = nxt.get(pw + 1, Fraction(0)) + c / (8 * (pw + 1))
            nxt[pw + 3] = nxt.get(pw + 3, Fraction(0)) - 5 * c / (8 * (pw + 3))
        polys.append({p: c for p, c in nxt.items() if c != 0})
    return polys


def uk_P_coeffs(kmax: int = KMAX):
    """P_k coefficients (ascending powers of t^2) with u_k(t) = t^k P_k(t^2)."""
    out = []
    for k, u in enumerate(uk_polynomials(kmax)):
        assert all((p - k) % 2 == 0 and k <= p <= 3 * k for p in u), (k, u)
        out.append([u.get(k + 2 * j, Fraction(0)) for j in range(k + 1)])
    return out


def rgamma_taylor(n: int = 28):
    """Taylor coefficients c_j of 1/Gamma(1+z) = sum_j c_j z^j (mpmath, 60 digits)."""
    import mpmath
    mpmath.mp.dps = 60
    return [float(c) for c in mpmath.taylor(lambda z: mpmath.rgamma(1 + z), 0, n - 1)]


ETA_TERMS = 14


def eta_root_taylor(nterms: int = ETA_TERMS):
    """Root z0 of eta(z) = sqrt(1+z^2) + log(z/(1+sqrt(1+z^2))) (the Laplace limit
    constant) as a double-double, and the Taylor coefficients c_1..c_n of eta
    around z0 (mpmath, 60 digits).  Used to evaluate v*eta without cancellation
    where eta ~ 0."""
    import mpmath
    mpmath.mp.dps = 60
    eta = lambda z: mpmath.sqrt(1 + z * z) + mpmath.log(z / (1 + mpmath.sqrt(1 + z * z)))
    z0 = mpmath.findroot(eta, mpmath.mpf("0.66"))
    hi = float(z0)
    lo = float(z0 - mpmath.mpf(hi))
    c = mpmath.taylor(eta, z0, nterms)
    return hi, lo, [float(ci) for ci in c[1:]]


# Table-driven f64 log/exp of csrc/fastmath.cuh.
LOG_TAB_BITS = 8
LOG_HI_OFF = 0x3FE6A09E      # high word of sqrt(1/2): mantissas are reduced to [sqrt(1/2), sqrt(2))
EXP_TAB_N = 64


def log_table():
    """Entry i covers the high words [OFF + i*2^12, OFF + (i+1)*2^12) of a number in
    [sqrt(1/2), sqrt(2)); invc_i = 1/(bucket centre) rounded to double and
    -log(invc_i) split into hi + lo (mpmath, 60 digits).  The bucket holding 1.0
    gets invc = 1 exactly so log(1 + r) keeps full relative accuracy near 1."""
    import struct

    import mpmath
    mpmath.mp.dps = 60

    def hw2d(h):
        return struct.unpack("<d", struct.pack("<Q", (h & 0xFFFFFFFF) << 32))[0]
    rows = []
    one_bucket = (0x3FF00000 - LOG_HI_OFF) >> (20 - LOG_TAB_BITS)
    for i in range(1 << LOG_TAB_BITS):
        lo = hw2d(LOG_HI_OFF + (i << (20 - LOG_TAB_BITS)))
        hi = hw2d(LOG_HI_OFF + ((i + 1) << (20 - LOG_TAB_BITS)))
        invc = 1.0 if i == one_bucket else float(2 / (mpmath.mpf(lo) + mpmath.mpf(hi)))
        t = -mpmath.log(mpmath.mpf(invc))
        th = float(t)
        tl = float(t - mpmath.mpf(th))
        rows.append((invc, th, tl))
    return rows


def exp_table(n: int = EXP_TAB_N):
    """2^(j/n), j = 0..n-1, as hi + lo (mpmath, 60 digits)."""
    import mpmath
    mpmath.mp.dps = 60
    out = []
    for j in range(n):
        t = mpmath.power(2, mpmath.mpf(j) / n)
        h = float(t)
        out.append((h, float(t - mpmath.mpf(h))))
    return out


# Dispatch thresholds as IEEE high words (csrc/bessel_math.cuh select_*):
# "a > C" is decided as hi(a) > HW(C), i.e. a > C' with C' the largest double
# sharing C's high word (C' - C < 2^-20 C; reading R3).
THRESHOLDS = {
    "X30": 30.0, "V15": 15.3919, "X59": 59.6925, "X19": 19.6931, "V07": 0.7, "V12": 12.6964,
    "X8": 8.0, "X2": 2.0, "X1E30": 1e30,
    "LO": 1e-140, "HI": 1e140,
    # f32 operating range (R13): every fast-path intermediate of the
    # float kernels (v^2 + x^2, 1/x, x/(v + rho), x^2/4) stays a normal float
    "LO32": 1e-18, "HI32": 1e18,
}


def u_term_thresholds(kmin: int = 3, kmax: int = KMAX - 1, bits: int = 56):
    """rho_K (integer, rounded up) from which K U-terms suffice (R12).

    The first omitted term of the U_K sum is P_{K+1}(t^2) w^{K+1} with w = 1/rho,
    rho = sqrt(v^2 + x^2) and |P_{K+1}| <= M_{K+1} := max over t^2 in [0, 1] (a
    fine grid plus the endpoints; the maximum sits at t^2 = 0), so it is
    <= 2^-bits once rho >= (M_{K+1} 2^bits)^(1/(K+1)).
    """
    import math
    P = uk_P_coeffs(kmax + 1)
    out = {}
    for K in range(kmin, kmax + 1):
        c = [float(a) for a in P[K + 1]]
        M = max(abs(sum(cj * (i / 4096.0) ** j for j, cj in enumerate(c))) for i in range(4097))
        out[K] = math.ceil((M * 2.0 ** bits) ** (1.0 / (K + 1)))
    return out


def f32_down_bits(c: float) -> int:
    """Bits of the largest float32 <= c (c > 0)."""
    import struct
    import numpy as np
    f = np.float32(c)
    if float(f) > c:
        f = np.nextafter(f, np.float32(0))
    return struct.unpack("<I", struct.pack("<f", float(f)))[0]


def hiword(c: float) -> int:
    import struct
    return struct.unpack("<Q", struct.pack("<d", c))[0] >> 32


SINPI_NT = 12


def sinpi_taylor(n: int = SINPI_NT):
    """c_k with sin(pi z) / (pi z) = sum_k c_k z^(2k), c_k = (-1)^k pi^(2k) / (2k+1)!
    (mpmath, 60 digits); 12 terms give 2^-60 for |z| <= 1/2."""
    import mpmath
    mpmath.mp.dps = 60
    return [float((-1) ** k * mpmath.pi ** (2 * k) / mpmath.factorial(2 * k + 1)) for k in range(n)]


def render() -> str:
    lines = [
        "// GENERATED by paper_2409_08729_b200/gen_tables.py -- do not edit.",
        "#pragma once",
        "",
        f"#define B200_UK_KMAX {KMAX}",
        "// u_k(t) = t^k * sum_j UK_P[k][j] * t^(2j)   (PAPER.md Eqs. (u0),(uk), lines 218-222)",
        "// row k holds k+1 coefficients; rows are packed with offsets UK_OFF[k].",
    ]
    P = uk_P_coeffs()
    flat, offs = [], []
    for row in P:
        offs.append(len(flat))
        flat.extend(row)
    lines.append("static const int UK_OFF[%d] = {%s};" % (len(offs), ", ".join(map(str, offs))))
    lines.append("#define B200_UK_NCOEF %d" % len(flat))
    lines.append("#define B200_UK_TABLE_INIT { \\")
    for k, row in enumerate(P):
        lines.append("    /* k=%2d */ %s, \\" % (k, ", ".join("%.17e" % float(c) for c in row)))
    lines.append("}")
    rg = rgamma_taylor()
    lines.append("")
    lines.append("// 1/Gamma(1+z) = sum_j RGAMMA_TAYLOR[j] z^j  (|z| <= 1/2 use), mpmath 60 digits")
    lines.append("#define B200_RGAMMA_NT %d" % len(rg))
    lines.append("#define B200_RGAMMA_INIT { %s }" % ", ".join("%.17e" % c for c in rg))
    lines.append("")
    lines.append("// 1/k, k = 0..400 (entry 0 unused)")
    lines.append("#define B200_INV_INIT { 0.0, %s }" % ", ".join("%.17e" % (1.0 / k) for k in range(1, 401)))
    import math
    from fractions import Fraction
    lines.append("// 1/k! for k = 0..30 (correctly rounded)")
    lines.append("#define B200_INVFACT_INIT { %s }" % ", ".join(
        "%.17e" % float(Fraction(1, math.factorial(k))) for k in range(0, 31)))
    lines.append("")
    lines.append("// f64 log table (csrc/fastmath.cuh): {1/c_i, -log(1/c_i) hi, lo, 0}, i = 0..%d" % ((1 << LOG_TAB_BITS) - 1))
    lines.append("#define B200_LOG_TAB_BITS %d" % LOG_TAB_BITS)
    lines.append("#define B200_LOG_HI_OFF 0x%08X" % LOG_HI_OFF)
    lines.append("#define B200_LOGTAB_INIT_STRUCT { %s }" % ", ".join(
        "{%.17e, %.17e, %.17e, 0.0}" % r for r in log_table()))
    lines.append("// f64 exp table: 2^(j/%d) hi, lo" % EXP_TAB_N)
    lines.append("#define B200_EXP_TAB_N %d" % EXP_TAB_N)
    lines.append("#define B200_EXPTAB_INIT_STRUCT { %s }" % ", ".join("{%.17e, %.17e}" % r for r in exp_table()))
    lines.append("")
    lines.append("// sin(pi z)/(pi z) = sum_k SINPI[k] z^(2k) (|z| <= 1/2), mpmath 60 digits")
    lines.append("#define B200_SINPI_NT %d" % SINPI_NT)
    lines.append("#define B200_SINPI_INIT { %s }" % ", ".join("%.17e" % c for c in sinpi_taylor()))
    lines.append("")
    lines.append("// dispatch thresholds: IEEE high words (gen_tables.THRESHOLDS)")
    for k, c in THRESHOLDS.items():
        lines.append("#define B200_HW_%s 0x%08Xu   // %r" % (k, hiword(c), c))
    lines.append("// f32 dispatch keys: float bit patterns (non-negative floats: bit order = value")
    lines.append("// order).  \"a > C\" is bits(a) > bits(C_dn), C_dn = the largest float <= C")
    lines.append("// (exact for float a); \"a >= rho_K\" is bits(a) >= bits(rho_K) (integers)")
    for k, c in THRESHOLDS.items():
        if k in ("LO", "HI"):
            continue                      # the f64 range; f32 uses LO32 / HI32
        lines.append("#define B200_F32_%s 0x%08Xu   // %r" % (k, f32_down_bits(c), c))
    for K, r in u_term_thresholds().items():
        lines.append("#define B200_F32_RHO_K%d 0x%08Xu   // %d" % (K, f32_down_bits(float(r)), r))
    lines.append("// f32 U bins: rho from which K terms leave a first omitted term <= 2^-28 (R17),")
    lines.append("// float bits; the f32 kernels use K = 2 / 3 / 5 / 9")
    for K, r in u_term_thresholds(kmin=1, kmax=12, bits=28).items():
        lines.append("#define B200_F32U_RHO_K%d 0x%08Xu   // %d" % (K, f32_down_bits(float(r)), r))
    lines.append("// rho from which K U-terms leave a first omitted term <= 2^-56 (R12):")
    lines.append("// B200_HW_RHO_K<K> = high word of that (integer) rho")
    for K, r in u_term_thresholds().items():
        lines.append("#define B200_HW_RHO_K%d 0x%08Xu   // %d" % (K, hiword(float(r)), r))
    lines.append("")
    hi, lo, ce = eta_root_taylor()
    lines.append("// eta(z) = sqrt(1+z^2) + log(z/(1+sqrt(1+z^2))): root z0 = HI + LO and")
    lines.append("// eta(z0 + d) = sum_{k=1..n} ETA_TAYLOR[k-1] d^k  (mpmath, 60 digits)")
    lines.append("#define B200_ETA_Z0_HI %.17e" % hi)
    lines.append("#define B200_ETA_Z0_LO %.17e" % lo)
    import numpy as np
    hf = float(np.float32(hi))
    lf = float(np.float32((hi - hf) + lo))
    lines.append("#define B200_ETA_Z0_HI_F %.9ef" % hf)
    lines.append("#define B200_ETA_Z0_LO_F %.9ef" % lf)
    lines.append("#define B200_ETA_NT %d" % len(ce))
    lines.append("#define B200_ETA_TAYLOR_INIT { %s }" % ", ".join("%.17e" % c for c in ce))
    lines.append("")
    return "\n".join(lines)


def write(path: str | None = None) -> str:
    path = path or os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "tables.h")
    txt = render()
    old = open(path).read() if os.path.exists(path) else None
    if old != txt:
        with open(path, "w") as f:
            f.write(txt)
    return path


if __name__ == "__main__":
    print(write())
