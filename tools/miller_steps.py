"""Truncation error of Miller's backward recurrence for r = I_{v+1}(x) / I_v(x).

Design tool for `log_ivkv_trap` (bessel_math.cuh): the fused
pass on 2 < x <= 30, v <= 12.7 starts y_{v+M+1} = 0, y_{v+M} = 1 and runs
y_{nu-1} = (2 nu / x) y_nu + y_{nu+1} down to nu = v + 1.  This script runs the
same recurrence in 80-bit long double for the kernel's step counts M(x) and
reports the largest relative deviation from a start at M = 120 (where the
start error is far below long-double resolution), plus the largest |y_v| (the
f32 path must stay below FLT_MAX).  CPU only; no kernel code involved.

  python tools/miller_steps.py
"""
import numpy as np

L = np.longdouble


def ratio(v, x, M):
    y1, y0 = L(0), L(1)
    v, x = L(v), L(x)
    for k in range(M, 0, -1):
        y1, y0 = y0, (2 * (v + k) / x) * y0 + y1
        if y0 > 1e300:
            y0 *= L(1e-300)
            y1 *= L(1e-300)
    return y1 / y0, y0


FORMULAS = {
    "f64": lambda x: int(min(12.0 + x, 20.0 + 0.55 * x)) + 1,
    "f32": lambda x: int(min(6.0 + x, 12.0 + 0.5 * x)) + 1,
}


def main():
    for name, Mf in FORMULAS.items():
        worst, where, ymax = 0.0, None, 0.0
        for x in np.arange(2.0, 30.0001, 0.1):
            M = Mf(x)
            for v in np.arange(0.0, 12.7001, 0.1):
                ref, _ = ratio(v, x, 120)
                r, y = ratio(v, x, M)
                e = float(abs(r - ref) / ref)
                ymax = max(ymax, float(y))
                if e > worst:
                    worst, where = e, (round(float(x), 2), round(float(v), 2), M)
        print(f"{name}: max truncation error of r {worst:.3g} at (x, v, M) = {where}; max |y_v| {ymax:.3g}")


if __name__ == "__main__":
    main()
