/*
 * bessel_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for log I_v(x) and log K_v(x),
 * evaluated in IEEE binary128 (__float128, libquadmath; 113-bit mantissa,
 * unit roundoff 9.6e-35).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path under
 * paper_2409_08729_b200/ and never calls it.
 *
 * Every function here is the PLAIN DEFINITION written out, not the paper's
 * approximation scheme:
 *
 *   oracle_log_iv -- the power series PAPER.md §3.1 Eq. (Iv infinite series)
 *                    (lines 126-128), terms generated with the recurrence of
 *                    Eqs. (ak recurrence base)/(ak recurrence) (lines 146-150),
 *                    summed to full binary128 precision (no truncation
 *                    heuristic: we stop only once the remaining tail is
 *                    provably below 2^-116 of the partial sum).  Corollary 1
 *                    (line 131-134) guarantees convergence for all inputs.
 *                    Overflow is avoided by an explicit power-of-two scale
 *                    counter, which is bookkeeping, not arithmetic.
 *
 *   oracle_log_kv -- K_v(x) is defined in PAPER.md §3 (lines 104-112) as the
 *                    solution of Eq. (modified bessel differential equation)
 *                    that diverges at 0.  We evaluate the standard integral
 *                    representation  K_v(x) = int_0^inf exp(-x cosh t) cosh(vt) dt
 *                    (DLMF 10.32.9), deliberately NOT the paper's
 *                    Eq. (log Kv integral) (line 251), so that oracle and
 *                    method do not share a formula.  Written as
 *                    1/2 int_{-inf}^{inf} exp(v t - x cosh t) dt and computed
 *                    with the trapezoidal rule (exponentially convergent for
 *                    this entire, doubly-exponentially decaying integrand),
 *                    halving the step until two successive sums agree to
 *                    1e-26 relative (ten orders below float64 resolution).
 *
 * Both return the value split as hi + lo (two doubles) so that callers can
 * form identities (Wronskian, recurrences) without losing the extra precision.
 *
 * Pins (tests/test_oracle_pins.py, -m "not gpu"): closed forms for
 * half-integer orders (PAPER.md never prints values; the closed forms
 * I_{1/2}(x)=sqrt(2/(pi x)) sinh x, K_{1/2}(x)=sqrt(pi/(2x)) e^-x are named in
 * BASELINE.json's north_star), the Wronskian I_v K_{v+1} + I_{v+1} K_v = 1/x,
 * the three-term recurrences, mpmath.besseli/besselk and scipy.special.ive/kve
 * as independent library routines, and the paper's Table 7 (lines 695-711)
 * through the vMF oracle.
 */
#include <quadmath.h>
#include <math.h>
#include <stdint.h>

#define EXPORT __attribute__((visibility("default")))

typedef __float128 q_t;

static const q_t Q_LN2 = 0.6931471805599453094172321214581765680755Q;

static void split_q(q_t v, double *hi, double *lo) {
    double h = (double)v;
    *hi = h;
    if (isinf(h) || isnan(h)) { *lo = 0.0; return; }
    *lo = (double)(v - (q_t)h);
}

/* ------------------------------------------------------------------------- */
/* log I_v(x), v >= 0, x >= 0 : direct series, PAPER.md Eq. (Iv infinite series)
 *   I_v(x) = (x/2)^v sum_k (x^2/4)^k / (k! Gamma(k+v+1))
 * with a_0 = 1/Gamma(v+1), a_{k+1} = a_k x^2 / (4 (k+1)(k+v+1)).
 * We sum b_k = a_k / a_0 (b_0 = 1) and return
 *   log I = v log(x/2) - lgamma(v+1) + log(sum_k b_k).
 */
static q_t log_iv_q(q_t v, q_t x) {
    if (x == 0) return (v == 0) ? (q_t)0 : -HUGE_VALQ;
    const q_t q = x * x / 4;
    /* peak of b_k: (k+1)(k+v+1) <= q  (Eq. (K)) */
    q_t b = 1, S = 1;
    int64_t scale = 0;               /* true sum = S * 2^scale            */
    const q_t BIG = 0x1p+8000Q, INV_BIG = 0x1p-8000Q;
    for (int64_t k = 0;; ++k) {
        q_t kk = (q_t)k;
        q_t r = q / ((kk + 1) * (kk + v + 1));   /* b_{k+1}/b_k */
        b = b * r;
        S = S + b;
        if (S > BIG) { S *= INV_BIG; b *= INV_BIG; scale += 8000; }
        /* past the peak, ratios are < 1 and decreasing, so the tail after
           this term is <= b r/(1-r); stop once that is negligible. */
        if (r < 0.5Q && b <= S * 0x1p-118Q) break;
        if (k > 100000000) break;   /* unreachable for the supported domain */
    }
    return v * logq(x / 2) - lgammaq(v + 1) + logq(S) + (q_t)scale * Q_LN2;
}

/* ------------------------------------------------------------------------- */
/* log K_v(x), x > 0: K_v(x) = 1/2 int_R exp(phi(t)) dt, phi(t) = v t - x cosh t
 * (DLMF 10.32.9).  phi is strictly concave with maximum at t* = asinh(v/x).
 */
static q_t phi_q(q_t v, q_t x, q_t t) { return v * t - x * coshq(t); }

static q_t log_kv_q(q_t v, q_t x) {
    if (x <= 0) return HUGE_VALQ;    /* pole at x = 0 */
    if (v < 0) v = -v;               /* K_{-v} = K_v */
    const q_t ts = asinhq(v / x);
    const q_t ps = phi_q(v, x, ts);
    const q_t DROP = 95;             /* exp(-95) ~ 5e-42 << 2^-113 */
    /* bracket the window where phi - ps >= -DROP (concavity => interval) */
    q_t dr = 1e-3Q, dl = 1e-3Q;
    while (phi_q(v, x, ts + dr) - ps > -DROP) dr *= 2;
    while (phi_q(v, x, ts - dl) - ps > -DROP) dl *= 2;
    const q_t lo = ts - dl, hi = ts + dr;
    /* trapezoid on the grid t = ts + j h, j in [-J_l, J_r]; the endpoints'
       contribution is < exp(-DROP) relative and is ignored.  Halve h until
       converged; each level reuses the previous sum (new midpoints only). */
    int64_t n = 64;
    q_t h = (hi - lo) / n;
    q_t sum = 0;
    for (int64_t j = 0; j <= n; ++j) sum += expq(phi_q(v, x, lo + j * h) - ps);
    q_t est = sum * h;
    for (int level = 0; level < 30; ++level) {
        q_t add = 0;
        for (int64_t j = 0; j < n; ++j) add += expq(phi_q(v, x, lo + (j + 0.5Q) * h) - ps);
        sum += add;
        n *= 2;
        h *= 0.5Q;
        q_t nest = sum * h;
        q_t diff = fabsq(nest - est);
        est = nest;
        /* the integrand itself carries rounding noise ~ eps_q * |v t| + |x cosh t|
           (up to ~1e-28 relative for v, x ~ 1e5), so converge to 1e-26: ten
           orders of magnitude below float64 resolution. */
        if (level >= 2 && diff <= est * 1e-26Q) break;
    }
    return -Q_LN2 + ps + logq(est);
}

/* ------------------------------------------------------------------------- */
/* C ABI (ctypes).  All arrays are host memory; n elements. */
EXPORT void oracle_log_iv(const double *v, const double *x, double *hi, double *lo, int64_t n) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i) split_q(log_iv_q((q_t)v[i], (q_t)x[i]), &hi[i], &lo[i]);
}

EXPORT void oracle_log_kv(const double *v, const double *x, double *hi, double *lo, int64_t n) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i) split_q(log_kv_q((q_t)v[i], (q_t)x[i]), &hi[i], &lo[i]);
}

/* Serial variants: used by bench.py's cpu_baseline so the thread count is explicit. */
EXPORT void oracle_log_iv_serial(const double *v, const double *x, double *hi, double *lo, int64_t n) {
    for (int64_t i = 0; i < n; ++i) split_q(log_iv_q((q_t)v[i], (q_t)x[i]), &hi[i], &lo[i]);
}

EXPORT void oracle_log_kv_serial(const double *v, const double *x, double *hi, double *lo, int64_t n) {
    for (int64_t i = 0; i < n; ++i) split_q(log_kv_q((q_t)v[i], (q_t)x[i]), &hi[i], &lo[i]);
}
