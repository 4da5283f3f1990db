// bessel_math.cuh -- per-element device math for log I_v(x) / log K_v(x).
//
// PAPER.md = arXiv 2409.08729.  Every function cites the passage it follows.
// Templated on the arithmetic type T (double for the f64 path, float for the
// f32 path).  Nothing here allocates, synchronises or touches global memory.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "fastmath.cuh"
#include "tables.h"

namespace b200 {

// ---------------------------------------------------------------- constants
static __constant__ double c_uk_d[B200_UK_NCOEF] = B200_UK_TABLE_INIT;
static __constant__ float c_uk_f[B200_UK_NCOEF] = B200_UK_TABLE_INIT;
static __constant__ double c_rg_d[B200_RGAMMA_NT] = B200_RGAMMA_INIT;
static __constant__ float c_rg_f[B200_RGAMMA_NT] = B200_RGAMMA_INIT;
static __constant__ double c_eta_d[B200_ETA_NT] = B200_ETA_TAYLOR_INIT;
static __constant__ double c_sinpi_d[B200_SINPI_NT] = B200_SINPI_INIT;
static __constant__ float c_eta_f[B200_ETA_NT] = B200_ETA_TAYLOR_INIT;

template <typename T> struct Tr;
template <> struct Tr<double> {
    static constexpr double eps = 1.1102230246251565e-16;   // 2^-53
    static constexpr int rg_terms = 28;
    __device__ static double uk(int i) { return c_uk_d[i]; }
    __device__ static double rg(int i) { return c_rg_d[i]; }
};
template <> struct Tr<float> {
    static constexpr float eps = 5.9604645e-08f;             // 2^-24
    static constexpr int rg_terms = 12;
    __device__ static float uk(int i) { return c_uk_f[i]; }
    __device__ static float rg(int i) { return c_rg_f[i]; }
};

// Constants used on every element of the mu / U paths.  In constant memory: a
// double literal with a non-zero low word costs two UMOVs per use in SASS, a
// __constant__ operand one LDCU (two per LDCU.128).
enum : int { HC_INV2PI = 0, HC_PIO2, HC_LNPI, HC_ETA_HI, HC_ETA_BAND, HC_PI2, HC_N };
static __constant__ double c_hot_d[HC_N] = {0.5 / CUDART_PI, CUDART_PI / 2.0, 1.1447298858494002,
                                            B200_ETA_Z0_HI, 0.03, CUDART_PI * CUDART_PI};
// f32: the eta band is |z - z0| < 0.12 (f64: 0.03): outside it rho + v log(x/(v+rho)) cancels
// up to ~6x at 0.12 against ~17x at 0.04, and float rounding times that cancellation came
// within 5% of the 1e-5 bar; the 8-term Taylor series of eta (radius |z0 - i| ~ 1.2) is
// accurate to < 1e-8 on the wider band (profiles/r62/acc32.txt)
static __constant__ float c_hot_f[HC_N] = {float(0.5 / CUDART_PI), float(CUDART_PI / 2.0), 1.1447298858494002f,
                                           B200_ETA_Z0_HI_F, 0.12f, float(CUDART_PI * CUDART_PI)};
template <typename T>
__device__ __forceinline__ T hc(int i) {
    if constexpr (sizeof(T) == 8) return c_hot_d[i]; else return c_hot_f[i];
}

// 1/k for k = 1..400 (recurrences divide by the term index)
#define B200_NINV 400
static __constant__ double c_inv_d[B200_NINV + 1] = B200_INV_INIT;
static __constant__ float c_inv_f[B200_NINV + 1] = B200_INV_INIT;
template <typename T>
__device__ __forceinline__ T c_inv_k(int k) {
    if constexpr (sizeof(T) == 8) return c_inv_d[k]; else return c_inv_f[k];
}

// 1/k! for k = 0..30 (the mu series carries k! term_k, B200_MUFACT)
static __constant__ double c_invfact_d[31] = B200_INVFACT_INIT;
static __constant__ float c_invfact_f[31] = B200_INVFACT_INIT;
template <typename T>
__device__ __forceinline__ T c_invfact(int k) {
    if constexpr (sizeof(T) == 8) return c_invfact_d[k]; else return c_invfact_f[k];
}

// Overload helpers so templates pick the right precision.
__device__ __forceinline__ double d_lgamma(double a) { return lgamma(a); }
__device__ __forceinline__ float d_lgamma(float a) { return lgammaf(a); }

// ---------------------------------------------------------------- dispatch
// Algorithm 1 / Table 1 (lines 338-352), with the
// GPU branch set: "When running on a GPU the branches for the mu_3, U_4, U_6,
// U_9 expressions are removed" (line 384).  Predicates are strict
// inequalities with natural logarithms (reading R3), decided on the
// IEEE high words of v >= 0 and x > 0 (bit order = value order for
// non-negative doubles): "a > C" is hi(a) > HW(C), one 32-bit integer compare
// on the ALU pipe, which is the strict inequality against C' = the largest
// double with C's high word (C' - C < 2^-20 C, far inside the precision of
// the fitted Table 1 constants).  Both precisions dispatch on the double value,
// so the f32 and f64 paths choose identical methods.
enum : int { M_MU = 0, M_U13 = 1, M_FALLBACK = 2 };

__device__ __forceinline__ long long dbits(double a) { return __double_as_longlong(a); }
__device__ __forceinline__ uint32_t hiw(double a) { return uint32_t(__double2hiint(a)); }

// The curved mu edge [0.5113 log x + 0.7939 > log v] is decided with the
// hardware log2 (MUFU.LG2, fp32) and re-evaluated in double only inside a
// 1e-4 guard band (and beyond the fp32 range), so the result equals the
// double-precision predicate.
// log2 by MUFU.LG2 with denormals flushed (no range fix-up instructions): x > 59 here,
// and a v that flushes to 0 gives -inf, i.e. "mu" -- as the exact predicate does
__device__ __forceinline__ float lg2_ftz(float a) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ bool mu_edge(double v, double x, uint32_t hx) {
    if (hx <= B200_HW_X1E30) {
        const float lx = lg2_ftz(float(x)), lv = lg2_ftz(float(v));
        const float d = 0.5113f * lx + 1.14535832f - lv;   // 0.7939 / ln 2 = 1.14535832
        if (fabsf(d) > 1e-4f) return d > 0.0f;
    }
    return 0.5113 * log(x) + 0.7939 > log(v);
}

// v >= 0, x >= 0 (callers filter the rest); hv, hx = high words
__device__ __forceinline__ bool is_mu_hw(double v, double x, uint32_t hv, uint32_t hx) {
    bool mu = hx > B200_HW_X30 && hv <= B200_HW_V15;                        // x > 30 && v < 15.3919
    // x > 59.6925 && (v <= 0 || edge).  For x > 5.08 the edge implies v < x,
    // so v >= x (hv >= hx) settles it without the logs.
    if (!mu && hx > B200_HW_X59 && hv < hx) mu = (hv == 0) || mu_edge(v, x, hx);
    return mu;
}
__device__ __forceinline__ bool is_u_hw(uint32_t hv, uint32_t hx) {
    return (hx > B200_HW_X19 && hv > B200_HW_V07) || hv > B200_HW_V12;     // Table 1, U13 region
}
__device__ __forceinline__ int select_method_hw(double v, double x, uint32_t hv, uint32_t hx) {
    return is_mu_hw(v, x, hv, hx) ? M_MU : is_u_hw(hv, hx) ? M_U13 : M_FALLBACK;
}

__device__ __forceinline__ int select_method(double v, double x) {
    return select_method_hw(v, x, hiw(v), hiw(x));
}

// Number of terms of the mu_K expansion.  The paper uses K = 20 (Table 1);
// we allow the same recurrence up to K = 26 so the truncation error stays
// below fp64 resolution on the whole region (reading R5), and stop
// as soon as a term no longer changes the sum (past the initial growth of
// the terms, k >= 4), which for x >= 60 is after 8-15 terms.
constexpr int KMU = 26;
#ifndef B200_MUEO
#define B200_MUEO 0
#endif
#ifndef B200_SERIES_UNROLL
#define B200_SERIES_UNROLL 1  // 1: the f64 power series of log I, terms 1..48 written out (0: rolled)
#endif
#ifndef B200_TEMME_UNROLL
#define B200_TEMME_UNROLL 1   // 1: Temme's series, terms 1..20 written out (0: rolled loop)
#endif
#ifndef B200_MUF
#define B200_MUF 1
#endif
#ifndef B200_MU2U
#define B200_MU2U 0
#endif
#ifndef B200_MUFACT
#define B200_MUFACT 2
#endif

// Wide-range guard: the fast paths form 1/x, v^2 + x^2 and 1/rho, which stay
// normal for arguments below BIG; beyond it the same formulas run rescaled or
// through the CUDA library functions (never on the tested domain).
template <typename T> struct Big;
template <> struct Big<double> { static constexpr double v = 1e150; };
template <> struct Big<float> { static constexpr float v = 1e18f; };

// ---------------------------------------------------------------- mu_K
// Eq. (log Iv mu k) (line 203-205) / Eq. (log Kv mu k) (line 234-236):
//   log I ~ x - 1/2 log(2 pi x) + log|1 + sum_k (-1)^k prod_{j<=k}(mu-(2j-1)^2) / (k! (8x)^k)|
//   log K ~ 1/2 (log pi - log 2x) - x + log|1 + sum_k prod_{j<=k}(mu-(2j-1)^2) / (k! (8x)^k)|
// mu = 4 v^2.  Terms by the paper's recurrence ("the terms in the series can
// also be calculated recursively", line 208):
//   term_k = term_{k-1} * s (mu - (2k-1)^2) / (8 x k),  s = -1 (I), +1 (K),
// fully unrolled so (2k-1)^2 and 1/k are compile-time constants; the stop
// test runs every fourth term.
template <typename T, bool IS_K>
__device__ __forceinline__ T mu_series(T v, T rx) {
#if B200_MUFACT
    // T_k = k! term_k (see log_bessel_mu_ik): T_k = T_{k-1} (c mu - c (2k-1)^2) with
    // c = +-1/(8x), s = sum T_k / k! by FMA -- 3 FP64 operations per term, written out
    const T c = (IS_K ? T(0.125) : T(-0.125)) * rx;
    const T z = c * (T(4) * v * v);
    T tk = T(1), s = T(1);
#define B200_MU1_T(k)                                                         \
    {                                                                         \
        tk *= fma(c, T(-double((2 * (k) - 1) * (2 * (k) - 1))), z);          \
        s = fma(tk, c_invfact<T>(k), s);                                      \
    }
#define B200_MU1_STOP(k) if (fabs(tk) * c_invfact<T>(k) <= Tr<T>::eps * T(0.25) * fabs(s)) goto mu1_done;
    B200_MU1_T(1) B200_MU1_T(2) B200_MU1_T(3) B200_MU1_T(4) B200_MU1_STOP(4)
    B200_MU1_T(5) B200_MU1_T(6) B200_MU1_T(7) B200_MU1_T(8) B200_MU1_STOP(8)
    B200_MU1_T(9) B200_MU1_T(10) B200_MU1_T(11) B200_MU1_T(12) B200_MU1_STOP(12)
    B200_MU1_T(13) B200_MU1_T(14) B200_MU1_T(15) B200_MU1_T(16) B200_MU1_STOP(16)
    B200_MU1_T(17) B200_MU1_T(18) B200_MU1_T(19) B200_MU1_T(20) B200_MU1_STOP(20)
    B200_MU1_T(21) B200_MU1_T(22) B200_MU1_T(23) B200_MU1_T(24) B200_MU1_STOP(24)
    B200_MU1_T(25) B200_MU1_T(26)
#undef B200_MU1_T
#undef B200_MU1_STOP
mu1_done:
    return fabs(s);
#else
    const T mu = T(4) * v * v;
    const T c = (IS_K ? T(0.125) : T(-0.125)) * rx;
#if B200_MUF
    const T z = c * mu;                          // factor = fma(c, -(2k-1)^2, c mu) / k
#endif
    T term = T(1), s = T(1);
#pragma unroll
    for (int k = 1; k <= KMU; k += 4) {        // four terms per stop test
#pragma unroll
        for (int u = 0; u < 4 && k + u <= KMU; ++u) {
            const int kk = k + u;
            const T inv_k = c_inv_k<T>(kk);
#if B200_MUF
            term *= fma(c, T(-(2 * kk - 1) * (2 * kk - 1)), z) * inv_k;
#else
            term *= (mu - T((2 * kk - 1) * (2 * kk - 1))) * (c * inv_k);
#endif
            s += term;
        }
        if (k >= 4 && fabs(term) <= Tr<T>::eps * T(0.25) * fabs(s)) break;
    }
    return fabs(s);
#endif
}

// log I = x - 1/2 log(2 pi x) + log S = x + 1/2 log(S^2 / (2 pi x))  (one log)
template <typename T, bool IS_K, bool SAFE>
__device__ __forceinline__ T log_bessel_mu(T v, T x, uint32_t tab = logtab_addr()) {
    if (!SAFE || x < Big<T>::v) {
        const T rx = fm_rcp(x);
        const T S = mu_series<T, IS_K>(v, rx);
        const T c = IS_K ? hc<T>(HC_PIO2) : hc<T>(HC_INV2PI);
        return (IS_K ? -x : x) + T(0.5) * fm_log(S * S * rx * c, tab);
    }
    const T S = mu_series<T, IS_K>(v, T(1) / x);
    const T l2 = IS_K ? T(-0.22579135264472743) : T(1.8378770664093453);   // log(2/pi), log(2 pi)
    return (IS_K ? -x : x) + log(S) - T(0.5) * (l2 + log(x));
}

// log(1 + d) for the U-expansion sums S = 1 + d: |d| <= sum_k M_k / rho^k with
// rho = sqrt(v^2 + x^2), i.e. |d| < 0.0105 in the U13 region (rho >= 12.69),
// 1.6e-3 for U9 (rho >= 80), 4.5e-4 for U6, 7e-5 for U4 (R12 bounds).  The
// Taylor polynomial of degree NP leaves |d|^(NP+1)/(NP+1) < 2^-60: NP = 9, 6,
// 5, 4.  Replaces a full log of S (one table log per function saved).
#ifndef B200_L1P56
#define B200_L1P56 1
#endif
#if B200_L1P56
// |d|^(NP+1)/(NP+1) < 2^-56 (absolute error of log S, below the 1e-13 target by 1e3):
// |d| < 0.0105 (U13) -> 7, 3e-3 (U10, rho >= 61) -> 5, 1.2e-3 (U8) -> 5, 4.5e-4 (U6) -> 4
template <int KU> struct Log1pDeg { static constexpr int v = KU >= 13 ? 7 : KU >= 8 ? 5 : 4; };
#else
template <int KU> struct Log1pDeg { static constexpr int v = KU >= 13 ? 9 : KU >= 9 ? 6 : KU >= 6 ? 5 : 4; };
#endif
static __constant__ double c_l1p[10] = {0.0, 1.0, -1.0 / 2, 1.0 / 3, -1.0 / 4, 1.0 / 5, -1.0 / 6, 1.0 / 7,
                                        -1.0 / 8, 1.0 / 9};
#if B200_IMM
// 1/k, with the odd tails 1/5, 1/7, 1/9 (and 1/3 for the U6 bound |d| < 4.5e-4) as
// 21-bit immediates: their rounding (< 2.4e-7 relative) times |d|^k stays < 1e-17
template <int K, bool SHORT3>
__device__ __forceinline__ double l1p_coef() {
    return K == 1 ? 1.0 : K == 2 ? -0.5 : K == 3 ? (SHORT3 ? 0.33333325386047363 : c_l1p[3]) : K == 4 ? -0.25
         : K == 5 ? 0.20000004768371582 : K == 6 ? -0.16666662693023682 : K == 7 ? 0.14285719394683838
         : K == 8 ? -0.125 : 0.1111111044883728;
}
template <typename T, int NP, int K>
__device__ __forceinline__ T l1p_step(T p, T d) {
    if constexpr (K < 1) return p;
    else return l1p_step<T, NP, K - 1>(fma(p, d, T(l1p_coef<K, (NP <= 5)>())), d);
}
#endif
// f32: first omitted U term <= 2^-28 (R17) -> log1p degree N with |d|^(N+1)/(N+1) <= 2^-28:
// |d| < 4.6e-4 (K = 2, rho >= 270), 1.7e-3 (K = 3, rho >= 75), 5.3e-3 (K = 5, rho >= 24),
// 0.011 (K = 9, rho >= 12)
template <int KU> struct Log1pDeg32 { static constexpr int v = KU >= 9 ? 4 : KU >= 5 ? 3 : 2; };
template <typename T, int KU> struct L1PDeg { static constexpr int v = Log1pDeg<KU>::v; };
template <int KU> struct L1PDeg<float, KU> { static constexpr int v = Log1pDeg32<KU>::v; };

template <typename T, int NP>
__device__ __forceinline__ T log1p_small(T d) {
#if B200_IMM
    if constexpr (sizeof(T) == 8) {
        const T p = l1p_step<T, NP, NP - 1>(T(l1p_coef<NP, (NP <= 5)>()), d);
        return p * d;
    }
#endif
    T p = T(c_l1p[NP]);
#pragma unroll
    for (int k = NP - 1; k >= 1; --k) p = fma(p, d, T(c_l1p[k]));
    return p * d;
}

// ---------------------------------------------------------------- U_13
// Eq. (log Iv u k) (lines 211-215) / Eq. (log Kv u k) (lines 241-245):
//   x' = x/v, t = 1/sqrt(1+x'^2), eta = sqrt(1+x'^2) + log(x'/(1+sqrt(1+x'^2)))
//   log I ~ -1/2 log(2 pi v) + v eta - 1/4 log(1+x'^2) + log|1 + sum_k u_k(t)/v^k|
//   log K ~  1/2 log(pi/(2v)) - v eta - 1/4 log(1+x'^2) + log|1 + sum_k (-1)^k u_k(t)/v^k|
// u_k(t) = t^k P_k(t^2) (tables.h, generated from Eqs. (u0),(uk)).  With
// w = +-t/v the sum is w (P_1 + w (P_2 + ... + w P_13)).
//
// Evaluated through rho = sqrt(v^2 + x^2) = v sqrt(1+x'^2), one reciprocal
// square root y = 1/rho giving all of
//   t = v y,   t/v = y,   v sqrt(1+x'^2) = rho,   x'/(1+sqrt(1+x'^2)) = x/(v+rho),
//   -1/2 log(2 pi v) - 1/4 log(1+x'^2) = 1/2 log(y / (2 pi)),
// so log I = rho + v log(x/(v+rho)) + 1/2 log(S^2 y / (2 pi)): two logs, no
// division, no sqrt (the algebra is exact; only rounding differs).
template <typename T>
__device__ __forceinline__ T uk_row(int k, T t2) {
    // P_k(t2) by Horner, k+1 coefficients starting at UK_OFF[k]
    const int off = (k * (k + 1)) / 2;
#if B200_IMM
    if constexpr (sizeof(T) == 8) {
        // first step as a separate multiply and add: both take their constant as a
        // uniform-register operand, where fma(c_k, t2, c_k-1) needs one of the two
        // constants in a vector register (a per-thread constant-bank load)
        T p = __dadd_rn(__dmul_rn(t2, Tr<T>::uk(off + k)), Tr<T>::uk(off + k - 1));
#pragma unroll
        for (int j = k - 2; j >= 0; --j) p = fma(p, t2, Tr<T>::uk(off + j));
        return p;
    }
#endif
#if 1
    T p = Tr<T>::uk(off + k);
#pragma unroll
    for (int j = k - 1; j >= 0; --j) p = fma(p, t2, Tr<T>::uk(off + j));
    return p;
#endif
}

// v * eta(x/v).  Where eta ~ 0 (z = x/v near the Laplace limit constant
// z0 = 0.6627...) the two terms of eta cancel and plain arithmetic leaves
// ~v*eps absolute error.  There eta is evaluated from its
// Taylor series around z0 with d = z - z0 formed from z = x/v in two-word
// precision (the remainder x - z*v is exact by FMA; z - z0_hi is exact by
// Sterbenz), so v*eta keeps full relative accuracy.
template <typename T> struct EtaC;
template <> struct EtaC<double> {
    static constexpr double hi = B200_ETA_Z0_HI, lo = B200_ETA_Z0_LO;
    static constexpr int nt = B200_ETA_NT;
    __device__ static double c(int k) { return c_eta_d[k]; }
};
template <> struct EtaC<float> {
    static constexpr float hi = B200_ETA_Z0_HI_F, lo = B200_ETA_Z0_LO_F;
    static constexpr int nt = 8;
    __device__ static float c(int k) { return c_eta_f[k]; }
};

// vs, xs, rhos: v, x, rho scaled by the same power of two s; returns v*eta.
template <typename T, bool SAFE>
__device__ __forceinline__ T v_times_eta(T v, T x, T vs, T xs, T rhos, T rho, uint32_t tab = logtab_addr()) {
    // band test on z = x/v without a division: |x - z0 v| < 0.03 v
    if (fabs(fma(-hc<T>(HC_ETA_HI), v, x)) < hc<T>(HC_ETA_BAND) * v) {
        // 1/v by the MUFU-seeded reciprocal (<= 2 ulp): its error enters z = x/v but not
        // z + zlo, whose residual x - z v is exact by FMA (z + zlo = x/v to ~2^-100)
        const T rv = SAFE ? T(1) / v : fm_rcp(v);
        const T z = x * rv;
        const T zlo = fma(-z, v, x) * rv;
        const T d = (z - EtaC<T>::hi) + (zlo - EtaC<T>::lo);
        T p = EtaC<T>::c(EtaC<T>::nt - 1);
#pragma unroll
        for (int k = EtaC<T>::nt - 2; k >= 0; --k) p = fma(p, d, EtaC<T>::c(k));
        return v * (p * d);
    }
    if constexpr (SAFE) {
        // log(x/(v + rho)): the quotient underflows when x << v (subnormal x, huge v);
        // then take the difference of the logs of the (scaled, normal) operands
        const T den = vs + rhos;
        const T lq = xs >= T(1e-30) * den ? fm_log_wide(xs * fm_rcp(den)) : log(xs) - log(den);
        return fma(v, lq, rho);
    }
    const T q = xs * fm_rcp(vs + rhos);
    return fma(v, fm_log_acc(q, tab), rho);
}

// Number of U_K terms.  The paper's Table 1 fits regions for U4/U6/U9/U13 and
// the GPU version keeps only U13 to avoid warp divergence (line 384).  With
// the in-CTA binning divergence is gone, so fewer terms come back where rho is
// large, selected by an a-priori truncation bound instead of the fitted regions
// (R12): u_k(t) = t^k P_k(t^2) with sup_{t in [0,1]} |P_k| = P_k(0) =:
// M_k, and w = t/v = 1/sqrt(v^2+x^2), so the first omitted term of U_K is at
// most M_{K+1} w^{K+1} <= 2^-56 once sqrt(v^2+x^2) >= rho_K (tables.h
// B200_HW_RHO_K*: 277 for K=6, 107 for K=8, 61 for K=10).  Tested on
// max(v, x) <= sqrt(v^2+x^2): conservative, never fewer terms than the bound
// allows.  The bins (select_eval_hw) use K = KU_A/KU_B/KU_C/13.

template <typename T, bool IS_K, int KU, bool SAFE>
__device__ __forceinline__ T log_bessel_u(T v, T x, uint32_t tab = logtab_addr()) {
    // rescale by s = 2^-e, e = the binary exponent of max(v, x), where v^2 + x^2 could
    // overflow (wide-range guard): then max(vs, xs) is in [1, 2)
    const bool big = SAFE && fmax(v, x) >= Big<T>::v;
    const int e = big ? ilogb(fmax(v, x)) : 0;
    const T s = big ? T(scalbn(1.0, -e)) : T(1);
    const T ls = big ? T(-double(e) * 0.6931471805599453) : T(0);          // log s
    const T vs = v * s, xs = x * s;
    const T rho2 = fma(vs, vs, xs * xs);
    const T y = fm_rsqrt(rho2);                  // 1 / (s rho)
    const T rhos = rho2 * y;
    const T rho = big ? T(scalbn(double(rhos), e)) : rhos;
    const T t = vs * y;
    const T t2 = t * t;
    const T w = (IS_K ? -y : y) * s;             // +-t/v
    T acc = uk_row<T>(KU, t2);
#pragma unroll
    for (int k = KU - 1; k >= 1; --k) acc = fma(acc, w, uk_row<T>(k, t2));
    const T d = acc * w;                         // S - 1
    const T veta = v_times_eta<T, SAFE>(v, x, vs, xs, rhos, rho, tab);
    // log S + 1/2 log(y_true c) with y_true = s y
    const T c = IS_K ? hc<T>(HC_PIO2) : hc<T>(HC_INV2PI);
    const T tail = log1p_small<T, L1PDeg<T, KU>::v>(d) + T(0.5) * (fm_log(y * c, tab) + ls);
    return IS_K ? tail - veta : veta + tail;
}

// ---------------------------------------------------------------- fused I + K
// Both functions at the same (v, x) share everything but the sign pattern of
// the expansion: with w = t/v, Eq. (log Iv u k) sums u_k(t) w^k and Eq. (log Kv
// u k) sums (-1)^k u_k(t) w^k, so with the even / odd parts E, O of the sum
// S_I = 1 + E + O and S_K = 1 + E - O; likewise the mu expansions differ only
// by (-1)^k.  One rsqrt, one Horner pass per P_k, one v*eta (its log) serve
// both results; only the final log per function is separate.
template <typename T, int KU>
__device__ __forceinline__ void log_bessel_u_ik(T v, T x, T &li, T &lk, uint32_t tab = logtab_addr()) {
    const T rho2 = fma(v, v, x * x);
    const T y = fm_rsqrt(rho2);                  // 1 / rho = t / v
    const T rho = rho2 * y;
    const T t = v * y;
    const T t2 = t * t, w2 = y * y;
    // E = sum_{k even >= 2} P_k w^k, O = sum_{k odd} P_k w^k (Horner in w^2)
    constexpr int KE = (KU / 2) * 2, KO = KU - ((KU + 1) % 2);
    T e = uk_row<T>(KE, t2);
#pragma unroll
    for (int k = KE - 2; k >= 2; k -= 2) e = fma(e, w2, uk_row<T>(k, t2));
    e *= w2;
    T o = uk_row<T>(KO, t2);
#pragma unroll
    for (int k = KO - 2; k >= 1; k -= 2) o = fma(o, w2, uk_row<T>(k, t2));
    o *= y;
    const T veta = v_times_eta<T, false>(v, x, v, x, rho, rho, tab);
    // log S_I = log1p(e + o), log S_K = log1p(e - o); one log of y for both:
    // 1/2 log(y pi/2) = 1/2 log(y/(2 pi)) + log(pi)
    const T hl = T(0.5) * fm_log(y * hc<T>(HC_INV2PI), tab);
    li = veta + (hl + log1p_small<T, L1PDeg<T, KU>::v>(e + o));
    lk = (hl + hc<T>(HC_LNPI)) + log1p_small<T, L1PDeg<T, KU>::v>(e - o) - veta;
}


template <typename T>
__device__ __forceinline__ void log_bessel_mu_ik(T v, T x, T &li, T &lk, uint32_t tab = logtab_addr()) {
#if B200_MUFACT
    // Carry T_k = k! term_k: T_k = T_{k-1} (c mu - c (2k-1)^2) (one FMA with an immediate
    // square, one multiply) and accumulate S_I, S_K with the constants (-1)^k / k!, 1/k!
    // by FMA: 4 FP64 operations per term.  |T_k| <= 26! max|term| < 1e30 (no overflow).
    // Written out term by term (the compiler declines to unroll this loop, and a rolled
    // loop pays an int -> double conversion and an indexed constant load per term).
    const T rx = fm_rcp(x);
    const T c = T(0.125) * rx;
    const T z = c * (T(4) * v * v);
    T tk = T(1), si = T(1), sk = T(1);
#define B200_MU_TERMS(T_, STOP_)                                              \
    T_(1) T_(2) T_(3) T_(4)                                                   \
    T_(5) T_(6) T_(7) T_(8) STOP_(8)                                          \
    T_(9) T_(10) T_(11) T_(12) STOP_(12)                                      \
    T_(13) T_(14) T_(15) T_(16) STOP_(16)                                     \
    T_(17) T_(18) T_(19) T_(20) STOP_(20)                                     \
    T_(21) T_(22) T_(23) T_(24) STOP_(24)                                     \
    T_(25) T_(26)
    // S_I alternates and cancels where the series converges slowest (x ~ 30, v ~ 15: terms
    // up to ~9 sum to ~0.02).  f64 sums even / odd parts (S_K = E + O, S_I = E - O: 3 FP64
    // operations per term, cancellation error ~1e-14 of log I); f32 accumulates S_I with
    // its signs term by term, whose rounding follows the partial sums (f32 log I at that
    // corner 1.7e-6 instead of 1.1e-5; R17)
#define B200_MU_F(k)                                                          \
    tk *= fma(c, T(-double((2 * (k) - 1) * (2 * (k) - 1))), z);
#if B200_MUFACT == 2
    if constexpr (sizeof(T) == 8) {
        T ev = T(1), od = T(0);
#define B200_MU_T(k)                                                          \
    {                                                                         \
        B200_MU_F(k)                                                          \
        if ((k) & 1) od = fma(tk, c_invfact<T>(k), od);                       \
        else ev = fma(tk, c_invfact<T>(k), ev);                               \
    }
#define B200_MU_STOP(k) if (fabs(tk) * c_invfact<T>(k) <= Tr<T>::eps * T(0.25) * fabs(ev - od)) goto mu_done_eo;
        B200_MU_TERMS(B200_MU_T, B200_MU_STOP)
#undef B200_MU_T
#undef B200_MU_STOP
    mu_done_eo:
        si = ev - od;
        sk = ev + od;
    } else
#endif
    {
#define B200_MU_T(k)                                                          \
    {                                                                         \
        B200_MU_F(k)                                                          \
        const T f = c_invfact<T>(k);                                          \
        si = fma(((k) & 1) ? -tk : tk, f, si);                                \
        sk = fma(tk, f, sk);                                                  \
    }
#define B200_MU_STOP(k) if (fabs(tk) * c_invfact<T>(k) <= Tr<T>::eps * T(0.25) * fabs(si)) goto mu_done_sg;
        B200_MU_TERMS(B200_MU_T, B200_MU_STOP)
#undef B200_MU_T
#undef B200_MU_STOP
    mu_done_sg:;
    }
#undef B200_MU_F
#undef B200_MU_TERMS
    const T SI = fabs(si), SK = fabs(sk);
    li = x + T(0.5) * fm_log(SI * SI * rx * hc<T>(HC_INV2PI), tab);
    lk = -x + T(0.5) * fm_log(SK * SK * rx * hc<T>(HC_PIO2), tab);
#elif B200_MUEO
    // The two series differ only by (-1)^k: with E = 1 + sum of the even terms and
    // O = sum of the odd ones, S_K = E + O and S_I = E - O, so every term is added
    // once.  term_k = term_{k-1} f_k with f_k = c (mu - (2k-1)^2) / k, c = 1/(8x),
    // formed as (c mu - c (2k-1)^2) / k = fma(c, -(2k-1)^2, z) * (1/k), z = c mu
    // ((2k-1)^2 is an immediate): 4 FP64 operations per term instead of 6.
    const T rx = fm_rcp(x);
    const T c = T(0.125) * rx;
    const T z = c * (T(4) * v * v);
    T term = T(1), E = T(1), O = T(0);
#pragma unroll
    for (int k = 1; k < KMU; k += 4) {
#pragma unroll
        for (int u = 0; u < 4 && k + u <= KMU; u += 2) {
            const int k1 = k + u;
            term *= fma(c, T(-(2 * k1 - 1) * (2 * k1 - 1)), z) * c_inv_k<T>(k1);
            O += term;
            term *= fma(c, T(-(2 * k1 + 1) * (2 * k1 + 1)), z) * c_inv_k<T>(k1 + 1);
            E += term;
        }
        if (k >= 3 && fabs(term) <= Tr<T>::eps * T(0.25) * fabs(E - O)) break;
    }
    const T SI = fabs(E - O), SK = fabs(E + O);
    li = x + T(0.5) * fm_log(SI * SI * rx * hc<T>(HC_INV2PI), tab);
    lk = -x + T(0.5) * fm_log(SK * SK * rx * hc<T>(HC_PIO2), tab);
#else
    const T rx = fm_rcp(x);
    const T mu = T(4) * v * v;
    const T c = T(0.125) * rx;
    T term = T(1), si = T(1), sk = T(1);          // K terms (all signs +); I alternates
#if B200_MUF
    // factor c (mu - (2k-1)^2) / k formed as fma(c, -(2k-1)^2, c mu) * (1/k): the odd
    // square is an immediate, one FP64 operation fewer per term than (mu - sq) * (c / k)
    const T z = c * mu;
#endif
    // terms in (odd, even) pairs, fully unrolled: (2k-1)^2 and 1/k are constants
#ifndef B200_MU_STEP
#define B200_MU_STEP 4
#endif
#pragma unroll
    for (int k = 1; k < KMU; k += B200_MU_STEP) {   // B200_MU_STEP terms per stop test (KMU = 26)
#pragma unroll
        for (int u = 0; u < B200_MU_STEP && k + u <= KMU; u += 2) {
            const int k1 = k + u;
            const T i1 = c_inv_k<T>(k1), i2 = c_inv_k<T>(k1 + 1);
#if B200_MUF
            term *= fma(c, T(-(2 * k1 - 1) * (2 * k1 - 1)), z) * i1;
#else
            term *= (mu - T((2 * k1 - 1) * (2 * k1 - 1))) * (c * i1);
#endif
            si -= term;                            // summed in order, as the separate
            sk += term;                            // series (no even/odd cancellation)
#if B200_MUF
            term *= fma(c, T(-(2 * k1 + 1) * (2 * k1 + 1)), z) * i2;
#else
            term *= (mu - T((2 * k1 + 1) * (2 * k1 + 1))) * (c * i2);
#endif
            si += term;
            sk += term;
        }
        if (k >= 3 && fabs(term) <= Tr<T>::eps * T(0.25) * fabs(si)) break;
    }
    const T SI = fabs(si), SK = fabs(sk);
    li = x + T(0.5) * fm_log(SI * SI * rx * hc<T>(HC_INV2PI), tab);
    lk = -x + T(0.5) * fm_log(SK * SK * rx * hc<T>(HC_PIO2), tab);
#endif
}

// ---------------------------------------------------------------- series (I)
// Eq. (Iv infinite series) (line 127) with the recurrence Eqs. (ak recurrence
// base)/(ak recurrence) (lines 148-150) and the logarithm-of-a-sum form
// Eq. (log Iv) (lines 153-155):
//   log I = v log(x/2) + log a_0 + log sum_k (a_k / a_0),  log a_0 = -lgamma(v+1).
// The ratios a_k/a_0 are carried in linear scale (b_{k+1} = b_k x^2 / (4(k+1)(k+v+1))):
// in the fallback region x <= 30, so sum_k b_k <= Gamma(v+1) e^x < 1e23 and
// nothing can overflow; pivoting the log-sum-exp on a_0 instead of the peak
// a_K (line 120) is therefore exact up to rounding (reading R6).
// Stop once past the peak term (Eq. (K)) and the term is below eps
// of the partial sum ("Terms less than machine precision, relative to the
// maximum value, are ignored", line 194).
//
// f64: the same sum without a division per term.  With D_k = k (v + k) and
// P_k = D_1 ... D_k, carry N_k = P_k * sum_{j<=k} b_j and Q_k = P_k b_k = q^k:
//   Q_k = q Q_{k-1},  N_k = N_{k-1} D_k + Q_k,  P_k = P_{k-1} D_k,
// so sum_k b_k = N_K / P_K (one division at the end) and the stop test
// b_k <= eps * sum reads Q_k <= eps * N_k.  In the fallback region (x <= 30,
// v <= 12.7, at most ~45 terms) P_K < 1e130 and N_K < 1e150: no rescaling.
template <typename T, bool SAFE>
__device__ __forceinline__ T log_iv_series(T v, T x, uint32_t tab = logtab_addr()) {
    if (x == T(0)) return v == T(0) ? T(0) : T(-CUDART_INF);
    if constexpr (sizeof(T) == 8) {
        const T q = T(0.25) * x * x;
        // M_k = N_k - P_k = P_k sum_{1<=j<=k} b_j (carried instead of N: the sum minus its
        // leading 1 keeps full relative accuracy when the sum is ~1, e.g. log I_0(x) ~ x^2/4)
        T M = T(0), P = T(1), Q = T(1), vk = v, kd = T(0);
#if B200_SERIES_UNROLL
        // terms 1..48 written out (x <= 30, the series region, needs at most ~45): D_k =
        // k (v + k) is one FMA with immediates k, k^2 instead of two counter additions and
        // a product (and one rounding instead of two)
#define B200_SR_T(k)                                                         \
        {                                                                    \
            const T d = fma(T(double(k)), v, T(double((k) * (k))));          \
            Q *= q;                                                          \
            M = fma(M, d, Q);                                                \
            P *= d;                                                          \
        }
#define B200_SR_4(k) B200_SR_T(k) B200_SR_T((k) + 1) B200_SR_T((k) + 2) B200_SR_T((k) + 3) \
        if (Q <= (M + P) * Tr<T>::eps) goto series_done;
        B200_SR_4(1) B200_SR_4(5) B200_SR_4(9) B200_SR_4(13) B200_SR_4(17) B200_SR_4(21)
        B200_SR_4(25) B200_SR_4(29) B200_SR_4(33) B200_SR_4(37) B200_SR_4(41) B200_SR_4(45)
#undef B200_SR_T
#undef B200_SR_4
        vk = v + T(48);
        kd = T(48);
        for (int k = 49; k < 400; k += 4) {     // not reached for x <= 30
#else
        for (int k = 1; k < 400; k += 4) {      // four terms per trip, one stop test
#endif
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                vk += T(1);
                kd += T(1);
                const T d = kd * vk;
                Q *= q;
                M = fma(M, d, Q);
                P *= d;
            }
            if (Q <= (M + P) * Tr<T>::eps) break;
        }
#if B200_SERIES_UNROLL
    series_done:
#endif
        // a_0 = 1/Gamma(v+1) = rg(mu) / prod_{j=1..n} (mu + j), v = n + mu, |mu| <= 1/2,
        // rg(z) = 1/Gamma(1+z) by its Taylor series (tables.h) -- no lgamma call;
        // rg(mu) = 1 + gm1 with gm1 = mu (c_1 + mu (c_2 + ...)) (c_0 = 1)
        const T fl = floor(v + T(0.5));
        const T mu = v - fl;
        const int nl = int(fl);
        T g = T(c_rg_d[B200_RGAMMA_NT - 1]);
#pragma unroll
        for (int j = B200_RGAMMA_NT - 2; j >= 1; --j) g = fma(g, mu, T(c_rg_d[j]));
        const T gm1 = g * mu;
        const T lx = SAFE ? fm_log_wide(x) - T(0.6931471805599453) : fm_log(T(0.5) * x, tab);   // log(x/2)
        if (nl == 0) {
            // v < 1/2: log I = v log(x/2) + log1p(gm1) + log1p(M/P) -- every term with
            // relative accuracy (|log I| < 1 here for small v and x: DESIGN.md R1)
            return fma(v, lx, fm_log1p(gm1, tab) + fm_log1p(fm_div(M, P), tab));
        }
        T pr = T(1), m = mu;
        for (int j = 1; j < nl; j += 2) {      // factor pairs (mu+j)(mu+j+1)
            const T a = m + T(1);
            m += T(2);
            pr *= a * m;
        }
        if (nl & 1) pr *= m + T(1);
        return fma(v, lx, fm_log(fm_div((M + P) * (T(1) + gm1), P * pr), tab));
    }
    const T q = T(0.25) * x * x;
    T b = T(1), S = T(1);
    // b_{k+1} = b_k * q * (1/(k+1)) * (1/(k+v+1)): 1/(k+1) from the table, the
    // reciprocal of (k+v+1) does not depend on b, so it is off the dependency chain.
    for (int k = 0; k < 200; k += 2) {
        const T r0 = q * c_inv_k<T>(k + 1) / (T(k) + v + T(1));
        const T r1 = q * c_inv_k<T>(k + 2) / (T(k) + v + T(2));
        const T b0 = b * r0;
        b = b0 * r1;
        S += b0 + b;
        if (r1 < T(1) && b <= S * Tr<T>::eps) break;
    }
    const T lx = SAFE ? log(x) - T(0.6931471805599453) : log(T(0.5) * x);   // log(x/2); 0.5 x underflows for tiny x
    return (v == T(0) ? T(0) : v * lx) - d_lgamma(v + T(1)) + log(S);
}

// ---------------------------------------------------------------- K fallback
// Small-argument region of K (x <= 30, v <= 12.7 after dispatch).  The paper
// evaluates Eq. (log Kv integral) with Simpson N = 600 (lines 248-324); its
// measured error against the binary128 oracle is up to 5.7e-10 (DESIGN.md
// §5), above the 1e-13 target.  Instead, for x <= 2 Temme's method:
// K_mu, K_{mu+1} for |mu| <= 1/2 by Temme's series, then the forward
// recurrence K_{nu+1} = K_{nu-1} + (2 nu / x) K_nu (stable for K) up to
// nu = v, with the running value kept as mantissa * 10^(30 e) so nothing
// overflows; the result is returned as a logarithm.  For 2 < x <= 30 the
// trapezoidal rule on DLMF 10.32.9 gives K_mu, K_{mu+1} (trap_kmu below), then
// the same recurrence.
template <typename T>
__device__ __forceinline__ void temme_gammas(T mu, T &gam1, T &gam2, T &gampl, T &gammi) {
    // 1/Gamma(1+z) = sum_j c_j z^j  (tables.h).  Even/odd parts give
    // gam2 = (1/G(1-mu) + 1/G(1+mu))/2 = sum_even c_j mu^j
    // gam1 = (1/G(1-mu) - 1/G(1+mu))/(2 mu) = -sum_odd c_j mu^(j-1)
    const T m2 = mu * mu;
    const int N = Tr<T>::rg_terms;
    T ev = Tr<T>::rg(N - 2), od = Tr<T>::rg(N - 1);
#pragma unroll
    for (int j = N - 4; j >= 0; j -= 2) {
        ev = fma(ev, m2, Tr<T>::rg(j));
        od = fma(od, m2, Tr<T>::rg(j + 1));
    }
    gam2 = ev;
    gam1 = -od;
    gampl = ev + mu * od;   // 1/Gamma(1+mu)
    gammi = ev - mu * od;   // 1/Gamma(1-mu)
}

// sinh(e)/e and cosh(e) from E = e^e (|e| <= 162 here)
template <typename T>
__device__ __forceinline__ void sinhc_cosh(T e, T E, T &shc, T &ch) {
    const T Ei = fm_rcp(E);
    ch = T(0.5) * (E + Ei);
    if (fabs(e) < T(0.5)) {
        // sinh(e)/e = sum_k e^{2k} / (2k+1)!, 9 terms for e^2 < 1/4
        const T e2 = e * e;
        T p = T(1.0 / 6402373705728000.0);                 // 1/18!
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            double f = 1.0;                                  // 1/(2k+1)!
            for (int j = 2; j <= 2 * k + 1; ++j) f /= j;
            p = fma(p, e2, T(f));
        }
        shc = p;
    } else {
        shc = T(0.5) * (E - Ei) * fm_rcp(e);
    }
}

// Temme's series for K_mu, K_{mu+1}, |mu| <= 1/2, 0 < x <= 2: N. M. Temme, "On the
// numerical evaluation of the modified Bessel function of the third kind",
// J. Comput. Phys. 19 (1975) 324-337; the step order follows the published
// formulation (f_k, p_k, q_k recurrences; the same lineage as Numerical Recipes'
// bessik and libstdc++'s tr1 __bessel_ik).  Re-worked for the GPU: one shared
// reciprocal of i^2 - mu^2 per term, multiplicative p/q updates, two terms per
// stop test, 1/Gamma(1 +- mu) and pi mu / sin(pi mu) from Taylor tables.
// Returns log K_mu(x) and the sums S = K_mu(x), S1 with K_{mu+1}(x) = (2/x) S1
// (callers form rho = K_{mu+1}/K_mu = 2 S1 / (x S), or the scaled ratio S1 / S).
// SAFE = false: elementary functions from fastmath.cuh (x >= 1e-140 on the fast
// path, so ln(2/x) <= 323, |mu ln(2/x)| <= 162, every reciprocal argument normal).
// SAFE = true (the slow bin): any x > 0 including subnormals -- ln(2/x) = ln 2 -
// log x by the library log (0.5 x would underflow), |mu ln(2/x)| <= 372.5.
template <typename T, bool SAFE = false>
__device__ __forceinline__ T temme_kmu(T mu, T x, T &sum, T &sum1, uint32_t tab = logtab_addr()) {
    const T eps = Tr<T>::eps;
    const T d = SAFE ? T(0.6931471805599453) - log(x) : -fm_log(T(0.5) * x, tab);   // ln(2/x)
    const T e = mu * d;
    // pi mu / sin(pi mu) = 1 / sum_k SINPI[k] mu^(2k)  (|mu| <= 1/2, tables.h)
    const T m2 = mu * mu;
    T sp = T(c_sinpi_d[B200_SINPI_NT - 1]);
#pragma unroll
    for (int k = B200_SINPI_NT - 2; k >= 0; --k) sp = fma(sp, m2, T(c_sinpi_d[k]));
    const T fact = fm_rcp(sp);
    const T ee = fm_exp(e);
    T fact2, che;
    sinhc_cosh<T>(e, ee, fact2, che);
    T gam1, gam2, gampl, gammi;
    temme_gammas<T>(mu, gam1, gam2, gampl, gammi);
    T ff = fact * (gam1 * che + gam2 * fact2 * d);
    sum = ff;
    T p = T(0.5) * ee * fm_rcp(gampl);                        // 1/2 (2/x)^mu Gamma(1+mu)
    T q = T(0.5) * fm_rcp(ee * gammi);                        // 1/2 (x/2)^mu Gamma(1-mu)
    T c = T(1);
    const T dd = T(0.25) * x * x;
    sum1 = p;
    T del;
#if B200_TEMME_UNROLL
    // terms 1..20 written out (x <= 2 needs at most ~19: c_k <= 1/k!), so k, k^2 and 1/k are
    // immediates / uniform constants instead of a floating counter and an indexed load
#define B200_TM_T(k)                                                         \
    {                                                                        \
        const T inv = fm_rcp(T(double((k) * (k))) - m2);                     \
        ff = (T(double(k)) * ff + p + q) * inv;                              \
        c *= dd * c_inv_k<T>(k);                                             \
        p *= (T(double(k)) + mu) * inv;                                      \
        q *= (T(double(k)) - mu) * inv;                                      \
        del = c * ff;                                                        \
        sum += del;                                                          \
        sum1 += c * (p - T(double(k)) * ff);                                 \
    }
#define B200_TM_STOP if (fabs(del) < fabs(sum) * eps) goto temme_done;
    B200_TM_T(1) B200_TM_T(2) B200_TM_STOP B200_TM_T(3) B200_TM_T(4) B200_TM_STOP
    B200_TM_T(5) B200_TM_T(6) B200_TM_STOP B200_TM_T(7) B200_TM_T(8) B200_TM_STOP
    B200_TM_T(9) B200_TM_T(10) B200_TM_STOP B200_TM_T(11) B200_TM_T(12) B200_TM_STOP
    B200_TM_T(13) B200_TM_T(14) B200_TM_STOP B200_TM_T(15) B200_TM_T(16) B200_TM_STOP
    B200_TM_T(17) B200_TM_T(18) B200_TM_STOP B200_TM_T(19) B200_TM_T(20) B200_TM_STOP
#undef B200_TM_T
#undef B200_TM_STOP
    {
        T fi = T(20);
        for (int i = 21; i < 100; i += 2) {      // not reached for x <= 2
#else
    {
        T fi = T(0);
        for (int i = 1; i < 100; i += 2) {      // two terms per stop test
#endif
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                fi += T(1);
                // 1/(i-mu), 1/(i+mu) and 1/(i^2-mu^2) share one reciprocal
                const T inv = fm_rcp(fma(fi, fi, -m2));
                ff = (fi * ff + p + q) * inv;
                c *= dd * c_inv_k<T>(i + u);
                p *= (fi + mu) * inv;
                q *= (fi - mu) * inv;
                del = c * ff;
                sum += del;
                sum1 += c * (p - fi * ff);
            }
            if (fabs(del) < fabs(sum) * eps) break;
        }
    }
#if B200_TEMME_UNROLL
temme_done:
#endif
    return SAFE ? log(sum) : fm_log(sum, tab);
}

// K_mu(x) and K_{mu+1}(x), |mu| <= 1/2, on the band 2 < x <= 30 of the
// fallback region, from the integral
//   K_nu(x) = int_0^inf exp(-x cosh t) cosh(nu t) dt        (DLMF 10.32.9)
// by the trapezoidal rule.  The integrand is entire and decays
// double-exponentially, so the rule converges geometrically in 1/h: the error
// is ~ exp(-2 pi d/h) M(d) for a strip of half-width d < pi/2, with M(d)
// growing like K_nu(x cos d) / K_nu(x).  For orders <= 3/2 the step
// h = pi^2 / (42 + 0.8 x) keeps it below 2^-53 on 2 < x <= 30 (measured
// largest admissible step: pi^2/(41..48 + 0.79 x)).  With
// t_k = k h the nodes are
//   K_nu = (h/2) e^{-x} [1 + sum_{k>=1} e^{-2x sinh^2(t_k/2)} (E_nu^k + E_nu^{-k})],  E_nu = e^{nu h},
// sinh(t_k/2) by the three-term recurrence s_{k+1} = 2 cosh(h/2) s_k - s_{k-1}
// and 2 cosh(k nu h) by C_{k+1} = 2 cosh(nu h) C_k - C_{k-1} (growing solutions
// dominate: forward-stable), one exp per node shared by both orders, all terms
// positive.  The integrand is unimodal in t and its first
// node is already O(1) of the k = 0 term (2x sinh^2(h/2) < 0.4), so a term
// below eps of the sum only occurs past the peak: stop at the first K_{mu+1}
// term (the wider integrand) below eps of its sum.
// 2 cosh(z) for |z| <= 0.36 by its Taylor series in z^2 (the z^16 term is < 2^-60 of the sum):
// eight FP64 operations instead of an exp and a reciprocal
template <typename T>
__device__ __forceinline__ T two_cosh_small(T z) {
    const T z2 = z * z;
    T p = T(2.0 / 87178291200.0);                                   // 2/14!
    p = fma(p, z2, T(2.0 / 479001600.0));                           // 2/12!
    p = fma(p, z2, T(2.0 / 3628800.0));                             // 2/10!
    p = fma(p, z2, T(2.0 / 40320.0));                               // 2/8!
    p = fma(p, z2, T(2.0 / 720.0));                                 // 2/6!
    p = fma(p, z2, T(2.0 / 24.0));                                  // 2/4!
    p = fma(p, z2, T(1));                                           // 2/2!
    return fma(p, z2, T(2));
}

// Returns log K_mu and rho = K_{mu+1} / K_mu.  12-17 nodes on the band.
// kl (optional): K_mu e^x = (h/2) A, so log K_mu = -x + log kl (callers that
// fold further factors into one log use it).
template <typename T>
__device__ __forceinline__ T trap_kmu(T mu, T x, T &rho, uint32_t tab = logtab_addr(), T *kl = nullptr) {
    // f64: h = pi^2 / (42 + 0.8 x) (measured largest admissible step for 2^-53, R14);
    // f32: the error ~ exp(-pi^2 / h) only has to reach ~2^-26: h = pi^2 / (24 + 0.45 x)
    const T h = hc<T>(HC_PI2) * fm_rcp(sizeof(T) == 8 ? fma(T(0.8), x, T(42)) : fma(T(0.45), x, T(24)));
    const T a = T(0.5) * h, a2 = a * a;
    // sinh(a) and 2 cosh(a) by their Taylor series (a <= 0.12: 5 terms exact to 2^-60)
    const T s1 = a * fma(a2 * T(1.0 / 6), fma(a2 * T(1.0 / 20), fma(a2 * T(1.0 / 42), fma(a2, T(1.0 / 72), T(1)), T(1)), T(1)), T(1));
    const T c = fma(a2, fma(a2 * T(1.0 / 12), fma(a2 * T(1.0 / 30), fma(a2, T(1.0 / 56), T(1)), T(1)), T(1)), T(2));
    // 2 cosh(k nu h) for nu = mu, mu+1 by the recurrence C_{k+1} = c C_k - C_{k-1},
    // c = 2 cosh(nu h) (forward-stable: the growing solution dominates); |mu h| <= 0.12,
    // (mu + 1) h <= 1.5 h <= 0.36 on 2 < x (h <= 0.235)
#if B200_TRAP_EXPCOSH
    const T Em = fm_exp(mu * h), Emi = fm_rcp(Em);
    const T eh = fm_exp(h);
    const T cm = Em + Emi, cp = fma(Em, eh, Emi * fm_rcp(eh));
#else
    const T cm = two_cosh_small<T>(mu * h), cp = two_cosh_small<T>((mu + T(1)) * h);
#endif
    // (a0, a1) = (C_{k-1}, C_k) for order mu, (b0, b1) for mu+1, (x0, x1) = (s_{k-1}, s_k):
    // each trip overwrites the older of every pair with the next value (no register
    // moves in the loop), k = 1 at entry
    T a0 = T(2), a1 = cm, b0 = T(2), b1 = cp;
    T A = T(1), B = T(1), x0 = T(0), x1 = s1;
    // f64: the node exponents -2x s_k^2 are formed scaled by 64/ln2 for fm_exp_prescaled
    // (a relative error |y| 2^-52 in a node of size e^y: < 2^-53 of the sum, R14)
    const T m2x = sizeof(T) == 8 ? T(-2.0 * 92.33248261689366) * x : T(-2) * x;
    for (int k = 1; k < 64; k += 2) {     // nodes k, k+1 per trip, stop test on the second
        x0 = fma(c, x1, -x0);                                           // s_{k+1}
        T e1, e2;
        if constexpr (sizeof(T) == 8) {
            e1 = fm_exp_prescaled(m2x * x1 * x1);
            e2 = fm_exp_prescaled(m2x * x0 * x0);
        } else {
            e1 = fm_exp_nc(m2x * x1 * x1);
            e2 = fm_exp_nc(m2x * x0 * x0);
        }
        a0 = fma(cm, a1, -a0);                                          // C_{k+1}
        b0 = fma(cp, b1, -b0);
        A = fma(e1, a1, A);
        B = fma(e1, b1, B);
        const T tb = e2 * b0;
        A = fma(e2, a0, A);
        B += tb;
        if (tb <= B * Tr<T>::eps) break;
        x1 = fma(c, x0, -x1);                                           // s_{k+2}
        a1 = fma(cm, a0, -a1);                                          // C_{k+2}
        b1 = fma(cp, b0, -b1);
    }
    rho = B * fm_rcp(A);
    if (kl) {
        *kl = T(0.5) * h * A;
        return T(0);   // unused by such callers
    }
    return -x + fm_log(T(0.5) * h * A, tab);
}

template <typename T, bool SAFE>
__device__ __forceinline__ T log_kv_fallback(T v, T x, uint32_t tab = logtab_addr()) {
    const int nl = int(floor(v + T(0.5)));
    const T mu = v - T(nl);
    // forward recurrence K_{nu+1} = K_{nu-1} + (2 nu / x) K_nu (stable for K)
    // on the ratios K_{mu+i} / K_mu, from i = 0, 1 up to i = nl
    if (x > T(2)) {
        T rho;
        const T lk = trap_kmu<T>(mu, x, rho, tab);
        const T tox = T(2) * fm_rcp(x);
        // x > 2, v <= 12.7: K_v / K_mu < 1e12, no rescaling needed.  The coefficient
        // 2 nu / x advances by one addition of 2/x per step (< 13 roundings)
        T km = T(1), kp = rho, a = mu * tox;
#pragma unroll 2
        for (int i = 1; i < nl; ++i) {
            a += tox;
            const T kn = fma(a, kp, km);
            km = kp;
            kp = kn;
        }
        return nl == 0 ? lk : lk + fm_log(kp, tab);
    }
    T S, S1;
    const T lk = temme_kmu<T, SAFE>(mu, x, S, S1, tab);
    if (nl == 0) return lk;
    if (x >= T(1e-6)) {
        // (2 * 13 / 1e-6)^13 < 1e97: the unscaled ratio stays in the double range
        // (double for both precisions)
        const double tx = double(T(2) * fm_rcp(x));
        double km = 1.0, kp = double(T(2) * S1 * fm_rcp(x * S)), a = double(mu) * tx;
#pragma unroll 2
        for (int i = 1; i < nl; ++i) {
            a += tx;                                  // 2 (mu + i) / x
            const double kn = fma(a, kp, km);
            km = kp;
            kp = kn;
        }
        return lk + T(fm_log(kp, tab));
    }
    // x < 1e-6 (any x > 0, subnormals included): scaled ratios.  With s = x/2 and
    // a = 2 max(-mu, 0), k_i = (K_{mu+i}/K_mu) s^(i-a) (i >= 1) is O(1) for every i
    // (K_{mu+i} ~ Gamma(mu+i) (2/x)^(mu+i) / 2 and K_mu ~ Gamma(|mu|) (2/x)^|mu| / 2), so
    // nothing overflows or underflows even at x = 5e-324:
    //   k_1 = (S1/S) s^-a,  k_2 = s^(2-a) + (mu+1) k_1,  k_{i+1} = s^2 k_{i-1} + (mu+i) k_i,
    //   log K_v = log K_mu + log k_nl - (nl - a) log s.
    const double ls = (SAFE ? fm_log_wide(double(x)) : fm_log(double(x), tab)) - 0.6931471805599453;   // log(x/2)
    const double a = mu < T(0) ? -2.0 * double(mu) : 0.0;
    const double k1 = mu < T(0) ? fm_exp(fm_log(double(S1), tab) - fm_log(double(S), tab) - a * ls) : double(S1) / double(S);
    if (nl == 1) return lk + T(fm_log(k1, tab) - (1.0 - a) * ls);
    const double s2 = 0.25 * double(x) * double(x);   // underflows harmlessly for tiny x
    double km = k1, kp = fm_exp((2.0 - a) * ls) + double(mu + T(1)) * k1, nu = double(mu) + 1.0;
    for (int i = 2; i < nl; ++i) {
        nu += 1.0;
        const double kn = fma(s2, km, nu * kp);
        km = kp;
        kp = kn;
    }
    return lk + T(fm_log(kp, tab) - (double(nl) - a) * ls);
}

// Fused fallback for 2 < x <= 30, v <= 12.7 (FN_IK): log K_v as in
// log_kv_fallback, and log I_v from the same K values by the Wronskian
//   I_v K_{v+1} + I_{v+1} K_v = 1/x   (DLMF 10.28.2; not in PAPER.md, whose small-x I is the
//   series of Eq. (Iv infinite series), line 127 -- a design choice of this implementation)
// => log I_v = -log(x (K_{v+1} + r K_v)),  r = I_{v+1} / I_v,
// with every term positive (no cancellation).  r comes from Miller's backward
// recurrence y_{nu-1} = (2 nu / x) y_nu + y_{nu+1} started at nu = v + M with
// y = (1, 0): the minimal solution I dominates.  Truncation error of r on the
// whole band (tools/miller_steps.py):
//   f64: M = floor(min(12 + x, 20 + 0.55 x)) + 1 (15-37 steps of 3 ops), < 8.1e-19;
//   f32: M = floor(min(6 + x, 12 + 0.5 x)) + 1, < 2.3e-10, |y| < 2e11.
// It replaces the power series (up to ~45 terms of 5 ops, 1/Gamma(v+1), two logs).
// TEMME = true: the same on 1e-6 <= x <= 2 with K_mu, K_{mu+1} from Temme's
// series (f64 only: there |y| < 4.1e98 and K_{v+1}/K_mu < 1e97, so neither
// the recurrences nor x (K_{v+1} + r K_v) / K_mu leave the double range).
template <typename T, bool TEMME = false>
__device__ __forceinline__ void log_ivkv_trap(T v, T x, T &ri, T &rk, uint32_t tab = logtab_addr()) {
    const int nl = int(floor(v + T(0.5)));
    const T mu = v - T(nl);
    const T tox = T(2) * fm_rcp(x);
    T rho;
    // K_mu = e^off * kl: off = -x, kl = (h/2) A (trapezoid), off = 0, kl = Temme's sum;
    // both logs below take kl as a factor (two logs per pair instead of three)
    T kl;
    if constexpr (TEMME) {
        T S1;
        (void)temme_kmu<T>(mu, x, kl, S1, tab);
        rho = T(2) * S1 * fm_rcp(x * kl);
    } else {
        (void)trap_kmu<T>(mu, x, rho, tab, &kl);
    }
    // kp = K_v / K_mu, kn = K_{v+1} / K_mu (one recurrence step past v); the
    // coefficient 2 nu / x advances by one addition of 2/x per step
    T km = T(1), kp = rho, a = mu * tox;
#pragma unroll 2
    for (int i = 1; i <= nl; ++i) {
        a += tox;
        const T kn = fma(a, kp, km);
        km = kp;
        kp = kn;
    }
    // after the loop: kp = K_{v+1}/K_mu, km = K_v/K_mu
    // M rounded up to a multiple of 4 (four steps per trip, no remainder; more steps only
    // shrink the start error; |y| grows by at most (2 (v + M + 3) / x)^3 < 1e24 over the
    // bounds of DESIGN.md §5: still far inside the double / float range)
    const int M = ((sizeof(T) == 8 ? int(fmin(T(12) + x, fma(T(0.55), x, T(20)))) + 1
                                   : int(fmin(T(6) + x, fma(T(0.5), x, T(12)))) + 1) + 3) & ~3;
    T y1 = T(0), y0 = T(1);                 // y_{v+k+1}, y_{v+k}
    // coefficient b = 2 (v + k) / x, stepped down by one subtraction of 2/x per step
    // (<= 40 roundings: relative error < 1e-14 in b, far inside the ratio's tolerance;
    // a multiply per step, or an int -> T conversion (I2F.F64), cost more)
    T b = (v + T(M)) * tox;
#pragma unroll 1
    for (int k = M; k >= 4; k -= 4) {       // the two values swap roles each step (no moves)
        y1 = fma(b, y0, y1);
        b -= tox;
        y0 = fma(b, y1, y0);
        b -= tox;
        y1 = fma(b, y0, y1);
        b -= tox;
        y0 = fma(b, y1, y0);
        b -= tox;
    }
    // y0 = y_v, y1 = y_{v+1}: r = y1 / y0;  1 / (I_v K_mu) = x (K_{v+1} + r K_v) / K_mu
    const T off = TEMME ? T(0) : -x;
    rk = off + fm_log(kl * km, tab);
    if constexpr (sizeof(T) == 8) {
        ri = -off - fm_log(kl * x * fma(km, y1, kp * y0) * fm_rcp(y0), tab);
    } else {
        // f32: kp y0 can pass FLT_MAX near x = 0.1 (~1e27 * 1e17); take the ratio first
        ri = -off - fm_log(kl * x * fma(km, y1 * fm_rcp(y0), kp), tab);
    }
}

// ---------------------------------------------------------------- paper K
// The paper's own small-argument K method (kept for fidelity studies):
// Eq. (log Kv integral) (lines 251-254), n = 8, beta = 2n/(2v+1),
//   log K = 1/2 log pi - lgamma(v+1/2) - v log(2x) - x + log int_0^1 (g + h) du,
// Simpson's 1/3 rule with N = 600 (line 269) and weights w_k (lines 272-275),
// each of G and H summed in log scale around the heuristic maxima u_g* = 1,
// u_h* = 1/2 (v < 2) or 1/(2v) (lines 305, 318-323).  The Simpson prefactor is
// h/3 = 1/(3N) (the printed 1/(6N), line 265-267, is read as a typo:
// DESIGN.md reading R7).  Only v >= 0 reaches here (|v| taken by the caller).
template <typename T>
__device__ __forceinline__ T log_kv_integral_paper(T v, T x) {
    const int N = 600;
    const T n = T(8);
    const T beta = T(2) * n / (T(2) * v + T(1));
    const T lbeta = log(beta);
    const T vm = v - T(0.5);
    const T twox = T(2) * x;
    // log g(u) = log beta - u^beta + (v-1/2) log(2x + u^beta) + (n-1) log u
    // log h(u) = -1/u - (2v+1) log u + (v-1/2) log(2xu + 1)
    const T lg_max = lbeta - T(1) + vm * log(twox + T(1));          // g at u* = 1
    const T uh = (v < T(2)) ? T(0.5) : T(0.5) / v;
    const T lh_max = -T(1) / uh - (T(2) * v + T(1)) * log(uh) + vm * log1p(twox * uh);
    T G = T(0), H = T(0);
    for (int k = 1; k <= N; ++k) {
        const T u = T(k) / T(N);
        const T w = (k == N) ? T(1) : ((k & 1) ? T(4) : T(2));
        const T lu = log(u);
        const T ub = exp(beta * lu);
        const T lg = lbeta - ub + vm * log(twox + ub) + (n - T(1)) * lu;
        const T lh = -T(1) / u - (T(2) * v + T(1)) * lu + vm * log1p(twox * u);
        G += w * exp(lg - lg_max);
        H += w * exp(lh - lh_max);
    }
    const T lG = lg_max + log(G), lH = lh_max + log(H);
    const T M = fmax(lG, lH);
    const T lint = -log(T(3 * N)) + M + log(exp(lG - M) + exp(lH - M));
    return T(0.5) * T(1.1447298858494002) - d_lgamma(v + T(0.5)) - v * log(twox) - x + lint;
}

// ---------------------------------------------------------------- entry points
// Evaluation sub-methods (bins): the region of Algorithm 1 refined by cost.
// The U region splits into four bins by the number of terms K (R12): KU_A > ...
// for large rho, 13 below; each bin's rho threshold is tables.h's bound for its K.
#ifndef B200_KU_A
#define B200_KU_A 6
#endif
#ifndef B200_KU_B
#define B200_KU_B 8
#endif
#ifndef B200_KU_C
#define B200_KU_C 10
#endif
#define B200_CAT_(a, b) a##b
#define B200_CAT(a, b) B200_CAT_(a, b)
#define B200_HW_RHO(K) B200_CAT(B200_HW_RHO_K, K)
constexpr int KU_A = B200_KU_A, KU_B = B200_KU_B, KU_C = B200_KU_C;
// U term count per bin and precision: f64 by the 2^-56 bound (R12), f32 by 2^-28 (R17)
template <typename T> struct KUs;
template <> struct KUs<double> { static constexpr int A = KU_A, B = KU_B, C = KU_C, D = 13; };
template <> struct KUs<float> { static constexpr int A = 2, B = 3, C = 5, D = 9; };
static_assert(KU_A < KU_B && KU_B < KU_C && KU_C < 13, "U bins: increasing term counts below 13");
enum : int { E_MU = 0, E_UA = 1, E_UB = 2, E_UC = 3, E_U13 = 4, E_FB_A = 5, E_FB_B = 6 };

__device__ __forceinline__ int select_eval_hw(double v, double x, uint32_t hv, uint32_t hx, uint32_t hw_split) {
    // selects, no nested branches: U sub-bin from max(v, x) (R12), fallback cost class from x
    const uint32_t m = hv > hx ? hv : hx;
    const int eu = m >= B200_HW_RHO(B200_KU_A) ? E_UA : m >= B200_HW_RHO(B200_KU_B) ? E_UB
                 : m >= B200_HW_RHO(B200_KU_C) ? E_UC : E_U13;
    const int ef = hx > hw_split ? E_FB_B : E_FB_A;
    const int e = is_u_hw(hv, hx) ? eu : ef;
#if B200_MU2U
    // mu region with rho >= rho_10 (61): the U expansion with the R12 term count meets
    // the same 2^-56 truncation bound for every t and costs less than the mu series
    if (m >= B200_HW_RHO(B200_KU_C)) return is_mu_hw(v, x, hv, hx) ? eu : e;
#endif
    return is_mu_hw(v, x, hv, hx) ? E_MU : e;
}
__device__ __forceinline__ int select_eval(double v, double x, uint32_t hw_split) {
    return select_eval_hw(v, x, hiw(v), hiw(x), hw_split);
}

// The same dispatch on float inputs with float keys (f32 kernels): the keys are the
// float bit patterns, each "a > C" is bits(a) > bits(C_dn) with C_dn the largest float
// <= C (exact for float a), each "a >= rho_K" bits(a) >= bits(rho_K) -- no conversion
// of the inputs to double (tables.h B200_F32_*; R3).
__device__ __forceinline__ bool mu_edge_f32(float v, float x) {
    const float d = 0.5113f * lg2_ftz(x) + 1.14535832f - lg2_ftz(v);   // 0.7939 / ln 2
    if (fabsf(d) > 1e-4f) return d > 0.0f;
    return 0.5113 * log(double(x)) + 0.7939 > log(double(v));         // guard band: the double predicate
}
__device__ __forceinline__ int select_eval_f32(float v, float x, uint32_t hv, uint32_t hx, uint32_t split) {
    const uint32_t m = hv > hx ? hv : hx;
    // f32 U bins: K = 2 / 3 / 5 / 9 (KUs<float>) from their 2^-28 thresholds (R17)
    const int eu = m >= B200_F32U_RHO_K2 ? E_UA : m >= B200_F32U_RHO_K3 ? E_UB
                 : m >= B200_F32U_RHO_K5 ? E_UC : E_U13;
    const int ef = hx > split ? E_FB_B : E_FB_A;
    const bool u = (hx > B200_F32_X19 && hv > B200_F32_V07) || hv > B200_F32_V12;
    bool mu = hx > B200_F32_X30 && hv <= B200_F32_V15;                   // x > 30 && v < 15.3919
    if (!mu && hx > B200_F32_X59 && hv < hx) mu = (hv == 0) || mu_edge_f32(v, x);
    return mu ? E_MU : (u ? eu : ef);
}

template <typename T, bool SAFE>
__device__ __forceinline__ T log_iv_eval(int e, T v, T x) {
    switch (e) {
        case E_MU: return log_bessel_mu<T, false, SAFE>(v, x);
        case E_UA: return log_bessel_u<T, false, KU_A, SAFE>(v, x);
        case E_UB: return log_bessel_u<T, false, KU_B, SAFE>(v, x);
        case E_UC: return log_bessel_u<T, false, KU_C, SAFE>(v, x);
        case E_U13: return log_bessel_u<T, false, 13, SAFE>(v, x);
        default: return log_iv_series<T, SAFE>(v, x);
    }
}

template <typename T, bool PAPER, bool SAFE>
__device__ __forceinline__ T log_kv_eval(int e, T v, T x) {
    switch (e) {
        case E_MU: return log_bessel_mu<T, true, SAFE>(v, x);
        case E_UA: return log_bessel_u<T, true, KU_A, SAFE>(v, x);
        case E_UB: return log_bessel_u<T, true, KU_B, SAFE>(v, x);
        case E_UC: return log_bessel_u<T, true, KU_C, SAFE>(v, x);
        case E_U13: return log_bessel_u<T, true, 13, SAFE>(v, x);
        default: return PAPER ? log_kv_integral_paper<T>(v, x) : log_kv_fallback<T, SAFE>(v, x);
    }
}

// Scalar entry (used by the vMF kernel): full dispatch for one element.
template <typename T>
__device__ __forceinline__ T log_iv_scalar_eval(T v, T x) {
    if (x == T(0)) return v == T(0) ? T(0) : T(-CUDART_INF);
    return log_iv_eval<T, true>(select_eval(double(v), double(x), B200_HW_X8), v, x);
}

}  // namespace b200
