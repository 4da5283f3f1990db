// fastmath.cuh -- f64 elementary functions for the evaluation kernels.
//
// CUDA's libdevice log/exp/sqrt/division handle every IEEE corner case
// (denormals, infinities, NaN, overflow) with range checks and slow-path
// branches; on sm_100a a double log() costs ~80 instructions, of which only
// ~20 issue on the FP64 pipe (ncu, profiles/r02).  The dispatch of Algorithm 1
// only ever hands these functions finite, normal, in-range arguments, so the
// kernels use the table-driven versions below instead:
//   fm_log : 256-entry table of 1/c_i and -log(1/c_i) (hi+lo), |r| < 2^-9,
//            degree-6 Taylor polynomial of log1p(r);  error < 1 ulp + 2^-60 abs.
//   fm_exp : 2^(j/64) table (hi+lo), |r| < ln2/128, degree-5 expm1 polynomial.
//   fm_rcp / fm_rsqrt : MUFU seed (rcp/rsqrt.approx.ftz.f64), a cubic and a Newton step.
// Argument contracts are stated per function; callers guarantee them.  The
// float overloads forward to the CUDA single-precision functions (the f32 path
// is not on the bench).  Tables: tables.h (paper_2409_08729_b200/gen_tables.py).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tables.h"

namespace b200 {

struct LogEnt { double invc, thi, tlo, pad; };
static __device__ const LogEnt g_logtab[1 << B200_LOG_TAB_BITS] = B200_LOGTAB_INIT_STRUCT;
static __device__ const double2 g_exptab[B200_EXP_TAB_N] = B200_EXPTAB_INIT_STRUCT;

// Polynomial and reduction constants.  Kept in constant memory rather than as
// literals: a double literal whose low word is non-zero costs two UMOVs per
// use in SASS, a __constant__ operand is fetched two at a time (LDCU.128).
struct FmConst {
    double log_c6, log_c5, log_c3;       // -1/6, 1/5, 1/3
    double ln2_hi, ln2_lo;               // ln 2 split so that e * ln2_hi is exact for |e| < 2^11 (fdlibm)
    double exp_inv, exp_chi, exp_clo;    // 64/ln2; ln2/64 = chi (33 significant bits) + clo
    double exp_c5, exp_c4, exp_c3;       // 1/120, 1/24, 1/6
    double ln2_lo20, exp_clo20;          // remainders of the 21-significant-bit splits below
    double exp_ln2o64;                   // ln2/64 (fm_exp_prescaled)
};
static __constant__ FmConst c_fm = {
    -1.0 / 6.0, 0.2, 1.0 / 3.0,
    6.93147180369123816490e-01, 1.90821492927058770002e-10,
    92.33248261689366, 0.010830424695086549, 1.162596423439437e-12,
    1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0,
    -1.904654299957768e-09, -2.9760223436840126e-11,
    0.010830424696249145,
};

#ifndef B200_IMM
#define B200_IMM 1
#endif
// Short constants (B200_IMM): a double whose low word is zero (21 significant bits)
// is an instruction immediate on sm_100a; any other constant costs a constant-bank
// load (LDC into a register, or LDCU into a uniform register).  Where the error
// analysis allows, the polynomial coefficients are rounded to 21 bits (relative
// error <= 2^-22): log1p's r^5, r^6 terms (|r| < 2^-9: contribution < 1e-18
// relative), exp's r^4, r^5 terms and the 64/ln2 range-reduction factor (|r|
// grows by < 4%); ln 2 and ln 2 / 64 are split at 21 bits (e * ln2_hi20 exact
// for |e| < 2^11, k * chi20 exact for |k| < 2^17) with full-precision remainders.
constexpr double IMM_LOG_C6 = -0.16666662693023682;     // -1/6 (0xBFC5555500000000)
constexpr double IMM_LOG_C5 = 0.20000004768371582;      //  1/5 (0x3FC9999A00000000)
constexpr double IMM_LN2_HI20 = 0.6931471824645996;     //  ln 2 (0x3FE62E4300000000)
constexpr double IMM_EXP_INV = 92.33245849609375;       //  64/ln2 (0x4057154700000000)
constexpr double IMM_EXP_CHI20 = 0.010830424726009369;  //  ln2/64 (0x3F862E4300000000)
constexpr double IMM_EXP_C5 = 0.00833333283662796;      //  1/120 (0x3F81111100000000)
constexpr double IMM_EXP_C4 = 0.041666656732559204;     //  1/24 (0x3FA5555500000000)

// exp(y) core, |y| <= 708 (result normal); shared by fm_exp / fm_exp_nc
__device__ __forceinline__ double fm_exp_core(double y) {
    constexpr double SHIFT = 6755399441055744.0;               // 1.5 * 2^52: round-to-int (immediate)
#if B200_IMM
    double kd = fma(y, IMM_EXP_INV, SHIFT);
    const int k = __double2loint(kd);
    kd -= SHIFT;
    double r = fma(kd, -IMM_EXP_CHI20, y);
    r = fma(kd, -c_fm.exp_clo20, r);                           // |r| <= 1.04 ln2/128
    // expm1(r) = r + r^2 (1/2 + r (1/6 + r (1/24 + r/120)))
    double p = fma(r, IMM_EXP_C5, IMM_EXP_C4);
#else
    double kd = fma(y, c_fm.exp_inv, SHIFT);
    const int k = __double2loint(kd);
    kd -= SHIFT;
    double r = fma(kd, -c_fm.exp_chi, y);
    r = fma(kd, -c_fm.exp_clo, r);                             // |r| <= ln2/128
    double p = fma(r, c_fm.exp_c5, c_fm.exp_c4);
#endif
    p = fma(p, r, c_fm.exp_c3);
    p = fma(p, r, 0.5);
    p = fma(p, r * r, r);
#if B200_SMEM_LOG && B200_SMEM_EXP
    const double2 T = s_exptab[k & (B200_EXP_TAB_N - 1)];
#else
    const double2 T = __ldg(&g_exptab[k & (B200_EXP_TAB_N - 1)]);
#endif
    const double res = T.x + fma(T.x, p, T.y);
    return __hiloint2double(__double2hiint(res) + ((k >> 6) << 20), __double2loint(res));
}

#ifndef B200_SMEM_LOG
#define B200_SMEM_LOG 1
#endif
#ifndef B200_SMEM_EXP
#define B200_SMEM_EXP 0
#endif
#if B200_SMEM_LOG
// {1/c_i, -log(1/c_i)} in shared memory (filled by fm_tables_init at kernel start)
static __shared__ double2 s_logtab[1 << B200_LOG_TAB_BITS];
#if B200_SMEM_EXP
static __shared__ double2 s_exptab[B200_EXP_TAB_N];
#endif
__device__ __forceinline__ void fm_tables_init() {
    for (int i = threadIdx.x; i < (1 << B200_LOG_TAB_BITS); i += blockDim.x)
        s_logtab[i] = make_double2(g_logtab[i].invc, g_logtab[i].thi);
#if B200_SMEM_EXP
    for (int i = threadIdx.x; i < B200_EXP_TAB_N; i += blockDim.x) s_exptab[i] = g_exptab[i];
#endif
    __syncthreads();
}
#else
__device__ __forceinline__ void fm_tables_init() {}
#endif

#if B200_SMEM_LOG
// 32-bit shared address of the log table.  The kernels compute it once and pass it down
// (fm_log(a, tab)): on sm_100a a shared address carries the CTA's cluster rank, and ptxas
// re-derives it (S2UR SR_CgaCtaId + three uniform operations) at every table access
// otherwise.
__device__ __forceinline__ uint32_t logtab_addr() { return uint32_t(__cvta_generic_to_shared(s_logtab)); }
#else
__device__ __forceinline__ uint32_t logtab_addr() { return 0u; }
#endif

// log(a) for finite normal a > 0; tab = logtab_addr() (computed by the caller).
__device__ __forceinline__ double fm_log(double a, uint32_t tab) {
    const int hi = __double2hiint(a), lo = __double2loint(a);
    const int t = hi - B200_LOG_HI_OFF;
    const int e = t >> 20;                                   // a = 2^e * m, m in [sqrt(1/2), sqrt(2))
    const int i = (t >> (20 - B200_LOG_TAB_BITS)) & ((1 << B200_LOG_TAB_BITS) - 1);
    const double m = __hiloint2double(hi - (e << 20), lo);
#if B200_SMEM_LOG
    double2 c;   // the table is written once at kernel start (fm_tables_init, then a barrier)
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c.x), "=d"(c.y) : "r"(tab + 16u * uint32_t(i)));
    const double tlo = 0.0;
#else
    const double2 c = __ldg(reinterpret_cast<const double2 *>(&g_logtab[i]));
    const double tlo = __ldg(&g_logtab[i].tlo);
#endif
    const double r = fma(m, c.x, -1.0);                      // m / c_i - 1, |r| < 0.00195
    // log1p(r) - r = r^2 (-1/2 + r (1/3 + r (-1/4 + r (1/5 - r/6))))
#if B200_IMM
    double p = fma(r, IMM_LOG_C6, IMM_LOG_C5);
#else
    double p = fma(r, c_fm.log_c6, c_fm.log_c5);
#endif
    p = fma(p, r, -0.25);
    p = fma(p, r, c_fm.log_c3);
    p = fma(p, r, -0.5);
    const double ed = double(e);   // I2F.F64 (a DADD-based magic-number conversion measured +1%: FP64 pipe)
#if B200_IMM
    const double h = fma(ed, IMM_LN2_HI20, c.y);
    const double l = fma(ed, c_fm.ln2_lo20, tlo);
#else
    const double h = fma(ed, c_fm.ln2_hi, c.y);
    const double l = fma(ed, c_fm.ln2_lo, tlo);
#endif
    return h + (r + fma(r * r, p, l));
}
__device__ __forceinline__ double fm_log(double a) { return fm_log(a, logtab_addr()); }

// exp(y) from yp = y * 64/ln2, already scaled by the caller (who folds the factor into a
// product it forms anyway), -65000 <= yp <= 0: the reduction is yp - round(yp), exact,
// and the 64/ln2 factor needs no register.  yp's own rounding (~2 ulp) is an absolute
// error |y| 2^-52 in the exponent, i.e. a relative error |y| 2^-52 of the result.
__device__ __forceinline__ double fm_exp_prescaled(double yp) {
    constexpr double SHIFT = 6755399441055744.0;               // 1.5 * 2^52: round-to-int (immediate)
    double kd = yp + SHIFT;
    const int k = __double2loint(kd);
    kd -= SHIFT;
    const double r = (yp - kd) * c_fm.exp_ln2o64;              // |r| <= ln2/128
    double p = fma(r, IMM_EXP_C5, IMM_EXP_C4);
    p = fma(p, r, c_fm.exp_c3);
    p = fma(p, r, 0.5);
    p = fma(p, r * r, r);
    const double2 T = __ldg(&g_exptab[k & (B200_EXP_TAB_N - 1)]);
    const double res = T.x + fma(T.x, p, T.y);
    return __hiloint2double(__double2hiint(res) + ((k >> 6) << 20), __double2loint(res));
}

// exp(y) for -708 <= y <= 709 (result normal); y < -708 is clamped (callers
// only use it where such terms are negligible).
__device__ __forceinline__ double fm_exp(double y) { return fm_exp_core(fmax(y, -708.0)); }

// exp(y) for -708 <= y <= 709 without the clamp (caller guarantees the range).
__device__ __forceinline__ double fm_exp_nc(double y) { return fm_exp_core(y); }

#ifndef B200_FASTRCP
#define B200_FASTRCP 1
#endif
// 1/a for finite normal |a| in [2^-1000, 2^1000].
__device__ __forceinline__ double fm_rcp(double a) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    double e = fma(-a, r, 1.0);
    r = fma(r, fma(e, e, e), r);              // cubic step: error e^3
#if B200_FASTRCP
    return r;                                 // seed error e < 2^-22 (tools/mufu_accuracy.cu): e^3 < 2^-66
#else
    e = fma(-a, r, 1.0);
    return fma(r, e, r);                      // Newton step
#endif
}

// x / y (y as for fm_rcp), with one residual correction (faithful).
__device__ __forceinline__ double fm_div(double x, double y) {
    const double r = fm_rcp(y);
    const double q = x * r;
    return fma(r, fma(-y, q, x), q);
}

// 1/sqrt(a) for finite normal a > 0 in [2^-1000, 2^1000].
__device__ __forceinline__ double fm_rsqrt(double a) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a * y, y, 1.0);           // 1 - a y^2
    y = fma(y, e * fma(e, 0.375, 0.5), y);    // y (1 + e/2 + 3e^2/8): error O(e^3)
#if B200_FASTRCP
    return y;
#else
    e = fma(-a * y, y, 1.0);
    return fma(0.5 * y, e, y);                // Newton step
#endif
}

// log(1 + d) for d > -1 with relative accuracy when |d| is small: u = 1 + d rounds,
// the first-order correction restores the lost low part of d (u - 1 is exact).
__device__ __forceinline__ double fm_log1p(double d, uint32_t tab) {
    const double u = 1.0 + d;
    if (u == 1.0) return d;
    return fm_log(u, tab) - ((u - 1.0) - d) * fm_rcp(u);
}
__device__ __forceinline__ double fm_log1p(double d) { return fm_log1p(d, logtab_addr()); }

__device__ __forceinline__ double fm_log_acc(double a, uint32_t tab) { return fm_log(a, tab); }
__device__ __forceinline__ double fm_log_acc(double a) { return fm_log(a); }

// log(a) for any finite a > 0 (subnormals through the library function).
__device__ __forceinline__ double fm_log_wide(double a) { return a >= 1e-300 ? fm_log(a) : log(a); }

#ifndef B200_F32FAST
#define B200_F32FAST 1
#endif
// f32 path.  B200_F32FAST: the hardware approximations (MUFU) -- log via lg2.approx
// (absolute error < 2^-21.4 on [1/2, 2], <= 3 ulp elsewhere), exp via ex2.approx of
// y log2 e, rcp / rsqrt .approx (1-2 ulp).  Every use is an O(1)-conditioned step of
// a result checked to 1e-5 against the oracle; the f32 operating range (R13) keeps
// the arguments normal.  The slow bin keeps the library functions (fm_log_wide).
__device__ __forceinline__ float fm_log_wide(float a) { return logf(a); }
// log whose absolute error is multiplied by a large factor (v log(x/(v+rho)) in the U
// expansion, where v eta cancels towards its root): the accurate library logf in f32
__device__ __forceinline__ float fm_log_acc(float a) { return logf(a); }
__device__ __forceinline__ float fm_log_acc(float a, uint32_t) { return logf(a); }
#if B200_F32FAST
__device__ __forceinline__ float fm_log(float a) { return __logf(a); }
__device__ __forceinline__ float fm_log(float a, uint32_t) { return __logf(a); }
__device__ __forceinline__ float fm_exp(float y) { return __expf(fmaxf(y, -87.0f)); }
__device__ __forceinline__ float fm_exp_nc(float y) { return __expf(y); }
__device__ __forceinline__ float fm_rcp(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ float fm_div(float x, float y) { return x * fm_rcp(y); }
__device__ __forceinline__ float fm_rsqrt(float a) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
#else
__device__ __forceinline__ float fm_log(float a) { return logf(a); }
__device__ __forceinline__ float fm_log(float a, uint32_t) { return logf(a); }
__device__ __forceinline__ float fm_exp(float y) { return expf(y); }
__device__ __forceinline__ float fm_exp_nc(float y) { return expf(y); }
__device__ __forceinline__ float fm_rcp(float a) { return __frcp_rn(a); }
__device__ __forceinline__ float fm_div(float x, float y) { return x / y; }
__device__ __forceinline__ float fm_rsqrt(float a) { return rsqrtf(a); }
#endif

}  // namespace b200
