// bessel_kernels.cu -- sm_100a kernels and the C ABI of include/bessel_b200.h.
//
// Hot path: batched log I_v(x) / log K_v(x) (§3-§4).  One persistent
// kernel per (function, precision, alignment); FN_IK evaluates both functions
// of each pair in one pass.  Each CTA processes tiles of TILE pairs:
//   0. one thread requests the NEXT tile with a bulk copy (TMA) into the other
//      half of a double-buffered shared-memory stage (per-thread cp.async for
//      8-byte-aligned pointers);
//   1. every thread classifies its elements (Algorithm 1 with the GPU branch
//      set plus cost sub-bins, integer predicates on IEEE high words);
//   2. an in-CTA counting sort of the element indices by bin (4-bit per-thread
//      counters widened to 8-bit warp fields, warp-shuffle scans) -- the paper's
//      "sort the input elements based on which expression is used" (§4.3, line
//      391) done per tile in shared memory instead of as a global sort, so no
//      extra HBM pass; a tile whose elements share one bin skips it;
//   3. every warp evaluates 32-slot chunks of the sorted order, gathering (v, x)
//      from the stage and writing the results over them.  The f64 fused pass
//      sorts costliest-first, pads every bin of a mixed tile to whole chunks (no
//      chunk runs two methods) and deals the chunks to the warps in snake order;
//      the other kernels keep the dense order (warp-uniform except at <= 7 bin
//      boundaries per tile) dealt round-robin;
//   4. one thread stores the results with a bulk copy.
// The loops address the stage, the slot words and the log table by 32-bit shared
// addresses computed once (sm_100a shared addresses carry the CTA's
// cluster rank, which ptxas otherwise re-derives per access).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "../../include/bessel_b200.h"
#include "bessel_math.cuh"

namespace b200 {

// Launch shape (overridable only by tools/variant_bench.py experiments).
#ifndef B200_TPB
#define B200_TPB 256
#endif
#ifndef B200_MINB
#define B200_MINB 4          // CTAs per SM for log I (64 registers)
#endif
#ifndef B200_MINB_K
#define B200_MINB_K 4        // CTAs per SM for log K
#endif
#ifndef B200_MINB_IK
#define B200_MINB_IK 4       // CTAs per SM for the fused I + K pass
#endif
#ifndef B200_ITEMS
#define B200_ITEMS 6         // elements per thread per tile (tile = 1536 pairs)
#endif
constexpr int TPB = B200_TPB;
#ifndef B200_ITEMS32
#define B200_ITEMS32 7       // elements per thread per tile in the f32 kernels (6: +3.3% on the f32 grid)
#endif
constexpr int ITEMS = B200_ITEMS;
constexpr int TILE = TPB * ITEMS;       // 1536 pairs per tile
static_assert(TILE <= 4096, "s_idx packs a 12-bit tile index with the bin");
// per-precision tile (f32 stages are half the bytes)
template <typename T> struct TileOf {
    static constexpr int items = sizeof(T) == 4 ? B200_ITEMS32 : B200_ITEMS;
    static constexpr int tile = TPB * items;
    static_assert(items <= 7 && tile <= 4096, "8-bit warp counters, 12-bit tile index");
};
constexpr int BIN_SLOW = 7;           // out-of-range / special inputs (slow_eval)
#ifndef B200_WS
#define B200_WS 0                     // 1: aligned operands take the pipelined kernel (bessel_ws_kernel)
#endif
#ifndef B200_HOMO
#define B200_HOMO 1                   // 1: tiles of a single bin skip the sort
#endif
#ifndef B200_C32
#define B200_C32 0                    // 1: 32-bit bin-counter increments
#endif
#ifndef B200_SADDR
#define B200_SADDR 1                  // 1: the fused f64 loop addresses the stage by 32-bit shared addresses
#endif
#ifndef B200_SADDR2
#define B200_SADDR2 1                 // 1: the same in the other kernels' evaluation loop
#endif
#ifndef B200_HOMOSKIP
#define B200_HOMOSKIP 1               // 1: homogeneous tiles skip the padded-base arithmetic (unused there)
#endif
#ifndef B200_REDUX
#define B200_REDUX 1                  // 1: warp totals by REDUX; the per-thread scan only for mixed tiles (0: scan always)
#endif
#ifndef B200_FULLTILE
#define B200_FULLTILE 1               // 1: full tiles classify without per-element bound checks
#endif
#ifndef B200_C4
#define B200_C4 1                     // 1: 4-bit per-thread bin counters, widened once per thread (0: 64-bit shifts)
#endif
#ifndef B200_PLOOP
#define B200_PLOOP 1                  // 1: the unpadded evaluation loop runs on the slot index (0: element counter)
#endif
#ifndef B200_IFCHAIN1
#define B200_IFCHAIN1 1               // 1: the single-function kernels dispatch mu, U6, U8 by compares (extending the chain to U10/U13 measured slower)
#endif
#ifndef B200_IFCHAIN
#define B200_IFCHAIN 1                // 1: fused pass dispatches the cheap bins by compares (0: jump table only)
#endif

std::atomic<int64_t> g_launches{0};
static thread_local char g_err[256] = "";

int set_err(int code, const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}
int cuda_err(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return B200_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return B200_ERR_CUDA;
}

// Function ids
enum : int { FN_I = 0, FN_K = 1, FN_K_PAPER = 2, FN_IK = 3 };   // FN_IK: both, one pass

#ifndef B200_BLKMAP
#define B200_BLKMAP 1        // 1: a thread bins ITEMS consecutive elements (odd ITEMS; see elem())
#endif
#ifndef B200_SB_ITEMS32
#define B200_SB_ITEMS32 11   // > 0: the f32 kernels on one stage of this many pairs per thread
#endif
#ifndef B200_SB
#define B200_SB 1            // 1: ONE stage buffer per CTA (f64: B200_SB_ITEMS, f32: B200_SB_ITEMS32 per thread)
#endif
#ifndef B200_SB_ITEMS
#define B200_SB_ITEMS 11     // 2816 pairs: 4 CTAs of 56.3 KB (+ 1 KB reserved each) fit the SM's 228 KB
#endif
// Tile shape of one kernel: double-buffered TileOf tiles, or (B200_SB) a
// single buffer of a larger tile -- more chunks per warp between two barriers; the load of
// the next tile is then exposed to this CTA and hidden by the SM's other CTAs
template <typename T, int FN> struct KTile {
    static constexpr bool sb = B200_SB && (sizeof(T) == 8 || B200_SB_ITEMS32 > 0);
    static constexpr int nbuf = sb ? 1 : 2;
    static constexpr int items = !sb ? TileOf<T>::items : sizeof(T) == 8 ? B200_SB_ITEMS : B200_SB_ITEMS32;
    static constexpr int tile = TPB * items;
    static_assert(items <= 15 && tile <= 4096, "4-bit thread counters, 12-bit tile index");
};

// ------------------------------------------------------------------ binning
// bins 0..6 = E_MU, E_UA, E_UB, E_UC, E_U13 (U by term count), fallback split by cost (series:
// x <= 8 / x > 8; K: Temme series x <= 2 / trapezoid x > 2); 7 = the slow bin.
// The fast evaluation paths (fastmath.cuh, SAFE = false) assume the operating
// range 1e-140 <= x <= 1e140, |v| <= 1e140: there every intermediate (1/x,
// v^2 + x^2, 1/rho, the log arguments) is a normal double.  Everything else
// -- non-finite or out-of-domain inputs and finite arguments outside that
// range -- goes to bin 7 and through slow_eval (library functions, rescaling).
// The tests run on the IEEE high words (integer pipe).
// Operating range per precision (R13): f64 [1e-140, 1e140]; f32 [1e-18, 1e18],
// where v^2 + x^2, 1/x, x/(v + rho) and x^2/4 are still normal floats.
template <typename T> struct Range;
template <> struct Range<double> { static constexpr uint32_t lo = B200_HW_LO, hi = B200_HW_HI; };
template <> struct Range<float> { static constexpr uint32_t lo = B200_F32_LO32, hi = B200_F32_HI32; };   // float bits

template <typename T, int FN>
__device__ __forceinline__ int bin_of(T v, T x) {
    constexpr uint32_t LO = Range<T>::lo, HI = Range<T>::hi;
    uint32_t hx, hvs;
    if constexpr (sizeof(T) == 8) {
        hx = hiw(x);
        hvs = hiw(v);
    } else {                                                            // f32: float bit patterns
        hx = __float_as_uint(x);
        hvs = __float_as_uint(v);
    }
    const uint32_t hv = hvs & 0x7FFFFFFFu;
    // x outside the range (or <= 0, NaN), |v| above it (inf, NaN), v < 0 for I (-0.0 is
    // handled there): one predicate and a final select, no early-return branches
    // I (alone or fused) needs v >= 0: a set sign bit puts the raw high word above HI, so
    // one unsigned compare covers |v| > range, NaN, v < 0 and -0.0 (K takes |v|)
    const bool slow = (hx - LO > HI - LO) | ((FN == FN_I || FN == FN_IK) ? hvs > HI : hv > HI);
    int e;
    if constexpr (sizeof(T) == 8)
        e = select_eval_hw(fabs(v), x, hv, hx, (FN == FN_I) ? B200_HW_X8 : B200_HW_X2);
    else
        e = select_eval_f32(fabsf(v), x, hv, hx, (FN == FN_I) ? B200_F32_X8 : B200_F32_X2);
    return slow ? BIN_SLOW : e;
}

// The slow bin: IEEE special cases, then the full-range (SAFE) evaluation.
template <typename T, int FN>
__device__ __noinline__ T slow_eval(T v, T x) {
    const T nan = T(CUDART_NAN);
    if (isnan(v) || isnan(x) || x < T(0)) return nan;
    if (FN == FN_I) {
        if (v < T(0)) return nan;
        if (x == T(0)) return v == T(0) ? T(0) : T(-CUDART_INF);
        if (isinf(v)) return T(-CUDART_INF);           // I_inf(x) = 0
        if (isinf(x)) return T(CUDART_INF);
        v = fabs(v);                                   // -0.0
        return log_iv_eval<T, true>(select_eval(double(v), double(x), B200_HW_X8), v, x);
    } else {
        if (x == T(0)) return T(CUDART_INF);           // pole
        if (isinf(v)) return T(CUDART_INF);
        if (isinf(x)) return T(-CUDART_INF);
        v = fabs(v);
        return log_kv_eval<T, FN == FN_K_PAPER, true>(select_eval(double(v), double(x), B200_HW_X2), v, x);
    }
}

template <typename T, int FN>
__device__ __forceinline__ T eval_bin(int bin, T v, T x, uint32_t tab) {
#ifdef B200_EVAL_NOP
    if (bin != BIN_SLOW) return v + x;   // experiment only: measures the tile machinery alone
#endif
#if B200_IFCHAIN1
    // the cheap bins by compare-and-branch (chunk-uniform after the sort), then the jump table
    if (FN == FN_I) {
        if (bin == E_MU) return log_bessel_mu<T, false, false>(v, x, tab);
        if (bin == E_UA) return log_bessel_u<T, false, KUs<T>::A, false>(v, x, tab);
        if (bin == E_UB) return log_bessel_u<T, false, KUs<T>::B, false>(v, x, tab);
    } else {
        if (bin == E_MU) return log_bessel_mu<T, true, false>(fabs(v), x, tab);
        if (bin == E_UA) return log_bessel_u<T, true, KUs<T>::A, false>(fabs(v), x, tab);
        if (bin == E_UB) return log_bessel_u<T, true, KUs<T>::B, false>(fabs(v), x, tab);
    }
#endif
    if (FN == FN_I) {
        switch (bin) {
            case E_MU: return log_bessel_mu<T, false, false>(v, x, tab);
            case E_UA: return log_bessel_u<T, false, KUs<T>::A, false>(v, x, tab);
            case E_UB: return log_bessel_u<T, false, KUs<T>::B, false>(v, x, tab);
            case E_UC: return log_bessel_u<T, false, KUs<T>::C, false>(v, x, tab);
            case E_U13: return log_bessel_u<T, false, KUs<T>::D, false>(v, x, tab);
            case E_FB_A:
            case E_FB_B: return log_iv_series<T, false>(v, x, tab);
            default: return slow_eval<T, FN>(v, x);
        }
    }
    const T av = fabs(v);
    switch (bin) {
        case E_MU: return log_bessel_mu<T, true, false>(av, x, tab);
        case E_UA: return log_bessel_u<T, true, KUs<T>::A, false>(av, x, tab);
        case E_UB: return log_bessel_u<T, true, KUs<T>::B, false>(av, x, tab);
        case E_UC: return log_bessel_u<T, true, KUs<T>::C, false>(av, x, tab);
        case E_U13: return log_bessel_u<T, true, KUs<T>::D, false>(av, x, tab);
        case E_FB_A:
        case E_FB_B: return FN == FN_K_PAPER ? log_kv_integral_paper<T>(av, x) : log_kv_fallback<T, false>(av, x, tab);
        default: return slow_eval<T, FN>(v, x);
    }
}

// Fused I + K: both results of one element (bins as for K, v >= 0 or slow).
template <typename T>
__device__ __forceinline__ void eval_bin_ik(int bin, T v, T x, T &ri, T &rk, uint32_t tab) {
#ifdef B200_EVAL_NOP
    if (bin != BIN_SLOW) { ri = v + x; rk = v - x; return; }
#endif
#if B200_IFCHAIN
    // the cheap bins by compare-and-branch (warp-uniform after the sort); no jump table
    if (bin == E_MU) { log_bessel_mu_ik<T>(v, x, ri, rk, tab); return; }
    if (bin == E_UA) { log_bessel_u_ik<T, KUs<T>::A>(v, x, ri, rk, tab); return; }
    if (bin == E_UB) { log_bessel_u_ik<T, KUs<T>::B>(v, x, ri, rk, tab); return; }
    if (bin == E_UC) { log_bessel_u_ik<T, KUs<T>::C>(v, x, ri, rk, tab); return; }
    if (bin == E_U13) { log_bessel_u_ik<T, KUs<T>::D>(v, x, ri, rk, tab); return; }
#endif
    switch (bin) {
        case E_MU: log_bessel_mu_ik<T>(v, x, ri, rk, tab); break;
        case E_UA: log_bessel_u_ik<T, KUs<T>::A>(v, x, ri, rk, tab); break;
        case E_UB: log_bessel_u_ik<T, KUs<T>::B>(v, x, ri, rk, tab); break;
        case E_UC: log_bessel_u_ik<T, KUs<T>::C>(v, x, ri, rk, tab); break;
        case E_U13: log_bessel_u_ik<T, KUs<T>::D>(v, x, ri, rk, tab); break;
        case E_FB_B:   // 2 < x <= 30
#ifndef B200_IK_SERIES   // experiment switch: the power series for I on this band too
            log_ivkv_trap<T>(v, x, ri, rk, tab);   // I from the K values (Wronskian + Miller ratio)
            break;
#endif
        case E_FB_A:   // x <= 2
#ifndef B200_IK_SERIES_A
            // v < 1/2 keeps the power series: there |log I| can be << 1 (log I_0(x) ~ x^2/4)
            // and log I = -log K_mu - log(...) would cancel to an absolute, not relative,
            // error (R1).  f32: from x = 0.1, where the Miller values stay below
            // ~(2 (v + M) / x)^M < 2e18 and K_{v+1} / K_mu < 1e27 (FLT_MAX 3.4e38)
            if (x >= T(sizeof(T) == 8 ? 1e-6 : 0.1) && x <= T(2) && v >= T(0.5)) {
                log_ivkv_trap<T, true>(v, x, ri, rk, tab);   // Temme K values, Wronskian + Miller ratio
                break;
            }
#endif
            ri = log_iv_series<T, false>(v, x, tab);
            rk = log_kv_fallback<T, false>(v, x, tab);
            break;
        default:
            ri = slow_eval<T, FN_I>(v, x);
            rk = slow_eval<T, FN_K>(v, x);
    }
}

// Counting-sort helpers.  A thread bins ITEMS <= 8 elements, so per-thread and
// warp-inclusive counts (<= 32 * ITEMS <= 255) fit 8-bit fields: all 8 bins in
// one 64-bit word, scanned across the warp with 64-bit shuffles.  Across warps
// (counts up to TILE) the fields are widened to 16 bits, bins 0-3 / 4-7.
__device__ __forceinline__ uint64_t widen_lo(uint64_t c8) {   // bytes 0..3 -> 16-bit fields
    const uint32_t a = uint32_t(c8);
    return uint64_t(__byte_perm(a, 0, 0x4140)) | (uint64_t(__byte_perm(a, 0, 0x4342)) << 32);
}
__device__ __forceinline__ uint64_t widen_hi(uint64_t c8) {   // bytes 4..7 -> 16-bit fields
    const uint32_t a = uint32_t(c8 >> 32);
    return uint64_t(__byte_perm(a, 0, 0x4140)) | (uint64_t(__byte_perm(a, 0, 0x4342)) << 32);
}
__device__ __forceinline__ uint64_t shfl_up64(uint64_t v, int o) { return __shfl_up_sync(0xffffffffu, v, o); }
__device__ __forceinline__ uint64_t shfl64(uint64_t v, int l) { return __shfl_sync(0xffffffffu, v, l); }

static_assert(ITEMS <= 7, "8-bit warp-level bin counters hold at most 255 = 32 * 7 + 31");

// ------------------------------------------------------------------ async copies
// Tiles move HBM <-> shared memory with the bulk-copy (TMA) engine: one thread
// issues a 1-D cp.async.bulk per array, completion is tracked by an mbarrier
// (loads) or a bulk group (stores).  Pointers that are only 8-byte aligned
// fall back to per-thread cp.async (LDGSTS) loads and plain stores.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
// 32-bit shared-memory accesses (B200_SADDR): volatile, so they keep their order
// relative to the barriers and to each other
__device__ __forceinline__ uint32_t opaque_u32(uint32_t a) {
    asm volatile("mov.b32 %0, %0;" : "+r"(a));
    return a;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double r;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float r;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
template <typename T> __device__ __forceinline__ T lds_t(uint32_t a) {
    if constexpr (sizeof(T) == 8) return lds_f64(a); else return lds_f32(a);
}
template <typename T> __device__ __forceinline__ void sts_t(uint32_t a, T v) {
    if constexpr (sizeof(T) == 8) sts_f64(a, v); else sts_f32(a, v);
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short r;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "B200_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra B200_WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int BYTES>
__device__ __forceinline__ void cp_async(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------------ evaluation kernel
// Persistent CTAs, tiles of TILE consecutive pairs, per tile:
//   0. (one thread) start the bulk load of the NEXT tile into the other half of
//      a double-buffered stage (v, x in tile order), so HBM reads overlap the
//      whole current tile;
//   1. wait for this tile's stage; every thread bins its ITEMS elements
//      (classification only -- values stay in the stage);
//   2. counting sort of the element indices by bin (packed 8-bit counters,
//      warp shuffles; every warp derives its own offsets from the per-warp
//      totals, no extra barrier);
//   3. every warp evaluates 32 consecutive sorted slots (warp-uniform method
//      except at <= 7 bin boundaries per tile), reading (v, x) from the stage
//      through the index and writing the result(s) over that element's own
//      (v, x) slots (each element is read and written by one thread only);
//   4. (one thread) bulk store of the stage's result arrays to HBM; the
//      buffer is reloaded only after the store has read it.
// The f64 kernels (KTile::sb) instead keep ONE stage of 2816 pairs and load the
// next tile after step 4: each warp then evaluates ~11 chunks between two barriers
// instead of ~6, which halves the barrier waits of tiles mixing costly and cheap bins;
// the exposed load is hidden by the SM's other three CTAs.
#ifndef B200_PAD
#define B200_PAD 1           // 1: f64 fused pass: sort keys costliest first, bins padded to 32-slot chunks
#endif
// slots of the sorted order: TILE, plus up to 8 * 31 = 248 padding slots (B200_PAD: every
// one of the 8 keys rounded up to a multiple of 32)
template <typename T, int FN> constexpr int idx_slots() { return KTile<T, FN>::tile + (B200_PAD && sizeof(T) == 8 ? 256 : 0); }
template <typename T, int FN>
constexpr int smem_bytes() {   // stage[nbuf][2][TILE] + idx
    return 2 * KTile<T, FN>::nbuf * KTile<T, FN>::tile * int(sizeof(T)) + idx_slots<T, FN>() * 2;
}

#ifndef B200_MINB32
#define B200_MINB32 6        // CTAs per SM for the f32 kernels (40 registers; 4 and 5 measured slower)
#endif
template <typename T, int FN, bool TMA>
__global__ void __launch_bounds__(TPB, sizeof(T) == 4 ? B200_MINB32 : FN == FN_I ? B200_MINB : FN == FN_IK ? B200_MINB_IK : B200_MINB_K)
    bessel_eval_kernel(const T *__restrict__ vin, const T *__restrict__ xin, T *__restrict__ out,
                       T *__restrict__ out2, int64_t n) {
    constexpr int NOUT = FN == FN_IK ? 2 : 1;         // results per element (out, out2)
    constexpr int ITEMS = KTile<T, FN>::items, TILE = KTile<T, FN>::tile;   // shadow the f64 defaults
    constexpr int NBUF = KTile<T, FN>::nbuf;
    constexpr bool W16 = ITEMS > 7;                   // warp sums need 16-bit fields (> 255 per key)
    // padded, costliest-first sort order with snake chunk dealing: the f64 fused pass only
    // (measured: it gains on tiles mixing the fallback with cheap bins; the f32 and
    // single-function kernels, whose fallback is cheap, lose 2-3% to the extra work)
    constexpr bool PADK = B200_PAD && sizeof(T) == 8 && FN == FN_IK;
    // dynamic shared memory (smem_bytes<T, FN>()): stage[2][2][TILE], idx[TILE]
    extern __shared__ __align__(128) unsigned char s_dyn[];
    auto s_stage = reinterpret_cast<T (*)[2][TILE]>(s_dyn);                       // [buffer][v|x][element]
    uint16_t *s_idx = reinterpret_cast<uint16_t *>(s_dyn + 2 * NBUF * TILE * sizeof(T));
    __shared__ uint64_t s_wtot[(W16 ? 2 : 1) * TPB / 32];   // per-warp bin totals, 8-bit (W16: 16-bit) fields
    __shared__ alignas(8) uint64_t s_bar[2];

    constexpr int VEC = 16 / int(sizeof(T));          // elements per 16 bytes (bulk-copy granule)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    fm_tables_init();   // the f64 log table (the f32 kernels use it in the double K recurrence)
    // its shared address, computed once and held where the compiler cannot re-derive it
    const uint32_t tab = opaque_u32(logtab_addr());
    auto tile_rem = [&](int64_t t) { return int(n - t * TILE < TILE ? n - t * TILE : TILE); };
    // the tile elements a thread loads (cp.async, ragged tail), bins and scatters.  B200_BLKMAP:
    // ITEMS consecutive elements per thread -- the scatter gives a thread's elements of one
    // key consecutive sorted slots, so a chunk then reads and writes consecutive (v, x)
    // words; with the strided map (tid + i TPB) those words share one bank pair (ITEMS-way
    // conflicts).  ITEMS is odd, so the binning reads (stride ITEMS) stay conflict-free.
    // (An even ITEMS keeps the strided map: with ITEMS = 6 the binning reads would
    // conflict 4-way.)
    auto elem = [&](int i) { return (B200_BLKMAP && (ITEMS & 1)) ? tid * ITEMS + i : tid + i * TPB; };

    // stage tile t into buffer (t / gridDim.x) & 1
    auto issue = [&](int64_t t, int buf) {
        const int rem = tile_rem(t);
        if constexpr (TMA) {
            if (tid == 0) {
                const int ra = rem & ~(VEC - 1);                  // bulk part (multiple of 16 bytes)
                if (NBUF == 1 && NOUT == 2) {
                    // the v half is free once the first store (out, from the v slots) has read
                    // it; the x half waits for the second
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    fence_proxy_async();
                    mbar_expect_tx(&s_bar[buf], uint32_t(2 * ra * sizeof(T)));
                    if (ra > 0) bulk_load(s_stage[buf][0], vin + t * TILE, uint32_t(ra * sizeof(T)), &s_bar[buf]);
                    bulk_wait_read();
                    fence_proxy_async();
                    if (ra > 0) bulk_load(s_stage[buf][1], xin + t * TILE, uint32_t(ra * sizeof(T)), &s_bar[buf]);
                } else {
                    bulk_wait_read();                             // this buffer's results are out
                    fence_proxy_async();
                    mbar_expect_tx(&s_bar[buf], uint32_t(2 * ra * sizeof(T)));
                    if (ra > 0) {
                        bulk_load(s_stage[buf][0], vin + t * TILE, uint32_t(ra * sizeof(T)), &s_bar[buf]);
                        bulk_load(s_stage[buf][1], xin + t * TILE, uint32_t(ra * sizeof(T)), &s_bar[buf]);
                    }
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int j = elem(i);
                if (j < rem) {
                    cp_async<sizeof(T)>(&s_stage[buf][0][j], vin + t * TILE + j);
                    cp_async<sizeof(T)>(&s_stage[buf][1][j], xin + t * TILE + j);
                }
            }
            cp_async_commit();
        }
    };

    if constexpr (TMA) {
        if (tid == 0) {
            mbar_init(&s_bar[0]);
            mbar_init(&s_bar[1]);
            fence_mbar_init();
        }
        __syncthreads();
    }
    if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
    uint32_t parity[2] = {0u, 0u};
    int buf = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= NBUF - 1) {
        const int64_t base = tile * TILE;
        const int rem = tile_rem(tile);
        // 0. prefetch the next tile into the other buffer (its readers finished
        //    before the last barrier of the previous tile)
        if (NBUF == 2 && tile + gridDim.x < ntiles) issue(tile + gridDim.x, buf ^ 1);
        // 1. wait for this tile, bin the owned elements
        T *sv = s_stage[buf][0], *sx = s_stage[buf][1];
        T *s_res[2] = {sv, sx};                    // results overwrite (v, x) of their own element
        if constexpr (TMA) {
            mbar_wait(&s_bar[buf], parity[buf]);
            parity[buf] ^= 1u;
            const int ra = rem & ~(VEC - 1);
            if (ra != rem) {                       // the (< VEC) elements past the bulk part,
#pragma unroll                                     // loaded by the thread that bins them
                for (int i = 0; i < ITEMS; ++i) {
                    const int j = elem(i);
                    if (j >= ra && j < rem) { sv[j] = vin[base + j]; sx[j] = xin[base + j]; }
                }
            }
        } else {
            // own copies of this tile are the older group: wait for all but the newest
            if (NBUF == 2 && tile + gridDim.x < ntiles) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else cp_async_wait_all();
        }
        int lb[ITEMS];
#if B200_C32
        static_assert(!PADK, "B200_C32 counts bins, B200_PAD sort keys");
        // packed 8-bit counters, incremented with 32-bit operations (a variable
        // 64-bit shift costs ~4 more instructions per element)
        uint32_t clo = 0, chi = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int j = elem(i);
            lb[i] = -1;
            if (j < rem) {
                const int b = bin_of<T, FN>(sv[j], sx[j]);
                lb[i] = b;
                const uint32_t inc = 1u << (8 * (b & 3));
                if (b < 4) clo += inc; else chi += inc;
            }
        }
        const uint64_t c8 = (uint64_t(chi) << 32) | clo;
#else
#if B200_C4
        // 4-bit per-thread counters (ITEMS <= 7 < 16 per key), one 32-bit shift and add per
        // element; widened once per thread to the 8-bit fields of the warp scan: the even
        // keys' nibbles go to bytes 0, 2, 4, 6 and the odd keys' to bytes 1, 3, 5, 7
        uint32_t c4 = 0;
#if B200_FULLTILE
        if (rem == TILE) {                         // every tile but the last: no bound checks
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int j = elem(i);
                lb[i] = bin_of<T, FN>(sv[j], sx[j]);
                c4 += 1u << (PADK ? 28 - 4 * lb[i] : 4 * lb[i]);
            }
        } else
#endif
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int j = elem(i);
            lb[i] = -1;
            if (j < rem) {
                lb[i] = bin_of<T, FN>(sv[j], sx[j]);
                c4 += 1u << (PADK ? 28 - 4 * lb[i] : 4 * lb[i]);     // PADK: sort key 7 - bin, costliest first
            }
        }
        const uint32_t ev = c4 & 0x0F0F0F0Fu, od = (c4 >> 4) & 0x0F0F0F0Fu;
        const uint64_t c8 = uint64_t(__byte_perm(ev, od, 0x5140)) | (uint64_t(__byte_perm(ev, od, 0x7362)) << 32);
#else
        uint64_t c8 = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int j = elem(i);
            lb[i] = -1;
            if (j < rem) {
                lb[i] = bin_of<T, FN>(sv[j], sx[j]);
                c8 += 1ull << (PADK ? 56 - 8 * lb[i] : 8 * lb[i]);   // PADK: sort key 7 - bin, costliest first
            }
        }
#endif
#endif
#if B200_REDUX
        // 2. per-warp totals (8-bit fields: <= 32 * 7 per key, no carries between fields)
        //    by two 32-bit REDUX sums; the per-thread warp scan is needed only by the
        //    scatter of a mixed tile (below)
        if constexpr (W16) {
            // per-thread 16-bit fields (keys 0-3 | 4-7), four 32-bit REDUX sums
            const uint64_t wl = widen_lo(c8), wh = widen_hi(c8);
            const uint32_t a0 = __reduce_add_sync(0xffffffffu, uint32_t(wl));
            const uint32_t a1 = __reduce_add_sync(0xffffffffu, uint32_t(wl >> 32));
            const uint32_t a2 = __reduce_add_sync(0xffffffffu, uint32_t(wh));
            const uint32_t a3 = __reduce_add_sync(0xffffffffu, uint32_t(wh >> 32));
            if (lane == 0) {
                s_wtot[2 * warp] = (uint64_t(a1) << 32) | a0;
                s_wtot[2 * warp + 1] = (uint64_t(a3) << 32) | a2;
            }
        } else {
            const uint32_t tl = __reduce_add_sync(0xffffffffu, uint32_t(c8));
            const uint32_t th = __reduce_add_sync(0xffffffffu, uint32_t(c8 >> 32));
            if (lane == 0) s_wtot[warp] = (uint64_t(th) << 32) | tl;
        }
        __syncthreads();
#else
        // 2. warp-inclusive scan of the packed counts, per-warp totals to smem
        uint64_t incl = c8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = shfl_up64(incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wtot[warp] = incl;
        __syncthreads();
#endif
        uint64_t plo = 0, phi = 0;
        int homo = 0;                // tile-homogeneous: 1 + its sort key (CTA-uniform)
        int nchunk = 0;              // B200_PAD: 32-slot chunks of the padded sorted order
        {
            // lanes 0..NW-1 of every warp scan the per-warp totals (16-bit fields);
            // the warp keeps the exclusive prefix of its own index
            constexpr int NW = TPB / 32;
            uint64_t lo, hi;
            if constexpr (W16) {
                lo = lane < NW ? s_wtot[2 * lane] : 0ull;
                hi = lane < NW ? s_wtot[2 * lane + 1] : 0ull;
            } else {
                const uint64_t t8 = lane < NW ? s_wtot[lane] : 0ull;
                lo = widen_lo(t8);
                hi = widen_hi(t8);
            }
            uint64_t ilo = lo, ihi = hi;
#pragma unroll
            for (int o = 1; o < NW; o <<= 1) {
                const uint64_t ylo = shfl_up64(ilo, o), yhi = shfl_up64(ihi, o);
                if (lane >= o) { ilo += ylo; ihi += yhi; }
            }
            const uint64_t tlo = shfl64(ilo, NW - 1), thi = shfl64(ihi, NW - 1);   // tile totals per bin
            // exclusive prefix over bins: field k of (x * 0x0001000100010001) is sum_{j<=k}
            constexpr uint64_t ONES = 0x0001000100010001ull;
#if B200_HOMO
            {
                // one bin holds all rem elements <=> a 16-bit field equals rem (fields < 2^15)
                constexpr uint64_t H = 0x8000800080008000ull;
                const uint64_t r4 = uint64_t(rem) * ONES;
                const uint64_t zl = tlo ^ r4, zh = thi ^ r4;
                const uint64_t ml = (zl - ONES) & ~zl & H, mh = (zh - ONES) & ~zh & H;
                if (ml | mh) homo = 1 + (ml ? (__ffsll(ml) - 16) >> 4 : 4 + ((__ffsll(mh) - 16) >> 4));
            }
#endif
            // PADK: key k = 7 - bin (the costliest bins first), and in a mixed tile each
            // key's run of slots starts on a 32-slot chunk boundary (sizes rounded up to
            // multiples of 32: fields < 2^15, no carries), so no warp evaluates two methods
            // in one chunk (a chunk mixing the fallback with a cheap bin runs the fallback's
            // ~1000 instructions beside the other method); the padding slots hold 0xFFFF.
            constexpr uint64_t F32 = 0xFFE0FFE0FFE0FFE0ull;
            uint64_t blo, bhi;
            if constexpr (PADK) {
#if B200_HOMOSKIP
              if (homo) {
                blo = bhi = 0;                                                     // unused: no scatter
              } else {
#endif
                // (a homogeneous tile computes the padded bases too and does not use them)
                const uint64_t qlo = (tlo + 31 * ONES) & F32, qhi = (thi + 31 * ONES) & F32;
                const uint64_t tp = qlo * ONES;
                blo = tp - qlo;                                                    // padded bases of keys 0..3
                bhi = qhi * ONES - qhi + (tp >> 48) * ONES;                        // padded bases of keys 4..7
                nchunk = int(((bhi + qhi) >> 48) >> 5);                            // chunks of the padded order
                // warp w fills the padding after key w: slots [base + count, base + round32(count))
                const int sh = 16 * (warp & 3);
                const int kb = int(((warp < 4 ? blo : bhi) >> sh) & 0xFFFFull);
                const int kc = int(((warp < 4 ? tlo : thi) >> sh) & 0xFFFFull);
                const int g = kb + kc + lane;
                if (!homo && g < kb + ((kc + 31) & ~31)) s_idx[g] = uint16_t(0xFFFF);
#if B200_HOMOSKIP
              }
#endif
            } else {
                const uint64_t tp = tlo * ONES;
                blo = tp - tlo;                                                    // bases of bins 0..3
                bhi = thi * ONES - thi + (tp >> 48) * ONES;                        // bases of bins 4..7
            }
#if B200_REDUX
            if (W16 && !homo) {
                // warp scan on the 16-bit fields (two words)
                const uint64_t cl = widen_lo(c8), ch = widen_hi(c8);
                uint64_t xl = cl, xh = ch;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t yl = shfl_up64(xl, o), yh = shfl_up64(xh, o);
                    if (lane >= o) { xl += yl; xh += yh; }
                }
                const uint64_t wlo = shfl64(blo + ilo - lo, warp), whi = shfl64(bhi + ihi - hi, warp);
                plo = wlo + (xl - cl);
                phi = whi + (xh - ch);
            } else if (!homo) {   // CTA-uniform: full-warp shuffles below
                uint64_t incl = c8;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t y = shfl_up64(incl, o);
                    if (lane >= o) incl += y;
                }
#else
            {
#endif
                const uint64_t wlo = shfl64(blo + ilo - lo, warp), whi = shfl64(bhi + ihi - hi, warp);
                // this thread's first slot per bin: warp offset + warp-exclusive count
                const uint64_t ex8 = incl - c8;
                plo = wlo + widen_lo(ex8);
                phi = whi + widen_hi(ex8);
            }
        }
        if (!homo) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int b = lb[i];
                if (b >= 0) {
                    const int kk = PADK ? 7 - b : b;
                    const int sh = 16 * (kk & 3);
                    const uint64_t word = kk < 4 ? plo : phi;
                    const int pos = int((word >> sh) & 0xFFFFull);
                    if (kk < 4) plo += 1ull << sh; else phi += 1ull << sh;
                    s_idx[pos] = uint16_t(elem(i) | (b << 12));   // tile index | bin
                }
            }
            __syncthreads();
        }
        // a homogeneous tile needs no sort: slot p = element p.  Its binning reads all precede
        // the barrier after the warp totals, and each element is then read and overwritten
        // by the one thread that evaluates its slot
        static_assert(!PADK || TPB / 32 == 8, "one warp per sort key fills that key's padding");
        const int hw = (PADK ? 7 - (homo - 1) : homo - 1) << 12;   // the tile's one bin (PADK: 7 - key)
        if constexpr (PADK) {
            // 3. evaluate the 32-slot chunks of the sorted order, dealt to the warps in
            //    snake order (w, 15 - w, 16 + w, 31 - w, ...): the costliest chunks come
            //    first and each round of eight runs opposite to the previous one.  A padded
            //    order spans up to TILE + 8 * 31 slots; its padding slots (0xFFFF) are skipped.
            //    On slot indices p = 32 c + lane the snake step needs neither the warp nor
            //    the lane: c -> c ^ 15 (16m + w -> 16m + 15 - w) then c -> (c ^ 15) + 16,
            //    i.e. p -> (p ^ 480) + ((p & 256) << 1), starting at p = tid (no SR_TID
            //    re-reads inside the loop).
            const int np = (homo ? (rem + 31) >> 5 : nchunk) << 5;
#pragma unroll 1
#if B200_SADDR
            // 32-bit shared addresses held in registers the compiler cannot re-derive:
            // without this it recomputes the shared window (S2R SR_CgaCtaId, LEA) per element
            const uint32_t a_st = opaque_u32(smem_u32(sv)), a_ix = opaque_u32(smem_u32(s_idx));
#endif
            for (int p = tid; p < np; p = (p ^ 480) + ((p & 256) << 1)) {
#if B200_SADDR
                const int w = homo ? (p < rem ? (p | hw) : 0xFFFF) : int(lds_u16(a_ix + 2 * p));
                if (w == 0xFFFF) continue;
                const uint32_t a = a_st + sizeof(T) * (w & 0xFFF);
                T ri, rk;
                eval_bin_ik<T>(w >> 12, lds_t<T>(a), lds_t<T>(a + sizeof(T) * TILE), ri, rk, tab);
                sts_t<T>(a, ri);
                sts_t<T>(a + sizeof(T) * TILE, rk);
#else
                const int w = homo ? (p < rem ? (p | hw) : 0xFFFF) : s_idx[p];
                if (w == 0xFFFF) continue;
                const int j = w & 0xFFF;
                if constexpr (FN == FN_IK) {
                    eval_bin_ik<T>(w >> 12, sv[j], sx[j], s_res[0][j], s_res[NOUT - 1][j], tab);
                } else {
                    s_res[0][j] = eval_bin<T, FN>(w >> 12, sv[j], sx[j], tab);
                }
#endif
            }
        } else {
            // 3. evaluate: sorted slot p -> element j of the stage (warp w takes the
            //    32-slot chunks w, w + 8, w + 16, w + 24: the expensive high bins at
            //    the end of the order land on different warps)
#if B200_PLOOP
#if B200_SADDR2
            const uint32_t a_st = opaque_u32(smem_u32(sv)), a_ix = opaque_u32(smem_u32(s_idx));
#endif
#pragma unroll 1
            for (int p = tid; p < rem; p += TPB) {   // the slot index is the loop variable
#if B200_SADDR2
                const int w = homo ? (p | hw) : int(lds_u16(a_ix + 2 * p));
                const uint32_t a = a_st + sizeof(T) * (w & 0xFFF);
                if constexpr (FN == FN_IK) {
                    T ri, rk;
                    eval_bin_ik<T>(w >> 12, lds_t<T>(a), lds_t<T>(a + sizeof(T) * TILE), ri, rk, tab);
                    sts_t<T>(a, ri);
                    sts_t<T>(a + sizeof(T) * TILE, rk);
                } else {
                    sts_t<T>(a, eval_bin<T, FN>(w >> 12, lds_t<T>(a), lds_t<T>(a + sizeof(T) * TILE), tab));
                }
#else
                const int w = homo ? (p | hw) : s_idx[p];
                const int j = w & 0xFFF;
                if constexpr (FN == FN_IK) {
                    eval_bin_ik<T>(w >> 12, sv[j], sx[j], s_res[0][j], s_res[NOUT - 1][j], tab);
                } else {
                    s_res[0][j] = eval_bin<T, FN>(w >> 12, sv[j], sx[j], tab);
                }
#endif
            }
#else
#pragma unroll 1
            for (int i = 0; i < ITEMS; ++i) {
                const int p = tid + i * TPB;
                if (p < rem) {
                    const int w = homo ? (p | hw) : s_idx[p];
                    const int j = w & 0xFFF;
                    if constexpr (FN == FN_IK) {
                        eval_bin_ik<T>(w >> 12, sv[j], sx[j], s_res[0][j], s_res[NOUT - 1][j], tab);
                    } else {
                        s_res[0][j] = eval_bin<T, FN>(w >> 12, sv[j], sx[j], tab);
                    }
                }
            }
#endif
        }
        __syncthreads();
        // 4. store
        if constexpr (TMA) {
            const int ra = rem & ~(VEC - 1);
            if (tid == 0 && ra > 0) {
                fence_proxy_async();
                bulk_store(out + base, s_res[0], uint32_t(ra * sizeof(T)));
                if (NOUT == 2) bulk_store(out2 + base, s_res[NOUT - 1], uint32_t(ra * sizeof(T)));
            }
            if (ra != rem && tid < rem - ra) {
                out[base + ra + tid] = s_res[0][ra + tid];
                if (NOUT == 2) out2[base + ra + tid] = s_res[NOUT - 1][ra + tid];
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int j = elem(i);
                if (j < rem) {
                    __stcs(out + base + j, s_res[0][j]);
                    if (NOUT == 2) __stcs(out2 + base + j, s_res[NOUT - 1][j]);
                }
            }
        }
        // single buffer: reload it once the store has read it (bulk_wait_read in issue; the
        // cp.async path: every thread reloads only the slots it just stored).  A ragged
        // tile is the last one, so the per-thread tail stores above never race the reload.
        if (NBUF == 1 && tile + gridDim.x < ntiles) issue(tile + gridDim.x, 0);
    }
    if constexpr (TMA) {
        if (tid == 0) bulk_wait_all();
    }
}

// ------------------------------------------------------------------ pipelined kernel
// The bench path (16-byte aligned operands): one CTA of 32 warps per SM, a ring
// of NST tile stages in shared memory, and no CTA-wide barrier in the steady
// state.  Per stage four mbarriers order the hand-offs:
//   full  (TMA transaction count)   tile's (v, x) landed
//   cnt   (32 warp arrivals)        every warp binned its share, warp totals posted
//   idx   (32 warp arrivals)        every warp scattered its indices (tile sorted)
//   done  (32 warp arrivals)        every warp stopped evaluating the tile
// Each warp runs, for the k-th tile of its CTA,
//   count(k+2)   bin its 1-2 elements of tile k+2 (Algorithm 1 dispatch), warp scan
//   eval(k)      claim 32-slot chunks of the sorted tile k from a shared counter
//                until none is left (dynamic balance; the sort puts the most
//                expensive bins first, longest-processing-time order)
//   scatter(k+2) from the 32 warp totals: its elements' sorted positions
// so a warp that finishes early starts the next tile instead of waiting at a
// barrier: the waits (cnt of k+2 across one eval phase, idx of k+1 across one
// iteration) have a whole evaluation phase of slack.  Thread 0 (warp 0) moves
// the data: at iteration k it waits done(k-2), bulk-stores tile k-2's results
// (in place over its (v, x)) and, once tile k-3's store has read its stage,
// bulk-loads tile k+3 into that stage.  Six stages: k-3 (store reading), k-2,
// k-1 (finishing), k (evaluated), k+1 (sorted), k+2 (binned/scattered), with
// k+3 loading into the stage of k-3.
namespace wsk {
constexpr int NWARP = 32;
constexpr int NTHR = NWARP * 32;          // 1024 threads: one CTA per SM, 64 registers each
constexpr int WTILE = 1536;               // pairs per tile
constexpr int NST = 6;                    // ring stages
constexpr int NCH = WTILE / 32;           // 32-slot chunks per tile
static_assert(WTILE <= 2 * NTHR, "count/scatter handle at most two elements per thread");
static_assert(WTILE <= 4096, "s_idx packs a 12-bit tile index with the bin");
template <typename T>
__host__ __device__ constexpr int data_bytes() { return NST * 2 * WTILE * int(sizeof(T)); }
constexpr int IDX_OFF_BYTES = NST * WTILE * 2;
template <typename T>
__host__ __device__ constexpr int smem_bytes() {
    // data[NST][2][WTILE] T | idx[NST][WTILE] u16 | tot[NST][NWARP] u64 | pre[NTHR] u64 |
    // bar[4][NST] u64 | claim[NST] int | bin[WTILE] u8
    return data_bytes<T>() + IDX_OFF_BYTES + NST * NWARP * 8 + NTHR * 8 + 4 * NST * 8 + NST * 4 + WTILE;
}
}  // namespace wsk

__device__ __forceinline__ void mbar_init_n(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store_nc(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

template <typename T, int FN>
__global__ void __launch_bounds__(wsk::NTHR, 1)
    bessel_ws_kernel(const T *__restrict__ vin, const T *__restrict__ xin, T *__restrict__ out, T *__restrict__ out2,
                     int64_t n) {
    using namespace wsk;
    constexpr int NOUT = FN == FN_IK ? 2 : 1;
    constexpr int VEC = 16 / int(sizeof(T));
    extern __shared__ __align__(128) unsigned char s_dyn[];
    auto s_data = reinterpret_cast<T (*)[2][WTILE]>(s_dyn);                                  // [stage][v|x][elem]
    auto s_idx = reinterpret_cast<uint16_t (*)[WTILE]>(s_dyn + data_bytes<T>());
    unsigned char *p8 = s_dyn + data_bytes<T>() + IDX_OFF_BYTES;
    auto s_tot = reinterpret_cast<uint64_t (*)[NWARP]>(p8);                                  // per-warp bin totals
    uint64_t *s_pre = reinterpret_cast<uint64_t *>(p8 + NST * NWARP * 8);                   // per-thread prefix
    uint64_t *s_bar = s_pre + NTHR;                                                           // [4][NST]
    uint64_t *b_full = s_bar, *b_cnt = s_bar + NST, *b_idx = s_bar + 2 * NST, *b_done = s_bar + 3 * NST;
    int *s_claim = reinterpret_cast<int *>(s_bar + 4 * NST);
    uint8_t *s_bin = reinterpret_cast<uint8_t *>(s_claim + NST);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + WTILE - 1) / WTILE;
    const int64_t K = int64_t(blockIdx.x) < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (tid == 0) {
        for (int st = 0; st < NST; ++st) {
            mbar_init_n(&b_full[st], 1);
            mbar_init_n(&b_cnt[st], NWARP);
            mbar_init_n(&b_idx[st], NWARP);
            mbar_init_n(&b_done[st], NWARP);
            s_claim[st] = 0;
        }
        fence_mbar_init();
    }
    fm_tables_init();   // log table to shared memory; ends with __syncthreads (covers the inits above)
    const uint32_t tab = logtab_addr();
    auto tile_of = [&](int64_t k) { return int64_t(blockIdx.x) + k * int64_t(gridDim.x); };
    auto rem_of = [&](int64_t t) { return int(n - t * WTILE < WTILE ? n - t * WTILE : WTILE); };
    auto par = [](int64_t k) { return uint32_t((k / NST) & 1); };

    // thread 0: bulk loads / stores (one commit group per stored tile)
    auto load = [&](int64_t k) {
        const int st = int(k % NST);
        const int64_t t = tile_of(k);
        const int ra = rem_of(t) & ~(VEC - 1);
        mbar_expect_tx(&b_full[st], uint32_t(2 * ra * sizeof(T)));
        if (ra > 0) {
            bulk_load(s_data[st][0], vin + t * WTILE, uint32_t(ra * sizeof(T)), &b_full[st]);
            bulk_load(s_data[st][1], xin + t * WTILE, uint32_t(ra * sizeof(T)), &b_full[st]);
        }
    };
    auto store = [&](int64_t k) {
        const int st = int(k % NST);
        mbar_wait(&b_done[st], par(k));
        const int64_t t = tile_of(k);
        const int rem = rem_of(t), ra = rem & ~(VEC - 1);
        fence_proxy_async();
        if (ra > 0) {
            bulk_store_nc(out + t * WTILE, s_data[st][0], uint32_t(ra * sizeof(T)));
            if (NOUT == 2) bulk_store_nc(out2 + t * WTILE, s_data[st][1], uint32_t(ra * sizeof(T)));
        }
        bulk_commit();
        for (int j = ra; j < rem; ++j) {          // < VEC elements past the bulk part
            out[t * WTILE + j] = s_data[st][0][j];
            if (NOUT == 2) out2[t * WTILE + j] = s_data[st][1][j];
        }
        s_claim[st] = 0;                          // the stage's next tile claims from 0
    };

    // count: bin this thread's elements of tile k, warp scan, post the warp totals
    auto count = [&](int64_t k) {
        const int st = int(k % NST);
        const int64_t t = tile_of(k);
        const int rem = rem_of(t), ra = rem & ~(VEC - 1);
        mbar_wait(&b_full[st], par(k));
        T *sv = s_data[st][0], *sx = s_data[st][1];
        uint64_t c8 = 0;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int j = tid + i * NTHR;
            if (j < rem) {
                if (j >= ra) { sv[j] = vin[t * WTILE + j]; sx[j] = xin[t * WTILE + j]; }   // tail past the bulk part
                const int b = bin_of<T, FN>(sv[j], sx[j]);
                c8 += 1ull << (8 * (7 - b));      // key 7 - b: expensive bins sort first
                s_bin[j] = uint8_t(b);
            }
        }
        uint64_t incl = c8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = shfl_up64(incl, o);
            if (lane >= o) incl += y;
        }
        s_pre[tid] = incl - c8;                   // this thread's warp-exclusive counts (8-bit fields)
        if (lane == 31) s_tot[st][warp] = incl;   // warp totals (<= 64 per key)
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_cnt[st]);
    };

    // scatter: sorted positions of this thread's elements of tile k
    auto scatter = [&](int64_t k) {
        const int st = int(k % NST);
        const int rem = rem_of(tile_of(k));
        mbar_wait(&b_cnt[st], par(k));
        const uint64_t t8 = s_tot[st][lane];      // lane w holds warp w's totals
        const uint64_t lo = widen_lo(t8), hi = widen_hi(t8);
        uint64_t ilo = lo, ihi = hi;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t ylo = shfl_up64(ilo, o), yhi = shfl_up64(ihi, o);
            if (lane >= o) { ilo += ylo; ihi += yhi; }
        }
        const uint64_t tlo = shfl64(ilo, 31), thi = shfl64(ihi, 31);     // tile totals per key
        constexpr uint64_t ONES = 0x0001000100010001ull;
        const uint64_t tp = tlo * ONES;
        const uint64_t blo = tp - tlo;                                     // bases of keys 0..3
        const uint64_t bhi = thi * ONES - thi + (tp >> 48) * ONES;         // bases of keys 4..7
        const uint64_t wlo = shfl64(blo + ilo - lo, warp), whi = shfl64(bhi + ihi - hi, warp);
        const uint64_t ex8 = s_pre[tid];
        uint64_t plo = wlo + widen_lo(ex8), phi = whi + widen_hi(ex8);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int j = tid + i * NTHR;
            if (j < rem) {
                const int b = s_bin[j], key = 7 - b;
                const int sh = 16 * (key & 3);
                const int pos = int(((key < 4 ? plo : phi) >> sh) & 0xFFFFull);
                if (key < 4) plo += 1ull << sh; else phi += 1ull << sh;
                s_idx[st][pos] = uint16_t(j | (b << 12));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_idx[st]);
    };

    // eval: claim 32-slot chunks of the sorted tile k until none is left
    auto eval = [&](int64_t k) {
        const int st = int(k % NST);
        const int rem = rem_of(tile_of(k));
        const int nch = (rem + 31) >> 5;
        mbar_wait(&b_idx[st], par(k));
        T *sv = s_data[st][0], *sx = s_data[st][1];
#pragma unroll 1
        for (;;) {
            int c = 0;
            if (lane == 0) c = atomicAdd(&s_claim[st], 1);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c >= nch) break;
            const int p = (c << 5) + lane;
            if (p < rem) {
                const int w = s_idx[st][p];
                const int j = w & 0xFFF;
                if constexpr (FN == FN_IK) {
                    eval_bin_ik<T>(w >> 12, sv[j], sx[j], sv[j], sx[j], tab);
                } else {
                    sv[j] = eval_bin<T, FN>(w >> 12, sv[j], sx[j], tab);
                }
            }
        }
        fence_proxy_async();                      // results -> visible to the bulk store
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_done[st]);
    };

    if (tid == 0)
        for (int64_t k = 0; k < 3 && k < K; ++k) load(k);
    if (K > 0) { count(0); scatter(0); }
    if (K > 1) { count(1); scatter(1); }
#pragma unroll 1
    for (int64_t k = 0; k < K; ++k) {
        if (tid == 0) {
            if (k >= 2) store(k - 2);
            if (k + 3 < K) {
                bulk_wait_read1();                // tile k-3's store has read the stage k+3 reuses
                fence_proxy_async();
                load(k + 3);
            }
        }
        if (k + 2 < K) count(k + 2);
        eval(k);
        if (k + 2 < K) scatter(k + 2);
    }
    if (tid == 0) {
        for (int64_t k = K >= 2 ? K - 2 : 0; k < K; ++k) store(k);
        bulk_wait_all();
    }
}

#ifdef B200_DIRECT
// Experiment only (tools/variant_bench.py): no staging, no sort -- every thread
// evaluates its own elements straight from global memory.  On method-homogeneous
// inputs this is the floor of the evaluation work alone.
template <typename T, int FN>
__global__ void __launch_bounds__(256, 4)
    bessel_direct_kernel(const T *__restrict__ vin, const T *__restrict__ xin, T *__restrict__ out,
                         T *__restrict__ out2, int64_t n) {
    fm_tables_init();
    const uint32_t tab = logtab_addr();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const T v = __ldcs(vin + i), x = __ldcs(xin + i);
        const int b = bin_of<T, FN>(v, x);
        if constexpr (FN == FN_IK) {
            T ri, rk;
            eval_bin_ik<T>(b, v, x, ri, rk, tab);
            __stcs(out + i, ri);
            __stcs(out2 + i, rk);
        } else {
            __stcs(out + i, eval_bin<T, FN>(b, v, x, tab));
        }
    }
}
#endif

__global__ void classify_kernel(const double *__restrict__ v, const double *__restrict__ x, int8_t *__restrict__ m,
                                int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double vv = v[i], xx = x[i];
        m[i] = (isfinite(vv) && isfinite(xx) && xx >= 0.0 && vv >= 0.0) ? int8_t(select_method(vv, xx)) : int8_t(-1);
    }
}

// ------------------------------------------------------------------ launch
template <typename T, int FN>
static int launch_eval(const T *v, const T *x, T *out, int64_t n, cudaStream_t s, T *out2 = nullptr) {
    if (n < 0) return set_err(B200_ERR_INVALID_ARGUMENT, "n < 0");
    if (n == 0) return B200_OK;
    if (!v || !x || !out || (FN == FN_IK && !out2)) return set_err(B200_ERR_INVALID_ARGUMENT, "null pointer");
    // bulk copies need 16-byte aligned global addresses
    const bool tma = ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(x) |
                       reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(out2)) & 15) == 0;
    constexpr int SMEM = smem_bytes<T, FN>();
    // the dynamic-shared-memory opt-in and the occupancy are per device
    constexpr int MAXDEV = 64;
    static std::atomic<int> occ[2][MAXDEV];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAXDEV)
        return set_err(B200_ERR_NO_DEVICE, "no current CUDA device (or device id >= 64)");
#ifdef B200_DIRECT
    {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        bessel_direct_kernel<T, FN><<<sms * 4, 256, 0, s>>>(v, x, out, out2, n);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cuda_err(cudaGetLastError(), "bessel_direct_kernel launch");
    }
#endif
#if B200_WS
    if (tma) {
        // pipelined kernel: one CTA of wsk::NTHR threads per SM
        static std::atomic<int> ws_ready[MAXDEV];
        constexpr int WSMEM = wsk::smem_bytes<T>();
        if (!ws_ready[dev].load(std::memory_order_relaxed)) {
            cudaError_t e = cudaFuncSetAttribute(bessel_ws_kernel<T, FN>, cudaFuncAttributeMaxDynamicSharedMemorySize, WSMEM);
            if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute (pipelined kernel)");
            ws_ready[dev].store(1, std::memory_order_relaxed);
        }
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
        const int64_t ntiles = (n + wsk::WTILE - 1) / wsk::WTILE;
        const int grid = int(ntiles < sms ? ntiles : sms);
        bessel_ws_kernel<T, FN><<<grid, wsk::NTHR, WSMEM, s>>>(v, x, out, out2, n);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cuda_err(cudaGetLastError(), "bessel_ws_kernel launch");
    }
#endif
    int o = occ[tma][dev].load(std::memory_order_relaxed);
    if (o == 0) {
        auto kern = tma ? bessel_eval_kernel<T, FN, true> : bessel_eval_kernel<T, FN, false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return cuda_err(e, "cudaFuncSetAttribute");
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, TPB, SMEM);
        if (o <= 0) o = 1;
        occ[tma][dev].store(o, std::memory_order_relaxed);
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    const int64_t ntiles = (n + KTile<T, FN>::tile - 1) / KTile<T, FN>::tile;
    const int64_t resident = int64_t(sms) * o;
    const int grid = int(ntiles < resident ? ntiles : resident);
    if (tma)
        bessel_eval_kernel<T, FN, true><<<grid, TPB, SMEM, s>>>(v, x, out, out2, n);
    else
        bessel_eval_kernel<T, FN, false><<<grid, TPB, SMEM, s>>>(v, x, out, out2, n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_err(cudaGetLastError(), "bessel_eval_kernel launch");
}

// ------------------------------------------------------------------ host-buffer pipeline
// Chunks of CH pairs cycle through NSLOT device slots, each with its own
// stream: H2D(v,x) -> kernel -> D2H(out).  Copies of one slot overlap the
// kernel of another and the two copy directions run on separate engines.
#ifndef B200_HOST_NSLOT
#define B200_HOST_NSLOT 4
#endif
#ifndef B200_HOST_CH_LOG2
#define B200_HOST_CH_LOG2 22
#endif

struct HostPipe {
    static constexpr int NSLOT = B200_HOST_NSLOT;
    // 4M pairs per chunk: measured against 0.5M-8M chunks, 3-8 slots, and a
    // ramp of chunk sizes (tools/host_bench.py): larger copies win until the
    // pipeline fill / drain dominates
    static constexpr int64_t CH = int64_t(1) << B200_HOST_CH_LOG2;
    std::mutex mu;
    bool ready = false;
    cudaStream_t st[NSLOT] = {};
    void *buf[NSLOT] = {};   // 4 arrays of CH doubles per slot: v, x, out, out2
};
// one pipeline per device, created on first use and kept for the process lifetime
constexpr int PIPE_MAXDEV = 64;
static HostPipe g_pipes[PIPE_MAXDEV];

template <int FN>
static int host_eval_f64(const double *v_h, const double *x_h, double *out_h, int64_t n, double *out2_h = nullptr) {
    if (n < 0) return set_err(B200_ERR_INVALID_ARGUMENT, "n < 0");
    if (n == 0) return B200_OK;
    if (!v_h || !x_h || !out_h || (FN == FN_IK && !out2_h)) return set_err(B200_ERR_INVALID_ARGUMENT, "null pointer");
    int dev = 0;
    int rc = cuda_err(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    if (dev < 0 || dev >= PIPE_MAXDEV) return set_err(B200_ERR_NO_DEVICE, "device id >= 64");
    HostPipe &g_pipe = g_pipes[dev];
    std::lock_guard<std::mutex> lk(g_pipe.mu);
    if (!g_pipe.ready) {
        for (int i = 0; i < HostPipe::NSLOT; ++i) {
            if ((rc = cuda_err(cudaStreamCreateWithFlags(&g_pipe.st[i], cudaStreamNonBlocking), "stream"))) return rc;
            if ((rc = cuda_err(cudaMalloc(&g_pipe.buf[i], 4 * HostPipe::CH * sizeof(double)), "cudaMalloc"))) return rc;
        }
        g_pipe.ready = true;
    }
    int64_t chunk = 0;
    for (int64_t off = 0; off < n && rc == B200_OK; off += HostPipe::CH, ++chunk) {
        const int slot = int(chunk % HostPipe::NSLOT);
        const int64_t m = (n - off < HostPipe::CH) ? n - off : HostPipe::CH;
        double *dv = static_cast<double *>(g_pipe.buf[slot]);
        double *dx = dv + HostPipe::CH;
        double *dout = dx + HostPipe::CH;
        double *dout2 = dout + HostPipe::CH;
        cudaStream_t s = g_pipe.st[slot];
        if ((rc = cuda_err(cudaMemcpyAsync(dv, v_h + off, m * sizeof(double), cudaMemcpyHostToDevice, s), "H2D")))
            break;
        if ((rc = cuda_err(cudaMemcpyAsync(dx, x_h + off, m * sizeof(double), cudaMemcpyHostToDevice, s), "H2D")))
            break;
        if ((rc = launch_eval<double, FN>(dv, dx, dout, m, s, dout2))) break;
        if ((rc = cuda_err(cudaMemcpyAsync(out_h + off, dout, m * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H")))
            break;
        if (FN == FN_IK &&
            (rc = cuda_err(cudaMemcpyAsync(out2_h + off, dout2, m * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H")))
            break;
    }
    // drain every slot, on success and on error alike: no copy into the caller's
    // buffers may still be running when this returns
    for (int i = 0; i < HostPipe::NSLOT; ++i) {
        const int r = cuda_err(cudaStreamSynchronize(g_pipe.st[i]), "sync");
        if (rc == B200_OK) rc = r;
    }
    return rc;
}

}  // namespace b200

// ====================================================================== C ABI
using namespace b200;

extern "C" {

int b200_log_iv_f64(const double *v, const double *x, double *out, int64_t n, void *stream) {
    return launch_eval<double, FN_I>(v, x, out, n, static_cast<cudaStream_t>(stream));
}
int b200_log_iv_f32(const float *v, const float *x, float *out, int64_t n, void *stream) {
    return launch_eval<float, FN_I>(v, x, out, n, static_cast<cudaStream_t>(stream));
}
int b200_log_kv_f64(const double *v, const double *x, double *out, int64_t n, void *stream) {
    return launch_eval<double, FN_K>(v, x, out, n, static_cast<cudaStream_t>(stream));
}
int b200_log_kv_f32(const float *v, const float *x, float *out, int64_t n, void *stream) {
    return launch_eval<float, FN_K>(v, x, out, n, static_cast<cudaStream_t>(stream));
}
int b200_log_ivkv_f64(const double *v, const double *x, double *out_i, double *out_k, int64_t n, void *stream) {
    return launch_eval<double, FN_IK>(v, x, out_i, n, static_cast<cudaStream_t>(stream), out_k);
}
int b200_log_ivkv_f32(const float *v, const float *x, float *out_i, float *out_k, int64_t n, void *stream) {
    return launch_eval<float, FN_IK>(v, x, out_i, n, static_cast<cudaStream_t>(stream), out_k);
}
int b200_log_kv_paper_f64(const double *v, const double *x, double *out, int64_t n, void *stream) {
    return launch_eval<double, FN_K_PAPER>(v, x, out, n, static_cast<cudaStream_t>(stream));
}

int b200_classify_f64(const double *v, const double *x, int8_t *m, int64_t n, void *stream) {
    if (n < 0) return set_err(B200_ERR_INVALID_ARGUMENT, "n < 0");
    if (n == 0) return B200_OK;
    if (!v || !x || !m) return set_err(B200_ERR_INVALID_ARGUMENT, "null pointer");
    const int64_t blocks64 = (n + 255) / 256;
    const int grid = int(blocks64 < 4096 ? blocks64 : 4096);
    classify_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(v, x, m, n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_err(cudaGetLastError(), "classify_kernel launch");
}

int b200_log_iv_f64_host(const double *v_h, const double *x_h, double *out_h, int64_t n) {
    return host_eval_f64<FN_I>(v_h, x_h, out_h, n);
}
int b200_log_kv_f64_host(const double *v_h, const double *x_h, double *out_h, int64_t n) {
    return host_eval_f64<FN_K>(v_h, x_h, out_h, n);
}
int b200_log_ivkv_f64_host(const double *v_h, const double *x_h, double *out_i_h, double *out_k_h, int64_t n) {
    return host_eval_f64<FN_IK>(v_h, x_h, out_i_h, n, out_k_h);
}

const char *b200_last_error(void) { return g_err; }
int64_t b200_launch_count(void) { return g_launches.load(); }

}  // extern "C"
