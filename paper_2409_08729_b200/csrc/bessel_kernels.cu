// bessel_kernels.cu -- sm_100a kernels and the C ABI of include/bessel_b200.h.
//
// Hot path: batched log I_v(x) / log K_v(x) (§3-§4).  One persistent
// kernel per (function, precision).  Each CTA processes tiles of TILE pairs:
//   1. coalesced load of (v, x) into registers, region id per element
//      (Algorithm 1 with the GPU branch set, plus a cost sub-bin);
//   2. an in-CTA counting sort of the tile by bin (packed 12-bit counters,
//      warp-shuffle scan) into shared memory -- the paper's "sort the input
//      elements based on which expression is used" (§4.3) done
//      per tile in SMEM instead of as a global sort, so no extra HBM pass;
//   3. every warp evaluates 32 consecutive binned elements (warp-uniform
//      method except at <= NBIN-1 bin boundaries per tile);
//   4. results scattered back to tile order in SMEM, coalesced store.
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
#define B200_MINB 4
#endif
#ifndef B200_ITEMS
#define B200_ITEMS 4
#endif
constexpr int TPB = B200_TPB;
constexpr int ITEMS = B200_ITEMS;
constexpr int TILE = TPB * ITEMS;       // 1024 pairs per tile
static_assert(TILE <= 4096, "s_idx packs a 12-bit tile index with the bin");
constexpr int BIN_SLOW = 7;

std::atomic<int64_t> g_launches{0};
static thread_local char g_err[256] = "";

static int set_err(int code, const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}
static int cuda_err(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return B200_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return B200_ERR_CUDA;
}

// Function ids
enum : int { FN_I = 0, FN_K = 1, FN_K_PAPER = 2 };

// ------------------------------------------------------------------ binning
// bins 0..6 = E_MU, E_U4, E_U6, E_U9, E_U13, fallback split by cost (series:
// x <= 8 / x > 8; K: Temme series x <= 2 / trapezoid x > 2); 7 = the slow bin.
// The fast evaluation paths (fastmath.cuh, SAFE = false) assume the operating
// range 1e-140 <= x <= 1e140, |v| <= 1e140: there every intermediate (1/x,
// v^2 + x^2, 1/rho, the log arguments) is a normal double.  Everything else
// -- non-finite or out-of-domain inputs and finite arguments outside that
// range -- goes to bin 7 and through slow_eval (library functions, rescaling).
// The tests run on the IEEE high words (integer pipe).
template <int FN>
__device__ __forceinline__ int bin_of(double v, double x) {
    const uint32_t hx = hiw(x), hvs = hiw(v), hv = hvs & 0x7FFFFFFFu;
    if (hx - B200_HW_LO > B200_HW_HI - B200_HW_LO) return BIN_SLOW;    // x outside [1e-140, 1e140] (or <= 0, NaN)
    if (hv > B200_HW_HI) return BIN_SLOW;                               // |v| > 1e140, inf, NaN
    if (FN == FN_I && hvs != hv) return BIN_SLOW;                       // v < 0 (or -0.0: handled there)
    return select_eval_hw(fabs(v), x, hv, hx, (FN == FN_I) ? B200_HW_X8 : B200_HW_X2);
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
__device__ __forceinline__ T eval_bin(int bin, T v, T x) {
#ifdef B200_EVAL_NOP
    if (bin != BIN_SLOW) return v + x;   // experiment only: measures the tile machinery alone
#endif
    if (FN == FN_I) {
        switch (bin) {
            case E_MU: return log_bessel_mu<T, false, false>(v, x);
            case E_U4: return log_bessel_u<T, false, 4, false>(v, x);
            case E_U6: return log_bessel_u<T, false, 6, false>(v, x);
            case E_U9: return log_bessel_u<T, false, 9, false>(v, x);
            case E_U13: return log_bessel_u<T, false, 13, false>(v, x);
            case E_FB_A:
            case E_FB_B: return log_iv_series<T, false>(v, x);
            default: return slow_eval<T, FN>(v, x);
        }
    }
    const T av = fabs(v);
    switch (bin) {
        case E_MU: return log_bessel_mu<T, true, false>(av, x);
        case E_U4: return log_bessel_u<T, true, 4, false>(av, x);
        case E_U6: return log_bessel_u<T, true, 6, false>(av, x);
        case E_U9: return log_bessel_u<T, true, 9, false>(av, x);
        case E_U13: return log_bessel_u<T, true, 13, false>(av, x);
        case E_FB_A:
        case E_FB_B: return FN == FN_K_PAPER ? log_kv_integral_paper<T>(av, x) : log_kv_fallback<T>(av, x);
        default: return slow_eval<T, FN>(v, x);
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

template <typename T, int FN>
__global__ void __launch_bounds__(TPB, B200_MINB) bessel_eval_kernel(const T *__restrict__ vin, const T *__restrict__ xin,
                                                          T *__restrict__ out, int64_t n) {
    __shared__ T s_v[TILE];
    __shared__ T s_x[TILE];
    __shared__ T s_res[TILE];
    __shared__ uint16_t s_idx[TILE];
    __shared__ uint64_t s_wtot[TPB / 32];          // per-warp bin totals, 8-bit fields
    __shared__ ulonglong2 s_off[TPB / 32];         // per-warp bin offsets, 16-bit fields

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + TILE - 1) / TILE;

    // Software pipeline: the (v, x) of the next tile are loaded into registers
    // while the current tile is binned and evaluated.
    T nv[ITEMS], nx[ITEMS];
    auto prefetch = [&](int64_t t) {
        if (t >= ntiles) return;
        const int64_t base = t * TILE;
        const int rem = int(n - base < TILE ? n - base : TILE);
        const T *pv = vin + base + tid, *px = xin + base + tid;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (tid + i * TPB < rem) {
                nv[i] = __ldcs(pv + i * TPB);
                nx[i] = __ldcs(px + i * TPB);
            }
        }
    };
    prefetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * TILE;
        const int rem = int(n - base < TILE ? n - base : TILE);
        T lv[ITEMS], lx[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) { lv[i] = nv[i]; lx[i] = nx[i]; }
        prefetch(tile + gridDim.x);
        int lb[ITEMS];
        uint64_t c8 = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            lb[i] = -1;
            if (tid + i * TPB < rem) {
                lb[i] = bin_of<FN>(double(lv[i]), double(lx[i]));
                c8 += 1ull << (8 * lb[i]);
            }
        }
        // warp-inclusive scan of the packed counts
        uint64_t incl = c8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = shfl_up64(incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wtot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            // lanes 0..NW-1: exclusive scan over warps of the per-bin totals (16-bit
            // fields), plus the bin bases from the tile totals (lane NW-1)
            constexpr int NW = TPB / 32;
            const uint64_t t8 = lane < NW ? s_wtot[lane] : 0ull;
            const uint64_t lo = widen_lo(t8), hi = widen_hi(t8);
            uint64_t ilo = lo, ihi = hi;
#pragma unroll
            for (int o = 1; o < NW; o <<= 1) {
                const uint64_t ylo = shfl_up64(ilo, o), yhi = shfl_up64(ihi, o);
                if (lane >= o) { ilo += ylo; ihi += yhi; }
            }
            const uint64_t tlo = shfl64(ilo, NW - 1), thi = shfl64(ihi, NW - 1);   // tile totals per bin
            // exclusive prefix over bins: field k of (x * 0x0001000100010001) is sum_{j<=k}
            constexpr uint64_t ONES = 0x0001000100010001ull;
            const uint64_t plo = tlo * ONES;
            const uint64_t blo = plo - tlo;                                        // bases of bins 0..3
            const uint64_t bhi = thi * ONES - thi + (plo >> 48) * ONES;            // bases of bins 4..7
            if (lane < NW) s_off[lane] = make_ulonglong2(blo + ilo - lo, bhi + ihi - hi);
        }
        __syncthreads();
        // this thread's first slot per bin: warp offset + warp-exclusive count
        const ulonglong2 wo = s_off[warp];
        const uint64_t ex8 = incl - c8;
        uint64_t plo = wo.x + widen_lo(ex8), phi = wo.y + widen_hi(ex8);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int b = lb[i];
            if (b >= 0) {
                const int sh = 16 * (b & 3);
                const uint64_t word = b < 4 ? plo : phi;
                const int pos = int((word >> sh) & 0xFFFFull);
                if (b < 4) plo += 1ull << sh; else phi += 1ull << sh;
                s_v[pos] = lv[i];
                s_x[pos] = lx[i];
                s_idx[pos] = uint16_t((tid + i * TPB) | (b << 12));   // tile index | bin
            }
        }
        __syncthreads();
#pragma unroll 1
        for (int i = 0; i < ITEMS; ++i) {
            const int p = tid + i * TPB;
            if (p < rem) {
                const int w = s_idx[p];
                s_res[w & 0xFFF] = eval_bin<T, FN>(w >> 12, s_v[p], s_x[p]);
            }
        }
        __syncthreads();
        // (no trailing barrier: the next tile writes shared memory only after its
        // first barrier, which every thread reaches after this store)
        T *po = out + base + tid;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (tid + i * TPB < rem) __stcs(po + i * TPB, s_res[tid + i * TPB]);
        }
    }
}

__global__ void classify_kernel(const double *__restrict__ v, const double *__restrict__ x, int8_t *__restrict__ m,
                                int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double vv = v[i], xx = x[i];
        m[i] = (isfinite(vv) && isfinite(xx) && xx >= 0.0 && vv >= 0.0) ? int8_t(select_method(vv, xx)) : int8_t(-1);
    }
}

// ------------------------------------------------------------------ launch
static int g_num_sms = 0;
static std::once_flag g_dev_once;

static int device_sms() {
    std::call_once(g_dev_once, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    });
    return g_num_sms;
}

template <typename T, int FN>
static int launch_eval(const T *v, const T *x, T *out, int64_t n, cudaStream_t s) {
    if (n < 0) return set_err(B200_ERR_INVALID_ARGUMENT, "n < 0");
    if (n == 0) return B200_OK;
    if (!v || !x || !out) return set_err(B200_ERR_INVALID_ARGUMENT, "null pointer");
    static int occ = 0;
    if (occ == 0) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, bessel_eval_kernel<T, FN>, TPB, 0);
        occ = o > 0 ? o : 1;
    }
    const int64_t ntiles = (n + TILE - 1) / TILE;
    const int64_t resident = int64_t(device_sms()) * occ;
    const int grid = int(ntiles < resident ? ntiles : resident);
    bessel_eval_kernel<T, FN><<<grid, TPB, 0, s>>>(v, x, out, n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_err(cudaGetLastError(), "bessel_eval_kernel launch");
}

// ------------------------------------------------------------------ host-buffer pipeline
// Chunks of CH pairs cycle through NSLOT device slots, each with its own
// stream: H2D(v,x) -> kernel -> D2H(out).  Copies of one slot overlap the
// kernel of another and the two copy directions run on separate engines.
struct HostPipe {
    static constexpr int NSLOT = 3;
    static constexpr int64_t CH = int64_t(1) << 23;   // 8M pairs per chunk
    std::mutex mu;
    int dev = -1;
    cudaStream_t st[NSLOT] = {};
    void *buf[NSLOT] = {};   // 3 arrays of CH doubles per slot
};
static HostPipe g_pipe;

template <int FN>
static int host_eval_f64(const double *v_h, const double *x_h, double *out_h, int64_t n) {
    if (n < 0) return set_err(B200_ERR_INVALID_ARGUMENT, "n < 0");
    if (n == 0) return B200_OK;
    if (!v_h || !x_h || !out_h) return set_err(B200_ERR_INVALID_ARGUMENT, "null pointer");
    std::lock_guard<std::mutex> lk(g_pipe.mu);
    int dev = 0;
    int rc = cuda_err(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc) return rc;
    if (g_pipe.dev != dev) {
        for (int i = 0; i < HostPipe::NSLOT; ++i) {
            if (g_pipe.buf[i]) cudaFree(g_pipe.buf[i]);
            if (g_pipe.st[i]) cudaStreamDestroy(g_pipe.st[i]);
            g_pipe.buf[i] = nullptr;
            g_pipe.st[i] = nullptr;
        }
        for (int i = 0; i < HostPipe::NSLOT; ++i) {
            if ((rc = cuda_err(cudaStreamCreateWithFlags(&g_pipe.st[i], cudaStreamNonBlocking), "stream"))) return rc;
            if ((rc = cuda_err(cudaMalloc(&g_pipe.buf[i], 3 * HostPipe::CH * sizeof(double)), "cudaMalloc"))) return rc;
        }
        g_pipe.dev = dev;
    }
    int64_t chunk = 0;
    for (int64_t off = 0; off < n; off += HostPipe::CH, ++chunk) {
        const int slot = int(chunk % HostPipe::NSLOT);
        const int64_t m = (n - off < HostPipe::CH) ? n - off : HostPipe::CH;
        double *dv = static_cast<double *>(g_pipe.buf[slot]);
        double *dx = dv + HostPipe::CH;
        double *dout = dx + HostPipe::CH;
        cudaStream_t s = g_pipe.st[slot];
        if ((rc = cuda_err(cudaMemcpyAsync(dv, v_h + off, m * sizeof(double), cudaMemcpyHostToDevice, s), "H2D")))
            return rc;
        if ((rc = cuda_err(cudaMemcpyAsync(dx, x_h + off, m * sizeof(double), cudaMemcpyHostToDevice, s), "H2D")))
            return rc;
        if ((rc = launch_eval<double, FN>(dv, dx, dout, m, s))) return rc;
        if ((rc = cuda_err(cudaMemcpyAsync(out_h + off, dout, m * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H")))
            return rc;
    }
    for (int i = 0; i < HostPipe::NSLOT; ++i)
        if ((rc = cuda_err(cudaStreamSynchronize(g_pipe.st[i]), "sync"))) return rc;
    return B200_OK;
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

const char *b200_last_error(void) { return g_err; }
int64_t b200_launch_count(void) { return g_launches.load(); }

}  // extern "C"
