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
#define B200_MINB 3
#endif
#ifndef B200_ITEMS
#define B200_ITEMS 4
#endif
constexpr int TPB = B200_TPB;
constexpr int ITEMS = B200_ITEMS;
constexpr int TILE = TPB * ITEMS;       // 1024 pairs per tile
static_assert(TILE <= 4096, "s_idx packs a 12-bit tile index with the bin");
constexpr int NBIN = 8;                 // 12-bit counters, 5 per 64-bit word, 2 words
constexpr int BIN_SPECIAL = 7;

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
// x <= 8 / x > 8; K: Temme series x <= 2 / Steed CF2 x > 2); 7 = special.
template <int FN>
__device__ __forceinline__ int bin_of(double v, double x) {
    if (!(x > 0.0) || !isfinite(x) || !isfinite(v)) return BIN_SPECIAL;   // x<=0, NaN, inf
    if (FN == FN_I) {
        if (v < 0.0) return BIN_SPECIAL;
    } else {
        v = fabs(v);
    }
    return select_eval(v, x, (FN == FN_I) ? 8.0 : 2.0);
}

// Values for the special bin: x == 0, non-finite or out-of-domain inputs.
template <typename T, int FN>
__device__ __forceinline__ T special_value(T v, T x) {
    const T nan = T(CUDART_NAN);
    if (isnan(v) || isnan(x) || x < T(0)) return nan;
    if (FN == FN_I) {
        if (v < T(0)) return nan;
        if (x == T(0)) return v == T(0) ? T(0) : T(-CUDART_INF);
        if (isinf(v)) return T(-CUDART_INF);           // I_inf(x) = 0
        return T(CUDART_INF);                          // x = +inf
    } else {
        if (x == T(0)) return T(CUDART_INF);           // pole
        if (isinf(v)) return T(CUDART_INF);
        return T(-CUDART_INF);                         // x = +inf
    }
}

template <typename T, int FN>
__device__ __forceinline__ T eval_bin(int bin, T v, T x) {
    if (bin == BIN_SPECIAL) return special_value<T, FN>(v, x);
#ifdef B200_EVAL_NOP
    return v + x;   // experiment only: measures the tile machinery alone
#endif
    if (FN == FN_I) return log_iv_eval<T>(bin, v, x);
    const T av = fabs(v);
    if (FN == FN_K) return log_kv_eval<T, false>(bin, av, x);
    return log_kv_eval<T, true>(bin, av, x);
}

// Two 64-bit words of five 12-bit counters each (a tile has <= 1024 < 4096 of a bin).
struct Cnt {
    uint64_t w[2];
    __device__ __forceinline__ void zero() { w[0] = w[1] = 0; }
    __device__ __forceinline__ void inc(int b) {
        const uint64_t one0 = b < 5 ? (1ull << (12 * b)) : 0ull;
        const uint64_t one1 = b < 5 ? 0ull : (1ull << (12 * (b - 5)));
        w[0] += one0;
        w[1] += one1;
    }
    __device__ __forceinline__ int get(int b) const {
        const uint64_t word = b < 5 ? w[0] : w[1];
        return int((word >> (12 * (b < 5 ? b : b - 5))) & 0xFFFull);
    }
    __device__ __forceinline__ void add(const Cnt &o) { w[0] += o.w[0]; w[1] += o.w[1]; }
    __device__ __forceinline__ void sub(const Cnt &o) { w[0] -= o.w[0]; w[1] -= o.w[1]; }
    __device__ __forceinline__ Cnt shfl_up(int o) const {
        Cnt r;
        r.w[0] = __shfl_up_sync(0xffffffffu, w[0], o);
        r.w[1] = __shfl_up_sync(0xffffffffu, w[1], o);
        return r;
    }
};

template <typename T, int FN>
__global__ void __launch_bounds__(TPB, B200_MINB) bessel_eval_kernel(const T *__restrict__ vin, const T *__restrict__ xin,
                                                          T *__restrict__ out, int64_t n) {
    __shared__ T s_v[TILE];
    __shared__ T s_x[TILE];
    __shared__ T s_res[TILE];
    __shared__ uint16_t s_idx[TILE];
    __shared__ Cnt s_warp[TPB / 32];
    __shared__ int s_base[NBIN + 1];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (n + TILE - 1) / TILE;

    // Software pipeline: the (v, x) of the next tile are loaded into registers
    // while the current tile is binned and evaluated.
    T nv[ITEMS], nx[ITEMS];
    auto prefetch = [&](int64_t t) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int64_t g = t * TILE + tid + i * TPB;
            if (t < ntiles && g < n) {
                nv[i] = __ldcs(vin + g);
                nx[i] = __ldcs(xin + g);
            }
        }
    };
    prefetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * TILE;
        T lv[ITEMS], lx[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) { lv[i] = nv[i]; lx[i] = nx[i]; }
        prefetch(tile + gridDim.x);
        int lb[ITEMS];
        Cnt cnt;
        cnt.zero();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int64_t g = base + tid + i * TPB;
            lb[i] = -1;
            if (g < n) {
                lb[i] = bin_of<FN>(double(lv[i]), double(lx[i]));
                cnt.inc(lb[i]);
            }
        }
        // block-wide exclusive scan of the packed per-thread bin counts (warp shuffles)
        Cnt incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const Cnt y = incl.shfl_up(o);
            if (lane >= o) incl.add(y);
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            Cnt wv;
            if (lane < TPB / 32) wv = s_warp[lane]; else wv.zero();
            Cnt wi = wv;
#pragma unroll
            for (int o = 1; o < TPB / 32; o <<= 1) {
                const Cnt y = wi.shfl_up(o);
                if (lane >= o) wi.add(y);
            }
            if (lane < TPB / 32) { Cnt ex = wi; ex.sub(wv); s_warp[lane] = ex; }   // exclusive warp offsets
            if (lane == TPB / 32 - 1) {
                int acc = 0;
                for (int b = 0; b < NBIN; ++b) { s_base[b] = acc; acc += wi.get(b); }
                s_base[NBIN] = acc;
            }
        }
        __syncthreads();
        Cnt excl = s_warp[warp];
        excl.add(incl);
        excl.sub(cnt);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (lb[i] >= 0) {
                const int b = lb[i];
                const int pos = s_base[b] + excl.get(b);
                excl.inc(b);
                s_v[pos] = lv[i];
                s_x[pos] = lx[i];
                s_idx[pos] = uint16_t((tid + i * TPB) | (b << 12));   // tile index | bin
            }
        }
        __syncthreads();
        const int total = s_base[NBIN];
#pragma unroll 1
        for (int i = 0; i < ITEMS; ++i) {
            const int p = tid + i * TPB;
            if (p < total) {
                const int w = s_idx[p];
                s_res[w & 0xFFF] = eval_bin<T, FN>(w >> 12, s_v[p], s_x[p]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int64_t g = base + tid + i * TPB;
            if (g < n) __stcs(out + g, s_res[tid + i * TPB]);
        }
        __syncthreads();
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
