// vmf_kernels.cu -- von Mises-Fisher fit (§6.3).
//
// Data-parallel part: the column sum of the n x d feature matrix (the mean
// x̄ of Eq. (mean direction estimate), line 672) -- an HBM-bound streaming
// reduction, two deterministic stages (per-row-slab partials, then a fixed
// order sum over slabs).  Scalar part: Rbar, mu, kappa0/1/2 (Eq. (kappa
// estimates), lines 676-680) and the MLE of kappa (lines 684-691) run in one
// CTA on the device with the same log I_v device code as the batch kernels.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <mutex>

#include "../../include/bessel_b200.h"
#include "bessel_math.cuh"

namespace b200 {

extern std::atomic<int64_t> g_launches;   // defined in bessel_kernels.cu
int set_err(int code, const char *msg);    // bessel_kernels.cu: per-thread last-error string
int cuda_err(cudaError_t e, const char *where);

// Programmatic dependent launch: the column-sum partial -> reduce -> fit chain is
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, so a dependent
// grid is scheduled while its producer drains and waits at griddepcontrol.wait for
// the producer's completion (memory visible); launched without the attribute, both
// instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

constexpr int CS_TPB = 256;
#ifndef B200_CS_ROWS
#define B200_CS_ROWS 8
#endif
constexpr int CS_ROWS = B200_CS_ROWS;       // rows in flight per thread in the column-sum stream
#ifndef B200_CS_CTAS
#define B200_CS_CTAS 8                      // column-sum CTAs per SM (row slabs x column slabs)
#endif
#ifndef B200_CS_CTAS_SMALL
#define B200_CS_CTAS_SMALL 3                // the same when d spans at most two column slabs (2/3/4 measured)
#endif

template <typename T> struct VecOf;
template <> struct VecOf<float> { using V = float4; static constexpr int N = 4; };
template <> struct VecOf<double> { using V = double2; static constexpr int N = 2; };

__device__ __forceinline__ void vadd(double *acc, const float4 &a) {
    acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
}
__device__ __forceinline__ void vadd(double *acc, const double2 &a) {
    acc[0] += a.x; acc[1] += a.y;
}

// Stage 1: CTA (bx, by) sums rows [by*rows_per, (by+1)*rows_per) of the
// column slab [bx*CW, bx*CW + CW).  Each thread owns VN consecutive columns
// and streams its rows with VN-wide loads (a warp reads 32*VN*sizeof(T)
// contiguous bytes per row); CS_ROWS rows in flight per thread.
template <typename T, bool VEC>
__global__ void __launch_bounds__(CS_TPB) colsum_partial_kernel(const T *__restrict__ X, int64_t n, int64_t d,
                                                                int64_t ld, int64_t rows_per,
                                                                double *__restrict__ part) {
    constexpr int VN = VEC ? VecOf<T>::N : 1;
    constexpr int CW = CS_TPB * VN;
    pdl_launch_dependents();   // the reduce kernel may be scheduled now; it waits for this grid
    const int64_t c0 = int64_t(blockIdx.x) * CW + int64_t(threadIdx.x) * VN;
    const int64_t r0 = int64_t(blockIdx.y) * rows_per;
    int64_t r1 = r0 + rows_per;
    if (r1 > n) r1 = n;
    double acc[VN];
#pragma unroll
    for (int j = 0; j < VN; ++j) acc[j] = 0.0;
    if (c0 < d) {
        if (VEC && c0 + VN <= d) {
            using V = typename VecOf<T>::V;
            const T *p = X + r0 * ld + c0;
            int64_t r = r0;
            // CS_ROWS rows in flight per thread (16-byte loads, streaming cache hint)
            for (; r + CS_ROWS <= r1; r += CS_ROWS) {
                V a[CS_ROWS];
#pragma unroll
                for (int q = 0; q < CS_ROWS; ++q) a[q] = __ldcs(reinterpret_cast<const V *>(p + q * ld));
#pragma unroll
                for (int q = 0; q < CS_ROWS; ++q) vadd(acc, a[q]);
                p += CS_ROWS * ld;
            }
            for (; r < r1; ++r, p += ld) vadd(acc, __ldcs(reinterpret_cast<const V *>(p)));
        } else {
            for (int j = 0; j < VN; ++j) {
                if (c0 + j >= d) break;
                const T *p = X + r0 * ld + c0 + j;
                double a = 0.0;
                for (int64_t r = r0; r < r1; ++r, p += ld) a += double(*p);
                acc[j] = a;
            }
        }
        double *o = part + int64_t(blockIdx.y) * d + c0;
#pragma unroll
        for (int j = 0; j < VN; ++j)
            if (c0 + j < d) o[j] = acc[j];
    }
}

// Stage 2: colsum[j] (+)= sum_s part[s*d + j] in a fixed order: warp w of an
// NW-warp CTA sums slabs w, w + NW, w + 2 NW, ... of 32 consecutive columns (one
// 256-byte row segment per load), eight slabs per pass loaded together (predicated,
// independent: one memory round trip per pass instead of a dependent chain) and added
// in a fixed tree; the NW warp partials are then added in warp order -- deterministic
// for a given slab count.  d/32 CTAs of 32 warps when there are more than 64 slabs
// (d = 2048: 222 slabs, 13 -> 3 us against 8 warps with dependent chains), else 8.
// Block 0 also writes the row-count slot colsum[d] (+)= n when with_count (no
// separate launch).
template <int CR_WARPS>
__global__ void __launch_bounds__(32 * CR_WARPS) colsum_reduce_kernel(const double *__restrict__ part, int64_t nslab,
                                                                     int64_t d, double *__restrict__ colsum,
                                                                     int accumulate, int with_count, double n_rows) {
    __shared__ double sh[CR_WARPS][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    pdl_wait();                // the partials of the preceding grid are complete and visible
    pdl_launch_dependents();
    if (with_count && blockIdx.x == 0 && threadIdx.x == 0) colsum[d] = accumulate ? colsum[d] + n_rows : n_rows;
    for (int64_t c0 = int64_t(blockIdx.x) * 32; c0 < d; c0 += int64_t(gridDim.x) * 32) {
        const int64_t j = c0 + lane;
        double s = 0.0;
        if (j < d) {
            const double *p = part + j;
            for (int64_t k0 = w; k0 < nslab; k0 += 8 * CR_WARPS) {
                double a[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int64_t k = k0 + int64_t(i) * CR_WARPS;
                    a[i] = k < nslab ? __ldcg(p + k * d) : 0.0;
                }
                s += ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
            }
        }
        sh[w][lane] = s;
        __syncthreads();
        if (w == 0 && j < d) {
            double t = sh[0][lane];
#pragma unroll
            for (int q = 1; q < CR_WARPS; ++q) t += sh[q][lane];
            colsum[j] = accumulate ? colsum[j] + t : t;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- scalar part
__device__ double log_iv_scalar(double v, double x) { return log_iv_scalar_eval<double>(v, x); }

// A_p(kappa) = I_{p/2}(kappa) / I_{p/2-1}(kappa)  (line 677).  Called by the
// 64 threads of warps 0 and 1 with the same arguments: lane 0 of warp w
// evaluates log I_{p/2 - w}(kappa), the two logs meet in shared memory behind
// a named barrier over the two warps, so the two evaluations run concurrently.
// lil = log I_{p/2-1}(kappa) (the log-likelihood needs it).
__device__ double a_p(double p, double kappa, double *s_l, double &lil) {
    const int w = threadIdx.x >> 5;
    if (kappa <= 0.0) { lil = 0.0; return 0.0; }
    if ((threadIdx.x & 31) == 0) s_l[w] = log_iv_scalar(0.5 * p - double(w), kappa);
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const double l0 = s_l[0];
    lil = s_l[1];
    asm volatile("bar.sync 1, 64;" ::: "memory");   // s_l is rewritten by the next call
    return exp(l0 - lil);
}

// F(kappa) of Eq. (kappa estimates)
__device__ double newton_F(double p, double rbar, double k, double *s_l) {
    double lil;
    const double A = a_p(p, k, s_l, lil);
    return k - (A - rbar) / (1.0 - A * A - (p - 1.0) / k * A);
}

constexpr int FIT_TPB = 256;

__global__ void __launch_bounds__(FIT_TPB) vmf_fit_kernel(const double *__restrict__ colsum, int64_t n_total,
                                                          int64_t d, double *__restrict__ mu,
                                                          double *__restrict__ stats) {
    fm_tables_init();
    pdl_wait();                // the column sums of the preceding grid (reduce / all-reduce) are visible
    __shared__ double s_red[FIT_TPB / 32];
    __shared__ double s_rbar;
    __shared__ double s_l[2];
    const double inv_n = 1.0 / (n_total > 0 ? double(n_total) : colsum[d]);
    double loc = 0.0;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
        const double m = colsum[j] * inv_n;
        loc = fma(m, m, loc);
    }
    // warp-shuffle reduction of ||xbar||^2, then across warps
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = loc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) s_rbar = sqrt(w);
    }
    __syncthreads();
    const double rbar = s_rbar;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) mu[j] = colsum[j] * inv_n / rbar;
    // the scalar part: warps 0 and 1 run it redundantly (identical control
    // flow), lane 0 of each evaluates one of the two logs per A_p; thread 0 writes
    if (threadIdx.x >= 64) return;
    const bool w0 = threadIdx.x == 0;

    const double p = double(d);
    if (w0) stats[0] = rbar;
    if (!(rbar > 0.0 && rbar < 1.0)) {
        if (w0)
            for (int i = 1; i < 8; ++i) stats[i] = CUDART_NAN;
        return;
    }
    // Eq. (kappa estimates)
    const double k0 = rbar * (p - rbar * rbar) / (1.0 - rbar * rbar);
    const double k1 = newton_F(p, rbar, k0, s_l);
    const double k2 = newton_F(p, rbar, k1, s_l);
    if (w0) {
        stats[1] = k0;
        stats[2] = k1;
        stats[3] = k2;
    }
    // MLE: d logLik/dkappa = Rbar - A_p(kappa) (A_p strictly increasing), so
    // the maximiser is the root; safeguarded Newton from kappa2 with a
    // bracket [lo, hi] (lo: A < Rbar, hi: A > Rbar), bisection fallback.
    // Stop rule: A_p is exp of a difference of two log I values, each carrying an
    // absolute error ~ eps |log I| (R15), so near the root g = A_p - Rbar
    // is noise of that size and Newton steps stop contracting instead of reaching
    // 4e-16 k.  Stop when |g| is inside that error bound, when a step is below
    // 4e-16 k or no longer at most half the previous one (quadratic convergence
    // over), and return the evaluated point with the smallest |g| together with its
    // A_p and log I (no re-evaluation).
    double lo = 0.0, hi = CUDART_INF;
    double k = (k2 > 0.0 && isfinite(k2)) ? k2 : k0;
    int it = 0;
    double A = 0.0, lil = 0.0;
    double kb = k, Ab = 0.0, lilb = 0.0, gb = CUDART_INF, prev = CUDART_INF;
    for (; it < 100; ++it) {
        A = a_p(p, k, s_l, lil);
        const double g = A - rbar;
        if (fabs(g) < gb) { gb = fabs(g); kb = k; Ab = A; lilb = lil; }
        // |g| within the error bound of A_p itself (64 eps max(|log I|, 1) relative, R15):
        // k is the root to the precision the Bessel values allow
        if (fabs(g) <= 64.0 * 1.1102230246251565e-16 * fmax(fabs(lil), 1.0) * A) { ++it; break; }
        if (g < 0.0) lo = k; else hi = k;
        const double dA = 1.0 - A * A - (p - 1.0) / k * A;
        double kn = k - g / dA;
        const bool newton = kn > lo && kn < hi && isfinite(kn);
        if (!newton) kn = isfinite(hi) ? 0.5 * (lo + hi) : 2.0 * k;
        const double step = fabs(kn - k);
        ++it;
        if (step <= 4e-16 * k) break;
        if (newton && step > 0.5 * prev) break;
        if (isfinite(hi) && (hi - lo) <= 4e-16 * hi) break;
        prev = newton ? step : CUDART_INF;
        k = kn;
    }
    k = kb;
    A = Ab;
    lil = lilb;
    if (w0) {
        stats[4] = k;
        stats[5] = (0.5 * p - 1.0) * log(k) - 0.5 * p * log(2.0 * CUDART_PI) - lil + k * rbar;
        stats[6] = A - rbar;
        stats[7] = double(it);
    }
}

// ---------------------------------------------------------------- scratch
// The per-slab partials live in a scratch buffer owned by the library, one per
// (device, stream): calls on one stream are ordered by the stream, and the
// mutex is held while a call enqueues both of its kernels, so two host threads
// sharing a stream cannot interleave partial / reduce pairs.  Calls on
// different streams use different buffers (no race).  A buffer that must grow
// is freed only after its stream has drained; buffers live for the process.
struct ScratchEnt {
    int dev;
    cudaStream_t stream;
    void *ptr;
    size_t bytes;
};
constexpr int SCRATCH_MAX = 256;
static std::mutex g_scratch_mu;
static ScratchEnt g_scratch[SCRATCH_MAX];
static int g_nscratch = 0;

// Called with g_scratch_mu held.
static int scratch_get(int dev, cudaStream_t s, size_t bytes, double **out) {
    ScratchEnt *e = nullptr;
    for (int i = 0; i < g_nscratch; ++i)
        if (g_scratch[i].dev == dev && g_scratch[i].stream == s) { e = &g_scratch[i]; break; }
    if (!e) {
        if (g_nscratch == SCRATCH_MAX) {
            // evict the oldest entry: wait for its stream's work, then free it
            ScratchEnt &o = g_scratch[0];
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(o.dev);
            cudaStreamSynchronize(o.stream);
            cudaFree(o.ptr);
            cudaSetDevice(cur);
            for (int i = 1; i < g_nscratch; ++i) g_scratch[i - 1] = g_scratch[i];
            --g_nscratch;
        }
        e = &g_scratch[g_nscratch++];
        *e = ScratchEnt{dev, s, nullptr, 0};
    }
    if (e->bytes < bytes) {
        if (e->ptr) {
            cudaError_t err = cudaStreamSynchronize(s);          // earlier calls may still read it
            if (err != cudaSuccess) return cuda_err(err, "vmf scratch: cudaStreamSynchronize");
            cudaFree(e->ptr);
            e->ptr = nullptr;
            e->bytes = 0;
        }
        cudaError_t err = cudaMalloc(&e->ptr, bytes);
        if (err != cudaSuccess) return cuda_err(err, "vmf scratch: cudaMalloc");
        e->bytes = bytes;
    }
    *out = static_cast<double *>(e->ptr);
    return B200_OK;
}

static int sms_count(int dev) {
    constexpr int MAXDEV = 64;
    static std::atomic<int> sms[MAXDEV];
    if (dev < 0 || dev >= MAXDEV) return 148;
    int v = sms[dev].load(std::memory_order_relaxed);
    if (!v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        sms[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// colsum[d] (+)= n as a double when with_count: the row count travels in the same
// buffer, so a sharded fit needs exactly one all-reduce of d + 1 doubles.
__global__ void count_slot_kernel(double *slot, double n, int accumulate) {
    *slot = accumulate ? *slot + n : n;
}

template <typename T>
static int colsum_impl(const T *X, int64_t n, int64_t d, int64_t ld, double *colsum, int accumulate,
                       int with_count, cudaStream_t s) {
    if (n < 0 || d < 0 || ld < d) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_colsum: n < 0, d < 0 or ld < d");
    if (d == 0 && !with_count) return B200_OK;
    if (!X && n > 0) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_colsum: null X");
    if (!colsum) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_colsum: null colsum");
    if (with_count && (d == 0 || n == 0)) {            // otherwise the reduce kernel writes the slot
        count_slot_kernel<<<1, 1, 0, s>>>(colsum + d, double(n), accumulate);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_err(e, "count_slot_kernel launch");
    }
    if (d == 0) return B200_OK;
    if (n == 0) {
        if (!accumulate) return cuda_err(cudaMemsetAsync(colsum, 0, size_t(d) * sizeof(double), s), "cudaMemsetAsync");
        return B200_OK;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return set_err(B200_ERR_NO_DEVICE, "no current CUDA device");
    constexpr int VN = VecOf<T>::N;
    const bool vec = ((reinterpret_cast<uintptr_t>(X) % 16) == 0) && ((ld * sizeof(T)) % 16 == 0);
    const int CW = CS_TPB * (vec ? VN : 1);
    const int64_t ncol = (d + CW - 1) / CW;
    // ~8 CTAs per SM in total; each CTA streams a slab of rows
    // few column slabs (d <= 2 CW): fewer row slabs -- the partials (nslab x d doubles) and
    // their reduce shrink, while 8 rows in flight per thread keep the stream fed
    const int ctas = ncol <= 2 ? B200_CS_CTAS_SMALL : B200_CS_CTAS;
    int64_t nslab = (ctas * int64_t(sms_count(dev)) + ncol - 1) / ncol;
    if (nslab > n) nslab = n;
    if (nslab < 1) nslab = 1;
    const int64_t rows_per = (n + nslab - 1) / nslab;
    nslab = (n + rows_per - 1) / rows_per;
    std::lock_guard<std::mutex> lk(g_scratch_mu);   // held over both launches (see scratch_get)
    double *part = nullptr;
    int rc = scratch_get(dev, s, size_t(nslab) * size_t(d) * sizeof(double), &part);
    if (rc) return rc;
    dim3 grid((unsigned)ncol, (unsigned)nslab);
    if (vec)
        colsum_partial_kernel<T, true><<<grid, CS_TPB, 0, s>>>(X, n, d, ld, rows_per, part);
    else
        colsum_partial_kernel<T, false><<<grid, CS_TPB, 0, s>>>(X, n, d, ld, rows_per, part);
    const int64_t rb = (d + 31) / 32;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_err(e, "vmf colsum partial launch");
    if (nslab > 64)
        e = launch_pdl(colsum_reduce_kernel<32>, dim3(unsigned(rb < 4096 ? rb : 4096)), dim3(32 * 32), s,
                       (const double *)part, nslab, d, colsum, accumulate, with_count, double(n));
    else
        e = launch_pdl(colsum_reduce_kernel<8>, dim3(unsigned(rb < 4096 ? rb : 4096)), dim3(32 * 8), s,
                       (const double *)part, nslab, d, colsum, accumulate, with_count, double(n));
    g_launches.fetch_add(2, std::memory_order_relaxed);
    return cuda_err(e, "vmf colsum reduce launch");
}

static int fit_from_colsum_impl(const double *colsum, int64_t n_total, int64_t d, double *mu, double *stats,
                                cudaStream_t s) {
    if (d < 2 || !colsum || !mu || !stats) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_fit: d < 2 or null pointer");
    if (n_total < 0) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_fit: n_total < 0");
    // n_total == 0: the row count is read from colsum[d] (b200_vmf_colsum_* with with_count)
    const cudaError_t e = launch_pdl(vmf_fit_kernel, dim3(1), dim3(FIT_TPB), s, colsum, n_total, d, mu, stats);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_err(e, "vmf_fit_kernel launch");
}

}  // namespace b200

using namespace b200;

extern "C" {

int b200_vmf_colsum_f32(const float *X, int64_t n, int64_t d, int64_t ld, double *colsum, int accumulate,
                        int with_count, void *stream) {
    return colsum_impl<float>(X, n, d, ld, colsum, accumulate, with_count, static_cast<cudaStream_t>(stream));
}
int b200_vmf_colsum_f64(const double *X, int64_t n, int64_t d, int64_t ld, double *colsum, int accumulate,
                        int with_count, void *stream) {
    return colsum_impl<double>(X, n, d, ld, colsum, accumulate, with_count, static_cast<cudaStream_t>(stream));
}
int b200_vmf_fit_from_colsum(const double *colsum, int64_t n_total, int64_t d, double *mu, double *stats,
                             void *stream) {
    return fit_from_colsum_impl(colsum, n_total, d, mu, stats, static_cast<cudaStream_t>(stream));
}
int b200_vmf_fit_f32(const float *X, int64_t n, int64_t d, double *ws, double *mu, double *stats, void *stream) {
    if (n <= 0) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_fit: n <= 0");
    int rc = colsum_impl<float>(X, n, d, d, ws, 0, 0, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
    return fit_from_colsum_impl(ws, n, d, mu, stats, static_cast<cudaStream_t>(stream));
}
int b200_vmf_fit_f64(const double *X, int64_t n, int64_t d, double *ws, double *mu, double *stats, void *stream) {
    if (n <= 0) return set_err(B200_ERR_INVALID_ARGUMENT, "vmf_fit: n <= 0");
    int rc = colsum_impl<double>(X, n, d, d, ws, 0, 0, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
    return fit_from_colsum_impl(ws, n, d, mu, stats, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
