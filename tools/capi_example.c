/* capi_example.c -- the C ABI of include/bessel_b200.h used from plain C (no Python, no torch).
 *
 * Build (nvcc only links; the file is C):
 *   nvcc -o capi_example tools/capi_example.c -Iinclude -Lpaper_2409_08729_b200/lib -lbessel_b200 \
 *        -Xlinker -rpath=paper_2409_08729_b200/lib
 * Checks the half-integer closed forms log I_{1/2}(x) = log(sqrt(2/(pi x)) sinh x) and
 * log K_{1/2}(x) = log(sqrt(pi/(2x))) - x through the device and the host-buffer entry points.
 * Exit status 0 on success.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "bessel_b200.h"

#define CK(e)                                                                         \
    do {                                                                              \
        cudaError_t _e = (e);                                                         \
        if (_e != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(_e)); \
            return 2;                                                                 \
        }                                                                             \
    } while (0)

int main(void) {
    const int64_t n = 100000;
    double *v = malloc(n * sizeof(double)), *x = malloc(n * sizeof(double));
    double *oi = malloc(n * sizeof(double)), *ok = malloc(n * sizeof(double));
    double *hi = malloc(n * sizeof(double)), *hk = malloc(n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        v[i] = 0.5;
        x[i] = 0.01 + 0.001 * (double)i;          /* 0.01 .. 100 */
    }
    double *dv, *dx, *di, *dk;
    CK(cudaMalloc((void **)&dv, n * sizeof(double)));
    CK(cudaMalloc((void **)&dx, n * sizeof(double)));
    CK(cudaMalloc((void **)&di, n * sizeof(double)));
    CK(cudaMalloc((void **)&dk, n * sizeof(double)));
    CK(cudaMemcpy(dv, v, n * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice));
    if (b200_log_ivkv_f64(dv, dx, di, dk, n, NULL) != B200_OK) {
        fprintf(stderr, "b200_log_ivkv_f64: %s\n", b200_last_error());
        return 1;
    }
    CK(cudaMemcpy(oi, di, n * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ok, dk, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (b200_log_ivkv_f64_host(v, x, hi, hk, n) != B200_OK) {
        fprintf(stderr, "b200_log_ivkv_f64_host: %s\n", b200_last_error());
        return 1;
    }
    /* argument errors are reported, not launched */
    if (b200_log_iv_f64(NULL, dx, di, n, NULL) != B200_ERR_INVALID_ARGUMENT) return 3;
    double emax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double xi = x[i];
        /* log(sqrt(2/(pi x)) sinh x) = x + log1p(-exp(-2x)) - log 2 + 0.5 log(2/(pi x)) */
        const double ri = xi + log1p(-exp(-2.0 * xi)) - log(2.0) + 0.5 * log(2.0 / (M_PI * xi));
        const double rk = 0.5 * log(M_PI / (2.0 * xi)) - xi;
        const double ei = fabs(oi[i] - ri) / fmax(fabs(ri), 1.0), ek = fabs(ok[i] - rk) / fmax(fabs(rk), 1.0);
        emax = fmax(emax, fmax(ei, ek));
        if (hi[i] != oi[i] || hk[i] != ok[i]) {
            fprintf(stderr, "host and device paths differ at %lld\n", (long long)i);
            return 1;
        }
    }
    printf("capi_example: %lld pairs, max rel err vs closed forms %.3e, launches %lld\n", (long long)n, emax,
           (long long)b200_launch_count());
    cudaFree(dv); cudaFree(dx); cudaFree(di); cudaFree(dk);
    free(v); free(x); free(oi); free(ok); free(hi); free(hk);
    return emax <= 1e-13 ? 0 : 1;
}
