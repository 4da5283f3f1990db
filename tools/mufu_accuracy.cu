// mufu_accuracy.cu -- accuracy of the MUFU-seeded reciprocal / reciprocal square
// root of fastmath.cuh with and without the final Newton step (diagnostic).
// Reports max relative error (in units of 2^-53) against the correctly rounded
// 1/a and 1/sqrt(a) (IEEE division / sqrt on the device).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstring>

__device__ double rcp_cubic(double a) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    double e = fma(-a, r, 1.0);
    return fma(r, fma(e, e, e), r);
}
__device__ double rcp_full(double a) {
    double r = rcp_cubic(a);
    double e = fma(-a, r, 1.0);
    return fma(r, e, r);
}
__device__ double rsq_cubic(double a) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    double e = fma(-a * y, y, 1.0);
    return fma(y, e * fma(e, 0.375, 0.5), y);
}
__device__ double rsq_full(double a) {
    double y = rsq_cubic(a);
    double e = fma(-a * y, y, 1.0);
    return fma(0.5 * y, e, y);
}
__device__ double seed_rcp(double a) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); return r; }
__device__ double seed_rsq(double a) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); return r; }

__device__ unsigned long long g_max[6];
__device__ __forceinline__ void upd(int i, double got, double ref) {
    double e = fabs(got - ref) / fabs(ref) * 9007199254740992.0;   // units of 2^-53
    atomicMax(&g_max[i], __double_as_longlong(e));
}
__global__ void k(uint64_t seed, int n) {
    uint64_t s = seed ^ (blockIdx.x * 0x9E3779B97F4A7C15ull + threadIdx.x * 0xBF58476D1CE4E5B9ull);
    for (int i = 0; i < n; ++i) {
        s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
        uint64_t m = s * 0x2545F4914F6CDD1Dull;
        // a = mantissa random, exponent in [-600, 600]
        int ex = int((m >> 52) % 1200) - 600;
        double a = __hiloint2double(int(((ex + 1023) << 20) | ((m >> 20) & 0xFFFFF)), int(m));
        double r1 = 1.0 / a, r2 = 1.0 / sqrt(a);
        upd(0, rcp_cubic(a), r1);
        upd(1, rcp_full(a), r1);
        upd(2, rsq_cubic(a), r2);
        upd(3, rsq_full(a), r2);
        upd(4, seed_rcp(a), r1);
        upd(5, seed_rsq(a), r2);
    }
}
int main() {
    k<<<1184, 256>>>(12345, 4096);
    unsigned long long h[6];
    cudaMemcpyFromSymbol(h, g_max, sizeof(h));
    const char *nm[6] = {"rcp_cubic", "rcp_full", "rsqrt_cubic", "rsqrt_full", "rcp_seed", "rsqrt_seed"};
    printf("{");
    for (int i = 0; i < 6; ++i) {
        double v;
        memcpy(&v, &h[i], 8);
        printf("\"%s_max_ulp53\": %.4g%s", nm[i], v, i < 5 ? ", " : "");
    }
    printf(", \"samples\": %lld}\n", 1184LL * 256 * 4096);
    return 0;
}
