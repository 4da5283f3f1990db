// initcheck_stores.cu -- does compute-sanitizer initcheck track each store flavour? (diagnostic)
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ics tools/initcheck_stores.cu
// compute-sanitizer --tool initcheck /tmp/ics   -> which D2H copies are reported
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void st_plain(double *o, int n) { int i = threadIdx.x; if (i < n) o[i] = i; }
__global__ void st_cs(double *o, int n) { int i = threadIdx.x; if (i < n) __stcs(o + i, double(i)); }
__global__ void st_bulk(double *o, int n) {
    __shared__ alignas(128) double s[256];
    int i = threadIdx.x;
    if (i < n) s[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (i == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o),
                     "r"(uint32_t(__cvta_generic_to_shared(s))), "r"(uint32_t(n * 8)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    const int n = 64;
    double *d, h[n];
    const char *names[3] = {"plain st.global", "st.global.cs (__stcs)", "cp.async.bulk store"};
    for (int k = 0; k < 3; ++k) {
        cudaMalloc(&d, n * sizeof(double));
        if (k == 0) st_plain<<<1, 256>>>(d, n);
        if (k == 1) st_cs<<<1, 256>>>(d, n);
        if (k == 2) st_bulk<<<1, 256>>>(d, n);
        cudaDeviceSynchronize();
        printf("== %s\n", names[k]);
        fflush(stdout);
        cudaMemcpy(h, d, n * sizeof(double), cudaMemcpyDeviceToHost);
        printf("   h[%d] = %g\n", n - 1, h[n - 1]);
        fflush(stdout);
        cudaFree(d);
    }
    return 0;
}
