// fp64_peak.cu -- measured FP64 FMA throughput of this GPU (the "alu" roofline
// denominator for the FP64-bound Bessel kernels).  8 independent DFMA chains
// per thread, enough warps per SM to cover the DFMA latency; CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
            r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int tpb = 256, bps = 8, iters = 4096;
    const int grid = sms * bps;
    double *out;
    cudaMalloc(&out, sizeof(double) * grid * tpb);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_kernel<<<grid, tpb>>>(out, 64, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_kernel<<<grid, tpb>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 16 * double(iters) * grid * tpb;
        double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    double per_sm_clk = best * 1e12 / 2.0 / (double(sms) * clk * 1e3);
    printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, \"dfma_per_sm_per_clk_at_attr_clock\": %.2f, "
           "\"source\": \"tools/fp64_peak.cu: 8 independent DFMA chains/thread, %d CTAs x %d threads, best of 5, CUDA events\"}\n",
           best, sms, clk, per_sm_clk, grid, tpb);
    return 0;
}
