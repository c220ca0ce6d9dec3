// fp64_peak.cu — measures the B200's sustained DFMA and DDIV throughput
// (the roofline denominator for the fp64-bound SL step; MEASURED_PEAKS.json
// carries no fp64 figure). Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>

#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ddiv_loop(double* out, int iters, double b) {
    double x0 = 1.0 + threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = b / x0 + 1.0; x1 = b / x1 + 1.0; x2 = b / x2 + 1.0; x3 = b / x3 + 1.0;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, threads = 256;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 3; ++rep) {
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = double(blocks) * threads * iters * 16 * 8;
        printf("{\"what\": \"dfma\", \"dfma_per_s\": %.4e, \"tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d}\n",
               n / (ms * 1e-3), 2 * n / (ms * 1e-3) / 1e12, ms, sms, clk / 1000);
    }
    const int diters = 2000;
    ddiv_loop<<<blocks, threads>>>(out, diters, 3.0);
    cudaEventRecord(e0);
    ddiv_loop<<<blocks, threads>>>(out, diters, 3.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = double(blocks) * threads * diters * 8 * 4;
    printf("{\"what\": \"ddiv\", \"ddiv_per_s\": %.4e, \"ms\": %.3f}\n", n / (ms * 1e-3), ms);
    cudaFree(out);
    return 0;
}
