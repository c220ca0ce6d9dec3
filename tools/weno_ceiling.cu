// weno_ceiling.cu — compute ceiling of the exact fast WENO arithmetic on one
// B200: fp64 dependent latencies (DFMA, DADD, MUFU.RCP64H) and the
// throughput of weno1_fast with ILP 1/2/4 independent lines per thread at
// several occupancies. No memory traffic: the stencil values are registers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false
//        -I include -I paper_2410_22205_b200/csrc -o tools/weno_ceiling tools/weno_ceiling.cu
#include <cstdio>

#include <cuda_runtime.h>

#include "sl_device.cuh"

using namespace lsr_dev;

__global__ void lat_dfma(double* out, long long* cyc, double a, double b) {
    double x = threadIdx.x * 1e-9;
    const long long t0 = clock64();
    for (int i = 0; i < 1024; ++i) x = __fma_rn(x, a, b);
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}

__global__ void lat_rcp(double* out, long long* cyc, double b) {
    double x = 1.5 + threadIdx.x * 1e-9;
    const long long t0 = clock64();
    for (int i = 0; i < 1024; ++i) x = rcp_approx_hi(x) + 1.0;
    const long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}

template <int ILP>
__global__ void __launch_bounds__(128) weno_tp(SlParams P, double* out, int iters, int* bad) {
    AxisW w;
    w.t = 0.37 + threadIdx.x * 1e-6;
    w.tt = w.t * w.t;
    w.cl = (2.0 - w.t) / 3.0;
    w.cr = (1.0 + w.t) / 3.0;
    w.omt = 1.0 - w.t;
    double v[ILP][4];
#pragma unroll
    for (int l = 0; l < ILP; ++l)
#pragma unroll
        for (int e = 0; e < 4; ++e) v[l][e] = 0.01 * (e + 1) * (l + 1) + threadIdx.x * 1e-7;
    bool ok = true;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int l = 0; l < ILP; ++l) {
            const double r = weno1_fast(P, w, v[l][0], v[l][1], v[l][2], v[l][3], ok);
            v[l][0] = v[l][1];
            v[l][1] = v[l][2];
            v[l][2] = v[l][3];
            v[l][3] = r;
        }
    }
    double s = 0;
#pragma unroll
    for (int l = 0; l < ILP; ++l) s += v[l][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (!ok) atomicAdd(bad, 1);
}

template <int ILP>
void run_tp(const SlParams& P, double* out, int* bad, int blocks_per_sm) {
    const int iters = 400;
    const int blocks = 148 * blocks_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    weno_tp<ILP><<<blocks, 128>>>(P, out, iters, bad);
    cudaEventRecord(e0);
    weno_tp<ILP><<<blocks, 128>>>(P, out, iters, bad);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double wenos = double(blocks) * 128 * iters * ILP;
    // 84 wenos per WENO-3D node-update
    printf("{\"ilp\": %d, \"blocks_per_sm\": %d, \"wenos_per_s\": %.4e, \"node_updates_equiv_per_s\": %.4e}\n", ILP,
           blocks_per_sm, wenos / (ms * 1e-3), wenos / 84.0 / (ms * 1e-3));
}

int main() {
    double* out;
    long long* cyc;
    int* bad;
    cudaMalloc(&out, sizeof(double) * 148 * 16 * 128);
    cudaMalloc(&cyc, sizeof(long long));
    cudaMalloc(&bad, sizeof(int));
    cudaMemset(bad, 0, sizeof(int));
    long long h = 0;
    lat_dfma<<<1, 32>>>(out, cyc, 0.999, 1e-3);
    cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("{\"dfma_latency_cycles\": %.2f}\n", h / 1024.0);
    lat_rcp<<<1, 32>>>(out, cyc, 1.5);
    cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("{\"rcp64h_plus_dadd_latency_cycles\": %.2f}\n", h / 1024.0);
    SlParams P{};
    P.dx = 2.0 / 511;
    P.dx2 = P.dx * P.dx;
    P.rdx = 1.0 / P.dx;
    P.rdx2 = 1.0 / P.dx2;
    P.r3 = 1.0 / 3.0;
    P.fast_div = 1;
    P.fast_weno = 1;
    for (int b : {2, 4, 6, 8}) {
        run_tp<1>(P, out, bad, b);
        run_tp<2>(P, out, bad, b);
        run_tp<4>(P, out, bad, b);
    }
    int hb = 0;
    cudaMemcpy(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost);
    printf("{\"guard_failures\": %d}\n", hb);
    return 0;
}
