// weno_mismatch.cu — prints the self-test samples (sl_step.cu weno_sample)
// on which weno1_fast / weno1_zt pass their guards but differ from weno1:
// the diagnostic behind lsr_cuda_selftest_weno's mismatch counts.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17
//        -I include -I paper_2410_22205_b200/csrc -o /tmp/weno_mismatch tools/weno_mismatch.cu
#include <cstdio>

#include "../paper_2410_22205_b200/csrc/sl_step.cu"

void lsr_note_launch() {}

struct Rec {
    long long i;
    double v[4], t, ref, fast, zt;
    int fast_ok, zt_ok;
};

__global__ void dump_kernel(SlParams P, unsigned long long seed, long long n, Rec* out, int cap, int* count) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        double v[4], t;
        weno_sample(seed, i, v, t);
        const AxisW w = axis_weights(P, t);
        const double ref = weno1(P, w, v[0], v[1], v[2], v[3]);
        bool ok = theta_in_range(t);
        const double fast = weno1_fast(P, w, v[0], v[1], v[2], v[3], ok);
        double sdK, SK, YK, sdK1, SK1, YK1;
        bool good = zt_node_terms(P, v[0], v[1], v[2], sdK, SK, YK);
        good = good & zt_node_terms(P, v[1], v[2], v[3], sdK1, SK1, YK1);
        const double c1 = v[2] - v[0], e2 = -3.0 * v[1] + 4.0 * v[2] - v[3];
        good = good & halvable(c1) & halvable(e2) & theta_in_range(t);
        const double zt = weno1_zt(w, make_double4(sdK, SK, YK, v[1]), make_double4(sdK1, SK1, YK1, v[2]),
                                   make_double2(c1, e2));
        const bool bad_f = ok && __double_as_longlong(fast) != __double_as_longlong(ref);
        const bool bad_z = good && __double_as_longlong(zt) != __double_as_longlong(ref);
        if (bad_f || bad_z) {
            const int q = atomicAdd(count, 1);
            if (q < cap) out[q] = Rec{i, {v[0], v[1], v[2], v[3]}, t, ref, fast, zt, ok ? 1 : 0, good ? 1 : 0};
        }
    }
}

int main(int argc, char** argv) {
    const double dx = argc > 1 ? atof(argv[1]) : 2.0 / 511;
    const long long n = argc > 2 ? atoll(argv[2]) : (1LL << 22);
    const unsigned long long seed = argc > 3 ? strtoull(argv[3], nullptr, 10) : 5;
    SlParams P{};
    P.dx = dx;
    P.dx2 = dx * dx;
    P.rdx = 1.0 / dx;
    P.rdx2 = 1.0 / P.dx2;
    P.r3 = 1.0 / 3.0;
    P.fast_div = 1;
    P.fast_weno = 1;
    const int cap = 40;
    Rec* d;
    int* c;
    cudaMalloc(&d, sizeof(Rec) * cap);
    cudaMalloc(&c, sizeof(int));
    cudaMemset(c, 0, sizeof(int));
    dump_kernel<<<148 * 8, 256>>>(P, seed, n, d, cap, c);
    Rec h[cap];
    int hc = 0;
    cudaMemcpy(&hc, c, sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(h, d, sizeof(Rec) * cap, cudaMemcpyDeviceToHost);
    std::printf("mismatches: %d\n", hc);
    for (int q = 0; q < (hc < cap ? hc : cap); ++q)
        std::printf("i=%lld cls=%lld v=[%a %a %a %a] t=%a ref=%a fast=%a(ok %d) zt=%a(ok %d)\n", h[q].i, h[q].i & 3,
                    h[q].v[0], h[q].v[1], h[q].v[2], h[q].v[3], h[q].t, h[q].ref, h[q].fast, h[q].fast_ok, h[q].zt,
                    h[q].zt_ok);
    return 0;
}
