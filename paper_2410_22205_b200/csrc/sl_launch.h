// Internal launcher interface between the C ABI (lsr_capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sl_device.cuh"

// per-line kernels (Q1, 2d, 3d WENO without the z-line table): 4 CTAs of 256
// threads at 64 registers (delta = 0 WENO 1.19 -> 1.10 ms, Q1 0.58 -> 0.56 ms
// at 512^3 against 7 x 128)
#ifndef LSR_SL_THREADS
#define LSR_SL_THREADS 256
#endif
#ifndef LSR_SL_MIN_BLOCKS
#define LSR_SL_MIN_BLOCKS 4
#endif
// 3d WENO with the z-line table (sl_step_zt_kernel): 4 CTAs of 256 threads at
// 64 registers (32 warps/SM). With one x-column per loop iteration
// (weno3_interior_zt) at 512^3: 4 x 256 2.74 ms, 8 x 128 2.75, 9 x 128 2.76,
// 6 x 192 (56 registers, the previous loop form's best) 2.77, 5 x 192 2.88,
// 10 x 128 2.96.
#ifndef LSR_SL_THREADS_W3
#define LSR_SL_THREADS_W3 256
#endif
#ifndef LSR_SL_MIN_BLOCKS_W3
#define LSR_SL_MIN_BLOCKS_W3 4
#endif
constexpr int kSlThreads = LSR_SL_THREADS;
constexpr int kSlThreadsW3 = LSR_SL_THREADS_W3;
constexpr int kSlMinBlocksW3 = LSR_SL_MIN_BLOCKS_W3;
constexpr int kSlMinBlocks = LSR_SL_MIN_BLOCKS;  // resident CTAs per SM the register budget must allow

// bumps the process-wide launch counter (lsr_cuda_kernel_launches)
void lsr_note_launch();

cudaError_t launch_sl_step(const lsr_dev::SlParams& P, int kind, const double* phi, const double* dist,
                           const int64_t* active, long long n_active, double* out, unsigned long long* bad,
                           cudaStream_t stream);

// the z-line table of the 3d WENO fast path (sl_step.cu): dense zt (4
// doubles per node) and zc (2 per node), written on the covered bricks;
// reach = foot reach per brick (cells), mark = covered bricks (the SL
// kernel's coverage map), list = covered brick ids, count[0] = listed
// bricks, count[1] = range-check failures (SlParams::ztab_bad)
struct ZtBuffers {
    double* zt;
    double* zc;
    unsigned char* mark;
    unsigned* reach;
    unsigned* list;
    unsigned* count;
};
inline long long zt_num_bricks(const int dims[3]) {
    return static_cast<long long>((dims[0] + kZtBrick - 1) / kZtBrick) * ((dims[1] + kZtBrick - 1) / kZtBrick) *
           ((dims[2] + kZtBrick - 1) / kZtBrick);
}
// covered bricks of an active set: depends on the ids, d, E and the step
// config (P.energy, dt, delta, p), not on phi — the context caches it
cudaError_t launch_zt_bricks(const lsr_dev::SlParams& P, const double* dist, const int64_t* active, long long n_active,
                             const ZtBuffers& Z, cudaStream_t stream);
// table entries of the listed bricks from phi (every step)
cudaError_t launch_zt_fill(const lsr_dev::SlParams& P, const double* phi, const ZtBuffers& Z, cudaStream_t stream);
// the device loop's form: per-brick maxima of d and |grad d| (once per d),
// then the covered bricks from the band's state bytes and E (sl_step.cu)
cudaError_t launch_brick_d(const lsr_dev::SlParams& P, const double* dist, double* bd, cudaStream_t stream);
cudaError_t launch_zt_bricks_state(const lsr_dev::SlParams& P, const unsigned char* state, const double* bd,
                                   const ZtBuffers& Z, cudaStream_t stream);

cudaError_t launch_check_sorted(const int64_t* ids, long long n, unsigned long long* bad, cudaStream_t stream);
cudaError_t launch_reach_max(const lsr_dev::SlParams& P, const double* dist, const int64_t* active, long long n,
                             unsigned long long* max_bits, cudaStream_t stream);
cudaError_t launch_check_ids(const int64_t* ids, long long n, long long n_nodes, unsigned long long* bad,
                             cudaStream_t stream);

cudaError_t launch_resync(const double* phi, double* out, const int64_t* ids, long long n, long long n_nodes,
                          cudaStream_t stream);

cudaError_t launch_weno_selftest(const lsr_dev::SlParams& P, unsigned long long seed, long long n,
                                 unsigned long long* counts);

cudaError_t launch_div_selftest(double c, double rc, unsigned long long seed, long long n,
                                unsigned long long* mismatches);

// field[desc[r].dst + l] = packed[desc[r].src + l] for the runs r in [r0, r1)
// (desc = (dst, src) pairs; a run ends where the next begins, the last at vend)
cudaError_t launch_scatter_runs(const double* packed, const long long* desc, long long r0, long long r1,
                                long long vend, double* field, cudaStream_t stream);

// res[t] = field[ids[t]] for t < n
cudaError_t launch_gather_ids(const double* field, const int64_t* ids, long long n, double* res, long long n_nodes,
                              cudaStream_t stream);

// the TMA brick form of the 3d WENO step (sl_step.cu, sl_node_box): active
// ids grouped by 8^3 brick; one CTA per non-empty brick stages the brick's
// phi (+ halo) with one TMA tensor copy
struct BoxBuffers {
    unsigned* count = nullptr;   // nbricks + 1
    unsigned* off = nullptr;     // nbricks + 1 (exclusive scan of count)
    unsigned* cursor = nullptr;  // nbricks
    unsigned* list = nullptr;    // non-empty bricks, ascending
    long long* d_listed = nullptr;
    int64_t* ids = nullptr;      // active ids grouped by brick
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
};
size_t box_tmp_bytes(long long nbricks);
cudaError_t launch_box_bricks(const lsr_dev::SlParams& P, const int64_t* active, long long n, const BoxBuffers& X,
                              long long* n_listed, cudaStream_t stream);
bool launch_sl_step_box(const lsr_dev::SlParams& P, const double* phi, const double* dist, const BoxBuffers& X,
                        long long n_listed, long long n_ids, double* out, unsigned long long* bad, cudaStream_t stream);
