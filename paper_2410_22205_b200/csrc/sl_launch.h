// Internal launcher interface between the C ABI (lsr_capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "sl_device.cuh"

#ifndef LSR_SL_THREADS
#define LSR_SL_THREADS 128
#endif
#ifndef LSR_SL_MIN_BLOCKS
#define LSR_SL_MIN_BLOCKS 7
#endif
constexpr int kSlThreads = LSR_SL_THREADS;
constexpr int kSlMinBlocks = LSR_SL_MIN_BLOCKS;  // resident CTAs per SM the register budget must allow

// bumps the process-wide launch counter (lsr_cuda_kernel_launches)
void lsr_note_launch();

cudaError_t launch_sl_step(const lsr_dev::SlParams& P, int kind, const double* phi, const double* dist,
                           const int64_t* active, long long n_active, double* out, unsigned long long* bad,
                           cudaStream_t stream);

cudaError_t launch_check_sorted(const int64_t* ids, long long n, unsigned long long* bad, cudaStream_t stream);

cudaError_t launch_resync(const double* phi, double* out, const int64_t* ids, long long n, cudaStream_t stream);

cudaError_t launch_div_selftest(double c, double rc, unsigned long long seed, long long n,
                                unsigned long long* mismatches);

// field[desc[r].dst + l] = packed[desc[r].src + l] for the runs r in [r0, r1)
// (desc = (dst, src) pairs; a run ends where the next begins, the last at vend)
cudaError_t launch_scatter_runs(const double* packed, const long long* desc, long long r0, long long r1,
                                long long vend, double* field, cudaStream_t stream);

// res[t] = field[ids[t]] for t < n
cudaError_t launch_gather_ids(const double* field, const int64_t* ids, long long n, double* res,
                              cudaStream_t stream);
