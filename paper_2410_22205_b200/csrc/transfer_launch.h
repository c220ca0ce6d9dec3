// Launchers of transfer.cu (bitmaps of the values one SL step reads, and the
// zero-copy pull of those values from mapped host memory).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

// words of one node bitmap (rows padded to 64-bit words)
long long lsr_bitmap_words(int nx, int ny, int nz);

// A = active ids (ids outside the grid bump *bad and are skipped), D = A and
// its axis neighbours, and for reach > 0 B = the Chebyshev ball of radius
// reach around A (T is scratch). All bitmaps hold lsr_bitmap_words words.
cudaError_t launch_build_bitmaps(int nx, int ny, int nz, const int64_t* ids, long long n, int reach,
                                 unsigned long long* A, unsigned long long* D, unsigned long long* B,
                                 unsigned long long* T, unsigned long long* bad, cudaStream_t s);

// for planes [z0, z1): dst_a[n] = src_a[n] where bm_a has node n (likewise b;
// a null bitmap skips that field). src_* may be mapped host memory.
cudaError_t launch_pull_planes(int nx, int ny, int nz, int z0, int z1, const unsigned long long* bm_a,
                               const double* src_a, double* dst_a, const unsigned long long* bm_b,
                               const double* src_b, double* dst_b, cudaStream_t s);

// *count += set bits of bm in planes [z0, z1)
cudaError_t launch_count_bits(int nx, int ny, int nz, int z0, int z1, const unsigned long long* bm,
                              unsigned long long* count, cudaStream_t s);
