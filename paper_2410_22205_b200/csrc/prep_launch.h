// Internal interface of the preprocessing / band / energy kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "lsr_cuda.h"
#include "sl_device.cuh"

void lsr_note_launch();

// lsr::build_distance_field on the device (distance.cu). d_field: N doubles,
// d_exact: N bytes (device). Returns an LSR_* status; *err holds the message.
int lsr_prep_build_distance(const lsr_grid* g, const double* h_pts, int64_t n, int dim, int seed_only,
                            double* d_field, unsigned char* d_exact, double* sentinel_out, int* rounds_out,
                            cudaStream_t s, std::string* err);

// lsr::fast_sweep (distance.cpp:72-142) of a device field in place.
int lsr_prep_fast_sweep(const lsr_grid* g, double* d_field, const unsigned char* d_exact, double sentinel,
                        int* rounds_out, cudaStream_t s, std::string* err);

// lsr::surface_energy on device fields (energy.cu); synchronous.
int lsr_prep_surface_energy(const lsr_dev::SlParams& P, const double* phi, const double* dist, int p, int refine,
                            double* energy, int64_t* n_cells, cudaStream_t s, std::string* err);

// lsr::compute_stats (cloud.cpp:480-489) with the NN sample on the device.
int lsr_prep_compute_stats(const double* h_pts, int64_t n, int dim, double fraction, double k_s, uint64_t seed,
                           double* h_s, double* gamma_s, double* bbox6, cudaStream_t s, std::string* err);
