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

// E_p for the device-controlled loop (energy.cu): the same kernels with the
// cell count kept in device memory and blocked_sum's final pass plus pow on
// the device; *d_e2 = E_p, *d_flags |= 1 when a 2d front leaves the hull
// (interp_q1 -> locate_cell throws, grid.cpp:40). Buffers sized for every
// cell of the grid are reserved first (no allocation while enqueueing).
struct EnergyLoopWork {
    unsigned char* flags = nullptr;
    int* cells = nullptr;
    double* contrib = nullptr;
    double* partial = nullptr;
    long long* nc = nullptr;  // [0] interface cells ([1], [2]: the dense and the tube selection's counts)
    int* ood = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    long long cap = 0;
    void release();
};
int lsr_energy_loop_reserve(const lsr_dev::SlParams& P, EnergyLoopWork& W, std::string* err);
int lsr_energy_enqueue(const lsr_dev::SlParams& P, const double* phi, const double* dist, int p, int refine,
                       EnergyLoopWork& W, long long est_cells, double* d_e2, int* d_flags, cudaStream_t s,
                       std::string* err, const long long* tube = nullptr, const long long* n_tube_dev = nullptr,
                       long long est_tube = 0, const int* hard = nullptr);

// lsr::compute_stats (cloud.cpp:480-489) with the NN sample on the device.
int lsr_prep_compute_stats(const double* h_pts, int64_t n, int dim, double fraction, double k_s, uint64_t seed,
                           double* h_s, double* gamma_s, double* bbox6, cudaStream_t s, std::string* err);

// z-slab surface energy (energy.cu): contributions of the owned cell planes
// [k_lo, k_hi), then this rank's pieces of blocked_sum given its global offset
struct EnergySlabWork {
    unsigned char* flags = nullptr;
    int* cells = nullptr;
    double* contrib = nullptr;
    double* partial = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    long long cap = 0, pcap = 0, nc = 0;
    void release();
};
int lsr_energy_slab_cells(const lsr_dev::SlParams& P, const double* phi_g, const double* dist_g, int p, int refine,
                          int k_lo, int k_hi, EnergySlabWork& W, long long* n_cells, cudaStream_t s,
                          std::string* err);
int lsr_energy_slab_pieces(EnergySlabWork& W, long long offset, double* h_blocks, long long* n_blocks, double* h_head,
                           long long* n_head, double* h_tail, long long* n_tail, cudaStream_t s, std::string* err);
