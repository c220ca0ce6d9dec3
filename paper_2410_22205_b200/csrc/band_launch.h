// Internal interface of the band rebuild and reinitialisation kernels
// (band_reinit.cu).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "sl_device.cuh"

void lsr_note_launch();

// BandMask on the device (grid.hpp:79-84): state per node, ascending
// active / tube id lists.
struct BandBuffers {
    unsigned char* state = nullptr;
    long long* active = nullptr;
    long long* tube = nullptr;
    long long* counts = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    long long cap = 0;
    long long n_active = 0, n_tube = 0;
    int reserve(long long n, std::string* err);
    void release();
};

// ReinitConfig (reinit.hpp:7-18)
struct ReinitParams {
    double dtau;
    int max_iters;
    double residual_tol;
    double sign_eps;
};

struct ReinitBuffers {
    unsigned char* frozen = nullptr;
    long long* nodes = nullptr;
    double* sgn = nullptr;
    unsigned char* nbr = nullptr;  // per node: which axis neighbours exist
    unsigned* nodes32 = nullptr;      // the node list as 4-byte ids (grids below 2^32 nodes)
    long long* frozen_ids = nullptr;  // nodes the one-step froze (ascending), n_frozen of them
    long long n_frozen = 0;
    int* clamp_outside = nullptr;  // device flag: the final clamp changed a node outside the tube
    unsigned long long* scal = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    long long cap = 0;
    int reserve(long long n, std::string* err);
    void release();
};

int lsr_band_build(const lsr_dev::SlParams& P, const double* phi, double gamma, BandBuffers& B, long long* n_active,
                   long long* n_tube, cudaStream_t s, std::string* err);
int lsr_clamp(double* f, long long n, double gamma, cudaStream_t s, std::string* err,
              const unsigned char* state = nullptr, int* outside = nullptr);
int lsr_reinit_one_step(const lsr_dev::SlParams& P, double** phi, double** scratch, ReinitBuffers& W,
                        int* had_interface, cudaStream_t s, std::string* err);
int lsr_reinit_iterate(const lsr_dev::SlParams& P, double** phi, double** scratch, const long long* tube,
                       long long n_tube, const ReinitParams& R, ReinitBuffers& W, bool scratch_differs_on_frozen,
                       int* iterations, cudaStream_t s, std::string* err);
int lsr_reinitialize(const lsr_dev::SlParams& P, double** phi, double** scratch, const BandBuffers& B, double gamma,
                     const ReinitParams& R, ReinitBuffers& W, int* iterations, int* had_interface, cudaStream_t s,
                     std::string* err, bool clamp_sparse = false);

// device-controlled loop (band_reinit.cu, lsr_cuda_loop_run): the words one
// iteration's reinit keeps in device memory instead of reading them back
struct ReinitLoopDev {
    int flags[2];            // the one-step's any_frozen, any_zero
    int clamp_outside;       // the dense clamp changed a node outside the tube
    int pad;
    long long counts[2];     // frozen ids, sweep nodes
    unsigned long long residual_bits;  // the sweeps' control (band_reinit.cu IterState)
    int done;
    int iterations;
    unsigned arrived;
    unsigned pad2;
    long long parts[4];      // list lengths of the dense ([0], [1]) and the tube ([2], [3]) selection
};
int lsr_band_enqueue(const lsr_dev::SlParams& P, const double* phi, double gamma, BandBuffers& B, cudaStream_t s,
                     std::string* err, const int* hard = nullptr);
int lsr_reinit_loop_reserve(long long n, ReinitBuffers& W, std::string* err);
// hard[0]: run the dense one-step (the field may hold a hard jump); hard[1]:
// set when this iteration finds one in phi^{n+1} (see band_reinit.cu
// OneStepGate); the caller moves hard[1] to hard[0] between iterations
int lsr_reinit_enqueue(const lsr_dev::SlParams& P, double* b, double* c, const BandBuffers& B, double gamma,
                       const ReinitParams& R, ReinitBuffers& W, ReinitLoopDev* L, bool clamp_sparse, int* hard,
                       cudaStream_t s, std::string* err);
int lsr_loop_sync_fields(const lsr_dev::SlParams& P, double* b, double* a, double* c, const BandBuffers& B,
                         ReinitBuffers& W, const ReinitLoopDev* L, double gamma, int* hard, bool clamp_sparse,
                         cudaStream_t s, std::string* err);

// z-slab forms (band_reinit.cu): owned planes [own_lo, own_hi) of buffers
// resident on [win_lo, win_hi), passed shifted to global node ids
int lsr_band_build_slab(const lsr_dev::SlParams& P, const double* phi_g, double gamma, BandBuffers& B, int win_lo,
                        int win_hi, int own_lo, int own_hi, long long* n_active, long long* n_tube, cudaStream_t s,
                        std::string* err);
int lsr_reinit_one_step_slab(const lsr_dev::SlParams& P, const double* prev_g, double* out_g, ReinitBuffers& W,
                             int win_lo, int win_hi, int own_lo, int own_hi, int* any_frozen, int* any_zero,
                             cudaStream_t s, std::string* err);
int lsr_reinit_slab_begin(const lsr_dev::SlParams& P, const double* cur_g, double* nxt_g, const long long* tube,
                          long long n_tube, const ReinitParams& R, ReinitBuffers& W, int win_lo, int win_hi,
                          long long* n_nodes, cudaStream_t s, std::string* err);
int lsr_reinit_slab_sweep(const lsr_dev::SlParams& P, const double* cur_g, double* nxt_g, ReinitBuffers& W,
                          long long nn, double dtau, double* residual, cudaStream_t s, std::string* err);
