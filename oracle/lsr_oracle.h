/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference's narrow-band semi-Lagrangian path
 * (arXiv 2410.22205 artifact, /root/reference/proj). Every function cites the
 * reference file:line it restates. Arithmetic follows the reference operation
 * order exactly and is compiled with -ffp-contract=off, so results are
 * bit-identical to the reference (pinned in tests/test_oracle.py against
 * oracle/_ref — the reference itself — and tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef LSR_ORACLE_H
#define LSR_ORACLE_H

#include <stdint.h>

#include "../include/lsr_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* --- grid helpers (grid.hpp:10-52, grid.cpp:39-74,126-143) --- */
int lsro_locate_cell(const lsr_grid* g, const double p[3], int32_t cell[3]);
void lsro_centered_gradient(const lsr_grid* g, const double* f, int i, int j, int k, double out[3]);
double lsro_cutoff_weight(double phi, double gamma, double beta);

/* --- interpolation (interp.cpp:7-119) --- */
double lsro_weno_1d(const double v[4], double dx, double theta);
int lsro_interp(int kind, const lsr_grid* g, const double* f, const double p[3], double* out);

/* --- evolve (evolve.cpp:10-118) --- */
void lsro_tangent_basis(int dim, const double grad[3], double v1[3], double v2[3]);
int lsro_scale_factor(double d_j, double energy_p, int p, double* out);
/* Full sl_step: validates, copies phi into out, updates the active ids.
 * Returns LSR_OK or an error status; *bad_node = smallest non-finite id. */
int lsro_sl_step(const lsr_grid* g, const double* phi, const double* dist, const int64_t* active,
                 int64_t n_active, const lsr_step_cfg* cfg, double energy_p, double* out,
                 int64_t* bad_node, int nthreads);

/* --- band (grid.cpp:76-134) --- */
int lsro_narrow_band(const lsr_grid* g, const double* phi, double gamma, uint8_t* state,
                     int64_t* active, int64_t* n_active, int64_t* tube, int64_t* n_tube);
int lsro_clamp_field(const lsr_grid* g, double* f, double gamma);

const char* lsro_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
