/* lsr_cuda.h — C ABI of the B200 (sm_100a) narrow-band semi-Lagrangian path.
 *
 * This is the drop-in boundary for the reference's hot path
 *     void lsr::sl_step(const ScalarField& phi, const DistanceField& dist,
 *                       const BandMask& mask, const StepConfig& cfg,
 *                       double energy_p, ScalarField& out);
 * declared at /root/reference/proj/include/lsr/evolve.hpp:42-43 and defined
 * at proj/src/evolve.cpp:40-118. The reference has no plugin/FFI layer, so
 * the entry points below are exactly what a C/C++/ctypes binding of that
 * free function (and of the neighbouring band helpers) needs: plain
 * pointers, sizes and POD structs, no C++ or torch types.
 *
 * Semantics (all match the reference unless stated):
 *  - fields are dense fp64, x fastest: id = (k*ny + j)*nx + i
 *    (grid.hpp:19-21); active ids are ascending int64 (grid.hpp:82).
 *  - out equals phi on every non-active node and the SL update on every
 *    active node, bit-for-bit (the kernels are built with --fmad=false and
 *    follow the reference operation order).
 *  - errors are returned as status codes; the message is available through
 *    lsr_cuda_last_error_string(). Config errors are detected before any
 *    device work, like StepConfig::validate() (evolve.hpp:25-30). A
 *    non-finite update yields LSR_ERR_NUMERICAL with *bad_node = the
 *    smallest offending id and `out` fully written (evolve.cpp:109-117; the
 *    reference reports whichever thread stored last, we report the minimum,
 *    which is deterministic).
 *  - every call is synchronous with respect to the host unless it says
 *    otherwise; one context per host thread.
 */
#ifndef LSR_CUDA_H
#define LSR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes — one per reference exception type (types.hpp:24-52) */
#define LSR_OK 0
#define LSR_ERR_CONFIG 1        /* lsr::ConfigError */
#define LSR_ERR 2               /* lsr::Error */
#define LSR_ERR_NUMERICAL 3     /* lsr::NumericalError */
#define LSR_ERR_OUT_OF_DOMAIN 4 /* lsr::OutOfDomainError */
#define LSR_ERR_CUDA 5          /* device / runtime failure (no reference analogue) */
#define LSR_ERR_NO_INTERFACE 6  /* lsr::NoInterfaceError */

/* lsr::InterpolatorKind (interp.hpp:9) */
#define LSR_INTERP_Q1 0
#define LSR_INTERP_WENO 1

/* resident fields of a context */
#define LSR_FIELD_PHI 0  /* phi^n (input of the step) */
#define LSR_FIELD_DIST 1 /* unsigned distance d (DistanceField::field) */
#define LSR_FIELD_OUT 2  /* phi^{n+1} (the double buffer `out`) */
#define LSR_FIELD_SCRATCH 3 /* reinitialisation double buffer (z-slab contexts) */

/* lsr::Grid (grid.hpp:10-52). dims[2] == 1 and origin[2] == 0 in 2d. */
typedef struct lsr_grid {
    int32_t dim;
    int32_t dims[3];
    double origin[3];
    double dx;
} lsr_grid;

/* lsr::StepConfig (evolve.hpp:16-31) with BandParams (grid.hpp:86-93) inlined. */
typedef struct lsr_step_cfg {
    int32_t p;      /* 1 or 2 */
    int32_t interp; /* LSR_INTERP_Q1 / LSR_INTERP_WENO */
    double delta;   /* [0, 1] */
    double dt;      /* > 0 */
    double fallback_c;     /* default 1e-3 */
    double fallback_alpha; /* default 1 */
    double gamma;   /* band half-width */
    double beta;    /* cutoff inner radius, 0 < beta < gamma */
} lsr_step_cfg;

typedef struct lsr_cuda_ctx lsr_cuda_ctx;

const char* lsr_cuda_last_error_string(void);
/* number of CUDA kernels this library has launched in this process */
int64_t lsr_cuda_kernel_launches(void);

/* ---- one-shot drop-in for lsr::sl_step (host buffers in, host buffer out) ----
 * Replaces evolve.cpp:40-118. phi, dist, out: num_nodes doubles; out must not
 * alias phi (evolve.cpp:48-50). */
int lsr_cuda_sl_step_host(const lsr_grid* grid, const double* phi, const double* dist,
                          const int64_t* active, int64_t n_active, const lsr_step_cfg* cfg,
                          double energy_p, double* out, int64_t* bad_node);
/* bytes the calling thread's last lsr_cuda_sl_step_host moved H2D / D2H (3d
 * grids move packed row runs: d where the gradients read it, phi around the
 * band, the band's updated values back; the host copies phi to out) */
void lsr_cuda_last_transfer_bytes(int64_t* h2d, int64_t* d2h);
/* Host-only view of the packed uploads (no GPU needed): for these ascending
 * active ids, copies into dist_field the d values the one-shot 3d step
 * uploads (active nodes and their axis neighbours) and, when reach > 0, into
 * phi_field the phi values of the Chebyshev ball of radius `reach` around
 * every active node. counts[4] = d values, d row runs, phi values, phi row
 * runs. LSR_ERR_CONFIG if the ids are not ascending in-grid (the one-shot
 * step then uploads the fields whole). */
int lsr_cuda_pack_host(const lsr_grid* grid, const int64_t* active, int64_t n_active, int32_t reach,
                       const double* dist, const double* phi, double* dist_field, double* phi_field,
                       int64_t* counts);

/* ---- device-resident context (the loop keeps phi, d, out and ids in HBM) ---- */
int lsr_cuda_create(int device, const lsr_grid* grid, lsr_cuda_ctx** ctx);
int lsr_cuda_destroy(lsr_cuda_ctx* ctx);
/* run on this cudaStream_t (NULL = the context's own stream) */
int lsr_cuda_set_stream(lsr_cuda_ctx* ctx, void* stream);
int lsr_cuda_upload_field(lsr_cuda_ctx* ctx, int which, const double* host);
int lsr_cuda_download_field(lsr_cuda_ctx* ctx, int which, double* host);
/* device pointer of a resident field (plumbing for torch / NCCL); a caller
 * that writes through it must call lsr_cuda_mark_dirty() afterwards */
int lsr_cuda_field_ptr(lsr_cuda_ctx* ctx, int which, double** dptr);
int lsr_cuda_mark_dirty(lsr_cuda_ctx* ctx, int which);
/* BandMask::active (grid.hpp:82): ascending ids, host memory */
int lsr_cuda_set_active(lsr_cuda_ctx* ctx, const int64_t* ids, int64_t n);
/* same, from device memory (e.g. a device-built band) */
int lsr_cuda_set_active_device(lsr_cuda_ctx* ctx, const int64_t* d_ids, int64_t n);
/* lsr::sl_step(PHI, DIST, active, cfg, energy_p, OUT) */
int lsr_cuda_sl_step(lsr_cuda_ctx* ctx, const lsr_step_cfg* cfg, double energy_p,
                     int64_t* bad_node);
/* the same step enqueued without any host synchronisation (device-resident
 * loops, CUDA-graph-style back-to-back submission); a non-finite update is
 * reported by the next lsr_cuda_sync (smallest bad id over the pending
 * steps). lsr_cuda_sl_step refuses to run while async steps are pending. */
int lsr_cuda_sl_step_async(lsr_cuda_ctx* ctx, const lsr_step_cfg* cfg, double energy_p);
/* waits for the pending async steps; LSR_ERR_NUMERICAL as lsr_cuda_sl_step */
int lsr_cuda_sync(lsr_cuda_ctx* ctx, int64_t* bad_node);
/* per-step device times (ms) of the async steps completed by the last sync:
 * SL kernel, whole step, z-line table fill; *n = min(cap, count) */
int lsr_cuda_async_times(lsr_cuda_ctx* ctx, float* kernel_ms, float* step_ms, float* table_ms, int cap,
                         int* n);
/* std::swap(phi.values, next.values) (driver.cpp:203): O(1) */
int lsr_cuda_swap(lsr_cuda_ctx* ctx);
/* 3d WENO step form: 0 = the z-line table kernel (default), 1 = each 8^3
 * brick's phi (+ halo) staged in shared memory by one TMA tensor copy
 * (the measured alternative); same bits either way */
int lsr_cuda_set_sl_mode(lsr_cuda_ctx* ctx, int mode);
/* device time (ms, CUDA events on the context stream) of the last SL kernel
 * and of the last whole sl_step (sync of out + kernel) */
int lsr_cuda_last_times(lsr_cuda_ctx* ctx, float* kernel_ms, float* step_ms);
/* device time (ms) of the last step's z-line table fill (3d WENO; 0 when the
 * step did not use the table); it is part of step_ms, not of kernel_ms */
int lsr_cuda_last_table_ms(lsr_cuda_ctx* ctx, float* table_ms);

/* ---- raw device entry (slab / multi-GPU plumbing) ----
 * Fields hold global planes [z_base, z_base + z_planes) of `grid` (3d) — a
 * z-slab plus halo; ids stay global. A node whose gradient or foot stencil
 * leaves the resident planes is counted in *halo_miss and its output is not
 * meaningful: the caller must widen the halo and redo.
 * Asynchronous on `stream`; bad_node/halo_miss are device int64 pointers
 * (bad_node initialised to INT64_MAX by the caller). */
int lsr_cuda_sl_step_device(const lsr_grid* grid, int32_t z_base, int32_t z_planes,
                            const double* d_phi, const double* d_dist, const int64_t* d_active,
                            int64_t n_active, const lsr_step_cfg* cfg, double energy_p,
                            double* d_out, int64_t* d_bad_node, int64_t* d_halo_miss,
                            void* stream);

/* Fused SL step + halo exchange (SURVEY §8(e) phase 2): as above with an
 * owned plane range [own_lo, own_hi); every update of a node in the first
 * push_lo_planes owned planes is ALSO stored into d_peer_lo_out (the lower
 * neighbour's resident out buffer, whose first resident plane is
 * peer_lo_zbase; a peer-mapped NVLink pointer from lsr_cuda_ipc_open), and
 * of a node in the last push_hi_planes owned planes into d_peer_hi_out. The
 * neighbours read those planes next step, so no plane exchange follows the
 * kernel; the caller only orders the ranks (a stream-ordered barrier). Peer
 * pointers may be NULL. */
int lsr_cuda_sl_step_device_fused(const lsr_grid* grid, int32_t z_base, int32_t z_planes, int32_t own_lo,
                                  int32_t own_hi, const double* d_phi, const double* d_dist, const int64_t* d_active,
                                  int64_t n_active, const lsr_step_cfg* cfg, double energy_p, double* d_out,
                                  double* d_peer_lo_out, int32_t peer_lo_zbase, int32_t push_lo_planes,
                                  double* d_peer_hi_out, int32_t peer_hi_zbase, int32_t push_hi_planes,
                                  int64_t* d_bad_node, int64_t* d_halo_miss, void* stream);
/* raw device buffers (whole allocations, so CUDA IPC handles cover them) and
 * CUDA IPC for the peer pointers of the fused path (handles are 64 bytes) */
int lsr_cuda_malloc(size_t bytes, void** dptr);
int lsr_cuda_free(void* dptr);
int lsr_cuda_ipc_handle(void* dptr, uint8_t* handle64);
int lsr_cuda_ipc_open(const uint8_t* handle64, void** dptr);
int lsr_cuda_ipc_close(void* dptr);

/* ---- point-cloud preprocessing ----
 * lsr::build_distance_field (distance.cpp:144-148; header distance.hpp:29):
 * seed_exact_distance (distance.cpp:8-52) then fast_sweep (:72-142),
 * bit-identical to the reference. pts: n points as x,y,z triples (host).
 * seed_only != 0 stops after seed_exact_distance (distance.hpp:24).
 * d_out (num_nodes doubles) and exact_out (num_nodes bytes) are host
 * buffers; either may be NULL. *rounds = fast_sweep's return value. */
int lsr_cuda_build_distance(const lsr_grid* grid, const double* pts, int64_t n, int dim, int seed_only,
                            double* d_out, uint8_t* exact_out, double* sentinel, int* rounds);
/* same, writing the context's resident DIST field */
int lsr_cuda_ctx_build_distance(lsr_cuda_ctx* ctx, const double* pts, int64_t n, int dim, int seed_only,
                                double* sentinel, int* rounds);

/* lsr::fast_sweep (distance.cpp:72-142) of the context's DIST field in
 * place, bit-identical: exact (num_nodes bytes, host; NULL = the flags of
 * the last lsr_cuda_ctx_build_distance) marks the nodes never modified,
 * values >= sentinel are unseeded. *rounds = fast_sweep's return value.
 * lsr_cuda_download_exact copies the context's exact flags to the host. */
int lsr_cuda_fast_sweep(lsr_cuda_ctx* ctx, const uint8_t* exact, double sentinel, int* rounds);
int lsr_cuda_download_exact(lsr_cuda_ctx* ctx, uint8_t* exact);

/* lsr::compute_stats (cloud.cpp:480-489; cloud.hpp:52-53): h_S =
 * estimate_resolution (mean exact nearest-neighbour distance over a seeded
 * Fisher-Yates sample of round(fraction*n) points, blocked_sum order),
 * gamma_S = k_s * h_S and the bounding box (bbox6 = lo[3], hi[3]).
 * Bit-identical to the reference. */
int lsr_cuda_compute_stats(const double* pts, int64_t n, int dim, double sample_fraction, double k_s, uint64_t seed,
                           double* h_s, double* gamma_s, double* bbox6);

/* ---- surface energy ----
 * lsr::surface_energy (metrics.cpp:186-189; header metrics.hpp:41-42): E_p
 * of the field `which` (LSR_FIELD_PHI or LSR_FIELD_OUT) against the
 * context's DIST field; 3d: energy_3d with `refine` subcells per axis, 2d:
 * energy_2d. Same cells, same quadrature, same blocked_sum order as the
 * reference; |d|^2 is computed as |d|*|d| where the reference calls glibc
 * pow (not correctly rounded), so E_p agrees to a few ulp. */
int lsr_cuda_surface_energy(lsr_cuda_ctx* ctx, int which, int p, int refine, double* energy);
int lsr_cuda_surface_energy_host(const lsr_grid* grid, const double* phi, const double* dist, int p, int refine,
                                 double* energy);

/* ---- band rebuild ----
 * lsr::narrow_band (grid.cpp:76-124; grid.hpp:105) of field `which` (PHI or
 * OUT): NodeState per node, ascending ACTIVE and tube (ACTIVE+REINIT_HALO)
 * lists, bit-identical; the ACTIVE list also becomes the context's active
 * set for lsr_cuda_sl_step. lsr_cuda_band_download copies the last band to
 * host (state: num_nodes bytes; active/tube: n_active/n_tube ids; any may be
 * NULL). lsr::clamp_field (grid.cpp:126-134) in place. */
int lsr_cuda_narrow_band(lsr_cuda_ctx* ctx, int which, double gamma, int64_t* n_active, int64_t* n_tube);
int lsr_cuda_band_download(lsr_cuda_ctx* ctx, uint8_t* state, int64_t* active, int64_t* tube);
int lsr_cuda_clamp_field(lsr_cuda_ctx* ctx, int which, double gamma);

/* ---- reinitialisation ----
 * lsr::reinitialize (reinit.cpp:133-145; reinit.hpp:43-44) of field `which`
 * on the band last built by lsr_cuda_narrow_band: interface_one_step,
 * Jacobi reinit_iterate on tube minus frozen, clamp to [-gamma, gamma].
 * Bit-identical, same iteration count. ReinitConfig (reinit.hpp:7-18): */
typedef struct lsr_reinit_cfg {
    double dtau;
    int32_t max_iters;
    double residual_tol;
    double sign_eps;
} lsr_reinit_cfg;
int lsr_cuda_reinitialize(lsr_cuda_ctx* ctx, int which, double gamma, const lsr_reinit_cfg* cfg, int* iterations,
                          int* had_interface);
/* A host BandMask (grid.hpp:79-84) as the context's band: state (num_nodes
 * bytes), ascending ACTIVE and tube ids; the ACTIVE list also becomes the
 * active set. (lsr_cuda_narrow_band builds the band on the device instead.) */
int lsr_cuda_set_band(lsr_cuda_ctx* ctx, const uint8_t* state, const int64_t* active, int64_t n_active,
                      const int64_t* tube, int64_t n_tube);
/* lsr::interface_one_step (reinit.cpp:18-59) of field `which` in place;
 * frozen (num_nodes bytes, may be NULL) receives the flags, which also stay
 * on the device for lsr_cuda_reinit_iterate. A field without sign change or
 * zero is left unchanged and LSR_ERR_NO_INTERFACE is returned (the
 * reference's NoInterfaceError). */
int lsr_cuda_interface_one_step(lsr_cuda_ctx* ctx, int which, uint8_t* frozen, int* had_interface);
/* lsr::reinit_iterate (reinit.cpp:88-131) of field `which` in place on the
 * context's band tube minus the frozen nodes (host flags, or NULL = those of
 * the last lsr_cuda_interface_one_step); *iterations = its return value. */
int lsr_cuda_reinit_iterate(lsr_cuda_ctx* ctx, int which, const uint8_t* frozen, const lsr_reinit_cfg* cfg,
                            int* iterations);
/* ReinitConfig::defaults(dx, gamma) (reinit.cpp:8-16) */
void lsr_cuda_reinit_defaults(double dx, double gamma, lsr_reinit_cfg* cfg);

/* ---- one iteration of the driver loop body on the device ----
 * driver.cpp:187-203 on a fixed grid: band of PHI, E_2 of PHI (or
 * energy_override when >= 0), sl_step PHI -> OUT, reinitialize OUT on the
 * band of PHI, swap. Per-phase device times in ms[0..3] (band, energy, SL,
 * reinit). */
typedef struct lsr_loop_stats {
    double energy;
    int64_t n_active;
    int64_t n_tube;
    int32_t reinit_iterations;
    int32_t had_interface;
    float ms[4];
    int32_t dense_one_step; /* the one-step visited every node (else the tube only: lsr_cuda_loop_run) */
    int32_t reserved;
} lsr_loop_stats;
int lsr_cuda_loop_step(lsr_cuda_ctx* ctx, const lsr_step_cfg* cfg, const lsr_reinit_cfg* rcfg, int energy_refine,
                       double energy_override, lsr_loop_stats* stats);
/* K iterations of the same loop body, device-controlled: the band counts,
 * the interface-cell count, E_2 (blocked_sum and pow on the device), the
 * p > 1 && E_2 == 0 skip, the NoInterface case and the Jacobi stop rule are
 * all decided on the device, so the K iterations are enqueued without a host
 * round trip and the host synchronises once, at the end, to read the K
 * records (stats[0..K), NULL = none; ms = device time per phase). use_graph:
 * iterations after the first are replays of a captured CUDA graph of one
 * iteration. *done = iterations completed (K, or the index of the first one
 * that failed: non-finite update, E_2 NaN, a 2d front outside the hull — the
 * reference throws there; the fields are then unspecified). E_2 differs from
 * lsr_cuda_loop_step's (host glibc pow) only where glibc's pow(x, 0.5) is
 * not the correctly rounded sqrt. The box SL form (lsr_cuda_set_sl_mode 1) is
 * not used here. */
int lsr_cuda_loop_run(lsr_cuda_ctx* ctx, const lsr_step_cfg* cfg, const lsr_reinit_cfg* rcfg, int energy_refine,
                      int iterations, int use_graph, lsr_loop_stats* stats, int* done);

/* ---- z-slab loop (driver.cpp:185-203 split over ranks) ----
 * A slab context holds the resident planes [win_lo, win_hi) of the global
 * grid (fields of (win_hi - win_lo) * nx * ny values; upload / download /
 * field_ptr move whole windows) and works on the owned planes
 * [own_lo, own_hi), win_lo <= max(own_lo - 1, 0), min(own_hi + 1, nz) <=
 * win_hi. Node ids (active / tube lists, bad_node) are global. Between the
 * phases the caller exchanges halo planes (lsr_cuda_slab_copy_planes) and
 * reduces over the ranks; every phase gives the owned nodes the bits the
 * whole-grid function gives them (paper_2410_22205_b200/zslab.py drives it). */
int lsr_cuda_slab_create(int device, const lsr_grid* grid, int32_t win_lo, int32_t win_hi, int32_t own_lo,
                         int32_t own_hi, lsr_cuda_ctx** ctx);
/* planes [plane0, plane0 + nplanes) of field `which` to (to_field = 0) or
 * from (1) nplanes * nx * ny doubles of device memory at dev */
int lsr_cuda_slab_copy_planes(lsr_cuda_ctx* ctx, int which, int32_t plane0, int32_t nplanes, void* dev,
                              int32_t to_field);
/* narrow_band (grid.cpp:76-124) of the owned planes; needs `which` valid on
 * the owned planes +- 1; the ACTIVE list becomes the active set */
int lsr_cuda_slab_band(lsr_cuda_ctx* ctx, int which, double gamma, int64_t* n_active, int64_t* n_tube);
/* surface_energy's interface cells of the owned cell planes and their
 * contributions (metrics.cpp:145-184); then, given the global position of
 * this rank's first contribution (the sum of the lower ranks' counts), its
 * pieces of blocked_sum (parallel.hpp:26-42): the sums of the 4096-blocks
 * wholly inside its range, and the raw contributions before its first
 * (head, < 4096) and after its last (tail, < 4096) block boundary. blocks
 * holds n_cells / 4096 + 1 values. */
int lsr_cuda_slab_energy_cells(lsr_cuda_ctx* ctx, int which, int p, int refine, int64_t* n_cells);
int lsr_cuda_slab_energy_pieces(lsr_cuda_ctx* ctx, int64_t offset, double* blocks, int64_t* n_blocks, double* head,
                                int64_t* n_head, double* tail, int64_t* n_tail);
/* largest foot displacement bound (cells) over the owned active nodes: the
 * halo must exceed it by the stencil radius + 1 (2 + 1 for WENO) */
int lsr_cuda_slab_max_reach(lsr_cuda_ctx* ctx, const lsr_step_cfg* cfg, double energy_p, double* cells);
/* sl_step on the owned active nodes: OUT = PHI on the window, then the
 * updates; *halo_miss = stencils that left the resident planes (then the
 * result is void: widen the halo and redo) */
int lsr_cuda_slab_sl_step(lsr_cuda_ctx* ctx, const lsr_step_cfg* cfg, double energy_p, int64_t* bad_node,
                          int64_t* halo_miss);
/* reinitialize (reinit.cpp:133-145) in phases: interface_one_step OUT ->
 * SCRATCH on the owned planes (OUT valid on owned +- 1); reinit_begin after
 * SCRATCH's halo planes are exchanged; sweep k reads buf[k & 1] and writes
 * buf[(k + 1) & 1], buf = {SCRATCH, OUT}, returning the owned max |upd|;
 * reinit_end clamps the result field's owned planes and makes it OUT */
int lsr_cuda_slab_one_step(lsr_cuda_ctx* ctx, int* any_frozen, int* any_zero);
int lsr_cuda_slab_reinit_begin(lsr_cuda_ctx* ctx, const lsr_reinit_cfg* rcfg, int64_t* n_nodes);
int lsr_cuda_slab_reinit_sweep(lsr_cuda_ctx* ctx, const lsr_reinit_cfg* rcfg, int32_t k, double* residual);
int lsr_cuda_slab_reinit_end(lsr_cuda_ctx* ctx, int which, double gamma);

/* ---- self-test hook ----
 * Divides n pseudo-random doubles by c with the kernels' constant-divisor
 * division and with the hardware IEEE division; *mismatches = how many
 * quotients differ in any bit (must be 0). */
int lsr_cuda_selftest_div_const(double c, int64_t n, uint64_t seed, int64_t* mismatches);
/* Differential test of the exact fast WENO forms (weno1_fast, and weno1_zt
 * fed the z-line table's terms) against weno_1d with the plain IEEE
 * operators, over n pseudo-random stencils and abscissae (smooth lines, raw
 * bit patterns, lines at the range/halving guards, tiny differences) at this
 * dx (in [2^-30, 1]). counts[4] = fast path taken, fast mismatches, table
 * path taken, table mismatches; both mismatch counts must be 0. */
int lsr_cuda_selftest_weno(double dx, int64_t n, uint64_t seed, int64_t* counts);

#ifdef __cplusplus
}
#endif
#endif /* LSR_CUDA_H */
