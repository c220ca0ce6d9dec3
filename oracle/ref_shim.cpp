// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A flat extern "C" face over the *unmodified* reference library, so the
// Python test harness and bench.py's CPU arm can drive the reference's own
// functions through ctypes. The reference sources are compiled where they
// lie (/root/reference/proj/src, see oracle/Makefile) with the reference's
// own FP flags (-ffp-contract=off, proj/CMakeLists.txt:28-30); nothing from
// the reference is copied into this repository.
//
// Each entry point builds the reference containers (ScalarField, BandMask,
// DistanceField) from plain arrays, calls the reference function, copies the
// result back and maps the reference exception hierarchy
// (proj/include/lsr/types.hpp:24-52) to integer status codes matching
// include/lsr_cuda.h.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "lsr/cloud.hpp"
#include "lsr/distance.hpp"
#include "lsr/evolve.hpp"
#include "lsr/grid.hpp"
#include "lsr/interp.hpp"
#include "lsr/metrics.hpp"
#include "lsr/parallel.hpp"
#include "lsr/reference.hpp"
#include "lsr/reinit.hpp"

namespace {

thread_local std::string g_msg;

struct RGrid {  // mirrors lsr_grid in include/lsr_cuda.h
    int32_t dim;
    int32_t dims[3];
    double origin[3];
    double dx;
};

struct RCfg {  // mirrors lsr_step_cfg in include/lsr_cuda.h
    int32_t p;
    int32_t interp;  // 0 = Q1, 1 = WENO
    double delta;
    double dt;
    double fallback_c;
    double fallback_alpha;
    double gamma;
    double beta;
};

lsr::Grid to_grid(const RGrid* g) {
    lsr::Grid out;
    out.dim = g->dim;
    out.dx = g->dx;
    for (int d = 0; d < 3; ++d) {
        out.origin[d] = g->origin[d];
        out.dims[d] = g->dims[d];
    }
    return out;
}

lsr::ScalarField to_field(const lsr::Grid& g, const double* v) {
    lsr::ScalarField f(g);
    std::memcpy(f.values.data(), v, sizeof(double) * f.values.size());
    return f;
}

lsr::StepConfig to_cfg(const RCfg* c) {
    lsr::StepConfig s;
    s.p = c->p;
    s.delta = c->delta;
    s.dt = c->dt;
    s.interp = c->interp == 0 ? lsr::InterpolatorKind::Q1 : lsr::InterpolatorKind::Weno;
    s.fallback_c = c->fallback_c;
    s.fallback_alpha = c->fallback_alpha;
    s.band.gamma = c->gamma;
    s.band.beta = c->beta;
    return s;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const lsr::ConfigError& e) {
        g_msg = e.what();
        return 1;
    } catch (const lsr::NumericalError& e) {
        g_msg = e.what();
        return 3;
    } catch (const lsr::OutOfDomainError& e) {
        g_msg = e.what();
        return 4;
    } catch (const lsr::NoInterfaceError& e) {
        g_msg = e.what();
        return 6;
    } catch (const lsr::Error& e) {
        g_msg = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 2;
    }
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* lsrref_last_error() { return g_msg.c_str(); }

void lsrref_set_threads(int n) { lsr::set_threads(n); }
int lsrref_max_threads() { return lsr::max_threads(); }

// lsr::sl_step (evolve.cpp:40) when serial == 0, lsr::ref::sl_step
// (reference.cpp:53) when serial != 0.
int lsrref_sl_step(int serial, const RGrid* rg, const double* phi, const double* dist,
                   const int64_t* active, int64_t n_active, const RCfg* rc, double energy_p,
                   double* out, double* seconds) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        const lsr::ScalarField f = to_field(g, phi);
        lsr::DistanceField d;
        d.field = to_field(g, dist);
        lsr::BandMask mask;
        mask.grid = g;
        mask.active.assign(active, active + n_active);
        const lsr::StepConfig cfg = to_cfg(rc);
        lsr::ScalarField next;
        const auto t0 = std::chrono::steady_clock::now();
        try {
            if (serial) lsr::ref::sl_step(f, d, mask, cfg, energy_p, next);
            else lsr::sl_step(f, d, mask, cfg, energy_p, next);
        } catch (...) {
            if (seconds) *seconds = seconds_since(t0);
            if (next.values.size() == f.values.size())
                std::memcpy(out, next.values.data(), sizeof(double) * next.values.size());
            throw;
        }
        if (seconds) *seconds = seconds_since(t0);
        std::memcpy(out, next.values.data(), sizeof(double) * next.values.size());
    });
}

// Pre-built inputs for timing the reference repeatedly (bench.py CPU arm):
// the container construction is kept outside the timed call.
struct LsrRefCtx {
    lsr::ScalarField phi;
    lsr::DistanceField dist;
    lsr::BandMask mask;
    lsr::ScalarField next;
};

void* lsrref_ctx_new(const RGrid* rg, const double* phi, const double* dist, const int64_t* active,
                     int64_t n_active) {
    auto* c = new LsrRefCtx;
    const lsr::Grid g = to_grid(rg);
    c->phi = to_field(g, phi);
    c->dist.field = to_field(g, dist);
    c->mask.grid = g;
    c->mask.active.assign(active, active + n_active);
    c->next = lsr::ScalarField(g);
    return c;
}

void lsrref_ctx_free(void* h) { delete static_cast<LsrRefCtx*>(h); }

int lsrref_ctx_sl_step(void* h, int serial, const RCfg* rc, double energy_p, double* seconds) {
    auto* c = static_cast<LsrRefCtx*>(h);
    return guarded([&] {
        const lsr::StepConfig cfg = to_cfg(rc);
        const auto t0 = std::chrono::steady_clock::now();
        if (serial) lsr::ref::sl_step(c->phi, c->dist, c->mask, cfg, energy_p, c->next);
        else lsr::sl_step(c->phi, c->dist, c->mask, cfg, energy_p, c->next);
        *seconds = seconds_since(t0);
    });
}

void lsrref_ctx_out(void* h, double* out) {
    auto* c = static_cast<LsrRefCtx*>(h);
    std::memcpy(out, c->next.values.data(), sizeof(double) * c->next.values.size());
}

// lsr::narrow_band (grid.cpp:76) / lsr::ref::narrow_band (reference.cpp:9).
// state: N bytes; active/tube: capacity N each.
int lsrref_narrow_band(int serial, const RGrid* rg, const double* phi, double gamma, uint8_t* state,
                       int64_t* active, int64_t* n_active, int64_t* tube, int64_t* n_tube) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        const lsr::ScalarField f = to_field(g, phi);
        const lsr::BandMask m = serial ? lsr::ref::narrow_band(f, gamma) : lsr::narrow_band(f, gamma);
        for (size_t i = 0; i < m.state.size(); ++i) state[i] = static_cast<uint8_t>(m.state[i]);
        std::memcpy(active, m.active.data(), sizeof(int64_t) * m.active.size());
        std::memcpy(tube, m.tube.data(), sizeof(int64_t) * m.tube.size());
        *n_active = static_cast<int64_t>(m.active.size());
        *n_tube = static_cast<int64_t>(m.tube.size());
    });
}

// lsr::clamp_field (grid.cpp:126), in place.
int lsrref_clamp_field(const RGrid* rg, double* phi, double gamma) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        lsr::ScalarField f = to_field(g, phi);
        lsr::clamp_field(f, gamma);
        std::memcpy(phi, f.values.data(), sizeof(double) * f.values.size());
    });
}

int lsrref_interp(int kind, const RGrid* rg, const double* f, const double* pts, int64_t n,
                  double* out) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        const lsr::ScalarField fld = to_field(g, f);
        const auto k = kind == 0 ? lsr::InterpolatorKind::Q1
                                 : (kind == 1 ? lsr::InterpolatorKind::Weno
                                              : static_cast<lsr::InterpolatorKind>(kind));
        for (int64_t i = 0; i < n; ++i)
            out[i] = lsr::interp(k, fld, lsr::Vec{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
    });
}

double lsrref_weno_1d(const double* v, double dx, double theta) {
    return lsr::weno_1d(lsr::Stencil4{{v[0], v[1], v[2], v[3]}, dx, theta});
}

void lsrref_weno_linear_weights(double theta, double* lr) {
    const lsr::WenoWeights w = lsr::weno_linear_weights(theta);
    lr[0] = w.left;
    lr[1] = w.right;
}

void lsrref_weno_indicators(const double* v, double dx, double* lr) {
    const lsr::WenoWeights w = lsr::weno_indicators(lsr::Stencil4{{v[0], v[1], v[2], v[3]}, dx, 0.0});
    lr[0] = w.left;
    lr[1] = w.right;
}

int lsrref_locate_cell(const RGrid* rg, const double* p, int32_t* cell) {
    return guarded([&] {
        const lsr::Index3 c = lsr::locate_cell(to_grid(rg), lsr::Vec{p[0], p[1], p[2]});
        for (int d = 0; d < 3; ++d) cell[d] = c[d];
    });
}

void lsrref_centered_gradient(const RGrid* rg, const double* f, int i, int j, int k, double* g3) {
    const lsr::Grid g = to_grid(rg);
    const lsr::ScalarField fld = to_field(g, f);
    const lsr::Vec v = lsr::centered_gradient(fld, i, j, k);
    for (int d = 0; d < 3; ++d) g3[d] = v[d];
}

void lsrref_tangent_basis(int dim, const double* grad, double* v1, double* v2) {
    const lsr::TangentBasis tb = lsr::tangent_basis(dim, lsr::Vec{grad[0], grad[1], grad[2]});
    for (int d = 0; d < 3; ++d) {
        v1[d] = tb.v1[d];
        v2[d] = tb.v2[d];
    }
}

int lsrref_scale_factor(double d_j, double energy_p, int p, double* out) {
    return guarded([&] { *out = lsr::scale_factor(d_j, energy_p, p); });
}

int lsrref_cutoff_weight(double phi, double gamma, double beta, double* out) {
    return guarded([&] { *out = lsr::cutoff_weight(phi, lsr::BandParams{gamma, beta}); });
}

// lsr::surface_energy (metrics.cpp:186) — what the driver feeds to sl_step.
int lsrref_surface_energy(const RGrid* rg, const double* phi, const double* dist, int p,
                          int refine, double* out) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        const lsr::ScalarField f = to_field(g, phi);
        lsr::DistanceField d;
        d.field = to_field(g, dist);
        *out = lsr::surface_energy(f, d, p, refine);
    });
}

// lsr::interface_cells (metrics.cpp:35). cells: capacity = number of cells.
int lsrref_interface_cells(const RGrid* rg, const double* phi, int64_t* cells, int64_t* n) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        const std::vector<int64_t> c = lsr::interface_cells(to_field(g, phi));
        std::memcpy(cells, c.data(), sizeof(int64_t) * c.size());
        *n = static_cast<int64_t>(c.size());
    });
}

// lsr::reinitialize (reinit.cpp:133) on the band computed by lsr::narrow_band
// of the *given* band field (the driver passes the band of phi^n while
// reinitialising phi^{n+1}, driver.cpp:187,196).
int lsrref_reinitialize(const RGrid* rg, double* phi, const double* band_phi, double gamma,
                        double dtau, int max_iters, double residual_tol, double sign_eps,
                        int* iterations, int* had_interface) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        lsr::ScalarField f = to_field(g, phi);
        const lsr::BandMask band = lsr::narrow_band(to_field(g, band_phi), gamma);
        lsr::ReinitConfig cfg;
        cfg.dtau = dtau;
        cfg.max_iters = max_iters;
        cfg.residual_tol = residual_tol;
        cfg.sign_eps = sign_eps;
        const lsr::ReinitResult r = lsr::reinitialize(f, band, gamma, cfg);
        *iterations = r.iterations;
        *had_interface = r.had_interface ? 1 : 0;
        std::memcpy(phi, f.values.data(), sizeof(double) * f.values.size());
    });
}

void lsrref_reinit_defaults(double dx, double gamma, double* dtau, int* max_iters, double* tol,
                            double* sign_eps) {
    const lsr::ReinitConfig c = lsr::ReinitConfig::defaults(dx, gamma);
    *dtau = c.dtau;
    *max_iters = c.max_iters;
    *tol = c.residual_tol;
    *sign_eps = c.sign_eps;
}

static lsr::PointCloud to_cloud(const double* pts, int64_t n, int dim) {
    lsr::PointCloud c;
    c.dim = dim;
    c.points.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) c.points[i] = lsr::Vec{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    return c;
}

// lsr::build_distance_field (distance.cpp:144); seed_only != 0 stops after
// seed_exact_distance (distance.cpp:8).
int lsrref_build_distance(const RGrid* rg, const double* pts, int64_t n, int dim, int seed_only,
                          double* d_out, uint8_t* exact_out, double* sentinel, int* rounds) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        const lsr::PointCloud cloud = to_cloud(pts, n, dim);
        lsr::DistanceField d = lsr::seed_exact_distance(g, cloud);
        *rounds = seed_only ? 0 : lsr::fast_sweep(d);
        std::memcpy(d_out, d.field.values.data(), sizeof(double) * d.field.values.size());
        std::memcpy(exact_out, d.exact.data(), d.exact.size());
        *sentinel = d.sentinel;
    });
}

// lsr::compute_stats (cloud.cpp:480).
int lsrref_compute_stats(const double* pts, int64_t n, int dim, double fraction, double k_s,
                         uint64_t seed, double* h_s, double* gamma_s, double* bbox6) {
    return guarded([&] {
        const lsr::CloudStats st = lsr::compute_stats(to_cloud(pts, n, dim), fraction, k_s, seed);
        *h_s = st.h_s;
        *gamma_s = st.gamma_s;
        for (int d = 0; d < 3; ++d) {
            bbox6[d] = st.bbox_min[d];
            bbox6[3 + d] = st.bbox_max[d];
        }
    });
}

// One iteration of the driver loop body (driver.cpp:185-203) on a fixed
// grid: band, E2, SL step, reinit, swap. phi is updated in place.
int lsrref_loop_step(const RGrid* rg, double* phi, const double* dist, const RCfg* rc,
                     int energy_refine, double* e2_out, int64_t* n_active, int* reinit_iters,
                     double* seconds4) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        lsr::ScalarField f = to_field(g, phi);
        lsr::DistanceField d;
        d.field = to_field(g, dist);
        const lsr::StepConfig step = to_cfg(rc);
        const lsr::ReinitConfig rcfg = lsr::ReinitConfig::defaults(g.dx, step.band.gamma);
        lsr::ScalarField next(g);
        auto t = std::chrono::steady_clock::now();
        const lsr::BandMask band = lsr::narrow_band(f, step.band.gamma);
        if (seconds4) seconds4[0] = seconds_since(t);
        t = std::chrono::steady_clock::now();
        const double e2 = lsr::surface_energy(f, d, 2, energy_refine);
        if (seconds4) seconds4[1] = seconds_since(t);
        t = std::chrono::steady_clock::now();
        if (step.p > 1 && e2 == 0.0) next.values = f.values;
        else lsr::sl_step(f, d, band, step, e2, next);
        if (seconds4) seconds4[2] = seconds_since(t);
        t = std::chrono::steady_clock::now();
        const lsr::ReinitResult rr = lsr::reinitialize(next, band, step.band.gamma, rcfg);
        if (seconds4) seconds4[3] = seconds_since(t);
        *e2_out = e2;
        *n_active = static_cast<int64_t>(band.active.size());
        *reinit_iters = rr.iterations;
        std::memcpy(phi, next.values.data(), sizeof(double) * next.values.size());
    });
}

// K iterations of the same loop body without leaving the library (the long
// end-to-end parity runs): per iteration the E2, |active| and reinit
// iteration count it used. phi is updated in place.
int lsrref_loop_run(const RGrid* rg, double* phi, const double* dist, const RCfg* rc, int energy_refine,
                    int iters, double* e2s, int64_t* n_active, int* reinit_iters) {
    return guarded([&] {
        const lsr::Grid g = to_grid(rg);
        lsr::ScalarField f = to_field(g, phi);
        lsr::DistanceField d;
        d.field = to_field(g, dist);
        const lsr::StepConfig step = to_cfg(rc);
        const lsr::ReinitConfig rcfg = lsr::ReinitConfig::defaults(g.dx, step.band.gamma);
        lsr::ScalarField next(g);
        for (int it = 0; it < iters; ++it) {
            const lsr::BandMask band = lsr::narrow_band(f, step.band.gamma);
            const double e2 = lsr::surface_energy(f, d, 2, energy_refine);
            if (step.p > 1 && e2 == 0.0) next.values = f.values;
            else lsr::sl_step(f, d, band, step, e2, next);
            const lsr::ReinitResult rr = lsr::reinitialize(next, band, step.band.gamma, rcfg);
            e2s[it] = e2;
            n_active[it] = static_cast<int64_t>(band.active.size());
            reinit_iters[it] = rr.iterations;
            std::swap(f.values, next.values);
        }
        std::memcpy(phi, f.values.data(), sizeof(double) * f.values.size());
    });
}

}  // extern "C"
