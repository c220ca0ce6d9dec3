// capi_snippet_main.cpp — INTEGRATION.md Option C as written: the
// reference's own types and functions (its headers, its compiled units,
// evolve.cpp included) plus include/lsr_cuda.h, with driver.cpp's
// lsr::sl_step(phi, dist, band, step, e2, next) call replaced by the
// snippet's lsr_cuda_sl_step_host call. On the same inputs (a reference
// sample cloud, its distance field, band and energy) both must write the
// same bytes into `next`. Test infrastructure only. Usage: capi_snippet.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "lsr/cloud.hpp"
#include "lsr/distance.hpp"
#include "lsr/evolve.hpp"
#include "lsr/grid.hpp"
#include "lsr/metrics.hpp"
#include "lsr_cuda.h"

namespace {

// the INTEGRATION.md Option C snippet, verbatim but for the function frame
void sl_step_gpu(const lsr::ScalarField& phi, const lsr::DistanceField& dist, const lsr::BandMask& band,
                 const lsr::StepConfig& step, double e2, lsr::ScalarField& next) {
    lsr_grid g{phi.grid.dim, {phi.grid.dims[0], phi.grid.dims[1], phi.grid.dims[2]},
               {phi.grid.origin[0], phi.grid.origin[1], phi.grid.origin[2]}, phi.grid.dx};
    lsr_step_cfg c{step.p, step.interp == lsr::InterpolatorKind::Q1 ? LSR_INTERP_Q1 : LSR_INTERP_WENO,
                   step.delta, step.dt, step.fallback_c, step.fallback_alpha, step.band.gamma, step.band.beta};
    if (next.values.size() != phi.values.size()) next = lsr::ScalarField(phi.grid);
    int64_t bad = -1;
    int st = lsr_cuda_sl_step_host(&g, phi.values.data(), dist.field.values.data(), band.active.data(),
                                   (int64_t)band.active.size(), &c, e2, next.values.data(), &bad);
    if (st == LSR_ERR_NUMERICAL) throw lsr::NumericalError(lsr_cuda_last_error_string());
    if (st == LSR_ERR_CONFIG) throw lsr::ConfigError(lsr_cuda_last_error_string());
    if (st != LSR_OK) throw lsr::Error(lsr_cuda_last_error_string());
}

int compare(const char* what, const lsr::ScalarField& a, const lsr::ScalarField& b) {
    if (a.values.size() != b.values.size()) {
        std::printf("%s: sizes differ\n", what);
        return 1;
    }
    long diff = 0;
    for (std::size_t q = 0; q < a.values.size(); ++q)
        diff += std::memcmp(&a.values[q], &b.values[q], sizeof(double)) != 0;
    std::printf("%s: %zu nodes, %ld differ\n", what, a.values.size(), diff);
    return diff != 0;
}

int run(int dim, int n, lsr::InterpolatorKind kind, int p, double delta) {
    lsr::ShapeSpec shape;
    shape.kind = dim == 2 ? lsr::ShapeKind::Circle : lsr::ShapeKind::Sphere;
    shape.size = 0.45;
    shape.n_points = dim == 2 ? 200 : 4000;
    const lsr::PointCloud cloud = lsr::sample_shape(shape, 11);
    lsr::Grid grid;
    grid.dim = dim;
    grid.dims = {n, n, dim == 2 ? 1 : n};
    grid.origin = {-1.0, -1.0, dim == 2 ? 0.0 : -1.0};
    grid.dx = 2.0 / (n - 1);
    const lsr::DistanceField dist = lsr::build_distance_field(grid, cloud);
    lsr::ScalarField phi(grid);
    for (int k = 0; k < grid.dims[2]; ++k)
        for (int j = 0; j < grid.dims[1]; ++j)
            for (int i = 0; i < grid.dims[0]; ++i) {
                const lsr::Vec x = grid.node(i, j, k);
                phi.values[grid.index(i, j, k)] = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]) - 0.8;
            }
    lsr::StepConfig step;
    step.p = p;
    step.delta = delta;
    step.dt = 0.25 * grid.dx;
    step.interp = kind;
    step.band = lsr::default_band_params(dim, grid.dx);
    const lsr::BandMask band = lsr::narrow_band(phi, step.band.gamma);
    const double e2 = lsr::surface_energy(phi, dist, 2, 5);
    lsr::ScalarField ref(grid), gpu(grid);
    lsr::sl_step(phi, dist, band, step, e2, ref);  // the reference (evolve.cpp)
    sl_step_gpu(phi, dist, band, step, e2, gpu);   // Option C
    char what[96];
    std::snprintf(what, sizeof what, "%dd n=%d %s p=%d delta=%g", dim, n,
                  kind == lsr::InterpolatorKind::Q1 ? "Q1" : "WENO", p, delta);
    return compare(what, ref, gpu);
}

}  // namespace

int main() {
    try {
        int bad = 0;
        bad += run(2, 129, lsr::InterpolatorKind::Q1, 1, 0.0);
        bad += run(2, 129, lsr::InterpolatorKind::Weno, 2, 1.0);
        bad += run(3, 48, lsr::InterpolatorKind::Weno, 2, 1.0);
        bad += run(3, 72, lsr::InterpolatorKind::Weno, 2, 0.5);  // >= 64 planes: the pipelined host path
        bad += run(3, 48, lsr::InterpolatorKind::Q1, 1, 0.0);
        if (bad) return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    std::printf("ok\n");
    return 0;
}
