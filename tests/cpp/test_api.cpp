// C++ API test: a program written against the reference's lsr:: headers
// (lsr/evolve.hpp, lsr/grid.hpp) compiles unchanged against include/lsr and
// runs its sl_step on the GPU. Cases restate the reference's known answers
// (proj/tests/test_evolve.cpp:78-123,195-225).
#include <cmath>
#include <cstdio>
#include <limits>

#include "lsr/evolve.hpp"
#include "lsr/grid.hpp"

static int failures = 0;
#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) {                                                   \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);   \
            ++failures;                                               \
        }                                                             \
    } while (0)

static lsr::Grid grid2(double lo, double dx, int n) {
    lsr::Grid g;
    g.dim = 2;
    g.origin = {lo, lo, 0.0};
    g.dx = dx;
    g.dims = {n, n, 1};
    return g;
}

static lsr::BandMask band_of(const lsr::ScalarField& phi, double gamma) {
    lsr::BandMask m;
    m.grid = phi.grid;
    for (std::int64_t id = 0; id < phi.grid.num_nodes(); ++id)
        if (std::abs(phi.values[id]) < gamma) m.active.push_back(id);
    return m;
}

int main() {
    const lsr::Grid g = grid2(-1.3, 0.1, 27);
    lsr::ScalarField phi(g);
    for (int j = 0; j < 27; ++j)
        for (int i = 0; i < 27; ++i) {
            const lsr::Vec p = g.node(i, j, 0);
            phi.at(i, j, 0) = std::sqrt(p[0] * p[0] + p[1] * p[1]) - 0.7;
        }
    lsr::DistanceField dist;
    dist.field = lsr::ScalarField(g, 0.5);
    lsr::StepConfig cfg;
    cfg.band = lsr::default_band_params(2, g.dx);
    cfg.dt = 0.025;
    const lsr::BandMask band = band_of(phi, cfg.band.gamma);
    CHECK(!band.active.empty());

    // identity with constant d and delta = 0 (test_evolve.cpp:78-92)
    lsr::ScalarField next;
    lsr::sl_step(phi, dist, band, cfg, 1.0, next);
    CHECK(next.values.size() == phi.values.size());
    double maxdiff = 0.0;
    for (size_t i = 0; i < phi.values.size(); ++i) maxdiff = std::fmax(maxdiff, std::abs(next.values[i] - phi.values[i]));
    CHECK(maxdiff < 1e-12);

    // zero field -> fallback -> stays exactly zero (test_evolve.cpp:114-123)
    lsr::ScalarField zero(g, 0.0);
    lsr::BandMask all;
    all.grid = g;
    for (std::int64_t id = 0; id < g.num_nodes(); ++id) all.active.push_back(id);
    lsr::sl_step(zero, dist, all, cfg, 1.0, next);
    for (double v : next.values) CHECK(v == 0.0);

    // NaN distance -> NumericalError naming the node (test_evolve.cpp:195-210)
    lsr::DistanceField bad = dist;
    bad.field.values[band.active[band.active.size() / 2]] = std::numeric_limits<double>::quiet_NaN();
    lsr::StepConfig c2 = cfg;
    c2.p = 2;
    c2.delta = 1.0;
    bool threw = false;
    try {
        lsr::sl_step(phi, bad, band, c2, 1.0, next);
    } catch (const lsr::NumericalError& e) {
        threw = std::string(e.what()).find("non-finite update at node") != std::string::npos;
    }
    CHECK(threw);

    // config validation (test_evolve.cpp:212-225) and energy check
    lsr::StepConfig c3 = cfg;
    c3.dt = 0.0;
    threw = false;
    try {
        lsr::sl_step(phi, dist, band, c3, 1.0, next);
    } catch (const lsr::ConfigError&) {
        threw = true;
    }
    CHECK(threw);
    c3 = cfg;
    c3.p = 2;
    threw = false;
    try {
        lsr::sl_step(phi, dist, band, c3, 0.0, next);
    } catch (const lsr::ConfigError&) {
    } catch (const lsr::Error&) {
        threw = true;
    }
    CHECK(threw);

    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
