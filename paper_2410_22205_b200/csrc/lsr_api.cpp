// lsr_api.cpp — definitions of the C++ `lsr::` face (include/lsr/lsr_b200.hpp)
// over the C ABI, grouped by the reference translation unit they replace.
//
// Error behaviour follows the reference: checks it performs before touching
// data throw before any device work, with the reference's exception classes
// and messages. The GPU-backed functions move host fields through one
// device context per host thread (kept across calls for the same grid), so
// a caller such as run_schedule (driver.cpp:139-230) runs unchanged; the
// device-resident loop without per-call PCIe traffic is lsr::cuda::Session.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "lsr/lsr_b200.hpp"

namespace lsr {

void throw_status(int status) {
    if (status == LSR_OK) return;
    const std::string msg = lsr_cuda_last_error_string();
    switch (status) {
        case LSR_ERR_CONFIG: throw ConfigError(msg);
        case LSR_ERR_NUMERICAL: throw NumericalError(msg);
        case LSR_ERR_OUT_OF_DOMAIN: throw OutOfDomainError(msg);
        case LSR_ERR_NO_INTERFACE: throw NoInterfaceError(msg);
        case LSR_ERR_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}

namespace {

// The calling thread's device context for grid g (re-created when the grid
// or the current device changes).
lsr_cuda_ctx* host_ctx(const Grid& g) {
    struct Cache {
        lsr_cuda_ctx* ctx = nullptr;
        lsr_grid grid{};
        int device = -1;
        ~Cache() { lsr_cuda_destroy(ctx); }
    };
    thread_local Cache cache;
    const lsr_grid cg = to_c(g);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    if (cache.ctx && (std::memcmp(&cache.grid, &cg, sizeof cg) != 0 || cache.device != dev)) {
        lsr_cuda_destroy(cache.ctx);
        cache.ctx = nullptr;
    }
    if (!cache.ctx) {
        throw_status(lsr_cuda_create(dev, &cg, &cache.ctx));
        cache.grid = cg;
        cache.device = dev;
    }
    return cache.ctx;
}

void upload(lsr_cuda_ctx* c, int which, const ScalarField& f) {
    throw_status(lsr_cuda_upload_field(c, which, f.values.data()));
}

void download(lsr_cuda_ctx* c, int which, ScalarField& f) {
    throw_status(lsr_cuda_download_field(c, which, f.values.data()));
}

void require_size(const ScalarField& f, const char* who) {
    if (f.values.size() != static_cast<std::size_t>(f.grid.num_nodes()))
        throw ConfigError(std::string(who) + ": field size does not match its grid");
}

void upload_band(lsr_cuda_ctx* c, const BandMask& band) {
    if (band.state.size() != static_cast<std::size_t>(band.grid.num_nodes()))
        throw ConfigError("band: state size does not match its grid");
    throw_status(lsr_cuda_set_band(c, reinterpret_cast<const uint8_t*>(band.state.data()), band.active.data(),
                                   static_cast<int64_t>(band.active.size()), band.tube.data(),
                                   static_cast<int64_t>(band.tube.size())));
}

std::vector<double> triples(const PointCloud& cloud) {  // Vec is a plain 3-double record
    std::vector<double> xyz(3 * cloud.points.size());
    for (std::size_t q = 0; q < cloud.points.size(); ++q)
        for (int d = 0; d < 3; ++d) xyz[3 * q + d] = cloud.points[q][d];
    return xyz;
}

}  // namespace

// ----------------------------------------------------- evolve.cpp (evolve.hpp)

TangentBasis tangent_basis(int dim, const Vec& grad) {  // evolve.cpp:10-30, same expressions
    TangentBasis tb;
    const double gn = norm(grad);
    if (dim == 2) {
        tb.v1 = gn == 0.0 ? Vec{1.0, 0.0, 0.0} : Vec{grad[1] / gn, -grad[0] / gn, 0.0};
        return tb;
    }
    const double r = std::sqrt(sqr(grad[0]) + sqr(grad[2]));
    if (gn == 0.0 || r < 1e-14 * gn) {  // degenerate: the fixed axes
        tb.v1 = {1.0, 0.0, 0.0};
        tb.v2 = {0.0, 0.0, 1.0};
        return tb;
    }
    const double rg = r * gn;
    tb.v1 = {-grad[2] / r, 0.0, grad[0] / r};
    tb.v2 = {-grad[0] * grad[1] / rg, r / gn, -grad[1] * grad[2] / rg};
    return tb;
}

double scale_factor(double d_j, double energy_p, int p) {  // evolve.cpp:32-38: (d_j / E)^(p-1)
    if (p == 1) return 1.0;
    if (!(energy_p > 0.0)) throw Error("scale_factor: energy must be positive for p > 1");
    double f = 1.0;
    for (int q = 1; q < p; ++q) f *= d_j / energy_p;
    return f;
}

void sl_step(const ScalarField& phi, const DistanceField& dist, const BandMask& mask, const StepConfig& cfg,
             double energy_p, ScalarField& out) {
    cfg.validate();  // evolve.cpp:42-46
    if (!(phi.grid == dist.field.grid) || !(phi.grid == mask.grid))
        throw ConfigError("sl_step: phi, dist and mask must share one grid");
    if (cfg.p > 1 && !(energy_p > 0.0)) throw Error("sl_step: energy must be positive for p > 1");
    require_size(phi, "sl_step");
    require_size(dist.field, "sl_step");
    const Grid& g = phi.grid;
    if (!(out.grid == g) || out.values.size() != phi.values.size()) out = ScalarField(g);
    const lsr_grid cg = to_c(g);
    const lsr_step_cfg cc = to_c(cfg);
    std::int64_t bad = -1;
    throw_status(lsr_cuda_sl_step_host(&cg, phi.values.data(), dist.field.values.data(), mask.active.data(),
                                       static_cast<std::int64_t>(mask.active.size()), &cc, energy_p,
                                       out.values.data(), &bad));
}

// --------------------------------------------------------- grid.cpp (grid.hpp)
// build_grid, locate_cell, default_band_params, centered_gradient and
// cutoff_weight are per-call scalar utilities of the API (no field-wide
// work), computed on the host with the reference's expressions.

Grid build_grid(const Vec& bbox_min, const Vec& bbox_max, int dim, double dx, int pad_cells,
                std::int64_t node_budget) {  // grid.cpp:9-37
    if (dim != 2 && dim != 3) throw ConfigError("build_grid: dim must be 2 or 3");
    if (!(dx > 0.0)) throw ConfigError("build_grid: dx must be positive");
    if (pad_cells < 2) throw ConfigError("build_grid: pad_cells must be >= 2");
    for (int d = 0; d < dim; ++d)
        if (!(bbox_min[d] < bbox_max[d])) throw ConfigError("build_grid: bbox_min must be < bbox_max componentwise");
    Grid g;
    g.dim = dim;
    g.dx = dx;
    std::int64_t nodes = 1;
    for (int d = 0; d < 3; ++d) {
        if (d >= dim) {  // unused axis
            g.origin[d] = 0.0;
            g.dims[d] = 1;
            continue;
        }
        g.origin[d] = bbox_min[d] - pad_cells * dx;
        const double extent = bbox_max[d] + pad_cells * dx - g.origin[d];
        g.dims[d] = 1 + static_cast<int>(std::ceil(extent / dx - 1e-9));
        nodes *= g.dims[d];
        if (nodes > node_budget)
            throw Error("build_grid: " + std::to_string(nodes) + "+ nodes exceed budget " + std::to_string(node_budget));
    }
    return g;
}

Index3 locate_cell(const Grid& g, const Vec& p) {  // grid.cpp:39-47
    if (!g.contains(p)) throw OutOfDomainError("locate_cell: point outside grid hull");
    Index3 cell{0, 0, 0};
    for (int d = 0; d < g.dim; ++d) {
        const int c = static_cast<int>(std::floor((p[d] - g.origin[d]) / g.dx));
        cell[d] = std::clamp(c, 0, g.dims[d] - 2);
    }
    return cell;
}

BandParams default_band_params(int dim, double dx) {  // grid.cpp:49-51
    if (dim == 2) return BandParams{4.0 * dx, 2.0 * dx};
    return BandParams{6.0 * dx, 3.0 * dx};
}

Vec centered_gradient(const ScalarField& f, int i, int j, int k) {  // grid.cpp:53-74
    const Grid& g = f.grid;
    const double inv2 = 1.0 / (2.0 * g.dx);
    const double inv1 = 1.0 / g.dx;
    const int at[3] = {i, j, k};
    Vec grad{0, 0, 0};
    for (int d = 0; d < g.dim; ++d) {
        int m[3] = {i, j, k}, p[3] = {i, j, k};
        if (at[d] == 0) {  // forward difference at the low hull
            p[d] = 1;
            grad[d] = (f.at(p[0], p[1], p[2]) - f.at(i, j, k)) * inv1;
        } else if (at[d] == g.dims[d] - 1) {  // backward difference at the high hull
            m[d] = g.dims[d] - 2;
            grad[d] = (f.at(i, j, k) - f.at(m[0], m[1], m[2])) * inv1;
        } else {
            m[d] -= 1;
            p[d] += 1;
            grad[d] = (f.at(p[0], p[1], p[2]) - f.at(m[0], m[1], m[2])) * inv2;
        }
    }
    return grad;
}

BandMask narrow_band(const ScalarField& phi, double gamma) {  // GPU (grid.cpp:76-124)
    require_size(phi, "narrow_band");
    lsr_cuda_ctx* c = host_ctx(phi.grid);
    upload(c, LSR_FIELD_PHI, phi);
    std::int64_t na = 0, nt = 0;
    throw_status(lsr_cuda_narrow_band(c, LSR_FIELD_PHI, gamma, &na, &nt));
    BandMask m;
    m.grid = phi.grid;
    m.state.resize(static_cast<std::size_t>(phi.grid.num_nodes()));
    m.active.resize(static_cast<std::size_t>(na));
    m.tube.resize(static_cast<std::size_t>(nt));
    throw_status(lsr_cuda_band_download(c, reinterpret_cast<uint8_t*>(m.state.data()), m.active.data(), m.tube.data()));
    return m;
}

void clamp_field(ScalarField& f, double gamma) {  // GPU (grid.cpp:126-134)
    if (!(gamma > 0.0)) throw ConfigError("clamp_field: gamma must be positive");
    require_size(f, "clamp_field");
    lsr_cuda_ctx* c = host_ctx(f.grid);
    upload(c, LSR_FIELD_PHI, f);
    throw_status(lsr_cuda_clamp_field(c, LSR_FIELD_PHI, gamma));
    download(c, LSR_FIELD_PHI, f);
}

double cutoff_weight(double phi, const BandParams& params) {  // grid.cpp:136-143
    params.validate();
    const double a = std::abs(phi);
    if (a <= params.beta) return 1.0;
    if (a > params.gamma) return 0.0;
    const double g = params.gamma, b = params.beta;
    return sqr(a - g) * (2.0 * a + g - 3.0 * b) / ((g - b) * (g - b) * (g - b));
}

// ------------------------------------------------- distance.cpp (distance.hpp)

namespace {

DistanceField distance_field(const Grid& grid, const PointCloud& cloud, int seed_only) {
    if (cloud.points.empty()) throw Error("seed_exact_distance: empty cloud");  // distance.cpp:9
    if (cloud.dim != grid.dim) throw ConfigError("seed_exact_distance: dimension mismatch");
    const lsr_grid cg = to_c(grid);
    DistanceField d;
    d.field = ScalarField(grid);
    d.exact.assign(static_cast<std::size_t>(grid.num_nodes()), 0);
    const std::vector<double> xyz = triples(cloud);
    int rounds = 0;
    throw_status(lsr_cuda_build_distance(&cg, xyz.data(), cloud.size(), cloud.dim, seed_only, d.field.values.data(),
                                         d.exact.data(), &d.sentinel, &rounds));
    return d;
}

}  // namespace

DistanceField seed_exact_distance(const Grid& grid, const PointCloud& cloud) {  // GPU (distance.cpp:8-52)
    return distance_field(grid, cloud, 1);
}

int fast_sweep(DistanceField& d) {  // GPU (distance.cpp:72-142)
    require_size(d.field, "fast_sweep");
    if (d.exact.size() != d.field.values.size()) throw ConfigError("fast_sweep: exact flags do not match the field");
    lsr_cuda_ctx* c = host_ctx(d.field.grid);
    upload(c, LSR_FIELD_DIST, d.field);
    int rounds = 0;
    throw_status(lsr_cuda_fast_sweep(c, d.exact.data(), d.sentinel, &rounds));
    download(c, LSR_FIELD_DIST, d.field);
    return rounds;
}

DistanceField build_distance_field(const Grid& grid, const PointCloud& cloud) {  // GPU (distance.cpp:144-148)
    return distance_field(grid, cloud, 0);
}

// ----------------------------------------------------- reinit.cpp (reinit.hpp)

ReinitConfig ReinitConfig::defaults(double dx, double gamma) {  // reinit.cpp:8-16
    lsr_reinit_cfg r{};
    lsr_cuda_reinit_defaults(dx, gamma, &r);
    ReinitConfig cfg;
    cfg.dtau = r.dtau;
    cfg.max_iters = r.max_iters;
    cfg.residual_tol = r.residual_tol;
    cfg.sign_eps = r.sign_eps;
    cfg.validate();
    return cfg;
}

std::vector<std::uint8_t> interface_one_step(ScalarField& phi) {  // GPU (reinit.cpp:18-59)
    require_size(phi, "interface_one_step");
    lsr_cuda_ctx* c = host_ctx(phi.grid);
    upload(c, LSR_FIELD_PHI, phi);
    std::vector<std::uint8_t> frozen(phi.values.size());
    int had = 0;
    throw_status(lsr_cuda_interface_one_step(c, LSR_FIELD_PHI, frozen.data(), &had));
    download(c, LSR_FIELD_PHI, phi);
    return frozen;
}

int reinit_iterate(ScalarField& phi, const BandMask& band, const std::vector<std::uint8_t>& frozen,
                   const ReinitConfig& cfg) {  // GPU (reinit.cpp:88-131)
    cfg.validate();
    if (!(phi.grid == band.grid)) throw ConfigError("reinit_iterate: grid mismatch");
    require_size(phi, "reinit_iterate");
    if (frozen.size() != phi.values.size()) throw ConfigError("reinit_iterate: frozen flags do not match the field");
    lsr_cuda_ctx* c = host_ctx(phi.grid);
    upload(c, LSR_FIELD_PHI, phi);
    upload_band(c, band);
    const lsr_reinit_cfg rc = to_c(cfg);
    int iters = 0;
    throw_status(lsr_cuda_reinit_iterate(c, LSR_FIELD_PHI, frozen.data(), &rc, &iters));
    download(c, LSR_FIELD_PHI, phi);
    return iters;
}

ReinitResult reinitialize(ScalarField& phi, const BandMask& band, double gamma, const ReinitConfig& cfg) {
    // GPU (reinit.cpp:133-145): one-step, iterate on the tube, clamp. With a
    // valid config the three run in one device pass; an invalid config goes
    // through the same sequence as the reference (the one-step has modified
    // phi when reinit_iterate's ConfigError propagates).
    require_size(phi, "reinitialize");
    const bool valid = cfg.dtau > 0.0 && cfg.max_iters >= 1;
    if (!valid || !(phi.grid == band.grid)) {
        ReinitResult res;
        try {
            const std::vector<std::uint8_t> frozen = interface_one_step(phi);
            res.had_interface = true;
            res.iterations = reinit_iterate(phi, band, frozen, cfg);
        } catch (const NoInterfaceError&) {
            res.had_interface = false;
        }
        clamp_field(phi, gamma);
        return res;
    }
    if (!(gamma > 0.0)) {  // the reference reaches clamp_field's check after the iterations
        ReinitResult res;
        try {
            const std::vector<std::uint8_t> frozen = interface_one_step(phi);
            res.had_interface = true;
            res.iterations = reinit_iterate(phi, band, frozen, cfg);
        } catch (const NoInterfaceError&) {
        }
        throw ConfigError("clamp_field: gamma must be positive");
    }
    lsr_cuda_ctx* c = host_ctx(phi.grid);
    upload(c, LSR_FIELD_PHI, phi);
    upload_band(c, band);
    const lsr_reinit_cfg rc = to_c(cfg);
    int iters = 0, had = 0;
    throw_status(lsr_cuda_reinitialize(c, LSR_FIELD_PHI, gamma, &rc, &iters, &had));
    download(c, LSR_FIELD_PHI, phi);
    ReinitResult res;
    res.had_interface = had != 0;
    res.iterations = iters;
    return res;
}

// ------------------------------------------------------------ lsr::cuda::Session

namespace cuda {

Session::Session(const Grid& grid, int device) : grid_(grid) {
    const lsr_grid cg = to_c(grid);
    throw_status(lsr_cuda_create(device, &cg, &ctx_));
}

Session::~Session() { lsr_cuda_destroy(ctx_); }

void Session::set_phi(const ScalarField& phi) {
    if (!(phi.grid == grid_)) throw ConfigError("session: grid mismatch");
    require_size(phi, "session");
    upload(ctx_, LSR_FIELD_PHI, phi);
}

void Session::set_distance(const DistanceField& dist) {
    if (!(dist.field.grid == grid_)) throw ConfigError("session: grid mismatch");
    require_size(dist.field, "session");
    upload(ctx_, LSR_FIELD_DIST, dist.field);
}

void Session::build_distance(const PointCloud& cloud) {
    if (cloud.points.empty()) throw Error("seed_exact_distance: empty cloud");
    const std::vector<double> xyz = triples(cloud);
    double sentinel = 0.0;
    int rounds = 0;
    throw_status(lsr_cuda_ctx_build_distance(ctx_, xyz.data(), cloud.size(), cloud.dim, 0, &sentinel, &rounds));
}

ScalarField Session::phi() const {
    ScalarField f(grid_);
    download(ctx_, LSR_FIELD_PHI, f);
    return f;
}

double Session::surface_energy(int p, int subcell_refine) const {
    double e = 0.0;
    throw_status(lsr_cuda_surface_energy(ctx_, LSR_FIELD_PHI, p, subcell_refine, &e));
    return e;
}

lsr_loop_stats Session::iterate(const StepConfig& step, const ReinitConfig& reinit, int energy_refine) {
    step.validate();
    const lsr_step_cfg sc = to_c(step);
    const lsr_reinit_cfg rc = to_c(reinit);
    lsr_loop_stats st{};
    throw_status(lsr_cuda_loop_step(ctx_, &sc, &rc, energy_refine, -1.0, &st));
    return st;
}

}  // namespace cuda

}  // namespace lsr
