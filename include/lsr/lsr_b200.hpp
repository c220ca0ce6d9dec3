// lsr_b200.hpp — the C++ `lsr::` face of the B200 path.
//
// One header that declares the whole public API of the reference headers it
// shadows (/root/reference/proj/include/lsr/{types,grid,interp,evolve,
// distance,cloud,reinit,metrics}.hpp): the same types with the same members,
// layouts and defaults, and the same function signatures, so the reference's
// own translation units compile against include/ unchanged and link with
// liblsr_b200.so. The forwarding headers include/lsr/*.hpp
// map each reference include path here; driver.hpp, io.hpp, reference.hpp
// and parallel.hpp are not shadowed (they come from the reference tree).
//
// Which definitions liblsr_b200.so provides (lsr_api.cpp), by the reference
// translation unit they replace:
//   evolve.cpp    sl_step (GPU), tangent_basis, scale_factor
//   grid.cpp      narrow_band, clamp_field (GPU); build_grid, locate_cell,
//                 default_band_params, centered_gradient, cutoff_weight
//                 (host scalar utilities, not on the per-node path)
//   distance.cpp  seed_exact_distance, fast_sweep, build_distance_field (GPU)
//   reinit.cpp    interface_one_step, reinit_iterate, reinitialize (GPU);
//                 ReinitConfig::defaults
// Everything else declared here (cloud.hpp's loaders and SpatialHash,
// interp.hpp's point interpolants, metrics.hpp) is defined by the
// reference's own cloud.cpp / interp.cpp / metrics.cpp, which a program
// links next to liblsr_b200.so. The device-resident loop, the GPU E_2 and
// the multi-GPU entries are in the C ABI (lsr_cuda.h) and lsr::cuda below.
//
//   reference (proj/include/lsr/)          here
//   types.hpp:12-61     Vec, Index3, Error hierarchy, dot/norm/sqr
//   grid.hpp:10-107     Grid, build_grid, locate_cell, ScalarField, NodeState,
//                       BandMask, BandParams, default_band_params,
//                       centered_gradient, narrow_band, clamp_field, cutoff_weight
//   cloud.hpp:11-85     PointCloud, CloudStats, ShapeKind, ShapeSpec, CloudFormat,
//                       loaders, estimate_resolution, compute_stats,
//                       sample_shape, exact_sdf, bounding_box, SpatialHash
//   interp.hpp:9-38     InterpolatorKind, Stencil4, WenoWeights, weno_*, interp*
//   distance.hpp:14-29  DistanceField, seed_exact_distance, fast_sweep,
//                       build_distance_field
//   evolve.hpp:11-43    TangentBasis, StepConfig, tangent_basis, scale_factor, sl_step
//   reinit.hpp:9-44     ReinitConfig, interface_one_step, reinit_iterate,
//                       ReinitResult, reinitialize
//   metrics.hpp:12-62   EnergyHistory, MetricsRecord, interface_cells, energy_2d,
//                       energy_3d, surface_energy, err_on_cloud, l1_update,
//                       l1_error_vs_exact, delta_energy, StopDecision, stopping_check
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "lsr_cuda.h"

namespace lsr {

// ---------------------------------------------------------------- types.hpp

struct Vec {  // fixed 3-vector; 2d data keeps z = 0
    double data[3];
    double& operator[](int i) { return data[i]; }
    double operator[](int i) const { return data[i]; }
    bool operator==(const Vec& o) const { return data[0] == o.data[0] && data[1] == o.data[1] && data[2] == o.data[2]; }
};
using Index3 = std::array<int, 3>;

// one class per C-ABI status code (lsr_cuda.h)
class Error : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
class ParseError : public Error {
  public:
    using Error::Error;
};
class ConfigError : public Error {
  public:
    using Error::Error;
};
class OutOfDomainError : public Error {
  public:
    using Error::Error;
};
class NumericalError : public Error {
  public:
    using Error::Error;
};
class NoInterfaceError : public Error {
  public:
    using Error::Error;
};
class CudaError : public Error {  // device / runtime failure (no reference analogue)
  public:
    using Error::Error;
};

inline Vec operator+(const Vec& a, const Vec& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline Vec operator-(const Vec& a, const Vec& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline Vec operator*(double s, const Vec& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline double dot(const Vec& a, const Vec& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double norm(const Vec& a) { return std::sqrt(dot(a, a)); }
inline double sqr(double x) { return x * x; }

// ----------------------------------------------------------------- grid.hpp

struct Grid {  // nodes x fastest: id = (k * ny + j) * nx + i
    int dim = 2;
    Vec origin{0, 0, 0};
    double dx = 1.0;
    Index3 dims{1, 1, 1};  // dims[2] == 1 in 2d

    std::int64_t num_nodes() const { return static_cast<std::int64_t>(dims[0]) * dims[1] * dims[2]; }
    std::int64_t index(int i, int j, int k) const { return (static_cast<std::int64_t>(k) * dims[1] + j) * dims[0] + i; }
    Index3 unflatten(std::int64_t id) const {
        const std::int64_t row = id / dims[0];
        return {static_cast<int>(id - row * dims[0]), static_cast<int>(row % dims[1]),
                static_cast<int>(id / (static_cast<std::int64_t>(dims[0]) * dims[1]))};
    }
    Vec node(int i, int j, int k) const { return {origin[0] + i * dx, origin[1] + j * dx, origin[2] + k * dx}; }
    Vec upper() const {
        return {origin[0] + (dims[0] - 1) * dx, origin[1] + (dims[1] - 1) * dx, origin[2] + (dims[2] - 1) * dx};
    }
    double diagonal() const { return norm(upper() - origin); }
    bool contains(const Vec& p) const {  // inside the hull [origin, upper] in the used axes
        const Vec hi = upper();
        for (int d = 0; d < dim; ++d)
            if (p[d] < origin[d] || p[d] > hi[d]) return false;
        return true;
    }
    Vec clamp_to_hull(const Vec& p) const {  // componentwise onto the hull; z := 0 in 2d
        const Vec hi = upper();
        Vec q = p;
        for (int d = 0; d < dim; ++d) q[d] = std::min(std::max(q[d], origin[d]), hi[d]);
        if (dim == 2) q[2] = 0.0;
        return q;
    }
    bool operator==(const Grid& o) const { return dim == o.dim && origin == o.origin && dx == o.dx && dims == o.dims; }
};

inline constexpr std::int64_t kDefaultNodeBudget = std::int64_t{1} << 28;

Grid build_grid(const Vec& bbox_min, const Vec& bbox_max, int dim, double dx, int pad_cells,
                std::int64_t node_budget = kDefaultNodeBudget);

// lower corner of the cell holding p (upper-hull points -> last cell);
// OutOfDomainError outside the hull
Index3 locate_cell(const Grid& g, const Vec& p);

struct ScalarField {
    Grid grid;
    std::vector<double> values;

    ScalarField() = default;
    explicit ScalarField(const Grid& g, double init = 0.0) : grid(g), values(static_cast<std::size_t>(g.num_nodes()), init) {}
    double& at(int i, int j, int k) { return values[static_cast<std::size_t>(grid.index(i, j, k))]; }
    double at(int i, int j, int k) const { return values[static_cast<std::size_t>(grid.index(i, j, k))]; }
};

enum class NodeState : unsigned char { Inactive = 0, Active = 1, ReinitHalo = 2 };

struct BandMask {
    Grid grid;
    std::vector<NodeState> state;
    std::vector<std::int64_t> active;  // ACTIVE ids, ascending
    std::vector<std::int64_t> tube;    // ACTIVE + REINIT_HALO ids, ascending
};

struct BandParams {
    double gamma = 0.0;  // band half-width
    double beta = 0.0;   // cutoff inner radius
    void validate() const {
        if (!(beta > 0.0) || !(beta < gamma)) throw ConfigError("band: need 0 < beta < gamma");
    }
};

BandParams default_band_params(int dim, double dx);            // (4dx, 2dx) in 2d, (6dx, 3dx) in 3d
Vec centered_gradient(const ScalarField& f, int i, int j, int k);  // one-sided at the hull
BandMask narrow_band(const ScalarField& phi, double gamma);     // GPU
void clamp_field(ScalarField& f, double gamma);                 // GPU
double cutoff_weight(double phi, const BandParams& params);

// ---------------------------------------------------------------- cloud.hpp

struct PointCloud {
    int dim = 0;  // 2 or 3
    std::vector<Vec> points;
    std::string source_id;
    std::int64_t size() const { return static_cast<std::int64_t>(points.size()); }
};

struct CloudStats {
    double h_s = 0.0;      // estimated cloud resolution
    double gamma_s = 0.0;  // k_s * h_s
    double k_s = 2.0;
    Vec bbox_min{0, 0, 0};
    Vec bbox_max{0, 0, 0};
    std::uint64_t sample_seed = 0;
};

enum class ShapeKind { Circle, Square45, Sphere, CubeSpheres };

struct ShapeSpec {
    ShapeKind kind = ShapeKind::Circle;
    double size = 1.0;
    Vec center{0, 0, 0};
    int n_points = 64;
    int dim() const { return (kind == ShapeKind::Circle || kind == ShapeKind::Square45) ? 2 : 3; }
    void validate() const;
};

enum class CloudFormat { Xyz, Ply };

PointCloud load_cloud(const std::string& path, CloudFormat format);
void write_cloud_xyz(const PointCloud& cloud, const std::string& path);
double estimate_resolution(const PointCloud& cloud, double sample_fraction, std::uint64_t seed);
CloudStats compute_stats(const PointCloud& cloud, double sample_fraction, double k_s, std::uint64_t seed);
PointCloud sample_shape(const ShapeSpec& spec, std::uint64_t seed);
double exact_sdf(const ShapeSpec& spec, const Vec& point);
void bounding_box(const PointCloud& cloud, Vec& lo, Vec& hi);

class SpatialHash {  // uniform bins, exact nearest-neighbour queries
  public:
    explicit SpatialHash(const PointCloud& cloud);
    double nearest_distance(const Vec& q, std::int64_t exclude = -1) const;

  private:
    const PointCloud* cloud_;
    int dim_;
    Vec lo_{0, 0, 0};
    double cell_ = 1.0;
    Index3 bins_{1, 1, 1};
    std::vector<std::int32_t> starts_;
    std::vector<std::int32_t> entries_;
    std::int64_t bin_index(int bx, int by, int bz) const {
        return (static_cast<std::int64_t>(bz) * bins_[1] + by) * bins_[0] + bx;
    }
};

// --------------------------------------------------------------- interp.hpp

enum class InterpolatorKind { Q1, Weno };

struct Stencil4 {  // (v_{j-1}, v_j, v_{j+1}, v_{j+2}), theta = (x - x_j)/dx
    std::array<double, 4> v{};
    double dx = 1.0;
    double theta = 0.0;
};

struct WenoWeights {
    double left = 0.0;
    double right = 0.0;
};
WenoWeights weno_linear_weights(double theta);
WenoWeights weno_indicators(const Stencil4& st);
double weno_1d(const Stencil4& st);
double interp_q1(const ScalarField& f, const Vec& p);
double interp_weno(const ScalarField& f, const Vec& p);
double interp(InterpolatorKind kind, const ScalarField& f, const Vec& p);

// ------------------------------------------------------------- distance.hpp

struct DistanceField {
    ScalarField field;
    std::vector<std::uint8_t> exact;  // 1 where the value is the exact cloud distance
    double sentinel = 0.0;
};

DistanceField seed_exact_distance(const Grid& grid, const PointCloud& cloud);  // GPU
int fast_sweep(DistanceField& d);                                            // GPU
DistanceField build_distance_field(const Grid& grid, const PointCloud& cloud);  // GPU

// --------------------------------------------------------------- evolve.hpp

struct TangentBasis {
    Vec v1{0, 0, 0};
    Vec v2{0, 0, 0};
};

struct StepConfig {
    int p = 1;
    double delta = 0.0;
    double dt = 0.0;
    InterpolatorKind interp = InterpolatorKind::Weno;
    double fallback_c = 1e-3;
    double fallback_alpha = 1.0;
    BandParams band{};

    void validate() const {
        if (p != 1 && p != 2) throw ConfigError("step: p must be 1 or 2");
        if (!(dt > 0.0)) throw ConfigError("step: dt must be positive");
        if (delta < 0.0 || delta > 1.0) throw ConfigError("step: delta must be in [0, 1]");
        band.validate();
    }
};

TangentBasis tangent_basis(int dim, const Vec& grad);
double scale_factor(double d_j, double energy_p, int p);

// One semi-Lagrangian step on the ACTIVE nodes (GPU); every other node of
// `out` equals phi; a non-finite update throws NumericalError naming the
// smallest such node after `out` is fully written.
void sl_step(const ScalarField& phi, const DistanceField& dist, const BandMask& mask, const StepConfig& cfg,
             double energy_p, ScalarField& out);

// --------------------------------------------------------------- reinit.hpp

struct ReinitConfig {
    double dtau = 0.0;
    int max_iters = 0;
    double residual_tol = 1e-3;
    double sign_eps = 0.0;

    static ReinitConfig defaults(double dx, double gamma);  // dx/2, 4 ceil(gamma/dx), 1e-3, dx
    void validate() const {
        if (!(dtau > 0.0)) throw ConfigError("reinit: dtau must be positive");
        if (max_iters < 1) throw ConfigError("reinit: max_iters must be >= 1");
    }
};

std::vector<std::uint8_t> interface_one_step(ScalarField& phi);  // GPU
int reinit_iterate(ScalarField& phi, const BandMask& band, const std::vector<std::uint8_t>& frozen,
                   const ReinitConfig& cfg);  // GPU

struct ReinitResult {
    bool had_interface = false;
    int iterations = 0;
};

ReinitResult reinitialize(ScalarField& phi, const BandMask& band, double gamma, const ReinitConfig& cfg);  // GPU

// -------------------------------------------------------------- metrics.hpp

struct EnergyHistory {
    std::vector<double> values;
    int k_window = 10;
};

struct MetricsRecord {
    int iter = 0;
    double e2 = 0.0;
    double delta_e = 0.0;
    double err_cloud = 0.0;
    double l1_update = 0.0;
    std::optional<double> l1_error;
    double wall_ms = 0.0;
};

std::vector<std::int64_t> interface_cells(const ScalarField& phi);
double energy_2d(const ScalarField& phi, const DistanceField& dist, int p);
double energy_3d(const ScalarField& phi, const DistanceField& dist, int p, int subcell_refine);
double surface_energy(const ScalarField& phi, const DistanceField& dist, int p, int subcell_refine = 5);
double err_on_cloud(const ScalarField& phi, const PointCloud& cloud, InterpolatorKind kind);
double l1_update(const ScalarField& prev, const ScalarField& next, const BandMask& band);
double l1_error_vs_exact(const ScalarField& phi, const ShapeSpec& spec, const BandMask& band);
double delta_energy(const EnergyHistory& hist, int n);

enum class StopDecision { Continue, Stop };

StopDecision stopping_check(const EnergyHistory& hist, int n, int min_iters, int max_iters, double tol);

// ------------------------------------------------------ B200 extensions

// Throws the exception class matching a C-ABI status (no-op on LSR_OK).
void throw_status(int status);

// C-ABI views of the host types
inline lsr_grid to_c(const Grid& g) {
    lsr_grid c{};
    c.dim = g.dim;
    c.dx = g.dx;
    for (int d = 0; d < 3; ++d) {
        c.dims[d] = g.dims[d];
        c.origin[d] = g.origin[d];
    }
    return c;
}
inline lsr_step_cfg to_c(const StepConfig& s) {
    lsr_step_cfg c{};
    c.p = s.p;
    c.interp = s.interp == InterpolatorKind::Q1 ? LSR_INTERP_Q1 : LSR_INTERP_WENO;
    c.delta = s.delta;
    c.dt = s.dt;
    c.fallback_c = s.fallback_c;
    c.fallback_alpha = s.fallback_alpha;
    c.gamma = s.band.gamma;
    c.beta = s.band.beta;
    return c;
}
inline lsr_reinit_cfg to_c(const ReinitConfig& r) { return lsr_reinit_cfg{r.dtau, r.max_iters, r.residual_tol, r.sign_eps}; }

namespace cuda {

// The device-resident driver loop (driver.cpp:185-203 on a fixed grid): phi,
// d and the band stay in HBM; one iteration = narrow_band, E_2 (GPU),
// sl_step, reinitialize, swap. Host traffic per iteration: the statistics.
class Session {
  public:
    Session(const Grid& grid, int device = 0);
    ~Session();
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    void set_phi(const ScalarField& phi);
    void set_distance(const DistanceField& dist);
    void build_distance(const PointCloud& cloud);  // build_distance_field on the device
    ScalarField phi() const;
    double surface_energy(int p = 2, int subcell_refine = 5) const;
    lsr_loop_stats iterate(const StepConfig& step, const ReinitConfig& reinit, int energy_refine = 5);
    lsr_cuda_ctx* handle() const { return ctx_; }

  private:
    Grid grid_;
    lsr_cuda_ctx* ctx_ = nullptr;
};

}  // namespace cuda

}  // namespace lsr
