// lsr_b200.hpp — C++ host API of the B200 path, source-compatible with the
// reference's `lsr::` API for the semi-Lagrangian step (SPEC.md:263-411,
// /root/reference/proj/include/lsr/*.hpp). A program written against the
// reference's grid/evolve headers compiles against these types unchanged and
// its lsr::sl_step calls run on the GPU through the C ABI (lsr_cuda.h).
//
//   reference                           here
//   types.hpp:12-61  Vec, Error...      same names below
//   grid.hpp:10-52   Grid               Grid
//   grid.hpp:63-75   ScalarField        ScalarField
//   grid.hpp:77-84   NodeState/BandMask NodeState/BandMask
//   grid.hpp:86-96   BandParams         BandParams, default_band_params
//   distance.hpp:14  DistanceField      DistanceField
//   interp.hpp:9     InterpolatorKind   InterpolatorKind
//   evolve.hpp:16-31 StepConfig         StepConfig
//   evolve.hpp:42-43 sl_step            sl_step  (GPU)
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "lsr_cuda.h"

namespace lsr {

struct Vec {
    double data[3];
    double& operator[](int i) { return data[i]; }
    double operator[](int i) const { return data[i]; }
    bool operator==(const Vec& o) const { return data[0] == o.data[0] && data[1] == o.data[1] && data[2] == o.data[2]; }
};
using Index3 = std::array<int, 3>;

inline Vec operator+(const Vec& a, const Vec& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline Vec operator-(const Vec& a, const Vec& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline Vec operator*(double s, const Vec& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline double dot(const Vec& a, const Vec& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double norm(const Vec& a) { return std::sqrt(dot(a, a)); }
inline double sqr(double x) { return x * x; }

// exception hierarchy, one class per C-ABI status code
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct OutOfDomainError : Error {
    using Error::Error;
};
struct NumericalError : Error {
    using Error::Error;
};
struct NoInterfaceError : Error {
    using Error::Error;
};
struct CudaError : Error {  // device failure; no reference analogue
    using Error::Error;
};

struct Grid {
    int dim = 2;
    Vec origin{0, 0, 0};
    double dx = 1.0;
    Index3 dims{1, 1, 1};

    std::int64_t num_nodes() const { return std::int64_t{dims[0]} * dims[1] * dims[2]; }
    std::int64_t index(int i, int j, int k) const { return (std::int64_t{k} * dims[1] + j) * dims[0] + i; }
    Index3 unflatten(std::int64_t id) const {
        const std::int64_t row = id / dims[0];
        return {static_cast<int>(id - row * dims[0]), static_cast<int>(row % dims[1]),
                static_cast<int>(row / dims[1])};
    }
    Vec node(int i, int j, int k) const { return {origin[0] + i * dx, origin[1] + j * dx, origin[2] + k * dx}; }
    Vec upper() const {
        return {origin[0] + (dims[0] - 1) * dx, origin[1] + (dims[1] - 1) * dx, origin[2] + (dims[2] - 1) * dx};
    }
    double diagonal() const { return norm(upper() - origin); }
    bool operator==(const Grid& o) const {
        return dim == o.dim && origin == o.origin && dx == o.dx && dims == o.dims;
    }
    lsr_grid c() const {
        lsr_grid g{};
        g.dim = dim;
        g.dx = dx;
        for (int d = 0; d < 3; ++d) {
            g.dims[d] = dims[d];
            g.origin[d] = origin[d];
        }
        return g;
    }
};

struct ScalarField {
    Grid grid;
    std::vector<double> values;
    ScalarField() = default;
    explicit ScalarField(const Grid& g, double init = 0.0) : grid(g), values(static_cast<size_t>(g.num_nodes()), init) {}
    double& at(int i, int j, int k) { return values[static_cast<size_t>(grid.index(i, j, k))]; }
    double at(int i, int j, int k) const { return values[static_cast<size_t>(grid.index(i, j, k))]; }
};

enum class NodeState : unsigned char { Inactive = 0, Active = 1, ReinitHalo = 2 };

struct BandMask {
    Grid grid;
    std::vector<NodeState> state;
    std::vector<std::int64_t> active;  // ascending
    std::vector<std::int64_t> tube;    // ascending
};

struct BandParams {
    double gamma = 0.0;
    double beta = 0.0;
    void validate() const {
        if (!(beta > 0.0) || !(beta < gamma)) throw ConfigError("band: need 0 < beta < gamma");
    }
};

inline BandParams default_band_params(int dim, double dx) {
    if (dim == 2) return BandParams{4.0 * dx, 2.0 * dx};
    return BandParams{6.0 * dx, 3.0 * dx};
}

struct DistanceField {
    ScalarField field;
    std::vector<std::uint8_t> exact;
    double sentinel = 0.0;
};

enum class InterpolatorKind { Q1, Weno };

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
    lsr_step_cfg c() const {
        lsr_step_cfg s{};
        s.p = p;
        s.interp = interp == InterpolatorKind::Q1 ? LSR_INTERP_Q1 : LSR_INTERP_WENO;
        s.delta = delta;
        s.dt = dt;
        s.fallback_c = fallback_c;
        s.fallback_alpha = fallback_alpha;
        s.gamma = band.gamma;
        s.beta = band.beta;
        return s;
    }
};

// Throws the exception class matching a C-ABI status (no-op on LSR_OK).
void throw_status(int status);

// One semi-Lagrangian step on the ACTIVE nodes (GPU). Same contract as the
// reference: all other nodes copy phi; `out` is resized if needed; a
// non-finite update throws NumericalError naming the node after `out` has
// been fully written.
void sl_step(const ScalarField& phi, const DistanceField& dist, const BandMask& mask, const StepConfig& cfg,
             double energy_p, ScalarField& out);

}  // namespace lsr
