// workloads.cpp — seeded synthetic clouds for the five BASELINE configs
// (include/lsr_workloads.h). Host-only input generation; not on the hot path.
#include <cmath>
#include <random>
#include <vector>

#include "lsr_workloads.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

struct Rng {
    std::mt19937_64 g;
    explicit Rng(uint64_t seed) : g(seed) {}
    double u() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }  // [0, 1)
    double normal() {                                                  // Box-Muller
        const double u1 = 1.0 - u();                                   // (0, 1]
        const double u2 = u();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    }
};

// uniform direction on the unit sphere: z = 2u - 1, phi = 2 pi u'
void unit_dir(Rng& r, double* d) {
    const double z = 2.0 * r.u() - 1.0;
    const double ph = 2.0 * kPi * r.u();
    const double s = std::sqrt(std::max(0.0, 1.0 - z * z));
    d[0] = s * std::cos(ph);
    d[1] = s * std::sin(ph);
    d[2] = z;
}

// distance from p to the core circle of a z-axis torus of radius R at (cx, 0, 0)
double torus_core_dist(const double* p, double cx, double R) {
    const double x = p[0] - cx, y = p[1];
    const double rho = std::sqrt(x * x + y * y);
    return std::sqrt((rho - R) * (rho - R) + p[2] * p[2]);
}

}  // namespace

extern "C" int lsr_cloud_generate(int config, int64_t n, uint64_t seed, double sigma, double* pts) {
    Rng r(seed);
    switch (config) {
        case LSR_CLOUD_CIRCLE:
            for (int64_t i = 0; i < n; ++i) {
                const double th = 2.0 * kPi * r.u();
                pts[3 * i] = 0.3 * std::cos(th);
                pts[3 * i + 1] = 0.3 * std::sin(th);
                pts[3 * i + 2] = 0.0;
            }
            return 0;
        case LSR_CLOUD_SPHERE:
            for (int64_t i = 0; i < n; ++i) {
                double d[3];
                unit_dir(r, d);
                for (int c = 0; c < 3; ++c) pts[3 * i + c] = 0.5 * d[c];
            }
            return 0;
        case LSR_CLOUD_TORUS:
            for (int64_t i = 0; i < n; ++i) {
                const double u = 2.0 * kPi * r.u(), v = 2.0 * kPi * r.u();
                const double R = 0.5, rr = 0.2;
                pts[3 * i] = (R + rr * std::cos(v)) * std::cos(u) + sigma * r.normal();
                pts[3 * i + 1] = (R + rr * std::cos(v)) * std::sin(u) + sigma * r.normal();
                pts[3 * i + 2] = rr * std::sin(v) + sigma * r.normal();
            }
            return 0;
        case LSR_CLOUD_BUMPY: {
            // uniform directions accepted with probability (1 + 9|cos t|)/10:
            // the surface density is 10x higher at the poles than at the equator
            int64_t i = 0;
            while (i < n) {
                double d[3];
                unit_dir(r, d);
                if (r.u() * 10.0 >= 1.0 + 9.0 * std::fabs(d[2])) continue;
                const double t = std::acos(std::max(-1.0, std::min(1.0, d[2])));
                const double ph = std::atan2(d[1], d[0]);
                const double rad = 0.5 * (1.0 + 0.1 * std::sin(5.0 * t) * std::cos(4.0 * ph));
                for (int c = 0; c < 3; ++c) pts[3 * i + c] = rad * d[c];
                ++i;
            }
            return 0;
        }
        case LSR_CLOUD_THREE_TORI: {
            const double R = 0.3, rr = 0.1, cx[3] = {-0.5, 0.0, 0.5};
            double cap[2][3];
            int ncap = 0;
            int64_t i = 0;
            while (i < n) {
                const int t = static_cast<int>(r.u() * 3.0);  // equal areas: pick a torus uniformly
                const double u = 2.0 * kPi * r.u(), v = 2.0 * kPi * r.u();
                if (r.u() * (R + rr) >= R + rr * std::cos(v)) continue;  // area element (R + r cos v)
                double p[3] = {cx[t] + (R + rr * std::cos(v)) * std::cos(u), (R + rr * std::cos(v)) * std::sin(u),
                               rr * std::sin(v)};
                bool inside = false;  // union surface: drop points inside another torus
                for (int o = 0; o < 3 && !inside; ++o)
                    if (o != t && torus_core_dist(p, cx[o], R) < rr) inside = true;
                if (inside) continue;
                if (ncap < 2) {  // the first two surface samples seed the removed caps
                    for (int c = 0; c < 3; ++c) cap[ncap][c] = p[c];
                    ++ncap;
                    continue;
                }
                bool in_cap = false;
                for (int k = 0; k < 2; ++k) {
                    const double dx = p[0] - cap[k][0], dy = p[1] - cap[k][1], dz = p[2] - cap[k][2];
                    if (dx * dx + dy * dy + dz * dz < 0.1 * 0.1) in_cap = true;
                }
                if (in_cap) continue;
                for (int c = 0; c < 3; ++c) pts[3 * i + c] = p[c] + sigma * r.normal();
                ++i;
            }
            return 0;
        }
    }
    return -1;
}
