// energy.cu — the surface energy E_p = (integral of |d|^p over the front)^(1/p)
// of lsr::surface_energy (/root/reference/proj/src/metrics.cpp:186-189), the
// producer of sl_step's energy_p (driver.cpp:188) — SURVEY §8(f) row 3.
//
//  * interface_cells (metrics.cpp:35-56): every cell is classified in
//    parallel; an order-preserving compaction (cub::DeviceSelect::Flagged)
//    reproduces the ascending cell list of the serial scan.
//  * energy_3d (metrics.cpp:145-184): one thread per interface cell runs the
//    r^3 subcell midpoint rule in the reference's loop order; energy_2d
//    (:113-143): marching squares with the reference's case table, saddle
//    rule and trapezoid sums.
//  * blocked_sum (parallel.hpp:26-42): the 4096-term blocks are summed
//    serially in index order (one thread per block), the block partials in
//    block order on the host, then pow(total, 1/p) with the host libm — the
//    reference's exact summation order.
//  The per-term |d|^p uses |d|*|d| for p = 2 (correctly rounded) where the
//  reference calls glibc pow, which is not correctly rounded,
//  so E_p agrees to a few ulp rather than bit for bit.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <cstdlib>

#include "compact.cuh"

#include <cmath>
#include <mutex>
#include <cstdint>
#include <string>
#include <vector>

#include "lsr_cuda.h"
#include "prep_launch.h"
#include "sl_device.cuh"

using lsr_dev::SlParams;

namespace {

__device__ __forceinline__ double powp(double a, int p) {
    if (p == 1) return a;
    if (p == 2) return a * a;
    return pow(a, static_cast<double>(p));
}

// interface_cells' corner test (metrics.cpp:23-31, 40-52)
// cells [base, end); flags indexed by global cell id
// (only_if, the device loop: nothing is done when *only_if == 0)
__global__ void flag_cells(SlParams P, const double* __restrict__ phi, long long base, long long end,
                           unsigned char* __restrict__ flags, const int* __restrict__ only_if = nullptr) {
    if (only_if != nullptr && *only_if == 0) return;
    const long long c = base + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= end) return;
    const unsigned cx = P.nx - 1, cy = P.ny - 1;  // cells < 2^31 (cub's int item count)
    const unsigned row = static_cast<unsigned>(c) / cx;
    const int i = static_cast<int>(static_cast<unsigned>(c) - row * cx);
    const int k = static_cast<int>(row / cy);
    const int j = static_cast<int>(row - static_cast<unsigned>(k) * cy);
    const long long b = (static_cast<long long>(k) * P.ny + j) * P.nx + i;
    bool pos = false, neg = false, zero = false;
    const int kz = P.dim == 3 ? 1 : 0;
    for (int dk = 0; dk <= kz; ++dk)
        for (int dj = 0; dj <= 1; ++dj)
            for (int di = 0; di <= 1; ++di) {
                const double v = __ldg(phi + b + dk * P.nxy + dj * P.nx + di);
                if (v > 0.0) pos = true;
                else if (v < 0.0) neg = true;
                else zero = true;
            }
    flags[c] = (zero || (pos && neg)) ? 1 : 0;
}

// flag_cells for 3d grids with nx % 4 == 0: four consecutive cells of a row
// per thread; the 5 x 4 corner nodes are loaded once (16-byte loads) and
// classified once instead of 8 loads per cell
__device__ __forceinline__ unsigned sign_class(double v) {  // bit0 pos, bit1 neg, bit2 zero (or NaN)
    return v > 0.0 ? 1u : (v < 0.0 ? 2u : 4u);
}

__global__ void flag_cells4(SlParams P, const double* __restrict__ phi, unsigned tpr, long long nthreads,
                            unsigned char* __restrict__ flags) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nthreads) return;
    const unsigned cx = P.nx - 1, cy = P.ny - 1;
    const unsigned row = static_cast<unsigned>(t / tpr);  // cell row (j, k)
    const int i0 = 4 * static_cast<int>(t - static_cast<long long>(row) * tpr);
    const int k = static_cast<int>(row / cy), j = static_cast<int>(row - static_cast<unsigned>(k) * cy);
    unsigned cls[5] = {0, 0, 0, 0, 0};  // per corner column: OR of the 4 rows' classes
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const long long b = (static_cast<long long>(k + (r >> 1)) * P.ny + j + (r & 1)) * P.nx + i0;
        const double2 a = __ldg(reinterpret_cast<const double2*>(phi + b));
        const double2 c = __ldg(reinterpret_cast<const double2*>(phi + b) + 1);
        cls[0] |= sign_class(a.x);
        cls[1] |= sign_class(a.y);
        cls[2] |= sign_class(c.x);
        cls[3] |= sign_class(c.y);
        if (i0 + 4 < P.nx) cls[4] |= sign_class(__ldg(phi + b + 4));
    }
    const long long c0 = static_cast<long long>(row) * cx + i0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (i0 + q >= static_cast<int>(cx)) break;
        const unsigned m = cls[q] | cls[q + 1];
        flags[c0 + q] = ((m & 4u) || (m & 3u) == 3u) ? 1 : 0;  // zero corner, or both signs
    }
}

// flag_cells4 marching along z: a thread owns 4 cells of a cell row (i0..,
// j) for kMarchCells consecutive cell planes; the classes of node rows
// (j, k) and (j+1, k) carry over from the previous plane, so each plane
// loads two node rows instead of four
constexpr int kMarchCells = 16;

__device__ __forceinline__ void row_classes(const SlParams& P, const double* __restrict__ phi, long long b, int i0,
                                            unsigned* cls) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(phi + b));
    const double2 c = __ldg(reinterpret_cast<const double2*>(phi + b) + 1);
    cls[0] = sign_class(a.x);
    cls[1] = sign_class(a.y);
    cls[2] = sign_class(c.x);
    cls[3] = sign_class(c.y);
    cls[4] = i0 + 4 < P.nx ? sign_class(__ldg(phi + b + 4)) : 0u;
}

// cell planes [k_lo, k_hi) (whole grid: 0, nz - 1); flags indexed by global cell id
__global__ void flag_cells_march(SlParams P, const double* __restrict__ phi, unsigned tpr,
                                 unsigned char* __restrict__ flags, int k_lo, int k_hi,
                                 const int* __restrict__ only_if = nullptr) {
    if (only_if != nullptr && *only_if == 0) return;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int cx = P.nx - 1, cy = P.ny - 1;
    const long long rows = static_cast<long long>(tpr) * cy;  // (x-quad, j) pairs
    if (t >= rows * ((k_hi - k_lo + kMarchCells - 1) / kMarchCells)) return;
    const int kb = static_cast<int>(t / rows);
    const long long r = t - kb * rows;
    const int j = static_cast<int>(r / tpr), i0 = 4 * static_cast<int>(r - static_cast<long long>(j) * tpr);
    const int k0 = k_lo + kb * kMarchCells, k1 = min(k_hi, k0 + kMarchCells);
    unsigned lo[5], lo1[5];  // classes of node rows (j, k) and (j+1, k)
    long long b = (static_cast<long long>(k0) * P.ny + j) * P.nx + i0;
    row_classes(P, phi, b, i0, lo);
    row_classes(P, phi, b + P.nx, i0, lo1);
    for (int k = k0; k < k1; ++k, b += P.nxy) {
        unsigned up[5], up1[5];
        row_classes(P, phi, b + P.nxy, i0, up);
        row_classes(P, phi, b + P.nxy + P.nx, i0, up1);
        const long long c0 = (static_cast<long long>(k) * cy + j) * cx + i0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (i0 + q >= cx) break;
            const unsigned m = lo[q] | lo[q + 1] | lo1[q] | lo1[q + 1] | up[q] | up[q + 1] | up1[q] | up1[q + 1];
            flags[c0 + q] = ((m & 4u) || (m & 3u) == 3u) ? 1 : 0;  // zero corner, or both signs
        }
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            lo[q] = up[q];
            lo1[q] = up1[q];
        }
    }
}

// The interface cells from the band's tube (the device loop, when phi has no
// hard jump: every axis pair of opposite signs then has an ACTIVE node, see
// band_reinit.cu OneStepGate). A cell with a zero corner, or with corners of
// both signs — hence an edge path between them, hence an opposite-sign edge
// or a zero corner on it — has an ACTIVE corner (|0| < gamma), and its base
// corner, at most one node below that corner on every axis, is in the tube
// (the ACTIVE set dilated by one, grid.cpp:98-116). So the tube entries whose
// node is a cell's base corner cover every interface cell, in ascending cell
// order (cell ids are monotone in base-node ids). tflags[t] = the corner test
// (metrics.cpp:23-31, 40-52) of the cell based at tube[t]; runs only when
// *hard == 0 (else the dense kernels above run).
__global__ void flag_cells_tube(SlParams P, const double* __restrict__ phi, const long long* __restrict__ tube,
                                const long long* __restrict__ n_dev, unsigned char* __restrict__ tflags,
                                const int* __restrict__ hard) {
    if (*hard != 0) return;
    const long long n = __ldg(n_dev);
    constexpr int kB = 1;  // entries per thread and round (2 measured slower)
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x * kB;
    const int kz = P.dim == 3 ? 1 : 0;
    for (long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x * kB; t0 < n; t0 += T) {
        long long id[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const long long t = t0 + u * blockDim.x + threadIdx.x;
            id[u] = t < n ? __ldg(tube + t) : -1;
        }
        double v[kB][8];
        bool cell[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            cell[u] = false;
            if (id[u] < 0) continue;
            int i, j, k;
            lsr_dev::unflatten(P, id[u], i, j, k);
            cell[u] = i < P.nx - 1 && j < P.ny - 1 && (P.dim != 3 || k < P.nz - 1);
            if (!cell[u]) continue;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int dk = (q >> 2) & kz;  // 2d: the four corners twice
                v[u][q] = __ldg(phi + id[u] + dk * P.nxy + ((q >> 1) & 1) * P.nx + (q & 1));
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            if (id[u] < 0) continue;
            unsigned m = 0;
            if (cell[u]) {
#pragma unroll
                for (int q = 0; q < 8; ++q) m |= sign_class(v[u][q]);
            }
            tflags[t0 + u * blockDim.x + threadIdx.x] = ((m & 4u) || (m & 3u) == 3u) ? 1 : 0;  // zero corner, or both signs
        }
    }
}

struct TubeCellId {  // the cell whose base corner is the node tube[t]
    const long long* tube;
    int nx, ny, dim;
    __device__ int operator()(long long t) const {
        const long long id = tube[t];
        const long long row = id / nx;
        const int i = static_cast<int>(id - row * nx);
        const long long k = dim == 3 ? row / ny : 0;
        const int j = static_cast<int>(row - k * ny);
        return static_cast<int>((k * (ny - 1) + j) * (nx - 1) + i);
    }
};

__global__ void add_counts(long long* __restrict__ nc) { nc[0] = nc[1] + nc[2]; }

// energy_3d per-cell contribution (metrics.cpp:161-178)
__global__ void contrib_3d(SlParams P, const double* __restrict__ phi, const double* __restrict__ dist,
                           const int* __restrict__ cells, long long nc, int r, double dxp, double select, int p,
                           double* __restrict__ contrib) {
    const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const long long cid = cells[c];
    const unsigned cx = P.nx - 1, cy = P.ny - 1;
    const unsigned row = static_cast<unsigned>(cid) / cx;
    const int i = static_cast<int>(static_cast<unsigned>(cid) - row * cx);
    const int k = static_cast<int>(row / cy);
    const int j = static_cast<int>(row - static_cast<unsigned>(k) * cy);
    const double bx = P.ox + i * P.dx, by = P.oy + j * P.dx, bz = P.oz + k * P.dx;  // Grid::node
    double acc = 0.0;
    for (int ck = 0; ck < r; ++ck)
        for (int cj = 0; cj < r; ++cj)
            for (int ci = 0; ci < r; ++ci) {
                const double x = bx + (ci + 0.5) * dxp, y = by + (cj + 0.5) * dxp, z = bz + (ck + 0.5) * dxp;
                if (fabs(lsr_dev::interp_q1<3>(P, phi, x, y, z)) >= select) continue;
                acc += powp(fabs(lsr_dev::interp_q1<3>(P, dist, x, y, z)), p) * dxp * dxp;
            }
    contrib[c] = acc;
}

// contrib_3d with the per-axis work hoisted (refinement r <= 8): a sample's
// x depends on ci only, so its cell and theta along x (locate_cell and the
// Markstein theta, interp.cpp:63-69) are computed once per ci, likewise y and
// z; the products wx*wy once per (ci, cj); the cell's 8 corner values of phi
// and d are loaded once and used whenever a sample locates in the cell
// itself (else its own corners are loaded). Every interpolant is the same
// expression as interp_q1's, so the result is bit-identical.
constexpr int kMaxRefine = 8;
constexpr int kEnergyMaxDevices = 64;

__device__ __forceinline__ double q1_corners(double w00, double w10, double w01, double w11, double uz, double tz,
                                             const double* f) {
    double value = 0.0;  // loop order dk, dj, di (interp.cpp:71-79); w = (wx*wy)*wz
    value += (w00 * uz) * f[0];
    value += (w10 * uz) * f[1];
    value += (w01 * uz) * f[2];
    value += (w11 * uz) * f[3];
    value += (w00 * tz) * f[4];
    value += (w10 * tz) * f[5];
    value += (w01 * tz) * f[6];
    value += (w11 * tz) * f[7];
    return value;
}

__device__ __forceinline__ void load_corners(const SlParams& P, const double* __restrict__ f, long long b, double* v) {
    v[0] = __ldg(f + b);
    v[1] = __ldg(f + b + 1);
    v[2] = __ldg(f + b + P.nx);
    v[3] = __ldg(f + b + P.nx + 1);
    v[4] = __ldg(f + b + P.nxy);
    v[5] = __ldg(f + b + P.nxy + 1);
    v[6] = __ldg(f + b + P.nxy + P.nx);
    v[7] = __ldg(f + b + P.nxy + P.nx + 1);
}

#ifndef LSR_EN_THREADS
#define LSR_EN_THREADS 128
#endif
#ifndef LSR_EN_MINB
#define LSR_EN_MINB 8  // 64 registers, 8 CTAs of 128 per SM (E_2 at 512^3: 1.06 -> 0.97 ms)
#endif
template <bool kDev>
__global__ void __launch_bounds__(LSR_EN_THREADS, LSR_EN_MINB) contrib_3d_hoisted(SlParams P, const double* __restrict__ phi, const double* __restrict__ dist,
                                   const int* __restrict__ cells, long long nc, int r, double dxp, double select,
                                   int p, double* __restrict__ contrib, const long long* __restrict__ nc_dev) {
    // kDev (the device loop): the cell count in device memory, grid-strided
    const long long n_ = kDev ? __ldg(nc_dev) : nc;
    for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < n_;
         c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long cid = cells[c];
    const unsigned cx = P.nx - 1, cy = P.ny - 1;
    const unsigned row = static_cast<unsigned>(cid) / cx;
    const int i = static_cast<int>(static_cast<unsigned>(cid) - row * cx);
    const int k = static_cast<int>(row / cy);
    const int j = static_cast<int>(row - static_cast<unsigned>(k) * cy);
    const double bx = P.ox + i * P.dx, by = P.oy + j * P.dx, bz = P.oz + k * P.dx;  // Grid::node
    int lx[kMaxRefine], ly[kMaxRefine], lz[kMaxRefine];
    double tx[kMaxRefine], ty[kMaxRefine], tz[kMaxRefine];
    for (int q = 0; q < r; ++q) {
        const double x = bx + (q + 0.5) * dxp, y = by + (q + 0.5) * dxp, z = bz + (q + 0.5) * dxp;
        lx[q] = lsr_dev::locate_axis(P, x, P.ox, P.nx);
        ly[q] = lsr_dev::locate_axis(P, y, P.oy, P.ny);
        lz[q] = lsr_dev::locate_axis(P, z, P.oz, P.nz);
        tx[q] = lsr_dev::axis_theta(P, x, P.ox, lx[q]);
        ty[q] = lsr_dev::axis_theta(P, y, P.oy, ly[q]);
        tz[q] = lsr_dev::axis_theta(P, z, P.oz, lz[q]);
    }
    const long long home = (static_cast<long long>(k) * P.ny + j) * P.nx + i;
    double fp[8], fd[8];
    load_corners(P, phi, home, fp);
    load_corners(P, dist, home, fd);
    double acc = 0.0;
    for (int ck = 0; ck < r; ++ck)
        for (int cj = 0; cj < r; ++cj)
            for (int ci = 0; ci < r; ++ci) {
                const double ux = 1.0 - tx[ci], uy = 1.0 - ty[cj], uz = 1.0 - tz[ck];
                const double w00 = ux * uy, w10 = tx[ci] * uy, w01 = ux * ty[cj], w11 = tx[ci] * ty[cj];
                const bool at_home = lx[ci] == i && ly[cj] == j && lz[ck] == k;
                double gp[8], gd[8];
                const long long b = (static_cast<long long>(lz[ck]) * P.ny + ly[cj]) * P.nx + lx[ci];
                if (!at_home) load_corners(P, phi, b, gp);
                const double vphi = q1_corners(w00, w10, w01, w11, uz, tz[ck], at_home ? fp : gp);
                if (fabs(vphi) >= select) continue;
                if (!at_home) load_corners(P, dist, b, gd);
                const double vd = q1_corners(w00, w10, w01, w11, uz, tz[ck], at_home ? fd : gd);
                acc += powp(fabs(vd), p) * dxp * dxp;
            }
    contrib[c] = acc;
    if (!kDev) break;
    }
}

struct Pt {
    double x, y;
};

// edge_crossing (metrics.cpp:65-77)
__device__ __forceinline__ Pt edge_crossing(const SlParams& P, const double* __restrict__ phi, int i, int j, int e) {
    const double x0 = P.ox + i * P.dx, y0 = P.oy + j * P.dx;
    const long long b = static_cast<long long>(j) * P.nx + i;
    auto lerp_t = [](double a, double c) { return a / (a - c); };
    switch (e) {
        case 0: return {x0 + lerp_t(__ldg(phi + b), __ldg(phi + b + 1)) * P.dx, y0};
        case 1: return {x0 + P.dx, y0 + lerp_t(__ldg(phi + b + 1), __ldg(phi + b + P.nx + 1)) * P.dx};
        case 2: return {x0 + lerp_t(__ldg(phi + b + P.nx), __ldg(phi + b + P.nx + 1)) * P.dx, y0 + P.dx};
        default: return {x0, y0 + lerp_t(__ldg(phi + b), __ldg(phi + b + P.nx)) * P.dx};
    }
}

__device__ __forceinline__ bool inside_hull(const SlParams& P, Pt a) {  // Grid::contains (grid.hpp:36-41)
    return !(a.x < P.ox || a.x > P.hx || a.y < P.oy || a.y > P.hy);
}

// energy_2d per-cell contribution (metrics.cpp:124-137, front_segments_2d :79-109)
template <bool kDev>
__global__ void contrib_2d(SlParams P, const double* __restrict__ phi, const double* __restrict__ dist,
                           const int* __restrict__ cells, long long nc, int p, double* __restrict__ contrib,
                           int* __restrict__ out_of_domain, const long long* __restrict__ nc_dev) {
    const long long n_ = kDev ? __ldg(nc_dev) : nc;
    for (long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; c < n_;
         c += static_cast<long long>(gridDim.x) * blockDim.x) {
    // segment table of the 16 corner cases (metrics.cpp:80-84)
    const signed char table[16][2] = {{-1, -1}, {3, 0}, {0, 1}, {3, 1}, {1, 2}, {-2, 0}, {0, 2}, {3, 2},
                                      {2, 3},   {0, 2}, {-2, 0}, {1, 2}, {1, 3}, {0, 1}, {3, 0}, {-1, -1}};
    const int cid = cells[c];
    const int i = cid % (P.nx - 1), j = cid / (P.nx - 1);
    const long long b = static_cast<long long>(j) * P.nx + i;
    const double f00 = __ldg(phi + b), f10 = __ldg(phi + b + 1), f11 = __ldg(phi + b + P.nx + 1),
                 f01 = __ldg(phi + b + P.nx);
    int cs = 0;  // cell_case_2d (metrics.cpp:14-21)
    if (f00 <= 0.0) cs |= 1;
    if (f10 <= 0.0) cs |= 2;
    if (f11 <= 0.0) cs |= 4;
    if (f01 <= 0.0) cs |= 8;
    int e[4];
    int ns = 0;
    if (table[cs][0] == -1) {
        ns = 0;
    } else if (table[cs][0] == -2) {
        const double avg = 0.25 * (f00 + f10 + f11 + f01);
        const bool center_inside = avg <= 0.0;
        const bool first = (cs == 5) ? center_inside : !center_inside;
        if (first) { e[0] = 0; e[1] = 1; e[2] = 2; e[3] = 3; }
        else { e[0] = 3; e[1] = 0; e[2] = 1; e[3] = 2; }
        ns = 2;
    } else {
        e[0] = table[cs][0];
        e[1] = table[cs][1];
        ns = 1;
    }
    double acc = 0.0;
    for (int s = 0; s < ns; ++s) {
        const Pt a = edge_crossing(P, phi, i, j, e[2 * s]);
        const Pt bb = edge_crossing(P, phi, i, j, e[2 * s + 1]);
        const double ddx = bb.x - a.x, ddy = bb.y - a.y, ddz = 0.0 - 0.0;
        const double len = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);  // norm(b - a)
        if (!inside_hull(P, a) || !inside_hull(P, bb)) {  // interp_q1 -> locate_cell throws (grid.cpp:40)
            atomicExch(out_of_domain, 1);
            continue;
        }
        const double da = lsr_dev::interp_q1<2>(P, dist, a.x, a.y, 0.0);
        const double db = lsr_dev::interp_q1<2>(P, dist, bb.x, bb.y, 0.0);
        acc += len * 0.5 * (powp(fabs(da), p) + powp(fabs(db), p));
    }
    contrib[c] = acc;
    if (!kDev) break;
    }
}

// blocked_sum's in-block serial sums (parallel.hpp:31-37)
// blocked_sum's per-block partials (parallel.hpp:39-40): one CTA per block
// of 4096 contributions stages them through shared memory with coalesced
// loads, then one thread adds them in index order (the reference's order)
struct FlagSet {
    __device__ bool operator()(unsigned v) const { return v != 0; }
};
struct CellId {  // cell ids fit int (cub's item count, as before)
    __device__ int operator()(long long c) const { return static_cast<int>(c); }
};
struct CellIdFrom {  // a z-slab's cells: index i of its range is global cell base + i
    long long base;
    __device__ int operator()(long long c) const { return static_cast<int>(base + c); }
};

__global__ void block_partials(const double* __restrict__ contrib, long long n, double* __restrict__ partial,
                               const long long* __restrict__ n_dev = nullptr) {
    __shared__ double buf[4096];
    // n_dev (the device loop): the count in device memory, CTAs stride over blocks
    const long long n_ = n_dev != nullptr ? __ldg(n_dev) : n;
    const long long nblk = (n_ + 4095) / 4096;
    for (long long blk = blockIdx.x; blk < nblk; blk += (n_dev != nullptr ? gridDim.x : nblk)) {
        const long long lo = blk * 4096;
        const int len = static_cast<int>(min(n_ - lo, 4096LL));
        for (int t = threadIdx.x; t < len; t += blockDim.x) buf[t] = contrib[lo + t];
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
#pragma unroll 16  // the loads of 16 terms ahead of the serial add chain (same order, same bits)
            for (int t = 0; t < len; ++t) s += buf[t];
            partial[blk] = s;
        }
        __syncthreads();
    }
}

// blocked_sum's final serial pass over the block partials in block order
// (parallel.hpp:39-40) and pow(total, 1/p) (metrics.cpp:142,183), on the
// device for the device-controlled loop: sqrt for p = 2 (the correctly
// rounded value, which glibc's pow returns except in rare hard cases), CUDA's
// pow otherwise. *e2 = the energy; flags bit 0 = out of domain (2d)
__global__ void energy_finish(const double* __restrict__ partial, const long long* __restrict__ n_dev, int p,
                              const int* __restrict__ ood, double* __restrict__ e2, int* __restrict__ flags) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const long long nblk = (*n_dev + 4095) / 4096;
    double total = 0.0;
    for (long long b = 0; b < nblk; ++b) total += partial[b];
    *e2 = p == 2 ? sqrt(total) : (p == 1 ? total : pow(total, 1.0 / p));
    if (*ood) *flags |= 1;
}

}  // namespace

int lsr_prep_surface_energy(const SlParams& P, const double* phi, const double* dist, int p, int refine,
                            double* energy, int64_t* n_cells, cudaStream_t s, std::string* err) {
#define EN_TRY(x)                                                       \
    do {                                                                \
        cudaError_t e_ = (x);                                           \
        if (e_ != cudaSuccess) {                                        \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_);     \
            return LSR_ERR_CUDA;                                        \
        }                                                               \
    } while (0)
    if (P.dim == 3 && (p < 1 || refine < 1)) {
        *err = "energy_3d: invalid p or refinement";  // metrics.cpp:147
        return LSR_ERR_CONFIG;
    }
    if (P.dim == 2 && p < 1) {
        *err = "energy_2d: p must be >= 1";  // metrics.cpp:115
        return LSR_ERR_CONFIG;
    }
    const long long ncells = static_cast<long long>(P.nx - 1) * (P.ny - 1) * (P.dim == 3 ? (P.nz - 1) : 1);
    if (ncells > 0x7fffffffLL) {  // interface cell ids are kept as int
        *err = "surface_energy: grids of 2^31 cells or more are not supported";
        return LSR_ERR_CONFIG;
    }
    // workspace per device, grown on demand (no per-call cudaMalloc); one
    // process may drive several devices (one context each)
    static std::mutex mu;
    struct Work {
        unsigned char* flags = nullptr;
        int* cells = nullptr;
        int* scal = nullptr;  // [0] selected count, [1] out-of-domain flag
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        long long cap = 0;
        double* contrib = nullptr;
        double* partial = nullptr;
        long long ccap = 0;
    };
    static Work works[kEnergyMaxDevices];
    int dev = 0;
    EN_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kEnergyMaxDevices) {
        *err = "surface_energy: device ordinal out of range";
        return LSR_ERR_CONFIG;
    }
    Work& W = works[dev];
    std::lock_guard<std::mutex> lock(mu);
    if (ncells > W.cap) {
        cudaFree(W.flags);
        cudaFree(W.cells);
        W.flags = nullptr;
        W.cells = nullptr;
        W.cap = 0;
        EN_TRY(cudaMalloc(&W.flags, ncells));
        EN_TRY(cudaMalloc(&W.cells, sizeof(int) * ncells));
        W.cap = ncells;
    }
    if (!W.scal) EN_TRY(cudaMalloc(&W.scal, sizeof(int) * 2));
    EN_TRY(cudaMemsetAsync(W.scal, 0, sizeof(int) * 2, s));
    const int T = 256;
    static const bool march = !(std::getenv("LSR_FLAG_MARCH") && std::atoi(std::getenv("LSR_FLAG_MARCH")) == 0);
    if (P.dim == 3 && P.nx % 4 == 0 && march) {
        const unsigned tpr = static_cast<unsigned>((P.nx - 1 + 3) / 4);
        const long long nt = static_cast<long long>(P.ny - 1) * tpr * ((P.nz - 1 + kMarchCells - 1) / kMarchCells);
        flag_cells_march<<<static_cast<unsigned>((nt + T - 1) / T), T, 0, s>>>(P, phi, tpr, W.flags, 0, P.nz - 1);
    } else if (P.dim == 3 && P.nx % 4 == 0) {
        const unsigned tpr = static_cast<unsigned>((P.nx - 1 + 3) / 4);
        const long long nt = static_cast<long long>(P.ny - 1) * (P.nz - 1) * tpr;
        flag_cells4<<<static_cast<unsigned>((nt + T - 1) / T), T, 0, s>>>(P, phi, tpr, nt, W.flags);
    } else {
        flag_cells<<<static_cast<unsigned>((ncells + T - 1) / T), T, 0, s>>>(P, phi, 0, ncells, W.flags);
    }
    lsr_note_launch();
    const size_t tb = lsr_compact::scratch_bytes(ncells) + sizeof(long long);
    if (tb > W.tmp_bytes) {
        cudaFree(W.tmp);
        W.tmp = nullptr;
        W.tmp_bytes = 0;
        EN_TRY(cudaMalloc(&W.tmp, tb));
        W.tmp_bytes = tb;
    }
    // interface cells in ascending order (metrics.cpp:150-156 visits them so)
    long long* d_nc = static_cast<long long*>(W.tmp);
    EN_TRY(lsr_compact::compact(lsr_compact::BytePred<FlagSet>{W.flags, {}}, CellId{}, ncells, W.cells, d_nc, d_nc + 1,
                                tb - sizeof(long long), s));
    lsr_note_launch();
    lsr_note_launch();
    long long nc = 0;
    EN_TRY(cudaMemcpyAsync(&nc, d_nc, sizeof nc, cudaMemcpyDeviceToHost, s));
    EN_TRY(cudaStreamSynchronize(s));
    *n_cells = nc;
    double total = 0.0;
    if (nc > 0) {
        const long long nblk = (nc + 4095) / 4096;
        if (nc > W.ccap) {
            cudaFree(W.contrib);
            cudaFree(W.partial);
            W.contrib = nullptr;
            W.partial = nullptr;
            W.ccap = 0;
            EN_TRY(cudaMalloc(&W.contrib, sizeof(double) * nc));
            EN_TRY(cudaMalloc(&W.partial, sizeof(double) * ((nc + 4095) / 4096)));
            W.ccap = nc;
        }
        if (P.dim == 3) {
            const int r = refine;
            const double dxp = P.dx / r;
            const double select = std::sqrt(3.0) / 2.0 * dxp;  // metrics.cpp:157
            const unsigned g = static_cast<unsigned>((nc + 127) / 128);
            if (r <= kMaxRefine)
                contrib_3d_hoisted<false><<<static_cast<unsigned>((nc + LSR_EN_THREADS - 1) / LSR_EN_THREADS), LSR_EN_THREADS,
                                     0, s>>>(P, phi, dist, W.cells, nc, r, dxp, select, p, W.contrib, nullptr);
            else
                contrib_3d<<<g, 128, 0, s>>>(P, phi, dist, W.cells, nc, r, dxp, select, p, W.contrib);
        } else {
            contrib_2d<false><<<static_cast<unsigned>((nc + 127) / 128), 128, 0, s>>>(P, phi, dist, W.cells, nc, p,
                                                                                W.contrib, W.scal + 1, nullptr);
        }
        lsr_note_launch();
        block_partials<<<static_cast<unsigned>(nblk), 256, 0, s>>>(W.contrib, nc, W.partial);
        lsr_note_launch();
        EN_TRY(cudaGetLastError());
        std::vector<double> h(nblk);
        int h_ood = 0;
        EN_TRY(cudaMemcpyAsync(h.data(), W.partial, sizeof(double) * nblk, cudaMemcpyDeviceToHost, s));
        EN_TRY(cudaMemcpyAsync(&h_ood, W.scal + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        EN_TRY(cudaStreamSynchronize(s));
        if (h_ood) {
            *err = "locate_cell: point outside grid hull";
            return LSR_ERR_OUT_OF_DOMAIN;
        }
        for (double v : h) total += v;  // blocked_sum (parallel.hpp:39-40)
    }
    *energy = std::pow(total, 1.0 / p);  // metrics.cpp:142,183
    return LSR_OK;
#undef EN_TRY
}

// ---------------------------------------------------------------------------
// z-slab E_p: the interface cells of the owned cell planes
// [k_lo, k_hi) and their contributions (ascending global cell order), then
// the pieces of blocked_sum (parallel.hpp:26-42) this rank can form on its
// own given the global position `offset` of its first contribution: the
// sums of the 4096-blocks that lie wholly in its range, and the raw
// contributions before its first and after its last block boundary. The
// ranks' pieces, laid end to end, give the reference's block partials bit for
// bit (the host adds the split blocks serially and then the partials in
// block order, and applies pow).
int lsr_energy_slab_cells(const SlParams& P, const double* phi_g, const double* dist_g, int p, int refine, int k_lo,
                          int k_hi, EnergySlabWork& W, long long* n_cells, cudaStream_t s, std::string* err) {
#define ES_TRY(x)                                                   \
    do {                                                            \
        cudaError_t e_ = (x);                                       \
        if (e_ != cudaSuccess) {                                    \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_); \
            return LSR_ERR_CUDA;                                    \
        }                                                           \
    } while (0)
    if (P.dim != 3 || p < 1 || refine < 1) {
        *err = "energy slab: 3d grids, p >= 1 and refinement >= 1";
        return LSR_ERR_CONFIG;
    }
    const long long cx = P.nx - 1, cy = P.ny - 1;
    const long long c0 = static_cast<long long>(k_lo) * cy * cx, c1 = static_cast<long long>(k_hi) * cy * cx;
    const long long nrange = c1 > c0 ? c1 - c0 : 0;
    if (c1 > 0x7fffffffLL) {
        *err = "surface_energy: grids of 2^31 cells or more are not supported";
        return LSR_ERR_CONFIG;
    }
    if (nrange > W.cap) {
        cudaFree(W.flags);
        cudaFree(W.cells);
        cudaFree(W.contrib);
        W.flags = nullptr;
        W.cells = nullptr;
        W.contrib = nullptr;
        W.cap = 0;
        ES_TRY(cudaMalloc(&W.flags, nrange + 16));
        ES_TRY(cudaMalloc(&W.cells, sizeof(int) * nrange));
        ES_TRY(cudaMalloc(&W.contrib, sizeof(double) * nrange));
        W.cap = nrange;
    }
    const size_t tb = lsr_compact::scratch_bytes(nrange > 0 ? nrange : 1) + sizeof(long long);
    if (tb > W.tmp_bytes) {
        cudaFree(W.tmp);
        W.tmp = nullptr;
        ES_TRY(cudaMalloc(&W.tmp, tb));
        W.tmp_bytes = tb;
    }
    W.nc = 0;
    *n_cells = 0;
    if (nrange == 0) return LSR_OK;
    unsigned char* flags_g = W.flags - c0;
    const int T = 256;
    if (P.nx % 4 == 0) {
        const unsigned tpr = static_cast<unsigned>((P.nx - 1 + 3) / 4);
        const long long nt = cy * tpr * ((k_hi - k_lo + kMarchCells - 1) / kMarchCells);
        flag_cells_march<<<static_cast<unsigned>((nt + T - 1) / T), T, 0, s>>>(P, phi_g, tpr, flags_g, k_lo, k_hi);
    } else {
        flag_cells<<<static_cast<unsigned>((nrange + T - 1) / T), T, 0, s>>>(P, phi_g, c0, c1, flags_g);
    }
    lsr_note_launch();
    long long* d_nc = static_cast<long long*>(W.tmp);
    ES_TRY(lsr_compact::compact(lsr_compact::BytePred<FlagSet>{W.flags, {}}, CellIdFrom{c0}, nrange, W.cells, d_nc,
                                d_nc + 1, tb - sizeof(long long), s));
    lsr_note_launch();
    lsr_note_launch();
    long long nc = 0;
    ES_TRY(cudaMemcpyAsync(&nc, d_nc, sizeof nc, cudaMemcpyDeviceToHost, s));
    ES_TRY(cudaStreamSynchronize(s));
    if (nc > 0) {
        const double dxp = P.dx / refine;
        const double select = std::sqrt(3.0) / 2.0 * dxp;  // metrics.cpp:157
        if (refine <= kMaxRefine)
            contrib_3d_hoisted<false><<<static_cast<unsigned>((nc + LSR_EN_THREADS - 1) / LSR_EN_THREADS), LSR_EN_THREADS, 0,
                                 s>>>(P, phi_g, dist_g, W.cells, nc, refine, dxp, select, p, W.contrib, nullptr);
        else
            contrib_3d<<<static_cast<unsigned>((nc + 127) / 128), 128, 0, s>>>(P, phi_g, dist_g, W.cells, nc, refine,
                                                                               dxp, select, p, W.contrib);
        lsr_note_launch();
        ES_TRY(cudaGetLastError());
    }
    W.nc = nc;
    *n_cells = nc;
    return LSR_OK;
}

int lsr_energy_slab_pieces(EnergySlabWork& W, long long offset, double* h_blocks, long long* n_blocks, double* h_head,
                           long long* n_head, double* h_tail, long long* n_tail, cudaStream_t s, std::string* err) {
    const long long nc = W.nc;
    const long long s0 = (4096 - offset % 4096) % 4096;  // first local index on a block boundary
    long long head = nc < s0 ? nc : s0, full = 0;
    if (nc > s0) full = (nc - s0) / 4096;
    const long long tail0 = head + 4096 * full;
    *n_head = head;
    *n_blocks = full;
    *n_tail = nc - tail0;
    if (full > 0) {
        if (full > W.pcap) {
            cudaFree(W.partial);
            W.partial = nullptr;
            ES_TRY(cudaMalloc(&W.partial, sizeof(double) * full));
            W.pcap = full;
        }
        block_partials<<<static_cast<unsigned>(full), 256, 0, s>>>(W.contrib + s0, 4096 * full, W.partial);
        lsr_note_launch();
        ES_TRY(cudaMemcpyAsync(h_blocks, W.partial, sizeof(double) * full, cudaMemcpyDeviceToHost, s));
    }
    if (head > 0) ES_TRY(cudaMemcpyAsync(h_head, W.contrib, sizeof(double) * head, cudaMemcpyDeviceToHost, s));
    if (nc - tail0 > 0)
        ES_TRY(cudaMemcpyAsync(h_tail, W.contrib + tail0, sizeof(double) * (nc - tail0), cudaMemcpyDeviceToHost, s));
    ES_TRY(cudaStreamSynchronize(s));
    return LSR_OK;
#undef ES_TRY
}

void EnergySlabWork::release() {
    cudaFree(flags);
    cudaFree(cells);
    cudaFree(contrib);
    cudaFree(partial);
    cudaFree(tmp);
    *this = EnergySlabWork{};
}

// ---------------------------------------------------------------------------
// E_p inside the device-controlled loop (lsr_cuda_loop_run): the interface
// cells, their contributions and blocked_sum with the cell count in device
// memory; nothing is read back.

void EnergyLoopWork::release() {
    cudaFree(flags);
    cudaFree(cells);
    cudaFree(contrib);
    cudaFree(partial);
    cudaFree(nc);
    cudaFree(ood);
    cudaFree(tmp);
    *this = EnergyLoopWork{};
}

int lsr_energy_loop_reserve(const SlParams& P, EnergyLoopWork& W, std::string* err) {
#define EL_TRY(x)                                                       \
    do {                                                                \
        cudaError_t e_ = (x);                                           \
        if (e_ != cudaSuccess) {                                        \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_);     \
            return LSR_ERR_CUDA;                                        \
        }                                                               \
    } while (0)
    const long long ncells = static_cast<long long>(P.nx - 1) * (P.ny - 1) * (P.dim == 3 ? (P.nz - 1) : 1);
    if (ncells > 0x7fffffffLL) {
        *err = "surface_energy: grids of 2^31 cells or more are not supported";
        return LSR_ERR_CONFIG;
    }
    if (ncells <= W.cap) return LSR_OK;
    W.release();
    const long long nodes = P.nxy * P.nz;  // the tube's flags are per tube entry (<= nodes)
    EL_TRY(cudaMalloc(&W.flags, nodes));
    EL_TRY(cudaMalloc(&W.cells, sizeof(int) * ncells));
    EL_TRY(cudaMalloc(&W.contrib, sizeof(double) * ncells));
    EL_TRY(cudaMalloc(&W.partial, sizeof(double) * ((ncells + 4095) / 4096 + 1)));
    EL_TRY(cudaMalloc(&W.nc, 3 * sizeof(long long)));  // [0] interface cells = [1] dense + [2] tube selection
    EL_TRY(cudaMalloc(&W.ood, sizeof(int)));
    W.tmp_bytes = lsr_compact::scratch_bytes(nodes);
    EL_TRY(cudaMalloc(&W.tmp, W.tmp_bytes));
    W.cap = ncells;
    return LSR_OK;
}

int lsr_energy_enqueue(const SlParams& P, const double* phi, const double* dist, int p, int refine,
                       EnergyLoopWork& W, long long est_cells, double* d_e2, int* d_flags, cudaStream_t s,
                       std::string* err, const long long* tube, const long long* n_tube_dev, long long est_tube,
                       const int* hard) {
    if (p < 1 || (P.dim == 3 && refine < 1)) {
        *err = "surface_energy: invalid p or refinement";  // metrics.cpp:115,147
        return LSR_ERR_CONFIG;
    }
    if (P.dim == 3 && refine > kMaxRefine) {
        *err = "surface_energy: the device loop supports subcell_refine <= 8";
        return LSR_ERR_CONFIG;
    }
    if (int st = lsr_energy_loop_reserve(P, W, err)) return st;
    const long long ncells = W.cap;
    EL_TRY(cudaMemsetAsync(W.ood, 0, sizeof(int), s));
    const int T = 256;
    // the interface cells, ascending (metrics.cpp:150-156): every cell tested
    // (when *hard != 0, or always without a tube), or the cells based at the
    // tube's nodes (flag_cells_tube); the device decides, both selections go
    // to W.cells and the one that did not run selects nothing
    const bool sparse = tube != nullptr && n_tube_dev != nullptr && hard != nullptr;
    const int* dense_if = sparse ? hard : nullptr;
    if (P.dim == 3 && P.nx % 4 == 0) {
        const unsigned tpr = static_cast<unsigned>((P.nx - 1 + 3) / 4);
        const long long nt = static_cast<long long>(P.ny - 1) * tpr * ((P.nz - 1 + kMarchCells - 1) / kMarchCells);
        flag_cells_march<<<static_cast<unsigned>((nt + T - 1) / T), T, 0, s>>>(P, phi, tpr, W.flags, 0, P.nz - 1,
                                                                                dense_if);
    } else {
        flag_cells<<<static_cast<unsigned>((ncells + T - 1) / T), T, 0, s>>>(P, phi, 0, ncells, W.flags, dense_if);
    }
    lsr_note_launch();
    EL_TRY(lsr_compact::compact_m(lsr_compact::GatedBytes{W.flags, nullptr, dense_if, 1}, CellId{}, ncells, W.cells,
                                  sparse ? W.nc + 1 : W.nc, W.tmp, W.tmp_bytes, s));
    for (int q = 0; q < 2; ++q) lsr_note_launch();
    if (sparse) {
        const long long nodes = P.nxy * P.nz;
        const long long est = est_tube > 0 ? est_tube : 1;
        flag_cells_tube<<<static_cast<unsigned>((est + T - 1) / T), T, 0, s>>>(P, phi, tube, n_tube_dev, W.flags, hard);
        EL_TRY(lsr_compact::compact_m(lsr_compact::GatedBytes{W.flags, n_tube_dev, hard, 0},
                                      TubeCellId{tube, P.nx, P.ny, P.dim}, nodes, W.cells, W.nc + 2, W.tmp,
                                      W.tmp_bytes, s));
        add_counts<<<1, 1, 0, s>>>(W.nc);
        for (int q = 0; q < 4; ++q) lsr_note_launch();
    }
    // the contributions: an estimate of the count sizes the grid, which strides past it
    const long long est = est_cells > 0 ? est_cells : 1;
    if (P.dim == 3) {
        const double dxp = P.dx / refine;
        const double select = std::sqrt(3.0) / 2.0 * dxp;  // metrics.cpp:157
        contrib_3d_hoisted<true><<<static_cast<unsigned>((est + LSR_EN_THREADS - 1) / LSR_EN_THREADS), LSR_EN_THREADS, 0,
                             s>>>(P, phi, dist, W.cells, 0, refine, dxp, select, p, W.contrib, W.nc);
    } else {
        contrib_2d<true><<<static_cast<unsigned>((est + 127) / 128), 128, 0, s>>>(P, phi, dist, W.cells, 0, p, W.contrib,
                                                                           W.ood, W.nc);
    }
    block_partials<<<148 * 4, 256, 0, s>>>(W.contrib, 0, W.partial, W.nc);
    energy_finish<<<1, 32, 0, s>>>(W.partial, W.nc, p, W.ood, d_e2, d_flags);
    for (int q = 0; q < 3; ++q) lsr_note_launch();
    EL_TRY(cudaGetLastError());
    return LSR_OK;
#undef EL_TRY
}
