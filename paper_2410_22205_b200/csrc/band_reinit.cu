// band_reinit.cu — the band rebuild and the constrained reinitialisation on
// the GPU, bit-identical to the reference.
//
//  narrow_band (/root/reference/proj/src/grid.cpp:76-124): one fused pass
//    classifies every node (ACTIVE if |phi| < gamma, else REINIT_HALO if any
//    of its 3^dim neighbours is ACTIVE). The reference's in-place halo pass
//    only reads ACTIVE flags and only writes INACTIVE nodes, so evaluating
//    the neighbours' ACTIVE test directly is the same function. The
//    ascending `active` and `tube` lists come from order-preserving
//    compactions (cub::DeviceSelect).
//  clamp_field (grid.cpp:126-134): elementwise std::min(std::max(v,-g), g).
//  interface_one_step (reinit.cpp:18-59): out of place (the reference reads a
//    full copy `prev`), so every node sees the pre-pass values.
//  reinit_iterate (reinit.cpp:88-131): the node list is the tube minus the
//    frozen nodes (order preserved); Jacobi sweeps write the other buffer;
//    the residual max is an integer atomicMax on the non-negative bits of
//    |upd| (max is order free); the two buffers only ever differ on the node
//    list, so the reference's `std::swap` is a pointer swap.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "compact.cuh"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "band_launch.h"
#include "lsr_cuda.h"
#include "sl_device.cuh"

using lsr_dev::SlParams;

namespace {

__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

// div_const's guard (sl_device.cuh) as a predicate: a == +0 or
// 2^-900 <= |a| < 2^900
__device__ __forceinline__ bool markstein_ok(double a) {
    const long long bits = __double_as_longlong(a);
    const unsigned e = static_cast<unsigned>(bits >> 32) & 0x7ff00000u;
    return ((e - 0x07b00000u) <= (0x78300000u - 0x07b00000u)) | (bits == 0);
}
__device__ __forceinline__ double markstein(double a, double c, double rc) {
    const double q = a * rc;
    return __fma_rn(__fma_rn(-q, c, a), rc, q);
}

constexpr int kTubeBatch = 4;  // list entries per thread and round in the device loop's list passes

struct IterState {  // device-side control of the Jacobi sweeps
    unsigned long long residual_bits;
    int done;
    int iterations;
    unsigned arrived;  // CTAs of the running sweep that have reduced their residual (jacobi_pipe's fused stop rule)
    unsigned pad;
};

// the stop rule after a sweep (reinit.cpp:125-128) on the sweep's residual
__device__ __forceinline__ void stop_rule(IterState* st, unsigned long long residual_bits, double tol) {
    st->iterations += 1;
    if (__longlong_as_double(static_cast<long long>(residual_bits)) < tol) st->done = 1;
}

// narrow_band state (grid.cpp:85-116): 1 ACTIVE, 2 REINIT_HALO, 0 INACTIVE.
// The halo test "some node of the 3^dim box is ACTIVE" is a separable
// max-dilation of the ACTIVE indicator: dilate along x (pass 1, which also
// evaluates |phi| < gamma), then y (pass 2), then z (pass 3). Per node:
// bit 0 = dilated indicator, bit 1 = the node itself is ACTIVE.
// (all passes take node ids [base, end); buffers are indexed by global id)
__global__ void band_pass_x(SlParams P, const double* __restrict__ phi, double gamma, long long base, long long end,
                            unsigned char* __restrict__ t) {
    const long long id = base + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= end) return;
    int i, j, k;
    lsr_dev::unflatten(P, id, i, j, k);
    const bool c = fabs(__ldg(phi + id)) < gamma;
    bool d = c;
    if (i > 0) d = d || fabs(__ldg(phi + id - 1)) < gamma;
    if (i < P.nx - 1) d = d || fabs(__ldg(phi + id + 1)) < gamma;
    t[id] = static_cast<unsigned char>((c ? 2 : 0) | (d ? 1 : 0));
}

__global__ void band_pass_y(SlParams P, const unsigned char* __restrict__ t, long long base, long long end,
                            unsigned char* __restrict__ u, unsigned char* __restrict__ state) {
    const long long id = base + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= end) return;
    int i, j, k;
    lsr_dev::unflatten(P, id, i, j, k);
    const unsigned char c = t[id];
    unsigned char d = c & 1;
    if (j > 0) d |= t[id - P.nx] & 1;
    if (j < P.ny - 1) d |= t[id + P.nx] & 1;
    const unsigned char v = static_cast<unsigned char>((c & 2) | d);
    if (P.dim == 2) state[id] = (v & 2) ? 1 : ((v & 1) ? 2 : 0);
    else u[id] = v;
}

__global__ void band_pass_z(SlParams P, const unsigned char* __restrict__ u, long long base, long long end,
                            unsigned char* __restrict__ state) {
    const long long id = base + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= end) return;
    int i, j, k;
    lsr_dev::unflatten(P, id, i, j, k);
    const unsigned char c = u[id];
    unsigned char d = c & 1;
    if (k > 0) d |= u[id - P.nxy] & 1;
    if (k < P.nz - 1) d |= u[id + P.nxy] & 1;
    state[id] = (c & 2) ? 1 : (d ? 2 : 0);
}

// Vector forms of the three passes for rows of a multiple of 16 nodes: the x
// pass makes 4 nodes per thread (two 16-byte loads of phi, one 4-byte store),
// the y/z passes 16 per thread (16-byte loads and stores, bytewise logic on
// 32-bit lanes). Same results as the scalar passes above.

// the x pass of a quad: the 4 output bytes of nodes id .. id + 3 (x0 = the first node's i)
__device__ __forceinline__ unsigned band_quad(const SlParams& P, const double* __restrict__ phi, double gamma,
                                              long long id, int x0) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(phi + id));
    const double2 b = __ldg(reinterpret_cast<const double2*>(phi + id) + 1);
    const bool c0 = fabs(a.x) < gamma, c1 = fabs(a.y) < gamma, c2 = fabs(b.x) < gamma, c3 = fabs(b.y) < gamma;
    const bool l = x0 > 0 && fabs(__ldg(phi + id - 1)) < gamma;
    const bool r = x0 + 4 < P.nx && fabs(__ldg(phi + id + 4)) < gamma;
    const unsigned o0 = (c0 ? 2u : 0u) | ((c0 || l || c1) ? 1u : 0u);
    const unsigned o1 = (c1 ? 2u : 0u) | ((c1 || c0 || c2) ? 1u : 0u);
    const unsigned o2 = (c2 ? 2u : 0u) | ((c2 || c1 || c3) ? 1u : 0u);
    const unsigned o3 = (c3 ? 2u : 0u) | ((c3 || c2 || r) ? 1u : 0u);
    return o0 | (o1 << 8) | (o2 << 16) | (o3 << 24);
}

__global__ void band_pass_x4(SlParams P, const double* __restrict__ phi, double gamma, long long base4, long long end4,
                             unsigned* __restrict__ t) {
    const long long q = base4 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= end4) return;
    const long long id = 4 * q;
    t[q] = band_quad(P, phi, gamma, id, static_cast<int>(id % P.nx));
}

// The device loop's x pass (rows of whole 16-node groups): 16 nodes per
// thread. old_state = the band's state bytes of the previous iteration; when
// *skip_if_clear == 0 the field differs from that iteration's only on its
// tube — SL on the ACTIVE nodes, one-step and sweeps on the tube, a clamp
// that only produces +-gamma — so a node off the old tube is not ACTIVE now
// either, and a quad whose nodes and x-neighbours were all off the tube
// gives 0 without phi being read (most of the grid).
__global__ void band_pass_x16(SlParams P, const double* __restrict__ phi, double gamma, long long n16,
                              uint4* __restrict__ t, const unsigned char* __restrict__ old_state,
                              const int* __restrict__ skip_if_clear) {
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n16) return;
    const long long id = 16 * q;
    const int x0 = static_cast<int>(id % P.nx);
    unsigned w[4] = {1u, 1u, 1u, 1u}, l = 1u, r = 1u;  // nonzero: the quad is evaluated
    if (*skip_if_clear == 0) {
        const uint4 o = __ldg(reinterpret_cast<const uint4*>(old_state + id));
        w[0] = o.x, w[1] = o.y, w[2] = o.z, w[3] = o.w;
        l = x0 > 0 ? __ldg(old_state + id - 1) : 0u;
        r = x0 + 16 < P.nx ? __ldg(old_state + id + 16) : 0u;
    }
    unsigned out[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const unsigned left = g == 0 ? l : (w[g - 1] >> 24), right = g == 3 ? r : (w[g + 1] & 0xffu);
        out[g] = (w[g] | left | right) ? band_quad(P, phi, gamma, id + 4 * g, x0 + 4 * g) : 0u;
    }
    t[q] = make_uint4(out[0], out[1], out[2], out[3]);
}

__device__ __forceinline__ uint4 or4(uint4 a, uint4 b) { return make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w); }

// per byte: core (bit 1) -> 1, else dilated (bit 0) -> 2, else 0
__device__ __forceinline__ unsigned state_bytes(unsigned core_bits, unsigned dil_bits) {
    const unsigned b1 = core_bits & 0x01010101u, b0 = dil_bits & 0x01010101u;
    return b1 | ((b0 & ~b1) << 1);
}

// (c1, c2, the device loop's final pass over the whole grid: the CTA's 4096
// nodes are one compaction tile (compact.cuh), whose ACTIVE and tube counts
// it leaves in c1[blockIdx.x], c2[blockIdx.x] — compact2's count pass)
__global__ void band_pass_yz16(SlParams P, int axis, const uint4* __restrict__ in, long long base16, long long end16,
                               uint4* __restrict__ out, uint4* __restrict__ state, long long* __restrict__ c1 = nullptr,
                               long long* __restrict__ c2 = nullptr) {
    const long long q = base16 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    int na = 0, nt = 0;
    if (q < end16) {
        const long long row = (16 * q) / P.nx;
        const int j = static_cast<int>(row % P.ny), k = static_cast<int>(row / P.ny);
        const long long st = (axis == 1 ? P.nx : P.nxy) / 16;
        const bool has_m = axis == 1 ? j > 0 : k > 0, has_p = axis == 1 ? j < P.ny - 1 : k < P.nz - 1;
        const uint4 c = in[q];
        uint4 d = c;
        if (has_m) d = or4(d, in[q - st]);
        if (has_p) d = or4(d, in[q + st]);
        const unsigned m = 0x01010101u;
        if (axis == 1 && P.dim == 3) {  // keep core (bit 1) and the y-dilated bit 0 for the z pass
            out[q] = make_uint4((c.x & (m << 1)) | (d.x & m), (c.y & (m << 1)) | (d.y & m),
                                (c.z & (m << 1)) | (d.z & m), (c.w & (m << 1)) | (d.w & m));
        } else {
            const uint4 sb = make_uint4(state_bytes(c.x >> 1, d.x), state_bytes(c.y >> 1, d.y),
                                        state_bytes(c.z >> 1, d.z), state_bytes(c.w >> 1, d.w));
            state[q] = sb;
            if (c1 != nullptr) {  // state bytes: 1 ACTIVE, 2 halo
                na = __popc(sb.x & m) + __popc(sb.y & m) + __popc(sb.z & m) + __popc(sb.w & m);
                nt = __popc((sb.x | (sb.x >> 1)) & m) + __popc((sb.y | (sb.y >> 1)) & m) +
                     __popc((sb.z | (sb.z >> 1)) & m) + __popc((sb.w | (sb.w >> 1)) & m);
            }
        }
    }
    if (c1 != nullptr) {  // uniform per launch
        const int v = __reduce_add_sync(0xffffffffu, (na << 16) | nt);  // both counts <= 4096 per CTA, 512 per warp
        __shared__ int wsum[8];
        if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            int a = 0, b = 0;
            for (int w = 0; w < 8; ++w) {
                a += wsum[w] >> 16;
                b += wsum[w] & 0xffff;
            }
            c1[blockIdx.x] = a;
            c2[blockIdx.x] = b;
        }
    }
}

struct StateIs1 {  // narrow_band ACTIVE
    __device__ bool operator()(unsigned v) const { return v == 1; }
};
struct NonZero {  // in the tube / frozen
    __device__ bool operator()(unsigned v) const { return v != 0; }
};


// clamp_field two nodes per thread; a node is stored only when clamping
// changes its bits (after the first loop iteration most of the grid already
// sits at +-gamma, so the pass is mostly reads)
// `state` (optional): the band of the previous step; a change at a node
// outside its tube (state 0) raises *outside, telling the loop that the
// field changed beyond the tube (else it resyncs only tube and frozen nodes)
__global__ void clamp_kernel2(double2* __restrict__ f, long long n2, double gamma,
                              const unsigned char* __restrict__ state, int* __restrict__ outside) {
    const long long id = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= n2) return;
    const double2 v = f[id];
    const double a = smin(smax(v.x, -gamma), gamma), b = smin(smax(v.y, -gamma), gamma);
    const bool ca = __double_as_longlong(a) != __double_as_longlong(v.x);
    const bool cb = __double_as_longlong(b) != __double_as_longlong(v.y);
    if (ca || cb) {
        f[id] = make_double2(a, b);
        if (state && ((ca && !state[2 * id]) || (cb && !state[2 * id + 1]))) *outside = 1;
    }
}

// four nodes per thread (two 16-byte loads issued together): twice the bytes
// in flight per thread of clamp_kernel2, for a read-mostly pass at HBM rate
__global__ void clamp_kernel4(double2* __restrict__ f, long long n4, double gamma,
                              const unsigned char* __restrict__ state, int* __restrict__ outside) {
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n4) return;
    const double2 v0 = f[2 * q], v1 = f[2 * q + 1];
    const double c[4] = {smin(smax(v0.x, -gamma), gamma), smin(smax(v0.y, -gamma), gamma),
                         smin(smax(v1.x, -gamma), gamma), smin(smax(v1.y, -gamma), gamma)};
    const double o[4] = {v0.x, v0.y, v1.x, v1.y};
    bool ch[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) ch[r] = __double_as_longlong(c[r]) != __double_as_longlong(o[r]);
    if (ch[0] || ch[1]) f[2 * q] = make_double2(c[0], c[1]);
    if (ch[2] || ch[3]) f[2 * q + 1] = make_double2(c[2], c[3]);
    if (state && (ch[0] || ch[1] || ch[2] || ch[3])) {
        bool out = false;
#pragma unroll
        for (int r = 0; r < 4; ++r) out = out || (ch[r] && !state[4 * q + r]);
        if (out) *outside = 1;
    }
}

__global__ void clamp_kernel(double* __restrict__ f, long long n, double gamma, const unsigned char* __restrict__ state,
                             int* __restrict__ outside) {
    const long long id = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= n) return;
    const double v = f[id], c = smin(smax(v, -gamma), gamma);
    f[id] = c;
    if (state && __double_as_longlong(c) != __double_as_longlong(v) && !state[id]) *outside = 1;
}

// The device loop's one-step gate (lsr_reinit_enqueue): the dense one-step
// runs only when *only_if is set (the field may have a "hard jump", below),
// and it reports hard jumps of its input in *hard. A hard jump is an axis
// pair of opposite signs with neither node ACTIVE (|phi| < gamma fails for
// both). Without one, every sign-change pair of the SL output has a node in
// the band's ACTIVE set, so every frozen node lies in the tube and the
// one-step can visit the tube only (one_step_tube).
struct OneStepGate {
    const int* only_if;
    int* hard;
    double gamma;
};

// (a NaN product counts as one: a NaN node is in no band, and the sparse
// forms of the loop — this one-step, the E_2 cell flags — must not miss it)
__device__ __forceinline__ bool hard_pair(double pj, double pk, double gamma) {
    const double pr = pj * pk;
    return pr != pr || (pr < 0.0 && !(fabs(pj) < gamma) && !(fabs(pk) < gamma));
}

// interface_one_step (reinit.cpp:24-46); `prev` is read-only, `out` gets every
// node. The two "any" flags are raised once per warp (a single-address store
// from every frozen node serialises in L2).
// (prev, out, frozen point at node `base`, items [0, n): a z-slab's owned ids)
template <bool kGate = false>
__global__ void one_step(SlParams P, const double* __restrict__ prev, double* __restrict__ out,
                         unsigned char* __restrict__ frozen, long long n, int* __restrict__ any_frozen,
                         int* __restrict__ any_zero, long long base, OneStepGate gate = {}) {
    if (kGate && !*gate.only_if) return;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool is_zero = false, is_frozen = false, is_hard = false;
    if (t < n) {
        const long long id = base + t;
        prev -= base;
        out -= base;
        frozen -= base;
        int i, j, k;
        lsr_dev::unflatten(P, id, i, j, k);
        // the node and its six neighbours are loaded up front (an absent
        // neighbour reads the node itself and is skipped below), so the seven
        // loads are in flight together
        const bool has[6] = {i > 0, i + 1 < P.nx, j > 0, j + 1 < P.ny, P.dim == 3 && k > 0, P.dim == 3 && k + 1 < P.nz};
        const long long st[3] = {1, P.nx, P.nxy};
        double v[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) v[q] = __ldg(prev + (has[q] ? id + ((q & 1) ? st[q >> 1] : -st[q >> 1]) : id));
        const double pj = __ldg(prev + id);
        double val = pj;
        if (pj == 0.0) {
            is_zero = true;
        } else {
            double best = -1.0;
#pragma unroll
            for (int q = 0; q < 6; ++q) {  // axes x, y, z; -1 before +1 (reinit.cpp:30-41)
                if (!has[q]) continue;
                const double pk = v[q];
                if (pj * pk >= 0.0) continue;
                if (kGate && hard_pair(pj, pk, gate.gamma)) is_hard = true;
                const double crossing = P.dx * fabs(pj) / (fabs(pj) + fabs(pk));
                best = best < 0.0 ? crossing : smin(best, crossing);
            }
            if (best >= 0.0) {
                val = pj > 0.0 ? best : -best;
                is_frozen = true;
            }
        }
        out[id] = val;
        frozen[id] = is_frozen ? 1 : 0;
    }
    const unsigned zb = __ballot_sync(0xffffffffu, is_zero), fb = __ballot_sync(0xffffffffu, is_frozen);
    if ((threadIdx.x & 31) == 0) {
        if (zb) *any_zero = 1;
        if (fb) *any_frozen = 1;
    }
    if (kGate && __any_sync(0xffffffffu, is_hard) && (threadIdx.x & 31) == 0) *gate.hard = 1;
}

// one_step for 3d grids with nx % 4 == 0: four consecutive nodes of a row
// per thread, the node values and their y/z neighbours as 16-byte loads;
// per node the same arithmetic in the same neighbour order as one_step
template <bool kGate = false>
__device__ __forceinline__ void one_node(const SlParams& P, double pj, const double* v, const bool* has,
                                         double& val, bool& is_zero, bool& is_frozen, bool* is_hard = nullptr,
                                         double gamma = 0.0) {
    val = pj;
    if (pj == 0.0) {
        is_zero = true;
        return;
    }
    // common case first: no existing neighbour of the opposite sign (a NaN
    // product fails the test and takes the full path below)
    bool quiet = true;
#pragma unroll
    for (int q = 0; q < 6; ++q) quiet = quiet && (!has[q] || pj * v[q] >= 0.0);
    if (quiet) return;
    double best = -1.0;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        if (!has[q]) continue;
        const double pk = v[q];
        if (pj * pk >= 0.0) continue;
        if (kGate && hard_pair(pj, pk, gamma)) *is_hard = true;
        const double crossing = P.dx * fabs(pj) / (fabs(pj) + fabs(pk));
        best = best < 0.0 ? crossing : smin(best, crossing);
    }
    if (best >= 0.0) {
        val = pj > 0.0 ? best : -best;
        is_frozen = true;
    }
}

__device__ __forceinline__ void load4(const double* src, double* dst) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(src));
    const double2 b = __ldg(reinterpret_cast<const double2*>(src) + 1);
    dst[0] = a.x;
    dst[1] = a.y;
    dst[2] = b.x;
    dst[3] = b.y;
}

// one_step marching along z: a thread owns 4 nodes of a row (x0.., j) for
// kMarch consecutive planes and keeps the planes k-1, k, k+1 of its row in
// registers, so each plane costs three row loads (z+1, y-1, y+1) instead of
// five; same per-node arithmetic as one_step
#ifndef LSR_MARCH_PLANES
#define LSR_MARCH_PLANES 16
#endif
constexpr int kMarch = LSR_MARCH_PLANES;

#ifndef LSR_MARCH_MINB
#define LSR_MARCH_MINB 4  // 64 registers: occupancy beats the few spills (reinit 4.82 -> 4.71 ms at 512^3)
#endif
// planes [k_lo, k_hi) (the whole grid: 0, nz; a z-slab: its owned planes)
template <bool kGate = false>
__global__ void __launch_bounds__(256, LSR_MARCH_MINB) one_step_march(SlParams P, const double* __restrict__ prev, double* __restrict__ out,
                               unsigned* __restrict__ frozen4, int* __restrict__ any_frozen,
                               int* __restrict__ any_zero, int k_lo, int k_hi, OneStepGate gate = {}) {
    if (kGate && !*gate.only_if) return;
    bool hard = false;
    const int qx = P.nx / 4;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long rows = static_cast<long long>(qx) * P.ny;  // (x-quad, j) pairs
    bool zero = false, froz = false;
    if (t < rows * ((k_hi - k_lo + kMarch - 1) / kMarch)) {
        const int kb = static_cast<int>(t / rows);
        const long long r = t - kb * rows;
        const int j = static_cast<int>(r / qx), x0 = 4 * static_cast<int>(r - static_cast<long long>(j) * qx);
        const int k0 = k_lo + kb * kMarch, k1 = min(k_hi, k0 + kMarch);
        const bool hy[2] = {j > 0, j + 1 < P.ny};
        long long id = (static_cast<long long>(k0) * P.ny + j) * P.nx + x0;
        double zm[4], c[4], zp[4];
        load4(prev + (k0 > 0 ? id - P.nxy : id), zm);
        load4(prev + id, c);
        for (int k = k0; k < k1; ++k, id += P.nxy) {
            const bool hz[2] = {k > 0, k + 1 < P.nz};
            double ym[4], yp[4];
            load4(prev + (hz[1] ? id + P.nxy : id), zp);
            load4(prev + (hy[0] ? id - P.nx : id), ym);
            load4(prev + (hy[1] ? id + P.nx : id), yp);
            const double xl = x0 > 0 ? __ldg(prev + id - 1) : 0.0;
            const double xr = x0 + 4 < P.nx ? __ldg(prev + id + 4) : 0.0;
            double res[4];
            unsigned fb = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double v[6] = {q > 0 ? c[q - 1] : xl, q < 3 ? c[q + 1] : xr, ym[q], yp[q], zm[q], zp[q]};
                const bool has[6] = {x0 + q > 0, x0 + q + 1 < P.nx, hy[0], hy[1], hz[0], hz[1]};
                bool z = false, f = false;
                one_node<kGate>(P, c[q], v, has, res[q], z, f, &hard, gate.gamma);
                zero |= z;
                froz |= f;
                fb |= (f ? 1u : 0u) << (8 * q);
            }
            reinterpret_cast<double2*>(out + id)[0] = make_double2(res[0], res[1]);
            reinterpret_cast<double2*>(out + id)[1] = make_double2(res[2], res[3]);
            frozen4[id / 4] = fb;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                zm[q] = c[q];
                c[q] = zp[q];
            }
        }
    }
    const unsigned zb = __ballot_sync(0xffffffffu, zero), fbal = __ballot_sync(0xffffffffu, froz);
    if ((threadIdx.x & 31) == 0) {
        if (zb) *any_zero = 1;
        if (fbal) *any_frozen = 1;
    }
    if (kGate && __any_sync(0xffffffffu, hard) && (threadIdx.x & 31) == 0) *gate.hard = 1;
}

// interface_one_step on the band's tube only (the device loop, when the field
// has no hard jump — see OneStepGate): the tube nodes' values and frozen
// flags, same per-node arithmetic and neighbour order as one_step. Nodes off
// the tube are neither frozen nor changed, and the loop keeps `out` equal to
// `prev` there. Runs only when *gate.only_if is clear.
// (ftube[t] = the frozen flag of entry t: the loop's lists come from it)
__global__ void one_step_tube(SlParams P, const double* __restrict__ prev, double* __restrict__ out,
                              unsigned char* __restrict__ frozen, const long long* __restrict__ tube,
                              const long long* __restrict__ n_dev, int* __restrict__ any_frozen,
                              int* __restrict__ any_zero, const int* __restrict__ dense,
                              unsigned char* __restrict__ ftube) {
    if (*dense) return;
    const long long n = __ldg(n_dev);
    bool zero = false, froz = false;
    // one entry per thread and round; the next round's id is loaded while this
    // round's seven values are in flight (as the sweeps do, jacobi_pipe)
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long st[3] = {1, P.nx, P.nxy};
    long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    long long id = t < n ? __ldg(tube + t) : -1;
    while (__any_sync(0xffffffffu, id >= 0)) {
        bool has[6] = {false, false, false, false, false, false};
        double v[6], pj = 0.0;
        if (id >= 0) {
            int i, j, k;
            lsr_dev::unflatten(P, id, i, j, k);
            has[0] = i > 0, has[1] = i + 1 < P.nx, has[2] = j > 0, has[3] = j + 1 < P.ny;
            has[4] = P.dim == 3 && k > 0, has[5] = P.dim == 3 && k + 1 < P.nz;
#pragma unroll
            for (int q = 0; q < 6; ++q)
                v[q] = __ldg(prev + (has[q] ? id + ((q & 1) ? st[q >> 1] : -st[q >> 1]) : id));
            pj = __ldg(prev + id);
        }
        const long long tn = t + T;
        const long long idn = tn < n ? __ldg(tube + tn) : -1;
        if (id >= 0) {
            double val;
            bool z = false, f = false;
            one_node(P, pj, v, has, val, z, f);
            out[id] = val;
            if (f) frozen[id] = 1;  // the flags are all clear on entry (lsr_loop_sync_fields clears them)
            ftube[t] = f ? 1 : 0;
            zero |= z;
            froz |= f;
        }
        id = idn;
        t = tn;
    }
    const unsigned zb = __ballot_sync(0xffffffffu, zero), fb = __ballot_sync(0xffffffffu, froz);
    if ((threadIdx.x & 31) == 0) {
        if (zb) *any_zero = 1;
        if (fb) *any_frozen = 1;
    }
}

struct NotFrozen {  // tube entries t whose node was not frozen by the one-step (reinit.cpp:94-98)
    const unsigned char* frozen;
    const long long* tube;
    __device__ bool operator()(long long t) const { return !frozen[tube[t]]; }
};
struct TubeId {
    const long long* tube;
    __device__ long long operator()(long long t) const { return tube[t]; }
};

// smoothed sign at entry (reinit.cpp:250-257); also each node's neighbour
// mask for the sweeps (bit 2*ax: the -1 neighbour along ax exists, bit
// 2*ax+1: the +1 one), so the sweeps need no index arithmetic
// (nn_dev: the count in device memory (the device loop), grid-strided)
__global__ void sign_kernel(SlParams P, const double* __restrict__ phi, const long long* __restrict__ nodes,
                            long long nn, double eps2, double* __restrict__ sgn, unsigned char* __restrict__ nbr,
                            unsigned* __restrict__ nodes32, const long long* __restrict__ nn_dev = nullptr) {
    const long long n_ = nn_dev != nullptr ? __ldg(nn_dev) : nn;
    // host count: one entry per thread; device count: the grid strides, a
    // thread taking kTubeBatch entries per round with their loads in flight together
    const int nb = nn_dev != nullptr ? kTubeBatch : 1;
    const long long step_ = nn_dev != nullptr ? static_cast<long long>(gridDim.x) * blockDim.x * nb : n_;
    for (long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x * nb; t0 < n_; t0 += step_) {
        long long id[kTubeBatch];
        double v[kTubeBatch];
#pragma unroll
        for (int u = 0; u < kTubeBatch; ++u) {
            const long long t = t0 + u * blockDim.x + threadIdx.x;
            id[u] = (u < nb && t < n_) ? nodes[t] : -1;
        }
#pragma unroll
        for (int u = 0; u < kTubeBatch; ++u) v[u] = id[u] >= 0 ? __ldg(phi + id[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kTubeBatch; ++u) {
            if (id[u] < 0) continue;
            const long long t = t0 + u * blockDim.x + threadIdx.x;
            if (nodes32) nodes32[t] = static_cast<unsigned>(id[u]);  // 4-byte ids for the sweeps when the grid allows
            sgn[t] = v[u] / sqrt(v[u] * v[u] + eps2);
            int i, j, k;
            lsr_dev::unflatten(P, id[u], i, j, k);
            unsigned m = (i > 0 ? 1u : 0u) | (i < P.nx - 1 ? 2u : 0u) | (j > 0 ? 4u : 0u) | (j < P.ny - 1 ? 8u : 0u);
            if (P.dim == 3) m |= (k > 0 ? 16u : 0u) | (k < P.nz - 1 ? 32u : 0u);
            nbr[t] = static_cast<unsigned char>(m);
        }
        if (nn_dev == nullptr) break;
    }
}

// godunov_norm (reinit.cpp:63-84) on values already loaded: pc = phi at the
// node, vm/vp = phi at its -1/+1 neighbours per axis (hm/hp: they exist). The
// one-sided differences are divided by dx with div_const's Markstein form;
// the six range guards are combined into one branch (they pass in practice),
// the plain division is the fallback.
__device__ __forceinline__ double godunov_vals(const SlParams& P, double pc, const double* vm, const double* vp,
                                               const bool* hm, const bool* hp, double sgn) {
    double dm[3], dp[3];
    bool fast = P.fast_div != 0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        dm[ax] = hm[ax] ? pc - vm[ax] : 0.0;
        dp[ax] = hp[ax] ? vp[ax] - pc : 0.0;
        fast = fast & markstein_ok(dm[ax]) & markstein_ok(dp[ax]);
    }
    double acc = 0.0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        if (ax >= P.dim) break;
        double dminus = 0.0, dplus = 0.0;
        if (fast) {
            if (hm[ax]) dminus = markstein(dm[ax], P.dx, P.rdx);
            if (hp[ax]) dplus = markstein(dp[ax], P.dx, P.rdx);
        } else {
            if (hm[ax]) dminus = dm[ax] / P.dx;
            if (hp[ax]) dplus = dp[ax] / P.dx;
        }
        if (sgn > 0.0) {
            const double a = smax(dminus, 0.0), b = smin(dplus, 0.0);
            acc += smax(a * a, b * b);
        } else {
            const double a = smin(dminus, 0.0), b = smax(dplus, 0.0);
            acc += smax(a * a, b * b);
        }
    }
    return sqrt(acc);
}

// godunov_norm of a node with all six neighbours (3d). Per axis only the
// larger-magnitude candidate is divided: with u = max(dm, 0), v = min(dp, 0)
// (or the mirrored pair for sgn <= 0), the reference's
// max(RN(u/dx)^2, RN(v/dx)^2) equals RN(RN(c/dx)^2) for c the one of u, v of
// larger magnitude, because x -> RN(RN(|x|/dx)^2) is non-decreasing and
// RN(+-x/dx) = +-RN(x/dx); ties give equal values, a zero's sign vanishes in
// the square, and a NaN u (v) is selected exactly when the reference's max
// returns its NaN (finite) term. Returns false (the caller takes
// godunov_vals) when a selected c is outside div_const's Markstein range.
__device__ __forceinline__ double flip_sign(double x, unsigned m) {  // x, or -x when m = 0x80000000 (exact)
    return __hiloint2double(__double2hiint(x) ^ static_cast<int>(m), __double2loint(x));
}
// markstein_ok also for -0 (the quotient is squared: the sign of a zero vanishes)
__device__ __forceinline__ bool markstein_ok_z(double a) {
    const long long bits = __double_as_longlong(a);
    const unsigned e = static_cast<unsigned>(bits >> 32) & 0x7ff00000u;
    return ((e - 0x07b00000u) <= (0x78300000u - 0x07b00000u)) | ((bits << 1) == 0);
}
// The sgn <= 0 pair min(dm, 0), max(dp, 0) is the negative of
// max(-dm, 0), min(-dp, 0): negating both differences (a sign-bit flip)
// reduces it to the sgn > 0 form with every magnitude unchanged (zeros may
// change sign, NaNs stay NaN), and only magnitudes reach the result.
__device__ __forceinline__ bool godunov_interior(const SlParams& P, double pc, const double* vm, const double* vp,
                                                 double sgn, double& gn) {
    double acc = 0.0;
    bool ok = P.fast_div != 0;
    const unsigned m = sgn > 0.0 ? 0u : 0x80000000u;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const double dm = pc - vm[ax], dp = vp[ax] - pc;
        const double u = smax(flip_sign(dm, m), 0.0);
        const double v = smin(flip_sign(dp, m), 0.0);
        const double c = fabs(u) < fabs(v) ? v : u;
        ok = ok & markstein_ok_z(c);
        const double q = markstein(c, P.dx, P.rdx);
        acc += q * q;
    }
    gn = sqrt(acc);
    return ok;
}

// one Jacobi iteration (reinit.cpp:111-124). Memory-latency bound (one id
// load, then 7 dependent gathers per node), so each thread takes kJacNPT
// nodes and issues all their loads before any arithmetic. The running max of
// |upd| is kept as the bits of a non-negative double (integer order = double
// order); std::max(residual, x) never lets a NaN in, nor does `a > 0`; it is
// reduced within each warp before one atomic per warp.
#ifndef LSR_JAC_INTERIOR
#define LSR_JAC_INTERIOR 1  // godunov_interior for nodes with all six neighbours
#endif
#ifndef LSR_JAC_NPT
#define LSR_JAC_NPT 4
#endif
#ifndef LSR_JAC_MINB
#define LSR_JAC_MINB 1
#endif
constexpr int kJacNPT = LSR_JAC_NPT;
#ifndef LSR_JAC_THREADS
#define LSR_JAC_THREADS 128
#endif
constexpr int kJacThreads = LSR_JAC_THREADS;

template <class IdT>
__global__ void __launch_bounds__(kJacThreads, LSR_JAC_MINB)
    jacobi(SlParams P, const double* __restrict__ cur, double* __restrict__ nxt, const IdT* __restrict__ nodes,
           const double* __restrict__ sgn, const unsigned char* __restrict__ nbr, long long nn, double dtau,
           IterState* __restrict__ st) {
    const long long base = static_cast<long long>(blockIdx.x) * (kJacThreads * kJacNPT) + threadIdx.x;
    long long id[kJacNPT];
    double sg[kJacNPT];
    unsigned mk[kJacNPT];
    // the node list loads are issued before the stop flag is read, so the
    // flag's latency overlaps them instead of preceding them
#pragma unroll
    for (int r = 0; r < kJacNPT; ++r) {
        const long long t = base + r * kJacThreads;
        id[r] = t < nn ? static_cast<long long>(nodes[t]) : -1;
        sg[r] = t < nn ? sgn[t] : 0.0;
        mk[r] = t < nn ? nbr[t] : 0u;
    }
    if (*reinterpret_cast<volatile int*>(&st->done)) return;
    const long long stv[3] = {1, P.nx, P.nxy};
    double pc[kJacNPT], vm[kJacNPT][3], vp[kJacNPT][3];
    bool hm[kJacNPT][3], hp[kJacNPT][3];
#pragma unroll
    for (int r = 0; r < kJacNPT; ++r) {
        pc[r] = id[r] >= 0 ? __ldg(cur + id[r]) : 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            hm[r][ax] = (mk[r] >> (2 * ax)) & 1u;
            hp[r][ax] = (mk[r] >> (2 * ax + 1)) & 1u;
            vm[r][ax] = hm[r][ax] ? __ldg(cur + id[r] - stv[ax]) : 0.0;
            vp[r][ax] = hp[r][ax] ? __ldg(cur + id[r] + stv[ax]) : 0.0;
        }
    }
    unsigned long long bitsmax = 0;
#pragma unroll
    for (int r = 0; r < kJacNPT; ++r) {
        if (id[r] < 0) continue;
        const double s = sg[r];
        double gn;
        if (!(LSR_JAC_INTERIOR && P.dim == 3 && mk[r] == 63u && godunov_interior(P, pc[r], vm[r], vp[r], s, gn)))
            gn = godunov_vals(P, pc[r], vm[r], vp[r], hm[r], hp[r], s);
        const double upd = -dtau * s * (gn - 1.0);
        nxt[id[r]] = pc[r] + upd;
        const double a = fabs(upd);
        if (a > 0.0) {
            const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(a));
            bitsmax = b > bitsmax ? b : bitsmax;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, bitsmax, off);
        bitsmax = o > bitsmax ? o : bitsmax;
    }
    // one atomic per CTA: same-address atomics serialise in L2, and one per
    // warp cost most of a sweep
    __shared__ unsigned long long wmax[kJacThreads / 32];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = bitsmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
#pragma unroll
        for (int w = 0; w < kJacThreads / 32; ++w) m = wmax[w] > m ? wmax[w] : m;
        if (m) atomicMax(&st->residual_bits, m);
    }
}

// The same sweep as a persistent, software-pipelined kernel: each thread
// walks the node list in rounds of kPipeNPT nodes (stride = the grid's
// thread count, so consecutive threads keep consecutive list entries) and
// issues the next round's id / sign / neighbour-mask loads before it waits
// on the current round's seven gathers, so a thread always has two rounds of
// loads in flight instead of one batch per CTA lifetime (the per-node
// arithmetic is jacobi's: same bits).
#ifndef LSR_JAC_PIPE
#define LSR_JAC_PIPE 1
#endif
#ifndef LSR_JAC_PIPE_NPT
#define LSR_JAC_PIPE_NPT 2
#endif
#ifndef LSR_JAC_PIPE_THREADS
#define LSR_JAC_PIPE_THREADS 256
#endif
#ifndef LSR_JAC_PIPE_MINB
#define LSR_JAC_PIPE_MINB 3
#endif
constexpr int kPipeNPT = LSR_JAC_PIPE_NPT;
constexpr int kPipeThreads = LSR_JAC_PIPE_THREADS;

template <class IdT>
__global__ void __launch_bounds__(kPipeThreads, LSR_JAC_PIPE_MINB)
    jacobi_pipe(SlParams P, const double* __restrict__ cur, double* __restrict__ nxt, const IdT* __restrict__ nodes,
                const double* __restrict__ sgn, const unsigned char* __restrict__ nbr, long long nn, double dtau,
                IterState* __restrict__ st, const long long* __restrict__ nn_dev, double tol, int rule) {
    if (nn_dev != nullptr) nn = __ldg(nn_dev);  // the device loop's node count
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long stv[3] = {1, P.nx, P.nxy};
    long long id[kPipeNPT];
    double sg[kPipeNPT];
    unsigned mk[kPipeNPT];
    long long t0 = g;  // this thread's first node of the round: t0 + r * T, r < kPipeNPT
#pragma unroll
    for (int r = 0; r < kPipeNPT; ++r) {
        const long long t = t0 + r * T;
        id[r] = t < nn ? static_cast<long long>(nodes[t]) : -1;
        sg[r] = t < nn ? sgn[t] : 0.0;
        mk[r] = t < nn ? nbr[t] : 0u;
    }
    if (*reinterpret_cast<volatile int*>(&st->done)) return;
    unsigned long long bitsmax = 0;
    while (__any_sync(0xffffffffu, id[0] >= 0)) {  // per warp: no CTA barrier inside the sweep
        // this round's gathers
        double pc[kPipeNPT], vm[kPipeNPT][3], vp[kPipeNPT][3];
        bool hm[kPipeNPT][3], hp[kPipeNPT][3];
#pragma unroll
        for (int r = 0; r < kPipeNPT; ++r) {
            pc[r] = id[r] >= 0 ? __ldg(cur + id[r]) : 0.0;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                hm[r][ax] = (mk[r] >> (2 * ax)) & 1u;
                hp[r][ax] = (mk[r] >> (2 * ax + 1)) & 1u;
                vm[r][ax] = hm[r][ax] ? __ldg(cur + id[r] - stv[ax]) : 0.0;
                vp[r][ax] = hp[r][ax] ? __ldg(cur + id[r] + stv[ax]) : 0.0;
            }
        }
        // the next round's list entries, in flight while this round computes
        const long long tn = t0 + kPipeNPT * T;
        long long idn[kPipeNPT];
        double sgn_n[kPipeNPT];
        unsigned mkn[kPipeNPT];
#pragma unroll
        for (int r = 0; r < kPipeNPT; ++r) {
            const long long t = tn + r * T;
            idn[r] = t < nn ? static_cast<long long>(nodes[t]) : -1;
            sgn_n[r] = t < nn ? sgn[t] : 0.0;
            mkn[r] = t < nn ? nbr[t] : 0u;
        }
#pragma unroll
        for (int r = 0; r < kPipeNPT; ++r) {
            if (id[r] < 0) continue;
            const double s = sg[r];
            double gn;
            if (!(LSR_JAC_INTERIOR && P.dim == 3 && mk[r] == 63u && godunov_interior(P, pc[r], vm[r], vp[r], s, gn)))
                gn = godunov_vals(P, pc[r], vm[r], vp[r], hm[r], hp[r], s);
            const double upd = -dtau * s * (gn - 1.0);
            nxt[id[r]] = pc[r] + upd;
            const double a = fabs(upd);
            if (a > 0.0) {
                const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(a));
                bitsmax = b > bitsmax ? b : bitsmax;
            }
        }
#pragma unroll
        for (int r = 0; r < kPipeNPT; ++r) {
            id[r] = idn[r];
            sg[r] = sgn_n[r];
            mk[r] = mkn[r];
        }
        t0 = tn;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, bitsmax, off);
        bitsmax = o > bitsmax ? o : bitsmax;
    }
    __shared__ unsigned long long wmax[kPipeThreads / 32];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = bitsmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
#pragma unroll
        for (int w = 0; w < kPipeThreads / 32; ++w) m = wmax[w] > m ? wmax[w] : m;
        if (m) atomicMax(&st->residual_bits, m);
        if (rule) {
            // the stop rule, applied by the last CTA to arrive (rule == 0: the
            // caller reads the residual itself, e.g. a z-slab's rank)
            __threadfence();
            if (atomicAdd(&st->arrived, 1u) == gridDim.x - 1) {
                __threadfence();
                const unsigned long long rb = atomicExch(&st->residual_bits, 0ULL);
                st->arrived = 0;
                stop_rule(st, rb, tol);
            }
        }
    }
}

// the stop rule after a sweep as its own launch (sweeps without the fused rule)
__global__ void iter_check(IterState* st, double tol) {
    if (st->done) return;
    const unsigned long long rb = st->residual_bits;
    st->residual_bits = 0;
    stop_rule(st, rb, tol);
}

// one sweep cur -> nxt over the node list (W.nodes32 when the ids fit 4 bytes)
// (tol != nullptr: the sweep also applies the stop rule with *tol — one
// launch per sweep; nullptr: the residual is left in st for the caller)
template <class IdT>
static void launch_jacobi(const SlParams& P, const double* cur, double* nxt, const IdT* ids, const ReinitBuffers& W,
                          long long nn, double dtau, IterState* st, cudaStream_t s,
                          const long long* nn_dev = nullptr, const double* tol = nullptr) {
    const double tolv = tol ? *tol : 0.0;
    const int rule = tol ? 1 : 0;
    if (nn_dev != nullptr) {  // device count: the persistent sweep on every resident CTA
        jacobi_pipe<<<148u * LSR_JAC_PIPE_MINB, kPipeThreads, 0, s>>>(P, cur, nxt, ids, W.sgn, W.nbr, 0, dtau, st,
                                                                      nn_dev, tolv, rule);
        lsr_note_launch();
        return;
    }
    if (nn <= 0 || !LSR_JAC_PIPE) {  // no sweep kernel, or the one without the fused rule
        if (nn > 0) {
            const unsigned g = static_cast<unsigned>((nn + kJacThreads * kJacNPT - 1) / (kJacThreads * kJacNPT));
            jacobi<<<g, kJacThreads, 0, s>>>(P, cur, nxt, ids, W.sgn, W.nbr, nn, dtau, st);
            lsr_note_launch();
        }
        if (rule) {
            iter_check<<<1, 1, 0, s>>>(st, tolv);
            lsr_note_launch();
        }
        return;
    }
    if (LSR_JAC_PIPE) {
        // persistent: the resident CTAs (148 SMs x LSR_JAC_PIPE_MINB), or fewer for short lists
        const long long want = (nn + kPipeThreads * kPipeNPT - 1) / (kPipeThreads * kPipeNPT);
        const long long cap = 148LL * LSR_JAC_PIPE_MINB;
        jacobi_pipe<<<static_cast<unsigned>(want < cap ? want : cap), kPipeThreads, 0, s>>>(P, cur, nxt, ids, W.sgn,
                                                                                            W.nbr, nn, dtau, st,
                                                                                            nullptr, tolv, rule);
    }
    lsr_note_launch();
}


// clamp_field on a node list (the sparse form of the loop's clamp, see
// lsr_reinitialize): same per-node expression as clamp_kernel
__global__ void clamp_ids(double* __restrict__ f, const long long* __restrict__ ids, long long n, double gamma) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long id = ids[t];
    const double v = f[id], c = smin(smax(v, -gamma), gamma);
    if (__double_as_longlong(c) != __double_as_longlong(v)) f[id] = c;
}

__global__ void copy_ids(const double* __restrict__ src, double* __restrict__ dst, const long long* __restrict__ ids,
                         long long n) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long id = ids[t];
    dst[id] = src[id];
}

// ---- device-loop forms (lsr_cuda_loop_run): list lengths in device memory,
// a fixed grid striding over them (no host round trip for the count)
constexpr unsigned kDevGrid = 148 * 8;

__global__ void copy_ids_dev(const double* __restrict__ src, double* __restrict__ dst,
                             const long long* __restrict__ ids, const long long* __restrict__ n_dev) {
    const long long n = __ldg(n_dev);
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long id = ids[t];
        dst[id] = src[id];
    }
}

// (only_if: nothing is done when *only_if == 0 — the loop's fused tail runs instead)
__global__ void clamp_ids_dev(double* __restrict__ f, const long long* __restrict__ ids,
                              const long long* __restrict__ n_dev, double gamma,
                              const int* __restrict__ only_if = nullptr) {
    if (only_if != nullptr && *only_if == 0) return;
    const long long n = __ldg(n_dev);
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long id = ids[t];
        const double v = f[id], c = smin(smax(v, -gamma), gamma);
        if (__double_as_longlong(c) != __double_as_longlong(v)) f[id] = c;
    }
}

// the list lengths of the selection that ran (the other one's are zero)
__global__ void add_parts(const long long* __restrict__ parts, long long* __restrict__ counts) {
    counts[0] = parts[0] + parts[2];
    counts[1] = parts[1] + parts[3];
}

// the sweeps start (or, without an interface, are skipped: reinit.cpp:140-142)
__global__ void reinit_begin(IterState* st, const int* __restrict__ flags) {
    st->residual_bits = 0;
    st->iterations = 0;
    st->done = (flags[0] || flags[1]) ? 0 : 1;
}

// after the sweeps the result is in b (an even sweep count) or c (odd): copy
// it over the node list into the other buffer, so that b holds the result
// and the two agree on the list
__global__ void sweep_parity(double* __restrict__ b, double* __restrict__ c, const long long* __restrict__ ids,
                             const long long* __restrict__ n_dev, const IterState* __restrict__ st,
                             const int* __restrict__ only_if = nullptr) {
    if (only_if != nullptr && *only_if == 0) return;
    const long long n = __ldg(n_dev);
    const bool odd = (st->iterations & 1) != 0;
    const double* src = odd ? c : b;
    double* dst = odd ? b : c;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long id = ids[t];
        dst[id] = src[id];
    }
}

// the end of a device-loop iteration over an id list (tube or frozen ids):
// a and c take b's values, the frozen flags (when given) are cleared, and a
// node of b that is not ACTIVE and has an axis neighbour of the opposite sign
// that is not ACTIVE either (a hard jump, see OneStepGate) raises *hard
__global__ void loop_finish(SlParams P, const double* __restrict__ b, double* __restrict__ a, double* __restrict__ c,
                            const long long* __restrict__ ids, const long long* __restrict__ n_dev,
                            unsigned char* __restrict__ frozen, double gamma, int* __restrict__ hard,
                            const int* __restrict__ only_if = nullptr) {
    if (only_if != nullptr && *only_if == 0) return;
    const long long n = __ldg(n_dev);
    bool h = false;
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x; t0 < n; t0 += T) {
        const long long t = t0 + threadIdx.x;
        if (t >= n) break;
        const long long id = ids[t];
        const double v = b[id];
        a[id] = v;
        c[id] = v;
        if (frozen) frozen[id] = 0;
        if (!(fabs(v) < gamma)) {
            int i, j, k;
            lsr_dev::unflatten(P, id, i, j, k);
            const bool has[6] = {i > 0, i + 1 < P.nx, j > 0, j + 1 < P.ny, P.dim == 3 && k > 0,
                                 P.dim == 3 && k + 1 < P.nz};
            const long long st[3] = {1, P.nx, P.nxy};
#pragma unroll
            for (int q = 0; q < 6; ++q)
                if (has[q] && hard_pair(v, b[id + ((q & 1) ? st[q >> 1] : -st[q >> 1])], gamma)) h = true;
        }
    }
    if (__any_sync(0xffffffffu, h) && (threadIdx.x & 31) == 0) *hard = 1;
}

// The tail of a device-loop iteration in one pass over the tube, for
// iterations that ran the tube one-step (*dense == 0: the frozen nodes lie in
// the tube) and the sparse clamp: sweep_parity, clamp_ids_dev on the tube and
// the frozen ids, and both loop_finish launches. The sweeps' result R is b
// (even count) or c (odd); off the sweep list b and c agree (frozen nodes:
// copy_ids_dev; off the tube: the loop's invariant a = b = c). Per tube node:
// v = clamp(R) goes to b, a and c, the frozen flag is cleared, and a node
// that is not ACTIVE is checked for hard jumps against its neighbours' final
// values clamp(R[nbr]) — the clamp is idempotent, so it does not matter
// whether a neighbour's entry of R has been rewritten by its own thread yet.
__global__ void loop_tail(SlParams P, double* __restrict__ b, double* __restrict__ a, double* __restrict__ c,
                          const long long* __restrict__ tube, const long long* __restrict__ n_dev,
                          unsigned char* __restrict__ frozen, const IterState* __restrict__ st, double gamma,
                          int* __restrict__ hard, const int* __restrict__ dense) {
    if (*dense != 0) return;
    const long long n = __ldg(n_dev);
    const double* R = (st->iterations & 1) ? c : b;
    bool h = false;
    // kTubeBatch entries per thread and round, their loads issued together
    // (one entry per round left the pass waiting on two dependent loads)
    const long long T = static_cast<long long>(gridDim.x) * blockDim.x * kTubeBatch;
    for (long long t0 = static_cast<long long>(blockIdx.x) * blockDim.x * kTubeBatch; t0 < n; t0 += T) {
        long long id[kTubeBatch];
        double r[kTubeBatch];
#pragma unroll
        for (int u = 0; u < kTubeBatch; ++u) {
            const long long t = t0 + u * blockDim.x + threadIdx.x;
            id[u] = t < n ? tube[t] : -1;
        }
#pragma unroll
        for (int u = 0; u < kTubeBatch; ++u) r[u] = id[u] >= 0 ? R[id[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < kTubeBatch; ++u) {
            if (id[u] < 0) continue;
            const double v = smin(smax(r[u], -gamma), gamma);  // clamp_field (grid.cpp:126-134)
            b[id[u]] = v;
            a[id[u]] = v;
            c[id[u]] = v;
            frozen[id[u]] = 0;
            if (!(fabs(v) < gamma)) {
                int i, j, k;
                lsr_dev::unflatten(P, id[u], i, j, k);
                const bool has[6] = {i > 0, i + 1 < P.nx, j > 0, j + 1 < P.ny, P.dim == 3 && k > 0,
                                     P.dim == 3 && k + 1 < P.nz};
                const long long sd[3] = {1, P.nx, P.nxy};
                double w[6];
#pragma unroll
                for (int q = 0; q < 6; ++q) w[q] = has[q] ? R[id[u] + ((q & 1) ? sd[q >> 1] : -sd[q >> 1])] : v;
#pragma unroll
                for (int q = 0; q < 6; ++q)
                    if (has[q] && hard_pair(v, smin(smax(w[q], -gamma), gamma), gamma)) h = true;
            }
        }
    }
    if (__any_sync(0xffffffffu, h) && (threadIdx.x & 31) == 0) *hard = 1;
}

// dst = src on every node when *flag is set (the dense clamp changed a node
// outside the tube), else nothing
__global__ void copy_all_if(const double* __restrict__ src, double* __restrict__ dst, long long n,
                            const int* __restrict__ flag) {
    if (!*flag) return;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x)
        dst[t] = src[t];
}

}  // namespace

#define BR_TRY(x)                                                    \
    do {                                                             \
        cudaError_t e_ = (x);                                        \
        if (e_ != cudaSuccess) {                                     \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_);  \
            return LSR_ERR_CUDA;                                     \
        }                                                            \
    } while (0)

int BandBuffers::reserve(long long n, std::string* err) {
    if (n <= cap) return LSR_OK;
    release();
    BR_TRY(cudaMalloc(&state, n));
    BR_TRY(cudaMalloc(&active, sizeof(long long) * n));
    BR_TRY(cudaMalloc(&tube, sizeof(long long) * n));
    BR_TRY(cudaMalloc(&counts, sizeof(long long) * 2));
    cap = n;
    return LSR_OK;
}

void BandBuffers::release() {
    cudaFree(state);
    cudaFree(active);
    cudaFree(tube);
    cudaFree(counts);
    cudaFree(tmp);
    state = nullptr;
    active = tube = nullptr;
    counts = nullptr;
    tmp = nullptr;
    tmp_bytes = 0;
    cap = 0;
}

static int ensure_tmp(BandBuffers& B, size_t bytes, std::string* err) {
    if (bytes <= B.tmp_bytes) return LSR_OK;
    cudaFree(B.tmp);
    B.tmp = nullptr;
    BR_TRY(cudaMalloc(&B.tmp, bytes));
    B.tmp_bytes = bytes;
    return LSR_OK;
}

// the three dilation passes: x and y over node ids [a0, a1), z (the state)
// over [b0, b1) within [a0, a1); every buffer indexed by global node id. A
// z-slab passes its owned ids as [b0, b1) and one plane more on each side as
// [a0, a1) (the z pass reads the y-dilated planes next to its own).
static void band_passes(const SlParams& P, const double* phi, double gamma, long long a0, long long a1, long long b0,
                        long long b1, unsigned char* t, unsigned char* u, unsigned char* state, cudaStream_t s,
                        const int* skip_if_clear = nullptr, long long* c1 = nullptr, long long* c2 = nullptr) {
    const auto grid = [](long long items) { return static_cast<unsigned>((items + 255) / 256); };
    if (P.nx % 16 == 0) {  // rows of whole 16-byte vectors
        if (skip_if_clear != nullptr && a0 == 0)
            band_pass_x16<<<grid(a1 / 16), 256, 0, s>>>(P, phi, gamma, a1 / 16, reinterpret_cast<uint4*>(t), state,
                                                       skip_if_clear);
        else
            band_pass_x4<<<grid((a1 - a0) / 4), 256, 0, s>>>(P, phi, gamma, a0 / 4, a1 / 4,
                                                             reinterpret_cast<unsigned*>(t));
        const uint4* t16 = reinterpret_cast<const uint4*>(t);
        const uint4* u16c = reinterpret_cast<const uint4*>(u);
        uint4* u16 = reinterpret_cast<uint4*>(u);
        uint4* st16 = reinterpret_cast<uint4*>(state);
        if (P.dim == 3) {
            band_pass_yz16<<<grid((a1 - a0) / 16), 256, 0, s>>>(P, 1, t16, a0 / 16, a1 / 16, u16, st16);
            band_pass_yz16<<<grid((b1 - b0) / 16), 256, 0, s>>>(P, 2, u16c, b0 / 16, b1 / 16, nullptr, st16, c1, c2);
        } else {
            band_pass_yz16<<<grid((b1 - b0) / 16), 256, 0, s>>>(P, 1, t16, b0 / 16, b1 / 16, u16, st16, c1, c2);
        }
    } else {
        band_pass_x<<<grid(a1 - a0), 256, 0, s>>>(P, phi, gamma, a0, a1, t);
        if (P.dim == 3) {
            band_pass_y<<<grid(a1 - a0), 256, 0, s>>>(P, t, a0, a1, u, state);
            band_pass_z<<<grid(b1 - b0), 256, 0, s>>>(P, u, b0, b1, state);
        } else {
            band_pass_y<<<grid(b1 - b0), 256, 0, s>>>(P, t, b0, b1, u, state);
        }
    }
    lsr_note_launch();
    lsr_note_launch();
    if (P.dim == 3) lsr_note_launch();
}

int lsr_band_build(const SlParams& P, const double* phi, double gamma, BandBuffers& B, long long* n_active,
                   long long* n_tube, cudaStream_t s, std::string* err) {
    if (!(gamma > 0.0)) {
        *err = "narrow_band: gamma must be positive";  // grid.cpp:77
        return LSR_ERR_CONFIG;
    }
    const long long n = P.nxy * P.nz;
    if (int st = B.reserve(n, err)) return st;
    // scratch bytes for the two dilation passes live in the active/tube id
    // buffers, which are only written by the compaction afterwards
    unsigned char* t = reinterpret_cast<unsigned char*>(B.active);
    unsigned char* u = reinterpret_cast<unsigned char*>(B.tube);
    band_passes(P, phi, gamma, 0, n, 0, n, t, u, B.state, s);
    // ACTIVE and tube lists from one count pass and one write pass over the state bytes
    const size_t tb = lsr_compact::scratch_bytes2(n);
    if (int st = ensure_tmp(B, tb, err)) return st;
    BR_TRY(lsr_compact::compact2(lsr_compact::BytePred<StateIs1>{B.state, {}}, NonZero{}, lsr_compact::Identity{}, n,
                                 B.active, B.tube, B.counts, B.tmp, tb, s));
    for (int q = 0; q < 2; ++q) lsr_note_launch();
    long long h[2];
    BR_TRY(cudaMemcpyAsync(h, B.counts, sizeof h, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    *n_active = h[0];
    *n_tube = h[1];
    B.n_active = h[0];
    B.n_tube = h[1];
    return LSR_OK;
}

int lsr_clamp(double* f, long long n, double gamma, cudaStream_t s, std::string* err, const unsigned char* state,
              int* outside) {
    if (!(gamma > 0.0)) {
        *err = "clamp_field: gamma must be positive";  // grid.cpp:127
        return LSR_ERR_CONFIG;
    }
    if (n % 4 == 0 && reinterpret_cast<uintptr_t>(f) % 16 == 0)
        clamp_kernel4<<<static_cast<unsigned>((n / 4 + 255) / 256), 256, 0, s>>>(reinterpret_cast<double2*>(f), n / 4,
                                                                                gamma, state, outside);
    else if (n % 2 == 0 && reinterpret_cast<uintptr_t>(f) % 16 == 0)
        clamp_kernel2<<<static_cast<unsigned>((n / 2 + 255) / 256), 256, 0, s>>>(reinterpret_cast<double2*>(f), n / 2,
                                                                                gamma, state, outside);
    else
        clamp_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(f, n, gamma, state, outside);
    lsr_note_launch();
    BR_TRY(cudaGetLastError());
    return LSR_OK;
}

int ReinitBuffers::reserve(long long n, std::string* err) {
    if (n <= cap) return LSR_OK;
    release();
    BR_TRY(cudaMalloc(&frozen, n));
    BR_TRY(cudaMalloc(&nodes, sizeof(long long) * n));
    BR_TRY(cudaMalloc(&sgn, sizeof(double) * n));
    BR_TRY(cudaMalloc(&nbr, n));
    BR_TRY(cudaMalloc(&frozen_ids, sizeof(long long) * n));
    BR_TRY(cudaMalloc(&nodes32, sizeof(unsigned) * n));
    BR_TRY(cudaMalloc(&clamp_outside, sizeof(int)));
    BR_TRY(cudaMalloc(&scal, sizeof(unsigned long long) * 4));
    cap = n;
    return LSR_OK;
}

void ReinitBuffers::release() {
    cudaFree(frozen);
    cudaFree(nodes);
    cudaFree(sgn);
    cudaFree(nbr);
    cudaFree(frozen_ids);
    cudaFree(nodes32);
    nodes32 = nullptr;
    cudaFree(clamp_outside);
    frozen_ids = nullptr;
    clamp_outside = nullptr;
    cudaFree(scal);
    cudaFree(tmp);
    frozen = nullptr;
    nodes = nullptr;
    sgn = nullptr;
    nbr = nullptr;
    scal = nullptr;
    tmp = nullptr;
    tmp_bytes = 0;
    cap = 0;
}

// reinitialize (reinit.cpp:133-145) of the field in *phi (device), on the
// band B (tube list + state of the band field). *phi and *scratch are two
// full-grid buffers; on return *phi holds the result (pointers may swap).
// interface_one_step (reinit.cpp:18-59): *phi -> *scratch on every node,
// frozen flags in W.frozen. With an interface the buffers are swapped (*phi
// = the one-step result, *scratch = the field before it) and *had = 1; a
// field with no sign change and no zero is left as it was, *had = 0 (the
// reference's NoInterfaceError).
int lsr_reinit_one_step(const SlParams& P, double** phi, double** scratch, ReinitBuffers& W, int* had_interface,
                        cudaStream_t s, std::string* err) {
    const long long n = P.nxy * P.nz;
    if (int st = W.reserve(n, err)) return st;
    *had_interface = 0;
    W.n_frozen = 0;
    int* flags = reinterpret_cast<int*>(W.scal);  // [0] any_frozen, [1] any_zero
    BR_TRY(cudaMemsetAsync(W.scal, 0, sizeof(unsigned long long) * 4, s));
    if (P.dim == 3 && P.nx % 4 == 0) {
        const long long threads = static_cast<long long>(P.nx / 4) * P.ny * ((P.nz + kMarch - 1) / kMarch);
        one_step_march<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
            P, *phi, *scratch, reinterpret_cast<unsigned*>(W.frozen), flags, flags + 1, 0, P.nz);
    } else {
        one_step<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(P, *phi, *scratch, W.frozen, n, flags,
                                                                         flags + 1, 0);
    }
    lsr_note_launch();
    int hf[2];
    BR_TRY(cudaMemcpyAsync(hf, flags, sizeof hf, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    if (!hf[0] && !hf[1]) return LSR_OK;
    std::swap(*phi, *scratch);
    *had_interface = 1;
    return LSR_OK;
}

// reinit_iterate (reinit.cpp:88-131) on the tube minus the nodes flagged in
// W.frozen. On entry *scratch must equal *phi except possibly on the frozen
// nodes (scratch_differs_on_frozen: right after lsr_reinit_one_step), or
// anywhere (otherwise: it is refreshed whole). On return *phi holds the
// result and *scratch equals it on the iterated nodes.
int lsr_reinit_iterate(const SlParams& P, double** phi, double** scratch, const long long* tube, long long n_tube,
                       const ReinitParams& R, ReinitBuffers& W, bool scratch_differs_on_frozen, int* iterations,
                       cudaStream_t s, std::string* err) {
    if (!(R.dtau > 0.0)) {
        *err = "reinit: dtau must be positive";  // reinit.hpp:14-17
        return LSR_ERR_CONFIG;
    }
    if (R.max_iters < 1) {
        *err = "reinit: max_iters must be >= 1";
        return LSR_ERR_CONFIG;
    }
    const long long n = P.nxy * P.nz;
    if (int st = W.reserve(n, err)) return st;
    *iterations = 0;
    long long* d_nn = reinterpret_cast<long long*>(W.scal + 2);
    const size_t tb = lsr_compact::scratch_bytes(n > n_tube ? n : n_tube);
    if (tb > W.tmp_bytes) {
        cudaFree(W.tmp);
        W.tmp = nullptr;
        BR_TRY(cudaMalloc(&W.tmp, tb));
        W.tmp_bytes = tb;
    }
    // `ScalarField next = phi` (reinit.cpp:109): after the one-step the two
    // buffers differ exactly on the frozen nodes -> copy those; otherwise copy
    // the field
    if (scratch_differs_on_frozen) {
        long long nf = 0;
        BR_TRY(lsr_compact::compact(lsr_compact::BytePred<NonZero>{W.frozen, {}}, lsr_compact::Identity{}, n,
                                    W.frozen_ids, d_nn, W.tmp, tb, s));
        BR_TRY(cudaMemcpyAsync(&nf, d_nn, sizeof nf, cudaMemcpyDeviceToHost, s));
        BR_TRY(cudaStreamSynchronize(s));
        W.n_frozen = nf;
        if (nf > 0) {
            copy_ids<<<static_cast<unsigned>((nf + 255) / 256), 256, 0, s>>>(*phi, *scratch, W.frozen_ids, nf);
            lsr_note_launch();
        }
    } else {
        BR_TRY(cudaMemcpyAsync(*scratch, *phi, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    }
    // nodes = tube minus frozen, ascending (reinit.cpp:94-98)
    BR_TRY(lsr_compact::compact(NotFrozen{W.frozen, tube}, TubeId{tube}, n_tube, W.nodes, d_nn, W.tmp, tb, s));
    lsr_note_launch();
    lsr_note_launch();
    long long nn = 0;
    BR_TRY(cudaMemcpyAsync(&nn, d_nn, sizeof nn, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    const unsigned gb = static_cast<unsigned>((nn + 255) / 256);
    if (nn > 0) {
        sign_kernel<<<gb, 256, 0, s>>>(P, *phi, W.nodes, nn, R.sign_eps * R.sign_eps, W.sgn, W.nbr,
                                       n <= 0xffffffffLL ? W.nodes32 : nullptr);
        lsr_note_launch();
    }
    // All max_iters sweeps are queued without host round trips: sweep k reads
    // buf[k&1] and writes buf[(k+1)&1]; a one-thread check after each sweep
    // applies the reference's stop rule (reinit.cpp:125-128) and raises a
    // device flag that turns the remaining sweeps into no-ops. The number of
    // sweeps done tells which buffer holds the result.
    const double tol = R.residual_tol * P.dx;
    IterState* st = reinterpret_cast<IterState*>(W.scal);  // reuses the flag words
    BR_TRY(cudaMemsetAsync(st, 0, sizeof(IterState), s));
    double* buf[2] = {*phi, *scratch};
    for (int k = 0; k < R.max_iters; ++k) {
        if (n <= 0xffffffffLL) launch_jacobi(P, buf[k & 1], buf[(k + 1) & 1], W.nodes32, W, nn, R.dtau, st, s, nullptr, &tol);
        else launch_jacobi(P, buf[k & 1], buf[(k + 1) & 1], W.nodes, W, nn, R.dtau, st, s, nullptr, &tol);
    }
    BR_TRY(cudaGetLastError());
    IterState h{};
    BR_TRY(cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    const int iter = static_cast<int>(h.iterations);
    *phi = buf[iter & 1];
    *scratch = buf[(iter + 1) & 1];
    // keep the two buffers equal on the node list for the caller's next use
    if (nn > 0) {
        copy_ids<<<gb, 256, 0, s>>>(*phi, *scratch, W.nodes, nn);
        lsr_note_launch();
    }
    *iterations = iter;
    return LSR_OK;
}

// clamp_sparse: the field equalled a fully clamped field except on the tube
// of B and the nodes the one-step / sweeps may change (the one-step's frozen
// nodes, the tube's nodes) — e.g. phi^{n+1} of the driver loop, built from a
// clamped phi^n by an SL step on the ACTIVE nodes (a subset of the tube).
// Clamping is elementwise and idempotent, so clamping just those nodes gives
// the bits of the full clamp_field (grid.cpp:126-134).
int lsr_reinitialize(const SlParams& P, double** phi, double** scratch, const BandBuffers& B, double gamma,
                     const ReinitParams& R, ReinitBuffers& W, int* iterations, int* had_interface, cudaStream_t s,
                     std::string* err, bool clamp_sparse) {
    if (!(R.dtau > 0.0)) {
        *err = "reinit: dtau must be positive";  // reinit.hpp:14-17
        return LSR_ERR_CONFIG;
    }
    if (R.max_iters < 1) {
        *err = "reinit: max_iters must be >= 1";
        return LSR_ERR_CONFIG;
    }
    const long long n = P.nxy * P.nz;
    if (int st = W.reserve(n, err)) return st;
    *iterations = 0;
    BR_TRY(cudaMemsetAsync(W.clamp_outside, 0, sizeof(int), s));
    if (int st = lsr_reinit_one_step(P, phi, scratch, W, had_interface, s, err)) return st;
    // NoInterfaceError is caught by reinitialize (reinit.cpp:140-142): phi is
    // left as it was, then clamped
    if (*had_interface)
        if (int st = lsr_reinit_iterate(P, phi, scratch, B.tube, B.n_tube, R, W, true, iterations, s, err)) return st;
    if (!clamp_sparse) return lsr_clamp(*phi, n, gamma, s, err, B.state, W.clamp_outside);
    if (!(gamma > 0.0)) {
        *err = "clamp_field: gamma must be positive";  // grid.cpp:127
        return LSR_ERR_CONFIG;
    }
    const long long nf = *had_interface ? W.n_frozen : 0;
    if (B.n_tube > 0) {
        clamp_ids<<<static_cast<unsigned>((B.n_tube + 255) / 256), 256, 0, s>>>(*phi, B.tube, B.n_tube, gamma);
        lsr_note_launch();
    }
    if (nf > 0) {
        clamp_ids<<<static_cast<unsigned>((nf + 255) / 256), 256, 0, s>>>(*phi, W.frozen_ids, nf, gamma);
        lsr_note_launch();
    }
    BR_TRY(cudaGetLastError());
    return LSR_OK;
}

// ---------------------------------------------------------------------------
// z-slab forms: the same kernels on the owned planes
// [own_lo, own_hi) of a rank whose buffers hold the resident planes
// [win_lo, win_hi) and are passed shifted to global node ids (phi_g[id] is
// node id's value for any resident id). Boundary tests stay those of the
// global grid; a node's stencil (one plane up and down) must be resident,
// i.e. win_lo <= max(own_lo - 1, 0) and min(own_hi + 1, nz) <= win_hi.

namespace {
struct OffsetId {  // compaction item: the index shifted to a global id
    long long base;
    __device__ long long operator()(long long i) const { return base + i; }
};
}  // namespace

int lsr_band_build_slab(const SlParams& P, const double* phi_g, double gamma, BandBuffers& B, int win_lo, int win_hi,
                        int own_lo, int own_hi, long long* n_active, long long* n_tube, cudaStream_t s,
                        std::string* err) {
    if (!(gamma > 0.0)) {
        *err = "narrow_band: gamma must be positive";  // grid.cpp:77
        return LSR_ERR_CONFIG;
    }
    const long long nw = static_cast<long long>(win_hi - win_lo) * P.nxy, off = static_cast<long long>(win_lo) * P.nxy;
    if (int st = B.reserve(nw, err)) return st;
    unsigned char* t = reinterpret_cast<unsigned char*>(B.active) - off;  // scratch bytes (see lsr_band_build)
    unsigned char* u = reinterpret_cast<unsigned char*>(B.tube) - off;
    unsigned char* state = B.state - off;
    const long long a0 = static_cast<long long>(max(own_lo - 1, win_lo)) * P.nxy;
    const long long a1 = static_cast<long long>(min(own_hi + 1, win_hi)) * P.nxy;
    const long long b0 = static_cast<long long>(own_lo) * P.nxy, b1 = static_cast<long long>(own_hi) * P.nxy;
    band_passes(P, phi_g, gamma, a0, a1, b0, b1, t, u, state, s);
    const size_t tb = lsr_compact::scratch_bytes2(b1 - b0);
    if (int st = ensure_tmp(B, tb, err)) return st;
    BR_TRY(lsr_compact::compact2(lsr_compact::BytePred<StateIs1>{state + b0, {}}, NonZero{}, OffsetId{b0}, b1 - b0,
                                 B.active, B.tube, B.counts, B.tmp, tb, s));
    for (int q = 0; q < 2; ++q) lsr_note_launch();
    long long h[2];
    BR_TRY(cudaMemcpyAsync(h, B.counts, sizeof h, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    *n_active = B.n_active = h[0];
    *n_tube = B.n_tube = h[1];
    return LSR_OK;
}

// interface_one_step (reinit.cpp:24-46) on the owned planes: prev_g -> out_g,
// frozen flags; any_frozen / any_zero of the owned nodes (the caller ORs them
// over the ranks: NoInterfaceError is a global verdict)
int lsr_reinit_one_step_slab(const SlParams& P, const double* prev_g, double* out_g, ReinitBuffers& W, int win_lo,
                             int win_hi, int own_lo, int own_hi, int* any_frozen, int* any_zero, cudaStream_t s,
                             std::string* err) {
    const long long nw = static_cast<long long>(win_hi - win_lo) * P.nxy, off = static_cast<long long>(win_lo) * P.nxy;
    if (int st = W.reserve(nw, err)) return st;
    int* flags = reinterpret_cast<int*>(W.scal);
    BR_TRY(cudaMemsetAsync(W.scal, 0, sizeof(unsigned long long) * 4, s));
    BR_TRY(cudaMemsetAsync(W.frozen, 0, static_cast<size_t>(nw), s));
    unsigned char* frozen_g = W.frozen - off;
    if (P.nx % 4 == 0) {
        const long long threads = static_cast<long long>(P.nx / 4) * P.ny * ((own_hi - own_lo + kMarch - 1) / kMarch);
        one_step_march<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
            P, prev_g, out_g, reinterpret_cast<unsigned*>(frozen_g), flags, flags + 1, own_lo, own_hi);
    } else {
        const long long b0 = static_cast<long long>(own_lo) * P.nxy, n = static_cast<long long>(own_hi - own_lo) * P.nxy;
        one_step<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(P, prev_g + b0, out_g + b0, frozen_g + b0, n,
                                                                         flags, flags + 1, b0);
    }
    lsr_note_launch();
    int hf[2];
    BR_TRY(cudaMemcpyAsync(hf, flags, sizeof hf, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    *any_frozen = hf[0];
    *any_zero = hf[1];
    return LSR_OK;
}

// reinit_iterate's set-up (reinit.cpp:94-109) on the owned planes: `cur_g`
// holds the one-step result on every resident plane (halo exchanged);
// `nxt_g` becomes a copy of it (next = phi), the node list is the owned tube
// minus the frozen nodes (ascending), and the signs / neighbour masks
// (sign_kernel) are taken from cur. Returns the node count.
int lsr_reinit_slab_begin(const SlParams& P, const double* cur_g, double* nxt_g, const long long* tube,
                          long long n_tube, const ReinitParams& R, ReinitBuffers& W, int win_lo, int win_hi,
                          long long* n_nodes, cudaStream_t s, std::string* err) {
    const long long nw = static_cast<long long>(win_hi - win_lo) * P.nxy, off = static_cast<long long>(win_lo) * P.nxy;
    if (int st = W.reserve(nw, err)) return st;
    BR_TRY(cudaMemcpyAsync(nxt_g + off, cur_g + off, sizeof(double) * nw, cudaMemcpyDeviceToDevice, s));
    long long* d_nn = reinterpret_cast<long long*>(W.scal + 2);
    const size_t tb = lsr_compact::scratch_bytes(n_tube > 0 ? n_tube : 1);
    if (tb > W.tmp_bytes) {
        cudaFree(W.tmp);
        W.tmp = nullptr;
        BR_TRY(cudaMalloc(&W.tmp, tb));
        W.tmp_bytes = tb;
    }
    BR_TRY(lsr_compact::compact(NotFrozen{W.frozen - off, tube}, TubeId{tube}, n_tube, W.nodes, d_nn, W.tmp, tb, s));
    lsr_note_launch();
    lsr_note_launch();
    long long nn = 0;
    BR_TRY(cudaMemcpyAsync(&nn, d_nn, sizeof nn, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    if (nn > 0) {
        const bool small = static_cast<long long>(P.nxy) * P.nz <= 0xffffffffLL;
        sign_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, s>>>(P, cur_g, W.nodes, nn,
                                                                             R.sign_eps * R.sign_eps, W.sgn, W.nbr,
                                                                             small ? W.nodes32 : nullptr);
        lsr_note_launch();
    }
    *n_nodes = nn;
    return LSR_OK;
}

// one Jacobi sweep (reinit.cpp:111-124) cur_g -> nxt_g on the node list of
// lsr_reinit_slab_begin; *residual = max |upd| over the owned nodes (the
// caller takes the max over the ranks for the stop rule, reinit.cpp:125-128)
int lsr_reinit_slab_sweep(const SlParams& P, const double* cur_g, double* nxt_g, ReinitBuffers& W, long long nn,
                          double dtau, double* residual, cudaStream_t s, std::string* err) {
    IterState* st = reinterpret_cast<IterState*>(W.scal);
    BR_TRY(cudaMemsetAsync(st, 0, sizeof(IterState), s));
    if (static_cast<long long>(P.nxy) * P.nz <= 0xffffffffLL)
        launch_jacobi(P, cur_g, nxt_g, W.nodes32, W, nn, dtau, st, s);
    else
        launch_jacobi(P, cur_g, nxt_g, W.nodes, W, nn, dtau, st, s);
    unsigned long long bits = 0;
    BR_TRY(cudaMemcpyAsync(&bits, &st->residual_bits, sizeof bits, cudaMemcpyDeviceToHost, s));
    BR_TRY(cudaStreamSynchronize(s));
    std::memcpy(residual, &bits, sizeof bits);
    return LSR_OK;
}

// ---------------------------------------------------------------------------
// The device-controlled loop (lsr_cuda_loop_run, lsr_capi.cu): the band and
// reinitialisation phases with every count kept in device memory, so that a
// loop iteration is enqueued (and captured into a CUDA graph) without a host
// round trip.

// narrow_band (grid.cpp:76-123): the dilation passes and the fused two-list
// compaction; the counts stay in B.counts ([0] ACTIVE, [1] tube)
int lsr_band_enqueue(const SlParams& P, const double* phi, double gamma, BandBuffers& B, cudaStream_t s,
                     std::string* err, const int* hard) {
    const long long n = P.nxy * P.nz;
    if (int st = B.reserve(n, err)) return st;
    const size_t tb = lsr_compact::scratch_bytes2(n);
    if (int st = ensure_tmp(B, tb, err)) return st;
    unsigned char* t = reinterpret_cast<unsigned char*>(B.active);
    unsigned char* u = reinterpret_cast<unsigned char*>(B.tube);
    // hard (the loop's hard[0], see OneStepGate): clear when phi differs from the
    // previous iteration's phi only on that iteration's tube, whose state
    // bytes B.state still holds — the x pass then skips quads off that tube
    // rows of whole 16-node groups: the final pass also counts per compaction tile
    const bool counted = P.nx % 16 == 0;
    long long *c1 = nullptr, *c2 = nullptr;
    if (counted) lsr_compact::compact2_counts(B.tmp, n, &c1, &c2);
    band_passes(P, phi, gamma, 0, n, 0, n, t, u, B.state, s, hard, c1, c2);
    BR_TRY(lsr_compact::compact2(lsr_compact::BytePred<StateIs1>{B.state, {}}, NonZero{}, lsr_compact::Identity{}, n,
                                 B.active, B.tube, B.counts, B.tmp, tb, s, counted));
    for (int q = 0; q < (counted ? 1 : 2); ++q) lsr_note_launch();
    return LSR_OK;
}

// buffers the loop's reinit needs, allocated before any capture
int lsr_reinit_loop_reserve(long long n, ReinitBuffers& W, std::string* err) {
    if (int st = W.reserve(n, err)) return st;
    const size_t tb = lsr_compact::scratch_bytes2(n);
    if (tb > W.tmp_bytes) {
        cudaFree(W.tmp);
        W.tmp = nullptr;
        BR_TRY(cudaMalloc(&W.tmp, tb));
        W.tmp_bytes = tb;
    }
    return LSR_OK;
}

// reinitialize (reinit.cpp:133-145) of b (phi^{n+1}) on the band B of phi^n,
// c = the scratch field; the result is left in b, and c agrees with b on the
// frozen and swept nodes. Same kernels and bits as lsr_reinitialize, but
// nothing is read back: the one-step's flags decide on the device whether
// the sweeps run (reinit_begin), the frozen ids and the sweep list come from
// one compaction over the frozen flags and the band state, the sweep count
// decides which buffer is copied where (sweep_parity). clamp_sparse: b
// equalled a clamped field except on the tube and the frozen nodes (see
// lsr_reinitialize); otherwise the dense clamp flags changes outside the
// tube in L->clamp_outside.
int lsr_reinit_enqueue(const SlParams& P, double* b, double* c, const BandBuffers& B, double gamma,
                       const ReinitParams& R, ReinitBuffers& W, ReinitLoopDev* L, bool clamp_sparse, int* hard,
                       cudaStream_t s, std::string* err) {
    if (!(R.dtau > 0.0)) {
        *err = "reinit: dtau must be positive";  // reinit.hpp:14-17
        return LSR_ERR_CONFIG;
    }
    if (R.max_iters < 1) {
        *err = "reinit: max_iters must be >= 1";
        return LSR_ERR_CONFIG;
    }
    if (!(gamma > 0.0)) {
        *err = "clamp_field: gamma must be positive";  // grid.cpp:127
        return LSR_ERR_CONFIG;
    }
    const long long n = P.nxy * P.nz;
    if (int st = lsr_reinit_loop_reserve(n, W, err)) return st;
    BR_TRY(cudaMemsetAsync(L, 0, sizeof(ReinitLoopDev), s));
    int* flags = L->flags;
    // interface_one_step (reinit.cpp:18-59), b -> c: on every node when hard[0]
    // is set (the field may hold a hard jump: the run's first iteration, or
    // one found by the last check), which also reports hard jumps of b in
    // hard[1]; otherwise on the tube only (one_step_tube; c equals b off it)
    const OneStepGate gate{hard, hard + 1, gamma};
    if (P.dim == 3 && P.nx % 4 == 0) {
        const long long threads = static_cast<long long>(P.nx / 4) * P.ny * ((P.nz + kMarch - 1) / kMarch);
        one_step_march<true><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
            P, b, c, reinterpret_cast<unsigned*>(W.frozen), flags, flags + 1, 0, P.nz, gate);
    } else {
        one_step<true><<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(P, b, c, W.frozen, n, flags, flags + 1,
                                                                              0, gate);
    }
    unsigned char* ftube = W.nbr;  // per tube entry, until sign_kernel rewrites nbr
    one_step_tube<<<kDevGrid, 256, 0, s>>>(P, b, c, W.frozen, B.tube, B.counts + 1, flags, flags + 1, hard, ftube);
    for (int q = 0; q < 2; ++q) lsr_note_launch();
    // frozen ids and the sweep list (tube minus frozen, reinit.cpp:94-98),
    // ascending: after the dense one-step from the node flags (a frozen node
    // may lie off the tube), after the tube one-step from the tube's entries
    // (9.8 M instead of 134 M items at 512^3); the device decides (hard[0]),
    // the selection that did not run selects nothing
    using lsr_compact::Gated;
    BR_TRY(lsr_compact::compact2m(Gated<lsr_compact::BytePred<NonZero>>{{W.frozen, {}}, hard, 1},
                                  Gated<lsr_compact::ByteAndNot>{{B.state, W.frozen}, hard, 1},
                                  lsr_compact::Identity{}, n, W.frozen_ids, W.nodes, L->parts, W.tmp, W.tmp_bytes,
                                  s));
    BR_TRY(lsr_compact::compact2m(Gated<lsr_compact::ListFlag>{{ftube, B.counts + 1, 1}, hard, 0},
                                  Gated<lsr_compact::ListFlag>{{ftube, B.counts + 1, 0}, hard, 0}, TubeId{B.tube}, n,
                                  W.frozen_ids, W.nodes, L->parts + 2, W.tmp, W.tmp_bytes, s));
    add_parts<<<1, 1, 0, s>>>(L->parts, L->counts);
    for (int q = 0; q < 5; ++q) lsr_note_launch();
    // b takes the one-step's values (`ScalarField next = phi` after it, reinit.cpp:109)
    copy_ids_dev<<<kDevGrid, 256, 0, s>>>(c, b, W.frozen_ids, L->counts);
    const bool small = n <= 0xffffffffLL;
    sign_kernel<<<kDevGrid, 256, 0, s>>>(P, b, W.nodes, 0, R.sign_eps * R.sign_eps, W.sgn, W.nbr,
                                         small ? W.nodes32 : nullptr, L->counts + 1);
    IterState* st = reinterpret_cast<IterState*>(&L->residual_bits);
    reinit_begin<<<1, 1, 0, s>>>(st, flags);
    for (int q = 0; q < 3; ++q) lsr_note_launch();
    const double tol = R.residual_tol * P.dx;
    double* buf[2] = {b, c};
    for (int k = 0; k < R.max_iters; ++k) {
        if (small) launch_jacobi(P, buf[k & 1], buf[(k + 1) & 1], W.nodes32, W, 0, R.dtau, st, s, L->counts + 1, &tol);
        else launch_jacobi(P, buf[k & 1], buf[(k + 1) & 1], W.nodes, W, 0, R.dtau, st, s, L->counts + 1, &tol);
    }
    // the sweeps' result into b, then clamp_field (reinit.cpp:144). With the
    // sparse clamp and the tube one-step (hard[0] clear) both are left to
    // loop_tail (lsr_loop_sync_fields), which does them in its one pass
    const int* tail_off = clamp_sparse ? hard : nullptr;
    sweep_parity<<<kDevGrid, 256, 0, s>>>(b, c, W.nodes, L->counts + 1, st, tail_off);
    lsr_note_launch();
    if (clamp_sparse) {
        clamp_ids_dev<<<kDevGrid, 256, 0, s>>>(b, B.tube, B.counts + 1, gamma, tail_off);
        clamp_ids_dev<<<kDevGrid, 256, 0, s>>>(b, W.frozen_ids, L->counts, gamma, tail_off);
        for (int q = 0; q < 2; ++q) lsr_note_launch();
    } else if (int e = lsr_clamp(b, n, gamma, s, err, B.state, &L->clamp_outside)) {
        return e;
    }
    BR_TRY(cudaGetLastError());
    return LSR_OK;
}

// after an iteration: a (phi^n, the next iteration's out) takes b's values
// (phi^{n+1}) where they may differ — the tube of phi^n, the frozen nodes,
// and (if the dense clamp reported it) anywhere — so that the two fields are
// equal when the next iteration's SL step writes its updates into a
// ... and c (the scratch field) too, the frozen flags are cleared, and the
// tube and frozen nodes of phi^{n+1} are checked for hard jumps (hard[1]):
// pairs with both nodes off them kept the values (and signs, and
// non-ACTIVE-ness: the clamp preserves both) they had in phi^n, which the
// previous check (or the dense one-step) cleared
int lsr_loop_sync_fields(const SlParams& P, double* b, double* a, double* c, const BandBuffers& B,
                         ReinitBuffers& W, const ReinitLoopDev* L, double gamma, int* hard, bool clamp_sparse,
                         cudaStream_t s, std::string* err) {
    const long long n = P.nxy * P.nz;
    const int* tail_off = clamp_sparse ? hard : nullptr;  // as in lsr_reinit_enqueue
    if (clamp_sparse) {
        const IterState* st = reinterpret_cast<const IterState*>(&L->residual_bits);
        loop_tail<<<kDevGrid, 256, 0, s>>>(P, b, a, c, B.tube, B.counts + 1, W.frozen, st, gamma, hard + 1, hard);
        lsr_note_launch();
    }
    loop_finish<<<kDevGrid, 256, 0, s>>>(P, b, a, c, B.tube, B.counts + 1, nullptr, gamma, hard + 1, tail_off);
    loop_finish<<<kDevGrid, 256, 0, s>>>(P, b, a, c, W.frozen_ids, L->counts, W.frozen, gamma, hard + 1, tail_off);
    copy_all_if<<<kDevGrid, 256, 0, s>>>(b, a, n, &L->clamp_outside);
    copy_all_if<<<kDevGrid, 256, 0, s>>>(b, c, n, &L->clamp_outside);
    for (int q = 0; q < 4; ++q) lsr_note_launch();
    BR_TRY(cudaGetLastError());
    return LSR_OK;
}
