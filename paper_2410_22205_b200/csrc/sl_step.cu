// sl_step.cu — sm_100a kernels of the narrow-band semi-Lagrangian step and
// their launchers. Replaces the OpenMP loop of lsr::sl_step
// (/root/reference/proj/src/evolve.cpp:56-111) and the O(N) field copy at
// evolve.cpp:50 (see the sparse resync below).
//
// Layout in HBM: phi, out, d are dense fp64 arrays, x fastest (grid.hpp:19);
// active ids are ascending int64 (grid.hpp:82). One thread owns one active
// node: consecutive lanes take consecutive ids, i.e. neighbouring nodes of
// the same x-row, so their WENO stencils overlap and the 4x4x4 gathers hit
// L1 and coalesce into few sectors per warp load.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>

#include "compact.cuh"
#include "sl_device.cuh"
#include "sl_launch.h"

namespace lsr_dev {

// ZT: 3d WENO launches that read the z-line table; their per-line chains are
// shorter, so they trade registers for a 9th resident CTA per SM
__device__ __forceinline__ void node_ijk(const SlParams& P, long long id, int& i, int& j, int& k) {
    if (P.nxy * P.nz < (1LL << 31)) {  // Grid::unflatten (grid.hpp:22-27) in 32 bits when it fits
        const unsigned u = static_cast<unsigned>(id);
        const unsigned row = u / static_cast<unsigned>(P.nx);
        i = static_cast<int>(u - row * static_cast<unsigned>(P.nx));
        k = static_cast<int>(row / static_cast<unsigned>(P.ny));
        j = static_cast<int>(row - static_cast<unsigned>(k) * static_cast<unsigned>(P.ny));
    } else {
        i = static_cast<int>(id % P.nx);
        j = static_cast<int>((id / P.nx) % P.ny);
        k = static_cast<int>(id / P.nxy);
    }
}

// an id outside the grid is never dereferenced: it is recorded as the
// node count N in *bad (atomicMin with the non-finite ids, which are < N),
// which the host reports as a ConfigError
__device__ __forceinline__ bool id_outside(const SlParams& P, long long id, unsigned long long* bad) {
    const unsigned long long n = static_cast<unsigned long long>(P.nxy * P.nz);
    if (static_cast<unsigned long long>(id) < n) return false;
    atomicMin(bad, n);
    return true;
}

// the write of one update (evolve.cpp:107-117): out, the smallest
// non-finite id, and the fused halo exchange — the neighbours read these
// planes next step, so the update goes straight into their resident buffers
// over NVLink (peer mapped) instead of a separate plane exchange after the
// kernel
__device__ __forceinline__ void store_update(const SlParams& P, long long id, int k, double next, double* out,
                                             unsigned long long* bad) {
    if (!isfinite(next)) atomicMin(bad, static_cast<unsigned long long>(id));
    out[id] = next;
    bool pushed = false;
    if (P.peer_lo != nullptr && k < P.push_lo_below) {
        P.peer_lo[id] = next;
        pushed = true;
    }
    if (P.peer_hi != nullptr && k >= P.push_hi_from) {
        P.peer_hi[id] = next;
        pushed = true;
    }
    if (pushed) __threadfence_system();
}

// The device-controlled loop (loop_device.cu) launches the SL kernels on an
// active count that lives in device memory (P.n_dev) and an E_2 the same
// iteration computed on the device (P.energy_dev): the launch covers an
// estimate of the count with one thread per node, and a TAIL launch of the
// same kernel (a grid-stride loop from `base`) takes whatever lies beyond the
// estimate. p > 1 with E_2 == 0 skips the step (driver.cpp:191-195: out keeps
// phi, which the loop already holds in out); a non-finite E_2 is reported by
// the loop. Host-driven launches: n_dev = energy_dev = null, base = 0.
__device__ __forceinline__ long long sl_count(const SlParams& P, long long n_active) {
    if (P.n_dev == nullptr) return n_active;
    if (P.energy_dev != nullptr && P.p > 1 && !(__ldg(P.energy_dev) > 0.0)) return 0;
    return __ldg(P.n_dev);
}

// one thread per active node (Q1, 2d)
template <int DIM, int KIND, bool TAIL>
__global__ void __launch_bounds__(kSlThreads, kSlMinBlocks) sl_step_kernel(SlParams P, const double* __restrict__ phi,
                                                                           const double* __restrict__ dist,
                                                                           const int64_t* __restrict__ active,
                                                                           long long n_active, double* __restrict__ out,
                                                                           unsigned long long* __restrict__ bad,
                                                                           long long base) {
    const long long n = sl_count(P, n_active);
    for (long long a = base + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; a < n;
         a += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long id = __ldg(active + a);
        if (!id_outside(P, id, bad)) {
            int i, j, k;
            node_ijk(P, id, i, j, k);
            if (slab_node_miss(P, k))  // nothing of a non-resident node is read or written
                atomicAdd(P.halo_miss, 1ULL);
            else
                store_update(P, id, k, sl_node<DIM, KIND>(P, phi, dist, id, i, j, k), out, bad);
        }
        if (!TAIL) break;
    }
}

// 3d WENO with the z-line table, one thread per active node (its own launch
// shape; the per-line kernel above runs Q1, 2d and table-less WENO). (Splitting a node's four feet over 2 or 4 lanes, each lane
// recomputing the node's gradients and basis, measured slower: 3.77 / 4.22
// ms against 2.93 ms at 512^3 — the feet of a warp's nodes then touch 2-4x
// as many L1 lines per table load, and L1 wavefronts are the busiest unit.)
template <bool TAIL>
__global__ void __launch_bounds__(kSlThreadsW3, kSlMinBlocksW3) sl_step_zt_kernel(
    SlParams P, const double* __restrict__ phi, const double* __restrict__ dist, const int64_t* __restrict__ active,
    long long n_active, double* __restrict__ out, unsigned long long* __restrict__ bad, long long base) {
    const long long n = sl_count(P, n_active);
    for (long long a = base + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; a < n;
         a += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long id = __ldg(active + a);
        if (!id_outside(P, id, bad)) {
            int i, j, k;
            node_ijk(P, id, i, j, k);
            if (slab_node_miss(P, k)) {
                atomicAdd(P.halo_miss, 1ULL);
            } else {
                const bool use_zt = __ldg(P.ztab_bad) == 0u;
                const double next = sl_node<3, 1>(P, phi, dist, id, i, j, k, use_zt);
                store_update(P, id, k, next, out, bad);
            }
        }
        if (!TAIL) break;
    }
}

// ---- the TMA brick form of the 3d WENO step (sl_node_box) ----------------

#ifndef LSR_BOX_MINB
#define LSR_BOX_MINB 4
#endif
constexpr int kBoxThreads = 256;
constexpr int kBoxMinBlocks = LSR_BOX_MINB;  // 4 x 52 KB of staged phi per SM
constexpr int kBoxBytes = kBoxEX * kBoxEY * kBoxEZ * 8;

__device__ __forceinline__ long long brick8_of(const SlParams& P, long long id, int nbx, int nby) {
    int i, j, k;
    unflatten(P, id, i, j, k);
    return (static_cast<long long>(k / kSlBrick) * nby + j / kSlBrick) * nbx + i / kSlBrick;
}

// count[b] = active nodes in brick b (one atomic per (warp, brick))
__global__ void box_count_kernel(SlParams P, const int64_t* __restrict__ active, long long n, int nbx, int nby,
                                 unsigned* __restrict__ count) {
    const long long a = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long b = a < n ? brick8_of(P, __ldg(active + a), nbx, nby) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, b);
    if (b >= 0 && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(same) - 1))
        atomicAdd(count + b, static_cast<unsigned>(__popc(same)));
}

// ids grouped by brick: ids[off[b] + r] for the r-th of brick b's nodes (any order inside a brick)
__global__ void box_scatter_kernel(SlParams P, const int64_t* __restrict__ active, long long n, int nbx, int nby,
                                   const unsigned* __restrict__ off, unsigned* __restrict__ cursor,
                                   int64_t* __restrict__ ids) {
    const long long a = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t id = a < n ? __ldg(active + a) : 0;
    const long long b = a < n ? brick8_of(P, id, nbx, nby) : -1;
    const unsigned same = __match_any_sync(0xffffffffu, b);
    const int lane = threadIdx.x & 31, lead = __ffs(same) - 1;
    unsigned base = 0;
    if (b >= 0 && lane == lead) base = atomicAdd(cursor + b, static_cast<unsigned>(__popc(same)));
    base = __shfl_sync(same, base, lead);
    if (b >= 0) ids[off[b] + base + __popc(same & ((1u << lane) - 1u))] = id;
}

struct NonEmpty {
    const unsigned* count;
    __device__ bool operator()(long long b) const { return count[b] != 0u; }
};

__device__ __forceinline__ unsigned box_smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(kBoxThreads, kBoxMinBlocks) sl_step_box_kernel(const __grid_constant__ CUtensorMap tmap, SlParams P,
                                                                  const double* __restrict__ phi,
                                                                  const double* __restrict__ dist,
                                                                  const unsigned* __restrict__ list,
                                                                  const unsigned* __restrict__ off, long long n_listed,
                                                                  const int64_t* __restrict__ ids, long long n_ids,
                                                                  int nbx, int nby, double* __restrict__ out,
                                                                  unsigned long long* __restrict__ bad) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
    double* box = reinterpret_cast<double*>(smem + 128);
    const long long q = blockIdx.x;
    const unsigned b = list[q];
    const long long lo = off[b], hi = q + 1 < n_listed ? off[list[q + 1]] : n_ids;
    const int bi = static_cast<int>(b % nbx), bj = static_cast<int>((b / nbx) % nby),
              bk = static_cast<int>(b / (static_cast<unsigned>(nbx) * nby));
    const int x0 = max(bi * kSlBrick - kBoxLoX, 0), y0 = max(bj * kSlBrick - kBoxLo, 0),
              z0 = max(bk * kSlBrick - kBoxLo, 0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(box_smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(box_smem_u32(bar)),
                     "r"(kBoxBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];\n" ::"r"(box_smem_u32(box)),
            "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(x0), "r"(y0), "r"(z0), "r"(box_smem_u32(bar))
            : "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            box_smem_u32(bar))
        : "memory");
    const PhiBox B{box, x0, y0, z0};
    for (long long t = lo + threadIdx.x; t < hi; t += blockDim.x) {
        const long long id = __ldg(ids + t);
        if (id_outside(P, id, bad)) continue;
        int i, j, k;
        node_ijk(P, id, i, j, k);
        store_update(P, id, k, sl_node_box(P, phi, dist, id, i, j, k, B), out, bad);
    }
}

// The z-line table of the 3d WENO fast path. For node n = (i, j, k),
// 1 <= k <= nz - 2, it holds the terms of weno1_fast that depend only on the
// z-line data (interp.cpp:11-33), computed once per node instead of once per
// z-line per foot (a node's z data is read by ~50 z-lines of nearby feet):
//   zt[n] = {sd, S, Y, phi}: sd = phi(k-1) - 2 phi(k) + phi(k+1), the second
//           difference of the lines whose v0 (sdl) or vp (sdr) is n;
//           S = (sd^2/dx^2 + dx^2)^2 (the alpha denominator), Y = recip_seq(S)
//   zc[n] = {c1, e2}: c1 = phi(k+1) - phi(k-1) (d1), e2 = -3 phi(k) +
//           4 phi(k+1) - phi(k+2) (d2), for the line whose v0 is n
// Same operations and operands as weno1_fast => same bits. A node outside
// weno1_fast's range argument (square_in_range of sd^2, halvable c1/e2)
// sets *bad, which switches the step back to the per-line arithmetic.
//
// The table is dense (indexed by node id) but written only on bricks of
// kZtBrick^3 nodes that some foot stencil may read: every active node bounds
// how far its feet can land (zt_reach_kernel: from d, grad d, E and the step
// config, evolve.cpp:83-101, with |nu1|, |nu2| <= 1), its brick keeps the
// maximum, and each such brick covers the bricks its reach spans
// (zt_cover_kernel). The SL kernel still checks, per foot, that the bricks
// of the stencil's table nodes are covered (zt_covered in sl_device.cuh), so
// the bound only decides speed, never the result: an uncovered foot takes
// the per-line arithmetic, which gives the same bits.

__device__ __forceinline__ long long brick_of(int i, int j, int k, int nbx, int nby) {
    return (static_cast<long long>(k / kZtBrick) * nby + j / kZtBrick) * nbx + i / kZtBrick;
}

// reach[brick] = max over its active nodes of the foot reach: with D the
// bound on a foot's displacement in cells along any axis, a foot cell lies in
// [i - ceil(D), i + floor(D)]; packed as ceil(D) << 8 | floor(D) (monotone in
// D, so atomicMax keeps the largest), D capped at kZtMaxReach
__device__ __forceinline__ void zt_reach_one(const SlParams& P, const double* __restrict__ dist,
                                             const int64_t* __restrict__ active, long long a, long long n, int nbx,
                                             int nby, unsigned* __restrict__ reach) {
    long long b = -1;
    unsigned r = 0;
    long long id = 0;
    int i = 0, j = 0, k = 0;
    const bool inside = a < n && static_cast<unsigned long long>(id = __ldg(active + a)) <
                                     static_cast<unsigned long long>(P.nxy * P.nz);
    if (inside) unflatten(P, id, i, j, k);
    if (inside && !slab_node_miss(P, k)) {  // (a non-resident node is counted by the SL kernel)
        b = brick_of(i, j, k, nbx, nby);
        const double d_j = __ldg(dist + id);
        const double c_j = P.p == 1 ? 1.0 : d_j / energy_of(P);  // scale_factor (evolve.cpp:32-38)
        const double s = c_j * P.dt;
        const double spread = sqrt(fmax(0.0, c_j * P.delta * d_j * P.dt / P.pd));
        double m = fabs(s * grad_axis(P, dist, id, i, P.nx, 1));
        m = fmax(m, fabs(s * grad_axis(P, dist, id, j, P.ny, P.nx)));
        if (P.dim == 3) m = fmax(m, fabs(s * grad_axis(P, dist, id, k, P.nz, P.nxy)));
        // feet = base +- spread nu1 +- spread nu2 (evolve.cpp:96-101); per axis
        // |nu1_x| + |nu2_x| <= sqrt(2) for orthonormal nu1, nu2
        const double cells = (m + 1.4143 * spread) / P.dx;
        if (cells < static_cast<double>(kZtMaxReach)) {
            const unsigned fl = static_cast<unsigned>(floor(cells)), ce = static_cast<unsigned>(ceil(cells));
            r = (ce << 8) | fl;
        } else {
            r = (kZtMaxReach << 8) | kZtMaxReach;
        }
        r = r ? r : 1u;  // a brick with an active node is nonzero
    }
    // one atomic per (warp, brick): consecutive ids share bricks
    const unsigned same = __match_any_sync(0xffffffffu, b);
    const unsigned rmax = __reduce_max_sync(same, r);
    if (b >= 0 && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(same) - 1)) atomicMax(reach + b, rmax);
}

// one thread per active id; with P.n_dev (the device loop) the count is read
// from device memory and the grid strides over it (whole warps per round,
// as the warp-level reduction needs)
__global__ void zt_reach_kernel(SlParams P, const double* __restrict__ dist, const int64_t* __restrict__ active,
                                long long n, int nbx, int nby, unsigned* __restrict__ reach) {
    const long long first = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (P.n_dev == nullptr) {
        zt_reach_one(P, dist, active, first, n, nbx, nby, reach);
        return;
    }
    const long long nd = __ldg(P.n_dev);
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long a = first; a - static_cast<long long>(threadIdx.x & 31) < nd; a += stride)
        zt_reach_one(P, dist, active, a, nd, nbx, nby, reach);
}

// the largest foot displacement bound (cells, as zt_reach_kernel) over the
// ids: *max_bits = max of the non-negative double bits (integer order =
// double order). A z-slab sizes its halo planes from the max over ranks.
__global__ void reach_max_kernel(SlParams P, const double* __restrict__ dist, const int64_t* __restrict__ active,
                                 long long n, unsigned long long* __restrict__ max_bits) {
    const long long a = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long b = 0;
    if (a < n) {
        const long long id = __ldg(active + a);
        int i, j, k;
        unflatten(P, id, i, j, k);
        const double d_j = __ldg(dist + id);
        const double c_j = P.p == 1 ? 1.0 : d_j / energy_of(P);
        const double s = c_j * P.dt;
        const double spread = sqrt(fmax(0.0, c_j * P.delta * d_j * P.dt / P.pd));
        double m = fabs(s * grad_axis(P, dist, id, i, P.nx, 1));
        m = fmax(m, fabs(s * grad_axis(P, dist, id, j, P.ny, P.nx)));
        if (P.dim == 3) m = fmax(m, fabs(s * grad_axis(P, dist, id, k, P.nz, P.nxy)));
        double cells = (m + 1.4143 * spread) / P.dx;
        if (!(cells >= 0.0)) cells = 1e300;  // NaN / inf d: no finite halo covers it
        b = static_cast<unsigned long long>(__double_as_longlong(cells));
    }
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, b, off);
        b = o > b ? o : b;
    }
    if ((threadIdx.x & 31) == 0 && b) atomicMax(max_bits, b);
}

__device__ __forceinline__ int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// a brick b0 whose feet reach [i - rn, i + rp] reads table nodes x, y in
// [b0 - rn - 1, b0 + B - 1 + rp + 2] and z in [b0 - rn, b0 + B - 1 + rp + 1]
// (stencil cell-1 .. cell+2; table at z = cell, cell+1); cover[] = 1 on the
// bricks overlapping them (benign same-value races)
__global__ void zt_cover_kernel(const unsigned* __restrict__ reach, int nbx, int nby, int nbz,
                                unsigned char* __restrict__ cover) {
    const long long b = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= static_cast<long long>(nbx) * nby * nbz) return;
    const unsigned r = reach[b];
    if (r == 0) return;
    const int rn = static_cast<int>(r >> 8), rp = static_cast<int>(r & 0xffu);
    const int bi = static_cast<int>(b % nbx), bj = static_cast<int>((b / nbx) % nby),
              bk = static_cast<int>(b / (static_cast<long long>(nbx) * nby));
    const int lo = floor_div(-rn - 1, kZtBrick), hi = floor_div(kZtBrick + 1 + rp, kZtBrick);
    const int loz = floor_div(-rn, kZtBrick), hiz = floor_div(kZtBrick + rp, kZtBrick);
    for (int dk = loz; dk <= hiz; ++dk) {
        const int z = bk + dk;
        if (z < 0 || z >= nbz) continue;
        for (int dj = lo; dj <= hi; ++dj) {
            const int y = bj + dj;
            if (y < 0 || y >= nby) continue;
            for (int di = lo; di <= hi; ++di) {
                const int x = bi + di;
                if (x < 0 || x >= nbx) continue;
                cover[(static_cast<long long>(z) * nby + y) * nbx + x] = 1;
            }
        }
    }
}

// ---- the covered bricks from the band's state bytes (the device loop) ----
// The per-node reach above needs a pass over the active ids and their d
// stencils every iteration. Its bound is monotone in d_j and in |grad d|, and
// both are fields of the run, not of the iteration: brick_d_kernel keeps, per
// brick, bd[2b] = max d and bd[2b + 1] = max |centered_gradient(d)| component
// over the brick's nodes (once per d), and zt_cover_state_kernel bounds the
// reach of every brick holding an ACTIVE node (state byte 1) from them and
// this iteration's E. The bound is looser than the per-node one by the
// variation of d over a brick; like it, it only decides which bricks the table
// covers (speed), never a result.

// one thread per (brick, row of the brick): its 4 nodes' d and gradient
// components; the 16 rows of a brick sit in 16 consecutive lanes
__global__ void brick_d_kernel(SlParams P, const double* __restrict__ dist, int nbx, int nby, int nbz,
                               double* __restrict__ bd) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long b = t >> 4;
    const int r = static_cast<int>(t & 15);
    double dm = 0.0, gm = 0.0;
    const bool live = b < static_cast<long long>(nbx) * nby * nbz;
    if (live) {
        const int bi = static_cast<int>(b % nbx), bj = static_cast<int>((b / nbx) % nby),
                  bk = static_cast<int>(b / (static_cast<long long>(nbx) * nby));
        const int j = bj * kZtBrick + (r & 3), k = bk * kZtBrick + (r >> 2);
        if (j < P.ny && k < P.nz) {
            for (int q = 0; q < kZtBrick; ++q) {
                const int i = bi * kZtBrick + q;
                if (i >= P.nx) break;
                const long long id = (static_cast<long long>(k) * P.ny + j) * P.nx + i;
                dm = fmax(dm, __ldg(dist + id));
                gm = fmax(gm, fabs(grad_axis(P, dist, id, i, P.nx, 1)));
                gm = fmax(gm, fabs(grad_axis(P, dist, id, j, P.ny, P.nx)));
                if (P.dim == 3) gm = fmax(gm, fabs(grad_axis(P, dist, id, k, P.nz, P.nxy)));
            }
        }
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
        dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, off));
        gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, off));
    }
    if (live && r == 0) {
        bd[2 * b] = dm;
        bd[2 * b + 1] = gm;
    }
}

// one thread per brick (nx % 4 == 0, so a brick row is one aligned 4-byte
// word of the state): any ACTIVE node -> reach from (max d, max |grad d|, E)
// as zt_reach_one computes it per node -> cover as zt_cover_kernel
__global__ void zt_cover_state_kernel(SlParams P, const unsigned char* __restrict__ state,
                                      const double* __restrict__ bd, int nbx, int nby, int nbz,
                                      unsigned char* __restrict__ cover) {
    const long long b = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= static_cast<long long>(nbx) * nby * nbz) return;
    const int bi = static_cast<int>(b % nbx), bj = static_cast<int>((b / nbx) % nby),
              bk = static_cast<int>(b / (static_cast<long long>(nbx) * nby));
    unsigned any = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const int j = bj * kZtBrick + (r & 3), k = bk * kZtBrick + (r >> 2);
        if (j < P.ny && k < P.nz) {
            const unsigned w = __ldg(reinterpret_cast<const unsigned*>(
                state + (static_cast<long long>(k) * P.ny + j) * P.nx + bi * kZtBrick));
            const unsigned x = w ^ 0x01010101u;  // a zero byte where the state is ACTIVE (1)
            any |= (x - 0x01010101u) & ~x & 0x80808080u;
        }
    }
    if (!any) return;
    const double dmax = bd[2 * b], gmax = bd[2 * b + 1];
    const double c_j = P.p == 1 ? 1.0 : dmax / energy_of(P);
    const double sdt = c_j * P.dt;
    const double spread = sqrt(fmax(0.0, c_j * P.delta * dmax * P.dt / P.pd));
    const double cells = (fabs(sdt * gmax) + 1.4143 * spread) / P.dx;
    int rn = kZtMaxReach, rp = kZtMaxReach;
    if (cells < static_cast<double>(kZtMaxReach)) {
        rp = static_cast<int>(floor(cells));
        rn = static_cast<int>(ceil(cells));
    }
    const int lo = floor_div(-rn - 1, kZtBrick), hi = floor_div(kZtBrick + 1 + rp, kZtBrick);
    const int loz = floor_div(-rn, kZtBrick), hiz = floor_div(kZtBrick + rp, kZtBrick);
    for (int dk = loz; dk <= hiz; ++dk) {
        const int z = bk + dk;
        if (z < 0 || z >= nbz) continue;
        for (int dj = lo; dj <= hi; ++dj) {
            const int y = bj + dj;
            if (y < 0 || y >= nby) continue;
            for (int di = lo; di <= hi; ++di) {
                const int x = bi + di;
                if (x < 0 || x >= nbx) continue;
                cover[(static_cast<long long>(z) * nby + y) * nbx + x] = 1;
            }
        }
    }
}

// list = the covered bricks (any order)
__global__ void zt_list_kernel(const unsigned char* __restrict__ cover, long long nbricks,
                               unsigned* __restrict__ list, unsigned* __restrict__ count) {
    const long long b = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool hit = b < nbricks && cover[b] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(count, static_cast<unsigned>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (hit) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<unsigned>(b);
}

// the table entries of the listed bricks: one thread per (x, y) column of a
// brick, marching up its kZtBrick planes with a sliding window of phi
__global__ void __launch_bounds__(256) zt_fill_kernel(SlParams P, const double* __restrict__ phi,
                                                      const unsigned* __restrict__ list,
                                                      const unsigned* __restrict__ count, int nbx, int nby,
                                                      double* __restrict__ zt, double* __restrict__ zc,
                                                      unsigned* __restrict__ bad) {
    constexpr int kCols = kZtBrick * kZtBrick;
    const unsigned nb = *count;
    const unsigned per_cta = blockDim.x / kCols;
    const int c = threadIdx.x % kCols;
    bool ok = true;
    for (unsigned q = blockIdx.x * per_cta + threadIdx.x / kCols; q < nb; q += gridDim.x * per_cta) {
        const unsigned b = __ldg(list + q);
        const int bi = static_cast<int>(b % nbx), bj = static_cast<int>((b / nbx) % nby),
                  bk = static_cast<int>(b / (static_cast<unsigned>(nbx) * nby));
        const int i = bi * kZtBrick + c % kZtBrick, j = bj * kZtBrick + c / kZtBrick;
        if (i >= P.nx || j >= P.ny) continue;
        // planes [k0, k1): interior planes whose z neighbours are resident
        // (whole grid: 1 .. nz-2; slab mode: z_base+1 .. z_base+z_planes-2)
        const int top = P.z_base + P.z_planes;
        const int k0 = max(bk * kZtBrick, P.z_base + 1), k1 = min(bk * kZtBrick + kZtBrick, top - 1);
        if (k0 >= k1) continue;
        long long id = (static_cast<long long>(k0) * P.ny + j) * P.nx + i;
        double vm = __ldg(phi + id - P.nxy), v0 = __ldg(phi + id), vp = __ldg(phi + id + P.nxy);
        for (int k = k0; k < k1; ++k, id += P.nxy) {
            const double vpp = k + 2 < top ? __ldg(phi + id + 2 * P.nxy) : 0.0;
            double sd, S, Y;  // weno1_fast's sdl / sdr and its alpha denominator
            bool good = zt_node_terms(P, vm, v0, vp, sd, S, Y);
            const double c1 = vp - vm;                      // d1
            const double e2 = -3.0 * v0 + 4.0 * vp - vpp;  // d2
            if (k + 2 < top) good = good & halvable(c1) & halvable(e2);  // else e2 is never read (no stencil has K = k)
            ok = ok & good;
            reinterpret_cast<double4*>(zt)[id] = make_double4(sd, S, Y, v0);
            reinterpret_cast<double2*>(zc)[id] = make_double2(c1, e2);
            vm = v0;
            v0 = vp;
            vp = vpp;
        }
    }
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// out[ids] = phi[ids]: re-establishes "out equals phi off the active set"
// after the previous step wrote out (or after a swap) without the O(N) copy.
__global__ void resync_kernel(const double* __restrict__ phi, double* __restrict__ out,
                              const int64_t* __restrict__ ids, long long n, long long n_nodes) {
    const long long a = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const long long id = __ldg(ids + a);
    if (static_cast<unsigned long long>(id) >= static_cast<unsigned long long>(n_nodes)) return;  // (reported by the step)
    out[id] = __ldg(phi + id);
}

// counts ids outside [0, n_nodes)
__global__ void check_ids_kernel(const int64_t* __restrict__ ids, long long n, long long n_nodes,
                                 unsigned long long* __restrict__ bad) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool wrong = i < n && static_cast<unsigned long long>(__ldg(ids + i)) >= static_cast<unsigned long long>(n_nodes);
    const unsigned b = __ballot_sync(0xffffffffu, wrong);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, static_cast<unsigned long long>(__popc(b)));
}

// counts positions where the id list is not strictly ascending
__global__ void check_sorted_kernel(const int64_t* __restrict__ ids, long long n, unsigned long long* __restrict__ bad) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool wrong = i + 1 < n && !(__ldg(ids + i) < __ldg(ids + i + 1));
    const unsigned b = __ballot_sync(0xffffffffu, wrong);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, static_cast<unsigned long long>(__popc(b)));
}

// Self-test of div_const against the hardware IEEE division: a splitmix64
// stream of bit patterns (all exponents, signs, zeros, subnormals, inf/NaN)
// divided by c; counts quotients whose bits differ.
__global__ void div_selftest_kernel(double c, double rc, unsigned long long seed, long long n,
                                    unsigned long long* mismatches) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long bad = 0;
    for (long long i = t; i < n; i += static_cast<long long>(gridDim.x) * blockDim.x) {
        unsigned long long z = seed + 0x9E3779B97F4A7C15ULL * static_cast<unsigned long long>(i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        double a = __longlong_as_double(static_cast<long long>(z));
        if ((i & 3) == 1) a = static_cast<double>(z >> 11) * 0x1.0p-53;  // [0,1): the common case
        if ((i & 3) == 2) a = (static_cast<double>(z >> 11) * 0x1.0p-53) * 1e-3;
        const double fast = div_const(a, c, rc, 1);
        const double ref = a / c;
        const bool same = __double_as_longlong(fast) == __double_as_longlong(ref) || (isnan(fast) && isnan(ref));
        bad += same ? 0 : 1;
    }
    if (bad) atomicAdd(mismatches, bad);
}

// Differential self-test of the exact fast WENO forms against weno1 (the
// plain IEEE operators, interp.cpp:16-33): for n pseudo-random stencils
// (vm, v0, vp, vpp) and abscissae theta, weno1_fast must return weno1's bits
// whenever its guards pass (theta_in_range and the in-function checks), and
// weno1_zt fed the table terms zt_fill_kernel would store (zt_node_terms of
// K = v0 and K + 1 = vp, d1, d2) must too whenever the fill's checks and
// theta_in_range pass. Sample classes (i mod 4): 0 smooth lines at random
// scales 2^-60..2^20; 1 raw random bit patterns (every exponent, zeros,
// subnormals, inf, NaN); 2 lines whose squared second differences sit at the
// range guards 2^-700 / 2^200 (+-few ulp) and differences at the halving
// guard 2^-1021; 3 tiny/subnormal/zero differences. theta is drawn from
// [-0.7, 1.7] or, one sample in four, from the guard values -1/2, 0, -0, 3/2,
// +-2^-510, +-2^-511 and their neighbours.
// counts: [0] fast taken, [1] fast mismatches, [2] table taken, [3] table
// mismatches.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double unit01(unsigned long long z) { return static_cast<double>(z >> 11) * 0x1.0p-53; }

__device__ __forceinline__ double nudge(double x, int ulps) {  // x moved by `ulps` units in the last place
    return __longlong_as_double(__double_as_longlong(x) + ulps);
}

// sample i of the self-test stream: a stencil v[4] and an abscissa t
__device__ __forceinline__ void weno_sample(unsigned long long seed, long long i, double* v, double& t) {
    unsigned long long z = seed + 0x9E3779B97F4A7C15ULL * static_cast<unsigned long long>(i + 1);
    auto next = [&z]() {
        z += 0x9E3779B97F4A7C15ULL;
        return mix64(z);
    };
    const int cls = static_cast<int>(i & 3);
    if (cls == 0) {  // smooth: quadratic + small noise, random scale
        const double sc = ldexp(1.0, static_cast<int>(next() % 81) - 60);
        const double a0 = unit01(next()) - 0.5, a1 = unit01(next()) - 0.5, a2 = (unit01(next()) - 0.5) * 0.1;
        for (int q = 0; q < 4; ++q)
            v[q] = sc * (a0 + a1 * (q - 1) + a2 * (q - 1) * (q - 1) + 1e-6 * (unit01(next()) - 0.5));
    } else if (cls == 1) {  // raw bit patterns
        for (int q = 0; q < 4; ++q) v[q] = __longlong_as_double(static_cast<long long>(next()));
    } else if (cls == 2) {  // at the guards
        const unsigned long long r = next();
        const int ulps = static_cast<int>(r % 9) - 4;
        const int which = static_cast<int>((r >> 8) % 6);
        const double s = (r >> 16) & 1 ? -1.0 : 1.0;
        for (int q = 0; q < 4; ++q) v[q] = 0.0;
        // sd^2 = 2^-700 <=> |sd| = 2^-350; sd^2 = 2^200 <=> |sd| = 2^100; d/2 exact down to 2^-1021
        const double mag = which == 0 ? 0x1.0p-350 : which == 1 ? 0x1.0p100 : which == 2 ? 0x1.0p-1021 : which == 3
            ? 0x1.6a09e667f3bcdp-351 /* sqrt(2^-701) */ : which == 4 ? 0x1.6a09e667f3bcdp+99 : 0x1.0p-1022;
        const int slot = static_cast<int>((r >> 20) & 3);
        v[slot] = s * nudge(mag, ulps);
        if ((r >> 24) & 1) v[(slot + 1) & 3] = 0.5 * v[slot];
    } else {  // tiny / subnormal / zero differences around a base value
        const double base = unit01(next()) - 0.5;
        for (int q = 0; q < 4; ++q) {
            const unsigned long long r = next();
            v[q] = (r & 3) == 0 ? base : (r & 3) == 1 ? 0.0 : (r & 3) == 2 ? nudge(base, static_cast<int>(r % 5) - 2)
                                                                           : __longlong_as_double(static_cast<long long>(r >> 12));
        }
    }
    {
        const unsigned long long r = next();
        if ((r & 3) != 0) {
            t = -0.7 + 2.4 * unit01(next());
        } else {
            const double special[8] = {-0.5, 0.0, -0.0, 1.5, 0x1.0p-510, -0x1.0p-510, 0x1.0p-511, -0x1.0p-511};
            t = special[(r >> 2) & 7];
            if ((r >> 5) & 1) t = nudge(t, ((r >> 6) & 1) ? 1 : -1);
            if (t == 0.0 && ((r >> 7) & 1)) t = __longlong_as_double(static_cast<long long>((r >> 8) & 0xfffff));
        }
    }
}

__global__ void weno_selftest_kernel(SlParams P, unsigned long long seed, long long n,
                                     unsigned long long* __restrict__ counts) {
    unsigned long long c[4] = {0, 0, 0, 0};
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        double v[4], t;
        weno_sample(seed, i, v, t);
        const AxisW w = axis_weights(P, t);
        const double ref = weno1(P, w, v[0], v[1], v[2], v[3]);
        bool ok = theta_in_range(t);
        const double fast = weno1_fast(P, w, v[0], v[1], v[2], v[3], ok);
        if (ok) {
            ++c[0];
            if (__double_as_longlong(fast) != __double_as_longlong(ref)) ++c[1];
        }
        double sdK, SK, YK, sdK1, SK1, YK1;
        bool good = zt_node_terms(P, v[0], v[1], v[2], sdK, SK, YK);
        good = good & zt_node_terms(P, v[1], v[2], v[3], sdK1, SK1, YK1);
        const double c1 = v[2] - v[0], e2 = -3.0 * v[1] + 4.0 * v[2] - v[3];
        good = good & halvable(c1) & halvable(e2) & theta_in_range(t);
        if (good) {
            ++c[2];
            const double zt = weno1_zt(w, make_double4(sdK, SK, YK, v[1]), make_double4(sdK1, SK1, YK1, v[2]),
                                       make_double2(c1, e2));
            if (__double_as_longlong(zt) != __double_as_longlong(ref)) ++c[3];
        }
    }
    for (int q = 0; q < 4; ++q)
        if (c[q]) atomicAdd(counts + q, c[q]);
}

// one warp per run of packed values (host_pack.h)
__global__ void scatter_runs_kernel(const double* __restrict__ packed, const long long* __restrict__ desc,
                                    long long r0, long long r1, long long vend, double* __restrict__ field) {
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long long r = r0 + ((static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); r < r1;
         r += nw) {
        const long long dst = desc[2 * r], src = desc[2 * r + 1];
        const long long len = (r + 1 < r1 ? desc[2 * r + 3] : vend) - src;
        for (long long l = lane; l < len; l += 32) field[dst + l] = packed[src + l];
    }
}

// res[t] = field[ids[t]]: the updated values of one chunk, packed for the D2H
__global__ void gather_ids_kernel(const double* __restrict__ field, const int64_t* __restrict__ ids, long long n,
                                  double* __restrict__ res, long long n_nodes) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long id = ids[t];
    res[t] = static_cast<unsigned long long>(id) < static_cast<unsigned long long>(n_nodes) ? field[id] : 0.0;
}

}  // namespace lsr_dev

using namespace lsr_dev;

cudaError_t launch_gather_ids(const double* field, const int64_t* ids, long long n, double* res, long long n_nodes,
                              cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    gather_ids_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(field, ids, n, res, n_nodes);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_scatter_runs(const double* packed, const long long* desc, long long r0, long long r1,
                                long long vend, double* field, cudaStream_t stream) {
    if (r1 <= r0) return cudaSuccess;
    const long long warps = r1 - r0;
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((warps + 7) / 8, 148LL * 16));
    scatter_runs_kernel<<<blocks, 256, 0, stream>>>(packed, desc, r0, r1, vend, field);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_div_selftest(double c, double rc, unsigned long long seed, long long n,
                                unsigned long long* mismatches) {
    div_selftest_kernel<<<148 * 8, 256>>>(c, rc, seed, n, mismatches);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_weno_selftest(const SlParams& P, unsigned long long seed, long long n, unsigned long long* counts) {
    weno_selftest_kernel<<<148 * 8, 256>>>(P, seed, n, counts);
    lsr_note_launch();
    return cudaGetLastError();
}

template <bool TAIL>
static void sl_launch_form(const SlParams& P, int kind, const double* phi, const double* dist, const int64_t* active,
                           long long n_active, double* out, unsigned long long* bad, long long base,
                           unsigned blocks, unsigned blocks_w3, cudaStream_t stream) {
    if (P.dim == 2) {
        if (kind == 0)
            sl_step_kernel<2, 0, TAIL><<<blocks, kSlThreads, 0, stream>>>(P, phi, dist, active, n_active, out, bad, base);
        else
            sl_step_kernel<2, 1, TAIL><<<blocks, kSlThreads, 0, stream>>>(P, phi, dist, active, n_active, out, bad, base);
    } else if (kind == 0) {
        sl_step_kernel<3, 0, TAIL><<<blocks, kSlThreads, 0, stream>>>(P, phi, dist, active, n_active, out, bad, base);
    } else if (LSR_ZTAB && P.ztab != nullptr) {
        sl_step_zt_kernel<TAIL><<<blocks_w3, kSlThreadsW3, 0, stream>>>(P, phi, dist, active, n_active, out, bad, base);
    } else {
        sl_step_kernel<3, 1, TAIL><<<blocks, kSlThreads, 0, stream>>>(P, phi, dist, active, n_active, out, bad, base);
    }
    lsr_note_launch();
}

cudaError_t launch_sl_step(const SlParams& P, int kind, const double* phi, const double* dist,
                           const int64_t* active, long long n_active, double* out, unsigned long long* bad,
                           cudaStream_t stream) {
    if (P.n_dev != nullptr) {
        // device count (the loop): n_active is the estimate the launch covers;
        // the tail launch takes any ids beyond it
        const long long est = n_active > 0 ? n_active : 1;
        const bool w3 = P.dim == 3 && kind != 0 && LSR_ZTAB && P.ztab != nullptr;
        const int T = w3 ? kSlThreadsW3 : kSlThreads;
        const long long blk = (est + T - 1) / T;
        sl_launch_form<false>(P, kind, phi, dist, active, est, out, bad, 0, static_cast<unsigned>(blk),
                              static_cast<unsigned>(blk), stream);
        sl_launch_form<true>(P, kind, phi, dist, active, est, out, bad, blk * T, 148u * 2u, 148u * 2u, stream);
        return cudaGetLastError();
    }
    if (n_active <= 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((n_active + kSlThreads - 1) / kSlThreads);
    const unsigned blocks_w3 = static_cast<unsigned>((n_active + kSlThreadsW3 - 1) / kSlThreadsW3);
    sl_launch_form<false>(P, kind, phi, dist, active, n_active, out, bad, 0, blocks, blocks_w3, stream);
    return cudaGetLastError();
}

cudaError_t launch_zt_bricks(const SlParams& P, const double* dist, const int64_t* active, long long n_active,
                             const ZtBuffers& Z, cudaStream_t stream) {
    const int nbx = (P.nx + kZtBrick - 1) / kZtBrick, nby = (P.ny + kZtBrick - 1) / kZtBrick,
              nbz = (P.nz + kZtBrick - 1) / kZtBrick;
    const long long nbricks = static_cast<long long>(nbx) * nby * nbz;
    cudaError_t e = cudaMemsetAsync(Z.mark, 0, static_cast<size_t>(nbricks), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(Z.reach, 0, sizeof(unsigned) * static_cast<size_t>(nbricks), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(Z.count, 0, sizeof(unsigned), stream);
    if (e != cudaSuccess || (n_active <= 0 && P.n_dev == nullptr)) return e;
    const unsigned gb = static_cast<unsigned>((nbricks + 255) / 256);
    // device count (P.n_dev): n_active is an estimate, the grid strides past it
    const long long est = n_active > 0 ? n_active : 1;
    zt_reach_kernel<<<static_cast<unsigned>((est + 255) / 256), 256, 0, stream>>>(P, dist, active, n_active, nbx, nby,
                                                                                 Z.reach);
    zt_cover_kernel<<<gb, 256, 0, stream>>>(Z.reach, nbx, nby, nbz, Z.mark);
    zt_list_kernel<<<gb, 256, 0, stream>>>(Z.mark, nbricks, Z.list, Z.count);
    for (int r = 0; r < 3; ++r) lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_brick_d(const SlParams& P, const double* dist, double* bd, cudaStream_t stream) {
    const int nbx = (P.nx + kZtBrick - 1) / kZtBrick, nby = (P.ny + kZtBrick - 1) / kZtBrick,
              nbz = (P.nz + kZtBrick - 1) / kZtBrick;
    const long long threads = 16LL * nbx * nby * nbz;
    brick_d_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(P, dist, nbx, nby, nbz, bd);
    lsr_note_launch();
    return cudaGetLastError();
}

// the covered bricks of the band whose state bytes are `state` (ACTIVE = 1);
// needs nx % 4 == 0 and bd from launch_brick_d of the same d
cudaError_t launch_zt_bricks_state(const SlParams& P, const unsigned char* state, const double* bd, const ZtBuffers& Z,
                                   cudaStream_t stream) {
    const int nbx = (P.nx + kZtBrick - 1) / kZtBrick, nby = (P.ny + kZtBrick - 1) / kZtBrick,
              nbz = (P.nz + kZtBrick - 1) / kZtBrick;
    const long long nbricks = static_cast<long long>(nbx) * nby * nbz;
    cudaError_t e = cudaMemsetAsync(Z.mark, 0, static_cast<size_t>(nbricks), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(Z.count, 0, sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    const unsigned gb = static_cast<unsigned>((nbricks + 255) / 256);
    zt_cover_state_kernel<<<gb, 256, 0, stream>>>(P, state, bd, nbx, nby, nbz, Z.mark);
    zt_list_kernel<<<gb, 256, 0, stream>>>(Z.mark, nbricks, Z.list, Z.count);
    for (int r = 0; r < 2; ++r) lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_zt_fill(const SlParams& P, const double* phi, const ZtBuffers& Z, cudaStream_t stream) {
    const int nbx = (P.nx + kZtBrick - 1) / kZtBrick, nby = (P.ny + kZtBrick - 1) / kZtBrick;
    cudaError_t e = cudaMemsetAsync(Z.count + 1, 0, sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    zt_fill_kernel<<<148 * 8, 256, 0, stream>>>(P, phi, Z.list, Z.count, nbx, nby, Z.zt, Z.zc, Z.count + 1);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_check_sorted(const int64_t* ids, long long n, unsigned long long* bad, cudaStream_t stream) {
    if (n <= 1) return cudaSuccess;
    check_sorted_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(ids, n, bad);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_reach_max(const SlParams& P, const double* dist, const int64_t* active, long long n,
                             unsigned long long* max_bits, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    reach_max_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(P, dist, active, n, max_bits);
    lsr_note_launch();
    return cudaGetLastError();
}

// the brick grouping of an active set for the TMA brick step
cudaError_t launch_box_bricks(const SlParams& P, const int64_t* active, long long n, const BoxBuffers& X,
                              long long* n_listed, cudaStream_t stream) {
    const int nbx = (P.nx + kSlBrick - 1) / kSlBrick, nby = (P.ny + kSlBrick - 1) / kSlBrick,
              nbz = (P.nz + kSlBrick - 1) / kSlBrick;
    const long long nb = static_cast<long long>(nbx) * nby * nbz;
    cudaError_t e = cudaMemsetAsync(X.count, 0, sizeof(unsigned) * (nb + 1), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(X.cursor, 0, sizeof(unsigned) * nb, stream);
    if (e != cudaSuccess) return e;
    *n_listed = 0;
    if (n <= 0) return cudaSuccess;
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    box_count_kernel<<<g, 256, 0, stream>>>(P, active, n, nbx, nby, X.count);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, X.count, X.off, static_cast<int>(nb + 1));
    if (tb > X.tmp_bytes) return cudaErrorMemoryAllocation;
    e = cub::DeviceScan::ExclusiveSum(X.tmp, tb, X.count, X.off, static_cast<int>(nb + 1), stream);
    if (e != cudaSuccess) return e;
    box_scatter_kernel<<<g, 256, 0, stream>>>(P, active, n, nbx, nby, X.off, X.cursor, X.ids);
    e = lsr_compact::compact(NonEmpty{X.count}, lsr_compact::Identity{}, nb, X.list, X.d_listed,
                             static_cast<char*>(X.tmp) + X.tmp_bytes / 2, X.tmp_bytes / 2, stream);
    if (e != cudaSuccess) return e;
    for (int r = 0; r < 4; ++r) lsr_note_launch();
    long long h = 0;
    e = cudaMemcpyAsync(&h, X.d_listed, sizeof h, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    *n_listed = h;
    return e;
}

size_t box_tmp_bytes(long long nbricks) {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, static_cast<unsigned*>(nullptr), static_cast<unsigned*>(nullptr),
                                  static_cast<int>(nbricks + 1));
    const size_t c = lsr_compact::scratch_bytes(nbricks);
    return 2 * ((std::max(tb + 256, c) + 255) / 256 * 256);  // two 256-byte-aligned halves
}

static bool box_tensor_map(const SlParams& P, const double* phi, CUtensorMap* map) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode || (P.nx * 8) % 16 != 0) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(P.nx), static_cast<cuuint64_t>(P.ny),
                                static_cast<cuuint64_t>(P.nz)};
    const cuuint64_t str[2] = {static_cast<cuuint64_t>(P.nx) * 8, static_cast<cuuint64_t>(P.nxy) * 8};
    const cuuint32_t box[3] = {kBoxEX, kBoxEY, kBoxEZ};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(phi), dims, str, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// false (nothing launched) when the tensor map cannot be made
bool launch_sl_step_box(const SlParams& P, const double* phi, const double* dist, const BoxBuffers& X,
                        long long n_listed, long long n_ids, double* out, unsigned long long* bad, cudaStream_t stream) {
    CUtensorMap map;
    if (!box_tensor_map(P, phi, &map)) return false;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        cudaFuncSetAttribute(sl_step_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBoxBytes + 128);
        attr_dev = dev;
    }
    if (n_listed <= 0) return true;
    const int nbx = (P.nx + kSlBrick - 1) / kSlBrick, nby = (P.ny + kSlBrick - 1) / kSlBrick;
    sl_step_box_kernel<<<static_cast<unsigned>(n_listed), kBoxThreads, kBoxBytes + 128, stream>>>(
        map, P, phi, dist, X.list, X.off, n_listed, X.ids, n_ids, nbx, nby, out, bad);
    lsr_note_launch();
    return true;
}

cudaError_t launch_check_ids(const int64_t* ids, long long n, long long n_nodes, unsigned long long* bad,
                             cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    check_ids_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(ids, n, n_nodes, bad);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_resync(const double* phi, double* out, const int64_t* ids, long long n, long long n_nodes,
                          cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    resync_kernel<<<blocks, 256, 0, stream>>>(phi, out, ids, n, n_nodes);
    lsr_note_launch();
    return cudaGetLastError();
}
