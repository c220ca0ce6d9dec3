// distance.cu — point-cloud preprocessing on the GPU:
// the unsigned distance d of lsr::build_distance_field
// (/root/reference/proj/src/distance.cpp:144-148), bit-identical to the
// reference.
//
//  * SpatialHash (cloud.cpp:390-452): the same uniform bins (geometry fixed
//    on the host with the reference's expressions), built with a counting
//    sort on the device. nearest_distance keeps the reference's shell loop
//    and break rule, so the set of examined points at each shell end — and
//    hence the min of the identical dot(diff,diff) terms — is the same.
//  * seed_exact_distance (distance.cpp:8-52): pass 1 flags the 4^dim node
//    block around each point's cell (all writers store 1), pass 2 evaluates
//    the exact NN distance at flagged nodes.
//  * fast_sweep (distance.cpp:72-142): Gauss–Seidel over the 2^dim orderings
//    as hyperplane sweeps. In ordering (+,+,+) the serial loop updates node
//    (i,j,k) after its -1 neighbours and before its +1 neighbours; sweeping
//    the hyperplanes i'+j'+k' = s in increasing s (with mirrored indices for
//    the other orderings) gives every node exactly the same inputs, and
//    nodes of one hyperplane are independent. max_change is a max (order
//    free), accumulated with an integer atomicMax on the non-negative bits.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>

#include <cub/cub.cuh>

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "lsr_cuda.h"
#include "prep_launch.h"

namespace {

struct HashP {
    int dim;
    double lox, loy, loz;
    double cell;
    int bx, by, bz;
};

__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ int iclamp(int v, int lo, int hi) { return v < lo ? lo : (hi < v ? hi : v); }

// bin_of (cloud.cpp:405-412)
__device__ __forceinline__ int bin_of(const HashP& H, const double* p) {
    int b[3] = {0, 0, 0};
    const double lo[3] = {H.lox, H.loy, H.loz};
    const int nb[3] = {H.bx, H.by, H.bz};
    for (int d = 0; d < H.dim; ++d) {
        b[d] = static_cast<int>((p[d] - lo[d]) / H.cell);
        b[d] = iclamp(b[d], 0, nb[d] - 1);
    }
    return (b[2] * H.by + b[1]) * H.bx + b[0];
}

__global__ void count_bins(HashP H, const double* __restrict__ pts, long long n, int* __restrict__ counts,
                           int* __restrict__ bin_id) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = bin_of(H, pts + 3 * i);
    bin_id[i] = b;
    atomicAdd(counts + b, 1);
}

__global__ void scatter_bins(const int* __restrict__ bin_id, long long n, int* __restrict__ cursor,
                             int* __restrict__ entries) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    entries[atomicAdd(cursor + bin_id[i], 1)] = static_cast<int>(i);
}

// SpatialHash::nearest_distance (cloud.cpp:420-452)
__device__ double nearest_distance(const HashP& H, const double* __restrict__ pts, const int* __restrict__ starts,
                                   const int* __restrict__ entries, double qx, double qy, double qz,
                                   int exclude = -1) {
    const double q[3] = {qx, qy, qz};
    const double lo[3] = {H.lox, H.loy, H.loz};
    const int nb[3] = {H.bx, H.by, H.bz};
    int bq[3] = {0, 0, 0};
    int rad_max = 0;
    for (int d = 0; d < H.dim; ++d) {
        bq[d] = static_cast<int>(floor((q[d] - lo[d]) / H.cell));
        rad_max = max(rad_max, max(bq[d], nb[d] - 1 - bq[d]));
    }
    double best2 = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    for (int rad = 0; rad <= rad_max + 1; ++rad) {
        if (rad > 0 && best2 <= ((rad - 1) * H.cell) * ((rad - 1) * H.cell)) break;
        const int zlo = H.dim == 3 ? bq[2] - rad : 0;
        const int zhi = H.dim == 3 ? bq[2] + rad : 0;
        for (int bz = max(0, zlo); bz <= min(nb[2] - 1, zhi); ++bz) {
            for (int by = max(0, bq[1] - rad); by <= min(nb[1] - 1, bq[1] + rad); ++by) {
                const int cyz = max(abs(by - bq[1]), abs(bz - bq[2]));
                for (int bx = max(0, bq[0] - rad); bx <= min(nb[0] - 1, bq[0] + rad); ++bx) {
                    if (max(abs(bx - bq[0]), cyz) != rad) continue;
                    const int b = (bz * nb[1] + by) * nb[0] + bx;
                    for (int e = starts[b]; e < starts[b + 1]; ++e) {
                        if (entries[e] == exclude) continue;
                        const double* p = pts + 3 * static_cast<long long>(entries[e]);
                        const double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
                        best2 = dmin(best2, dx * dx + dy * dy + dz * dz);  // dot(diff, diff)
                    }
                }
            }
        }
    }
    return sqrt(best2);
}

struct GridP {
    int dim, nx, ny, nz;
    long long nxy;
    double ox, oy, oz, dx;
};

// seed pass 1 (distance.cpp:25-39): flag the 4^dim block around each point's cell
__global__ void seed_flag(GridP G, const double* __restrict__ pts, long long n, unsigned char* __restrict__ exact) {
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double* p = pts + 3 * q;
    // locate_cell (grid.cpp:39-47); the host has checked Grid::contains
    const double o[3] = {G.ox, G.oy, G.oz};
    const int nn[3] = {G.nx, G.ny, G.nz};
    int c[3] = {0, 0, 0};
    for (int d = 0; d < G.dim; ++d) c[d] = iclamp(static_cast<int>(floor((p[d] - o[d]) / G.dx)), 0, nn[d] - 2);
    const int kz = G.dim == 3 ? 1 : 0;
    for (int dk = -kz; dk <= 2 * kz; ++dk)
        for (int dj = -1; dj <= 2; ++dj)
            for (int di = -1; di <= 2; ++di) {
                const int i = c[0] + di, j = c[1] + dj, k = c[2] + dk;
                if (i < 0 || j < 0 || k < 0 || i >= G.nx || j >= G.ny || k >= G.nz) continue;
                exact[(static_cast<long long>(k) * G.ny + j) * G.nx + i] = 1;
            }
}

// seed pass 2 (distance.cpp:42-50) + the sentinel fill of every other node
__global__ void seed_values(GridP G, HashP H, const double* __restrict__ pts, const int* __restrict__ starts,
                            const int* __restrict__ entries, const unsigned char* __restrict__ exact, double sentinel,
                            double* __restrict__ d) {
    const long long id = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= G.nxy * G.nz) return;
    if (!exact[id]) {
        d[id] = sentinel;
        return;
    }
    const int i = static_cast<int>(id % G.nx);
    const int j = static_cast<int>((id / G.nx) % G.ny);
    const int k = static_cast<int>(id / G.nxy);
    d[id] = nearest_distance(H, pts, starts, entries, G.ox + i * G.dx, G.oy + j * G.dx, G.oz + k * G.dx);
}

__global__ void any_below(const double* __restrict__ d, long long n, double sentinel, int* __restrict__ flag) {
    for (long long id = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; id < n;
         id += static_cast<long long>(gridDim.x) * blockDim.x)
        if (d[id] < sentinel) {
            *flag = 1;
            return;
        }
}

// eikonal_update (distance.cpp:57-68)
__device__ __forceinline__ double eikonal_update(const double* a, int m, double h) {
    double x = a[0] + h;
    if (m >= 2 && x > a[1]) {
        x = 0.5 * (a[0] + a[1] + sqrt(2.0 * h * h - (a[0] - a[1]) * (a[0] - a[1])));
        if (m >= 3 && x > a[2]) {
            const double s = a[0] + a[1] + a[2];
            const double s2 = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
            x = (s + sqrt(s * s - 3.0 * (s2 - h * h))) / 3.0;
        }
    }
    return x;
}

// one hyperplane i'+j'+k' = s of ordering `ord` (update_node, distance.cpp:86-116)
__global__ void sweep_plane(GridP G, int ord, int s, int k_lo, int k_cnt, double sentinel,
                            const unsigned char* __restrict__ exact, double* __restrict__ d,
                            unsigned long long* __restrict__ max_change) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int kp = k_lo + t / G.ny;  // mirrored k', j'
    const int jp = t % G.ny;
    if (t / G.ny >= k_cnt) return;
    const int ip = s - jp - kp;
    if (ip < 0 || ip >= G.nx) return;
    const int i = (ord & 1) ? G.nx - 1 - ip : ip;
    const int j = (ord & 2) ? G.ny - 1 - jp : jp;
    const int k = (ord & 4) ? G.nz - 1 - kp : kp;
    const long long id = (static_cast<long long>(k) * G.ny + j) * G.nx + i;
    if (exact[id]) return;
    double a[3];
    int m = 0;
    {
        double best = sentinel;
        if (i > 0) best = dmin(best, d[id - 1]);
        if (i < G.nx - 1) best = dmin(best, d[id + 1]);
        if (best < sentinel) a[m++] = best;
    }
    {
        double best = sentinel;
        if (j > 0) best = dmin(best, d[id - G.nx]);
        if (j < G.ny - 1) best = dmin(best, d[id + G.nx]);
        if (best < sentinel) a[m++] = best;
    }
    if (G.dim == 3) {
        double best = sentinel;
        if (k > 0) best = dmin(best, d[id - G.nxy]);
        if (k < G.nz - 1) best = dmin(best, d[id + G.nxy]);
        if (best < sentinel) a[m++] = best;
    }
    if (m == 0) return;
    // std::sort of <= 3 values: the sorted sequence is unique
    if (m >= 2 && a[1] < a[0]) { const double t0 = a[0]; a[0] = a[1]; a[1] = t0; }
    if (m == 3) {
        if (a[2] < a[1]) { const double t1 = a[1]; a[1] = a[2]; a[2] = t1; }
        if (a[1] < a[0]) { const double t0 = a[0]; a[0] = a[1]; a[1] = t0; }
    }
    const double v = d[id];
    const double cand = eikonal_update(a, m, G.dx);
    if (cand < v) {
        d[id] = cand;
        const double change = v - cand;
        atomicMax(max_change, static_cast<unsigned long long>(__double_as_longlong(change)));
    }
}

// Tiled wavefront form of one 3d Gauss-Seidel sweep (fast_sweep's inner
// triple loop for one ordering, distance.cpp:80-139). In the mirrored
// coordinates of the ordering every update reads its -1 neighbours already
// updated and its +1 neighbours not yet updated. Tiles of kTile^3 nodes whose
// mirrored tile coordinates sum to S run in the S-th launch (their -1 face
// neighbours finished at S-1, their +1 ones start at S+1); inside a tile one
// CTA walks the kTile*3-2 inner planes in order, one node per thread and
// plane, with the tile and a one-node halo in shared memory. Every node sees
// exactly the neighbour values the lexicographic sweep gives it, so the
// result is bit-identical, with 3*n/kTile launches per sweep instead of 3*n.
#ifndef LSR_SWEEP_TILE
#define LSR_SWEEP_TILE 16
#endif
constexpr int kTile = LSR_SWEEP_TILE;
#ifndef LSR_SWEEP_TMA_FLAGS
#define LSR_SWEEP_TMA_FLAGS 1
#endif
constexpr int kTH = kTile + 2;   // y and z extent of the box + halo
constexpr int kTHX = kTile + 4;  // x extent: the box starts two nodes early so its start stays 16-byte aligned

// dynamic shared memory of one tile: the box + halo of d, the box's exact
// flags, the TMA mbarrier and the per-warp maxima
constexpr int kSdBytes = kTH * kTH * kTHX * 8;
constexpr int kSdOff = 128;  // after the mbarrier and the per-warp maxima; TMA destinations are 128-byte aligned
constexpr int kSxOff = kSdOff + (kSdBytes + 127) / 128 * 128;
constexpr int kSxBytes = kTile * kTile * kTile;
constexpr int kTileSmem = kSxOff + kSxBytes;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// With kTma the box + halo of d (kTH x kTH x kTHX doubles) and the box's
// exact flags (kTile^3 bytes) arrive by two TMA tensor copies
// (cp.async.bulk.tensor) on one mbarrier; otherwise by per-thread loads. A
// TMA box must start at a non-negative coordinate whose innermost offset is
// 16-byte aligned (an odd fp64 x start faults with an illegal instruction),
// so along x the box starts two nodes before the tile (the tile starts at a
// multiple of 16 when nx % 16 == 0) and along any axis where that start
// would be negative it starts at 0 and the shared-memory index shifts (the
// nodes before 0 are outside the grid and never read; the box then reaches
// past the far halo, zero-filled or unused).
template <bool kTma>
__global__ void __launch_bounds__(kTile * kTile) sweep_tiles(const __grid_constant__ CUtensorMap tmap_d,
                                                             const __grid_constant__ CUtensorMap tmap_x, GridP G,
                                                             int ord, int S, int nti, int ntj, int ntk, int tk_lo,
                                                             double sentinel, const unsigned char* __restrict__ exact,
                                                             double* __restrict__ d,
                                                             unsigned long long* __restrict__ max_change) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem);
    unsigned long long* wmax = mbar + 1;
    double* sd = reinterpret_cast<double*>(smem + kSdOff);
    unsigned char* sx = smem + kSxOff;
    const int tkp = tk_lo + blockIdx.x / ntj, tjp = blockIdx.x % ntj;
    const int tip = S - tjp - tkp;
    if (tip < 0 || tip >= nti || tkp >= ntk) return;  // uniform per CTA
    // the tile's real box [x0, x0 + bx) etc. (mirrored tiles map to contiguous boxes)
    const int mlo[3] = {tip * kTile, tjp * kTile, tkp * kTile};
    const int n3[3] = {G.nx, G.ny, G.nz};
    int lo[3], bsz[3];
    for (int a = 0; a < 3; ++a) {
        const int mhi = min(mlo[a] + kTile, n3[a]);
        bsz[a] = mhi - mlo[a];
        lo[a] = (ord >> a) & 1 ? n3[a] - mhi : mlo[a];
    }
    // box start per axis (x two nodes early, y and z one) and the shared index
    // of the real local node (l0, l1, l2), l in [-1, kTile]
    const int bx0 = kTma ? max(lo[0] - 2, 0) : lo[0] - 2, by0 = kTma ? max(lo[1] - 1, 0) : lo[1] - 1,
              bz0 = kTma ? max(lo[2] - 1, 0) : lo[2] - 1;
    const int ebase = ((lo[2] - bz0) * kTH + lo[1] - by0) * kTHX + lo[0] - bx0;
    if (kTma) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(mbar)));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
                         "r"(kSdBytes + (LSR_SWEEP_TMA_FLAGS ? kSxBytes : 0))
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];\n" ::"r"(smem_u32(sd)),
                "l"(reinterpret_cast<unsigned long long>(&tmap_d)), "r"(bx0), "r"(by0), "r"(bz0), "r"(smem_u32(mbar))
                : "memory");
#if LSR_SWEEP_TMA_FLAGS
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];\n" ::"r"(smem_u32(sx)),
                "l"(reinterpret_cast<unsigned long long>(&tmap_x)), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(smem_u32(mbar))
                : "memory");
#endif
        }
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}\n" ::"r"(
                smem_u32(mbar))
            : "memory");
#if !LSR_SWEEP_TMA_FLAGS
        for (int e = threadIdx.x; e < bsz[0] * bsz[1] * bsz[2]; e += blockDim.x) {
            const int z = e / (bsz[0] * bsz[1]), y = (e / bsz[0]) % bsz[1], x = e % bsz[0];
            sx[(z * kTile + y) * kTile + x] =
                exact[(static_cast<long long>(lo[2] + z) * G.ny + lo[1] + y) * G.nx + lo[0] + x];
        }
        __syncthreads();
#endif
    } else {
        // box + halo into shared memory (outside the grid: never read)
        for (int e = threadIdx.x; e < kTH * kTH * kTHX; e += blockDim.x) {
            const int hz = e / (kTH * kTHX), hy = (e / kTHX) % kTH, hx = e % kTHX;
            const int gx = bx0 + hx, gy = by0 + hy, gz = bz0 + hz;
            if (hx >= 1 && hx <= bsz[0] + 2 && hy <= bsz[1] + 1 && hz <= bsz[2] + 1 && gx >= 0 && gx < G.nx &&
                gy >= 0 && gy < G.ny && gz >= 0 && gz < G.nz)
                sd[e] = d[(static_cast<long long>(gz) * G.ny + gy) * G.nx + gx];
        }
        // the flags too: a global load inside the plane loop would put its
        // latency on every one of the 3*kTile-2 dependent steps
        for (int e = threadIdx.x; e < bsz[0] * bsz[1] * bsz[2]; e += blockDim.x) {
            const int z = e / (bsz[0] * bsz[1]), y = (e / bsz[0]) % bsz[1], x = e % bsz[0];
            sx[(z * kTile + y) * kTile + x] =
                exact[(static_cast<long long>(lo[2] + z) * G.ny + lo[1] + y) * G.nx + lo[0] + x];
        }
        __syncthreads();
    }
    const int ljp = threadIdx.x % kTile, lkp = threadIdx.x / kTile;  // this thread's mirrored row
    const bool row_ok = ljp < bsz[1] && lkp < bsz[2];
    const int lj = (ord & 2) ? bsz[1] - 1 - ljp : ljp, lk = (ord & 4) ? bsz[2] - 1 - lkp : lkp;
    const int gj = lo[1] + lj, gk = lo[2] + lk;
    unsigned long long cmax = 0;
    const int planes = bsz[0] + bsz[1] + bsz[2] - 2;
    for (int sp = 0; sp < planes; ++sp) {
        const int lip = sp - ljp - lkp;
        if (row_ok && lip >= 0 && lip < bsz[0]) {
            const int li = (ord & 1) ? bsz[0] - 1 - lip : lip;
            const int gi = lo[0] + li;
            if (!sx[(lk * kTile + lj) * kTile + li]) {
                const int e = ebase + (lk * kTH + lj) * kTHX + li;
                double a[3];
                int m = 0;
                {
                    double best = sentinel;
                    if (gi > 0) best = dmin(best, sd[e - 1]);
                    if (gi < G.nx - 1) best = dmin(best, sd[e + 1]);
                    if (best < sentinel) a[m++] = best;
                }
                {
                    double best = sentinel;
                    if (gj > 0) best = dmin(best, sd[e - kTHX]);
                    if (gj < G.ny - 1) best = dmin(best, sd[e + kTHX]);
                    if (best < sentinel) a[m++] = best;
                }
                {
                    double best = sentinel;
                    if (gk > 0) best = dmin(best, sd[e - kTH * kTHX]);
                    if (gk < G.nz - 1) best = dmin(best, sd[e + kTH * kTHX]);
                    if (best < sentinel) a[m++] = best;
                }
                if (m > 0) {
                    if (m >= 2 && a[1] < a[0]) { const double t0 = a[0]; a[0] = a[1]; a[1] = t0; }
                    if (m == 3) {
                        if (a[2] < a[1]) { const double t1 = a[1]; a[1] = a[2]; a[2] = t1; }
                        if (a[1] < a[0]) { const double t0 = a[0]; a[0] = a[1]; a[1] = t0; }
                    }
                    const double v = sd[e];
                    const double cand = eikonal_update(a, m, G.dx);
                    if (cand < v) {
                        sd[e] = cand;
                        const unsigned long long c =
                            static_cast<unsigned long long>(__double_as_longlong(v - cand));
                        cmax = c > cmax ? c : cmax;
                    }
                }
            }
        }
        __syncthreads();
    }
    // write the box back
    for (int e = threadIdx.x; e < bsz[0] * bsz[1] * bsz[2]; e += blockDim.x) {
        const int z = e / (bsz[0] * bsz[1]), y = (e / bsz[0]) % bsz[1], x = e % bsz[0];
        d[(static_cast<long long>(lo[2] + z) * G.ny + lo[1] + y) * G.nx + lo[0] + x] =
            sd[ebase + (z * kTH + y) * kTHX + x];
    }
    // the largest change: one atomic per CTA (max is order free)
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, cmax, off);
        cmax = o > cmax ? o : cmax;
    }
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = cmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long mm = 0;
        for (int w = 0; w < kTile * kTile / 32; ++w) mm = wmax[w] > mm ? wmax[w] : mm;
        if (mm) atomicMax(max_change, mm);
    }
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link dependency)
static bool make_tile_maps(const GridP& G, double* d, const unsigned char* exact, CUtensorMap* maps) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        // the 12.0 ABI of the symbol (the typedef below), whatever the driver's default
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(G.nx), static_cast<cuuint64_t>(G.ny),
                                static_cast<cuuint64_t>(G.nz)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint64_t sd_str[2] = {static_cast<cuuint64_t>(G.nx) * 8, static_cast<cuuint64_t>(G.nxy) * 8};
    const cuuint32_t sd_box[3] = {kTHX, kTH, kTH};
    const cuuint64_t sx_str[2] = {static_cast<cuuint64_t>(G.nx), static_cast<cuuint64_t>(G.nxy)};
    const cuuint32_t sx_box[3] = {kTile, kTile, kTile};
    if (encode(&maps[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, sd_str, sd_box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (encode(&maps[1], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<unsigned char*>(exact), dims, sx_str, sx_box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    return true;
}

namespace {

// estimate_resolution's terms (cloud.cpp:473-476): the exact NN distance of
// sampled point idx[i] to the rest of the cloud
__global__ void sample_nn(HashP H, const double* __restrict__ pts, const int* __restrict__ starts,
                          const int* __restrict__ entries, const int* __restrict__ idx, long long m,
                          double* __restrict__ term) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int id = idx[i];
    const double* q = pts + 3 * static_cast<long long>(id);
    term[i] = nearest_distance(H, pts, starts, entries, q[0], q[1], q[2], id);
}

// blocked_sum's in-block serial sums (parallel.hpp:31-37)
__global__ void block_sums(const double* __restrict__ term, long long n, double* __restrict__ partial) {
    const long long b = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long lo = b * 4096;
    if (lo >= n) return;
    const long long hi = min(n, lo + 4096);
    double acc = 0.0;
    for (long long i = lo; i < hi; ++i) acc += term[i];
    partial[b] = acc;
}

}  // namespace

// ---------------------------------------------------------------------------

// fast_sweep (distance.cpp:72-142) of the device field d_field with the
// exact flags d_exact and the sentinel (values >= sentinel are unseeded):
// Gauss-Seidel over the 2^dim orderings as tiled wavefronts, until the
// largest change of a round is below 1e-3 dx or after 8 rounds.
int lsr_prep_fast_sweep(const lsr_grid* g, double* d_field, const unsigned char* d_exact, double sentinel,
                        int* rounds_out, cudaStream_t s, std::string* err) {
    auto fail = [&](int code, const char* m) {
        *err = m;
        return code;
    };
#define PREP_TRY(x)                                         \
    do {                                                    \
        cudaError_t e_ = (x);                               \
        if (e_ != cudaSuccess) {                            \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_); \
            return LSR_ERR_CUDA;                            \
        }                                                   \
    } while (0)
    GridP G{g->dim, g->dims[0], g->dims[1], g->dims[2], static_cast<long long>(g->dims[0]) * g->dims[1],
            g->origin[0], g->origin[1], g->origin[2], g->dx};
    const long long N = G.nxy * G.nz;
    const int T = 256;
    int* flag = nullptr;
    unsigned long long* dmax = nullptr;
    struct Guard {
        int*& f;
        unsigned long long*& m;
        ~Guard() {
            cudaFree(f);
            cudaFree(m);
        }
    } guard{flag, dmax};
    PREP_TRY(cudaMalloc(&flag, sizeof(int)));
    PREP_TRY(cudaMalloc(&dmax, sizeof(unsigned long long)));
    int h_flag = 0;
    PREP_TRY(cudaMemsetAsync(flag, 0, sizeof(int), s));
    any_below<<<148 * 4, 256, 0, s>>>(d_field, N, sentinel, flag);
    lsr_note_launch();
    PREP_TRY(cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    PREP_TRY(cudaStreamSynchronize(s));
    if (!h_flag) return fail(LSR_ERR, "fast_sweep: no finite seed value");
    const int orderings = g->dim == 3 ? 8 : 4;
    const double tol = 1e-3 * g->dx;
    const int max_rounds = 8;
    static const bool tiled = !(std::getenv("LSR_SWEEP_TILES") && std::atoi(std::getenv("LSR_SWEEP_TILES")) == 0);
    // TMA tensor maps of d (fp64) and the exact flags (u8) over the grid for
    // the tiled sweep; global strides must be multiples of 16 bytes
    CUtensorMap tmaps[2] = {};
    bool use_tma = false;
    if (G.dim == 3 && tiled) {
        static const int tma_env = std::getenv("LSR_SWEEP_TMA") ? std::atoi(std::getenv("LSR_SWEEP_TMA")) : 1;
        use_tma = tma_env != 0 && G.nx % 16 == 0 && make_tile_maps(G, d_field, d_exact, tmaps);
        // the dynamic shared-memory limit is a per-device function attribute
        static std::atomic<unsigned long long> attr_set{0};
        int dev = 0;
        PREP_TRY(cudaGetDevice(&dev));
        if (dev >= 64 || !(attr_set.load() >> dev & 1ULL)) {
            PREP_TRY(cudaFuncSetAttribute(sweep_tiles<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
            PREP_TRY(cudaFuncSetAttribute(sweep_tiles<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmem));
            if (dev < 64) attr_set.fetch_or(1ULL << dev);
        }
    }
    const int smax = (G.nx - 1) + (G.ny - 1) + (G.dim == 3 ? G.nz - 1 : 0);
    int round = 0;
    for (; round < max_rounds; ++round) {
        PREP_TRY(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), s));
        for (int ord = 0; ord < orderings; ++ord) {
            if (G.dim == 3 && tiled) {
                const int nti = (G.nx + kTile - 1) / kTile, ntj = (G.ny + kTile - 1) / kTile,
                          ntk = (G.nz + kTile - 1) / kTile;
                for (int S = 0; S <= (nti - 1) + (ntj - 1) + (ntk - 1); ++S) {
                    const int tk_lo = std::max(0, S - (nti - 1) - (ntj - 1)), tk_hi = std::min(ntk - 1, S);
                    const unsigned ctas = static_cast<unsigned>((tk_hi - tk_lo + 1) * ntj);
                    if (use_tma)
                        sweep_tiles<true><<<ctas, kTile * kTile, kTileSmem, s>>>(
                            tmaps[0], tmaps[1], G, ord, S, nti, ntj, ntk, tk_lo, sentinel, d_exact, d_field, dmax);
                    else
                        sweep_tiles<false><<<ctas, kTile * kTile, kTileSmem, s>>>(
                            tmaps[0], tmaps[1], G, ord, S, nti, ntj, ntk, tk_lo, sentinel, d_exact, d_field, dmax);
                    lsr_note_launch();
                }
                continue;
            }
            for (int sp = 0; sp <= smax; ++sp) {
                const int k_lo = G.dim == 3 ? std::max(0, sp - (G.nx - 1) - (G.ny - 1)) : 0;
                const int k_hi = G.dim == 3 ? std::min(G.nz - 1, sp) : 0;
                const int k_cnt = k_hi - k_lo + 1;
                const long long threads = static_cast<long long>(k_cnt) * G.ny;
                sweep_plane<<<static_cast<unsigned>((threads + T - 1) / T), T, 0, s>>>(G, ord, sp, k_lo, k_cnt,
                                                                                      sentinel, d_exact, d_field, dmax);
                lsr_note_launch();
            }
        }
        PREP_TRY(cudaGetLastError());
        unsigned long long h_max = 0;
        PREP_TRY(cudaMemcpyAsync(&h_max, dmax, sizeof h_max, cudaMemcpyDeviceToHost, s));
        PREP_TRY(cudaStreamSynchronize(s));
        double max_change;
        std::memcpy(&max_change, &h_max, sizeof max_change);
        if (max_change < tol) {
            ++round;
            break;
        }
    }
    *rounds_out = round;
    return LSR_OK;
#undef PREP_TRY
}

int lsr_prep_build_distance(const lsr_grid* g, const double* h_pts, int64_t n, int dim, int seed_only,
                            double* d_field, unsigned char* d_exact, double* sentinel_out, int* rounds_out,
                            cudaStream_t s, std::string* err) {
    auto fail = [&](int code, const char* m) {
        *err = m;
        return code;
    };
#define PREP_TRY(x)                                         \
    do {                                                    \
        cudaError_t e_ = (x);                               \
        if (e_ != cudaSuccess) {                            \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_); \
            return LSR_ERR_CUDA;                            \
        }                                                   \
    } while (0)
    if (n <= 0) return fail(LSR_ERR, "seed_exact_distance: empty cloud");          // distance.cpp:9
    if (dim != g->dim) return fail(LSR_ERR_CONFIG, "seed_exact_distance: dimension mismatch");  // :10
    // Grid::diagonal (grid.hpp:35) and the sentinel (distance.cpp:13)
    double up[3], diff[3];
    for (int d = 0; d < 3; ++d) {
        up[d] = g->origin[d] + (g->dims[d] - 1) * g->dx;
        diff[d] = up[d] - g->origin[d];
    }
    const double sentinel = 10.0 * std::sqrt(diff[0] * diff[0] + diff[1] * diff[1] + diff[2] * diff[2]);
    *sentinel_out = sentinel;
    // Grid::contains for every point (distance.cpp:18-20), bounding box (cloud.cpp:380-388)
    double lo[3] = {h_pts[0], h_pts[1], h_pts[2]}, hi[3] = {h_pts[0], h_pts[1], h_pts[2]};
    for (int64_t q = 0; q < n; ++q) {
        const double* p = h_pts + 3 * q;
        for (int d = 0; d < g->dim; ++d)
            if (p[d] < g->origin[d] || p[d] > up[d])
                return fail(LSR_ERR_OUT_OF_DOMAIN, "seed_exact_distance: cloud point outside grid hull");
        for (int d = 0; d < 3; ++d) {
            lo[d] = std::min(lo[d], p[d]);
            hi[d] = std::max(hi[d], p[d]);
        }
    }
    // SpatialHash geometry (cloud.cpp:390-399)
    HashP H{};
    H.dim = dim;
    H.lox = lo[0];
    H.loy = lo[1];
    H.loz = lo[2];
    const double span[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    const double diag = std::sqrt(span[0] * span[0] + span[1] * span[1] + span[2] * span[2]);
    const double n_axis = std::pow(static_cast<double>(n), 1.0 / dim);
    H.cell = diag > 0.0 ? diag / std::max(1.0, n_axis) : 1.0;
    int nb[3];
    for (int d = 0; d < 3; ++d) nb[d] = d < dim ? 1 + static_cast<int>(span[d] / H.cell) : 1;
    H.bx = nb[0];
    H.by = nb[1];
    H.bz = nb[2];
    const long long nbins = static_cast<long long>(nb[0]) * nb[1] * nb[2];

    GridP G{g->dim, g->dims[0], g->dims[1], g->dims[2], static_cast<long long>(g->dims[0]) * g->dims[1],
            g->origin[0], g->origin[1], g->origin[2], g->dx};
    const long long N = G.nxy * G.nz;

    double* pts = nullptr;
    int *counts = nullptr, *starts = nullptr, *bin_id = nullptr, *entries = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    auto cleanup = [&] {
        cudaFree(pts);
        cudaFree(counts);
        cudaFree(starts);
        cudaFree(bin_id);
        cudaFree(entries);
        cudaFree(tmp);
    };
    struct Guard {
        decltype(cleanup)& f;
        ~Guard() { f(); }
    } guard{cleanup};
    PREP_TRY(cudaMalloc(&pts, sizeof(double) * 3 * n));
    PREP_TRY(cudaMalloc(&counts, sizeof(int) * (nbins + 1)));
    PREP_TRY(cudaMalloc(&starts, sizeof(int) * (nbins + 1)));
    PREP_TRY(cudaMalloc(&bin_id, sizeof(int) * n));
    PREP_TRY(cudaMalloc(&entries, sizeof(int) * n));
    PREP_TRY(cudaMemcpyAsync(pts, h_pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    PREP_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * (nbins + 1), s));
    const int T = 256;
    const unsigned pb = static_cast<unsigned>((n + T - 1) / T);
    count_bins<<<pb, T, 0, s>>>(H, pts, n, counts, bin_id);
    lsr_note_launch();
    PREP_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, starts, static_cast<int>(nbins + 1), s));
    PREP_TRY(cudaMalloc(&tmp, tmp_bytes));
    PREP_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, starts, static_cast<int>(nbins + 1), s));
    PREP_TRY(cudaMemcpyAsync(counts, starts, sizeof(int) * (nbins + 1), cudaMemcpyDeviceToDevice, s));
    scatter_bins<<<pb, T, 0, s>>>(bin_id, n, counts, entries);
    lsr_note_launch();

    PREP_TRY(cudaMemsetAsync(d_exact, 0, N, s));
    seed_flag<<<pb, T, 0, s>>>(G, pts, n, d_exact);
    lsr_note_launch();
    seed_values<<<static_cast<unsigned>((N + T - 1) / T), T, 0, s>>>(G, H, pts, starts, entries, d_exact, sentinel,
                                                                      d_field);
    lsr_note_launch();
    PREP_TRY(cudaGetLastError());
    if (seed_only) {
        *rounds_out = 0;
        PREP_TRY(cudaStreamSynchronize(s));
        return LSR_OK;
    }

    return lsr_prep_fast_sweep(g, d_field, d_exact, sentinel, rounds_out, s, err);
#undef PREP_TRY
}

// SpatialHash geometry (cloud.cpp:390-399) from a host cloud, plus its CSR
// bins built on the device (counting sort).
struct DeviceHash {
    HashP H{};
    double* pts = nullptr;
    int* starts = nullptr;
    int* entries = nullptr;
    ~DeviceHash() {
        cudaFree(pts);
        cudaFree(starts);
        cudaFree(entries);
    }
};

static int build_hash(const double* h_pts, int64_t n, int dim, DeviceHash& D, cudaStream_t s, std::string* err) {
#define HB_TRY(x)                                                    \
    do {                                                             \
        cudaError_t e_ = (x);                                        \
        if (e_ != cudaSuccess) {                                     \
            *err = std::string(#x) + ": " + cudaGetErrorString(e_);  \
            return LSR_ERR_CUDA;                                     \
        }                                                            \
    } while (0)
    double lo[3] = {h_pts[0], h_pts[1], h_pts[2]}, hi[3] = {h_pts[0], h_pts[1], h_pts[2]};
    for (int64_t q = 0; q < n; ++q)  // bounding_box (cloud.cpp:380-388)
        for (int d = 0; d < 3; ++d) {
            lo[d] = std::min(lo[d], h_pts[3 * q + d]);
            hi[d] = std::max(hi[d], h_pts[3 * q + d]);
        }
    HashP& H = D.H;
    H.dim = dim;
    H.lox = lo[0];
    H.loy = lo[1];
    H.loz = lo[2];
    const double span[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    const double diag = std::sqrt(span[0] * span[0] + span[1] * span[1] + span[2] * span[2]);
    const double n_axis = std::pow(static_cast<double>(n), 1.0 / dim);
    H.cell = diag > 0.0 ? diag / std::max(1.0, n_axis) : 1.0;
    int nb[3];
    for (int d = 0; d < 3; ++d) nb[d] = d < dim ? 1 + static_cast<int>(span[d] / H.cell) : 1;
    H.bx = nb[0];
    H.by = nb[1];
    H.bz = nb[2];
    const long long nbins = static_cast<long long>(nb[0]) * nb[1] * nb[2];
    int *counts = nullptr, *bin_id = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    struct G {
        int** a;
        int** b;
        void** c;
        ~G() {
            cudaFree(*a);
            cudaFree(*b);
            cudaFree(*c);
        }
    } guard{&counts, &bin_id, &tmp};
    HB_TRY(cudaMalloc(&D.pts, sizeof(double) * 3 * n));
    HB_TRY(cudaMalloc(&D.starts, sizeof(int) * (nbins + 1)));
    HB_TRY(cudaMalloc(&D.entries, sizeof(int) * n));
    HB_TRY(cudaMalloc(&counts, sizeof(int) * (nbins + 1)));
    HB_TRY(cudaMalloc(&bin_id, sizeof(int) * n));
    HB_TRY(cudaMemcpyAsync(D.pts, h_pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    HB_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * (nbins + 1), s));
    const unsigned pb = static_cast<unsigned>((n + 255) / 256);
    count_bins<<<pb, 256, 0, s>>>(H, D.pts, n, counts, bin_id);
    lsr_note_launch();
    HB_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, D.starts, static_cast<int>(nbins + 1), s));
    HB_TRY(cudaMalloc(&tmp, tb));
    HB_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, D.starts, static_cast<int>(nbins + 1), s));
    HB_TRY(cudaMemcpyAsync(counts, D.starts, sizeof(int) * (nbins + 1), cudaMemcpyDeviceToDevice, s));
    scatter_bins<<<pb, 256, 0, s>>>(bin_id, n, counts, D.entries);
    lsr_note_launch();
    HB_TRY(cudaStreamSynchronize(s));
    return LSR_OK;
#undef HB_TRY
}

// compute_stats (cloud.cpp:480-489) with estimate_resolution (:454-478):
// the seeded Fisher-Yates prefix stays on the host (mt19937_64 and the
// unbiased bounded draw, cloud.cpp:20-27); the sampled exact NN distances
// run on the device; blocked_sum order is kept (serial 4096-term blocks,
// block partials summed in order on the host).
int lsr_prep_compute_stats(const double* h_pts, int64_t n, int dim, double fraction, double k_s, uint64_t seed,
                           double* h_s, double* gamma_s, double* bbox6, cudaStream_t s, std::string* err) {
    if (n < 2) {
        *err = "estimate_resolution: need at least 2 points";
        return LSR_ERR;
    }
    if (!(fraction > 0.0) || fraction > 1.0) {
        *err = "estimate_resolution: sample_fraction must be in (0, 1]";
        return LSR_ERR_CONFIG;
    }
    int64_t m = std::llround(fraction * static_cast<double>(n));
    m = std::min<int64_t>(std::max<int64_t>(m, 1), n);
    std::vector<int> idx(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) idx[i] = static_cast<int>(i);
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < m; ++i) {
        const uint64_t range = static_cast<uint64_t>(n - i);
        const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
        uint64_t x = rng();
        while (x >= limit) x = rng();
        std::swap(idx[i], idx[i + static_cast<int64_t>(x % range)]);
    }
    DeviceHash D;
    if (int st = build_hash(h_pts, n, dim, D, s, err)) return st;
    int* d_idx = nullptr;
    double* term = nullptr;
    double* partial = nullptr;
    const long long nblk = (m + 4095) / 4096;
    struct G {
        int** a;
        double** b;
        double** c;
        ~G() {
            cudaFree(*a);
            cudaFree(*b);
            cudaFree(*c);
        }
    } guard{&d_idx, &term, &partial};
    auto cuda_fail = [&](cudaError_t e, const char* w) {
        *err = std::string(w) + ": " + cudaGetErrorString(e);
        return LSR_ERR_CUDA;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&d_idx, sizeof(int) * m)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&term, sizeof(double) * m)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&partial, sizeof(double) * nblk)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMemcpyAsync(d_idx, idx.data(), sizeof(int) * m, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync");
    sample_nn<<<static_cast<unsigned>((m + 127) / 128), 128, 0, s>>>(D.H, D.pts, D.starts, D.entries, d_idx, m, term);
    lsr_note_launch();
    block_sums<<<static_cast<unsigned>((nblk + 127) / 128), 128, 0, s>>>(term, m, partial);
    lsr_note_launch();
    std::vector<double> hp(static_cast<size_t>(nblk));
    if ((e = cudaMemcpyAsync(hp.data(), partial, sizeof(double) * nblk, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    double total = 0.0;
    for (double v : hp) total += v;
    *h_s = total / static_cast<double>(m);
    *gamma_s = k_s * *h_s;
    double lo[3] = {h_pts[0], h_pts[1], h_pts[2]}, hi[3] = {h_pts[0], h_pts[1], h_pts[2]};
    for (int64_t q = 0; q < n; ++q)
        for (int d = 0; d < 3; ++d) {
            lo[d] = std::min(lo[d], h_pts[3 * q + d]);
            hi[d] = std::max(hi[d], h_pts[3 * q + d]);
        }
    for (int d = 0; d < 3; ++d) {
        bbox6[d] = lo[d];
        bbox6[3 + d] = hi[d];
    }
    return LSR_OK;
}
