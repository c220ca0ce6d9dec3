// Device side of the one-shot host entry when the caller's phi and d are in
// mapped (pinned) host memory: the GPU works out which values one SL step
// reads (node bitmaps built from the active ids) and pulls exactly those over
// PCIe with zero-copy loads — no host thread packs anything.
//
// Bitmaps: one bit per node, each grid row padded to W = ceil(nx / 64) words,
// word index (k * ny + j) * W + x / 64.
//   active A     : the active ids
//   d set   D    : A and its axis neighbours (the centered gradient of d,
//                  reference src/grid.cpp:53-74 via src/evolve.cpp:57-66)
//   phi set B    : the Chebyshev ball of radius R around A (feet stencils
//                  and the fallback's neighbour interpolations; the SL kernel
//                  counts any foot whose stencil may leave it)
#include <cuda_runtime.h>

#include <cstdint>

#include "transfer_launch.h"

void lsr_note_launch();

namespace {

struct Bits {
    int nx, ny, nz, W;
    __device__ __forceinline__ long long row(int j, int k) const { return (static_cast<long long>(k) * ny + j) * W; }
    __device__ __forceinline__ unsigned long long last_mask() const {
        const int r = nx & 63;
        return r == 0 ? ~0ULL : ((1ULL << r) - 1);
    }
};

__global__ void set_active_bits(Bits b, const int64_t* __restrict__ ids, long long n, unsigned long long* bm,
                                unsigned long long* bad) {
    const long long N = static_cast<long long>(b.nx) * b.ny * b.nz;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long id = ids[t];
        if (id < 0 || id >= N) {  // never dereferenced: the step falls back
            atomicAdd(bad, 1ULL);
            continue;
        }
        const long long jk = id / b.nx;
        const int x = static_cast<int>(id - jk * b.nx);
        atomicOr(bm + jk * b.W + (x >> 6), 1ULL << (x & 63));
    }
}

// word w of a row shifted so that bit x takes the value of bit x - s (s > 0:
// towards higher x) or x + |s| (s < 0), zero-filled at the row ends
__device__ __forceinline__ unsigned long long shifted(const unsigned long long* row, int w, int W, int s) {
    if (s > 0) {
        const unsigned long long lo = w > 0 ? row[w - 1] : 0ULL;
        return s == 64 ? lo : (row[w] << s) | (lo >> (64 - s));
    }
    const int u = -s;
    const unsigned long long hi = w + 1 < W ? row[w + 1] : 0ULL;
    return u == 64 ? hi : (row[w] >> u) | (hi << (64 - u));
}

// D = A | A(x +- 1) | A(j +- 1) | A(k +- 1)
__global__ void axis_dilate(Bits b, const unsigned long long* __restrict__ A, unsigned long long* __restrict__ D) {
    const long long words = static_cast<long long>(b.ny) * b.nz * b.W;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < words;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = t / b.W;
        const int w = static_cast<int>(t - r * b.W);
        const int j = static_cast<int>(r % b.ny), k = static_cast<int>(r / b.ny);
        const unsigned long long* row = A + r * b.W;
        unsigned long long v = row[w] | shifted(row, w, b.W, 1) | shifted(row, w, b.W, -1);
        if (j > 0) v |= A[b.row(j - 1, k) + w];
        if (j + 1 < b.ny) v |= A[b.row(j + 1, k) + w];
        if (k > 0) v |= A[b.row(j, k - 1) + w];
        if (k + 1 < b.nz) v |= A[b.row(j, k + 1) + w];
        if (w == b.W - 1) v &= b.last_mask();
        D[t] = v;
    }
}

// one separable pass of the Chebyshev dilation by R: axis 0 = x (within the
// row's words), 1 = y (rows), 2 = z (planes)
__global__ void ball_pass(Bits b, int axis, int R, const unsigned long long* __restrict__ in,
                          unsigned long long* __restrict__ out) {
    const long long words = static_cast<long long>(b.ny) * b.nz * b.W;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < words;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = t / b.W;
        const int w = static_cast<int>(t - r * b.W);
        const int j = static_cast<int>(r % b.ny), k = static_cast<int>(r / b.ny);
        unsigned long long v = 0;
        if (axis == 0) {
            const unsigned long long* row = in + r * b.W;
            v = row[w];
            for (int s = 1; s <= R; ++s) v |= shifted(row, w, b.W, s) | shifted(row, w, b.W, -s);
            if (w == b.W - 1) v &= b.last_mask();
        } else if (axis == 1) {
            for (int jj = max(0, j - R); jj <= min(b.ny - 1, j + R); ++jj) v |= in[b.row(jj, k) + w];
        } else {
            for (int kk = max(0, k - R); kk <= min(b.nz - 1, k + R); ++kk) v |= in[b.row(j, kk) + w];
        }
        out[t] = v;
    }
}

// zero-copy pull of planes [z0, z1): dst[n] = src[n] where the node's bit is
// set, two fields at once. One warp per 64-node bitmap word: lane l moves
// nodes 2l and 2l+1 with one 16-byte load when both are set, so a warp's
// reads of a run are contiguous and wide; empty words are skipped whole.
__device__ __forceinline__ void pull_pair(unsigned long long word, int l, const double* __restrict__ src,
                                          double* __restrict__ dst, long long n) {
    const unsigned pair = static_cast<unsigned>(word >> (2 * l)) & 3u;
    if (pair == 3u && ((n & 1) == 0)) {
        *reinterpret_cast<double2*>(dst + n) = *reinterpret_cast<const double2*>(src + n);
    } else {
        if (pair & 1u) dst[n] = src[n];
        if (pair & 2u) dst[n + 1] = src[n + 1];
    }
}

__global__ void pull_planes(Bits b, int z0, int z1, const unsigned long long* __restrict__ bm_a,
                            const double* __restrict__ src_a, double* __restrict__ dst_a,
                            const unsigned long long* __restrict__ bm_b, const double* __restrict__ src_b,
                            double* __restrict__ dst_b) {
    const long long w0 = static_cast<long long>(z0) * b.ny * b.W, w1 = static_cast<long long>(z1) * b.ny * b.W;
    const int l = threadIdx.x & 31;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    for (long long w = w0 + ((static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); w < w1; w += nw) {
        const unsigned long long wa = bm_a ? bm_a[w] : 0ULL, wb = bm_b ? bm_b[w] : 0ULL;
        if ((wa | wb) == 0ULL) continue;
        const long long r = w / b.W;
        const int x0 = static_cast<int>(w - r * b.W) << 6;
        const long long n = r * b.nx + x0 + 2 * l;  // rows are unpadded in the fields
        if (x0 + 2 * l >= b.nx) continue;
        if (wa) pull_pair(wa, l, src_a, dst_a, n);
        if (wb) pull_pair(wb, l, src_b, dst_b, n);
    }
}

__global__ void count_bits(Bits b, int z0, int z1, const unsigned long long* __restrict__ bm,
                           unsigned long long* count) {
    const long long w0 = static_cast<long long>(z0) * b.ny * b.W, w1 = static_cast<long long>(z1) * b.ny * b.W;
    unsigned long long c = 0;
    for (long long t = w0 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < w1;
         t += static_cast<long long>(gridDim.x) * blockDim.x)
        c += __popcll(bm[t]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

unsigned grid_for(long long work, int threads) {
    long long blocks = (work + threads - 1) / threads;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    return static_cast<unsigned>(blocks < 1 ? 1 : blocks);
}

}  // namespace

long long lsr_bitmap_words(int nx, int ny, int nz) {
    return static_cast<long long>(ny) * nz * ((nx + 63) / 64);
}

cudaError_t launch_build_bitmaps(int nx, int ny, int nz, const int64_t* ids, long long n, int reach,
                                 unsigned long long* A, unsigned long long* D, unsigned long long* B,
                                 unsigned long long* T, unsigned long long* bad, cudaStream_t s) {
    const Bits b{nx, ny, nz, (nx + 63) / 64};
    const long long words = lsr_bitmap_words(nx, ny, nz);
    cudaError_t e = cudaMemsetAsync(A, 0, sizeof(unsigned long long) * words, s);
    if (e != cudaSuccess) return e;
    set_active_bits<<<grid_for(n, 256), 256, 0, s>>>(b, ids, n, A, bad);
    axis_dilate<<<grid_for(words, 256), 256, 0, s>>>(b, A, D);
    lsr_note_launch();
    lsr_note_launch();
    if (reach > 0) {
        ball_pass<<<grid_for(words, 256), 256, 0, s>>>(b, 0, reach, A, B);
        ball_pass<<<grid_for(words, 256), 256, 0, s>>>(b, 1, reach, B, T);
        ball_pass<<<grid_for(words, 256), 256, 0, s>>>(b, 2, reach, T, B);
        lsr_note_launch();
        lsr_note_launch();
        lsr_note_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_pull_planes(int nx, int ny, int nz, int z0, int z1, const unsigned long long* bm_a,
                               const double* src_a, double* dst_a, const unsigned long long* bm_b,
                               const double* src_b, double* dst_b, cudaStream_t s) {
    if (z1 <= z0) return cudaSuccess;
    const Bits b{nx, ny, nz, (nx + 63) / 64};
    const long long warps = static_cast<long long>(z1 - z0) * ny * b.W;
    pull_planes<<<grid_for(32 * warps, 256), 256, 0, s>>>(b, z0, z1, bm_a, src_a, dst_a, bm_b, src_b, dst_b);
    lsr_note_launch();
    return cudaGetLastError();
}

cudaError_t launch_count_bits(int nx, int ny, int nz, int z0, int z1, const unsigned long long* bm,
                              unsigned long long* count, cudaStream_t s) {
    if (z1 <= z0) return cudaSuccess;
    const Bits b{nx, ny, nz, (nx + 63) / 64};
    count_bits<<<grid_for(static_cast<long long>(z1 - z0) * ny * b.W, 256), 256, 0, s>>>(b, z0, z1, bm, count);
    lsr_note_launch();
    return cudaGetLastError();
}
