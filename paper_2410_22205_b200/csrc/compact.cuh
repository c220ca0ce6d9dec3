// Order-preserving stream compaction for the loop's selections (the band's
// ACTIVE / tube lists, the energy's interface cells, the non-frozen tube
// nodes): out = the indices i (or items src[i]) whose predicate holds, in
// ascending order — the same lists cub::DeviceSelect yields, made in three
// bandwidth-shaped passes:
//   1. per tile of kTile items, count the selected items;
//   2. exclusive scan of the tile counts (cub::DeviceScan, a few 10k items);
//   3. per tile, rank the selected items (warp ballots + a block scan) and
//      write them at tile offset + rank.
// The predicate is evaluated twice (passes 1 and 3): for the byte-flag
// predicates used here that is cheaper than cub's single-pass look-back with
// a 64-bit counting iterator, whose tile policy for 64-bit items runs at a
// third of the occupancy.
#pragma once

#include <cuda_runtime.h>

#include <cub/cub.cuh>

namespace lsr_compact {

constexpr int kThreads = 256;
constexpr int kItems = 16;  // per thread; contiguous per thread
constexpr int kTile = kThreads * kItems;

template <class Pred>
__global__ void __launch_bounds__(kThreads) count_tiles(Pred pred, long long n, long long* __restrict__ counts) {
    const long long base = static_cast<long long>(blockIdx.x) * kTile + static_cast<long long>(threadIdx.x) * kItems;
    int c = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) c += (base + q < n && pred(base + q)) ? 1 : 0;
    using Reduce = cub::BlockReduce<int, kThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const int total = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

// Item maps the selected index to the value written (the index itself, or
// a list entry for list filters)
template <class Pred, class Item, class Out>
__global__ void __launch_bounds__(kThreads) write_tiles(Pred pred, Item item, long long n,
                                                        const long long* __restrict__ offsets,
                                                        Out* __restrict__ out) {
    const long long base = static_cast<long long>(blockIdx.x) * kTile + static_cast<long long>(threadIdx.x) * kItems;
    unsigned mask = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) mask |= ((base + q < n && pred(base + q)) ? 1u : 0u) << q;
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage tmp;
    int rank;
    Scan(tmp).ExclusiveSum(__popc(mask), rank);
    Out* o = out + offsets[blockIdx.x] + rank;
    while (mask) {
        const int q = __ffs(mask) - 1;
        mask &= mask - 1;
        *o++ = item(base + q);
    }
}

// Byte-flag predicates (pred(i) = test(a[i])) read their 16 bytes per thread
// with one 16-byte load; a must be 16-byte aligned.
template <class Test>
struct BytePred {
    const unsigned char* a;
    Test test;
    __device__ __forceinline__ unsigned mask16(long long base, long long n) const {
        unsigned m = 0;
        if (base + kItems <= n) {
            const uint4 v = *reinterpret_cast<const uint4*>(a + base);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < kItems; ++q) m |= (test((w[q >> 2] >> (8 * (q & 3))) & 0xffu) ? 1u : 0u) << q;
        } else {
            for (int q = 0; q < kItems && base + q < n; ++q) m |= (test(a[base + q]) ? 1u : 0u) << q;
        }
        return m;
    }
};

template <class Test>
__global__ void __launch_bounds__(kThreads) count_tiles_bytes(BytePred<Test> pred, long long n,
                                                              long long* __restrict__ counts) {
    const long long base = static_cast<long long>(blockIdx.x) * kTile + static_cast<long long>(threadIdx.x) * kItems;
    const int c = base < n ? __popc(pred.mask16(base, n)) : 0;
    using Reduce = cub::BlockReduce<int, kThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const int total = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

template <class Test, class Item, class Out>
__global__ void __launch_bounds__(kThreads) write_tiles_bytes(BytePred<Test> pred, Item item, long long n,
                                                              const long long* __restrict__ offsets,
                                                              Out* __restrict__ out) {
    const long long base = static_cast<long long>(blockIdx.x) * kTile + static_cast<long long>(threadIdx.x) * kItems;
    unsigned mask = base < n ? pred.mask16(base, n) : 0u;
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage tmp;
    int rank;
    Scan(tmp).ExclusiveSum(__popc(mask), rank);
    Out* o = out + offsets[blockIdx.x] + rank;
    while (mask) {
        const int q = __ffs(mask) - 1;
        mask &= mask - 1;
        *o++ = item(base + q);
    }
}

struct Identity {
    __device__ long long operator()(long long i) const { return i; }
};

// The loop's compactions run as persistent launches: a CTA per resident slot
// walks the tiles (most of them empty — a band's tiles, a gated-off twin, a
// list far shorter than its capacity), instead of one CTA launch per tile.
inline unsigned persistent_grid(long long tiles) {
    const long long cap = 148LL * 8;
    return static_cast<unsigned>(tiles < cap ? tiles : cap);
}

// A tile's selected items, ranked: their offsets within the tile go to shared
// memory, and consecutive threads then store consecutive entries
// out[x] = item(tile + offset[x]) (the per-thread runs written straight to
// global memory made 8-byte stores at 16 scattered addresses per warp
// instruction, and an item that is itself a load — a list entry — was
// fetched by 16 dependent iterations per thread). All threads of the CTA call it.
template <class Item, class Out>
__device__ __forceinline__ void staged_write(unsigned short* __restrict__ stage, Out* __restrict__ out, int total,
                                             int rank, unsigned mask, long long tile, Item item) {
    const unsigned local = threadIdx.x * kItems;
    while (mask) {
        const int q = __ffs(mask) - 1;
        mask &= mask - 1;
        stage[rank++] = static_cast<unsigned short>(local + q);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < total; x += kThreads) out[x] = item(tile + stage[x]);
    __syncthreads();
}

// scratch bytes compact() needs for n items
inline size_t scratch_bytes(long long n) {
    const long long tiles = (n + kTile - 1) / kTile;
    size_t scan = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan, static_cast<long long*>(nullptr), static_cast<long long*>(nullptr),
                                  static_cast<int>(tiles + 1));
    return (2 * (tiles + 1)) * sizeof(long long) + scan + 256;
}

namespace detail {
template <class Pred, class Item, class Out>
void launch_count(Pred pred, Item, long long n, long long tiles, long long* counts, Out*, cudaStream_t s) {
    count_tiles<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(pred, n, counts);
}
template <class Test, class Item, class Out>
void launch_count(BytePred<Test> pred, Item, long long n, long long tiles, long long* counts, Out*, cudaStream_t s) {
    count_tiles_bytes<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(pred, n, counts);
}
template <class Pred, class Item, class Out>
void launch_write(Pred pred, Item item, long long n, long long tiles, const long long* offsets, Out* out,
                  cudaStream_t s) {
    write_tiles<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(pred, item, n, offsets, out);
}
template <class Test, class Item, class Out>
void launch_write(BytePred<Test> pred, Item item, long long n, long long tiles, const long long* offsets, Out* out,
                  cudaStream_t s) {
    write_tiles_bytes<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(pred, item, n, offsets, out);
}
}  // namespace detail

// out[0..*d_count) = item(i) for the i in [0, n) with pred(i), ascending.
// *d_count is written on the device (stream order); scratch holds
// scratch_bytes(n) bytes.
template <class Pred, class Item, class Out>
cudaError_t compact(Pred pred, Item item, long long n, Out* out, long long* d_count, void* scratch,
                    size_t scratch_size, cudaStream_t s) {
    if (n <= 0) return cudaMemsetAsync(d_count, 0, sizeof(long long), s);
    const long long tiles = (n + kTile - 1) / kTile;
    long long* counts = static_cast<long long*>(scratch);
    long long* offsets = counts + (tiles + 1);
    void* scan_tmp = offsets + (tiles + 1);
    size_t scan_bytes = scratch_size - 2 * (tiles + 1) * sizeof(long long);
    cudaError_t e = cudaMemsetAsync(counts + tiles, 0, sizeof(long long), s);
    if (e != cudaSuccess) return e;
    detail::launch_count(pred, item, n, tiles, counts, out, s);
    e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, offsets, static_cast<int>(tiles + 1), s);
    if (e != cudaSuccess) return e;
    detail::launch_write(pred, item, n, tiles, offsets, out, s);
    e = cudaMemcpyAsync(d_count, offsets + tiles, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Two order-preserving selections from one byte array in one pass each:
// out1 = the i with test1(a[i]), out2 = the i with test2(a[i]) (items
// base + i), as two compact() calls would make them — one count pass reads
// the bytes once for both counts, one write pass writes both lists.
template <class T1, class T2>
__global__ void __launch_bounds__(kThreads) count_tiles_bytes2(BytePred<T1> p1, T2 test2, long long n,
                                                               long long* __restrict__ c1, long long* __restrict__ c2) {
    const long long base = static_cast<long long>(blockIdx.x) * kTile + static_cast<long long>(threadIdx.x) * kItems;
    BytePred<T2> p2{p1.a, test2};
    const int a = base < n ? __popc(p1.mask16(base, n)) : 0;
    const int b = base < n ? __popc(p2.mask16(base, n)) : 0;
    using Reduce = cub::BlockReduce<int, kThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const int ta = Reduce(tmp).Sum(a);
    __syncthreads();
    const int tb = Reduce(tmp).Sum(b);
    if (threadIdx.x == 0) {
        c1[blockIdx.x] = ta;
        c2[blockIdx.x] = tb;
    }
}

template <class T1, class T2, class Item, class Out>
__global__ void __launch_bounds__(kThreads) write_tiles_bytes2(BytePred<T1> p1, T2 test2, Item item, long long n,
                                                               long long tiles, const long long* __restrict__ o1,
                                                               const long long* __restrict__ o2, Out* __restrict__ out1,
                                                               Out* __restrict__ out2) {
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned short stage[kTile];
    BytePred<T2> p2{p1.a, test2};
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const long long a0 = o1[t], a1 = o1[t + 1], b0 = o2[t], b1 = o2[t + 1];
        if (a1 == a0 && b1 == b0) continue;  // nothing selected in this tile
        const long long tile = t * kTile, base = tile + static_cast<long long>(threadIdx.x) * kItems;
        const unsigned m1 = base < n ? p1.mask16(base, n) : 0u, m2 = base < n ? p2.mask16(base, n) : 0u;
        int r1, r2;
        Scan(tmp).ExclusiveSum(__popc(m1), r1);
        __syncthreads();
        Scan(tmp).ExclusiveSum(__popc(m2), r2);
        staged_write(stage, out1 + a0, static_cast<int>(a1 - a0), r1, m1, tile, item);
        staged_write(stage, out2 + b0, static_cast<int>(b1 - b0), r2, m2, tile, item);
    }
}

inline size_t scratch_bytes2(long long n) { return 2 * scratch_bytes(n); }

// where compact2 keeps its per-tile counts (a producer of the bytes may fill
// them itself and pass counted = true)
inline void compact2_counts(void* scratch, long long n, long long** c1, long long** c2) {
    const long long tiles = (n + kTile - 1) / kTile;
    *c1 = static_cast<long long*>(scratch);
    *c2 = *c1 + 2 * (tiles + 1);
}

template <class T1, class T2, class Item, class Out>
cudaError_t compact2(BytePred<T1> p1, T2 test2, Item item, long long n, Out* out1, Out* out2, long long* d_count2,
                     void* scratch, size_t scratch_size, cudaStream_t s, bool counted = false) {
    if (n <= 0) return cudaMemsetAsync(d_count2, 0, 2 * sizeof(long long), s);
    const long long tiles = (n + kTile - 1) / kTile;
    long long* c1 = static_cast<long long*>(scratch);
    long long* off1 = c1 + (tiles + 1);
    long long* c2 = off1 + (tiles + 1);
    long long* off2 = c2 + (tiles + 1);
    void* scan_tmp = off2 + (tiles + 1);
    size_t scan_bytes = scratch_size - 4 * (tiles + 1) * sizeof(long long);
    cudaError_t e = cudaMemsetAsync(c1 + tiles, 0, sizeof(long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(c2 + tiles, 0, sizeof(long long), s);
    if (e != cudaSuccess) return e;
    if (!counted) count_tiles_bytes2<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(p1, test2, n, c1, c2);
    e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, c1, off1, static_cast<int>(tiles + 1), s);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, c2, off2, static_cast<int>(tiles + 1), s);
    if (e != cudaSuccess) return e;
    // (a CTA per tile: the band's live tiles gain more from independent CTAs than from fewer launches)
    write_tiles_bytes2<<<static_cast<unsigned>(tiles), kThreads, 0, s>>>(p1, test2, item, n, tiles, off1, off2, out1, out2);
    e = cudaMemcpyAsync(d_count2, off1 + tiles, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_count2 + 1, off2 + tiles, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// a[i] != 0 && b[i] == 0 over two byte arrays (16 of each per thread)
struct ByteAndNot {
    const unsigned char* a;
    const unsigned char* b;
    __device__ __forceinline__ unsigned mask16(long long base, long long n) const {
        unsigned m = 0;
        if (base + kItems <= n) {
            const uint4 va = *reinterpret_cast<const uint4*>(a + base);
            const uint4 vb = *reinterpret_cast<const uint4*>(b + base);
            const unsigned wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                const unsigned x = (wa[q >> 2] >> (8 * (q & 3))) & 0xffu, y = (wb[q >> 2] >> (8 * (q & 3))) & 0xffu;
                m |= (x != 0 && y == 0 ? 1u : 0u) << q;
            }
        } else {
            for (int q = 0; q < kItems && base + q < n; ++q) m |= (a[base + q] != 0 && b[base + q] == 0 ? 1u : 0u) << q;
        }
        return m;
    }
};

// compact2 over two mask providers (anything with mask16(base, n), e.g. a
// BytePred and a ByteAndNot over different arrays): both lists in one count
// and one write pass
template <class M1, class M2>
__global__ void __launch_bounds__(kThreads) count_tiles_m2(M1 p1, M2 p2, long long n, long long tiles,
                                                           long long* __restrict__ c1, long long* __restrict__ c2) {
    using Reduce = cub::BlockReduce<int, kThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const long long base = t * kTile + static_cast<long long>(threadIdx.x) * kItems;
        const int a = base < n ? __popc(p1.mask16(base, n)) : 0;
        const int b = base < n ? __popc(p2.mask16(base, n)) : 0;
        const int ta = Reduce(tmp).Sum(a);
        __syncthreads();
        const int tb = Reduce(tmp).Sum(b);
        if (threadIdx.x == 0) {
            c1[t] = ta;
            c2[t] = tb;
        }
        __syncthreads();
    }
}

template <class M1, class M2, class Item, class Out>
__global__ void __launch_bounds__(kThreads) write_tiles_m2(M1 p1, M2 p2, Item item, long long n, long long tiles,
                                                           const long long* __restrict__ o1,
                                                           const long long* __restrict__ o2, Out* __restrict__ out1,
                                                           Out* __restrict__ out2) {
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned short stage[kTile];
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const long long a0 = o1[t], a1 = o1[t + 1], b0 = o2[t], b1 = o2[t + 1];
        if (a1 == a0 && b1 == b0) continue;  // nothing selected in this tile
        const long long tile = t * kTile, base = tile + static_cast<long long>(threadIdx.x) * kItems;
        const unsigned m1 = base < n ? p1.mask16(base, n) : 0u, m2 = base < n ? p2.mask16(base, n) : 0u;
        int r1, r2;
        Scan(tmp).ExclusiveSum(__popc(m1), r1);
        __syncthreads();
        Scan(tmp).ExclusiveSum(__popc(m2), r2);
        staged_write(stage, out1 + a0, static_cast<int>(a1 - a0), r1, m1, tile, item);
        staged_write(stage, out2 + b0, static_cast<int>(b1 - b0), r2, m2, tile, item);
    }
}

template <class M1, class M2, class Item, class Out>
cudaError_t compact2m(M1 p1, M2 p2, Item item, long long n, Out* out1, Out* out2, long long* d_count2, void* scratch,
                      size_t scratch_size, cudaStream_t s) {
    if (n <= 0) return cudaMemsetAsync(d_count2, 0, 2 * sizeof(long long), s);
    const long long tiles = (n + kTile - 1) / kTile;
    long long* c1 = static_cast<long long*>(scratch);
    long long* off1 = c1 + (tiles + 1);
    long long* c2 = off1 + (tiles + 1);
    long long* off2 = c2 + (tiles + 1);
    void* scan_tmp = off2 + (tiles + 1);
    size_t scan_bytes = scratch_size - 4 * (tiles + 1) * sizeof(long long);
    cudaError_t e = cudaMemsetAsync(c1 + tiles, 0, sizeof(long long), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(c2 + tiles, 0, sizeof(long long), s);
    if (e != cudaSuccess) return e;
    count_tiles_m2<<<persistent_grid(tiles), kThreads, 0, s>>>(p1, p2, n, tiles, c1, c2);
    e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, c1, off1, static_cast<int>(tiles + 1), s);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, c2, off2, static_cast<int>(tiles + 1), s);
    if (e != cudaSuccess) return e;
    write_tiles_m2<<<persistent_grid(tiles), kThreads, 0, s>>>(p1, p2, item, n, tiles, off1, off2, out1, out2);
    e = cudaMemcpyAsync(d_count2, off1 + tiles, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_count2 + 1, off2 + tiles, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// compact() over one mask provider (anything with mask16(base, n), e.g. a
// GatedBytes): the same three passes; tiles the provider reports empty cost
// one predicate evaluation
template <class M>
__global__ void __launch_bounds__(kThreads) count_tiles_m(M p, long long n, long long tiles,
                                                          long long* __restrict__ counts) {
    using Reduce = cub::BlockReduce<int, kThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const long long base = t * kTile + static_cast<long long>(threadIdx.x) * kItems;
        const int c = base < n ? __popc(p.mask16(base, n)) : 0;
        const int total = Reduce(tmp).Sum(c);
        if (threadIdx.x == 0) counts[t] = total;
        __syncthreads();
    }
}

template <class M, class Item, class Out>
__global__ void __launch_bounds__(kThreads) write_tiles_m(M p, Item item, long long n, long long tiles,
                                                          const long long* __restrict__ offsets,
                                                          Out* __restrict__ out) {
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned short stage[kTile];
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        const long long a0 = offsets[t], a1 = offsets[t + 1];
        if (a1 == a0) continue;  // nothing selected in this tile
        const long long tile = t * kTile, base = tile + static_cast<long long>(threadIdx.x) * kItems;
        const unsigned mask = base < n ? p.mask16(base, n) : 0u;
        int rank;
        Scan(tmp).ExclusiveSum(__popc(mask), rank);
        staged_write(stage, out + a0, static_cast<int>(a1 - a0), rank, mask, tile, item);
    }
}

// flag bytes a[0 .. min(n, *n_dev)) (n_dev null: a[0 .. n)), selected where
// nonzero — but nothing at all unless (*gate != 0) == open (gate null: always
// open). Lets two alternative selections be enqueued back to back into one
// output, the device deciding which of them runs.
struct GatedBytes {
    const unsigned char* a;
    const long long* n_dev;
    const int* gate;
    int open;
    __device__ __forceinline__ unsigned mask16(long long base, long long n) const {
        if (gate != nullptr && (*gate != 0) != (open != 0)) return 0u;
        if (n_dev != nullptr) {
            const long long nd = *n_dev;
            n = nd < n ? nd : n;
        }
        unsigned m = 0;
        if (base + kItems <= n) {
            const uint4 v = *reinterpret_cast<const uint4*>(a + base);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < kItems; ++q) m |= (((w[q >> 2] >> (8 * (q & 3))) & 0xffu) != 0 ? 1u : 0u) << q;
        } else {
            for (int q = 0; q < kItems && base + q < n; ++q) m |= (a[base + q] != 0 ? 1u : 0u) << q;
        }
        return m;
    }
};

// any mask provider behind a device-side gate: selects nothing unless
// (*gate != 0) == open
template <class M>
struct Gated {
    M m;
    const int* gate;
    int open;
    __device__ __forceinline__ unsigned mask16(long long base, long long n) const {
        if ((*gate != 0) != (open != 0)) return 0u;
        return m.mask16(base, n);
    }
};

// entries t < *n_dev of a list whose flag byte a[t] is nonzero (want = 1) or zero (want = 0)
struct ListFlag {
    const unsigned char* a;
    const long long* n_dev;
    int want;
    __device__ __forceinline__ unsigned mask16(long long base, long long n) const {
        const long long nd = *n_dev;
        n = nd < n ? nd : n;
        unsigned m = 0;
        if (base + kItems <= n) {
            const uint4 v = *reinterpret_cast<const uint4*>(a + base);
            const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < kItems; ++q) m |= (((w[q >> 2] >> (8 * (q & 3))) & 0xffu) != 0 ? 1u : 0u) << q;
            return want ? m : (~m & 0xffffu);
        }
        for (int q = 0; q < kItems && base + q < n; ++q) m |= ((a[base + q] != 0) == (want != 0) ? 1u : 0u) << q;
        return m;
    }
};

template <class M, class Item, class Out>
cudaError_t compact_m(M p, Item item, long long n, Out* out, long long* d_count, void* scratch, size_t scratch_size,
                      cudaStream_t s) {
    if (n <= 0) return cudaMemsetAsync(d_count, 0, sizeof(long long), s);
    const long long tiles = (n + kTile - 1) / kTile;
    long long* counts = static_cast<long long*>(scratch);
    long long* offsets = counts + (tiles + 1);
    void* scan_tmp = offsets + (tiles + 1);
    size_t scan_bytes = scratch_size - 2 * (tiles + 1) * sizeof(long long);
    cudaError_t e = cudaMemsetAsync(counts + tiles, 0, sizeof(long long), s);
    if (e != cudaSuccess) return e;
    count_tiles_m<<<persistent_grid(tiles), kThreads, 0, s>>>(p, n, tiles, counts);
    e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, offsets, static_cast<int>(tiles + 1), s);
    if (e != cudaSuccess) return e;
    write_tiles_m<<<persistent_grid(tiles), kThreads, 0, s>>>(p, item, n, tiles, offsets, out);
    e = cudaMemcpyAsync(d_count, offsets + tiles, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace lsr_compact
