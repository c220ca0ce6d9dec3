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

}  // namespace lsr_compact
