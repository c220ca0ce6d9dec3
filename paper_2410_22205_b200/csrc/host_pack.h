// Host-side packing for the pipelined one-shot entry (lsr_capi.cu).
//
// One SL step (reference src/evolve.cpp:40-118) reads
//   * the distance field d only at the active nodes and their axis
//     neighbours (the centered gradient, src/grid.cpp:53-74), and
//   * phi only inside a small neighbourhood of each active node: its axis
//     neighbours, the 4x4x4 (WENO) / 2x2x2 (Q1) stencils around its feet and
//     the fallback's neighbour interpolations.
// So the one-shot call uploads d as exactly that set and phi as the
// Chebyshev ball of radius R around every active node (the kernel checks
// each foot stencil against the ball and counts any miss, which reruns the
// step on fully uploaded fields), both packed as x-runs of grid rows.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace lsr_host {

// A fixed set of worker threads that run fn(0..n-1) jobs, items handed out in
// ascending order. run() blocks until the job is done; post() returns at once
// (wait() joins it). One job at a time per pool.
class Pool {
  public:
    explicit Pool(int threads);
    ~Pool();
    int size() const { return static_cast<int>(workers_.size()); }
    void post(int n, std::function<void(int)> fn);
    void wait();
    void run(int n, std::function<void(int)> fn) {
        post(n, std::move(fn));
        wait();
    }

  private:
    void loop();
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    std::function<void(int)> fn_;
    int n_ = 0;
    std::atomic<int> next_{0};
    int busy_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// dst = src for `bytes` bytes with streaming (non-temporal) stores where the
// CPU has them: the destination is not read first and does not evict the
// cache, which matters when host memory bandwidth is the bound
void copy_stream(void* dst, const void* src, size_t bytes);

// one run of consecutive nodes on a grid row: node ids [dst, dst + len)
// live at packed[src, src + len). len is implied by the next run's src.
struct RunDesc {
    int64_t dst;
    int64_t src;
};

struct Run {
    int32_t j, x0, x1;  // row j of a plane, inclusive x range
};

// Per-plane runs of one packed set with the offsets of each plane's values
// and runs in the packed buffers.
struct PackSet {
    std::vector<std::vector<Run>> runs;
    std::vector<int64_t> val_off, run_off;  // nz + 1 prefix sums
    int64_t values_before(int k) const { return val_off[k]; }
    int64_t runs_before(int k) const { return run_off[k]; }
    int64_t total_values() const { return val_off.back(); }
    int64_t total_runs() const { return run_off.back(); }
    void finish_offsets();
};

class StepPacker {
  public:
    // Validates that ids are non-decreasing inside the grid and builds, per
    // z-plane, the runs of the d set ({active} ∪ axis neighbours) and, when
    // reach > 0, of the phi set (all nodes within Chebyshev distance `reach`
    // of an active node). Returns false (nothing planned) when the ids are
    // not ascending.
    bool plan(const int64_t* ids, int64_t n, int nx, int ny, int nz, int reach, int threads);

    const PackSet& dset() const { return d_; }
    const PackSet& phiset() const { return phi_; }
    int reach() const { return reach_; }

    // Copies plane k's values of the planned sets out of the fields (phi_*
    // may be null when no phi set was planned).
    void gather_plane(int k, const double* dist, double* d_vals, RunDesc* d_desc, const double* phi,
                      double* phi_vals, RunDesc* phi_desc) const;

    Pool& pool() { return *pool_; }  // exists after the first plan()
    void wait() {                     // joins a job posted on the pool, if any
        if (pool_) pool_->wait();
    }

  private:
    int nx_ = 0, ny_ = 0, nz_ = 0, reach_ = 0;
    std::vector<std::vector<Run>> active_;  // per plane: runs of active nodes, ascending (j, x0)
    int words_ = 0;                         // 64-bit words per row bitmap
    std::vector<uint64_t> bits_;            // per plane: active runs widened by R in x, row bitmaps
    std::vector<std::vector<Run>> scratch_;
    PackSet d_, phi_;
    std::unique_ptr<Pool> pool_;
};

}  // namespace lsr_host
