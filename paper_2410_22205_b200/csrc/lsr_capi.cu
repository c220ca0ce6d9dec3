// lsr_capi.cu — the C ABI (include/lsr_cuda.h): validation with the
// reference's error semantics, device-resident contexts, and the one-shot
// host entry that stands in for lsr::sl_step (evolve.cpp:40-118).
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>

#include "lsr_cuda.h"
#include "band_launch.h"
#include "prep_launch.h"
#include "sl_launch.h"
#include "host_pack.h"
#include "transfer_launch.h"

using lsr_dev::SlParams;

namespace {

thread_local std::string g_err;
// bytes the last lsr_cuda_sl_step_host call moved host->device / device->host
thread_local int64_t g_h2d_bytes = 0, g_d2h_bytes = 0;
std::atomic<long long> g_launches{0};

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_err(cudaError_t e, const char* what) {
    return set_err(LSR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define LSR_CUDA_TRY(expr)                                     \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_err(_e, #expr);     \
    } while (0)

int64_t num_nodes(const lsr_grid& g) {
    return static_cast<int64_t>(g.dims[0]) * g.dims[1] * g.dims[2];
}

int check_grid(const lsr_grid* g) {
    if (!g) return set_err(LSR_ERR_CONFIG, "grid: null");
    if (g->dim != 2 && g->dim != 3) return set_err(LSR_ERR_CONFIG, "grid: dim must be 2 or 3");
    if (!(g->dx > 0.0)) return set_err(LSR_ERR_CONFIG, "grid: dx must be positive");
    for (int d = 0; d < g->dim; ++d)
        if (g->dims[d] < 2) return set_err(LSR_ERR_CONFIG, "grid: need at least 2 nodes per axis");
    if (g->dim == 2 && g->dims[2] != 1) return set_err(LSR_ERR_CONFIG, "grid: dims[2] must be 1 in 2d");
    return LSR_OK;
}

// StepConfig::validate (evolve.hpp:25-30), BandParams::validate
// (grid.hpp:90-92), the energy check (evolve.cpp:45-46) and the interp
// dispatch error (interp.cpp:118) — all before any device work.
int check_cfg(const lsr_step_cfg* c, double energy_p) {
    if (!c) return set_err(LSR_ERR_CONFIG, "step: null config");
    if (c->p != 1 && c->p != 2) return set_err(LSR_ERR_CONFIG, "step: p must be 1 or 2");
    if (!(c->dt > 0.0)) return set_err(LSR_ERR_CONFIG, "step: dt must be positive");
    if (c->delta < 0.0 || c->delta > 1.0) return set_err(LSR_ERR_CONFIG, "step: delta must be in [0, 1]");
    if (!(c->beta > 0.0) || !(c->beta < c->gamma)) return set_err(LSR_ERR_CONFIG, "band: need 0 < beta < gamma");
    if (c->interp != LSR_INTERP_Q1 && c->interp != LSR_INTERP_WENO)
        return set_err(LSR_ERR_CONFIG, "interp: unknown interpolator kind");
    if (c->p > 1 && !(energy_p > 0.0)) return set_err(LSR_ERR, "sl_step: energy must be positive for p > 1");
    return LSR_OK;
}

bool pow2_range(double c) {  // div_const precondition (sl_device.cuh)
    const double a = std::fabs(c);
    return a >= std::ldexp(1.0, -100) && a <= std::ldexp(1.0, 100);
}

// Host-side precomputation with the reference's own expressions.
SlParams make_params(const lsr_grid& g, const lsr_step_cfg& c, double energy_p) {
    SlParams P{};
    P.dim = g.dim;
    P.nx = g.dims[0];
    P.ny = g.dims[1];
    P.nz = g.dims[2];
    P.nxy = static_cast<long long>(P.nx) * P.ny;
    P.ox = g.origin[0];
    P.oy = g.origin[1];
    P.oz = g.origin[2];
    P.dx = g.dx;
    P.hx = g.origin[0] + (g.dims[0] - 1) * g.dx;  // Grid::upper (grid.hpp:31-34)
    P.hy = g.origin[1] + (g.dims[1] - 1) * g.dx;
    P.hz = g.origin[2] + (g.dims[2] - 1) * g.dx;
    P.inv2 = 1.0 / (2.0 * g.dx);  // grid.cpp:55
    P.inv1 = 1.0 / g.dx;          // grid.cpp:56
    P.dx2 = g.dx * g.dx;
    P.rdx = 1.0 / g.dx;
    P.rdx2 = 1.0 / P.dx2;
    P.r3 = 1.0 / 3.0;
    P.fast_div = (pow2_range(g.dx) && pow2_range(P.dx2)) ? 1 : 0;
    P.fast_weno = (P.fast_div && g.dx >= std::ldexp(1.0, -30) && g.dx <= 1.0) ? 1 : 0;  // weno1_fast's range argument
    P.p = c.p;
    P.pd = static_cast<double>(c.p);
    P.dt = c.dt;
    P.delta = c.delta;
    P.energy = energy_p;
    P.grad_threshold = c.fallback_c * std::pow(c.dt, c.fallback_alpha);  // evolve.cpp:52
    P.gamma = c.gamma;
    P.beta = c.beta;
    P.cut_den = (c.gamma - c.beta) * (c.gamma - c.beta) * (c.gamma - c.beta);  // grid.cpp:142
    P.z_base = 0;
    P.z_planes = g.dims[2];
    P.own_lo = 0;
    P.own_hi = g.dims[2];
    return P;
}

// points the SL kernel at a filled z-line table
void zt_attach(SlParams& P, const ZtBuffers& Z) {
    P.ztab = Z.zt;
    P.zcoef = Z.zc;
    P.ztab_bad = Z.count + 1;
    P.zt_cover = Z.mark;
    P.zt_nbx = (P.nx + kZtBrick - 1) / kZtBrick;
    P.zt_nby = (P.ny + kZtBrick - 1) / kZtBrick;
}

int numerical_error(const lsr_grid& g, unsigned long long bad, int64_t* bad_node) {
    if (bad >= static_cast<unsigned long long>(num_nodes(g)))  // the kernels' mark of an id outside the grid
        return set_err(LSR_ERR_CONFIG, "sl_step: ids must be node ids of the grid");
    if (bad_node) *bad_node = static_cast<int64_t>(bad);
    const int64_t id = static_cast<int64_t>(bad);
    const int i = static_cast<int>(id % g.dims[0]);
    const int j = static_cast<int>((id / g.dims[0]) % g.dims[1]);
    const int k = static_cast<int>(id / (static_cast<int64_t>(g.dims[0]) * g.dims[1]));
    char buf[160];
    std::snprintf(buf, sizeof buf, "sl_step: non-finite update at node (%d, %d, %d)", i, j, k);  // evolve.cpp:115
    return set_err(LSR_ERR_NUMERICAL, buf);
}

}  // namespace

void lsr_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

constexpr int kMaxAsyncSteps = 4096;

struct lsr_cuda_ctx {
    int device = 0;
    lsr_grid grid{};
    int64_t n = 0;
    double* phi = nullptr;
    double* out = nullptr;
    double* dist = nullptr;
    unsigned char* exact = nullptr;  // DistanceField::exact (distance.hpp:16)
    int64_t* active = nullptr;
    int64_t n_active = 0, cap_active = 0;
    int64_t* dirty = nullptr;  // ids where out may differ from phi
    int64_t n_dirty = 0, cap_dirty = 0;
    bool consistent = false;   // out == phi except at `dirty`
    unsigned long long* d_bad = nullptr;
    unsigned long long* h_bad = nullptr;  // pinned
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // start, table filled, SL start, SL done
    float kernel_ms = 0.f, step_ms = 0.f, table_ms = 0.f;
    int64_t n_interface_cells = 0;
    BandBuffers band;        // last narrow_band built on the device
    ReinitBuffers rb;        // reinitialisation scratch
    double* scratch = nullptr;  // third full-grid field (reinit double buffer)
    // z-slab context (lsr_cuda_slab_create): fields hold the resident planes
    // [win_lo, win_hi) of the global grid `grid`; work is done on the owned
    // planes [own_lo, own_hi); n = resident nodes
    // the loop's clamp bookkeeping: `phi` was fully clamped to clamped_gamma
    // by the loop step that set clamped_seq, and no entry point that may
    // write phi or out (each bumps seq) ran since
    uint64_t seq = 1, clamped_seq = 0;
    const double* clamped_phi = nullptr;
    double clamped_gamma = 0.0;
    // SL step form for 3d WENO: 0 = z-line table (default), 1 = TMA bricks
    // (sl_step_box_kernel); the brick grouping is kept per active set
    int sl_mode = 0;
    BoxBuffers box{};
    long long box_nb = 0, box_cap_ids = 0, box_listed = 0;
    bool box_valid = false;
    bool slab = false;
    int win_lo = 0, win_hi = 0, own_lo = 0, own_hi = 0;
    EnergySlabWork ew;
    // the device-controlled loop (lsr_cuda_loop_run): its device words,
    // per-iteration records, count estimates and captured iteration graphs
    struct LoopRun {
        EnergyLoopWork ew;
        ReinitLoopDev* rl = nullptr;
        double* e2 = nullptr;
        int* flags = nullptr;
        int* k = nullptr;
        int* hard = nullptr;    // [0] dense one-step this iteration, [1] a hard jump found for the next
        void* stats = nullptr;  // LoopDevStat[cap]
        int cap = 0;
        long long est_active = 0, est_cells = 0;
        cudaGraphExec_t exec[2] = {nullptr, nullptr};
        std::string key[2];
        int64_t launches[2] = {0, 0};  // kernels per replay (for lsr_cuda_kernel_launches)
    } lr;
    long long reinit_nn = 0;
    unsigned long long* d_aux = nullptr;  // [0] halo misses, [1] reach bits
    // pipelined host entry: compute / D2H streams, per-chunk events, miss counter
    cudaStream_t s_cmp = nullptr, s_down = nullptr;
    cudaEvent_t ev_up[32] = {}, ev_cmp[32] = {};
    unsigned long long* d_miss = nullptr;
    int64_t pipeline_fallbacks = 0;
    // pipelined host entry, packed transfers (host_pack.h): pinned staging and
    // device copies of the packed d and phi sets and of the chunk results
    lsr_host::StepPacker packer;
    std::unique_ptr<lsr_host::Pool> copy_pool;  // host out = phi copy and result scatter
    int reach = 5;  // Chebyshev radius of the packed phi set; 0 = upload phi whole
    cudaEvent_t ev_down[32] = {};
    struct Packed {
        double* h_vals = nullptr;
        lsr_host::RunDesc* h_desc = nullptr;
        double* d_vals = nullptr;
        long long* d_desc = nullptr;  // RunDesc pairs (dst, src)
        int64_t cap_hv = 0, cap_hd = 0, cap_dv = 0, cap_dd = 0;
    } pk_d, pk_phi;
    double* h_res = nullptr;
    double* d_res = nullptr;
    int64_t cap_hres = 0, cap_dres = 0;
    unsigned long long* bm = nullptr;  // node bitmaps of the zero-copy pull (transfer.cu)
    int64_t cap_bm = 0;
    ZtBuffers zt{};  // z-line table of the 3d WENO path (sl_launch.h)
    double* bd = nullptr;    // per-brick max d and max |grad d| (launch_brick_d); valid for the current d:
    bool bd_valid = false;
    bool zt_bricks = false;  // zt.list holds the covered bricks of the current active set ...
    double zt_key[4] = {0, 0, 0, 0};  // ... for this (E, dt, delta, p) (and the current d)
    cudaStream_t s_aux = nullptr;  // resync beside the table fill
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool dirty_is_active = false;  // `dirty` holds the current active ids
    // asynchronous steps since the last lsr_cuda_sync: their timing events,
    // whether they used the table, and the times read at the sync
    int async_n = 0;
    std::vector<std::array<cudaEvent_t, 4>> aev;
    bool aused[kMaxAsyncSteps] = {};
    std::vector<float> async_kernel_ms, async_step_ms, async_table_ms;
};

namespace {

int ensure_ids(int64_t** buf, int64_t* cap, int64_t n) {
    if (n <= *cap) return LSR_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    const int64_t c = n + n / 4 + 1024;
    LSR_CUDA_TRY(cudaMalloc(buf, sizeof(int64_t) * c));
    *cap = c;
    return LSR_OK;
}

// every id a node of the grid (0 <= id < n)? Active ids are dereferenced
// by the kernels and by the host scatter, so they are checked before any of
// that (the reference's BandMask holds node ids by construction,
// grid.hpp:79-84). Large lists are scanned by several threads.
bool ids_in_grid(const int64_t* ids, int64_t n, int64_t n_nodes) {
    const auto scan = [=](int64_t t0, int64_t t1) {
        bool ok = true;
        for (int64_t t = t0; t < t1; ++t) ok &= static_cast<uint64_t>(ids[t]) < static_cast<uint64_t>(n_nodes);
        return ok;
    };
    const int64_t kSerial = 1 << 20;
    if (n <= kSerial) return scan(0, n);
    const int nt = static_cast<int>(std::min<int64_t>(8, n / kSerial + 1));
    std::vector<std::thread> th;
    std::vector<char> ok(nt, 1);
    for (int q = 0; q < nt; ++q)
        th.emplace_back([&, q] { ok[q] = scan(n * q / nt, n * (q + 1) / nt); });
    for (auto& t : th) t.join();
    for (char v : ok)
        if (!v) return false;
    return true;
}

double** field_slot(lsr_cuda_ctx* c, int which) {
    switch (which) {
        case LSR_FIELD_PHI: return &c->phi;
        case LSR_FIELD_DIST: return &c->dist;
        case LSR_FIELD_OUT: return &c->out;
        case LSR_FIELD_SCRATCH: return c->scratch ? &c->scratch : nullptr;  // once allocated
    }
    return nullptr;
}

}  // namespace

extern "C" {

const char* lsr_cuda_last_error_string(void) { return g_err.c_str(); }

int64_t lsr_cuda_kernel_launches(void) { return g_launches.load(); }

void lsr_cuda_last_transfer_bytes(int64_t* h2d, int64_t* d2h) {
    if (h2d) *h2d = g_h2d_bytes;
    if (d2h) *d2h = g_d2h_bytes;
}

int lsr_cuda_create(int device, const lsr_grid* grid, lsr_cuda_ctx** out) {
    if (!out) return set_err(LSR_ERR_CONFIG, "create: null out");
    *out = nullptr;
    if (int st = check_grid(grid)) return st;
    LSR_CUDA_TRY(cudaSetDevice(device));
    auto* c = new lsr_cuda_ctx;
    c->device = device;
    c->grid = *grid;
    c->n = num_nodes(*grid);
    const size_t bytes = sizeof(double) * static_cast<size_t>(c->n);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&c->phi, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->out, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->dist, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_bad, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_bad, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e != cudaSuccess) {
        lsr_cuda_destroy(c);
        return cuda_err(e, "lsr_cuda_create");
    }
    c->stream = c->own;
    *out = c;
    return LSR_OK;
}

int lsr_cuda_destroy(lsr_cuda_ctx* c) {
    if (!c) return LSR_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->phi);
    cudaFree(c->out);
    cudaFree(c->dist);
    cudaFree(c->exact);
    cudaFree(c->scratch);
    c->ew.release();
    c->lr.ew.release();
    cudaFree(c->lr.rl);
    cudaFree(c->lr.e2);
    cudaFree(c->lr.flags);
    cudaFree(c->lr.k);
    cudaFree(c->lr.hard);
    cudaFree(c->lr.stats);
    for (auto& g : c->lr.exec)
        if (g) cudaGraphExecDestroy(g);
    cudaFree(c->d_aux);
    c->band.release();
    c->rb.release();
    cudaFree(c->d_miss);
    c->copy_pool.reset();
    for (auto* q : {&c->pk_d, &c->pk_phi}) {
        if (q->h_vals) cudaFreeHost(q->h_vals);
        if (q->h_desc) cudaFreeHost(q->h_desc);
        cudaFree(q->d_vals);
        cudaFree(q->d_desc);
    }
    if (c->h_res) cudaFreeHost(c->h_res);
    cudaFree(c->d_res);
    cudaFree(c->bm);
    cudaFree(c->zt.zt);
    cudaFree(c->zt.zc);
    cudaFree(c->zt.mark);
    cudaFree(c->zt.reach);
    cudaFree(c->zt.list);
    cudaFree(c->zt.count);
    cudaFree(c->bd);
    cudaFree(c->box.count);
    cudaFree(c->box.off);
    cudaFree(c->box.cursor);
    cudaFree(c->box.list);
    cudaFree(c->box.d_listed);
    cudaFree(c->box.ids);
    cudaFree(c->box.tmp);
    for (auto& e : c->ev_down)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->ev_up)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->ev_cmp)
        if (e) cudaEventDestroy(e);
    if (c->s_cmp) cudaStreamDestroy(c->s_cmp);
    if (c->s_aux) cudaStreamDestroy(c->s_aux);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    for (auto& e : c->aev)
        for (auto& x : e) cudaEventDestroy(x);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->s_down) cudaStreamDestroy(c->s_down);
    cudaFree(c->active);
    cudaFree(c->dirty);
    cudaFree(c->d_bad);
    if (c->h_bad) cudaFreeHost(c->h_bad);
    for (auto& ev : c->ev)
        if (ev) cudaEventDestroy(ev);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
    return LSR_OK;
}

int lsr_cuda_set_stream(lsr_cuda_ctx* c, void* stream) {
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
    return LSR_OK;
}

int lsr_cuda_upload_field(lsr_cuda_ctx* c, int which, const double* host) {
    if (!c || !host) return set_err(LSR_ERR_CONFIG, "upload: null argument");
    double** slot = field_slot(c, which);
    if (!slot) return set_err(LSR_ERR_CONFIG, "upload: unknown field");
    c->seq++;  // may write phi or out
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    LSR_CUDA_TRY(cudaMemcpyAsync(*slot, host, sizeof(double) * c->n, cudaMemcpyHostToDevice, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (which != LSR_FIELD_DIST) c->consistent = false;
    else c->zt_bricks = c->bd_valid = false;  // d changed: its covered bricks and per-brick maxima
    c->box_valid = false;  // the covered bricks depend on d
    return LSR_OK;
}

int lsr_cuda_download_field(lsr_cuda_ctx* c, int which, double* host) {
    if (!c || !host) return set_err(LSR_ERR_CONFIG, "download: null argument");
    double** slot = field_slot(c, which);
    if (!slot) return set_err(LSR_ERR_CONFIG, "download: unknown field");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    LSR_CUDA_TRY(cudaMemcpyAsync(host, *slot, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LSR_OK;
}

int lsr_cuda_field_ptr(lsr_cuda_ctx* c, int which, double** dptr) {
    if (!c || !dptr) return set_err(LSR_ERR_CONFIG, "field_ptr: null argument");
    double** slot = field_slot(c, which);
    if (!slot) return set_err(LSR_ERR_CONFIG, "field_ptr: unknown field");
    c->seq++;  // may write phi or out
    *dptr = *slot;
    return LSR_OK;
}

int lsr_cuda_mark_dirty(lsr_cuda_ctx* c, int which) {
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    c->seq++;  // may write phi or out
    if (which != LSR_FIELD_DIST) c->consistent = false;
    else c->zt_bricks = c->bd_valid = false;  // d changed: its covered bricks and per-brick maxima
    c->box_valid = false;
    return LSR_OK;
}

int lsr_cuda_set_active(lsr_cuda_ctx* c, const int64_t* ids, int64_t n) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "set_active: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || (n > 0 && !ids) || n < 0) return set_err(LSR_ERR_CONFIG, "set_active: bad argument");
    if (!ids_in_grid(ids, n, c->n)) return set_err(LSR_ERR_CONFIG, "set_active: ids must be node ids of the grid");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (int st = ensure_ids(&c->active, &c->cap_active, n)) return st;
    if (n > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->n_active = n;
    c->zt_bricks = false;
    c->box_valid = false;
    c->dirty_is_active = false;
    return LSR_OK;
}

int lsr_cuda_set_active_device(lsr_cuda_ctx* c, const int64_t* d_ids, int64_t n) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "set_active_device: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || (n > 0 && !d_ids) || n < 0) return set_err(LSR_ERR_CONFIG, "set_active_device: bad argument");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (int st = ensure_ids(&c->active, &c->cap_active, n)) return st;
    if (n > 0) {
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, d_ids, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c->stream));
        // the range check before any kernel dereferences them
        LSR_CUDA_TRY(cudaMemsetAsync(c->d_bad, 0, sizeof(unsigned long long), c->stream));
        LSR_CUDA_TRY(launch_check_ids(c->active, n, c->n, c->d_bad, c->stream));
        LSR_CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                     c->stream));
        LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (*c->h_bad != 0) {
            c->n_active = 0;
            return set_err(LSR_ERR_CONFIG, "set_active_device: ids must be node ids of the grid");
        }
    }
    c->n_active = n;
    c->zt_bricks = false;
    c->box_valid = false;
    c->dirty_is_active = false;
    return LSR_OK;
}

namespace {

// Enqueues one SL step on the context stream (resync of out, z-line table,
// SL kernel, dirty-id bookkeeping) with timing events ev[0..3] = start, table
// filled, SL kernel start, SL kernel end; no host synchronisation.
int enqueue_step(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, double energy_p, bool reset_bad, cudaEvent_t* ev,
                 bool* used_table) {
    SlParams P = make_params(c->grid, *cfg, energy_p);
    cudaStream_t s = c->stream;
    // delta = 0: the four feet coincide and one interpolation per node does
    // not amortise the fill (1.31 vs 1.27 ms at 512^3), so no table
    const bool use_box = c->sl_mode == 1 && c->grid.dim == 3 && cfg->interp == 1 && P.fast_weno;
    const bool use_table = !use_box && LSR_ZTAB && c->grid.dim == 3 && cfg->interp == 1 && P.fast_weno &&
                           c->grid.dims[2] >= 4 && cfg->delta > 0.0;
    if (use_box && !c->box_valid) {
        const long long nb = static_cast<long long>((c->grid.dims[0] + 7) / 8) * ((c->grid.dims[1] + 7) / 8) *
                             ((c->grid.dims[2] + 7) / 8);
        if (nb > c->box_nb) {
            for (void* q : {static_cast<void*>(c->box.count), static_cast<void*>(c->box.off),
                            static_cast<void*>(c->box.cursor), static_cast<void*>(c->box.list), c->box.tmp})
                cudaFree(q);
            c->box.tmp_bytes = box_tmp_bytes(nb);
            LSR_CUDA_TRY(cudaMalloc(&c->box.count, sizeof(unsigned) * (nb + 1)));
            LSR_CUDA_TRY(cudaMalloc(&c->box.off, sizeof(unsigned) * (nb + 1)));
            LSR_CUDA_TRY(cudaMalloc(&c->box.cursor, sizeof(unsigned) * nb));
            LSR_CUDA_TRY(cudaMalloc(&c->box.list, sizeof(unsigned) * nb));
            LSR_CUDA_TRY(cudaMalloc(&c->box.tmp, c->box.tmp_bytes));
            if (!c->box.d_listed) LSR_CUDA_TRY(cudaMalloc(&c->box.d_listed, sizeof(long long)));
            c->box_nb = nb;
        }
        if (c->n_active > c->box_cap_ids) {
            cudaFree(c->box.ids);
            LSR_CUDA_TRY(cudaMalloc(&c->box.ids, sizeof(int64_t) * static_cast<size_t>(c->n_active)));
            c->box_cap_ids = c->n_active;
        }
        LSR_CUDA_TRY(launch_box_bricks(P, c->active, c->n_active, c->box, &c->box_listed, s));
        c->box_valid = true;
    }
    if (use_table && !c->s_aux) {
        LSR_CUDA_TRY(cudaStreamCreateWithFlags(&c->s_aux, cudaStreamNonBlocking));
        LSR_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        LSR_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    // the resync runs beside the table fill (different buffers) on s_aux
    cudaStream_t sr = use_table ? c->s_aux : s;
    LSR_CUDA_TRY(cudaEventRecord(ev[0], s));
    if (use_table) {
        LSR_CUDA_TRY(cudaEventRecord(c->ev_fork, s));
        LSR_CUDA_TRY(cudaStreamWaitEvent(sr, c->ev_fork, 0));
    }
    // "non-active nodes carry phi over" (evolve.cpp:50) without the O(N) copy
    // when out is known to equal phi except at the previous step's ids.
    if (!c->consistent) {
        LSR_CUDA_TRY(cudaMemcpyAsync(c->out, c->phi, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, sr));
    } else {
        LSR_CUDA_TRY(launch_resync(c->phi, c->out, c->dirty, c->n_dirty, c->n, sr));
    }
    if (reset_bad) LSR_CUDA_TRY(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), sr));
    // 3d WENO: the z-line table of phi on the bricks around the active set
    // (sl_step.cu); the brick list depends on the ids only and is kept until
    // the active set changes
    if (use_table) {
        if (!c->zt.zt) {
            const long long nb = zt_num_bricks(c->grid.dims);
            LSR_CUDA_TRY(cudaMalloc(&c->zt.zt, sizeof(double) * 4 * static_cast<size_t>(c->n)));
            LSR_CUDA_TRY(cudaMalloc(&c->zt.zc, sizeof(double) * 2 * static_cast<size_t>(c->n)));
            LSR_CUDA_TRY(cudaMalloc(&c->zt.mark, static_cast<size_t>(nb)));
            LSR_CUDA_TRY(cudaMalloc(&c->zt.reach, sizeof(unsigned) * static_cast<size_t>(nb)));
            LSR_CUDA_TRY(cudaMalloc(&c->zt.list, sizeof(unsigned) * static_cast<size_t>(nb)));
            LSR_CUDA_TRY(cudaMalloc(&c->zt.count, 2 * sizeof(unsigned)));
        }
        const double key[4] = {energy_p, cfg->dt, cfg->delta, static_cast<double>(cfg->p)};
        if (!c->zt_bricks || std::memcmp(key, c->zt_key, sizeof key) != 0) {
            LSR_CUDA_TRY(launch_zt_bricks(P, c->dist, c->active, c->n_active, c->zt, s));
            std::memcpy(c->zt_key, key, sizeof key);
            c->zt_bricks = true;
        }
        LSR_CUDA_TRY(launch_zt_fill(P, c->phi, c->zt, s));
        zt_attach(P, c->zt);
    }
    LSR_CUDA_TRY(cudaEventRecord(ev[1], s));
    if (use_table) {
        LSR_CUDA_TRY(cudaEventRecord(c->ev_join, sr));
        LSR_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_join, 0));
    }
    LSR_CUDA_TRY(cudaEventRecord(ev[2], s));
    if (!(use_box && launch_sl_step_box(P, c->phi, c->dist, c->box, c->box_listed, c->n_active, c->out, c->d_bad, s)))
        LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, c->phi, c->dist, c->active, c->n_active, c->out, c->d_bad, s));
    LSR_CUDA_TRY(cudaGetLastError());
    LSR_CUDA_TRY(cudaEventRecord(ev[3], s));
    // the ids written now are where out may differ from phi after the swap
    if (!c->dirty_is_active) {
        if (int st = ensure_ids(&c->dirty, &c->cap_dirty, c->n_active)) return st;
        if (c->n_active > 0)
            LSR_CUDA_TRY(cudaMemcpyAsync(c->dirty, c->active, sizeof(int64_t) * c->n_active,
                                         cudaMemcpyDeviceToDevice, s));
        c->n_dirty = c->n_active;
        c->dirty_is_active = true;
    }
    c->consistent = true;
    *used_table = use_table;
    return LSR_OK;
}

}  // namespace

int lsr_cuda_sl_step(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, double energy_p, int64_t* bad_node) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "sl_step: a z-slab context (use lsr_cuda_slab_*)");
    if (bad_node) *bad_node = -1;
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    c->seq++;  // may write phi or out
    if (int st = check_cfg(cfg, energy_p)) return st;
    if (c->async_n > 0) return set_err(LSR_ERR_CONFIG, "sl_step: asynchronous steps pending (call lsr_cuda_sync)");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    bool use_table = false;
    if (int st = enqueue_step(c, cfg, energy_p, true, c->ev, &use_table)) return st;
    cudaStream_t s = c->stream;
    LSR_CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    LSR_CUDA_TRY(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&c->kernel_ms, c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&c->step_ms, c->ev[0], c->ev[3]);
    c->table_ms = 0.f;
    if (use_table) cudaEventElapsedTime(&c->table_ms, c->ev[0], c->ev[1]);
    if (*c->h_bad != ~0ULL) return numerical_error(c->grid, *c->h_bad, bad_node);
    return LSR_OK;
}

int lsr_cuda_sl_step_async(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, double energy_p) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "sl_step_async: a z-slab context (use lsr_cuda_slab_*)");
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    c->seq++;  // may write phi or out
    if (int st = check_cfg(cfg, energy_p)) return st;
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (c->async_n >= kMaxAsyncSteps) return set_err(LSR_ERR_CONFIG, "sl_step_async: too many pending steps");
    while (static_cast<int>(c->aev.size()) <= c->async_n) {
        std::array<cudaEvent_t, 4> e{};
        for (auto& x : e) LSR_CUDA_TRY(cudaEventCreate(&x));
        c->aev.push_back(e);
    }
    bool use_table = false;
    if (int st = enqueue_step(c, cfg, energy_p, c->async_n == 0, c->aev[c->async_n].data(), &use_table)) return st;
    c->aused[c->async_n] = use_table;
    ++c->async_n;
    return LSR_OK;
}

int lsr_cuda_sync(lsr_cuda_ctx* c, int64_t* bad_node) {
    if (bad_node) *bad_node = -1;
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int n = c->async_n;
    if (n > 0) LSR_CUDA_TRY(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    LSR_CUDA_TRY(cudaStreamSynchronize(s));
    c->async_kernel_ms.assign(n, 0.f);
    c->async_step_ms.assign(n, 0.f);
    c->async_table_ms.assign(n, 0.f);
    for (int i = 0; i < n; ++i) {
        const auto& e = c->aev[i];
        cudaEventElapsedTime(&c->async_kernel_ms[i], e[2], e[3]);
        cudaEventElapsedTime(&c->async_step_ms[i], e[0], e[3]);
        if (c->aused[i]) cudaEventElapsedTime(&c->async_table_ms[i], e[0], e[1]);
    }
    c->async_n = 0;
    if (n > 0 && *c->h_bad != ~0ULL) return numerical_error(c->grid, *c->h_bad, bad_node);
    return LSR_OK;
}

int lsr_cuda_async_times(lsr_cuda_ctx* c, float* kernel_ms, float* step_ms, float* table_ms, int cap, int* n) {
    if (!c || !n) return set_err(LSR_ERR_CONFIG, "async_times: null argument");
    const int m = std::min<int>(cap, static_cast<int>(c->async_kernel_ms.size()));
    for (int i = 0; i < m; ++i) {
        if (kernel_ms) kernel_ms[i] = c->async_kernel_ms[i];
        if (step_ms) step_ms[i] = c->async_step_ms[i];
        if (table_ms) table_ms[i] = c->async_table_ms[i];
    }
    *n = m;
    return LSR_OK;
}

int lsr_cuda_set_sl_mode(lsr_cuda_ctx* c, int mode) {
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    if (mode != 0 && mode != 1) return set_err(LSR_ERR_CONFIG, "set_sl_mode: 0 (z-line table) or 1 (TMA bricks)");
    c->sl_mode = mode;
    return LSR_OK;
}

int lsr_cuda_swap(lsr_cuda_ctx* c) {
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    c->seq++;  // may write phi or out
    std::swap(c->phi, c->out);  // out and phi still differ only at `dirty`
    return LSR_OK;
}

int lsr_cuda_last_table_ms(lsr_cuda_ctx* c, float* table_ms) {
    if (!c || !table_ms) return set_err(LSR_ERR_CONFIG, "null argument");
    *table_ms = c->table_ms;
    return LSR_OK;
}

int lsr_cuda_last_times(lsr_cuda_ctx* c, float* kernel_ms, float* step_ms) {
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    if (kernel_ms) *kernel_ms = c->kernel_ms;
    if (step_ms) *step_ms = c->step_ms;
    return LSR_OK;
}

namespace {

// z-line table buffers of the stateless device entries (slab mode), one set
// per host thread, device and stream (launches on one stream are ordered, so
// reusing the set is safe), grown on demand; the brick list is rebuilt every
// call since the caller's ids may change between calls
struct SlabTable {
    int device = -1;
    cudaStream_t stream = nullptr;
    long long nodes = 0, bricks = 0;
    ZtBuffers Z{};
    void release() {
        cudaFree(Z.zt);
        cudaFree(Z.zc);
        cudaFree(Z.mark);
        cudaFree(Z.reach);
        cudaFree(Z.list);
        cudaFree(Z.count);
        Z = ZtBuffers{};
        nodes = bricks = 0;
    }
    ~SlabTable() { release(); }
};
thread_local std::vector<std::unique_ptr<SlabTable>> g_slab_tables;

// attaches a z-line table of the resident planes to P (3d WENO only);
// P.z_base/z_planes must be set, phi_g is the global-id-shifted phi
int attach_slab_table(SlParams& P, const lsr_grid& g, int interp, const double* phi_g, const double* dist_g,
                      const int64_t* d_active, int64_t n_active, cudaStream_t s) {
    if (!(LSR_ZTAB && g.dim == 3 && interp == 1 && P.fast_weno && P.z_planes >= 4 && n_active > 0 && P.delta > 0.0))
        return LSR_OK;
    int dev = 0;
    LSR_CUDA_TRY(cudaGetDevice(&dev));
    SlabTable* tp = nullptr;
    for (auto& t : g_slab_tables)
        if (t->device == dev && t->stream == s) tp = t.get();
    if (!tp) {
        g_slab_tables.push_back(std::make_unique<SlabTable>());
        tp = g_slab_tables.back().get();
        tp->device = dev;
        tp->stream = s;
    }
    SlabTable& T = *tp;
    const long long nodes = static_cast<long long>(P.z_planes) * P.nxy;
    const long long bricks = zt_num_bricks(g.dims);
    if (T.nodes < nodes || T.bricks < bricks) {
        T.release();
        LSR_CUDA_TRY(cudaMalloc(&T.Z.zt, sizeof(double) * 4 * static_cast<size_t>(nodes)));
        LSR_CUDA_TRY(cudaMalloc(&T.Z.zc, sizeof(double) * 2 * static_cast<size_t>(nodes)));
        LSR_CUDA_TRY(cudaMalloc(&T.Z.mark, static_cast<size_t>(bricks)));
        LSR_CUDA_TRY(cudaMalloc(&T.Z.reach, sizeof(unsigned) * static_cast<size_t>(bricks)));
        LSR_CUDA_TRY(cudaMalloc(&T.Z.list, sizeof(unsigned) * static_cast<size_t>(bricks)));
        LSR_CUDA_TRY(cudaMalloc(&T.Z.count, 2 * sizeof(unsigned)));
        T.nodes = nodes;
        T.bricks = bricks;
    }
    const long long shift = static_cast<long long>(P.z_base) * P.nxy;
    ZtBuffers Zg = T.Z;  // indexed by global node id
    Zg.zt -= 4 * shift;
    Zg.zc -= 2 * shift;
    LSR_CUDA_TRY(launch_zt_bricks(P, dist_g, d_active, n_active, Zg, s));
    LSR_CUDA_TRY(launch_zt_fill(P, phi_g, Zg, s));
    zt_attach(P, Zg);
    return LSR_OK;
}

}  // namespace

int lsr_cuda_sl_step_device(const lsr_grid* grid, int32_t z_base, int32_t z_planes, const double* d_phi,
                            const double* d_dist, const int64_t* d_active, int64_t n_active,
                            const lsr_step_cfg* cfg, double energy_p, double* d_out, int64_t* d_bad_node,
                            int64_t* d_halo_miss, void* stream) {
    if (int st = check_grid(grid)) return st;
    if (int st = check_cfg(cfg, energy_p)) return st;
    const bool slab = z_base != 0 || z_planes != grid->dims[2];
    if (slab && (grid->dim != 3 || z_base < 0 || z_planes < 1 || z_base + z_planes > grid->dims[2]))
        return set_err(LSR_ERR_CONFIG, "sl_step_device: slabs are z-plane ranges of a 3d grid");
    if (slab && !d_halo_miss) return set_err(LSR_ERR_CONFIG, "sl_step_device: slab mode needs a halo_miss counter");
    SlParams P = make_params(*grid, *cfg, energy_p);
    P.z_base = z_base;
    P.z_planes = z_planes;
    P.own_lo = z_base;  // ids outside the resident planes are counted, never read or written
    P.own_hi = z_base + z_planes;
    P.halo_miss = slab ? reinterpret_cast<unsigned long long*>(d_halo_miss) : nullptr;
    // the resident planes start at global plane z_base: shift the bases so
    // that global ids index them directly
    const long long shift = static_cast<long long>(z_base) * grid->dims[0] * grid->dims[1];
    if (int st = attach_slab_table(P, *grid, cfg->interp, d_phi - shift, d_dist - shift, d_active, n_active,
                                   static_cast<cudaStream_t>(stream)))
        return st;
    LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, d_phi - shift, d_dist - shift, d_active, n_active, d_out - shift,
                                reinterpret_cast<unsigned long long*>(d_bad_node), static_cast<cudaStream_t>(stream)));
    return LSR_OK;
}

int lsr_cuda_sl_step_device_fused(const lsr_grid* grid, int32_t z_base, int32_t z_planes, int32_t own_lo,
                                  int32_t own_hi, const double* d_phi, const double* d_dist, const int64_t* d_active,
                                  int64_t n_active, const lsr_step_cfg* cfg, double energy_p, double* d_out,
                                  double* d_peer_lo_out, int32_t peer_lo_zbase, int32_t push_lo_planes,
                                  double* d_peer_hi_out, int32_t peer_hi_zbase, int32_t push_hi_planes,
                                  int64_t* d_bad_node, int64_t* d_halo_miss, void* stream) {
    if (int st = check_grid(grid)) return st;
    if (int st = check_cfg(cfg, energy_p)) return st;
    if (grid->dim != 3 || z_base < 0 || z_planes < 1 || z_base + z_planes > grid->dims[2] || own_lo < z_base ||
        own_hi > z_base + z_planes || own_lo >= own_hi || !d_halo_miss)
        return set_err(LSR_ERR_CONFIG, "sl_step_device_fused: bad slab description");
    SlParams P = make_params(*grid, *cfg, energy_p);
    const long long nxy = static_cast<long long>(grid->dims[0]) * grid->dims[1];
    P.z_base = z_base;
    P.z_planes = z_planes;
    P.own_lo = own_lo;
    P.own_hi = own_hi;
    P.halo_miss = reinterpret_cast<unsigned long long*>(d_halo_miss);
    // peer buffers hold their owners' resident planes: shift to global ids
    P.peer_lo = d_peer_lo_out ? d_peer_lo_out - static_cast<long long>(peer_lo_zbase) * nxy : nullptr;
    P.peer_hi = d_peer_hi_out ? d_peer_hi_out - static_cast<long long>(peer_hi_zbase) * nxy : nullptr;
    P.push_lo_below = own_lo + push_lo_planes;
    P.push_hi_from = own_hi - push_hi_planes;
    const long long shift = static_cast<long long>(z_base) * nxy;
    if (int st = attach_slab_table(P, *grid, cfg->interp, d_phi - shift, d_dist - shift, d_active, n_active,
                                   static_cast<cudaStream_t>(stream)))
        return st;
    LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, d_phi - shift, d_dist - shift, d_active, n_active, d_out - shift,
                                reinterpret_cast<unsigned long long*>(d_bad_node), static_cast<cudaStream_t>(stream)));
    return LSR_OK;
}

int lsr_cuda_malloc(size_t bytes, void** dptr) {
    if (!dptr) return set_err(LSR_ERR_CONFIG, "malloc: null out");
    LSR_CUDA_TRY(cudaMalloc(dptr, bytes));
    return LSR_OK;
}

int lsr_cuda_free(void* dptr) {
    LSR_CUDA_TRY(cudaFree(dptr));
    return LSR_OK;
}

int lsr_cuda_ipc_handle(void* dptr, uint8_t* handle64) {
    cudaIpcMemHandle_t h;
    LSR_CUDA_TRY(cudaIpcGetMemHandle(&h, dptr));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle64, &h, sizeof h);
    return LSR_OK;
}

int lsr_cuda_ipc_open(const uint8_t* handle64, void** dptr) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    LSR_CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return LSR_OK;
}

int lsr_cuda_ipc_close(void* dptr) {
    LSR_CUDA_TRY(cudaIpcCloseMemHandle(dptr));
    return LSR_OK;
}

// The one-shot host entry, pipelined over z-chunks for 3d grids: the H2D
// of phi (plane order) and of the packed d values, the SL kernel of each
// chunk (as soon as its planes plus a halo are resident) and the D2H of
// finished out planes run on three streams, so the PCIe directions overlap
// each other and the compute. d is read only at active nodes and their axis
// neighbours, so host threads gather exactly those values (as row runs,
// host_pack.h) into pinned staging while phi streams up, and a device kernel
// scatters them into place. Each chunk runs the kernel in slab mode: a
// stencil that reaches a plane not yet uploaded is counted, and any count
// makes the whole step rerun unpipelined with all of d resident (exact
// either way). Ids that are not ascending skip the pipeline altogether.
static constexpr int kNotPipelined = -1000;

static int host_threads() {
    static const int n = [] {
        if (const char* e = std::getenv("LSR_HOST_THREADS")) return std::max(1, std::atoi(e));
        return static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
    }();
    return n;
}

extern "C++" {
template <class T>
static int ensure_pinned(T** buf, int64_t* cap, int64_t n) {
    if (n <= *cap) return LSR_OK;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *cap = 0;
    const int64_t c = n + n / 4 + 4096;
    LSR_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(buf), sizeof(T) * c, cudaHostAllocDefault));
    *cap = c;
    return LSR_OK;
}

template <class T>
static int ensure_device(T** buf, int64_t* cap, int64_t n) {
    if (n <= *cap) return LSR_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    const int64_t c = n + n / 4 + 4096;
    LSR_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(buf), sizeof(T) * c));
    *cap = c;
    return LSR_OK;
}

}  // extern "C++"

// copies one packed set's chunk [z0, z1) to the device and counts the bytes
static int upload_set(const lsr_host::PackSet& ps, lsr_cuda_ctx::Packed& q, int z0, int z1, cudaStream_t s,
                      int64_t* h2d) {
    const int64_t v0 = ps.values_before(z0), v1 = ps.values_before(z1);
    const int64_t r0 = ps.runs_before(z0), r1 = ps.runs_before(z1);
    if (v1 <= v0) return LSR_OK;
    LSR_CUDA_TRY(cudaMemcpyAsync(q.d_vals + v0, q.h_vals + v0, sizeof(double) * (v1 - v0), cudaMemcpyHostToDevice, s));
    LSR_CUDA_TRY(cudaMemcpyAsync(q.d_desc + 2 * r0, q.h_desc + r0, sizeof(lsr_host::RunDesc) * (r1 - r0),
                                 cudaMemcpyHostToDevice, s));
    *h2d += static_cast<int64_t>(sizeof(double)) * (v1 - v0) +
            static_cast<int64_t>(sizeof(lsr_host::RunDesc)) * (r1 - r0);
    return LSR_OK;
}

static int ensure_set(const lsr_host::PackSet& ps, lsr_cuda_ctx::Packed& q) {
    if (int st = ensure_pinned(&q.h_vals, &q.cap_hv, ps.total_values())) return st;
    if (int st = ensure_pinned(&q.h_desc, &q.cap_hd, ps.total_runs())) return st;
    if (int st = ensure_device(&q.d_vals, &q.cap_dv, ps.total_values())) return st;
    return ensure_device(reinterpret_cast<lsr_host::RunDesc**>(&q.d_desc), &q.cap_dd, ps.total_runs());
}

// the device address of n doubles of mapped (pinned) host memory, or null
// when the GPU cannot read the whole range directly
static const double* mapped_ptr(const double* h, int64_t n) {
    cudaPointerAttributes a{}, b{};
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess || cudaPointerGetAttributes(&b, h + (n - 1)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type != cudaMemoryTypeHost || b.type != cudaMemoryTypeHost || !a.devicePointer || !b.devicePointer)
        return nullptr;
    const double* d = static_cast<const double*>(a.devicePointer);
    return static_cast<const double*>(b.devicePointer) == d + (n - 1) ? d : nullptr;
}

struct Finally {
    std::function<void()> f;
    ~Finally() { f(); }
};

static int sl_step_host_pipelined(lsr_cuda_ctx* c, const double* phi, const double* dist, const int64_t* active,
                                  int64_t n_active, const lsr_step_cfg* cfg, double energy_p, double* out,
                                  int64_t* bad_node) {
    const lsr_grid& g = c->grid;
    const int nx = g.dims[0], ny = g.dims[1], nz = g.dims[2];
    const long long nxy = static_cast<long long>(nx) * ny;
    const int kChunks = 16;
    const int zc = (nz + kChunks - 1) / kChunks;
    const int nch = (nz + zc - 1) / zc;
    const int halo = 8;  // lead of the upload over the compute (planes); >= the packed reach
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->s_cmp) {
        LSR_CUDA_TRY(cudaStreamCreateWithFlags(&c->s_cmp, cudaStreamNonBlocking));
        LSR_CUDA_TRY(cudaStreamCreateWithFlags(&c->s_down, cudaStreamNonBlocking));
        for (auto& e : c->ev_up) LSR_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : c->ev_cmp) LSR_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : c->ev_down) LSR_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        LSR_CUDA_TRY(cudaMalloc(&c->d_miss, sizeof(unsigned long long)));
    }
    if (nch > static_cast<int>(sizeof(c->ev_up) / sizeof(c->ev_up[0]))) return kNotPipelined;
    cudaStream_t up = c->stream, cmp = c->s_cmp, down = c->s_down;
    const auto chunk_off = [&](int ch) { return static_cast<long long>(std::min(nz, ch * zc)) * nxy; };
    const auto upload_chunk_for = [&](int ch) {  // last upload chunk compute chunk ch needs
        return std::min(nch - 1, (std::min(nz, std::min(nz, (ch + 1) * zc) + halo) - 1) / zc);
    };
    const int R = std::min(c->reach, halo);
    const bool packed = R >= 3;  // >= 3 covers the degenerate-gradient fallback's stencils
    // phi and d in mapped pinned memory: the GPU pulls the values it needs
    // itself (transfer.cu); otherwise host threads pack them (host_pack.h)
    static const bool zero_copy = !(std::getenv("LSR_ZERO_COPY") && std::atoi(std::getenv("LSR_ZERO_COPY")) == 0);
    const double* phi_map = zero_copy ? mapped_ptr(phi, c->n) : nullptr;
    const double* dist_map = zero_copy ? mapped_ptr(dist, c->n) : nullptr;
    const bool mapped = phi_map && dist_map;
    const int threads = host_threads();
    static const int copy_env = std::getenv("LSR_COPY_THREADS") ? std::atoi(std::getenv("LSR_COPY_THREADS")) : 0;
    const int copy_threads = !packed ? 0
                             : copy_env > 0 ? std::min(copy_env, threads)
                             : mapped       ? threads
                                            : std::max(1, threads / 2);
    static const bool trace = std::getenv("LSR_PIPE_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    const auto ms_since = [&] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    };
    // the ids (and, unpacked, phi's first chunks) go up while the host plans
    if (int st = ensure_ids(&c->active, &c->cap_active, n_active)) return st;
    cudaEvent_t tev[4] = {};  // trace: device timeline (start, ids up, uploads done, compute done)
    if (trace) {
        for (auto& e : tev) LSR_CUDA_TRY(cudaEventCreate(&e));
        LSR_CUDA_TRY(cudaEventRecord(tev[0], up));
    }
    LSR_CUDA_TRY(cudaMemcpyAsync(c->active, active, sizeof(int64_t) * n_active, cudaMemcpyHostToDevice, up));
    if (trace) LSR_CUDA_TRY(cudaEventRecord(tev[1], up));
    LSR_CUDA_TRY(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), up));
    LSR_CUDA_TRY(cudaMemsetAsync(c->d_miss, 0, sizeof(unsigned long long), up));
    // packed: chunks [0, nfull) still move phi and out whole over PCIe (the
    // DMA engines are idle otherwise), the rest move packed values and the
    // host threads copy phi to out for them — balancing PCIe time against
    // host memory bandwidth. Unpacked: every chunk moves whole.
    static const double full_env = std::getenv("LSR_PIPE_FULL") ? std::atof(std::getenv("LSR_PIPE_FULL")) : 0.125;
    const int nfull = packed ? std::max(0, std::min(nch, static_cast<int>(std::lround(full_env * nch)))) : nch;
    const int zfull = std::min(nz, nfull * zc);  // planes [0, zfull) move whole
    const int prefetch = packed ? nfull : std::min(nch, 2);
    if (prefetch)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->phi, phi, sizeof(double) * chunk_off(prefetch), cudaMemcpyHostToDevice, up));
    c->n_active = n_active;
    c->zt_bricks = false;
    c->bd_valid = false;
    c->box_valid = false;
    c->dirty_is_active = false;
    c->consistent = false;
    // per-chunk ranges of the (ascending) ids
    std::vector<int64_t> first(nch + 1);
    for (int ch = 0; ch <= nch; ++ch) first[ch] = std::lower_bound(active, active + n_active, chunk_off(ch)) - active;
    first[nch] = n_active;
    // packed: the host's out = phi copy starts at once on its own threads;
    // each chunk's results are scattered into out once both its planes are
    // copied and its results are back (event). Items run in ascending order.
    std::unique_ptr<std::atomic<int>[]> copied(new std::atomic<int>[nz]), recorded(new std::atomic<int>[nch]),
        gathered(new std::atomic<int>[nz]);
    for (int k = 0; k < nz; ++k) copied[k].store(0, std::memory_order_relaxed);
    for (int k = 0; k < nz; ++k) gathered[k].store(0, std::memory_order_relaxed);
    for (int ch = 0; ch < nch; ++ch) recorded[ch].store(0, std::memory_order_relaxed);
    std::atomic<int> copy_error{0};
    std::atomic<bool> cancel{false};
    std::atomic<int> n_copied{0};
    double t_copied = 0.0, t_last_res = 0.0;  // trace: host copy finished, last results back
    const bool host_copy = nfull < nch;
    if (host_copy) {
        if (int st = ensure_pinned(&c->h_res, &c->cap_hres, n_active)) return st;
        if (int st = ensure_device(&c->d_res, &c->cap_dres, n_active)) return st;
        if (!c->copy_pool || c->copy_pool->size() != copy_threads)
            c->copy_pool.reset(new lsr_host::Pool(std::max(1, copy_threads)));
        double* h_res = c->h_res;
        cudaEvent_t* ev_down = c->ev_down;
        constexpr int kParts = 8;  // scatter items per chunk, so the last chunk's scatter runs wide
        c->copy_pool->post(nz - zfull + (nch - nfull) * kParts, [&, h_res, ev_down](int item) {
            if (item < nz - zfull) {
                const int k = zfull + item;
                const long long o = static_cast<long long>(k) * nxy;
                lsr_host::copy_stream(out + o, phi + o, sizeof(double) * nxy);
                copied[k].store(1, std::memory_order_release);
                if (trace && ++n_copied == nz - zfull) t_copied = ms_since();
                return;
            }
            const int ch = nfull + (item - (nz - zfull)) / kParts, part = (item - (nz - zfull)) % kParts;
            for (int k = ch * zc; k < std::min(nz, (ch + 1) * zc); ++k)
                while (!copied[k].load(std::memory_order_acquire)) std::this_thread::yield();
            // the chunk's results: wait until this call has queued their D2H
            while (!recorded[ch].load(std::memory_order_acquire) && !cancel.load()) std::this_thread::yield();
            if (cancel.load()) return;
            if (cudaEventSynchronize(ev_down[ch]) != cudaSuccess) {
                copy_error = 1;
                return;
            }
            if (trace && ch == nch - 1 && part == 0) t_last_res = ms_since();
            const int64_t len = first[ch + 1] - first[ch];
            const int64_t t0 = first[ch] + len * part / kParts, t1 = first[ch] + len * (part + 1) / kParts;
            const uint64_t nn = static_cast<uint64_t>(c->n);
            for (int64_t t = t0; t < t1; ++t)
                if (static_cast<uint64_t>(active[t]) < nn) out[active[t]] = h_res[t];  // else reported by the step
        });
    }
    // on every exit the host jobs (which reference this frame) are joined;
    // on an early exit, copy items whose results were never queued give up
    bool copy_joined = !host_copy;
    const Finally copy_guard{[&] {
        if (copy_joined) return;
        cancel.store(true);
        c->copy_pool->wait();
    }};
    lsr_host::StepPacker& pk = c->packer;
    const Finally gather_guard{[&] { pk.wait(); }};
    const long long words = lsr_bitmap_words(nx, ny, nz);
    unsigned long long *bmA = nullptr, *bmD = nullptr, *bmB = nullptr;
    if (mapped) {
        // bitmaps of what the step reads; unsorted or out-of-grid ids count
        // as misses (the chunking needs ascending ids) and rerun the step whole
        if (int st = ensure_device(&c->bm, &c->cap_bm, 4 * words + 8)) return st;
        bmA = c->bm;
        bmD = c->bm + words;
        bmB = c->bm + 2 * words;
        LSR_CUDA_TRY(cudaMemsetAsync(c->bm + 4 * words, 0, 8 * sizeof(unsigned long long), up));
        LSR_CUDA_TRY(launch_build_bitmaps(nx, ny, nz, c->active, n_active, packed ? R : 0, bmA, bmD, bmB,
                                          c->bm + 3 * words, c->d_miss, up));
        LSR_CUDA_TRY(launch_check_sorted(c->active, n_active, c->d_miss, up));
        LSR_CUDA_TRY(launch_count_bits(nx, ny, nz, 0, nz, bmD, c->bm + 4 * words, up));
        if (packed) LSR_CUDA_TRY(launch_count_bits(nx, ny, nz, zfull, nz, bmB, c->bm + 4 * words + 1, up));
    } else if (!pk.plan(active, n_active, nx, ny, nz, packed ? R : 0, std::max(1, threads - copy_threads))) {
        LSR_CUDA_TRY(cudaStreamSynchronize(up));  // the unpipelined path reuses these buffers
        return kNotPipelined;
    }
    const double t_plan = ms_since();
    const lsr_host::PackSet& dset = pk.dset();
    const lsr_host::PackSet& pset = pk.phiset();
    int status = LSR_OK;
    if (!mapped) status = ensure_set(dset, c->pk_d);
    if (status == LSR_OK && !mapped && packed) status = ensure_set(pset, c->pk_phi);
    if (status != LSR_OK) return status;
    if (!mapped) {
        const lsr_cuda_ctx::Packed qd = c->pk_d, qp = c->pk_phi;
        pk.pool().post(nz, [&, qd, qp](int k) {
            pk.gather_plane(k, dist, qd.h_vals, qd.h_desc, packed && k >= zfull ? phi : nullptr, qp.h_vals,
                            qp.h_desc);
            gathered[k].store(1, std::memory_order_release);
        });
    }
    SlParams P = make_params(g, *cfg, energy_p);
    P.halo_miss = c->d_miss;
    if (packed) P.reach = (R - 1.5) * g.dx;
    int64_t h2d = static_cast<int64_t>(sizeof(int64_t)) * n_active;
    int scattered = 0;  // chunks whose packed runs are in place on the device
    int computed = 0;   // chunks whose kernel is issued
    const auto issue_compute = [&](int ch) -> int {
        const int z0 = ch * zc, z1 = std::min(nz, (ch + 1) * zc);
        const int up_ch = upload_chunk_for(ch);
        LSR_CUDA_TRY(cudaStreamWaitEvent(cmp, c->ev_up[up_ch], 0));
        for (; !mapped && scattered <= up_ch; ++scattered) {
            const int s0 = scattered * zc, s1 = std::min(nz, (scattered + 1) * zc);
            LSR_CUDA_TRY(launch_scatter_runs(c->pk_d.d_vals, c->pk_d.d_desc, dset.runs_before(s0),
                                             dset.runs_before(s1), dset.values_before(s1), c->dist, cmp));
            if (scattered >= nfull)
                LSR_CUDA_TRY(launch_scatter_runs(c->pk_phi.d_vals, c->pk_phi.d_desc, pset.runs_before(s0),
                                                 pset.runs_before(s1), pset.values_before(s1), c->phi, cmp));
        }
        P.z_base = 0;
        P.z_planes = std::min(nz, (up_ch + 1) * zc);
        P.own_lo = z0;
        P.own_hi = z1;
        const long long n = first[ch + 1] - first[ch];
        LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, c->phi, c->dist, c->active + first[ch], n, c->out, c->d_bad, cmp));
        const bool whole = ch < nfull;
        if (!whole) LSR_CUDA_TRY(launch_gather_ids(c->out, c->active + first[ch], n, c->d_res + first[ch], c->n, cmp));
        LSR_CUDA_TRY(cudaEventRecord(c->ev_cmp[ch], cmp));
        LSR_CUDA_TRY(cudaStreamWaitEvent(down, c->ev_cmp[ch], 0));
        if (!whole) {
            if (n > 0)
                LSR_CUDA_TRY(cudaMemcpyAsync(c->h_res + first[ch], c->d_res + first[ch], sizeof(double) * n,
                                             cudaMemcpyDeviceToHost, down));
            LSR_CUDA_TRY(cudaEventRecord(c->ev_down[ch], down));
            recorded[ch].store(1, std::memory_order_release);
        } else {
            const long long o = chunk_off(ch), cnt = chunk_off(ch + 1) - o;
            LSR_CUDA_TRY(cudaMemcpyAsync(out + o, c->out + o, sizeof(double) * cnt, cudaMemcpyDeviceToHost, down));
        }
        return LSR_OK;
    };
    const auto issue_upload = [&](int ch) -> int {
        const int z0 = ch * zc, z1 = std::min(nz, (ch + 1) * zc);
        const long long o = chunk_off(ch), cnt = chunk_off(ch + 1) - o;
        const bool whole = ch < nfull;
        if (whole && ch >= prefetch)
            LSR_CUDA_TRY(cudaMemcpyAsync(c->phi + o, phi + o, sizeof(double) * cnt, cudaMemcpyHostToDevice, up));
        if (whole) h2d += static_cast<int64_t>(sizeof(double)) * cnt;
        if (mapped) {
            LSR_CUDA_TRY(launch_pull_planes(nx, ny, nz, z0, z1, bmD, dist_map, c->dist, whole ? nullptr : bmB, phi_map,
                                            c->phi, up));
        } else {
            for (int k = z0; k < z1; ++k)
                while (!gathered[k].load(std::memory_order_acquire)) std::this_thread::yield();
            if (int st = upload_set(dset, c->pk_d, z0, z1, up, &h2d)) return st;
            if (!whole)
                if (int st = upload_set(pset, c->pk_phi, z0, z1, up, &h2d)) return st;
        }
        if (whole)
            LSR_CUDA_TRY(cudaMemcpyAsync(c->out + o, c->phi + o, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, up));
        LSR_CUDA_TRY(cudaEventRecord(c->ev_up[ch], up));
        return LSR_OK;
    };
    for (int ch = 0; ch < nch && status == LSR_OK; ++ch) {  // uploads in plane order
        status = issue_upload(ch);
        // compute every chunk whose planes (plus the halo) are now queued
        while (status == LSR_OK && computed < nch && upload_chunk_for(computed) <= ch)
            status = issue_compute(computed++);
    }
    pk.wait();
    if (trace && status == LSR_OK) {
        cudaEventRecord(tev[2], up);
        cudaEventRecord(tev[3], cmp);
    }
    const double t_issued = ms_since();
    if (status != LSR_OK) return status;
    unsigned long long h[2] = {0, 0};
    LSR_CUDA_TRY(cudaStreamSynchronize(down));
    LSR_CUDA_TRY(cudaStreamSynchronize(cmp));
    if (host_copy) c->copy_pool->wait();
    copy_joined = true;
    if (copy_error) return set_err(LSR_ERR_CUDA, "sl_step: result download failed");
    if (trace) {
        float ms[3] = {0, 0, 0};
        for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&ms[i], tev[0], tev[i + 1]);
        std::fprintf(stderr, "[lsr pipe] device: ids up %.2f ms, uploads done %.2f ms, compute done %.2f ms\n", ms[0],
                     ms[1], ms[2]);
        for (auto& e : tev) cudaEventDestroy(e);
    }
    if (trace)
        std::fprintf(stderr,
                     "[lsr pipe] %s, whole chunks %d/%d, threads %d+%d reach %d plan %.2f ms, issued %.2f ms, copied %.2f ms, last results "
                     "%.2f ms, done %.2f ms; d %lld values %lld runs, phi %lld values %lld runs\n",
                     mapped ? "zero-copy" : "host-packed", nfull, nch, std::max(1, threads - copy_threads), copy_threads, packed ? R : 0, t_plan, t_issued, t_copied,
                     t_last_res, ms_since(),
                     static_cast<long long>(mapped ? 0 : dset.total_values()),
                     static_cast<long long>(mapped ? 0 : dset.total_runs()),
                     static_cast<long long>(packed && !mapped ? pset.total_values() : 0),
                     static_cast<long long>(packed && !mapped ? pset.total_runs() : 0));
    LSR_CUDA_TRY(cudaMemcpy(&h[0], c->d_miss, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    LSR_CUDA_TRY(cudaMemcpy(&h[1], c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (mapped) {  // values pulled over PCIe
        unsigned long long cnt[2] = {0, 0};
        LSR_CUDA_TRY(cudaMemcpy(cnt, c->bm + 4 * words, sizeof cnt, cudaMemcpyDeviceToHost));
        h2d += static_cast<int64_t>(sizeof(double)) * static_cast<int64_t>(cnt[0] + cnt[1]);
    }
    if (h[0] != 0) {  // rerun unpipelined with phi and d whole
        LSR_CUDA_TRY(cudaMemcpyAsync(c->phi, phi, sizeof(double) * c->n, cudaMemcpyHostToDevice, up));
        LSR_CUDA_TRY(cudaMemcpyAsync(c->dist, dist, sizeof(double) * c->n, cudaMemcpyHostToDevice, up));
        LSR_CUDA_TRY(cudaMemcpyAsync(c->out, c->phi, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, up));
        P = make_params(g, *cfg, energy_p);
        LSR_CUDA_TRY(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), up));
        LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, c->phi, c->dist, c->active, n_active, c->out, c->d_bad, up));
        LSR_CUDA_TRY(cudaMemcpyAsync(out, c->out, sizeof(double) * c->n, cudaMemcpyDeviceToHost, up));
        LSR_CUDA_TRY(cudaMemcpyAsync(&h[1], c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, up));
        LSR_CUDA_TRY(cudaStreamSynchronize(up));
        c->pipeline_fallbacks++;
        // the feet reach beyond the packed ball: widen it for the next calls
        c->reach = std::min(halo, c->reach + 3);
        h2d += 2 * static_cast<int64_t>(sizeof(double)) * c->n;
    }
    g_h2d_bytes = h2d;
    g_d2h_bytes = static_cast<int64_t>(sizeof(double)) * (n_active - first[nfull] + chunk_off(nfull)) +
                  (h[0] != 0 ? static_cast<int64_t>(sizeof(double)) * c->n : 0);
    if (h[1] != ~0ULL) return numerical_error(g, h[1], bad_node);
    return LSR_OK;
}

int lsr_cuda_pack_host(const lsr_grid* grid, const int64_t* active, int64_t n_active, int32_t reach,
                       const double* dist, const double* phi, double* dist_field, double* phi_field,
                       int64_t* counts) {
    if (int st = check_grid(grid)) return st;
    if (grid->dim != 3 || !dist || !dist_field || (n_active > 0 && !active) || reach < 0 ||
        (reach > 0 && (!phi || !phi_field)))
        return set_err(LSR_ERR_CONFIG, "pack_host: needs a 3d grid and non-null buffers");
    lsr_host::StepPacker pk;
    if (!pk.plan(active, n_active, grid->dims[0], grid->dims[1], grid->dims[2], reach, host_threads()))
        return set_err(LSR_ERR_CONFIG, "pack_host: ids are not ascending inside the grid");
    const lsr_host::PackSet& ds = pk.dset();
    const lsr_host::PackSet& ps = pk.phiset();
    std::vector<double> dv(ds.total_values()), pv(reach > 0 ? ps.total_values() : 0);
    std::vector<lsr_host::RunDesc> dd(ds.total_runs()), pd(reach > 0 ? ps.total_runs() : 0);
    for (int k = 0; k < grid->dims[2]; ++k) pk.gather_plane(k, dist, dv.data(), dd.data(), phi, pv.data(), pd.data());
    const auto scatter = [](const std::vector<double>& v, const std::vector<lsr_host::RunDesc>& d, double* f) {
        for (size_t r = 0; r < d.size(); ++r) {
            const int64_t end = r + 1 < d.size() ? d[r + 1].src : static_cast<int64_t>(v.size());
            std::memcpy(f + d[r].dst, v.data() + d[r].src, sizeof(double) * (end - d[r].src));
        }
    };
    scatter(dv, dd, dist_field);
    if (reach > 0) scatter(pv, pd, phi_field);
    if (counts) {
        counts[0] = ds.total_values();
        counts[1] = ds.total_runs();
        counts[2] = reach > 0 ? ps.total_values() : 0;
        counts[3] = reach > 0 ? ps.total_runs() : 0;
    }
    return LSR_OK;
}

// One-shot host entry. A per-thread context is cached across calls with the
// same grid, so repeated calls do not re-allocate device memory.
int lsr_cuda_sl_step_host(const lsr_grid* grid, const double* phi, const double* dist, const int64_t* active,
                          int64_t n_active, const lsr_step_cfg* cfg, double energy_p, double* out,
                          int64_t* bad_node) {
    if (bad_node) *bad_node = -1;
    if (int st = check_grid(grid)) return st;
    if (int st = check_cfg(cfg, energy_p)) return st;
    if (!phi || !dist || !out || (n_active > 0 && !active)) return set_err(LSR_ERR_CONFIG, "sl_step: null argument");
    if (out == phi) return set_err(LSR_ERR_CONFIG, "sl_step: out must not alias phi");
    // ids outside the grid are never dereferenced on the device or in the
    // host scatter; the step reports them as a ConfigError (numerical_error)
    struct Cache {
        lsr_cuda_ctx* ctx = nullptr;
        ~Cache() { lsr_cuda_destroy(ctx); }
    };
    thread_local Cache cache;
    int dev = 0;
    LSR_CUDA_TRY(cudaGetDevice(&dev));
    if (cache.ctx && (std::memcmp(&cache.ctx->grid, grid, sizeof(lsr_grid)) != 0 || cache.ctx->device != dev)) {
        lsr_cuda_destroy(cache.ctx);
        cache.ctx = nullptr;
    }
    if (!cache.ctx)
        if (int st = lsr_cuda_create(dev, grid, &cache.ctx)) return st;
    lsr_cuda_ctx* c = cache.ctx;
    if (grid->dim == 3 && grid->dims[2] >= 64 && n_active > 0) {
        const int st = sl_step_host_pipelined(c, phi, dist, active, n_active, cfg, energy_p, out, bad_node);
        if (st != kNotPipelined) return st;
    }
    const size_t bytes = sizeof(double) * c->n;
    cudaStream_t s = c->stream;
    LSR_CUDA_TRY(cudaMemcpyAsync(c->phi, phi, bytes, cudaMemcpyHostToDevice, s));
    LSR_CUDA_TRY(cudaMemcpyAsync(c->dist, dist, bytes, cudaMemcpyHostToDevice, s));
    if (int st = ensure_ids(&c->active, &c->cap_active, n_active)) return st;
    if (n_active > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, active, sizeof(int64_t) * n_active, cudaMemcpyHostToDevice, s));
    c->n_active = n_active;
    c->zt_bricks = false;
    c->bd_valid = false;
    c->box_valid = false;
    c->dirty_is_active = false;
    c->consistent = false;
    int64_t bad = -1;
    const int st = lsr_cuda_sl_step(c, cfg, energy_p, &bad);
    if (bad_node) *bad_node = bad;
    if (st != LSR_OK && st != LSR_ERR_NUMERICAL) return st;
    const std::string msg = g_err;
    g_h2d_bytes = static_cast<int64_t>(2 * bytes + sizeof(int64_t) * n_active);
    g_d2h_bytes = static_cast<int64_t>(bytes);
    // out is fully written even when a node went non-finite (evolve.cpp:110-117)
    LSR_CUDA_TRY(cudaMemcpyAsync(out, c->out, bytes, cudaMemcpyDeviceToHost, s));
    LSR_CUDA_TRY(cudaStreamSynchronize(s));
    if (st == LSR_ERR_NUMERICAL) return set_err(st, msg);
    return st;
}

int lsr_cuda_ctx_build_distance(lsr_cuda_ctx* c, const double* pts, int64_t n, int dim, int seed_only,
                                double* sentinel, int* rounds) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "ctx_build_distance: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || (n > 0 && !pts)) return set_err(LSR_ERR_CONFIG, "build_distance: null argument");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->exact) LSR_CUDA_TRY(cudaMalloc(&c->exact, static_cast<size_t>(c->n)));
    c->zt_bricks = false;
    c->bd_valid = false;
    c->box_valid = false;  // the covered bricks depend on d
    std::string err;
    double sent = 0.0;
    int r = 0;
    const int st = lsr_prep_build_distance(&c->grid, pts, n, dim, seed_only, c->dist, c->exact, &sent, &r, c->stream,
                                           &err);
    if (st) return set_err(st, err);
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (sentinel) *sentinel = sent;
    if (rounds) *rounds = r;
    return LSR_OK;
}

int lsr_cuda_surface_energy(lsr_cuda_ctx* c, int which, int p, int refine, double* energy) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "surface_energy: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || !energy) return set_err(LSR_ERR_CONFIG, "surface_energy: null argument");
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "surface_energy: phi must be PHI or OUT");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    lsr_step_cfg dummy{1, LSR_INTERP_Q1, 0.0, 1.0, 1e-3, 1.0, 2.0, 1.0};
    const SlParams P = make_params(c->grid, dummy, 1.0);
    std::string err;
    int64_t nc = 0;
    const int st = lsr_prep_surface_energy(P, *slot, c->dist, p, refine, energy, &nc, c->stream, &err);
    if (st) return set_err(st, err);
    c->n_interface_cells = nc;
    return LSR_OK;
}

int lsr_cuda_surface_energy_host(const lsr_grid* grid, const double* phi, const double* dist, int p, int refine,
                                 double* energy) {
    if (int st = check_grid(grid)) return st;
    if (!phi || !dist || !energy) return set_err(LSR_ERR_CONFIG, "surface_energy: null argument");
    int dev = 0;
    LSR_CUDA_TRY(cudaGetDevice(&dev));
    lsr_cuda_ctx* c = nullptr;
    if (int st = lsr_cuda_create(dev, grid, &c)) return st;
    int st = lsr_cuda_upload_field(c, LSR_FIELD_PHI, phi);
    if (st == LSR_OK) st = lsr_cuda_upload_field(c, LSR_FIELD_DIST, dist);
    if (st == LSR_OK) st = lsr_cuda_surface_energy(c, LSR_FIELD_PHI, p, refine, energy);
    lsr_cuda_destroy(c);
    return st;
}

int lsr_cuda_build_distance(const lsr_grid* grid, const double* pts, int64_t n, int dim, int seed_only,
                            double* d_out, uint8_t* exact_out, double* sentinel, int* rounds) {
    if (int st = check_grid(grid)) return st;
    int dev = 0;
    LSR_CUDA_TRY(cudaGetDevice(&dev));
    lsr_cuda_ctx* c = nullptr;
    if (int st = lsr_cuda_create(dev, grid, &c)) return st;
    int st = lsr_cuda_ctx_build_distance(c, pts, n, dim, seed_only, sentinel, rounds);
    if (st == LSR_OK && d_out) st = lsr_cuda_download_field(c, LSR_FIELD_DIST, d_out);
    if (st == LSR_OK && exact_out) {
        const cudaError_t e = cudaMemcpy(exact_out, c->exact, static_cast<size_t>(c->n), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = cuda_err(e, "download exact");
    }
    lsr_cuda_destroy(c);
    return st;
}

// ---- band rebuild / reinitialisation / the whole loop body ----------------

static SlParams grid_params(const lsr_grid& g) {
    const lsr_step_cfg dummy{1, LSR_INTERP_Q1, 0.0, 1.0, 1e-3, 1.0, 2.0, 1.0};
    return make_params(g, dummy, 1.0);
}

int lsr_cuda_narrow_band(lsr_cuda_ctx* c, int which, double gamma, int64_t* n_active, int64_t* n_tube) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "narrow_band: a z-slab context (use lsr_cuda_slab_*)");
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "narrow_band: phi must be PHI or OUT");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    long long na = 0, nt = 0;
    if (int st = lsr_band_build(grid_params(c->grid), *slot, gamma, c->band, &na, &nt, c->stream, &err))
        return set_err(st, err);
    // the band's ACTIVE list becomes the context's active set
    if (int st = ensure_ids(&c->active, &c->cap_active, na)) return st;
    if (na > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, c->band.active, sizeof(int64_t) * na, cudaMemcpyDeviceToDevice,
                                     c->stream));
    c->n_active = na;
    c->zt_bricks = false;
    c->box_valid = false;
    c->dirty_is_active = false;
    if (n_active) *n_active = na;
    if (n_tube) *n_tube = nt;
    return LSR_OK;
}

int lsr_cuda_band_download(lsr_cuda_ctx* c, uint8_t* state, int64_t* active, int64_t* tube) {
    if (!c || !c->band.state) return set_err(LSR_ERR_CONFIG, "band_download: no band built");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (state) LSR_CUDA_TRY(cudaMemcpyAsync(state, c->band.state, c->n, cudaMemcpyDeviceToHost, c->stream));
    if (active && c->band.n_active)
        LSR_CUDA_TRY(cudaMemcpyAsync(active, c->band.active, sizeof(int64_t) * c->band.n_active,
                                     cudaMemcpyDeviceToHost, c->stream));
    if (tube && c->band.n_tube)
        LSR_CUDA_TRY(cudaMemcpyAsync(tube, c->band.tube, sizeof(int64_t) * c->band.n_tube, cudaMemcpyDeviceToHost,
                                     c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LSR_OK;
}

int lsr_cuda_clamp_field(lsr_cuda_ctx* c, int which, double gamma) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "clamp_field: a z-slab context (use lsr_cuda_slab_*)");
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    double** slot = field_slot(c, which);
    if (!slot) return set_err(LSR_ERR_CONFIG, "clamp_field: unknown field");
    c->seq++;  // may write phi or out
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    if (int st = lsr_clamp(*slot, c->n, gamma, c->stream, &err)) return set_err(st, err);
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (which != LSR_FIELD_DIST) c->consistent = false;
    else c->zt_bricks = c->bd_valid = false;  // d changed: its covered bricks and per-brick maxima
    c->box_valid = false;  // the covered bricks depend on d
    return LSR_OK;
}

static int reinitialize_impl(lsr_cuda_ctx* c, int which, double gamma, const lsr_reinit_cfg* rc, int* iterations,
                             int* had_interface, bool clamp_sparse) {
    if (!c || !rc) return set_err(LSR_ERR_CONFIG, "reinitialize: null argument");
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "reinitialize: phi must be PHI or OUT");
    c->seq++;  // may write phi or out
    if (!c->band.state) return set_err(LSR_ERR_CONFIG, "reinitialize: build the band first (lsr_cuda_narrow_band)");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->scratch) LSR_CUDA_TRY(cudaMalloc(&c->scratch, sizeof(double) * c->n));
    const ReinitParams R{rc->dtau, rc->max_iters, rc->residual_tol, rc->sign_eps};
    std::string err;
    int it = 0, had = 0;
    const int st = lsr_reinitialize(grid_params(c->grid), slot, &c->scratch, c->band, gamma, R, c->rb, &it, &had,
                                    c->stream, &err, clamp_sparse);
    if (st) return set_err(st, err);
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->consistent = false;  // the clamp may touch any node
    if (iterations) *iterations = it;
    if (had_interface) *had_interface = had;
    return LSR_OK;
}

int lsr_cuda_reinitialize(lsr_cuda_ctx* c, int which, double gamma, const lsr_reinit_cfg* rc, int* iterations,
                          int* had_interface) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "reinitialize: a z-slab context (use lsr_cuda_slab_*)");
    return reinitialize_impl(c, which, gamma, rc, iterations, had_interface, false);
}

int lsr_cuda_set_band(lsr_cuda_ctx* c, const uint8_t* state, const int64_t* active, int64_t n_active,
                      const int64_t* tube, int64_t n_tube) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "set_band: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || !state || (n_active > 0 && !active) || (n_tube > 0 && !tube))
        return set_err(LSR_ERR_CONFIG, "set_band: null argument");
    if (n_active < 0 || n_tube < 0 || n_active > c->n || n_tube > c->n)
        return set_err(LSR_ERR_CONFIG, "set_band: bad list sizes");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    if (int st = c->band.reserve(c->n, &err)) return set_err(st, err);
    cudaStream_t s = c->stream;
    LSR_CUDA_TRY(cudaMemcpyAsync(c->band.state, state, static_cast<size_t>(c->n), cudaMemcpyHostToDevice, s));
    if (n_active > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->band.active, active, sizeof(int64_t) * n_active, cudaMemcpyHostToDevice, s));
    if (n_tube > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->band.tube, tube, sizeof(int64_t) * n_tube, cudaMemcpyHostToDevice, s));
    c->band.n_active = n_active;
    c->band.n_tube = n_tube;
    // the band's ACTIVE list becomes the context's active set (as narrow_band)
    if (int st = ensure_ids(&c->active, &c->cap_active, n_active)) return st;
    if (n_active > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, active, sizeof(int64_t) * n_active, cudaMemcpyHostToDevice, s));
    c->n_active = n_active;
    c->zt_bricks = false;
    c->box_valid = false;
    c->dirty_is_active = false;
    LSR_CUDA_TRY(cudaStreamSynchronize(s));
    return LSR_OK;
}

int lsr_cuda_interface_one_step(lsr_cuda_ctx* c, int which, uint8_t* frozen, int* had_interface) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "interface_one_step: a z-slab context (use lsr_cuda_slab_*)");
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    c->seq++;  // may write phi or out
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "interface_one_step: phi must be PHI or OUT");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->scratch) LSR_CUDA_TRY(cudaMalloc(&c->scratch, sizeof(double) * c->n));
    std::string err;
    int had = 0;
    if (int st = lsr_reinit_one_step(grid_params(c->grid), slot, &c->scratch, c->rb, &had, c->stream, &err))
        return set_err(st, err);
    if (had_interface) *had_interface = had;
    if (frozen) {
        LSR_CUDA_TRY(cudaMemcpyAsync(frozen, c->rb.frozen, static_cast<size_t>(c->n), cudaMemcpyDeviceToHost, c->stream));
        LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    c->consistent = false;
    if (!had) return set_err(LSR_ERR_NO_INTERFACE, "interface_one_step: phi has no sign change");  // reinit.cpp:56
    return LSR_OK;
}

int lsr_cuda_reinit_iterate(lsr_cuda_ctx* c, int which, const uint8_t* frozen, const lsr_reinit_cfg* rc,
                            int* iterations) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "reinit_iterate: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || !rc) return set_err(LSR_ERR_CONFIG, "reinit_iterate: null argument");
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "reinit_iterate: phi must be PHI or OUT");
    c->seq++;  // may write phi or out
    if (!c->band.state) return set_err(LSR_ERR_CONFIG, "reinit_iterate: no band (lsr_cuda_narrow_band / set_band)");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->scratch) LSR_CUDA_TRY(cudaMalloc(&c->scratch, sizeof(double) * c->n));
    std::string err;
    if (int st = c->rb.reserve(c->n, &err)) return set_err(st, err);
    if (frozen)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->rb.frozen, frozen, static_cast<size_t>(c->n), cudaMemcpyHostToDevice, c->stream));
    const ReinitParams R{rc->dtau, rc->max_iters, rc->residual_tol, rc->sign_eps};
    int it = 0;
    if (int st = lsr_reinit_iterate(grid_params(c->grid), slot, &c->scratch, c->band.tube, c->band.n_tube, R, c->rb,
                                    false, &it, c->stream, &err))
        return set_err(st, err);
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->consistent = false;
    if (iterations) *iterations = it;
    return LSR_OK;
}

int lsr_cuda_fast_sweep(lsr_cuda_ctx* c, const uint8_t* exact, double sentinel, int* rounds) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "fast_sweep: a z-slab context (use lsr_cuda_slab_*)");
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (!c->exact) {
        if (!exact) return set_err(LSR_ERR_CONFIG, "fast_sweep: no exact flags");
        LSR_CUDA_TRY(cudaMalloc(&c->exact, static_cast<size_t>(c->n)));
    }
    if (exact)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->exact, exact, static_cast<size_t>(c->n), cudaMemcpyHostToDevice, c->stream));
    std::string err;
    int r = 0;
    if (int st = lsr_prep_fast_sweep(&c->grid, c->dist, c->exact, sentinel, &r, c->stream, &err))
        return set_err(st, err);
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->zt_bricks = false;
    c->bd_valid = false;
    c->box_valid = false;  // the covered bricks depend on d
    if (rounds) *rounds = r;
    return LSR_OK;
}

int lsr_cuda_download_exact(lsr_cuda_ctx* c, uint8_t* exact) {
    if (!c || !exact) return set_err(LSR_ERR_CONFIG, "download_exact: null argument");
    if (!c->exact) return set_err(LSR_ERR_CONFIG, "download_exact: no distance field built");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    LSR_CUDA_TRY(cudaMemcpyAsync(exact, c->exact, static_cast<size_t>(c->n), cudaMemcpyDeviceToHost, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LSR_OK;
}

void lsr_cuda_reinit_defaults(double dx, double gamma, lsr_reinit_cfg* rc) {  // ReinitConfig::defaults (reinit.cpp:8-16)
    rc->dtau = 0.5 * dx;
    rc->max_iters = 4 * static_cast<int>(std::ceil(gamma / dx));
    rc->residual_tol = 1e-3;
    rc->sign_eps = dx;
}

int lsr_cuda_loop_step(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, const lsr_reinit_cfg* rc, int energy_refine,
                       double energy_override, lsr_loop_stats* stats) {
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "loop_step: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || !cfg || !rc) return set_err(LSR_ERR_CONFIG, "loop_step: null argument");
    if (int st = check_cfg(cfg, 1.0)) return st;
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    cudaEvent_t ev[5];
    for (auto& e : ev) LSR_CUDA_TRY(cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
        }
    } evg{ev};
    lsr_loop_stats S{};
    // phi^n fully clamped by the previous loop step and untouched since: phi^{n+1}
    // can then differ from a clamped field only on the band's tube and the
    // one-step's frozen nodes, and the final clamp visits just those
    const bool clamp_sparse = c->clamped_seq == c->seq && c->clamped_phi == c->phi && c->clamped_gamma == cfg->gamma;
    cudaEventRecord(ev[0], c->stream);
    int64_t na = 0, nt = 0;
    // 1. band of phi^n (driver.cpp:187)
    if (int st = lsr_cuda_narrow_band(c, LSR_FIELD_PHI, cfg->gamma, &na, &nt)) return st;
    cudaEventRecord(ev[1], c->stream);
    // 2. E_2 of phi^n (driver.cpp:188)
    double e2 = energy_override;
    if (!(energy_override >= 0.0)) {
        if (int st = lsr_cuda_surface_energy(c, LSR_FIELD_PHI, 2, energy_refine, &e2)) return st;
    }
    cudaEventRecord(ev[2], c->stream);
    // 3. the SL step, skipped when p > 1 and E_2 == 0 (driver.cpp:191-195)
    if (cfg->p > 1 && e2 == 0.0) {
        LSR_CUDA_TRY(cudaMemcpyAsync(c->out, c->phi, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream));
        c->consistent = false;
    } else {
        int64_t bad = -1;
        if (int st = lsr_cuda_sl_step(c, cfg, e2, &bad)) return st;
    }
    cudaEventRecord(ev[3], c->stream);
    // 4. reinitialise phi^{n+1} on the band of phi^n (driver.cpp:196)
    int it = 0, had = 0;
    if (int st = reinitialize_impl(c, LSR_FIELD_OUT, cfg->gamma, rc, &it, &had, clamp_sparse)) return st;
    cudaEventRecord(ev[4], c->stream);
    // 5. swap (driver.cpp:203). phi^{n+1} differs from phi^n (the buffer that
    // becomes `out`) only where the SL step, the one-step, the sweeps or the
    // clamp changed it: inside the tube of phi^n (ACTIVE is in it), at the
    // frozen nodes, or — reported by the clamp — elsewhere. Unless the clamp
    // reported a change outside the tube, the next SL step resyncs just the
    // tube and frozen nodes instead of copying the whole field.
    int outside = 1;
    LSR_CUDA_TRY(cudaMemcpyAsync(&outside, c->rb.clamp_outside, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const int64_t nd = c->band.n_tube + c->rb.n_frozen;
    if (!outside) {
        if (int st = ensure_ids(&c->dirty, &c->cap_dirty, nd)) return st;
        if (c->band.n_tube > 0)
            LSR_CUDA_TRY(cudaMemcpyAsync(c->dirty, c->band.tube, sizeof(int64_t) * c->band.n_tube,
                                         cudaMemcpyDeviceToDevice, c->stream));
        if (c->rb.n_frozen > 0)
            LSR_CUDA_TRY(cudaMemcpyAsync(c->dirty + c->band.n_tube, c->rb.frozen_ids, sizeof(int64_t) * c->rb.n_frozen,
                                         cudaMemcpyDeviceToDevice, c->stream));
        c->n_dirty = nd;
        c->dirty_is_active = false;
        c->consistent = true;
    } else {
        c->consistent = false;
    }
    std::swap(c->phi, c->out);
    c->clamped_seq = ++c->seq;
    c->clamped_phi = c->phi;
    c->clamped_gamma = cfg->gamma;
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    S.energy = e2;
    S.n_active = na;
    S.n_tube = nt;
    S.reinit_iterations = it;
    S.had_interface = had;
    S.dense_one_step = 1;
    cudaEventElapsedTime(&S.ms[0], ev[0], ev[1]);
    cudaEventElapsedTime(&S.ms[1], ev[1], ev[2]);
    cudaEventElapsedTime(&S.ms[2], ev[2], ev[3]);
    cudaEventElapsedTime(&S.ms[3], ev[3], ev[4]);
    if (stats) *stats = S;
    return LSR_OK;
}

// ---- the device-controlled loop ------------------------------------------

extern "C++" {
namespace {

// one iteration's record, written by the device (globaltimer marks at the
// phase boundaries: start, band, E_2, SL, reinit)
struct LoopDevStat {
    double energy;
    long long n_active, n_tube, n_cells, n_frozen;
    int iterations, had_interface;
    unsigned long long bad;
    int flags, pad;
    unsigned long long t[5];
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void loop_mark(LoopDevStat* st, const int* k, int phase) { st[*k].t[phase] = global_ns(); }

// the iteration's record; clears the SL bad-node word and the flags for the
// next iteration and advances the index
__global__ void loop_record(LoopDevStat* st, int* k, const double* e2, const long long* band_counts,
                            const long long* n_cells, const ReinitLoopDev* rl, unsigned long long* bad, int* flags,
                            int p, int* hard) {
    LoopDevStat& r = st[*k];
    r.t[4] = global_ns();
    r.energy = *e2;
    r.n_active = band_counts[0];
    r.n_tube = band_counts[1];
    r.n_cells = *n_cells;
    r.n_frozen = rl->counts[0];
    r.had_interface = (rl->flags[0] || rl->flags[1]) ? 1 : 0;
    r.iterations = r.had_interface ? rl->iterations : 0;
    r.bad = *bad;
    // bit 0: a 2d front left the hull (E_2); bit 1: E_2 is NaN with p > 1
    // (sl_step's "energy must be positive", evolve.cpp:45-46)
    r.flags = *flags | ((p > 1 && isnan(*e2)) ? 2 : 0);
    r.pad = hard[0];  // this iteration ran the dense one-step
    *bad = ~0ULL;
    *flags = 0;
    hard[0] = hard[1];
    hard[1] = 0;
    *k += 1;
}

int loop_reserve(lsr_cuda_ctx* c, int iterations) {
    auto& L = c->lr;
    if (!L.rl) LSR_CUDA_TRY(cudaMalloc(&L.rl, sizeof(ReinitLoopDev)));
    if (!L.e2) LSR_CUDA_TRY(cudaMalloc(&L.e2, sizeof(double)));
    if (!L.flags) LSR_CUDA_TRY(cudaMalloc(&L.flags, sizeof(int)));
    if (!L.k) LSR_CUDA_TRY(cudaMalloc(&L.k, sizeof(int)));
    if (!L.hard) LSR_CUDA_TRY(cudaMalloc(&L.hard, 2 * sizeof(int)));
    if (iterations > L.cap) {
        cudaFree(L.stats);
        L.stats = nullptr;
        L.cap = 0;
        LSR_CUDA_TRY(cudaMalloc(&L.stats, sizeof(LoopDevStat) * static_cast<size_t>(iterations)));
        L.cap = iterations;
    }
    if (!c->scratch) LSR_CUDA_TRY(cudaMalloc(&c->scratch, sizeof(double) * c->n));
    std::string err;
    if (int st = c->band.reserve(c->n, &err)) return set_err(st, err);
    if (int st = lsr_reinit_loop_reserve(c->n, c->rb, &err)) return set_err(st, err);
    if (int st = lsr_energy_loop_reserve(grid_params(c->grid), L.ew, &err)) return set_err(st, err);
    if (!c->zt.zt && c->grid.dim == 3) {
        const long long nb = zt_num_bricks(c->grid.dims);
        LSR_CUDA_TRY(cudaMalloc(&c->zt.zt, sizeof(double) * 4 * static_cast<size_t>(c->n)));
        LSR_CUDA_TRY(cudaMalloc(&c->zt.zc, sizeof(double) * 2 * static_cast<size_t>(c->n)));
        LSR_CUDA_TRY(cudaMalloc(&c->zt.mark, static_cast<size_t>(nb)));
        LSR_CUDA_TRY(cudaMalloc(&c->zt.reach, sizeof(unsigned) * static_cast<size_t>(nb)));
        LSR_CUDA_TRY(cudaMalloc(&c->zt.list, sizeof(unsigned) * static_cast<size_t>(nb)));
        LSR_CUDA_TRY(cudaMalloc(&c->zt.count, 2 * sizeof(unsigned)));
    }
    if (!c->bd && c->grid.dim == 3) {
        LSR_CUDA_TRY(cudaMalloc(&c->bd, sizeof(double) * 2 * static_cast<size_t>(zt_num_bricks(c->grid.dims))));
        c->bd_valid = false;
    }
    return LSR_OK;
}

// enqueues one loop iteration (driver.cpp:187-203) on the context stream: phi^n
// in a, out (equal to a on entry) in b; afterwards both hold phi^{n+1}. No
// host round trip and no allocation: capturable into a CUDA graph.
int enqueue_loop_iteration(lsr_cuda_ctx* c, double* a, double* b, const lsr_step_cfg* cfg, const lsr_reinit_cfg* rc,
                           int refine, bool clamp_sparse) {
    auto& L = c->lr;
    cudaStream_t s = c->stream;
    const SlParams G = grid_params(c->grid);
    LoopDevStat* st = static_cast<LoopDevStat*>(L.stats);
    std::string err;
    loop_mark<<<1, 1, 0, s>>>(st, L.k, 0);
    // 1. band of phi^n (driver.cpp:187)
    if (int e = lsr_band_enqueue(G, a, cfg->gamma, c->band, s, &err, L.hard)) return set_err(e, err);
    loop_mark<<<1, 1, 0, s>>>(st, L.k, 1);
    // 2. E_2 of phi^n (driver.cpp:188)
    // (interface cells from the band's tube unless phi^n may hold a hard jump, L.hard[0])
    if (int e = lsr_energy_enqueue(G, a, c->dist, 2, refine, L.ew, L.est_cells, L.e2, L.flags, s, &err, c->band.tube,
                                   c->band.counts + 1, L.est_active + L.est_active / 4, L.hard))
        return set_err(e, err);
    loop_mark<<<1, 1, 0, s>>>(st, L.k, 2);
    // 3. sl_step a -> b on the band's ACTIVE ids, E_2 read on the device; the
    // kernels skip when p > 1 and E_2 == 0 (driver.cpp:191-195; b already
    // equals a)
    SlParams P = make_params(c->grid, *cfg, 1.0);
    P.energy_dev = L.e2;
    P.n_dev = c->band.counts;
    const int64_t* ids = reinterpret_cast<const int64_t*>(c->band.active);
    const bool use_table = LSR_ZTAB && c->grid.dim == 3 && cfg->interp == 1 && P.fast_weno &&
                           c->grid.dims[2] >= 4 && cfg->delta > 0.0;
    if (use_table) {
        // covered bricks: from the band's state bytes and the per-brick maxima
        // of d (rows of whole 4-node brick words), else from the active ids
        if (c->grid.dims[0] % 4 == 0 && c->bd_valid)
            LSR_CUDA_TRY(launch_zt_bricks_state(P, c->band.state, c->bd, c->zt, s));
        else
            LSR_CUDA_TRY(launch_zt_bricks(P, c->dist, ids, L.est_active, c->zt, s));
        LSR_CUDA_TRY(launch_zt_fill(P, a, c->zt, s));
        zt_attach(P, c->zt);
    }
    LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, a, c->dist, ids, L.est_active, b, c->d_bad, s));
    loop_mark<<<1, 1, 0, s>>>(st, L.k, 3);
    // 4. reinitialise phi^{n+1} on the band of phi^n (driver.cpp:196), then a
    // takes phi^{n+1} where it may differ (the swap, driver.cpp:203, is the
    // caller's exchange of a and b)
    const ReinitParams R{rc->dtau, rc->max_iters, rc->residual_tol, rc->sign_eps};
    if (int e = lsr_reinit_enqueue(G, b, c->scratch, c->band, cfg->gamma, R, c->rb, L.rl, clamp_sparse, L.hard, s,
                                   &err))
        return set_err(e, err);
    if (int e = lsr_loop_sync_fields(G, b, a, c->scratch, c->band, c->rb, L.rl, cfg->gamma, L.hard, clamp_sparse, s,
                                      &err))
        return set_err(e, err);
    loop_record<<<1, 1, 0, s>>>(st, L.k, L.e2, c->band.counts, L.ew.nc, L.rl, c->d_bad, L.flags, cfg->p, L.hard);
    for (int q = 0; q < 5; ++q) lsr_note_launch();
    LSR_CUDA_TRY(cudaGetLastError());
    return LSR_OK;
}

std::string loop_key(const lsr_cuda_ctx* c, const double* a, const double* b, const lsr_step_cfg* cfg,
                     const lsr_reinit_cfg* rc, int refine) {
    std::string k;
    const auto put = [&k](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
    put(&a, sizeof a);
    put(&b, sizeof b);
    put(&c->scratch, sizeof c->scratch);
    put(&c->dist, sizeof c->dist);
    put(cfg, sizeof *cfg);
    put(rc, sizeof *rc);
    put(&refine, sizeof refine);
    put(&c->lr.est_active, sizeof c->lr.est_active);
    put(&c->lr.est_cells, sizeof c->lr.est_cells);
    put(&c->bd_valid, sizeof c->bd_valid);
    return k;
}

// the graph of one iteration with (a, b) in slot q, captured on first use and
// whenever its key changes
int loop_graph(lsr_cuda_ctx* c, int q, double* a, double* b, const lsr_step_cfg* cfg, const lsr_reinit_cfg* rc,
               int refine, cudaGraphExec_t* out) {
    auto& L = c->lr;
    const std::string key = loop_key(c, a, b, cfg, rc, refine);
    if (L.exec[q] && L.key[q] == key) {
        *out = L.exec[q];
        return LSR_OK;
    }
    if (L.exec[q]) cudaGraphExecDestroy(L.exec[q]);
    L.exec[q] = nullptr;
    const int64_t n0 = lsr_cuda_kernel_launches();
    LSR_CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int st = enqueue_loop_iteration(c, a, b, cfg, rc, refine, true);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (st) {
        if (g) cudaGraphDestroy(g);
        return st;
    }
    LSR_CUDA_TRY(ce);
    const cudaError_t ie = cudaGraphInstantiate(&L.exec[q], g, 0);
    cudaGraphDestroy(g);
    LSR_CUDA_TRY(ie);
    L.key[q] = key;
    L.launches[q] = lsr_cuda_kernel_launches() - n0;
    g_launches.fetch_sub(L.launches[q], std::memory_order_relaxed);  // counted when replayed
    *out = L.exec[q];
    return LSR_OK;
}

}  // namespace
}  // extern "C++"

int lsr_cuda_loop_run(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, const lsr_reinit_cfg* rc, int energy_refine,
                      int iterations, int use_graph, lsr_loop_stats* stats, int* done) {
    if (done) *done = 0;
    if (c && c->slab) return set_err(LSR_ERR_CONFIG, "loop_run: a z-slab context (use lsr_cuda_slab_*)");
    if (!c || !cfg || !rc) return set_err(LSR_ERR_CONFIG, "loop_run: null argument");
    if (iterations < 1) return set_err(LSR_ERR_CONFIG, "loop_run: iterations must be >= 1");
    if (int st = check_cfg(cfg, 1.0)) return st;
    if (!(rc->dtau > 0.0) || rc->max_iters < 1) return set_err(LSR_ERR_CONFIG, "reinit: invalid configuration");
    if (!(cfg->gamma > 0.0)) return set_err(LSR_ERR_CONFIG, "narrow_band: gamma must be positive");
    if (c->grid.dim == 3 && (energy_refine < 1 || energy_refine > 8))
        return set_err(LSR_ERR_CONFIG, "loop_run: energy_refine must be in [1, 8]");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    auto& L = c->lr;
    if (int st = loop_reserve(c, iterations)) return st;
    cudaStream_t s = c->stream;
    // count estimates size the grids of the count-driven launches (the
    // kernels stride past them, so they decide speed only): the last run's
    // counts, or the band of phi now
    if (L.est_active <= 0) {
        long long na = 0, nt = 0;
        std::string err;
        if (int st = lsr_band_build(grid_params(c->grid), c->phi, cfg->gamma, c->band, &na, &nt, s, &err))
            return set_err(st, err);
        L.est_active = na > 0 ? na : 1;
        L.est_cells = na / 4 + 1;
    }
    if (c->grid.dim == 3 && c->grid.dims[0] % 4 == 0 && !c->bd_valid) {
        LSR_CUDA_TRY(launch_brick_d(grid_params(c->grid), c->dist, c->bd, s));
        c->bd_valid = true;
    }
    const bool first_sparse =
        c->clamped_seq == c->seq && c->clamped_phi == c->phi && c->clamped_gamma == cfg->gamma;
    c->seq++;
    LSR_CUDA_TRY(cudaMemsetAsync(L.k, 0, sizeof(int), s));
    LSR_CUDA_TRY(cudaMemsetAsync(L.flags, 0, sizeof(int), s));
    LSR_CUDA_TRY(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), s));
    // the first iteration runs the dense one-step (nothing is known of phi's
    // hard jumps yet; its one-step and checks tell the next iteration)
    const int hard0[2] = {1, 0};
    LSR_CUDA_TRY(cudaMemcpyAsync(L.hard, hard0, sizeof hard0, cudaMemcpyHostToDevice, s));
    // out = phi on entry (afterwards every iteration leaves the two equal)
    LSR_CUDA_TRY(cudaMemcpyAsync(c->out, c->phi, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s));
    double* a = c->phi;
    double* b = c->out;
    for (int it = 0; it < iterations; ++it) {
        if (it == 0 || !use_graph) {
            if (int st = enqueue_loop_iteration(c, a, b, cfg, rc, energy_refine, it > 0 || first_sparse)) return st;
        } else {
            cudaGraphExec_t g = nullptr;
            const int q = (a == c->phi) ? 0 : 1;
            if (int st = loop_graph(c, q, a, b, cfg, rc, energy_refine, &g)) return st;
            LSR_CUDA_TRY(cudaGraphLaunch(g, s));
            g_launches.fetch_add(L.launches[q], std::memory_order_relaxed);
        }
        std::swap(a, b);
    }
    // the one host synchronisation of the run: the per-iteration records
    std::vector<LoopDevStat> h(static_cast<size_t>(iterations));
    LSR_CUDA_TRY(cudaMemcpyAsync(h.data(), L.stats, sizeof(LoopDevStat) * h.size(), cudaMemcpyDeviceToHost, s));
    LSR_CUDA_TRY(cudaStreamSynchronize(s));
    // the context after the run: phi = phi^{n+K} (fully clamped), out equal
    // to it, the active set = the band of the last iteration's phi^n
    c->phi = a;
    c->out = b;
    c->consistent = true;
    c->n_dirty = 0;
    c->dirty_is_active = false;
    c->zt_bricks = false;
    c->box_valid = false;
    c->clamped_seq = ++c->seq;
    c->clamped_phi = c->phi;
    c->clamped_gamma = cfg->gamma;
    const LoopDevStat& last = h.back();
    c->band.n_active = last.n_active;
    c->band.n_tube = last.n_tube;
    c->rb.n_frozen = last.n_frozen;
    if (int st = ensure_ids(&c->active, &c->cap_active, last.n_active)) return st;
    if (last.n_active > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, c->band.active, sizeof(int64_t) * last.n_active,
                                     cudaMemcpyDeviceToDevice, s));
    c->n_active = last.n_active;
    L.est_active = last.n_active + last.n_active / 16 + 256;
    L.est_cells = last.n_cells + last.n_cells / 16 + 256;
    for (int it = 0; it < iterations; ++it) {
        const LoopDevStat& r = h[static_cast<size_t>(it)];
        if (stats) {
            lsr_loop_stats& o = stats[it];
            o.energy = r.energy;
            o.n_active = r.n_active;
            o.n_tube = r.n_tube;
            o.reinit_iterations = r.iterations;
            o.had_interface = r.had_interface;
            for (int q = 0; q < 4; ++q) o.ms[q] = static_cast<float>(1e-6 * static_cast<double>(r.t[q + 1] - r.t[q]));
            o.dense_one_step = r.pad;
            o.reserved = 0;
        }
        // the first failing iteration ends the run (the reference throws
        // there; later iterations' results are unspecified)
        if (r.flags & 1) {
            if (done) *done = it;
            return set_err(LSR_ERR_OUT_OF_DOMAIN, "locate_cell: point outside grid hull");
        }
        if (r.flags & 2) {
            if (done) *done = it;
            return set_err(LSR_ERR, "sl_step: energy must be positive for p > 1");
        }
        if (r.bad != ~0ULL) {
            if (done) *done = it;
            return numerical_error(c->grid, r.bad, nullptr);
        }
    }
    if (done) *done = iterations;
    return LSR_OK;
}

int lsr_cuda_compute_stats(const double* pts, int64_t n, int dim, double sample_fraction, double k_s, uint64_t seed,
                           double* h_s, double* gamma_s, double* bbox6) {
    if ((n > 0 && !pts) || !h_s || !gamma_s || !bbox6) return set_err(LSR_ERR_CONFIG, "compute_stats: null argument");
    if (dim != 2 && dim != 3) return set_err(LSR_ERR_CONFIG, "compute_stats: dim must be 2 or 3");
    std::string err;
    const int st = lsr_prep_compute_stats(pts, n, dim, sample_fraction, k_s, seed, h_s, gamma_s, bbox6, nullptr, &err);
    if (st) return set_err(st, err);
    return LSR_OK;
}

int lsr_cuda_selftest_div_const(double c, int64_t n, uint64_t seed, int64_t* mismatches) {
    if (!pow2_range(c)) return set_err(LSR_ERR_CONFIG, "selftest: divisor outside [2^-100, 2^100]");
    unsigned long long* d = nullptr;
    LSR_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long)));
    LSR_CUDA_TRY(cudaMemset(d, 0, sizeof(unsigned long long)));
    LSR_CUDA_TRY(launch_div_selftest(c, 1.0 / c, seed, n, d));
    unsigned long long h = 0;
    LSR_CUDA_TRY(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost));
    cudaFree(d);
    *mismatches = static_cast<int64_t>(h);
    return LSR_OK;
}

int lsr_cuda_selftest_weno(double dx, int64_t n, uint64_t seed, int64_t* counts) {
    if (!counts || n < 0) return set_err(LSR_ERR_CONFIG, "selftest_weno: bad arguments");
    lsr_grid g{};
    g.dim = 3;
    g.dims[0] = g.dims[1] = g.dims[2] = 8;
    g.dx = dx;
    lsr_step_cfg c{};
    c.p = 1;
    c.interp = LSR_INTERP_WENO;
    c.dt = dx;
    c.gamma = 2.0;
    c.beta = 1.0;
    const SlParams P = make_params(g, c, 1.0);
    if (!P.fast_weno) return set_err(LSR_ERR_CONFIG, "selftest_weno: dx outside the fast path's range [2^-30, 1]");
    unsigned long long* d = nullptr;
    LSR_CUDA_TRY(cudaMalloc(&d, 4 * sizeof(unsigned long long)));
    LSR_CUDA_TRY(cudaMemset(d, 0, 4 * sizeof(unsigned long long)));
    LSR_CUDA_TRY(launch_weno_selftest(P, seed, n, d));
    unsigned long long h[4] = {0, 0, 0, 0};
    LSR_CUDA_TRY(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
    cudaFree(d);
    for (int q = 0; q < 4; ++q) counts[q] = static_cast<int64_t>(h[q]);
    return LSR_OK;
}


// ---------------------------------------------------------------------------
// z-slab loop: one rank's share of driver.cpp:185-203 on its
// owned planes; the caller (paper_2410_22205_b200/zslab.py) does the plane
// exchanges and the reductions between the phases.

static int slab_check(lsr_cuda_ctx* c) {
    if (!c) return set_err(LSR_ERR_CONFIG, "null context");
    if (!c->slab) return set_err(LSR_ERR_CONFIG, "slab: not a slab context (lsr_cuda_slab_create)");
    return LSR_OK;
}

static long long slab_off(const lsr_cuda_ctx* c) {
    return static_cast<long long>(c->win_lo) * c->grid.dims[0] * c->grid.dims[1];
}

int lsr_cuda_slab_create(int device, const lsr_grid* grid, int32_t win_lo, int32_t win_hi, int32_t own_lo,
                         int32_t own_hi, lsr_cuda_ctx** out) {
    if (!out) return set_err(LSR_ERR_CONFIG, "slab_create: null out");
    *out = nullptr;
    if (int st = check_grid(grid)) return st;
    const int nz = grid->dims[2];
    if (grid->dim != 3 || own_lo < 0 || own_hi > nz || own_lo >= own_hi || win_lo > std::max(own_lo - 1, 0) ||
        win_hi < std::min(own_hi + 1, nz) || win_lo < 0 || win_hi > nz)
        return set_err(LSR_ERR_CONFIG,
                       "slab_create: need a 3d grid and 0 <= win_lo <= own_lo - 1 < own_hi + 1 <= win_hi <= nz");
    const long long nxy = static_cast<long long>(grid->dims[0]) * grid->dims[1];
    if (nxy % 16 != 0) return set_err(LSR_ERR_CONFIG, "slab_create: planes must hold a multiple of 16 nodes");
    LSR_CUDA_TRY(cudaSetDevice(device));
    auto* c = new lsr_cuda_ctx;
    c->device = device;
    c->grid = *grid;
    c->slab = true;
    c->win_lo = win_lo;
    c->win_hi = win_hi;
    c->own_lo = own_lo;
    c->own_hi = own_hi;
    c->n = static_cast<int64_t>(win_hi - win_lo) * nxy;
    const size_t bytes = sizeof(double) * static_cast<size_t>(c->n);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&c->phi, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->out, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->dist, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->scratch, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_bad, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_aux, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_bad, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e != cudaSuccess) {
        lsr_cuda_destroy(c);
        return cuda_err(e, "lsr_cuda_slab_create");
    }
    c->stream = c->own;
    *out = c;
    return LSR_OK;
}

int lsr_cuda_slab_copy_planes(lsr_cuda_ctx* c, int which, int32_t plane0, int32_t nplanes, void* dev,
                              int32_t to_field) {
    if (int st = slab_check(c)) return st;
    double** slot = field_slot(c, which);
    if (!slot || !dev || nplanes < 0 || plane0 < c->win_lo || plane0 + nplanes > c->win_hi)
        return set_err(LSR_ERR_CONFIG, "slab_copy_planes: bad field or planes outside the resident window");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    const long long nxy = static_cast<long long>(c->grid.dims[0]) * c->grid.dims[1];
    double* f = *slot + (static_cast<long long>(plane0) - c->win_lo) * nxy;
    const size_t bytes = sizeof(double) * static_cast<size_t>(nplanes) * nxy;
    if (bytes == 0) return LSR_OK;
    if (to_field) LSR_CUDA_TRY(cudaMemcpyAsync(f, dev, bytes, cudaMemcpyDeviceToDevice, c->stream));
    else LSR_CUDA_TRY(cudaMemcpyAsync(dev, f, bytes, cudaMemcpyDeviceToDevice, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (to_field && which != LSR_FIELD_DIST) c->consistent = false;
    return LSR_OK;
}

int lsr_cuda_slab_band(lsr_cuda_ctx* c, int which, double gamma, int64_t* n_active, int64_t* n_tube) {
    if (int st = slab_check(c)) return st;
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "slab_band: phi must be PHI or OUT");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    long long na = 0, nt = 0;
    if (int st = lsr_band_build_slab(grid_params(c->grid), *slot - slab_off(c), gamma, c->band, c->win_lo, c->win_hi,
                                     c->own_lo, c->own_hi, &na, &nt, c->stream, &err))
        return set_err(st, err);
    if (int st = ensure_ids(&c->active, &c->cap_active, na)) return st;
    if (na > 0)
        LSR_CUDA_TRY(cudaMemcpyAsync(c->active, c->band.active, sizeof(int64_t) * na, cudaMemcpyDeviceToDevice,
                                     c->stream));
    c->n_active = na;
    if (n_active) *n_active = na;
    if (n_tube) *n_tube = nt;
    return LSR_OK;
}

int lsr_cuda_slab_energy_cells(lsr_cuda_ctx* c, int which, int p, int refine, int64_t* n_cells) {
    if (int st = slab_check(c)) return st;
    double** slot = field_slot(c, which);
    if (!slot || which == LSR_FIELD_DIST) return set_err(LSR_ERR_CONFIG, "slab_energy: phi must be PHI or OUT");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    long long nc = 0;
    const int k_hi = std::min(c->own_hi, c->grid.dims[2] - 1);  // cells (k, k+1) of the owned planes
    const long long off = slab_off(c);
    if (int st = lsr_energy_slab_cells(grid_params(c->grid), *slot - off, c->dist - off, p, refine, c->own_lo,
                                       std::max(k_hi, c->own_lo), c->ew, &nc, c->stream, &err))
        return set_err(st, err);
    if (n_cells) *n_cells = nc;
    return LSR_OK;
}

int lsr_cuda_slab_energy_pieces(lsr_cuda_ctx* c, int64_t offset, double* blocks, int64_t* n_blocks, double* head,
                                int64_t* n_head, double* tail, int64_t* n_tail) {
    if (int st = slab_check(c)) return st;
    if (!blocks || !head || !tail || !n_blocks || !n_head || !n_tail || offset < 0)
        return set_err(LSR_ERR_CONFIG, "slab_energy_pieces: null argument");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    long long nb = 0, nh = 0, nt = 0;
    if (int st = lsr_energy_slab_pieces(c->ew, offset, blocks, &nb, head, &nh, tail, &nt, c->stream, &err))
        return set_err(st, err);
    *n_blocks = nb;
    *n_head = nh;
    *n_tail = nt;
    return LSR_OK;
}

int lsr_cuda_slab_max_reach(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, double energy_p, double* cells) {
    if (int st = slab_check(c)) return st;
    if (int st = check_cfg(cfg, energy_p)) return st;
    if (!cells) return set_err(LSR_ERR_CONFIG, "slab_max_reach: null argument");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    SlParams P = make_params(c->grid, *cfg, energy_p);
    LSR_CUDA_TRY(cudaMemsetAsync(c->d_aux + 1, 0, sizeof(unsigned long long), c->stream));
    LSR_CUDA_TRY(launch_reach_max(P, c->dist - slab_off(c), c->active, c->n_active, c->d_aux + 1, c->stream));
    unsigned long long bits = 0;
    LSR_CUDA_TRY(cudaMemcpyAsync(&bits, c->d_aux + 1, sizeof bits, cudaMemcpyDeviceToHost, c->stream));
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    std::memcpy(cells, &bits, sizeof bits);
    return LSR_OK;
}

int lsr_cuda_slab_sl_step(lsr_cuda_ctx* c, const lsr_step_cfg* cfg, double energy_p, int64_t* bad_node,
                          int64_t* halo_miss) {
    if (bad_node) *bad_node = -1;
    if (halo_miss) *halo_miss = 0;
    if (int st = slab_check(c)) return st;
    if (int st = check_cfg(cfg, energy_p)) return st;
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    // out = phi on every resident node (evolve.cpp:50), then the owned active updates
    LSR_CUDA_TRY(cudaMemcpyAsync(c->out, c->phi, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s));
    LSR_CUDA_TRY(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), s));
    LSR_CUDA_TRY(cudaMemsetAsync(c->d_aux, 0, sizeof(unsigned long long), s));
    if (!(cfg->p > 1 && energy_p == 0.0) && c->n_active > 0) {  // driver.cpp:191-195
        SlParams P = make_params(c->grid, *cfg, energy_p);
        P.z_base = c->win_lo;
        P.z_planes = c->win_hi - c->win_lo;
        P.own_lo = c->own_lo;
        P.own_hi = c->own_hi;
        P.halo_miss = c->d_aux;
        const long long off = slab_off(c);
        if (int st = attach_slab_table(P, c->grid, cfg->interp, c->phi - off, c->dist - off, c->active, c->n_active, s))
            return st;
        LSR_CUDA_TRY(launch_sl_step(P, cfg->interp, c->phi - off, c->dist - off, c->active, c->n_active, c->out - off,
                                    c->d_bad, s));
    }
    unsigned long long h[2] = {0, 0};
    LSR_CUDA_TRY(cudaMemcpyAsync(&h[0], c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    LSR_CUDA_TRY(cudaMemcpyAsync(&h[1], c->d_aux, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    LSR_CUDA_TRY(cudaStreamSynchronize(s));
    c->consistent = false;
    if (halo_miss) *halo_miss = static_cast<int64_t>(h[1]);
    if (h[0] != ~0ULL) return numerical_error(c->grid, h[0], bad_node);
    return LSR_OK;
}

int lsr_cuda_slab_one_step(lsr_cuda_ctx* c, int* any_frozen, int* any_zero) {
    if (int st = slab_check(c)) return st;
    if (!any_frozen || !any_zero) return set_err(LSR_ERR_CONFIG, "slab_one_step: null argument");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    const long long off = slab_off(c);
    if (int st = lsr_reinit_one_step_slab(grid_params(c->grid), c->out - off, c->scratch - off, c->rb, c->win_lo,
                                          c->win_hi, c->own_lo, c->own_hi, any_frozen, any_zero, c->stream, &err))
        return set_err(st, err);
    return LSR_OK;
}

int lsr_cuda_slab_reinit_begin(lsr_cuda_ctx* c, const lsr_reinit_cfg* rc, int64_t* n_nodes) {
    if (int st = slab_check(c)) return st;
    if (!rc || !n_nodes) return set_err(LSR_ERR_CONFIG, "slab_reinit_begin: null argument");
    if (!c->band.state) return set_err(LSR_ERR_CONFIG, "slab_reinit_begin: build the band first (lsr_cuda_slab_band)");
    if (!(rc->dtau > 0.0) || rc->max_iters < 1) return set_err(LSR_ERR_CONFIG, "reinit: bad configuration");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    const ReinitParams R{rc->dtau, rc->max_iters, rc->residual_tol, rc->sign_eps};
    const long long off = slab_off(c);
    long long nn = 0;
    if (int st = lsr_reinit_slab_begin(grid_params(c->grid), c->scratch - off, c->out - off, c->band.tube,
                                       c->band.n_tube, R, c->rb, c->win_lo, c->win_hi, &nn, c->stream, &err))
        return set_err(st, err);
    c->reinit_nn = nn;
    *n_nodes = nn;
    return LSR_OK;
}

// sweep k reads buf[k & 1] and writes buf[(k + 1) & 1], buf = {SCRATCH, OUT}
int lsr_cuda_slab_reinit_sweep(lsr_cuda_ctx* c, const lsr_reinit_cfg* rc, int32_t k, double* residual) {
    if (int st = slab_check(c)) return st;
    if (!rc || !residual || k < 0) return set_err(LSR_ERR_CONFIG, "slab_reinit_sweep: bad argument");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    std::string err;
    const long long off = slab_off(c);
    double* buf[2] = {c->scratch - off, c->out - off};
    if (int st = lsr_reinit_slab_sweep(grid_params(c->grid), buf[k & 1], buf[(k + 1) & 1], c->rb, c->reinit_nn,
                                       rc->dtau, residual, c->stream, &err))
        return set_err(st, err);
    return LSR_OK;
}

// the reinitialised field is `which` (SCRATCH or OUT): clamp its owned
// planes (reinit.cpp:143) and make it the context's OUT field
int lsr_cuda_slab_reinit_end(lsr_cuda_ctx* c, int which, double gamma) {
    if (int st = slab_check(c)) return st;
    if (which != LSR_FIELD_SCRATCH && which != LSR_FIELD_OUT)
        return set_err(LSR_ERR_CONFIG, "slab_reinit_end: the result is SCRATCH or OUT");
    LSR_CUDA_TRY(cudaSetDevice(c->device));
    if (which == LSR_FIELD_SCRATCH) std::swap(c->out, c->scratch);
    const long long nxy = static_cast<long long>(c->grid.dims[0]) * c->grid.dims[1];
    std::string err;
    if (int st = lsr_clamp(c->out + (static_cast<long long>(c->own_lo) - c->win_lo) * nxy,
                           static_cast<long long>(c->own_hi - c->own_lo) * nxy, gamma, c->stream, &err))
        return set_err(st, err);
    LSR_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->consistent = false;
    return LSR_OK;
}

}  // extern "C"
