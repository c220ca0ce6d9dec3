// Host-side packing of the distance values one SL step reads. See host_pack.h.
#include "host_pack.h"

#include <algorithm>
#include <cstring>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace lsr_host {

void copy_stream(void* dst, const void* src, size_t bytes) {
#if defined(__SSE2__)
    auto* d = static_cast<unsigned char*>(dst);
    auto* s = static_cast<const unsigned char*>(src);
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
    if (bytes < head + 64) {
        std::memcpy(d, s, bytes);
        return;
    }
    std::memcpy(d, s, head);
    d += head;
    s += head;
    bytes -= head;
    const size_t body = bytes & ~static_cast<size_t>(63);
    for (size_t i = 0; i < body; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
        const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
    }
    _mm_sfence();
    std::memcpy(d + body, s + body, bytes - body);
#else
    std::memcpy(dst, src, bytes);
#endif
}

Pool::Pool(int threads) {
    for (int t = 0; t < std::max(1, threads); ++t) workers_.emplace_back([this] { loop(); });
}

Pool::~Pool() {
    {
        std::lock_guard<std::mutex> l(m_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& th : workers_) th.join();
}

void Pool::post(int n, std::function<void(int)> fn) {
    {
        std::lock_guard<std::mutex> l(m_);
        fn_ = std::move(fn);
        n_ = n;
        next_.store(0);
        busy_ = size();
        ++gen_;
    }
    cv_.notify_all();
}

void Pool::wait() {
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [this] { return busy_ == 0; });
}

void Pool::loop() {
    uint64_t seen = 0;
    for (;;) {
        std::function<void(int)>* fn;
        int n;
        {
            std::unique_lock<std::mutex> l(m_);
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            fn = &fn_;
            n = n_;
        }
        for (int k = next_.fetch_add(1); k < n; k = next_.fetch_add(1)) (*fn)(k);
        std::lock_guard<std::mutex> l(m_);
        if (--busy_ == 0) done_cv_.notify_all();
    }
}

namespace {

// a sorted interval source for row_union: rows shift by dj, x ranges widen by
// grow (clipped to the grid)
struct Src {
    const Run* p;
    const Run* e;
    int dj, grow;
};

// Appends to out the union of the sources' intervals, row by row in
// ascending order: each source is ascending in (j, x0), so a scan of the
// source heads finds the next row; its intervals are insertion-sorted by x0
// (a row holds a handful) and overlapping or touching ones are fused.
void row_union(Src* src, int ns, int nx, int ny, std::vector<Run>& row, std::vector<Run>& out) {
    constexpr int kNone = 1 << 30;
    for (;;) {
        int j = kNone;
        for (int s = 0; s < ns; ++s) {
            Src& q = src[s];
            while (q.p < q.e && (q.p->j + q.dj < 0 || q.p->j + q.dj >= ny)) ++q.p;
            if (q.p < q.e) j = std::min(j, q.p->j + q.dj);
        }
        if (j == kNone) return;
        row.clear();
        for (int s = 0; s < ns; ++s) {
            Src& q = src[s];
            for (; q.p < q.e && q.p->j + q.dj == j; ++q.p) {
                const Run w{j, std::max(0, q.p->x0 - q.grow), std::min(nx - 1, q.p->x1 + q.grow)};
                size_t at = row.size();
                row.push_back(w);
                while (at > 0 && row[at - 1].x0 > w.x0) {
                    row[at] = row[at - 1];
                    --at;
                }
                row[at] = w;
            }
        }
        const size_t first = out.size();
        for (const Run& r : row) {
            if (out.size() > first && r.x0 <= out.back().x1 + 1)
                out.back().x1 = std::max(out.back().x1, r.x1);
            else
                out.push_back(r);
        }
    }
}

// sets bits [x0, x1] of a row bitmap
void set_bits(uint64_t* row, int x0, int x1) {
    int w0 = x0 >> 6, w1 = x1 >> 6;
    const uint64_t lo = ~0ULL << (x0 & 63), hi = ~0ULL >> (63 - (x1 & 63));
    if (w0 == w1) {
        row[w0] |= lo & hi;
        return;
    }
    row[w0] |= lo;
    for (int w = w0 + 1; w < w1; ++w) row[w] = ~0ULL;
    row[w1] |= hi;
}

// appends the runs of set bits of a row bitmap (nx bits) as row j's runs
void bit_runs(const uint64_t* row, int words, int nx, int j, std::vector<Run>& out) {
    int x = 0;
    while (x < nx) {
        // next set bit at or after x
        int w = x >> 6;
        uint64_t v = row[w] & (~0ULL << (x & 63));
        while (!v && ++w < words) v = row[w];
        if (w >= words) return;
        const int s = (w << 6) + __builtin_ctzll(v);
        if (s >= nx) return;
        // next clear bit after s
        w = s >> 6;
        v = ~row[w] & (~0ULL << (s & 63));
        while (!v && ++w < words) v = ~row[w];
        const int e = w >= words ? nx : std::min(nx, (w << 6) + __builtin_ctzll(v));
        out.push_back({j, s, e - 1});
        x = e;
    }
}

int64_t count_values(const std::vector<Run>& runs) {
    int64_t v = 0;
    for (const Run& r : runs) v += r.x1 - r.x0 + 1;
    return v;
}

}  // namespace

void PackSet::finish_offsets() {
    // on entry val_off[k + 1] / run_off[k + 1] hold plane k's own counts
    for (size_t k = 1; k < val_off.size(); ++k) {
        val_off[k] += val_off[k - 1];
        run_off[k] += run_off[k - 1];
    }
}

bool StepPacker::plan(const int64_t* ids, int64_t n, int nx, int ny, int nz, int reach, int threads) {
    if (!pool_ || pool_->size() != threads) pool_.reset(new Pool(threads));
    nx_ = nx;
    ny_ = ny;
    nz_ = nz;
    reach_ = reach;
    const int64_t nxy = static_cast<int64_t>(nx) * ny;
    std::vector<int64_t> first(nz + 1);
    for (int k = 0; k <= nz; ++k) first[k] = std::lower_bound(ids, ids + n, k * nxy) - ids;
    if (first[0] != 0 || first[nz] != n) return false;  // ids below 0 or beyond the grid
    active_.resize(nz);  // vectors keep their capacity across calls
    scratch_.resize(nz);
    for (PackSet* ps : {&d_, &phi_}) {
        ps->runs.resize(nz);
        ps->val_off.assign(nz + 1, 0);
        ps->run_off.assign(nz + 1, 0);
    }
    words_ = (nx + 63) / 64;
    if (reach > 0) bits_.resize(static_cast<size_t>(nz) * ny * words_);
    std::atomic<bool> ok{true};
    // 1. runs of active nodes per plane; every plane's slice of the ids must
    //    be non-decreasing and inside the plane, which (with the slices in
    //    plane order covering [0, n)) makes the whole list non-decreasing.
    pool_->run(nz, [&](int k) {
        const int64_t a = first[k], b = first[k + 1];
        const int64_t base = k * nxy;
        if (a > b || (a < b && (ids[a] < base || ids[b - 1] >= base + nxy))) {
            ok = false;
            return;
        }
        std::vector<Run> runs;  // local: pushing through active_[k] would false-share the vector headers
        runs.swap(active_[k]);
        runs.clear();
        const auto push = [&](int64_t rs, int64_t re) {
            const int32_t j = static_cast<int32_t>((rs - base) / nx);
            const int64_t row = base + static_cast<int64_t>(j) * nx;
            runs.push_back({j, static_cast<int32_t>(rs - row), static_cast<int32_t>(re - row)});
        };
        if (a < b) {
            // the current run [rs, re] (node ids) is held in registers
            int64_t rs = ids[a], re = rs;
            int64_t row_end = base + ((rs - base) / nx + 1) * nx;  // one past the run's row
            for (int64_t i = a + 1; i < b; ++i) {
                const int64_t id = ids[i];
                if (id < re) {  // descending
                    ok = false;
                    return;
                }
                if (id <= re + 1 && id < row_end) {  // extends (or repeats into) the run
                    re = id;
                    continue;
                }
                push(rs, re);
                rs = re = id;
                if (id >= row_end) row_end = base + ((id - base) / nx + 1) * nx;
            }
            push(rs, re);
        }
        if (reach > 0) {  // plane k's active runs widened by R in x, as a bitmap
            uint64_t* bm = bits_.data() + static_cast<size_t>(k) * ny * words_;
            std::fill(bm, bm + static_cast<size_t>(ny) * words_, 0ULL);
            for (const Run& r : runs) set_bits(bm + static_cast<size_t>(r.j) * words_, std::max(0, r.x0 - reach),
                                               std::min(nx - 1, r.x1 + reach));
        }
        active_[k].swap(runs);
    });
    if (!ok) return false;
    // 2. per plane: the d set = the plane's runs widened by one in x, the
    //    same runs on rows j-1 and j+1, and the runs of planes k-1 and k+1;
    //    the phi set = the union of planes k-R..k+R's runs, then of that
    //    union's rows j-R..j+R, widened by R in x.
    pool_->run(nz, [&](int k) {
        static const std::vector<Run> none;
        const auto src_of = [&](const std::vector<Run>& v, int dj, int grow) {
            return Src{v.data(), v.data() + v.size(), dj, grow};
        };
        std::vector<Run> row, out;
        row.swap(scratch_[k]);
        {
            const std::vector<Run>& A = active_[k];
            Src src[5] = {src_of(A, 0, 1), src_of(A, -1, 0), src_of(A, 1, 0),
                          src_of(k > 0 ? active_[k - 1] : none, 0, 0),
                          src_of(k + 1 < nz ? active_[k + 1] : none, 0, 0)};
            out.swap(d_.runs[k]);
            out.clear();
            row_union(src, 5, nx, ny, row, out);
            d_.val_off[k + 1] = count_values(out);
            d_.run_off[k + 1] = static_cast<int64_t>(out.size());
            d_.runs[k].swap(out);
        }
        if (reach > 0) {
            // the ball = OR of the widened bitmaps over planes k-R..k+R, then
            // over rows j-R..j+R; its runs are read off the bitmap
            const size_t plane = static_cast<size_t>(ny) * words_;
            std::vector<uint64_t> zor(plane, 0ULL), yor(plane);
            for (int kk = std::max(0, k - reach); kk <= std::min(nz - 1, k + reach); ++kk) {
                const uint64_t* b = bits_.data() + static_cast<size_t>(kk) * plane;
                for (size_t w = 0; w < plane; ++w) zor[w] |= b[w];
            }
            for (int j = 0; j < ny; ++j) {
                uint64_t* dst = yor.data() + static_cast<size_t>(j) * words_;
                std::fill(dst, dst + words_, 0ULL);
                for (int jj = std::max(0, j - reach); jj <= std::min(ny - 1, j + reach); ++jj) {
                    const uint64_t* b = zor.data() + static_cast<size_t>(jj) * words_;
                    for (int w = 0; w < words_; ++w) dst[w] |= b[w];
                }
            }
            out.swap(phi_.runs[k]);
            out.clear();
            for (int j = 0; j < ny; ++j) bit_runs(yor.data() + static_cast<size_t>(j) * words_, words_, nx, j, out);
            phi_.val_off[k + 1] = count_values(out);
            phi_.run_off[k + 1] = static_cast<int64_t>(out.size());
            phi_.runs[k].swap(out);
        } else {
            phi_.runs[k].clear();
        }
        scratch_[k].swap(row);
    });
    d_.finish_offsets();
    phi_.finish_offsets();
    return true;
}

namespace {

void gather_set(const PackSet& ps, int k, int64_t base, int nx, const double* field, double* vals, RunDesc* desc) {
    int64_t src = ps.val_off[k];
    RunDesc* d = desc + ps.run_off[k];
    for (const Run& r : ps.runs[k]) {
        const int64_t dst = base + static_cast<int64_t>(r.j) * nx + r.x0;
        const int64_t len = r.x1 - r.x0 + 1;
        std::memcpy(vals + src, field + dst, sizeof(double) * len);
        *d++ = {dst, src};
        src += len;
    }
}

}  // namespace

void StepPacker::gather_plane(int k, const double* dist, double* d_vals, RunDesc* d_desc, const double* phi,
                              double* phi_vals, RunDesc* phi_desc) const {
    const int64_t base = static_cast<int64_t>(k) * nx_ * ny_;
    gather_set(d_, k, base, nx_, dist, d_vals, d_desc);
    if (reach_ > 0 && phi) gather_set(phi_, k, base, nx_, phi, phi_vals, phi_desc);
}

}  // namespace lsr_host
