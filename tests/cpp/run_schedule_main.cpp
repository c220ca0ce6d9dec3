// run_schedule_main.cpp — drives the reference's own lsr::run_schedule
// (driver.cpp:139-230) on small seeded clouds and writes every run's final
// phi and the per-iteration log as raw bytes, so that builds of the same
// program can be compared bit for bit:
//   run_schedule_ref   all reference sources (oracle/_ref, pure CPU)
//   run_schedule_optA  the reference sources minus evolve.cpp, compiled
//                      against include/ and linked with liblsr_b200.so
//                      (INTEGRATION.md Option A: sl_step on the GPU)
//   run_schedule_optB  minus evolve.cpp, grid.cpp, distance.cpp and
//                      reinit.cpp (Option B: band, clamp, distance field
//                      and reinitialisation on the GPU as well)
// Usage: run_schedule_<x> <out-file>. Test infrastructure only.
#include <cstdio>
#include <cstring>
#include <vector>

#include "lsr/driver.hpp"

namespace {

void put(std::FILE* f, const void* p, std::size_t n) { std::fwrite(p, 1, n, f); }

void dump(std::FILE* f, const lsr::ScheduleResult& res) {
    put(f, &res.h_s, sizeof res.h_s);
    put(f, &res.gamma_s, sizeof res.gamma_s);
    for (const lsr::RunResult& r : res.runs) {
        put(f, &r.iterations, sizeof r.iterations);
        put(f, &r.dx, sizeof r.dx);
        put(f, &r.final_e2, sizeof r.final_e2);
        put(f, &r.final_err_s, sizeof r.final_err_s);
        const std::int64_t n = static_cast<std::int64_t>(r.phi.values.size());
        put(f, &n, sizeof n);
        put(f, r.phi.values.data(), sizeof(double) * r.phi.values.size());
    }
    for (const lsr::LogRow& row : res.log) {
        put(f, &row.run, sizeof row.run);
        put(f, &row.rec.iter, sizeof row.rec.iter);
        put(f, &row.rec.e2, sizeof row.rec.e2);
        put(f, &row.rec.delta_e, sizeof row.rec.delta_e);
        put(f, &row.rec.err_cloud, sizeof row.rec.err_cloud);
        put(f, &row.rec.l1_update, sizeof row.rec.l1_update);
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s out-file\n", argv[0]);
        return 2;
    }
    std::FILE* f = std::fopen(argv[1], "wb");
    if (!f) return 2;
    try {
        // 2d circle (radius 0.4, 96 points), Q1, three runs (Table 1 schedule)
        lsr::ShapeSpec circle;
        circle.kind = lsr::ShapeKind::Circle;
        circle.size = 0.4;
        circle.n_points = 96;
        lsr::ScheduleConfig c2;
        c2.interp = lsr::InterpolatorKind::Q1;
        c2.max_iters = 40;
        dump(f, lsr::run_schedule(lsr::sample_shape(circle, 7), c2));
        // 3d sphere (radius 0.5, 1500 Fibonacci points), WENO, three runs
        lsr::ShapeSpec sphere;
        sphere.kind = lsr::ShapeKind::Sphere;
        sphere.size = 0.5;
        sphere.n_points = 1500;
        lsr::ScheduleConfig c3;
        c3.interp = lsr::InterpolatorKind::Weno;
        c3.max_iters = 12;
        dump(f, lsr::run_schedule(lsr::sample_shape(sphere, 7), c3));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        std::fclose(f);
        return 1;
    }
    std::fclose(f);
    std::printf("ok\n");
    return 0;
}
