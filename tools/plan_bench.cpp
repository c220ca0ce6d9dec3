// Times StepPacker::plan and the gathers (csrc/host_pack.cpp) on the 512^3 sphere band:
//   g++ -O3 -march=native -std=c++17 -I paper_2410_22205_b200/csrc tools/plan_bench.cpp \
//       paper_2410_22205_b200/csrc/host_pack.cpp -pthread -o /tmp/pb && /tmp/pb THREADS REACH
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "host_pack.h"
using namespace lsr_host;

int main(int argc, char** argv) {
    const int n = 512, T = argc > 1 ? atoi(argv[1]) : 8, R = argc > 2 ? atoi(argv[2]) : 5;
    std::vector<int64_t> ids;
    const double dx = 2.0 / (n - 1), gamma = 6 * dx;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const double x = -1 + i * dx, y = -1 + j * dx, z = -1 + k * dx;
                if (std::fabs(std::sqrt(x * x + y * y + z * z) - 0.9) < gamma) ids.push_back((int64_t(k) * n + j) * n + i);
            }
    std::vector<double> d(size_t(n) * n * n, 1.0);
    StepPacker pk;
    std::vector<double> dv(20000000), pv(40000000);
    std::vector<RunDesc> dd(2000000), pd(2000000);
    for (int it = 0; it < 5; ++it) {
        const auto t0 = std::chrono::steady_clock::now();
        pk.plan(ids.data(), ids.size(), n, n, n, R, T);
        const auto t1 = std::chrono::steady_clock::now();
        pk.pool().run(n, [&](int k) { pk.gather_plane(k, d.data(), dv.data(), dd.data(), d.data(), pv.data(), pd.data()); });
        const auto t2 = std::chrono::steady_clock::now();
        std::printf("plan %.2f ms gather %.2f ms (%zu ids; d %lld, phi %lld values)\n",
                    std::chrono::duration<double, std::milli>(t1 - t0).count(),
                    std::chrono::duration<double, std::milli>(t2 - t1).count(), ids.size(),
                    static_cast<long long>(pk.dset().total_values()), static_cast<long long>(pk.phiset().total_values()));
    }
}
