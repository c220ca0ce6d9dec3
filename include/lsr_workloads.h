/* lsr_workloads.h — seeded synthetic point clouds of the five BASELINE
 * configurations (BASELINE.json "configs"). The benchmark
 * clouds are not part of the reference, so these generators
 * stand in for them: same shapes, sizes and value distributions. Randomness
 * is std::mt19937_64 with 53-bit uniforms ((x >> 11) * 2^-53, the reference
 * tests' convention, test_interp.cpp:52-53) and Box-Muller normals, so a
 * (config, n, seed) triple gives the same cloud on every platform.
 *
 * Host-only helpers for tests and bench.py; not on the SL hot path.
 */
#ifndef LSR_WORKLOADS_H
#define LSR_WORKLOADS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* config ids */
#define LSR_CLOUD_CIRCLE 1       /* 2d circle r = 0.3, uniform seeded angles, no noise */
#define LSR_CLOUD_SPHERE 2       /* sphere r = 0.5, uniform on the surface */
#define LSR_CLOUD_TORUS 3        /* torus R = 0.5, r = 0.2 about z, (u,v) uniform + N(0, sigma^2 I) */
#define LSR_CLOUD_BUMPY 4        /* r(t,p) = 0.5(1 + 0.1 sin 5t cos 4p), density 1 + 9|cos t| (poles 10x) */
#define LSR_CLOUD_THREE_TORI 5   /* union of tori R = 0.3, r = 0.1 at x = -0.5, 0, 0.5, two caps removed, noise */

/* Writes n points (x, y, z; z = 0 in 2d) into pts[3n]. sigma is the noise
 * standard deviation (configs 3 and 5; ignored elsewhere). Returns 0, or -1
 * for an unknown config. */
int lsr_cloud_generate(int config, int64_t n, uint64_t seed, double sigma, double* pts);

#ifdef __cplusplus
}
#endif
#endif
