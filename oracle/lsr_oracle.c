/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference's narrow-band semi-Lagrangian step
 * and its helpers (arXiv 2410.22205 artifact, /root/reference/proj). The
 * operation order of every floating-point expression follows the cited
 * reference line; build with -ffp-contract=off (oracle/Makefile) so no FMA
 * is formed, exactly like the reference (proj/CMakeLists.txt:28-30).
 *
 * Parity of this restatement is pinned by tests/test_oracle.py against the
 * reference library itself (oracle/_ref, built from the reference sources)
 * and against the committed golden vectors in tests/golden/.
 */
#include "lsr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_msg[256];

const char* lsro_last_error(void) { return g_msg; }

static int fail(int code, const char* msg) {
    snprintf(g_msg, sizeof g_msg, "%s", msg);
    return code;
}

/* std::min / std::max semantics: max(a,b) = (a < b) ? b : a, min(a,b) = (b < a) ? b : a */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double sqr(double x) { return x * x; } /* types.hpp:61 */

static inline int64_t gidx(const lsr_grid* g, int i, int j, int k) { /* grid.hpp:19-21 */
    return ((int64_t)k * g->dims[1] + j) * g->dims[0] + i;
}

static inline double at(const lsr_grid* g, const double* f, int i, int j, int k) {
    return f[gidx(g, i, j, k)];
}

/* Grid::node (grid.hpp:28-30) */
static inline void node(const lsr_grid* g, int i, int j, int k, double out[3]) {
    out[0] = g->origin[0] + i * g->dx;
    out[1] = g->origin[1] + j * g->dx;
    out[2] = g->origin[2] + k * g->dx;
}

/* Grid::upper (grid.hpp:31-34) */
static inline void upper(const lsr_grid* g, double hi[3]) {
    for (int d = 0; d < 3; ++d) hi[d] = g->origin[d] + (g->dims[d] - 1) * g->dx;
}

/* Grid::contains (grid.hpp:36-41) */
static int contains(const lsr_grid* g, const double p[3]) {
    double hi[3];
    upper(g, hi);
    for (int d = 0; d < g->dim; ++d)
        if (p[d] < g->origin[d] || p[d] > hi[d]) return 0;
    return 1;
}

/* Grid::clamp_to_hull (grid.hpp:42-48) */
static void clamp_to_hull(const lsr_grid* g, const double p[3], double q[3]) {
    double hi[3];
    upper(g, hi);
    q[0] = p[0];
    q[1] = p[1];
    q[2] = p[2];
    for (int d = 0; d < g->dim; ++d) q[d] = smin(smax(q[d], g->origin[d]), hi[d]);
    if (g->dim == 2) q[2] = 0.0;
}

/* locate_cell (grid.cpp:39-47) */
int lsro_locate_cell(const lsr_grid* g, const double p[3], int32_t c[3]) {
    if (!contains(g, p)) return fail(LSR_ERR_OUT_OF_DOMAIN, "locate_cell: point outside grid hull");
    c[0] = c[1] = c[2] = 0;
    for (int d = 0; d < g->dim; ++d) {
        int cd = (int)floor((p[d] - g->origin[d]) / g->dx);
        int hi = g->dims[d] - 2;
        c[d] = cd < 0 ? 0 : (hi < cd ? hi : cd); /* std::clamp */
    }
    return LSR_OK;
}

/* centered_gradient (grid.cpp:53-74) */
void lsro_centered_gradient(const lsr_grid* g, const double* f, int i, int j, int k, double gr[3]) {
    const double inv2 = 1.0 / (2.0 * g->dx);
    const double inv1 = 1.0 / g->dx;
    const int id[3] = {i, j, k};
    gr[0] = gr[1] = gr[2] = 0.0;
    for (int d = 0; d < g->dim; ++d) {
        int lo[3] = {i, j, k}, hi[3] = {i, j, k};
        if (id[d] == 0) {
            hi[d] = 1;
            gr[d] = (at(g, f, hi[0], hi[1], hi[2]) - at(g, f, i, j, k)) * inv1;
        } else if (id[d] == g->dims[d] - 1) {
            lo[d] = g->dims[d] - 2;
            gr[d] = (at(g, f, i, j, k) - at(g, f, lo[0], lo[1], lo[2])) * inv1;
        } else {
            lo[d] -= 1;
            hi[d] += 1;
            gr[d] = (at(g, f, hi[0], hi[1], hi[2]) - at(g, f, lo[0], lo[1], lo[2])) * inv2;
        }
    }
}

/* cutoff_weight (grid.cpp:136-143); validation hoisted to the caller */
double lsro_cutoff_weight(double phi, double gamma, double beta) {
    const double a = fabs(phi);
    if (a <= beta) return 1.0;
    if (a > gamma) return 0.0;
    return sqr(a - gamma) * (2.0 * a + gamma - 3.0 * beta) /
           ((gamma - beta) * (gamma - beta) * (gamma - beta));
}

/* weno_1d (interp.cpp:16-33) with weno_indicators (:11-14) and
 * weno_linear_weights (:7-9) inlined in the same operation order */
double lsro_weno_1d(const double v[4], double dx, double t) {
    const double vm = v[0], v0 = v[1], vp = v[2], vpp = v[3];
    const double pl = v0 + t * (0.5 * (vp - vm)) + t * t * (0.5 * (vm - 2.0 * v0 + vp));
    const double pr = v0 + t * (0.5 * (-3.0 * v0 + 4.0 * vp - vpp)) + t * t * (0.5 * (v0 - 2.0 * vp + vpp));
    const double il = sqr(v[0] - 2.0 * v[1] + v[2]) / (dx * dx);
    const double ir = sqr(v[1] - 2.0 * v[2] + v[3]) / (dx * dx);
    const double cl = (2.0 - t) / 3.0, cr = (1.0 + t) / 3.0;
    const double eps = dx * dx;
    const double al = cl / sqr(il + eps);
    const double ar = cr / sqr(ir + eps);
    const double wl = al / (al + ar);
    const double wr = ar / (al + ar);
    return wl * pl + wr * pr;
}

/* AxisStencil / axis_stencil / blend_1d (interp.cpp:37-59) */
typedef struct {
    int base, count;
    double theta;
} axis_st;

static axis_st axis_stencil(const lsr_grid* g, int axis, int cell, double coord) {
    axis_st s;
    s.theta = (coord - (g->origin[axis] + cell * g->dx)) / g->dx;
    if (cell - 1 >= 0 && cell + 2 <= g->dims[axis] - 1) {
        s.base = cell - 1;
        s.count = 4;
    } else {
        s.base = cell;
        s.count = 2;
    }
    return s;
}

static double blend_1d(const axis_st* s, const double* v, double dx) {
    if (s->count == 2) return (1.0 - s->theta) * v[0] + s->theta * v[1];
    return lsro_weno_1d(v, dx, s->theta);
}

/* interp_q1 (interp.cpp:63-81) */
static int interp_q1(const lsr_grid* g, const double* f, const double p[3], double* out) {
    int32_t c[3];
    int st = lsro_locate_cell(g, p, c);
    if (st) return st;
    double t[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < g->dim; ++d) t[d] = (p[d] - (g->origin[d] + c[d] * g->dx)) / g->dx;
    double value = 0.0;
    const int kz = g->dim == 3 ? 1 : 0;
    for (int dk = 0; dk <= kz; ++dk)
        for (int dj = 0; dj <= 1; ++dj)
            for (int di = 0; di <= 1; ++di) {
                const double w = (di ? t[0] : 1.0 - t[0]) * (dj ? t[1] : 1.0 - t[1]) *
                                 (g->dim == 3 ? (dk ? t[2] : 1.0 - t[2]) : 1.0);
                value += w * at(g, f, c[0] + di, c[1] + dj, c[2] + dk);
            }
    *out = value;
    return LSR_OK;
}

/* interp_weno (interp.cpp:83-111) */
static int interp_weno(const lsr_grid* g, const double* f, const double p[3], double* out) {
    int32_t c[3];
    int st = lsro_locate_cell(g, p, c);
    if (st) return st;
    const axis_st sx = axis_stencil(g, 0, c[0], p[0]);
    const axis_st sy = axis_stencil(g, 1, c[1], p[1]);
    double col[4];
    if (g->dim == 2) {
        for (int a = 0; a < sx.count; ++a) {
            double line[4];
            for (int b = 0; b < sy.count; ++b) line[b] = at(g, f, sx.base + a, sy.base + b, 0);
            col[a] = blend_1d(&sy, line, g->dx);
        }
        *out = blend_1d(&sx, col, g->dx);
        return LSR_OK;
    }
    const axis_st sz = axis_stencil(g, 2, c[2], p[2]);
    for (int a = 0; a < sx.count; ++a) {
        double plane[4];
        for (int b = 0; b < sy.count; ++b) {
            double line[4];
            for (int e = 0; e < sz.count; ++e) line[e] = at(g, f, sx.base + a, sy.base + b, sz.base + e);
            plane[b] = blend_1d(&sz, line, g->dx);
        }
        col[a] = blend_1d(&sy, plane, g->dx);
    }
    *out = blend_1d(&sx, col, g->dx);
    return LSR_OK;
}

/* interp (interp.cpp:113-119) */
int lsro_interp(int kind, const lsr_grid* g, const double* f, const double p[3], double* out) {
    if (kind == LSR_INTERP_Q1) return interp_q1(g, f, p, out);
    if (kind == LSR_INTERP_WENO) return interp_weno(g, f, p, out);
    return fail(LSR_ERR_CONFIG, "interp: unknown interpolator kind");
}

/* norm / dot (types.hpp:58-60) */
static inline double vnorm(const double a[3]) { return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

/* tangent_basis (evolve.cpp:10-30) */
void lsro_tangent_basis(int dim, const double g[3], double v1[3], double v2[3]) {
    v1[0] = v1[1] = v1[2] = 0.0;
    v2[0] = v2[1] = v2[2] = 0.0;
    const double gnorm = vnorm(g);
    if (dim == 2) {
        if (gnorm == 0.0) {
            v1[0] = 1.0;
            return;
        }
        v1[0] = g[1] / gnorm;
        v1[1] = -g[0] / gnorm;
        v1[2] = 0.0;
        return;
    }
    const double r = sqrt(sqr(g[0]) + sqr(g[2]));
    if (gnorm == 0.0 || r < 1e-14 * gnorm) {
        v1[0] = 1.0;
        v2[2] = 1.0;
        return;
    }
    v1[0] = -g[2] / r;
    v1[1] = 0.0;
    v1[2] = g[0] / r;
    v2[0] = -g[0] * g[1] / (r * gnorm);
    v2[1] = r / gnorm;
    v2[2] = -g[1] * g[2] / (r * gnorm);
}

/* scale_factor (evolve.cpp:32-38) */
int lsro_scale_factor(double d_j, double energy_p, int p, double* out) {
    if (p == 1) {
        *out = 1.0;
        return LSR_OK;
    }
    if (!(energy_p > 0.0)) return fail(LSR_ERR, "scale_factor: energy must be positive for p > 1");
    double f = 1.0;
    for (int i = 1; i < p; ++i) f *= d_j / energy_p;
    *out = f;
    return LSR_OK;
}

/* StepConfig::validate (evolve.hpp:25-30) + BandParams::validate (grid.hpp:90-92) */
static int validate_cfg(const lsr_step_cfg* c) {
    if (c->p != 1 && c->p != 2) return fail(LSR_ERR_CONFIG, "step: p must be 1 or 2");
    if (!(c->dt > 0.0)) return fail(LSR_ERR_CONFIG, "step: dt must be positive");
    if (c->delta < 0.0 || c->delta > 1.0) return fail(LSR_ERR_CONFIG, "step: delta must be in [0, 1]");
    if (!(c->beta > 0.0) || !(c->beta < c->gamma)) return fail(LSR_ERR_CONFIG, "band: need 0 < beta < gamma");
    if (c->interp != LSR_INTERP_Q1 && c->interp != LSR_INTERP_WENO)
        return fail(LSR_ERR_CONFIG, "interp: unknown interpolator kind");
    return LSR_OK;
}

/* One active node of sl_step (evolve.cpp:58-110). Returns next. */
static double sl_node(const lsr_grid* g, const double* phi, const double* dist, int64_t id,
                      const lsr_step_cfg* cfg, double energy_p, double grad_threshold) {
    const int nx = g->dims[0], ny = g->dims[1];
    const int i = (int)(id % nx);
    const int j = (int)((id / nx) % ny);
    const int k = (int)(id / ((int64_t)nx * ny));
    const double phi_j = phi[id];
    double grad_phi[3];
    lsro_centered_gradient(g, phi, i, j, k, grad_phi);
    double star;
    if (vnorm(grad_phi) < grad_threshold) { /* evolve.cpp:65-78 */
        double sum = 0.0;
        int count = 0;
        for (int ax = 0; ax < g->dim; ++ax)
            for (int s = -1; s <= 1; s += 2) {
                int nb[3] = {i, j, k};
                nb[ax] += s;
                if (nb[ax] < 0 || nb[ax] >= g->dims[ax]) continue;
                double p[3], v;
                node(g, nb[0], nb[1], nb[2], p);
                lsro_interp(cfg->interp, g, phi, p, &v);
                sum += v;
                ++count;
            }
        star = sum / count;
    } else { /* evolve.cpp:79-105 */
        const double d_j = dist[id];
        double grad_d[3];
        lsro_centered_gradient(g, dist, i, j, k, grad_d);
        double c_j;
        lsro_scale_factor(d_j, energy_p, cfg->p, &c_j); /* energy checked by the caller */
        double nd[3], base[3];
        node(g, i, j, k, nd);
        const double s = c_j * cfg->dt;
        for (int d = 0; d < 3; ++d) base[d] = nd[d] + s * grad_d[d];
        const double spread = sqrt(smax(0.0, c_j * cfg->delta * d_j * cfg->dt / cfg->p));
        double v1[3], v2[3];
        lsro_tangent_basis(g->dim, grad_phi, v1, v2);
        double sum = 0.0;
        const int nfeet = g->dim == 2 ? 2 : 4;
        for (int f = 0; f < nfeet; ++f) {
            double foot[3];
            if (g->dim == 2) {
                const int sg = f == 0 ? -1 : 1;
                const double a = sg * spread;
                for (int d = 0; d < 3; ++d) foot[d] = base[d] + a * v1[d];
            } else {
                const int s1 = f < 2 ? -1 : 1, s2 = (f & 1) ? 1 : -1;
                const double a = s1 * spread, b = s2 * spread;
                for (int d = 0; d < 3; ++d) foot[d] = base[d] + a * v1[d] + b * v2[d];
            }
            double val;
            if (!isfinite(foot[0]) || !isfinite(foot[1]) || !isfinite(foot[2])) {
                val = NAN;
            } else {
                double q[3];
                clamp_to_hull(g, foot, q);
                lsro_interp(cfg->interp, g, phi, q, &val);
            }
            sum += val;
        }
        star = g->dim == 2 ? sum / 2.0 : sum / 4.0;
    }
    const double c = lsro_cutoff_weight(phi_j, cfg->gamma, cfg->beta);
    return phi_j + c * (star - phi_j);
}

/* sl_step (evolve.cpp:40-118) */
int lsro_sl_step(const lsr_grid* g, const double* phi, const double* dist, const int64_t* active,
                 int64_t n_active, const lsr_step_cfg* cfg, double energy_p, double* out,
                 int64_t* bad_node, int nthreads) {
    int st = validate_cfg(cfg);
    if (st) return st;
    if (cfg->p > 1 && !(energy_p > 0.0)) return fail(LSR_ERR, "sl_step: energy must be positive for p > 1");
    const int64_t n = (int64_t)g->dims[0] * g->dims[1] * g->dims[2];
    memcpy(out, phi, sizeof(double) * (size_t)n); /* evolve.cpp:50 */
    const double grad_threshold = cfg->fallback_c * pow(cfg->dt, cfg->fallback_alpha);
    int64_t bad = INT64_MAX;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(min : bad)
#else
    (void)nthreads;
#endif
    for (int64_t a = 0; a < n_active; ++a) {
        const int64_t id = active[a];
        const double next = sl_node(g, phi, dist, id, cfg, energy_p, grad_threshold);
        if (!isfinite(next) && id < bad) bad = id;
        out[id] = next;
    }
    if (bad_node) *bad_node = bad == INT64_MAX ? -1 : bad;
    if (bad != INT64_MAX) {
        const int nx = g->dims[0], ny = g->dims[1];
        snprintf(g_msg, sizeof g_msg, "sl_step: non-finite update at node (%d, %d, %d)",
                 (int)(bad % nx), (int)((bad / nx) % ny), (int)(bad / ((int64_t)nx * ny)));
        return LSR_ERR_NUMERICAL;
    }
    return LSR_OK;
}

/* narrow_band (grid.cpp:76-124) */
int lsro_narrow_band(const lsr_grid* g, const double* phi, double gamma, uint8_t* state,
                     int64_t* active, int64_t* n_active, int64_t* tube, int64_t* n_tube) {
    if (!(gamma > 0.0)) return fail(LSR_ERR_CONFIG, "narrow_band: gamma must be positive");
    const int64_t n = (int64_t)g->dims[0] * g->dims[1] * g->dims[2];
    for (int64_t id = 0; id < n; ++id) state[id] = fabs(phi[id]) < gamma ? 1 : 0;
    const int kz = g->dim == 3 ? 1 : 0;
    for (int k = 0; k < g->dims[2]; ++k)
        for (int j = 0; j < g->dims[1]; ++j)
            for (int i = 0; i < g->dims[0]; ++i) {
                const int64_t id = gidx(g, i, j, k);
                if (state[id] != 0) continue;
                int near = 0;
                for (int dk = -kz; dk <= kz && !near; ++dk)
                    for (int dj = -1; dj <= 1 && !near; ++dj)
                        for (int di = -1; di <= 1 && !near; ++di) {
                            const int ni = i + di, nj = j + dj, nk = k + dk;
                            if (ni < 0 || nj < 0 || nk < 0 || ni >= g->dims[0] || nj >= g->dims[1] ||
                                nk >= g->dims[2])
                                continue;
                            near = state[gidx(g, ni, nj, nk)] == 1;
                        }
                if (near) state[id] = 2;
            }
    int64_t na = 0, nt = 0;
    for (int64_t id = 0; id < n; ++id) {
        if (state[id] == 1) active[na++] = id;
        if (state[id] != 0) tube[nt++] = id;
    }
    *n_active = na;
    *n_tube = nt;
    return LSR_OK;
}

/* clamp_field (grid.cpp:126-134) */
int lsro_clamp_field(const lsr_grid* g, double* f, double gamma) {
    if (!(gamma > 0.0)) return fail(LSR_ERR_CONFIG, "clamp_field: gamma must be positive");
    const int64_t n = (int64_t)g->dims[0] * g->dims[1] * g->dims[2];
    for (int64_t id = 0; id < n; ++id) f[id] = smin(smax(f[id], -gamma), gamma);
    return LSR_OK;
}
