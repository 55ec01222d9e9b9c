/*
 * oracle/difform_oracle.c — TEST INFRASTRUCTURE ONLY (see difform_oracle.h).
 *
 * fp64 restatement of the reference hot path, written from the reference's
 * published behaviour.  Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).  Layout: x-fastest
 * voxels, vector fields interleaved (AoS) with ndim components per voxel.
 */
#define _POSIX_C_SOURCE 200809L
#include "difform_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_msg[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    return code;
}

size_t orc_last_error(char* buf, size_t cap) {
    size_t n = strlen(g_msg);
    if (buf && cap) {
        size_t k = n < cap - 1 ? n : cap - 1;
        memcpy(buf, g_msg, k);
        buf[k] = 0;
    }
    return n;
}

#define CHECK(expr)              \
    do {                         \
        int rc_ = (expr);        \
        if (rc_) return rc_;     \
    } while (0)

static int64_t nvox(const dfm_grid* g) { return g->dims[0] * g->dims[1] * g->dims[2]; }

static int same_grid(const dfm_grid* a, const dfm_grid* b) {
    return a->ndim == b->ndim && a->dims[0] == b->dims[0] && a->dims[1] == b->dims[1] &&
           a->dims[2] == b->dims[2];
}

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* core.cpp:26-37 validate_meta */
int orc_validate_grid(const dfm_grid* g) {
    if (g->ndim != 2 && g->ndim != 3) return fail(1, "grid must have 2 or 3 axes");
    for (int a = 0; a < g->ndim; ++a) {
        if (g->dims[a] < 2) return fail(1, "grid dims must be >= 2 per axis");
        if (!(g->spacing[a] > 0.0) || !isfinite(g->spacing[a]))
            return fail(1, "grid spacing must be > 0");
    }
    if (g->ndim == 2 && g->dims[2] != 1) return fail(1, "2D grid must have dims[2] == 1");
    return 0;
}

/* ---------------------------------------------------------------------- */
/* trilinear sampling: interp.cpp:19-57 (locate / corner_weight / cell)    */

typedef struct {
    int64_t i0[3];
    double f[3];
    int clamped[3];
} cell_t;

static cell_t locate(const dfm_grid* m, const double p_in[3]) {
    cell_t c;
    for (int a = 0; a < 3; ++a) {
        if (a >= m->ndim || m->dims[a] == 1) {
            c.i0[a] = 0;
            c.f[a] = 0.0;
            c.clamped[a] = 0;
            continue;
        }
        double p = p_in[a];
        const double hi = (double)(m->dims[a] - 1);
        c.clamped[a] = (p < 0.0 || p > hi);
        if (p < 0.0) p = 0.0;
        if (hi < p) p = hi;
        int64_t i = (int64_t)floor(p);
        if (i < 0) i = 0;
        if (m->dims[a] - 2 < i) i = m->dims[a] - 2;
        c.i0[a] = i;
        c.f[a] = p - (double)i;
    }
    return c;
}

static double corner_w(const cell_t* c, int cx, int cy, int cz, int skip) {
    const int k[3] = {cx, cy, cz};
    double w = 1.0;
    for (int a = 0; a < 3; ++a) {
        if (a == skip) continue;
        w *= k[a] ? c->f[a] : (1.0 - c->f[a]);
    }
    return w;
}

static int64_t corner_index(const dfm_grid* m, const cell_t* c, int cx, int cy, int cz) {
    const int64_t x = c->i0[0] + (m->dims[0] > 1 ? cx : 0);
    const int64_t y = c->i0[1] + (m->dims[1] > 1 ? cy : 0);
    const int64_t z = (m->ndim == 3 && m->dims[2] > 1) ? c->i0[2] + cz : 0;
    return (z * m->dims[1] + y) * m->dims[0] + x;
}

static int nzc(const dfm_grid* m) { return (m->ndim == 3 && m->dims[2] > 1) ? 2 : 1; }

/* interp.cpp:155-164 */
static double sample_linear(const dfm_grid* m, const double* img, const double p[3]) {
    const cell_t c = locate(m, p);
    double acc = 0.0;
    for (int cz = 0; cz < nzc(m); ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx)
                acc += corner_w(&c, cx, cy, cz, -1) * img[corner_index(m, &c, cx, cy, cz)];
    return acc;
}

/* interp.cpp:166-186 */
static void sample_linear_gradient(const dfm_grid* m, const double* img, const double p[3],
                                   double g[3]) {
    const cell_t c = locate(m, p);
    g[0] = g[1] = g[2] = 0.0;
    for (int a = 0; a < m->ndim; ++a) {
        if (m->dims[a] == 1 || c.clamped[a]) continue;
        double acc = 0.0;
        for (int cz = 0; cz < nzc(m); ++cz)
            for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                    const int k[3] = {cx, cy, cz};
                    const double sgn = k[a] ? 1.0 : -1.0;
                    acc += sgn * corner_w(&c, cx, cy, cz, a) * img[corner_index(m, &c, cx, cy, cz)];
                }
        g[a] = acc;
    }
}

/* interp.cpp:188-203 */
static void sample_field(const dfm_grid* m, const double* f, const double p[3], double out[3]) {
    const cell_t c = locate(m, p);
    const int d = m->ndim;
    out[0] = out[1] = out[2] = 0.0;
    for (int cz = 0; cz < nzc(m); ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx) {
                const double w = corner_w(&c, cx, cy, cz, -1);
                const int64_t j = corner_index(m, &c, cx, cy, cz);
                for (int k = 0; k < d; ++k) out[k] += w * f[j * d + k];
            }
}

static void voxel_xyz(const dfm_grid* m, int64_t i, double p[3]) {
    p[0] = (double)(i % m->dims[0]);
    p[1] = (double)((i / m->dims[0]) % m->dims[1]);
    p[2] = (double)(i / (m->dims[0] * m->dims[1]));
}

int orc_sample_linear_points(const dfm_grid* g, const double* img, int64_t npts,
                             const double* pts, double* values, double* grads) {
    CHECK(orc_validate_grid(g));
    for (int64_t i = 0; i < npts; ++i) {
        values[i] = sample_linear(g, img, pts + 3 * i);
        if (grads) sample_linear_gradient(g, img, pts + 3 * i, grads + 3 * i);
    }
    return 0;
}

/* interp.cpp:229-246 */
int orc_warp_image(const dfm_grid* g, const double* img, const double* phi, double* out) {
    CHECK(orc_validate_grid(g));
    const int64_t n = nvox(g);
    for (int64_t i = 0; i < n; ++i) {
        double p[3];
        voxel_xyz(g, i, p);
        for (int c = 0; c < g->ndim; ++c) p[c] += phi[i * g->ndim + c];
        out[i] = sample_linear(g, img, p);
    }
    return 0;
}

/* interp.cpp:248-267 (llround = round half away from zero, then clamp) */
int orc_warp_labels(const dfm_grid* g, const int32_t* labels, const double* phi, int32_t* out) {
    CHECK(orc_validate_grid(g));
    const int64_t n = nvox(g);
    for (int64_t i = 0; i < n; ++i) {
        double p[3];
        int64_t q[3];
        voxel_xyz(g, i, p);
        for (int c = 0; c < 3; ++c) q[c] = (int64_t)p[c];
        for (int c = 0; c < g->ndim; ++c) {
            int64_t r = llround((double)q[c] + phi[i * g->ndim + c]);
            if (r < 0) r = 0;
            if (r > g->dims[c] - 1) r = g->dims[c] - 1;
            q[c] = r;
        }
        out[i] = labels[(q[2] * g->dims[1] + q[1]) * g->dims[0] + q[0]];
    }
    return 0;
}

/* interp.cpp:269-289 */
static void compose_raw(const dfm_grid* g, const double* phi, const double* psi, double* out) {
    const int64_t n = nvox(g);
    const int d = g->ndim;
    for (int64_t i = 0; i < n; ++i) {
        double p[3], up[3];
        voxel_xyz(g, i, p);
        for (int c = 0; c < d; ++c) p[c] += psi[i * d + c];
        sample_field(g, phi, p, up);
        for (int c = 0; c < d; ++c) out[i * d + c] = psi[i * d + c] + up[c];
    }
}

int orc_compose(const dfm_grid* g, const double* phi, const double* psi, double* out) {
    CHECK(orc_validate_grid(g));
    compose_raw(g, phi, psi, out);
    return 0;
}

/* ---------------------------------------------------------------------- */
/* SVF: diffeo.cpp:66-167                                                   */

/* diffeo.cpp:66-77: u = v / 2^M, then M self-compositions */
static void exp_map_raw(const dfm_grid* g, const double* v, int M, double* u, double* tmp) {
    const int64_t nd = nvox(g) * g->ndim;
    const double scale = ldexp(1.0, -M);
    for (int64_t i = 0; i < nd; ++i) u[i] = v[i] * scale;
    for (int k = 0; k < M; ++k) {
        compose_raw(g, u, u, tmp);
        memcpy(u, tmp, (size_t)nd * sizeof(double));
    }
}

int orc_exp_map(const dfm_grid* g, const double* v, int M, double* out) {
    if (M < 0) return fail(1, "exp_map: M must be >= 0");
    CHECK(orc_validate_grid(g));
    double* tmp = dalloc(nvox(g) * g->ndim);
    exp_map_raw(g, v, M, out, tmp);
    free(tmp);
    return 0;
}

/* interp.cpp:205-227 sample_field_jacobian: J[comp][a] over the cell corners
 * in (cz, cy, cx) order, zero on flat or clamped axes */
static void sample_field_jacobian(const dfm_grid* m, const double* f, const double p[3],
                                  double J[3][3]) {
    const cell_t c = locate(m, p);
    const int d = m->ndim;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) J[a][b] = 0.0;
    for (int a = 0; a < d; ++a) {
        if (m->dims[a] == 1 || c.clamped[a]) continue;
        for (int cz = 0; cz < nzc(m); ++cz)
            for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                    const int k[3] = {cx, cy, cz};
                    const double sgn = k[a] ? 1.0 : -1.0;
                    const double w = sgn * corner_w(&c, cx, cy, cz, a);
                    const int64_t j = corner_index(m, &c, cx, cy, cz);
                    for (int comp = 0; comp < d; ++comp) J[comp][a] += w * f[j * d + comp];
                }
    }
}

/* diffeo.cpp:79-167: discrete adjoint of exp_map.  Per level (reverse order):
 * wn = w + J(u_k)(x+u_k)^T w (voxel-parallel in the reference), then the
 * serial scatter of the lerp weights of every voxel's sample onto its cell
 * corners, in voxel order; finally w * 2^-M. */
int orc_svf_pullback(const dfm_grid* g, const double* v, const double* grad_phi, int M,
                     double* out) {
    if (M < 0) return fail(1, "svf_pullback: M must be >= 0");
    CHECK(orc_validate_grid(g));
    const int d = g->ndim;
    const int64_t n = nvox(g), nd = n * d;
    const double scale = ldexp(1.0, -M);
    double* levels = dalloc(nd * (M + 1));
    for (int64_t i = 0; i < nd; ++i) levels[i] = v[i] * scale;
    for (int k = 0; k < M; ++k) compose_raw(g, levels + k * nd, levels + k * nd, levels + (k + 1) * nd);
    double* w = dalloc(nd);
    double* wn = dalloc(nd);
    double* pts = dalloc(n * 3);
    memcpy(w, grad_phi, (size_t)nd * sizeof(double));
    const int nz = (d == 3) ? 2 : 1;
    for (int k = M - 1; k >= 0; --k) {
        const double* uk = levels + k * nd;
        memcpy(wn, w, (size_t)nd * sizeof(double));
        for (int64_t i = 0; i < n; ++i) {
            double* p = pts + 3 * i;
            voxel_xyz(g, i, p);
            for (int c = 0; c < d; ++c) p[c] += uk[i * d + c];
            double J[3][3];
            sample_field_jacobian(g, uk, p, J);
            const double* wi = w + i * d;
            double* wo = wn + i * d;
            for (int a = 0; a < d; ++a) {
                double acc = 0.0;
                for (int comp = 0; comp < d; ++comp) acc += J[comp][a] * wi[comp];
                wo[a] += acc;
            }
        }
        for (int64_t i = 0; i < n; ++i) {
            const double* p = pts + 3 * i;
            int64_t i0[3] = {0, 0, 0};
            double f[3] = {0.0, 0.0, 0.0};
            for (int a = 0; a < 3; ++a) {
                if (a >= d || g->dims[a] == 1) continue;
                double pc = p[a];
                const double hi = (double)(g->dims[a] - 1);
                if (pc < 0.0) pc = 0.0;
                if (hi < pc) pc = hi;
                int64_t q = (int64_t)floor(pc);
                if (q < 0) q = 0;
                if (g->dims[a] - 2 < q) q = g->dims[a] - 2;
                i0[a] = q;
                f[a] = pc - (double)q;
            }
            const double* wi = w + i * d;
            for (int cz = 0; cz < nz; ++cz)
                for (int cy = 0; cy < 2; ++cy)
                    for (int cx = 0; cx < 2; ++cx) {
                        const double wt = (cx ? f[0] : 1.0 - f[0]) * (cy ? f[1] : 1.0 - f[1]) *
                                          ((nz == 2) ? (cz ? f[2] : 1.0 - f[2]) : 1.0);
                        if (wt == 0.0) continue;
                        const int64_t zz = (nz == 2) ? i0[2] + cz : 0;
                        const int64_t idx = (zz * g->dims[1] + (i0[1] + cy)) * g->dims[0] + i0[0] + cx;
                        for (int c = 0; c < d; ++c) wn[idx * d + c] += wt * wi[c];
                    }
        }
        memcpy(w, wn, (size_t)nd * sizeof(double));
    }
    for (int64_t i = 0; i < nd; ++i) out[i] = w[i] * scale;
    free(levels);
    free(w);
    free(wn);
    free(pts);
    return 0;
}

/* interp.cpp:291-328: J = I + central differences (one-sided at borders),
 * row = component, column = axis. */
static void jacobian_at(const dfm_grid* m, const double* phi, int64_t i, double J[9]) {
    const int d = m->ndim;
    const int64_t pos[3] = {i % m->dims[0], (i / m->dims[0]) % m->dims[1],
                            i / (m->dims[0] * m->dims[1])};
    for (int k = 0; k < 9; ++k) J[k] = 0.0;
    for (int a = 0; a < d; ++a) {
        int64_t lo[3] = {pos[0], pos[1], pos[2]}, hi[3] = {pos[0], pos[1], pos[2]};
        double den;
        if (pos[a] == 0) {
            hi[a] = 1;
            den = 1.0;
        } else if (pos[a] == m->dims[a] - 1) {
            lo[a] = m->dims[a] - 2;
            den = 1.0;
        } else {
            lo[a] = pos[a] - 1;
            hi[a] = pos[a] + 1;
            den = 2.0;
        }
        const int64_t jl = (lo[2] * m->dims[1] + lo[1]) * m->dims[0] + lo[0];
        const int64_t jh = (hi[2] * m->dims[1] + hi[1]) * m->dims[0] + hi[0];
        for (int c = 0; c < d; ++c)
            J[c * d + a] = (phi[jh * d + c] - phi[jl * d + c]) / den + (c == a ? 1.0 : 0.0);
    }
}

/* interp.cpp:330-349 */
static double det_of(const double* j, int d) {
    if (d == 2) return j[0] * j[3] - j[1] * j[2];
    return j[0] * (j[4] * j[8] - j[5] * j[7]) - j[1] * (j[3] * j[8] - j[5] * j[6]) +
           j[2] * (j[3] * j[7] - j[4] * j[6]);
}

int orc_jacobian_det(const dfm_grid* g, const double* phi, double* out) {
    CHECK(orc_validate_grid(g));
    const int64_t n = nvox(g);
    for (int64_t i = 0; i < n; ++i) {
        double J[9];
        jacobian_at(g, phi, i, J);
        out[i] = det_of(J, g->ndim);
    }
    return 0;
}

/* analysis.cpp:160-167 */
int orc_singularity_fraction(const dfm_grid* g, const double* phi, double* frac) {
    CHECK(orc_validate_grid(g));
    const int64_t n = nvox(g);
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        double J[9];
        jacobian_at(g, phi, i, J);
        if (det_of(J, g->ndim) <= 0.0) ++bad;
    }
    *frac = (double)bad / (double)n;
    return 0;
}

/* ---------------------------------------------------------------------- */
/* separable filters                                                        */

/* interp.cpp:110-151: truncated Gaussian along one axis of an interleaved
 * buffer with `comps` components; taps renormalised over the in-range part. */
static void smooth_axis(double* data, const dfm_grid* m, int comps, int axis, double sigma) {
    if (sigma <= 0.0 || m->dims[axis] == 1) return;
    const int64_t R = (int64_t)ceil(3.0 * sigma);
    double* taps = dalloc(2 * R + 1);
    double tsum = 0.0;
    for (int64_t j = -R; j <= R; ++j) {
        const double q = (double)j / sigma;
        taps[j + R] = exp(-0.5 * q * q);
        tsum += taps[j + R];
    }
    for (int64_t j = 0; j < 2 * R + 1; ++j) taps[j] /= tsum;
    const int64_t n = m->dims[axis];
    int64_t stride = comps;
    for (int a = 0; a < axis; ++a) stride *= m->dims[a];
    const int64_t total = nvox(m) * comps;
    const int64_t lines = total / n;
    double* out = dalloc(total);
    for (int64_t line = 0; line < lines; ++line) {
        const int64_t start = (line / stride) * stride * n + line % stride;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t jlo = (-R > -i) ? -R : -i;
            const int64_t jhi = (R < n - 1 - i) ? R : n - 1 - i;
            double acc = 0.0, ws = 0.0;
            for (int64_t j = jlo; j <= jhi; ++j) {
                acc += taps[j + R] * data[start + (i + j) * stride];
                ws += taps[j + R];
            }
            out[start + i * stride] = acc / ws;
        }
    }
    memcpy(data, out, (size_t)total * sizeof(double));
    free(out);
    free(taps);
}

static int smooth_generic(const dfm_grid* g, const double* in, int comps, const double sigma[3],
                          double* out, const char* what) {
    CHECK(orc_validate_grid(g));
    for (int a = 0; a < g->ndim; ++a)
        if (sigma[a] < 0.0) return fail(1, "%s: sigma must be >= 0", what);
    memmove(out, in, (size_t)(nvox(g) * comps) * sizeof(double));
    for (int a = 0; a < g->ndim; ++a) smooth_axis(out, g, comps, a, sigma[a]);
    return 0;
}

/* interp.cpp:351-360 */
int orc_gaussian_smooth(const dfm_grid* g, const double* img, const double sigma[3], double* out) {
    return smooth_generic(g, img, 1, sigma, out, "gaussian_smooth");
}

/* interp.cpp:362-371 */
int orc_gaussian_smooth_field(const dfm_grid* g, const double* f, const double sigma[3],
                              double* out) {
    return smooth_generic(g, f, g->ndim, sigma, out, "gaussian_smooth_field");
}

/* similarity.cpp:48-77: clipped box sum [i-r, i+r] along every active axis */
static void box_sum(double* v, const dfm_grid* m, int r) {
    const int64_t total = nvox(m);
    double* out = dalloc(total);
    for (int axis = 0; axis < m->ndim; ++axis) {
        const int64_t n = m->dims[axis];
        int64_t stride = 1;
        for (int a = 0; a < axis; ++a) stride *= m->dims[a];
        const int64_t lines = total / n;
        for (int64_t line = 0; line < lines; ++line) {
            const int64_t start = (line / stride) * stride * n + line % stride;
            for (int64_t i = 0; i < n; ++i) {
                const int64_t jlo = i - r > 0 ? i - r : 0;
                const int64_t jhi = i + r < n - 1 ? i + r : n - 1;
                double acc = 0.0;
                for (int64_t j = jlo; j <= jhi; ++j) acc += v[start + j * stride];
                out[start + i * stride] = acc;
            }
        }
        memcpy(v, out, (size_t)total * sizeof(double));
    }
    free(out);
}

/* parallel.cpp:153-169: partial sums over fixed 4096-element blocks, then the
 * partials summed in block order. */
static double block_sum(const double* t, int64_t n) {
    double total = 0.0;
    for (int64_t lo = 0; lo < n; lo += 4096) {
        const int64_t hi = lo + 4096 < n ? lo + 4096 : n;
        double acc = 0.0;
        for (int64_t i = lo; i < hi; ++i) acc += t[i];
        total += acc;
    }
    return total;
}

/* ---------------------------------------------------------------------- */
/* similarity losses                                                        */

static int check_loss(const dfm_grid* fg, const dfm_grid* mg, const char* what) {
    CHECK(orc_validate_grid(fg));
    CHECK(orc_validate_grid(mg));
    if (fg->ndim != mg->ndim) return fail(1, "%s: dimensionality mismatch", what);
    return 0;
}

/* similarity.cpp:25-45: W = M(x+u), G = grad of the interpolant there */
static void warp_with_gradient(const dfm_grid* fg, const dfm_grid* mg, const double* moving,
                               const double* phi, double* W, double* G) {
    const int64_t n = nvox(fg);
    const int d = fg->ndim;
    for (int64_t i = 0; i < n; ++i) {
        double p[3], gr[3];
        voxel_xyz(fg, i, p);
        for (int c = 0; c < d; ++c) p[c] += phi[i * d + c];
        W[i] = sample_linear(mg, moving, p);
        sample_linear_gradient(mg, moving, p, gr);
        for (int c = 0; c < d; ++c) G[i * d + c] = gr[c];
    }
}

/* similarity.cpp:81-104 (gradient omits the factor 2) */
int orc_ssd_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                 const double* moving, const double* phi, double* value, double* grad) {
    CHECK(check_loss(fg, mg, "ssd_eval"));
    const int64_t n = nvox(fg);
    const int d = fg->ndim;
    double* W = dalloc(n);
    double* G = dalloc(n * d);
    double* t = dalloc(n);
    warp_with_gradient(fg, mg, moving, phi, W, G);
    for (int64_t i = 0; i < n; ++i) {
        const double r = fixed[i] - W[i];
        t[i] = r * r;
    }
    *value = block_sum(t, n) / (double)n;
    if (grad)
        for (int64_t i = 0; i < n; ++i) {
            const double r = W[i] - fixed[i];
            for (int c = 0; c < d; ++c) grad[i * d + c] = r * G[i * d + c] / (double)n;
        }
    free(W);
    free(G);
    free(t);
    return 0;
}

/* similarity.cpp:106-190 */
int orc_lncc_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                  const double* moving, const double* phi, int r, double* value, double* grad) {
    CHECK(check_loss(fg, mg, "lncc_eval"));
    if (r < 1) return fail(1, "lncc_eval: window_radius must be >= 1");
    for (int a = 0; a < fg->ndim; ++a)
        if (2 * (int64_t)r + 1 > fg->dims[a]) return fail(1, "lncc_eval: window larger than image");
    const int64_t n = nvox(fg);
    const int d = fg->ndim;
    double* W = dalloc(n);
    double* G = dalloc(n * d);
    warp_with_gradient(fg, mg, moving, phi, W, G);
    /* moments: cnt, F, W, F^2, W^2, FW */
    double* mom[6];
    for (int k = 0; k < 6; ++k) mom[k] = dalloc(n);
    for (int64_t i = 0; i < n; ++i) {
        mom[0][i] = 1.0;
        mom[1][i] = fixed[i];
        mom[2][i] = W[i];
        mom[3][i] = fixed[i] * fixed[i];
        mom[4][i] = W[i] * W[i];
        mom[5][i] = fixed[i] * W[i];
    }
    for (int k = 0; k < 6; ++k) box_sum(mom[k], fg, r);
    double* cf[4];
    for (int k = 0; k < 4; ++k) cf[k] = dalloc(n);
    double* cc2 = dalloc(n);
    for (int64_t i = 0; i < n; ++i) {
        const double cnt = mom[0][i];
        const double muF = mom[1][i] / cnt;
        const double muW = mom[2][i] / cnt;
        double vF = mom[3][i] / cnt - muF * muF;
        double vW = mom[4][i] / cnt - muW * muW;
        if (vF < 0.0) vF = 0.0;
        if (vW < 0.0) vW = 0.0;
        const double cv = mom[5][i] / cnt - muF * muW;
        if (vF < 1e-5 || vW < 1e-5) { /* similarity.cpp:13 variance floor */
            cc2[i] = cf[0][i] = cf[1][i] = cf[2][i] = cf[3][i] = 0.0;
            continue;
        }
        const double cc = cv / sqrt(vF * vW);
        cc2[i] = cc * cc;
        const double alpha = cv / (vF * vW);
        const double beta = cv * cv / (vF * vW * vW);
        cf[0][i] = alpha / cnt;
        cf[1][i] = alpha * muF / cnt;
        cf[2][i] = beta / cnt;
        cf[3][i] = beta * muW / cnt;
    }
    *value = -block_sum(cc2, n) / (double)n;
    if (grad) {
        for (int k = 0; k < 4; ++k) box_sum(cf[k], fg, r);
        for (int64_t i = 0; i < n; ++i) {
            const double dW =
                -2.0 / (double)n * (fixed[i] * cf[0][i] - cf[1][i] - W[i] * cf[2][i] + cf[3][i]);
            for (int c = 0; c < d; ++c) grad[i * d + c] = dW * G[i * d + c];
        }
    }
    for (int k = 0; k < 6; ++k) free(mom[k]);
    for (int k = 0; k < 4; ++k) free(cf[k]);
    free(cc2);
    free(W);
    free(G);
    return 0;
}

/* similarity.cpp:192-231 */
int orc_dice_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                  const double* moving, const double* phi, double* value, double* grad) {
    CHECK(check_loss(fg, mg, "dice_soft_eval"));
    for (int64_t i = 0; i < nvox(fg); ++i)
        if (!(fixed[i] >= 0.0 && fixed[i] <= 1.0))
            return fail(1, "dice_soft_eval: fixed mask values outside [0,1]");
    for (int64_t i = 0; i < nvox(mg); ++i)
        if (!(moving[i] >= 0.0 && moving[i] <= 1.0))
            return fail(1, "dice_soft_eval: moving mask values outside [0,1]");
    const int64_t n = nvox(fg);
    const int d = fg->ndim;
    double* W = dalloc(n);
    double* G = dalloc(n * d);
    double* t = dalloc(n);
    warp_with_gradient(fg, mg, moving, phi, W, G);
    for (int64_t i = 0; i < n; ++i) t[i] = fixed[i] * W[i];
    const double P = block_sum(t, n);
    const double SF = block_sum(fixed, n);
    const double SM = block_sum(W, n);
    const double D = SF + SM + 1e-7;
    *value = 1.0 - 2.0 * P / D;
    if (grad)
        for (int64_t i = 0; i < n; ++i) {
            const double dW = -2.0 * fixed[i] / D + 2.0 * P / (D * D);
            for (int c = 0; c < d; ++c) grad[i * d + c] = dW * G[i * d + c];
        }
    free(W);
    free(G);
    free(t);
    return 0;
}

/* ---------------------------------------------------------------------- */
/* optimiser                                                                */

/* optim.cpp:22-42 */
int orc_adam_step(const dfm_grid* g, double* m, double* nu, int64_t* t, double b1, double b2,
                  double eps, const double* v, double* dir) {
    CHECK(orc_validate_grid(g));
    *t += 1;
    const double c1 = 1.0 - pow(b1, (double)*t);
    const double c2 = 1.0 - pow(b2, (double)*t);
    const int64_t n = nvox(g) * g->ndim;
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * v[i];
        nu[i] = b2 * nu[i] + (1.0 - b2) * v[i] * v[i];
        const double mh = m[i] / c1;
        const double nh = nu[i] / c2;
        dir[i] = mh / (sqrt(nh) + eps);
    }
    return 0;
}

/* interp.cpp:381-406; `rescale` (per axis) applied when non-NULL */
static void resample_linear_raw(const dfm_grid* g, const double* f, const dfm_grid* ng,
                                const double* rescale, double* out) {
    double step[3] = {0.0, 0.0, 0.0};
    const int d = ng->ndim;
    for (int a = 0; a < d; ++a)
        step[a] = ng->dims[a] > 1 ? (double)(g->dims[a] - 1) / (double)(ng->dims[a] - 1) : 0.0;
    const int64_t n = nvox(ng);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t x = i % ng->dims[0];
        const int64_t y = (i / ng->dims[0]) % ng->dims[1];
        const int64_t z = i / (ng->dims[0] * ng->dims[1]);
        const double p[3] = {x * step[0], y * step[1], z * step[2]};
        double v[3];
        sample_field(g, f, p, v);
        for (int c = 0; c < d; ++c) out[i * d + c] = rescale ? v[c] * rescale[c] : v[c];
    }
}

static int dims_equal(const dfm_grid* a, const dfm_grid* b) {
    return a->dims[0] == b->dims[0] && a->dims[1] == b->dims[1] && a->dims[2] == b->dims[2];
}

int orc_resample_field_linear(const dfm_grid* g, const double* f, const dfm_grid* ng,
                              double* out) {
    CHECK(orc_validate_grid(g));
    CHECK(orc_validate_grid(ng));
    if (ng->ndim != g->ndim) return fail(1, "resample_field_linear: dimensionality mismatch");
    if (dims_equal(g, ng)) {
        memmove(out, f, (size_t)(nvox(g) * g->ndim) * sizeof(double));
        return 0;
    }
    resample_linear_raw(g, f, ng, NULL, out);
    return 0;
}

static void displacement_rescale(const dfm_grid* g, const dfm_grid* ng, double r[3]) {
    r[0] = r[1] = r[2] = 1.0;
    for (int a = 0; a < ng->ndim; ++a)
        r[a] = (double)(ng->dims[a] - 1) / (double)(g->dims[a] - 1);
}

/* interp.cpp:408-445 (linear method) */
int orc_upsample_field(const dfm_grid* g, const double* phi, const dfm_grid* ng, double* out) {
    CHECK(orc_validate_grid(g));
    CHECK(orc_validate_grid(ng));
    if (ng->ndim != g->ndim) return fail(1, "upsample_field: dimensionality mismatch");
    for (int a = 0; a < g->ndim; ++a)
        if (ng->dims[a] < g->dims[a]) return fail(1, "upsample_field: shrinking not allowed");
    if (dims_equal(g, ng)) {
        memmove(out, phi, (size_t)(nvox(g) * g->ndim) * sizeof(double));
        return 0;
    }
    double r[3];
    displacement_rescale(g, ng, r);
    resample_linear_raw(g, phi, ng, r, out);
    return 0;
}

/* interp.cpp:447-465: resample then multiply (two roundings, as the reference) */
int orc_resample_displacement(const dfm_grid* g, const double* phi, const dfm_grid* ng,
                              double* out) {
    CHECK(orc_validate_grid(g));
    CHECK(orc_validate_grid(ng));
    if (ng->ndim != g->ndim) return fail(1, "resample_displacement: dimensionality mismatch");
    if (dims_equal(g, ng)) {
        memmove(out, phi, (size_t)(nvox(g) * g->ndim) * sizeof(double));
        return 0;
    }
    resample_linear_raw(g, phi, ng, NULL, out);
    double r[3];
    displacement_rescale(g, ng, r);
    for (int64_t i = 0; i < nvox(ng); ++i)
        for (int c = 0; c < ng->ndim; ++c) out[i * ng->ndim + c] *= r[c];
    return 0;
}

/* optim.cpp:59-85 */
int orc_upsample_state(const dfm_grid* g, const double* m, const double* nu, const dfm_grid* ng,
                       double* m_out, double* nu_out) {
    CHECK(orc_validate_grid(ng));
    for (int a = 0; a < ng->ndim; ++a)
        if (ng->dims[a] < g->dims[a]) return fail(1, "upsample_state: shrinking not allowed");
    CHECK(orc_upsample_field(g, m, ng, m_out));
    CHECK(orc_resample_field_linear(g, nu, ng, nu_out));
    double sq[3] = {1.0, 1.0, 1.0};
    for (int a = 0; a < ng->ndim; ++a) {
        const double r = (double)(ng->dims[a] - 1) / (double)(g->dims[a] - 1);
        sq[a] = r * r;
    }
    for (int64_t i = 0; i < nvox(ng); ++i)
        for (int c = 0; c < ng->ndim; ++c) nu_out[i * ng->ndim + c] *= sq[c];
    return 0;
}

/* ---------------------------------------------------------------------- */
/* group update                                                             */

/* diffeo.cpp:11-40 */
int orc_eulerian_direction(const dfm_grid* g, const double* grad, const double* phi,
                           int use_jac, double* out) {
    CHECK(orc_validate_grid(g));
    const int d = g->ndim;
    const int64_t n = nvox(g);
    if (!use_jac) {
        for (int64_t i = 0; i < n * d; ++i) out[i] = -grad[i];
        return 0;
    }
    for (int64_t i = 0; i < n; ++i) {
        double J[9];
        jacobian_at(g, phi, i, J);
        for (int a = 0; a < d; ++a) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += J[c * d + a] * grad[i * d + c];
            out[i * d + a] = -acc;
        }
    }
    return 0;
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* diffeo.cpp:42-64 */
int orc_apply_update(const dfm_grid* g, const double* phi, const double* v, double eta,
                     double sigma_warp, double cap, double* out) {
    CHECK(orc_validate_grid(g));
    const int d = g->ndim;
    const int64_t n = nvox(g) * d;
    double* step = dalloc(n);
    int bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double s = eta * v[i];
        if (!isfinite(s)) bad = 1;
        step[i] = clampd(s, -cap, cap);
    }
    if (bad) {
        free(step);
        return fail(2, "apply_update: non-finite step");
    }
    compose_raw(g, phi, step, out);
    free(step);
    if (sigma_warp > 0.0) {
        const double s3[3] = {sigma_warp, sigma_warp, sigma_warp};
        for (int a = 0; a < d; ++a) smooth_axis(out, g, d, a, s3[a]);
    }
    return 0;
}

/* ---------------------------------------------------------------------- */
/* pyramid                                                                  */

/* core.cpp:58-74 (output grid) */
int orc_downsample_grid(const dfm_grid* g, const double factor[3], dfm_grid* out) {
    CHECK(orc_validate_grid(g));
    *out = *g;
    for (int a = 0; a < g->ndim; ++a) {
        if (!(factor[a] >= 1.0)) return fail(1, "downsample factor must be >= 1");
        out->dims[a] = (int64_t)ceil((double)g->dims[a] / factor[a]);
        if (out->dims[a] < 2) return fail(1, "downsample would leave < 2 samples on an axis");
        out->spacing[a] = g->spacing[a] * ((double)g->dims[a] / (double)out->dims[a]);
    }
    return 0;
}

/* core.cpp:58-96 */
int orc_downsample_image(const dfm_grid* g, const double* img, const double factor[3],
                         dfm_grid* og, double* out) {
    CHECK(orc_downsample_grid(g, factor, og));
    double sigma[3] = {0.0, 0.0, 0.0};
    int any_blur = 0;
    for (int a = 0; a < g->ndim; ++a)
        if (factor[a] > 1.0) {
            sigma[a] = factor[a] / 2.0;
            any_blur = 1;
        }
    const int64_t n = nvox(g);
    if (dims_equal(g, og) && !any_blur) {
        memmove(out, img, (size_t)n * sizeof(double));
        return 0;
    }
    double* blurred = dalloc(n);
    memcpy(blurred, img, (size_t)n * sizeof(double));
    if (any_blur)
        for (int a = 0; a < g->ndim; ++a) smooth_axis(blurred, g, 1, a, sigma[a]);
    double step[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < g->ndim; ++a)
        step[a] = (double)(g->dims[a] - 1) / (double)(og->dims[a] - 1);
    for (int64_t z = 0; z < og->dims[2]; ++z)
        for (int64_t y = 0; y < og->dims[1]; ++y)
            for (int64_t x = 0; x < og->dims[0]; ++x) {
                const double p[3] = {x * step[0], y * step[1], z * step[2]};
                out[(z * og->dims[1] + y) * og->dims[0] + x] = sample_linear(g, blurred, p);
            }
    free(blurred);
    return 0;
}

/* ---------------------------------------------------------------------- */
/* driver: register_images, direct mode (pipeline.cpp:121-224)              */

/* pipeline.cpp:83-96 */
static int validate_schedule(const double* scales, const int32_t* iters, int32_t ns) {
    if (ns < 1) return fail(1, "schedule: at least one scale required");
    for (int i = 0; i < ns; ++i) {
        if (!(scales[i] >= 1.0) || !isfinite(scales[i]))
            return fail(1, "schedule: scales must be finite and >= 1");
        if (i > 0 && !(scales[i] < scales[i - 1]))
            return fail(1, "schedule: scales must be strictly decreasing");
        if (iters[i] < 0) return fail(1, "schedule: iterations must be >= 0");
    }
    return 0;
}

/* pipeline.cpp:98-119 */
static int validate_config(const dfm_config* c) {
    if (!(c->eta > 0.0) || !isfinite(c->eta)) return fail(1, "config: eta must be positive and finite");
    if (c->sigma_grad < 0.0 || c->sigma_warp < 0.0) return fail(1, "config: sigmas must be >= 0");
    if (c->lncc_radius < 1) return fail(1, "config: lncc_radius must be >= 1");
    if (c->svf_M < 0) return fail(1, "config: svf_M must be >= 0");
    if (!(c->beta1 >= 0.0 && c->beta1 < 1.0) || !(c->beta2 >= 0.0 && c->beta2 < 1.0))
        return fail(1, "config: betas must lie in [0, 1)");
    if (!(c->eps_adam > 0.0)) return fail(1, "config: eps_adam must be positive");
    if (!(c->step_cap > 0.0)) return fail(1, "config: step_cap must be positive");
    if (c->conv_window < 1) return fail(1, "config: conv_window must be >= 1");
    if (c->conv_tol < 0.0) return fail(1, "config: conv_tol must be >= 0");
    if (c->mode == DFM_MODE_SVF && c->loss == DFM_LOSS_DICE)
        return fail(1, "config: dice loss is not available in svf mode");
    if (c->mode != DFM_MODE_DIRECT && c->mode != DFM_MODE_SVF) return fail(1, "config: unknown mode");
    return 0;
}

/* pipeline.cpp:45-53 */
static int converged(const double* L, int64_t n, int w, double tol) {
    if (n < (int64_t)w + 1) return 0;
    const double prev = L[n - 1 - w];
    const double cur = L[n - 1];
    const double den = fabs(prev) > 1e-30 ? fabs(prev) : 1e-30;
    const double rel = ((prev - cur) / w) / den;
    return rel < tol;
}

static int eval_loss(const dfm_grid* g, const double* f, const double* mv, const double* phi,
                     const dfm_config* c, double* value, double* grad) {
    switch (c->loss) {
        case DFM_LOSS_SSD: return orc_ssd_eval(g, f, g, mv, phi, value, grad);
        case DFM_LOSS_LNCC: return orc_lncc_eval(g, f, g, mv, phi, c->lncc_radius, value, grad);
        case DFM_LOSS_DICE: return orc_dice_eval(g, f, g, mv, phi, value, grad);
    }
    return fail(1, "unknown loss");
}

/* affine.cpp:26-48 working_field: u(x) = S^-1 (A S x + t) - x */
static void affine_working_field(const dfm_init* T, const dfm_grid* m, const double S[3],
                                 double* u) {
    const int d = m->ndim;
    for (int64_t i = 0; i < nvox(m); ++i) {
        double xw[3];
        voxel_xyz(m, i, xw);
        for (int r = 0; r < d; ++r) {
            double acc = T->t[r];
            for (int c = 0; c < d; ++c) acc += T->A[r * d + c] * S[c] * xw[c];
            u[i * d + r] = acc / S[r] - xw[r];
        }
    }
}

/* pipeline.cpp:57-79 */
static int initial_field(const dfm_init* init, const dfm_grid* work, const dfm_grid* full,
                         double* u) {
    const int64_t n = nvox(work) * work->ndim;
    if (!init || init->kind == DFM_INIT_NONE) {
        memset(u, 0, (size_t)n * sizeof(double));
        return 0;
    }
    if (init->kind == DFM_INIT_AFFINE) {
        double S[3] = {1.0, 1.0, 1.0};
        for (int a = 0; a < work->ndim; ++a) {
            const int64_t den = work->dims[a] - 1 > 1 ? work->dims[a] - 1 : 1;
            S[a] = (double)(full->dims[a] - 1) / (double)den;
        }
        if (init->affine_ndim != work->ndim)
            return fail(1, "affine_to_working_field: dimensionality mismatch");
        affine_working_field(init, work, S, u);
        return 0;
    }
    const dfm_grid* fg = &init->field_grid;
    if (fg->ndim != work->ndim)
        return fail(1, "register_images: init field dimensionality mismatch");
    if (dims_equal(fg, work)) {
        memcpy(u, init->field, (size_t)n * sizeof(double));
        return 0;
    }
    if (dims_equal(fg, full)) return orc_resample_displacement(fg, init->field, work, u);
    return fail(1, "register_images: init field must live on the full or coarsest grid");
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

int orc_register(const dfm_grid* g, const double* fixed, const double* moving,
                 const dfm_config* cfg, const double* scales, const int32_t* iters,
                 int32_t nscales, const dfm_init* init, double* out_field,
                 dfm_iter_record* records, int64_t max_records, dfm_runlog* log) {
    CHECK(orc_validate_grid(g));
    CHECK(validate_config(cfg));
    CHECK(validate_schedule(scales, iters, nscales));
    const double t0 = now_ms();
    const int d = g->ndim;
    const int64_t nfull = nvox(g);
    int rc = 0;
    /* buffers sized for the full grid, reused at every scale */
    double* f = dalloc(nfull);
    double* mv = dalloc(nfull);
    double* u = dalloc(nfull * d);
    double* m = dalloc(nfull * d);
    double* nu = dalloc(nfull * d);
    double* tmp = dalloc(nfull * d);
    double* tmp2 = dalloc(nfull * d);
    double* grad = dalloc(nfull * d);
    double* phis = dalloc(nfull * d); /* exp(v) in svf mode */
    int64_t total_iters = 0;
    for (int i = 0; i < nscales; ++i) total_iters += iters[i];
    double* losses = dalloc(total_iters + 1);
    dfm_grid cur;
    int have = 0;
    int64_t t_adam = 0, global = 0, nrec = 0;

    for (int si = 0; si < nscales && !rc; ++si) {
        const double fac[3] = {scales[si], scales[si], scales[si]};
        dfm_grid wg;
        if ((rc = orc_downsample_image(g, fixed, fac, &wg, f))) break;
        if ((rc = orc_downsample_image(g, moving, fac, &wg, mv))) break;
        const int64_t n = nvox(&wg);
        if (!have) {
            if ((rc = initial_field(init, &wg, g, u))) break;
            memset(m, 0, (size_t)(n * d) * sizeof(double));
            memset(nu, 0, (size_t)(n * d) * sizeof(double));
            have = 1;
        } else if (!dims_equal(&cur, &wg)) {
            if ((rc = orc_upsample_field(&cur, u, &wg, tmp))) break;
            memcpy(u, tmp, (size_t)(n * d) * sizeof(double));
            if ((rc = orc_upsample_state(&cur, m, nu, &wg, tmp, tmp2))) break;
            memcpy(m, tmp, (size_t)(n * d) * sizeof(double));
            memcpy(nu, tmp2, (size_t)(n * d) * sizeof(double));
        }
        cur = wg;
        int64_t nl = 0;
        for (int it = 0; it < iters[si]; ++it) {
            const double t_it = now_ms();
            double value;
            const double* phi = u;
            if (cfg->mode == DFM_MODE_SVF) {  /* pipeline.cpp:166-167 */
                exp_map_raw(&wg, u, cfg->svf_M, phis, tmp);
                phi = phis;
            }
            if ((rc = eval_loss(&wg, f, mv, phi, cfg, &value, grad))) break;
            if (!isfinite(value)) {
                rc = fail(2, "register_images: non-finite loss at scale %f, iteration %d",
                          scales[si], it);
                break;
            }
            losses[nl++] = value;
            dfm_iter_record rec = {si, scales[si], it, global++, value, 0.0, 0.0};
            if (converged(losses, nl, cfg->conv_window, cfg->conv_tol)) {
                rec.wall_ms = now_ms() - t_it;
                if (nrec < max_records) records[nrec] = rec;
                ++nrec;
                break;
            }
            if (cfg->mode == DFM_MODE_SVF) {  /* pipeline.cpp:189-206 */
                if ((rc = orc_svf_pullback(&wg, u, grad, cfg->svf_M, tmp))) break;
                if (cfg->sigma_grad > 0.0)
                    for (int a = 0; a < d; ++a) smooth_axis(tmp, &wg, d, a, cfg->sigma_grad);
                for (int64_t i = 0; i < n * d; ++i) tmp[i] = -tmp[i];
                if ((rc = orc_adam_step(&wg, m, nu, &t_adam, cfg->beta1, cfg->beta2,
                                        cfg->eps_adam, tmp, tmp2)))
                    break;
                double mx = 0.0;
                for (int64_t i = 0; i < n * d; ++i) {
                    const double sv = fabs(clampd(cfg->eta * tmp2[i], -cfg->step_cap, cfg->step_cap));
                    mx = mx > sv ? mx : sv;
                }
                rec.max_step = mx;
                for (int64_t i = 0; i < n * d; ++i)
                    u[i] += clampd(cfg->eta * tmp2[i], -cfg->step_cap, cfg->step_cap);
                if (cfg->sigma_warp > 0.0)
                    for (int a = 0; a < d; ++a) smooth_axis(u, &wg, d, a, cfg->sigma_warp);
                rec.wall_ms = now_ms() - t_it;
                if (nrec < max_records) records[nrec] = rec;
                ++nrec;
                continue;
            }
            if (cfg->sigma_grad > 0.0) {
                const double s3[3] = {cfg->sigma_grad, cfg->sigma_grad, cfg->sigma_grad};
                for (int a = 0; a < d; ++a) smooth_axis(grad, &wg, d, a, s3[a]);
            }
            if ((rc = orc_eulerian_direction(&wg, grad, u, cfg->use_jac, tmp))) break;
            if ((rc = orc_adam_step(&wg, m, nu, &t_adam, cfg->beta1, cfg->beta2, cfg->eps_adam,
                                    tmp, tmp2)))
                break;
            /* pipeline.cpp:36-41 max_abs_step (serial) */
            double mx = 0.0;
            for (int64_t i = 0; i < n * d; ++i) {
                const double s = fabs(clampd(cfg->eta * tmp2[i], -cfg->step_cap, cfg->step_cap));
                mx = mx > s ? mx : s;
            }
            rec.max_step = mx;
            if ((rc = orc_apply_update(&wg, u, tmp2, cfg->eta, cfg->sigma_warp, cfg->step_cap, tmp)))
                break;
            memcpy(u, tmp, (size_t)(n * d) * sizeof(double));
            rec.wall_ms = now_ms() - t_it;
            if (nrec < max_records) records[nrec] = rec;
            ++nrec;
        }
    }
    if (!rc && !dims_equal(&cur, g)) {
        rc = orc_upsample_field(&cur, u, g, tmp);
        if (!rc) memcpy(u, tmp, (size_t)(nfull * d) * sizeof(double));
    }
    double final_loss = 0.0, sing = 0.0;
    if (!rc && cfg->mode == DFM_MODE_SVF) {  /* pipeline.cpp:214-215: phi = exp(v) */
        exp_map_raw(g, u, cfg->svf_M, phis, tmp);
        memcpy(u, phis, (size_t)(nfull * d) * sizeof(double));
    }
    if (!rc) rc = eval_loss(g, fixed, moving, u, cfg, &final_loss, NULL);
    if (!rc) rc = orc_singularity_fraction(g, u, &sing);
    if (!rc) {
        if (out_field) memcpy(out_field, u, (size_t)(nfull * d) * sizeof(double));
        log->n_records = nrec < max_records ? nrec : max_records;
        log->n_total = nrec;
        log->final_loss = final_loss;
        log->final_singularity_fraction = sing;
        log->total_ms = now_ms() - t0;
        if (cfg->mode == DFM_MODE_DIRECT && sing > 0.0)
            rc = fail(2, "register_images: folded warp (det J <= 0 somewhere)");
    }
    free(f);
    free(mv);
    free(u);
    free(m);
    free(nu);
    free(tmp);
    free(tmp2);
    free(grad);
    free(phis);
    free(losses);
    return rc;
}

/* ---------------------------------------------------------------------- */
/* affine pre-alignment: affine.cpp:50-183                                  */

static int affine_eval(const dfm_grid* g, const double* f, const double* mv, int loss, int r,
                       double* phi, double* value, double* grad) {
    dfm_config c;
    memset(&c, 0, sizeof(c));
    c.loss = loss;
    c.lncc_radius = r;
    return eval_loss(g, f, mv, phi, &c, value, grad);
}

/* affine.cpp:72-77 */
int orc_affine_to_field(const dfm_grid* g, const double A[9], const double t[3], double* out) {
    CHECK(orc_validate_grid(g));
    dfm_init T;
    memset(&T, 0, sizeof(T));
    memcpy(T.A, A, sizeof(T.A));
    memcpy(T.t, t, sizeof(T.t));
    const double S[3] = {1.0, 1.0, 1.0};
    affine_working_field(&T, g, S, out);
    return 0;
}

/* affine.cpp:95-122: dL/dA_rc = sum_x (g_r / S_r) S_c x_c, dL/dt_r = sum_x g_r / S_r,
 * each a 4096-block ordered sum (parallel.cpp:153-169) */
int orc_affine_param_gradient(const dfm_grid* g, const double* fixed, const double* moving,
                              int loss, const double A[9], const double t[3], const double S[3],
                              int lncc_radius, double* value, double dA[9], double dt[3]) {
    CHECK(orc_validate_grid(g));
    const int d = g->ndim;
    const int64_t n = nvox(g);
    dfm_init T;
    memset(&T, 0, sizeof(T));
    memcpy(T.A, A, sizeof(T.A));
    memcpy(T.t, t, sizeof(T.t));
    double* u = dalloc(n * d);
    double* gr = dalloc(n * d);
    double* term = dalloc(n);
    affine_working_field(&T, g, S, u);
    int rc = affine_eval(g, fixed, moving, loss, lncc_radius, u, value, gr);
    for (int k = 0; k < 9; ++k) dA[k] = 0.0;
    for (int k = 0; k < 3; ++k) dt[k] = 0.0;
    if (!rc) {
        for (int r = 0; r < d; ++r) {
            for (int c = 0; c < d; ++c) {
                for (int64_t i = 0; i < n; ++i) {
                    double xw[3];
                    voxel_xyz(g, i, xw);
                    term[i] = gr[i * d + r] / S[r] * S[c] * xw[c];
                }
                dA[r * d + c] = block_sum(term, n);
            }
            for (int64_t i = 0; i < n; ++i) term[i] = gr[i * d + r] / S[r];
            dt[r] = block_sum(term, n);
        }
    }
    free(u);
    free(gr);
    free(term);
    return rc;
}

/* affine.cpp:124-183 */
int orc_affine_register(const dfm_grid* g, const double* fixed, const double* moving, int loss,
                        const double* scales, const int32_t* iters, int32_t nscales, double eta,
                        int lncc_radius, dfm_affine_result* out) {
    CHECK(orc_validate_grid(g));
    if (nscales < 1) return fail(1, "affine_register: bad schedule");
    const int d = g->ndim, np = d * d + d;
    const int64_t nfull = nvox(g);
    double A[9] = {0}, t[3] = {0}, bA[9], bt[3];
    for (int i = 0; i < d; ++i) A[i * d + i] = 1.0;
    memcpy(bA, A, sizeof(A));
    memcpy(bt, t, sizeof(t));
    double best = INFINITY;
    double am[12] = {0}, anu[12] = {0};
    int64_t ta = 0, total = 0;
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    double* f = dalloc(nfull);
    double* mv = dalloc(nfull);
    int rc = 0, diverged = 0;
    for (int si = 0; si < nscales && !rc && !diverged; ++si) {
        const double fac[3] = {scales[si], scales[si], scales[si]};
        dfm_grid wg;
        if ((rc = orc_downsample_image(g, fixed, fac, &wg, f))) break;
        if ((rc = orc_downsample_image(g, moving, fac, &wg, mv))) break;
        double S[3] = {1.0, 1.0, 1.0};
        for (int a = 0; a < d; ++a) S[a] = (double)(g->dims[a] - 1) / (double)(wg.dims[a] - 1);
        for (int it = 0; it < iters[si]; ++it) {
            double value, dA[9], dt[3];
            if ((rc = orc_affine_param_gradient(&wg, f, mv, loss, A, t, S, lncc_radius, &value,
                                                dA, dt)))
                break;
            ++total;
            if (!isfinite(value)) {
                diverged = 1;
                break;
            }
            if (value < best) {
                best = value;
                memcpy(bA, A, sizeof(A));
                memcpy(bt, t, sizeof(t));
            }
            ++ta;
            const double c1 = 1.0 - pow(b1, (double)ta);
            const double c2 = 1.0 - pow(b2, (double)ta);
            for (int p = 0; p < np; ++p) {
                const double gp = p < d * d ? dA[p] : dt[p - d * d];
                am[p] = b1 * am[p] + (1.0 - b1) * gp;
                anu[p] = b2 * anu[p] + (1.0 - b2) * gp * gp;
                const double dir = (am[p] / c1) / (sqrt(anu[p] / c2) + eps);
                if (p < d * d)
                    A[p] -= eta * dir;
                else
                    t[p - d * d] -= eta * dir;
            }
        }
    }
    free(f);
    free(mv);
    if (rc) return rc;
    out->ndim = d;
    memcpy(out->A, bA, sizeof(bA));
    memcpy(out->t, bt, sizeof(bt));
    out->loss = best;
    out->diverged = diverged;
    out->iterations = total;
    if (!diverged) {
        const double det = d == 2 ? bA[0] * bA[3] - bA[1] * bA[2]
                                  : bA[0] * (bA[4] * bA[8] - bA[5] * bA[7]) -
                                        bA[1] * (bA[3] * bA[8] - bA[5] * bA[6]) +
                                        bA[2] * (bA[3] * bA[7] - bA[4] * bA[6]);
        if (fabs(det) < 1e-3) return fail(2, "affine_register: transform collapsed (|det A| < 1e-3)");
    }
    return 0;
}

/* analysis.cpp:169-247, MO (Dice) columns only.  Labels are ints; regions are
 * visited in ascending label order like std::map. */
int orc_overlap_dice(const dfm_grid* g, const int32_t* warped, const int32_t* fixed,
                     double* mo_mean, double* mo_klein) {
    const int64_t n = nvox(g);
    int32_t maxl = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (warped[i] > maxl) maxl = warped[i];
        if (fixed[i] > maxl) maxl = fixed[i];
    }
    int64_t* S = calloc((size_t)maxl + 1, sizeof(int64_t));
    int64_t* T = calloc((size_t)maxl + 1, sizeof(int64_t));
    int64_t* I = calloc((size_t)maxl + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        const int32_t s = warped[i], t = fixed[i];
        if (s > 0) ++S[s];
        if (t > 0) ++T[t];
        if (s > 0 && s == t) ++I[s];
    }
    double mo = 0.0;
    int cnt = 0;
    int64_t ps = 0, pt = 0, pi = 0;
    for (int32_t l = 1; l <= maxl; ++l) {
        if (S[l] + T[l] == 0) continue;
        mo += 2.0 * (double)I[l] / (double)(S[l] + T[l]);
        ++cnt;
        ps += S[l];
        pt += T[l];
        pi += I[l];
    }
    *mo_mean = cnt ? mo / cnt : 0.0;
    *mo_klein = (ps + pt) ? 2.0 * (double)pi / (double)(ps + pt) : 0.0;
    free(S);
    free(T);
    free(I);
    return 0;
}

/* analysis.cpp:169-247: full report; regions in ascending label order */
int orc_overlap_report(const dfm_grid* gw, const int32_t* warped, const dfm_grid* gf,
                       const int32_t* fixed, dfm_overlap_summary* rep,
                       dfm_region_overlap* regions, int64_t cap) {
    CHECK(orc_validate_grid(gw));
    CHECK(orc_validate_grid(gf));
    if (!same_grid(gw, gf)) return fail(1, "overlap_report: grid mismatch");
    const int64_t n = nvox(gw);
    int32_t maxl = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (warped[i] > maxl) maxl = warped[i];
        if (fixed[i] > maxl) maxl = fixed[i];
    }
    int64_t* S = calloc((size_t)maxl + 1, sizeof(int64_t));
    int64_t* T = calloc((size_t)maxl + 1, sizeof(int64_t));
    int64_t* I = calloc((size_t)maxl + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        const int32_t s = warped[i], t = fixed[i];
        if (s > 0) ++S[s];
        if (t > 0) ++T[t];
        if (s > 0 && s == t) ++I[s];
    }
    memset(rep, 0, sizeof(*rep));
    int64_t ps = 0, pt = 0, pi = 0, pfn = 0, pfp = 0, nr = 0;
    int to_n = 0, fp_n = 0, vs_n = 0;
    for (int32_t l = 1; l <= maxl; ++l) {
        if (S[l] == 0 && T[l] == 0) continue;
        dfm_region_overlap r;
        memset(&r, 0, sizeof(r));
        r.label = l;
        r.warped_count = S[l];
        r.fixed_count = T[l];
        r.intersection = I[l];
        const int64_t fn = T[l] - I[l], fp = S[l] - I[l];
        if (T[l] > 0) {
            r.has_to = r.has_fn = 1;
            r.to = (double)I[l] / (double)T[l];
            r.fn = (double)fn / (double)T[l];
            rep->to_mean += r.to;
            rep->fn_mean += r.fn;
            ++to_n;
        }
        if (S[l] > 0) {
            r.has_fp = 1;
            r.fp = (double)fp / (double)S[l];
            rep->fp_mean += r.fp;
            ++fp_n;
        }
        const int64_t den = S[l] + T[l];
        r.mo = 2.0 * (double)I[l] / (double)den;
        r.vs = 2.0 * (double)(S[l] - T[l]) / (double)den;
        rep->mo_mean += r.mo;
        rep->vs_mean += r.vs;
        ++vs_n;
        ps += S[l];
        pt += T[l];
        pi += I[l];
        pfn += fn;
        pfp += fp;
        if (nr < cap) regions[nr] = r;
        ++nr;
    }
    if (to_n > 0) {
        rep->to_mean /= to_n;
        rep->fn_mean /= to_n;
    }
    if (fp_n > 0) rep->fp_mean /= fp_n;
    if (vs_n > 0) {
        rep->mo_mean /= vs_n;
        rep->vs_mean /= vs_n;
    }
    if (pt > 0) {
        rep->to_klein = (double)pi / (double)pt;
        rep->fn_klein = (double)pfn / (double)pt;
    }
    if (ps > 0) rep->fp_klein = (double)pfp / (double)ps;
    if (ps + pt > 0) {
        rep->mo_klein = 2.0 * (double)pi / (double)(ps + pt);
        rep->vs_klein = 2.0 * (double)(ps - pt) / (double)(ps + pt);
    }
    rep->n_regions = nr;
    free(S);
    free(T);
    free(I);
    return 0;
}

/* analysis.cpp:249-283 */
int orc_landmark_error(const dfm_grid* fg, const dfm_grid* mg, const dfm_grid* pg,
                       const double* phi, int64_t n, const double* fixed_mm,
                       const double* moving_mm, double* dist, double* mean, double* mx) {
    if (!same_grid(pg, fg)) /* core.hpp:20-22: ndim and dims */
        return fail(1, "landmark_error: field must live on the fixed grid");
    *mean = 0.0;
    *mx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double vox[3] = {0.0, 0.0, 0.0}, u[3];
        for (int a = 0; a < fg->ndim; ++a)
            vox[a] = (fixed_mm[3 * i + a] - fg->origin[a]) / fg->spacing[a];
        sample_field(pg, phi, vox, u);
        double d2 = 0.0;
        for (int a = 0; a < fg->ndim; ++a) {
            const double mapped = (vox[a] + u[a]) * mg->spacing[a] + mg->origin[a];
            const double diff = mapped - moving_mm[3 * i + a];
            d2 += diff * diff;
        }
        const double d = sqrt(d2);
        dist[i] = d;
        *mean += d;
        *mx = *mx > d ? *mx : d;
    }
    if (n > 0) *mean /= (double)n;
    return 0;
}

/* pipeline.cpp:226-313 sweep, serial (workers = 1): config k = (ei*n_sw + wi)*n_sg + gi */
int orc_sweep(const dfm_sweep_pair* pairs, int npairs, const dfm_config* base,
              const double* scales, const int32_t* iters, int32_t nscales, const double* etas,
              int n_eta, const double* sws, int n_sw, const double* sgs, int n_sg, int metric,
              dfm_sweep_row* rows) {
    if (npairs < 1) return fail(1, "sweep: at least one image pair required");
    if (n_eta < 1 || n_sw < 1 || n_sg < 1) return fail(1, "sweep: grid axes must be non-empty");
    if (metric == DFM_SWEEP_OVERLAP)
        for (int p = 0; p < npairs; ++p)
            if (!pairs[p].fixed_labels || !pairs[p].moving_labels)
                return fail(1, "sweep: overlap metric needs label maps on every pair");
    const int64_t n_cfg = (int64_t)n_eta * n_sw * n_sg;
    int64_t cap = 1;
    for (int i = 0; i < nscales; ++i) cap += iters[i];
    dfm_iter_record* recs = calloc((size_t)cap, sizeof(dfm_iter_record));
    for (int64_t k = 0; k < n_cfg; ++k) {
        const int64_t gi = k % n_sg, wi = (k / n_sg) % n_sw, ei = k / ((int64_t)n_sg * n_sw);
        dfm_sweep_row* row = &rows[k];
        memset(row, 0, sizeof(*row));
        row->eta = etas[ei];
        row->sigma_warp = sws[wi];
        row->sigma_grad = sgs[gi];
        row->computed = 1;
        dfm_config cfg = *base;
        cfg.eta = row->eta;
        cfg.sigma_warp = row->sigma_warp;
        cfg.sigma_grad = row->sigma_grad;
        cfg.seed = base->seed + (uint64_t)k;
        const double t0 = now_ms();
        double sum = 0.0, sum2 = 0.0;
        int failed = 0;
        for (int p = 0; p < npairs && !failed; ++p) {
            const dfm_grid* g = pairs[p].grid;
            const int64_t n = nvox(g);
            double* phi = dalloc(n * g->ndim);
            dfm_runlog log;
            double m = 0.0;
            int rc = orc_register(g, pairs[p].fixed, pairs[p].moving, &cfg, scales, iters, nscales,
                                  NULL, phi, recs, cap, &log);
            if (!rc) {
                if (metric == DFM_SWEEP_LOSS) {
                    m = log.final_loss;
                } else {
                    int32_t* w = calloc((size_t)n, sizeof(int32_t));
                    orc_warp_labels(g, pairs[p].moving_labels, phi, w);
                    dfm_overlap_summary rep;
                    orc_overlap_report(g, w, g, pairs[p].fixed_labels, &rep, NULL, 0);
                    m = rep.to_mean;
                    free(w);
                }
            } else {
                failed = 1;
                orc_last_error(row->error, sizeof(row->error));
            }
            free(phi);
            sum += m;
            sum2 += m * m;
        }
        if (failed) {
            row->failed = 1;
            row->metric_mean = NAN;
            row->metric_sd = NAN;
        } else {
            const double nn = (double)npairs;
            row->metric_mean = sum / nn;
            const double v = sum2 / nn - row->metric_mean * row->metric_mean;
            row->metric_sd = sqrt(v > 0.0 ? v : 0.0);
        }
        row->wall_ms = now_ms() - t0;
    }
    free(recs);
    return 0;
}
