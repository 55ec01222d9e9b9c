// kernels_exact.cu — the bit-exact fp64 parity mode (DFM_OPT_EXACT).
//
// The tuned loop reassociates sums (separable filters in fp64/fp32 rings,
// reciprocal multiplies, FMA contraction, fused kernels).  On chaotic inputs
// those last-bit differences grow: on BASELINE's LNCC phantoms the fp64 loop
// drifts from the reference by 1e-4..1e-3 in the loss after 350 iterations —
// as far as the reference drifts from its own FMA build.  This
// mode instead evaluates register_images (direct mode, SSD / LNCC,
// use_jac on or off, any init) with the reference's arithmetic in the
// reference's order, one IEEE operation at a time: every sum accumulates in
// the reference's loop order (clipped box sums and Gaussian taps from the
// window's low end, corner loops cz-cy-cx, 4096-element blocks for the loss),
// every quotient is a division, and this file is compiled with -fmad=false
// (no contraction anywhere).  Fields are AoS doubles as in the reference.  The
// result is bit-identical to the reference's register_images
// (tests/test_exact_gpu.py): it is the parity mode, not the fast path —
// one thread per output element, no fusion.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/difform_gpu.h"

namespace dfm {
namespace exact {

struct Meta {
    int ndim;
    int64_t d[3];
    __host__ __device__ int64_t n() const { return d[0] * d[1] * d[2]; }
};

constexpr int kNT = 256;

inline unsigned grid_for(int64_t n) {
    int64_t b = (n + kNT - 1) / kNT;
    if (b < 1) b = 1;
    if (b > (int64_t(1) << 30)) b = int64_t(1) << 30;
    return static_cast<unsigned>(b);
}

#define EX_LOOP(i, n) \
    for (int64_t i = blockIdx.x * int64_t(kNT) + threadIdx.x; i < (n); i += int64_t(gridDim.x) * kNT)

struct Cell {
    int64_t i0[3];
    double f[3];
    bool cl[3];
};

// interp.cpp:19-37
__device__ __forceinline__ Cell locate(const Meta& m, const double p_in[3]) {
    Cell c;
    for (int a = 0; a < 3; ++a) {
        if (a >= m.ndim || m.d[a] == 1) {
            c.i0[a] = 0;
            c.f[a] = 0.0;
            c.cl[a] = false;
            continue;
        }
        double p = p_in[a];
        const double hi = static_cast<double>(m.d[a] - 1);
        c.cl[a] = (p < 0.0 || p > hi);
        p = p < 0.0 ? 0.0 : (hi < p ? hi : p);  // std::clamp
        int64_t i = static_cast<int64_t>(floor(p));
        i = i < 0 ? 0 : (m.d[a] - 2 < i ? m.d[a] - 2 : i);
        c.i0[a] = i;
        c.f[a] = p - static_cast<double>(i);
    }
    return c;
}

// interp.cpp:40-49
__device__ __forceinline__ double corner_weight(const Cell& c, int cx, int cy, int cz, int skip) {
    const int k[3] = {cx, cy, cz};
    double w = 1.0;
    for (int a = 0; a < 3; ++a) {
        if (a == skip) continue;
        w *= k[a] ? c.f[a] : (1.0 - c.f[a]);
    }
    return w;
}

// interp.cpp:51-57 (voxel index of a corner)
__device__ __forceinline__ int64_t corner_index(const Meta& m, const Cell& c, int cx, int cy,
                                                int cz) {
    const int64_t x = c.i0[0] + (m.d[0] > 1 ? cx : 0);
    const int64_t y = c.i0[1] + (m.d[1] > 1 ? cy : 0);
    const int64_t z = (m.ndim == 3 && m.d[2] > 1) ? c.i0[2] + cz : 0;
    return (z * m.d[1] + y) * m.d[0] + x;
}

__device__ __forceinline__ int ncz(const Meta& m) { return (m.ndim == 3 && m.d[2] > 1) ? 2 : 1; }

// interp.cpp:155-164
__device__ __forceinline__ double sample_linear(const Meta& m, const double* img,
                                                const double p[3]) {
    const Cell c = locate(m, p);
    double acc = 0.0;
    for (int cz = 0; cz < ncz(m); ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx)
                acc += corner_weight(c, cx, cy, cz, -1) * img[corner_index(m, c, cx, cy, cz)];
    return acc;
}

// interp.cpp:166-186
__device__ __forceinline__ void sample_gradient(const Meta& m, const double* img,
                                                const double p[3], double g[3]) {
    const Cell c = locate(m, p);
    g[0] = g[1] = g[2] = 0.0;
    for (int a = 0; a < m.ndim; ++a) {
        if (m.d[a] == 1 || c.cl[a]) continue;
        double acc = 0.0;
        for (int cz = 0; cz < ncz(m); ++cz)
            for (int cy = 0; cy < 2; ++cy)
                for (int cx = 0; cx < 2; ++cx) {
                    const int k[3] = {cx, cy, cz};
                    const double sgn = k[a] ? 1.0 : -1.0;
                    acc += sgn * corner_weight(c, cx, cy, cz, a) *
                           img[corner_index(m, c, cx, cy, cz)];
                }
        g[a] = acc;
    }
}

// interp.cpp:188-203 (AoS field with ndim components)
__device__ __forceinline__ void sample_field(const Meta& m, const double* f, const double p[3],
                                             double out[3]) {
    const Cell c = locate(m, p);
    const int d = m.ndim;
    out[0] = out[1] = out[2] = 0.0;
    for (int cz = 0; cz < ncz(m); ++cz)
        for (int cy = 0; cy < 2; ++cy)
            for (int cx = 0; cx < 2; ++cx) {
                const double w = corner_weight(c, cx, cy, cz, -1);
                const int64_t j = corner_index(m, c, cx, cy, cz);
                for (int k = 0; k < d; ++k) out[k] += w * f[j * d + k];
            }
}

__device__ __forceinline__ void voxel_xyz(const Meta& m, int64_t i, double p[3]) {
    p[0] = static_cast<double>(i % m.d[0]);
    p[1] = static_cast<double>((i / m.d[0]) % m.d[1]);
    p[2] = static_cast<double>(i / (m.d[0] * m.d[1]));
}

// interp.cpp:291-328
__device__ __forceinline__ void jacobian_at(const Meta& m, const double* phi, int64_t i,
                                            double J[9]) {
    const int d = m.ndim;
    const int64_t pos[3] = {i % m.d[0], (i / m.d[0]) % m.d[1], i / (m.d[0] * m.d[1])};
    for (int k = 0; k < 9; ++k) J[k] = 0.0;
    for (int a = 0; a < d; ++a) {
        int64_t lo[3] = {pos[0], pos[1], pos[2]}, hi[3] = {pos[0], pos[1], pos[2]};
        double den;
        if (pos[a] == 0) {
            hi[a] = 1;
            den = 1.0;
        } else if (pos[a] == m.d[a] - 1) {
            lo[a] = m.d[a] - 2;
            den = 1.0;
        } else {
            lo[a] = pos[a] - 1;
            hi[a] = pos[a] + 1;
            den = 2.0;
        }
        const int64_t jl = (lo[2] * m.d[1] + lo[1]) * m.d[0] + lo[0];
        const int64_t jh = (hi[2] * m.d[1] + hi[1]) * m.d[0] + hi[0];
        for (int c = 0; c < d; ++c)
            J[c * d + a] = (phi[jh * d + c] - phi[jl * d + c]) / den + (c == a ? 1.0 : 0.0);
    }
}

// ---------------------------------------------------------------------------
// kernels

// similarity.cpp:25-45
__global__ void k_warp_grad(const double* __restrict__ mov, Meta mm, const double* __restrict__ phi,
                            Meta fm, double* __restrict__ W, double* __restrict__ G) {
    const int d = fm.ndim;
    EX_LOOP(i, fm.n()) {
        double p[3], g[3];
        voxel_xyz(fm, i, p);
        for (int c = 0; c < d; ++c) p[c] += phi[i * d + c];
        W[i] = sample_linear(mm, mov, p);
        if (G) {
            sample_gradient(mm, mov, p, g);
            for (int c = 0; c < d; ++c) G[i * d + c] = g[c];
        }
    }
}

// similarity.cpp:131-136: the six moment images (cnt, F, W, F^2, W^2, FW)
__global__ void k_moments(const double* __restrict__ F, const double* __restrict__ W, int64_t n,
                          double* __restrict__ mo) {
    EX_LOOP(i, n) {
        mo[i] = 1.0;
        mo[n + i] = F[i];
        mo[2 * n + i] = W[i];
        mo[3 * n + i] = F[i] * F[i];
        mo[4 * n + i] = W[i] * W[i];
        mo[5 * n + i] = F[i] * W[i];
    }
}

// similarity.cpp:48-68: clipped box sum along `axis` of `nimg` scalar images
__global__ void k_box_axis(const double* __restrict__ in, double* __restrict__ out, Meta m,
                           int axis, int r, int nimg) {
    const int64_t n = m.n(), na = m.d[axis];
    int64_t stride = 1;
    for (int a = 0; a < axis; ++a) stride *= m.d[a];
    EX_LOOP(e, n * nimg) {
        const int64_t img = e / n, v = e - img * n;
        const int64_t i = (v / stride) % na;
        const int64_t jlo = i - r > 0 ? i - r : 0;
        const int64_t jhi = i + r < na - 1 ? i + r : na - 1;
        const double* src = in + img * n + (v - i * stride);
        double acc = 0.0;
        for (int64_t j = jlo; j <= jhi; ++j) acc += src[j * stride];
        out[e] = acc;
    }
}

// similarity.cpp:144-168
__global__ void k_lncc_coef(const double* __restrict__ mo, int64_t n, double* __restrict__ cf,
                            double* __restrict__ cc2) {
    EX_LOOP(i, n) {
        const double cnt = mo[i];
        const double muF = mo[n + i] / cnt;
        const double muW = mo[2 * n + i] / cnt;
        const double vFr = mo[3 * n + i] / cnt - muF * muF;
        const double vWr = mo[4 * n + i] / cnt - muW * muW;
        const double vF = 0.0 < vFr ? vFr : 0.0;  // std::max(0.0, x)
        const double vW = 0.0 < vWr ? vWr : 0.0;
        const double cv = mo[5 * n + i] / cnt - muF * muW;
        if (vF < 1e-5 || vW < 1e-5) {
            cc2[i] = cf[i] = cf[n + i] = cf[2 * n + i] = cf[3 * n + i] = 0.0;
            continue;
        }
        const double cc = cv / sqrt(vF * vW);
        cc2[i] = cc * cc;
        const double alpha = cv / (vF * vW);
        const double beta = cv * cv / (vF * vW * vW);
        cf[i] = alpha / cnt;
        cf[n + i] = alpha * muF / cnt;
        cf[2 * n + i] = beta / cnt;
        cf[3 * n + i] = beta * muW / cnt;
    }
}

// similarity.cpp:178-189
__global__ void k_lncc_grad(const double* __restrict__ F, const double* __restrict__ W,
                            const double* __restrict__ bs, const double* __restrict__ G,
                            int64_t n, int d, double* __restrict__ grad) {
    const double N = static_cast<double>(n);
    EX_LOOP(i, n) {
        const double dW =
            -2.0 / N * (F[i] * bs[i] - bs[n + i] - W[i] * bs[2 * n + i] + bs[3 * n + i]);
        for (int c = 0; c < d; ++c) grad[i * d + c] = dW * G[i * d + c];
    }
}

// similarity.cpp:81-104
__global__ void k_ssd_terms(const double* __restrict__ F, const double* __restrict__ W,
                            const double* __restrict__ G, int64_t n, int d,
                            double* __restrict__ t, double* __restrict__ grad) {
    const double N = static_cast<double>(n);
    EX_LOOP(i, n) {
        const double r = F[i] - W[i];
        t[i] = r * r;
        if (grad) {
            const double q = W[i] - F[i];
            for (int c = 0; c < d; ++c) grad[i * d + c] = q * G[i * d + c] / N;
        }
    }
}

// parallel.cpp:55-71: the sum of every 4096-element block in order
__global__ void k_block_sums(const double* __restrict__ t, int64_t n, double* __restrict__ part) {
    const int64_t nb = (n + 4095) / 4096;
    EX_LOOP(b, nb) {
        const int64_t lo = b * 4096, hi = lo + 4096 < n ? lo + 4096 : n;
        double acc = 0.0;
        for (int64_t i = lo; i < hi; ++i) acc += t[i];
        part[b] = acc;
    }
}

// interp.cpp:110-151: one axis of an interleaved buffer, renormalised taps
__global__ void k_smooth_axis(const double* __restrict__ in, double* __restrict__ out, Meta m,
                              int comps, int axis, const double* __restrict__ taps, int64_t R) {
    const int64_t n = m.n(), na = m.d[axis];
    int64_t stride = 1;
    for (int a = 0; a < axis; ++a) stride *= m.d[a];
    EX_LOOP(e, n * comps) {
        const int64_t v = e / comps, c = e - v * comps;
        const int64_t i = (v / stride) % na;
        const int64_t jlo = -R > -i ? -R : -i;
        const int64_t jhi = R < na - 1 - i ? R : na - 1 - i;
        double acc = 0.0, ws = 0.0;
        for (int64_t j = jlo; j <= jhi; ++j) {
            const double w = taps[j + R];
            acc += w * in[(v + j * stride) * comps + c];
            ws += w;
        }
        out[e] = acc / ws;
    }
}

// diffeo.cpp:11-40
__global__ void k_eulerian(const double* __restrict__ g, const double* __restrict__ phi, Meta m,
                           int use_jac, double* __restrict__ out) {
    const int d = m.ndim;
    EX_LOOP(i, m.n()) {
        if (!use_jac) {
            for (int c = 0; c < d; ++c) out[i * d + c] = -g[i * d + c];
            continue;
        }
        double J[9];
        jacobian_at(m, phi, i, J);
        for (int a = 0; a < d; ++a) {
            double acc = 0.0;
            for (int c = 0; c < d; ++c) acc += J[c * d + a] * g[i * d + c];
            out[i * d + a] = -acc;
        }
    }
}

// optim.cpp:22-42 (corr1/corr2 by std::pow on the host)
__global__ void k_adam(double* __restrict__ m, double* __restrict__ nu,
                       const double* __restrict__ v, double* __restrict__ dir, int64_t n, double b1,
                       double b2, double c1, double c2, double eps) {
    EX_LOOP(i, n) {
        m[i] = b1 * m[i] + (1.0 - b1) * v[i];
        nu[i] = b2 * nu[i] + (1.0 - b2) * v[i] * v[i];
        const double mh = m[i] / c1;
        const double nh = nu[i] / c2;
        dir[i] = mh / (sqrt(nh) + eps);
    }
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// pipeline.cpp:36-41 (max |step|, a record only) + diffeo.cpp:47-55
__global__ void k_step(const double* __restrict__ dir, int64_t n, double eta, double cap,
                       double* __restrict__ step, unsigned long long* mx, int* bad) {
    EX_LOOP(i, n) {
        const double s = eta * dir[i];
        if (!isfinite(s)) atomicOr(bad, 1);
        const double c = clampd(s, -cap, cap);
        step[i] = c;
        const double a = fabs(c);
        if (a == a) atomicMax(mx, static_cast<unsigned long long>(__double_as_longlong(a)));
    }
}

// interp.cpp:269-289: out = psi + phi(x + psi)
__global__ void k_compose(const double* __restrict__ phi, const double* __restrict__ psi, Meta m,
                          double* __restrict__ out) {
    const int d = m.ndim;
    EX_LOOP(i, m.n()) {
        double p[3], up[3];
        voxel_xyz(m, i, p);
        for (int c = 0; c < d; ++c) p[c] += psi[i * d + c];
        sample_field(m, phi, p, up);
        for (int c = 0; c < d; ++c) out[i * d + c] = psi[i * d + c] + up[c];
    }
}

// interp.cpp:381-445 / core.cpp:86-91: corner-aligned resample (field or image)
__global__ void k_resample(const double* __restrict__ f, Meta om, Meta nm, int comps, double st0,
                           double st1, double st2, double r0, double r1, double r2, int scale,
                           double* __restrict__ out) {
    const double rs[3] = {r0, r1, r2};
    EX_LOOP(i, nm.n()) {
        const int64_t x = i % nm.d[0];
        const int64_t y = (i / nm.d[0]) % nm.d[1];
        const int64_t z = i / (nm.d[0] * nm.d[1]);
        const double p[3] = {x * st0, y * st1, z * st2};
        if (comps == 0) {  // scalar image (downsample_image)
            out[i] = sample_linear(om, f, p);
            continue;
        }
        double v[3];
        sample_field(om, f, p, v);
        for (int c = 0; c < comps; ++c) out[i * comps + c] = scale ? v[c] * rs[c] : v[c];
    }
}

__global__ void k_scale_comps(double* __restrict__ f, int64_t n, int d, double s0, double s1,
                              double s2) {
    const double s[3] = {s0, s1, s2};
    EX_LOOP(i, n) for (int c = 0; c < d; ++c) f[i * d + c] *= s[c];
}

// affine.cpp:26-48: u(x) = S^-1 (A S x + t) - x
__global__ void k_affine_working(Meta m, const dfm_init T, double S0, double S1, double S2,
                                 double* __restrict__ u) {
    const double S[3] = {S0, S1, S2};
    const int d = m.ndim;
    EX_LOOP(i, m.n()) {
        double xw[3];
        voxel_xyz(m, i, xw);
        for (int r = 0; r < d; ++r) {
            double acc = T.t[r];
            for (int c = 0; c < d; ++c) acc += T.A[r * d + c] * S[c] * xw[c];
            u[i * d + r] = acc / S[r] - xw[r];
        }
    }
}

// analysis.cpp:160-167 + interp.cpp:330-349
__global__ void k_fold_count(const double* __restrict__ phi, Meta m,
                             unsigned long long* __restrict__ cnt) {
    const int d = m.ndim;
    EX_LOOP(i, m.n()) {
        double J[9];
        jacobian_at(m, phi, i, J);
        double det;
        if (d == 2)
            det = J[0] * J[3] - J[1] * J[2];
        else
            det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                  J[2] * (J[3] * J[7] - J[4] * J[6]);
        if (det <= 0.0) atomicAdd(cnt, 1ull);
    }
}

// ---------------------------------------------------------------------------
// host driver: pipeline.cpp:121-224, direct mode

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(DFM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct Dev {
    std::vector<void*> ptrs;
    double* alloc(int64_t n) {
        void* p = nullptr;
        ck(cudaMalloc(&p, sizeof(double) * static_cast<size_t>(n > 0 ? n : 1)), "cudaMalloc");
        ptrs.push_back(p);
        return static_cast<double*>(p);
    }
    ~Dev() {
        for (void* p : ptrs) cudaFree(p);
    }
};

Meta meta_of(const dfm_grid* g) {
    Meta m;
    m.ndim = g->ndim;
    for (int a = 0; a < 3; ++a) m.d[a] = g->dims[a];
    return m;
}

bool same_dims(const Meta& a, const Meta& b) {
    return a.d[0] == b.d[0] && a.d[1] == b.d[1] && a.d[2] == b.d[2];
}

struct Runner {
    cudaStream_t s;
    int64_t* launches;
    Dev dev;
    double* taps = nullptr;  // scratch for the Gaussian taps
    double* scratch = nullptr;

    void bump() { ++*launches; }

    // interp.cpp:117-130: taps of one axis, normalised (host libm, as the reference)
    void smooth(double* data, const Meta& m, int comps, const double sigma[3]) {
        for (int a = 0; a < m.ndim; ++a) {
            if (sigma[a] <= 0.0 || m.d[a] == 1) continue;
            const int64_t R = static_cast<int64_t>(std::ceil(3.0 * sigma[a]));
            std::vector<double> h(static_cast<size_t>(2 * R + 1));
            double tsum = 0.0;
            for (int64_t j = -R; j <= R; ++j) {
                const double t = std::exp(-0.5 * (j / sigma[a]) * (j / sigma[a]));
                h[static_cast<size_t>(j + R)] = t;
                tsum += t;
            }
            for (double& t : h) t /= tsum;
            ck(cudaMemcpyAsync(taps, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice,
                               s),
               "taps");
            const int64_t ne = m.n() * comps;
            k_smooth_axis<<<grid_for(ne), kNT, 0, s>>>(data, scratch, m, comps, a, taps, R);
            bump();
            ck(cudaMemcpyAsync(data, scratch, sizeof(double) * ne, cudaMemcpyDeviceToDevice, s),
               "smooth copy");
            ck(cudaStreamSynchronize(s), "smooth sync");  // taps reused by the next axis
        }
    }

    double block_total(const double* t, int64_t n, double* part) {
        const int64_t nb = (n + 4095) / 4096;
        k_block_sums<<<grid_for(nb), kNT, 0, s>>>(t, n, part);
        bump();
        std::vector<double> h(static_cast<size_t>(nb));
        ck(cudaMemcpyAsync(h.data(), part, sizeof(double) * nb, cudaMemcpyDeviceToHost, s),
           "partials");
        ck(cudaStreamSynchronize(s), "partials sync");
        double total = 0.0;
        for (double p : h) total += p;
        return total;
    }

    // core.cpp:58-96
    void downsample(const double* img, const Meta& m, const double fac, Meta& om, double* out,
                    double* tmp) {
        om = m;
        double sigma[3] = {0, 0, 0};
        bool blur = false;
        for (int a = 0; a < m.ndim; ++a) {
            om.d[a] = static_cast<int64_t>(std::ceil(m.d[a] / fac));
            if (fac > 1.0) {
                sigma[a] = fac / 2.0;
                blur = true;
            }
        }
        if (same_dims(m, om) && !blur) {
            ck(cudaMemcpyAsync(out, img, sizeof(double) * m.n(), cudaMemcpyDeviceToDevice, s),
               "copy");
            return;
        }
        ck(cudaMemcpyAsync(tmp, img, sizeof(double) * m.n(), cudaMemcpyDeviceToDevice, s), "copy");
        if (blur) smooth(tmp, m, 1, sigma);
        double st[3] = {0, 0, 0};
        for (int a = 0; a < m.ndim; ++a)
            st[a] = static_cast<double>(m.d[a] - 1) / (om.d[a] - 1);
        k_resample<<<grid_for(om.n()), kNT, 0, s>>>(tmp, m, om, 0, st[0], st[1], st[2], 1, 1, 1, 0,
                                                    out);
        bump();
    }

    // interp.cpp:381-445: resample_field_linear (scale 0) / upsample_field (scale 1)
    void resample_field(const double* f, const Meta& m, const Meta& nm, bool rescale,
                        double* out) {
        double st[3] = {0, 0, 0}, r[3] = {1, 1, 1};
        for (int a = 0; a < nm.ndim; ++a) {
            st[a] = nm.d[a] > 1 ? static_cast<double>(m.d[a] - 1) / (nm.d[a] - 1) : 0.0;
            r[a] = static_cast<double>(nm.d[a] - 1) / (m.d[a] - 1);
        }
        k_resample<<<grid_for(nm.n()), kNT, 0, s>>>(f, m, nm, nm.ndim, st[0], st[1], st[2], r[0],
                                                    r[1], r[2], rescale ? 1 : 0, out);
        bump();
    }
};

}  // namespace exact

// register_images (pipeline.cpp:121-224) with the reference's arithmetic; F, M
// are full-resolution device images (doubles); the AoS field lands in
// d_field_aos (voxel_count * ndim doubles).  Records as dfm_register.
void exact_register(cudaStream_t stream, int64_t* launches, const dfm_grid* g, const double* F,
                    const double* M, const dfm_config* cfg, const double* scales,
                    const int32_t* iters, int ns, const dfm_init* init, double* d_field_aos,
                    std::vector<dfm_iter_record>& recs, double* final_loss, double* sing) {
    using namespace exact;
    if (cfg->mode != DFM_MODE_DIRECT)
        fail(DFM_E_INVALID, "exact mode: direct mode only");
    if (cfg->loss != DFM_LOSS_LNCC && cfg->loss != DFM_LOSS_SSD)
        fail(DFM_E_INVALID, "exact mode: LNCC or SSD loss only");
    Runner X;
    X.s = stream;
    X.launches = launches;
    const Meta full = meta_of(g);
    const int d = full.ndim;
    const int64_t nf = full.n();
    double* f = X.dev.alloc(nf);
    double* mv = X.dev.alloc(nf);
    double* u = X.dev.alloc(nf * d);
    double* m = X.dev.alloc(nf * d);
    double* nu = X.dev.alloc(nf * d);
    double* tmp = X.dev.alloc(nf * d);
    double* tmp2 = X.dev.alloc(nf * d);
    double* grad = X.dev.alloc(nf * d);
    double* W = X.dev.alloc(nf);
    double* G = X.dev.alloc(nf * d);
    double* mo = X.dev.alloc(6 * nf);
    double* bs = X.dev.alloc(6 * nf);
    double* cc2 = X.dev.alloc(nf);
    double* part = X.dev.alloc((nf + 4095) / 4096 + 1);
    X.taps = X.dev.alloc(64);
    X.scratch = X.dev.alloc(nf * (d > 1 ? d : 1) + 6 * nf);
    auto* mx = reinterpret_cast<unsigned long long*>(X.dev.alloc(1));
    auto* bad = reinterpret_cast<int*>(X.dev.alloc(1));
    auto* cnt = reinterpret_cast<unsigned long long*>(X.dev.alloc(1));

    // eval_loss (pipeline.cpp:26-34) at phi on grid wm: value, grad (optional)
    auto eval_loss = [&](const double* Fi, const double* Mi, const double* phi, const Meta& wm,
                         bool want_grad) -> double {
        const int64_t n = wm.n();
        k_warp_grad<<<grid_for(n), kNT, 0, stream>>>(Mi, wm, phi, wm, W, want_grad ? G : nullptr);
        X.bump();
        if (cfg->loss == DFM_LOSS_SSD) {
            k_ssd_terms<<<grid_for(n), kNT, 0, stream>>>(Fi, W, G, n, d, cc2,
                                                         want_grad ? grad : nullptr);
            X.bump();
            return X.block_total(cc2, n, part) / static_cast<double>(n);
        }
        const int r = cfg->lncc_radius;
        k_moments<<<grid_for(n), kNT, 0, stream>>>(Fi, W, n, mo);
        X.bump();
        for (int a = 0; a < d; ++a) {  // similarity.cpp:72-77: axes x, y, z of all six images
            k_box_axis<<<grid_for(6 * n), kNT, 0, stream>>>(mo, X.scratch, wm, a, r, 6);
            X.bump();
            ck(cudaMemcpyAsync(mo, X.scratch, sizeof(double) * 6 * n, cudaMemcpyDeviceToDevice,
                               stream),
               "box copy");
        }
        k_lncc_coef<<<grid_for(n), kNT, 0, stream>>>(mo, n, bs, cc2);
        X.bump();
        const double value = -X.block_total(cc2, n, part) / static_cast<double>(n);
        if (want_grad) {
            for (int a = 0; a < d; ++a) {
                k_box_axis<<<grid_for(4 * n), kNT, 0, stream>>>(bs, X.scratch, wm, a, r, 4);
                X.bump();
                ck(cudaMemcpyAsync(bs, X.scratch, sizeof(double) * 4 * n,
                                   cudaMemcpyDeviceToDevice, stream),
                   "box copy");
            }
            k_lncc_grad<<<grid_for(n), kNT, 0, stream>>>(Fi, W, bs, G, n, d, grad);
            X.bump();
        }
        return value;
    };

    Meta cur{};
    bool have = false;
    int64_t t_adam = 0, global = 0;
    for (int si = 0; si < ns; ++si) {
        Meta wm;
        X.downsample(F, full, scales[si], wm, f, tmp);
        X.downsample(M, full, scales[si], wm, mv, tmp);
        const int64_t n = wm.n();
        if (!have) {  // pipeline.cpp:57-79 initial_field
            if (!init || init->kind == DFM_INIT_NONE) {
                ck(cudaMemsetAsync(u, 0, sizeof(double) * n * d, stream), "memset");
            } else if (init->kind == DFM_INIT_AFFINE) {
                if (init->affine_ndim != d)
                    fail(DFM_E_INVALID, "affine_to_working_field: dimensionality mismatch");
                double S[3] = {1.0, 1.0, 1.0};
                for (int a = 0; a < d; ++a) {
                    const int64_t den = wm.d[a] - 1 > 1 ? wm.d[a] - 1 : 1;
                    S[a] = static_cast<double>(full.d[a] - 1) / static_cast<double>(den);
                }
                k_affine_working<<<grid_for(n), kNT, 0, stream>>>(wm, *init, S[0], S[1], S[2], u);
                X.bump();
            } else {
                const Meta im = meta_of(&init->field_grid);
                if (im.ndim != d)
                    fail(DFM_E_INVALID, "register_images: init field dimensionality mismatch");
                if (same_dims(im, wm)) {
                    ck(cudaMemcpyAsync(u, init->field, sizeof(double) * n * d,
                                       cudaMemcpyHostToDevice, stream),
                       "init");
                } else if (same_dims(im, full)) {  // resample_displacement (interp.cpp:447-465)
                    ck(cudaMemcpyAsync(tmp2, init->field, sizeof(double) * nf * d,
                                       cudaMemcpyHostToDevice, stream),
                       "init");
                    X.resample_field(tmp2, im, wm, false, u);
                    double r[3] = {1, 1, 1};
                    for (int a = 0; a < d; ++a)
                        r[a] = static_cast<double>(wm.d[a] - 1) / (im.d[a] - 1);
                    k_scale_comps<<<grid_for(n), kNT, 0, stream>>>(u, n, d, r[0], r[1], r[2]);
                    X.bump();
                } else {
                    fail(DFM_E_INVALID,
                         "register_images: init field must live on the full or coarsest grid");
                }
            }
            ck(cudaMemsetAsync(m, 0, sizeof(double) * n * d, stream), "memset");
            ck(cudaMemsetAsync(nu, 0, sizeof(double) * n * d, stream), "memset");
            have = true;
        } else if (!same_dims(cur, wm)) {  // upsample_field + upsample_state
            X.resample_field(u, cur, wm, true, tmp);
            ck(cudaMemcpyAsync(u, tmp, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, stream),
               "copy");
            X.resample_field(m, cur, wm, true, tmp);
            ck(cudaMemcpyAsync(m, tmp, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, stream),
               "copy");
            X.resample_field(nu, cur, wm, false, tmp);
            double sq[3] = {1, 1, 1};
            for (int a = 0; a < d; ++a) {
                const double r = static_cast<double>(wm.d[a] - 1) / (cur.d[a] - 1);
                sq[a] = r * r;
            }
            k_scale_comps<<<grid_for(n), kNT, 0, stream>>>(tmp, n, d, sq[0], sq[1], sq[2]);
            X.bump();
            ck(cudaMemcpyAsync(nu, tmp, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, stream),
               "copy");
        }
        cur = wm;
        std::vector<double> losses;
        for (int it = 0; it < iters[si]; ++it) {
            for (int a = 0; a < d; ++a)  // loss needs 2r+1 <= dims (similarity.cpp:112-114)
                if (cfg->loss == DFM_LOSS_LNCC && 2 * int64_t(cfg->lncc_radius) + 1 > wm.d[a])
                    fail(DFM_E_INVALID, "lncc_eval: window larger than image");
            const double value = eval_loss(f, mv, u, wm, true);
            if (!std::isfinite(value)) {
                char b[128];
                snprintf(b, sizeof b, "register_images: non-finite loss at scale %f, iteration %d",
                         scales[si], it);
                fail(DFM_E_NUMERICAL, b);
            }
            losses.push_back(value);
            dfm_iter_record rec{};
            rec.scale_index = si;
            rec.scale = scales[si];
            rec.iter = it;
            rec.global_iter = global++;
            rec.loss = value;
            const size_t nl = losses.size();  // pipeline.cpp:45-53 converged
            if (nl >= static_cast<size_t>(cfg->conv_window) + 1) {
                const double prev = losses[nl - 1 - static_cast<size_t>(cfg->conv_window)];
                const double den = std::fabs(prev) > 1e-30 ? std::fabs(prev) : 1e-30;
                if (((prev - value) / cfg->conv_window) / den < cfg->conv_tol) {
                    recs.push_back(rec);
                    break;
                }
            }
            if (cfg->sigma_grad > 0.0) {
                const double s3[3] = {cfg->sigma_grad, cfg->sigma_grad, cfg->sigma_grad};
                X.smooth(grad, wm, d, s3);
            }
            k_eulerian<<<grid_for(n), kNT, 0, stream>>>(grad, u, wm, cfg->use_jac, tmp);
            X.bump();
            ++t_adam;
            const double c1 = 1.0 - std::pow(cfg->beta1, static_cast<double>(t_adam));
            const double c2 = 1.0 - std::pow(cfg->beta2, static_cast<double>(t_adam));
            k_adam<<<grid_for(n * d), kNT, 0, stream>>>(m, nu, tmp, tmp2, n * d, cfg->beta1,
                                                         cfg->beta2, c1, c2, cfg->eps_adam);
            X.bump();
            ck(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), stream), "memset");
            ck(cudaMemsetAsync(bad, 0, sizeof(int), stream), "memset");
            k_step<<<grid_for(n * d), kNT, 0, stream>>>(tmp2, n * d, cfg->eta, cfg->step_cap,
                                                        grad, mx, bad);
            X.bump();
            unsigned long long hmx = 0;
            int hbad = 0;
            ck(cudaMemcpyAsync(&hmx, mx, sizeof(hmx), cudaMemcpyDeviceToHost, stream), "mx");
            ck(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, stream), "bad");
            ck(cudaStreamSynchronize(stream), "step sync");
            std::memcpy(&rec.max_step, &hmx, sizeof(double));
            if (hbad) fail(DFM_E_NUMERICAL, "apply_update: non-finite step");
            k_compose<<<grid_for(n), kNT, 0, stream>>>(u, grad, wm, tmp);
            X.bump();
            if (cfg->sigma_warp > 0.0) {
                const double s3[3] = {cfg->sigma_warp, cfg->sigma_warp, cfg->sigma_warp};
                X.smooth(tmp, wm, d, s3);
            }
            ck(cudaMemcpyAsync(u, tmp, sizeof(double) * n * d, cudaMemcpyDeviceToDevice, stream),
               "copy");
            recs.push_back(rec);
        }
    }
    if (!same_dims(cur, full)) {
        X.resample_field(u, cur, full, true, tmp);
        ck(cudaMemcpyAsync(u, tmp, sizeof(double) * nf * d, cudaMemcpyDeviceToDevice, stream),
           "copy");
    }
    *final_loss = eval_loss(F, M, u, full, false);
    ck(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), stream), "memset");
    k_fold_count<<<grid_for(nf), kNT, 0, stream>>>(u, full, cnt);
    X.bump();
    unsigned long long hc = 0;
    ck(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, stream), "count");
    ck(cudaMemcpyAsync(d_field_aos, u, sizeof(double) * nf * d, cudaMemcpyDeviceToDevice, stream),
       "field");
    ck(cudaStreamSynchronize(stream), "final sync");
    *sing = static_cast<double>(hc) / static_cast<double>(nf);
}

// status-returning wrapper for engine.cu (its own error type stays local)
int exact_register_status(cudaStream_t stream, int64_t* launches, const dfm_grid* g,
                          const double* F, const double* M, const dfm_config* cfg,
                          const double* scales, const int32_t* iters, int ns,
                          const dfm_init* init, double* d_field_aos,
                          std::vector<dfm_iter_record>& recs, double* final_loss, double* sing,
                          std::string& msg) {
    try {
        exact_register(stream, launches, g, F, M, cfg, scales, iters, ns, init, d_field_aos, recs,
                       final_loss, sing);
        return DFM_OK;
    } catch (const exact::Fail& e) {
        msg = e.msg;
        return e.code;
    }
}

}  // namespace dfm
