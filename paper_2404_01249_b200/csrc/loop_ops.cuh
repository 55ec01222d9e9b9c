// loop_ops.cuh — per-voxel math of the hot loop shared by the plane-streaming
// (kernels_tma.cu) and brick (kernels_brick.cu) kernel families, plus the
// CTA reductions and the fused convergence-monitor tail.  Keeping one copy of
// the arithmetic means both tilings compute identical values per voxel.
#pragma once

#include <cstdint>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"

namespace dfm {

struct Red2 {
    double sum;
    double mx;
};

// ---------------------------------------------------------------------------
// CTA reductions (fixed order: warp shuffles, then warp 0 over the warp sums)
template <int NTH>
__device__ double bsum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = 0.0;
    if (w == 0) {
        v = l < NTH / 32 ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    __syncthreads();
    return v;
}

template <int NTH>
__device__ double bmax(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = 0.0;
    if (w == 0) {
        v = l < NTH / 32 ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;
}

// Fused loss + convergence monitor tail: every CTA has written its partial;
// the last CTA to arrive sums all partials in fixed order (deterministic) and
// runs monitor_commit (pipeline.cpp:157-179) on sign * sum / nvox (LNCC -1,
// SSD +1).  nvox = global voxel count.
template <int NTH>
__device__ void monitor_tail(const MonitorArgs& mon, const double* partials, int nb, double nvox,
                             double* s_red, double sign = -1.0) {
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&mon.st->arrive, 1u) == static_cast<unsigned>(nb - 1);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        double acc = 0.0;
        for (int k = threadIdx.x; k < nb; k += NTH) acc += __ldcg(partials + k);
        const double tot = bsum<NTH>(acc, s_red);
        if (threadIdx.x == 0) {
            mon.st->arrive = 0;
            monitor_commit(mon.st, sign * tot / nvox, 0.0, 0.0, mon.loss, mon.stamp,
                           mon.window, mon.tol);
        }
    }
}

// ---------------------------------------------------------------------------
// LNCC window coefficients from the five box moments s = (ΣF, ΣW, ΣF², ΣW², ΣFW)
// over a clipped window of n voxels (similarity.cpp:145-162), with 2 divisions
// instead of 12: 1/n and 1/(vF vW).  Returns cc² (the loss term).
struct LnccCoef {
    double cc2, an, amu, bn, bmu;
};

// The fixed image's window statistics (similarity.cpp:145-150, F half),
// given inv_n = 1 / (clipped window size):
// constant over the iterations of a pyramid level, so computable once per
// level.  Products and differences are explicit (no FMA contraction) so the
// split and the fused forms below round identically.
__device__ __forceinline__ void lncc_fstats(double sF, double sF2, double inv_n, double& muF,
                                            double& vF) {
    muF = __dmul_rn(sF, inv_n);
    vF = __dsub_rn(__dmul_rn(sF2, inv_n), __dmul_rn(muF, muF));
    vF = vF < 0.0 ? 0.0 : vF;
}

// window coefficients given the F statistics and the three W moments
// (ΣW, ΣW², ΣFW)
__device__ __forceinline__ LnccCoef lncc_coef_f(double muF, double vF, double sW, double sW2,
                                                double sFW, double inv_n) {
    LnccCoef r{0.0, 0.0, 0.0, 0.0, 0.0};
    const double muW = __dmul_rn(sW, inv_n);
    double vW = __dsub_rn(__dmul_rn(sW2, inv_n), __dmul_rn(muW, muW));
    vW = vW < 0.0 ? 0.0 : vW;
    const double cv = __dsub_rn(__dmul_rn(sFW, inv_n), __dmul_rn(muF, muW));
    if (!(vF < 1e-5 || vW < 1e-5)) {  // similarity.cpp:13, 151-154
        const double inv_den = 1.0 / (vF * vW);
        const double alpha = cv * inv_den;         // cv / (vF vW)
        r.cc2 = alpha * cv;                        // cv^2 / (vF vW)
        const double beta = r.cc2 * vF * inv_den;  // cv^2 / (vF vW^2)
        r.an = alpha * inv_n;
        r.amu = r.an * muF;
        r.bn = beta * inv_n;
        r.bmu = r.bn * muW;
    }
    return r;
}

// from the five raw moments: the same two steps, hence bit-identical to the
// precomputed-F form
__device__ __forceinline__ LnccCoef lncc_coef(const double s[5], double inv_n) {
    double muF, vF;
    lncc_fstats(s[0], s[2], inv_n, muF, vF);
    return lncc_coef_f(muF, vF, s[1], s[3], s[4], inv_n);
}

// 1 / (clipped window size) at voxel (x, y, z local; zoff/gnz from the view):
// interior voxels take the compile-time constant (the same correctly rounded
// value a division would give), border voxels divide
template <int R>
__device__ __forceinline__ double window_inv(int x, int y, int z, const Dims& d) {
    constexpr double K = 2 * R + 1;
    const int gz = d.gz(), zg = z + d.zoff;
    const bool three = gz > 1;
    // R <= i < n - R as one unsigned compare per axis (bounds are loop-invariant)
    if (static_cast<unsigned>(x - R) < static_cast<unsigned>(max(d.nx - 2 * R, 0)) &&
        static_cast<unsigned>(y - R) < static_cast<unsigned>(max(d.ny - 2 * R, 0)) &&
        (!three || static_cast<unsigned>(zg - R) < static_cast<unsigned>(max(gz - 2 * R, 0))))
        return three ? 1.0 / (K * K * K) : 1.0 / (K * K);
    const double n = static_cast<double>(box_len(x, d.nx, R) * box_len(y, d.ny, R) *
                                         (three ? box_len(zg, gz, R) : 1));
    return 1.0 / n;
}

// Box sums of the 4 LNCC coefficients in the backward: fp64 (0, default) or
// fp32 (1, fp32 context only; A/B builds).  fp32 sums cancel: dW combines
// F*S[an] - S[amu] - W*S[bn] + S[bmu], and at 160x192x224 the fp32-summed
// gradient misses the per-kernel criterion (1e-5 relative + 1e-6 of peak) by
// up to 2.3x on 167 of 20.6M components; fp64 sums of the same fp32-stored
// coefficients stay within 0.2 of it (tests/test_fullsize_parity_gpu.py).
#ifndef DFM_BWD_ACC32
#define DFM_BWD_ACC32 0
#endif

// dL/dW at one voxel from the box sums of the 4 coefficients (similarity.cpp:182)
__device__ __forceinline__ double lncc_dw(double m2n, double f, double w, const double s[4]) {
    return m2n * (f * s[0] - s[1] - w * s[2] + s[3]);
}

// ---------------------------------------------------------------------------
// Adam division / square root: fp32 uses the MUFU approximations (<= 2 ulp;
// the fp32 path is held to 1e-5 relative), fp64 the IEEE operations.
__device__ __forceinline__ float adam_div(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double adam_div(double a, double b) { return a / b; }
__device__ __forceinline__ float adam_sqrt(float a) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ double adam_sqrt(double a) { return sqrt(a); }

// Adam constants of one launch (optim.cpp:22-42, diffeo.cpp:47-57)
template <class T>
struct AdamK {
    T b1, omb1, b2, omb2, eps, eta, cap;
};

template <class T>
inline AdamK<T> adam_k(const AdamParams& ap) {
    return AdamK<T>{T(ap.b1), T(1.0 - ap.b1), T(ap.b2), T(1.0 - ap.b2),
                    T(ap.eps), T(ap.eta),     T(ap.cap)};
}

// One component: v = -smoothed grad (diffeo.cpp:17-24); m, nu updated in
// place; returns the capped step; sets bad on a non-finite step.
template <class T>
__device__ __forceinline__ T adam_component(const AdamK<T>& k, T g, T& m, T& nu, T ic1, T ic2,
                                            bool& bad) {
    const T v = -g;
    m = k.b1 * m + k.omb1 * v;
    nu = k.b2 * nu + k.omb2 * v * v;
    const T dir = adam_div(m * ic1, adam_sqrt(nu * ic2) + k.eps);  // (m/c1)/(sqrt(nu/c2)+eps)
    const T sv = k.eta * dir;
    bad |= !isfinite(sv);
    return fmin(fmax(sv, -k.cap), k.cap);
}

// ---------------------------------------------------------------------------
// compose at one voxel (interp.cpp:269-289 with psi = step): the composed
// value step + u(x + step), u read from global memory (3 packed planes of the
// volume view d; zg = global z of the voxel).  Same arithmetic as the staged
// compose of kernels_tma.cu (Compose2::stage / stage_point) so both give
// bit-identical values; CAPH bounds |step| (cap <= CAPH - 0.5).
// the 8 corner values of each component and the weights, fetched at one
// plane and combined at the next (the gathers' latency hides behind a plane)
template <class T>
struct ComposeCarry {
    bool valid;
    int64_t i;
    T s[3];
    T fx, fy, fz;
    T a[3][8];
};

template <class T, int CAPH>
__device__ __forceinline__ void compose_fetch(const T* __restrict__ u, const Dims& d, int x,
                                              int y, int zg, const T s[3], int64_t i,
                                              ComposeCarry<T>& c) {
    const int64_t n = d.n;
    const int gz = d.gz();
    // one clamped cell search for every voxel (equal to the unclamped one
    // where nothing clamps): no divergent interior/border split in a warp
    const AxisCell<T> ax = locate_axis(x, s[0], d.nx);
    const AxisCell<T> ay = locate_axis(y, s[1], d.ny);
    const AxisCell<T> az = locate_axis(zg, s[2], gz);
    const int ix = ax.i0, iy = ay.i0, iz = az.i0;
    c.fx = ax.f;
    c.fy = ay.f;
    c.fz = az.f;
    const int sy = d.nx;
    const int64_t sz = static_cast<int64_t>(d.nx) * d.ny;
    const int64_t base = (static_cast<int64_t>(iz - d.zoff) * d.ny + iy) * d.nx + ix;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T* a = u + k * n + base;
        c.a[k][0] = a[0];
        c.a[k][1] = a[1];
        c.a[k][2] = a[sy];
        c.a[k][3] = a[sy + 1];
        c.a[k][4] = a[sz];
        c.a[k][5] = a[sz + 1];
        c.a[k][6] = a[sz + sy];
        c.a[k][7] = a[sz + sy + 1];
        c.s[k] = s[k];
    }
    c.i = i;
    c.valid = true;
}

// trilinear combination of the 8 corners, as explicit fma chains: every
// compose path (fused, folded, split, brick, register or cp.async gather)
// rounds identically whatever the compiler would contract around it
template <class T>
__device__ __forceinline__ T bilerp4(T w00, T w10, T w01, T w11, T a0, T a1, T a2, T a3) {
    T r = mul_rn(w00, a0);
    r = fma(w10, a1, r);
    r = fma(w01, a2, r);
    return fma(w11, a3, r);
}
template <class T>
__device__ __forceinline__ T zlerp(T wz0, T lo, T wz1, T hi) {
    return fma(wz0, lo, mul_rn(wz1, hi));
}

template <class T>
__device__ __forceinline__ void compose_finish(const ComposeCarry<T>& c, T out[3]) {
    const T wx0 = T(1) - c.fx, wy0 = T(1) - c.fy, wz0 = T(1) - c.fz;
    const T w00 = wx0 * wy0, w10 = c.fx * wy0, w01 = wx0 * c.fy, w11 = c.fx * c.fy;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T* a = c.a[k];
        const T lo = bilerp4(w00, w10, w01, w11, a[0], a[1], a[2], a[3]);
        const T hi = bilerp4(w00, w10, w01, w11, a[4], a[5], a[6], a[7]);
        out[k] = c.s[k] + zlerp(wz0, lo, c.fz, hi);
    }
}

// the same compose with the 24 corner values gathered by cp.async into
// shared memory (buf[(k * 8 + j) * ss], k component, j corner): the carry
// holds 7 values instead of 30 registers of loads in flight
template <class T>
struct ComposeCarryA {
    bool valid;
    int slot;
    int64_t i;
    T s[3];
    T fx, fy, fz;
};

template <class T, int CAPH>
__device__ __forceinline__ void compose_fetch_async(const T* const* u, const Dims& d, int x,
                                                    int y, int zg, const T s[3], int64_t i,
                                                    ComposeCarryA<T>& c, T* buf, int ss) {
    const int gz = d.gz();
    // one clamped cell search for every voxel (equal to the unclamped one
    // where nothing clamps): no divergent interior/border split in a warp
    const AxisCell<T> ax = locate_axis(x, s[0], d.nx);
    const AxisCell<T> ay = locate_axis(y, s[1], d.ny);
    const AxisCell<T> az = locate_axis(zg, s[2], gz);
    const int ix = ax.i0, iy = ay.i0, iz = az.i0;
    c.fx = ax.f;
    c.fy = ay.f;
    c.fz = az.f;
    const int sy = d.nx;
    const int64_t sz = static_cast<int64_t>(d.nx) * d.ny;
    const int64_t base = (static_cast<int64_t>(iz - d.zoff) * d.ny + iy) * d.nx + ix;
    const int64_t off[8] = {0, 1, sy, sy + 1, sz, sz + 1, sz + sy, sz + sy + 1};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T* a = u[k] + base;
#pragma unroll
        for (int j = 0; j < 8; ++j) cp_async<int(sizeof(T))>(buf + (k * 8 + j) * ss, a + off[j]);
        c.s[k] = s[k];
    }
    cp_async_commit();
    c.i = i;
    c.valid = true;
}

// after cp_async_wait_all()
template <class T>
__device__ __forceinline__ void compose_finish_async(const ComposeCarryA<T>& c, const T* buf,
                                                     int ss, T out[3]) {
    const T wx0 = T(1) - c.fx, wy0 = T(1) - c.fy, wz0 = T(1) - c.fz;
    const T w00 = wx0 * wy0, w10 = c.fx * wy0, w01 = wx0 * c.fy, w11 = c.fx * c.fy;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T* a = buf + k * 8 * ss;
        const T lo = bilerp4(w00, w10, w01, w11, a[0], a[ss], a[2 * ss], a[3 * ss]);
        const T hi = bilerp4(w00, w10, w01, w11, a[4 * ss], a[5 * ss], a[6 * ss], a[7 * ss]);
        out[k] = c.s[k] + zlerp(wz0, lo, c.fz, hi);
    }
}

template <class T, int CAPH>
__device__ __forceinline__ void compose_at(const T* __restrict__ u, const Dims& d, int x, int y,
                                           int zg, const T s[3], T out[3]) {
    ComposeCarry<T> c;
    compose_fetch<T, CAPH>(u, d, x, y, zg, s, 0, c);
    compose_finish(c, out);
}

}  // namespace dfm
