// dfm_device.cuh — device-side building blocks shared by every kernel.
//
// Layout in HBM: every scalar volume is one
// x-fastest plane array of T (float or double); every vector field is three
// such arrays (SoA: x-, y-, z-component planes), so a warp reading 32
// consecutive voxels of one component issues one 128 B (fp32) transaction.
// 2-D grids are 3-D grids with nz == 1 and a zero z component.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include "tma_util.cuh"

namespace dfm {

struct Dims {
    int nx, ny, nz;  // nz == 1 for 2-D grids
    int ndim;
    int64_t n;       // nx*ny*nz
    // z-slab view (all 0 for a whole volume): local plane 0 is global plane
    // zoff of a volume with gnz planes; kernels produce local planes [zb, ze).
    int zoff = 0, gnz = 0, zb = 0, ze = 0;
    __host__ __device__ int gz() const { return gnz ? gnz : nz; }
    __host__ __device__ int out_begin() const { return zb; }
    __host__ __device__ int out_end() const { return ze ? ze : nz; }
    __host__ __device__ int64_t idx(int x, int y, int z) const {
        return (static_cast<int64_t>(z) * ny + y) * nx + x;
    }
    // 32-bit index math (volumes are validated to < 2^31 voxels)
    __host__ __device__ int idx32(int x, int y, int z) const { return (z * ny + y) * nx + x; }
    __host__ __device__ bool is3d() const { return nz > 1; }
};

// Programmatic dependent launch (sm_90+): a kernel launched with
// programmatic stream serialization may start while its predecessor drains;
// pdl_wait() blocks until the predecessor grid has completed and its writes
// are visible (a no-op for a normally launched kernel); pdl_trigger() lets the
// successor's CTAs be scheduled once every CTA of this grid has issued it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class T>
struct Planes3 {  // SoA vector field
    T* c[3];
};

template <class T>
struct CPlanes3 {
    const T* c[3];
};

// ---------------------------------------------------------------------------
// Trilinear interpolation with clamp-to-edge, the reference's `locate`
// (interp.cpp:19-37): p clamped to [0, n-1]; lower node clamped to [0, n-2];
// `clamped` marks points that were outside [0, n-1] (zero gradient there,
// interp.cpp:171-173).
//
// fp64 follows the reference formulation (p = x + u in double, floor).  fp32
// splits the sample position into integer x + floor(u) and the exact fraction
// u - floor(u), so the fp32 cell decision is the exact real-number one
// (SURVEY.md §7 hard part 2) instead of rounding x + u first.
template <class T>
struct AxisCell {
    int i0;
    T f;
    bool clamped;
};

// kFlat = false: the caller guarantees n >= 2 (no flat-axis branch)
template <bool kFlat = true>
__device__ __forceinline__ AxisCell<double> locate_axis(int xi, double u, int n) {
    AxisCell<double> c;
    if (kFlat && n == 1) {
        c.i0 = 0;
        c.f = 0.0;
        c.clamped = false;
        return c;
    }
    double p = static_cast<double>(xi) + u;
    const double hi = static_cast<double>(n - 1);
    c.clamped = (p < 0.0 || p > hi);
    p = p < 0.0 ? 0.0 : (hi < p ? hi : p);
    double fl = floor(p);
    int i = (fl == fl) ? static_cast<int>(fl) : 0;  // NaN -> 0 like the cast
    i = i < 0 ? 0 : (i > n - 2 ? n - 2 : i);
    c.i0 = i;
    c.f = p - static_cast<double>(i);
    return c;
}

template <bool kFlat = true>
__device__ __forceinline__ AxisCell<float> locate_axis(int xi, float u, int n) {
    AxisCell<float> c;
    if (kFlat && n == 1) {
        c.i0 = 0;
        c.f = 0.f;
        c.clamped = false;
        return c;
    }
    float fl = floorf(u);
    const float fr = u - fl;  // exact
    fl = fminf(fmaxf(fl, -1.0e9f), 1.0e9f);
    const int i = xi + static_cast<int>(fl);
    if (i < 0) {
        c.clamped = true;
        c.i0 = 0;
        c.f = 0.f;
    } else if (i >= n - 1) {
        c.clamped = (i > n - 1) || (fr > 0.f);
        c.i0 = n - 2;
        c.f = 1.f;
    } else {
        c.clamped = false;
        c.i0 = i;
        c.f = fr;
    }
    return c;
}

template <class T>
struct Cell3 {
    int64_t base;  // index of the lower corner
    int sx, sy;    // +x / +y corner offsets (0 on flat axes)
    int64_t sz;    // +z corner offset (0 for 2-D)
    T fx, fy, fz;
    bool clx, cly, clz;
    bool three;
};

// The three axes of a 3-D gather cell at once.  fp32 fast path
// (DFM_LOCATE_FAST): when all three lower corners are strictly inside
// [0, n-2] nothing clamps and locate_axis would return (i, u - floor(u),
// false) — the same values without its border selects; otherwise (borders,
// flat axes, huge or NaN displacements) the general per-axis search.
#ifndef DFM_LOCATE_FAST
#define DFM_LOCATE_FAST 1
#endif
template <class T, bool kFlat = true>
__device__ __forceinline__ void locate_cells3(int x, int y, int z, T ux, T uy, T uz, int nx,
                                              int ny, int nz, AxisCell<T>& ax, AxisCell<T>& ay,
                                              AxisCell<T>& az) {
    if constexpr (DFM_LOCATE_FAST != 0 && sizeof(T) == 4) {
        const float flx = floorf(ux), fly = floorf(uy), flz = floorf(uz);
        const int ix = x + static_cast<int>(fminf(fmaxf(flx, -1.0e9f), 1.0e9f));
        const int iy = y + static_cast<int>(fminf(fmaxf(fly, -1.0e9f), 1.0e9f));
        const int iz = z + static_cast<int>(fminf(fmaxf(flz, -1.0e9f), 1.0e9f));
        if (static_cast<unsigned>(ix) < static_cast<unsigned>(nx - 1) &&
            static_cast<unsigned>(iy) < static_cast<unsigned>(ny - 1) &&
            static_cast<unsigned>(iz) < static_cast<unsigned>(nz - 1)) {
            ax.i0 = ix, ax.f = ux - flx, ax.clamped = false;
            ay.i0 = iy, ay.f = uy - fly, ay.clamped = false;
            az.i0 = iz, az.f = uz - flz, az.clamped = false;
            return;
        }
    }
    ax = locate_axis<kFlat>(x, ux, nx);
    ay = locate_axis<kFlat>(y, uy, ny);
    az = locate_axis<kFlat>(z, uz, nz);
}

template <class T>
__device__ __forceinline__ Cell3<T> locate3(const Dims& m, int x, int y, int z, T ux, T uy,
                                            T uz) {
    Cell3<T> c;
    const AxisCell<T> ax = locate_axis(x, ux, m.nx);
    const AxisCell<T> ay = locate_axis(y, uy, m.ny);
    c.three = m.nz > 1;
    AxisCell<T> az;
    if (c.three) {
        az = locate_axis(z, uz, m.nz);
    } else {
        az.i0 = 0;
        az.f = T(0);
        az.clamped = false;
    }
    c.fx = ax.f;
    c.fy = ay.f;
    c.fz = az.f;
    c.clx = ax.clamped;
    c.cly = ay.clamped;
    c.clz = az.clamped;
    c.sx = m.nx > 1 ? 1 : 0;
    c.sy = m.ny > 1 ? m.nx : 0;
    c.sz = c.three ? static_cast<int64_t>(m.nx) * m.ny : 0;
    c.base = m.idx(ax.i0, ay.i0, az.i0);
    return c;
}

// Sample point given as grid coordinate (x,y,z) of a voxel of the FIXED grid
// plus displacement u — the only form the hot path needs.
template <class T>
struct Corners {
    T v[8];  // order (cz, cy, cx) as in interp.cpp:159-162
};

// NC = true reads through the non-coherent (read-only) path: only for data
// that no thread writes during the kernel.
template <class S, bool NC>
__device__ __forceinline__ S ld_(const S* p) {
    if constexpr (NC) return __ldg(p);
    else return *p;
}

template <class T, class S, bool NC = true>
__device__ __forceinline__ Corners<T> fetch_corners(const S* __restrict__ img, const Cell3<T>& c) {
    Corners<T> k;
    const S* p = img + c.base;
    k.v[0] = static_cast<T>(ld_<S, NC>(p));
    k.v[1] = static_cast<T>(ld_<S, NC>(p + c.sx));
    k.v[2] = static_cast<T>(ld_<S, NC>(p + c.sy));
    k.v[3] = static_cast<T>(ld_<S, NC>(p + c.sy + c.sx));
    if (c.three) {
        k.v[4] = static_cast<T>(ld_<S, NC>(p + c.sz));
        k.v[5] = static_cast<T>(ld_<S, NC>(p + c.sz + c.sx));
        k.v[6] = static_cast<T>(ld_<S, NC>(p + c.sz + c.sy));
        k.v[7] = static_cast<T>(ld_<S, NC>(p + c.sz + c.sy + c.sx));
    } else {
        k.v[4] = k.v[5] = k.v[6] = k.v[7] = T(0);
    }
    return k;
}

// value (interp.cpp:155-164)
template <class T>
__device__ __forceinline__ T lerp_value(const Cell3<T>& c, const Corners<T>& k) {
    const T wx0 = T(1) - c.fx, wx1 = c.fx;
    const T wy0 = T(1) - c.fy, wy1 = c.fy;
    const T wz0 = T(1) - c.fz, wz1 = c.fz;
    T acc = (wx0 * wy0 * wz0) * k.v[0] + (wx1 * wy0 * wz0) * k.v[1] +
            (wx0 * wy1 * wz0) * k.v[2] + (wx1 * wy1 * wz0) * k.v[3];
    if (c.three)
        acc += (wx0 * wy0 * wz1) * k.v[4] + (wx1 * wy0 * wz1) * k.v[5] +
               (wx0 * wy1 * wz1) * k.v[6] + (wx1 * wy1 * wz1) * k.v[7];
    return acc;
}

// exact interpolant gradient (interp.cpp:166-186); zero on clamped/flat axes
template <class T>
__device__ __forceinline__ void lerp_grad(const Cell3<T>& c, const Corners<T>& k, int ndim,
                                          T g[3]) {
    const T wx0 = T(1) - c.fx, wx1 = c.fx;
    const T wy0 = T(1) - c.fy, wy1 = c.fy;
    const T wz0 = T(1) - c.fz, wz1 = c.fz;
    g[0] = g[1] = g[2] = T(0);
    if (!c.clx && c.sx) {
        T a = (wy0 * wz0) * (k.v[1] - k.v[0]) + (wy1 * wz0) * (k.v[3] - k.v[2]);
        if (c.three) a += (wy0 * wz1) * (k.v[5] - k.v[4]) + (wy1 * wz1) * (k.v[7] - k.v[6]);
        g[0] = a;
    }
    if (!c.cly && c.sy) {
        T a = (wx0 * wz0) * (k.v[2] - k.v[0]) + (wx1 * wz0) * (k.v[3] - k.v[1]);
        if (c.three) a += (wx0 * wz1) * (k.v[6] - k.v[4]) + (wx1 * wz1) * (k.v[7] - k.v[5]);
        g[1] = a;
    }
    if (ndim == 3 && c.three && !c.clz) {
        g[2] = (wx0 * wy0) * (k.v[4] - k.v[0]) + (wx1 * wy0) * (k.v[5] - k.v[1]) +
               (wx0 * wy1) * (k.v[6] - k.v[2]) + (wx1 * wy1) * (k.v[7] - k.v[3]);
    }
}

// ---------------------------------------------------------------------------
// 3-D fast form of warp_with_gradient at one voxel (similarity.cpp:25-45):
// all dims >= 2 (validate_meta), 32-bit offsets, no flat-axis cases.  Same
// arithmetic as locate3 + lerp_value + lerp_grad, in fewer instructions.
template <class T>
struct WG3 {
    int base;       // lower corner index
    T fx, fy, fz;
    unsigned clamp;  // bit a: axis a clamped (zero gradient)
    T v[8];          // corners in (cz, cy, cx) order
};

template <class T, bool NC = true, bool kFlat = true>
__device__ __forceinline__ void wg3_fetch(const T* __restrict__ M, const Dims& m, int x, int y,
                                          int z, T ux, T uy, T uz, WG3<T>& w) {
    AxisCell<T> ax, ay, az;
    locate_cells3<T, kFlat>(x, y, z, ux, uy, uz, m.nx, m.ny, m.nz, ax, ay, az);
    w.fx = ax.f;
    w.fy = ay.f;
    w.fz = az.f;
    w.clamp = (ax.clamped ? 1u : 0u) | (ay.clamped ? 2u : 0u) | (az.clamped ? 4u : 0u);
    const int sy = m.nx, sz = m.nx * m.ny;
    w.base = (az.i0 * m.ny + ay.i0) * m.nx + ax.i0;
    const T* p = M + w.base;
    w.v[0] = ld_<T, NC>(p);
    w.v[1] = ld_<T, NC>(p + 1);
    w.v[2] = ld_<T, NC>(p + sy);
    w.v[3] = ld_<T, NC>(p + sy + 1);
    w.v[4] = ld_<T, NC>(p + sz);
    w.v[5] = ld_<T, NC>(p + sz + 1);
    w.v[6] = ld_<T, NC>(p + sz + sy);
    w.v[7] = ld_<T, NC>(p + sz + sy + 1);
}

// the same gather issued as cp.async copies of the 8 corners into s[k * ss]
// (shared memory); wg3_load pulls them into w.v once cp_async_wait_all() ran
template <class T, bool kFlat = true>
__device__ __forceinline__ void wg3_fetch_async(const T* __restrict__ M, const Dims& m, int x,
                                                int y, int z, T ux, T uy, T uz, WG3<T>& w,
                                                T* s, int ss) {
    AxisCell<T> ax, ay, az;
    locate_cells3<T, kFlat>(x, y, z, ux, uy, uz, m.nx, m.ny, m.nz, ax, ay, az);
    w.fx = ax.f;
    w.fy = ay.f;
    w.fz = az.f;
    w.clamp = (ax.clamped ? 1u : 0u) | (ay.clamped ? 2u : 0u) | (az.clamped ? 4u : 0u);
    const int sy = m.nx, sz = m.nx * m.ny;
    w.base = (az.i0 * m.ny + ay.i0) * m.nx + ax.i0;
    const T* p = M + w.base;
    const int off[8] = {0, 1, sy, sy + 1, sz, sz + 1, sz + sy, sz + sy + 1};
    const uint32_t sa = smem_u32(s);
#pragma unroll
    for (int k = 0; k < 8; ++k)  // one generic->shared conversion for the 8 copies
        cp_async_u32<int(sizeof(T))>(sa + k * ss * int(sizeof(T)), p + off[k]);
    cp_async_commit();
}

template <class T>
__device__ __forceinline__ void wg3_load(WG3<T>& w, const T* s, int ss) {
#pragma unroll
    for (int k = 0; k < 8; ++k) w.v[k] = s[k * ss];
}

// The 8-corner sums below are written as explicit fma chains: left to the
// compiler, mul+add contraction depends on the surrounding code, and the
// gather's kernels (fused, split, brick, streamed, synchronous or cp.async
// gather) must round identically.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <class T>
__device__ __forceinline__ T wg3_value(const WG3<T>& w) {
    const T wx0 = T(1) - w.fx, wx1 = w.fx;
    const T wy0 = T(1) - w.fy, wy1 = w.fy;
    const T wz0 = T(1) - w.fz, wz1 = w.fz;
    const T a00 = mul_rn(wy0, wz0), a10 = mul_rn(wy1, wz0), a01 = mul_rn(wy0, wz1),
            a11 = mul_rn(wy1, wz1);
    T acc = mul_rn(mul_rn(wx0, a00), w.v[0]);
    acc = fma(mul_rn(wx1, a00), w.v[1], acc);
    acc = fma(mul_rn(wx0, a10), w.v[2], acc);
    acc = fma(mul_rn(wx1, a10), w.v[3], acc);
    acc = fma(mul_rn(wx0, a01), w.v[4], acc);
    acc = fma(mul_rn(wx1, a01), w.v[5], acc);
    acc = fma(mul_rn(wx0, a11), w.v[6], acc);
    acc = fma(mul_rn(wx1, a11), w.v[7], acc);
    return acc;
}

template <class T>
__device__ __forceinline__ void wg3_grad(const WG3<T>& w, T g[3]) {
    const T wx0 = T(1) - w.fx, wx1 = w.fx;
    const T wy0 = T(1) - w.fy, wy1 = w.fy;
    const T wz0 = T(1) - w.fz, wz1 = w.fz;
    const T* k = w.v;
    T a = mul_rn(mul_rn(wy0, wz0), k[1] - k[0]);
    a = fma(mul_rn(wy1, wz0), k[3] - k[2], a);
    a = fma(mul_rn(wy0, wz1), k[5] - k[4], a);
    a = fma(mul_rn(wy1, wz1), k[7] - k[6], a);
    g[0] = (w.clamp & 1u) ? T(0) : a;
    T b = mul_rn(mul_rn(wx0, wz0), k[2] - k[0]);
    b = fma(mul_rn(wx1, wz0), k[3] - k[1], b);
    b = fma(mul_rn(wx0, wz1), k[6] - k[4], b);
    b = fma(mul_rn(wx1, wz1), k[7] - k[5], b);
    g[1] = (w.clamp & 2u) ? T(0) : b;
    T c = mul_rn(mul_rn(wx0, wy0), k[4] - k[0]);
    c = fma(mul_rn(wx1, wy0), k[5] - k[1], c);
    c = fma(mul_rn(wx0, wy1), k[6] - k[2], c);
    c = fma(mul_rn(wx1, wy1), k[7] - k[3], c);
    g[2] = (w.clamp & 4u) ? T(0) : c;
}

// per-component field sample (interp.cpp:188-203)
template <class T, bool NC = true>
__device__ __forceinline__ void lerp_field(const Cell3<T>& c, const T* __restrict__ f0,
                                           const T* __restrict__ f1, const T* __restrict__ f2,
                                           int ndim, T out[3]) {
    Corners<T> k = fetch_corners<T, T, NC>(f0, c);
    out[0] = lerp_value(c, k);
    k = fetch_corners<T, T, NC>(f1, c);
    out[1] = lerp_value(c, k);
    if (ndim == 3) {
        k = fetch_corners<T, T, NC>(f2, c);
        out[2] = lerp_value(c, k);
    } else {
        out[2] = T(0);
    }
}

// clipped box-window length along one axis: |[i-r, i+r] ∩ [0, n-1]|
__device__ __forceinline__ int box_len(int i, int n, int r) {
    const int lo = i - r < 0 ? 0 : i - r;
    const int hi = i + r > n - 1 ? n - 1 : i + r;
    return hi - lo + 1;
}

template <class T>
__device__ __forceinline__ bool finite_(T v) {
    return isfinite(v);
}

// non-negative float/double -> monotone unsigned key for atomicMax
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
    atomicMax(slot, static_cast<unsigned long long>(__double_as_longlong(v)));
}

// jacobian (interp.cpp:291-328) at one voxel: J[c][a] = du_c/dx_a + delta
template <class T>
__device__ __forceinline__ void jacobian_at(CPlanes3<T> u, const Dims& d, int x, int y, int z,
                                            T J[9]) {
    // boundary decisions in global coordinates (z-slab views carry halos)
    const int pos[3] = {x, y, z + d.zoff};
    const int n[3] = {d.nx, d.ny, d.gz()};
    const int64_t stride[3] = {1, d.nx, static_cast<int64_t>(d.nx) * d.ny};
    const int64_t i = d.idx(x, y, z);
    for (int k = 0; k < 9; ++k) J[k] = T(0);
    for (int a = 0; a < d.ndim; ++a) {
        int64_t lo, hi;
        T scale;  // 1/den: x / 2 == x * 0.5 exactly, x / 1 == x
        if (pos[a] == 0) {
            lo = i;
            hi = i + stride[a];
            scale = T(1);
        } else if (pos[a] == n[a] - 1) {
            lo = i - stride[a];
            hi = i;
            scale = T(1);
        } else {
            lo = i - stride[a];
            hi = i + stride[a];
            scale = T(0.5);
        }
        for (int c = 0; c < d.ndim; ++c)
            J[c * d.ndim + a] =
                (__ldg(u.c[c] + hi) - __ldg(u.c[c] + lo)) * scale + (c == a ? T(1) : T(0));
    }
}

// the same for a 3-D grid with compile-time indices (J stays in registers)
template <class T>
__device__ __forceinline__ void jacobian_at3(CPlanes3<T> u, const Dims& d, int x, int y, int z,
                                             T J[9]) {
    const int pos[3] = {x, y, z + d.zoff};
    const int n[3] = {d.nx, d.ny, d.gz()};
    const int64_t stride[3] = {1, d.nx, static_cast<int64_t>(d.nx) * d.ny};
    const int64_t i = d.idx(x, y, z);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int64_t lo = i - stride[a], hi = i + stride[a];
        T scale = T(0.5);
        if (pos[a] == 0) {
            lo = i;
            scale = T(1);
        } else if (pos[a] == n[a] - 1) {
            hi = i;
            scale = T(1);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c)
            J[c * 3 + a] =
                (__ldg(u.c[c] + hi) - __ldg(u.c[c] + lo)) * scale + (c == a ? T(1) : T(0));
    }
}

template <class T>
__device__ __forceinline__ T det_of(const T* j, int nd) {
    if (nd == 2) return j[0] * j[3] - j[1] * j[2];
    return j[0] * (j[4] * j[8] - j[5] * j[7]) - j[1] * (j[3] * j[8] - j[5] * j[6]) +
           j[2] * (j[3] * j[7] - j[4] * j[6]);
}

}  // namespace dfm
