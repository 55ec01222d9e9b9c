// kernels_point.cu — pointwise, gather and reduction kernels of the path:
// staging conversions, warps, compose, Jacobian determinant, Adam, resampling,
// SSD / soft-Dice losses, and the on-device convergence monitor.
#include <cstdint>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"
#include "loop_ops.cuh"

namespace dfm {

namespace {

constexpr int kNT = 256;
constexpr int kRedBlocks = 1184;  // fixed => partial-sum order independent of the device

inline int grid_for(int64_t n, int cap = 0x7fffffff) {  // callers with a cap grid-stride
    int64_t b = (n + kNT - 1) / kNT;
    if (b < 1) b = 1;
    return static_cast<int>(b < cap ? b : cap);
}

// per-voxel kernels over (x, row) with 32 x 8 blocks: x from the block's x
// index, rows (y, z) grid-strided over blockIdx.y — one 32-bit division per
// row instead of two 64-bit ones per voxel, and whole warps on one row
constexpr int kRX = 32, kRY = 8;
inline dim3 rows_grid(int nx, int64_t rows) {
    const int64_t by = (rows + kRY - 1) / kRY;
    return dim3(static_cast<unsigned>((nx + kRX - 1) / kRX),
                static_cast<unsigned>(by < 65535 ? (by < 1 ? 1 : by) : 65535));
}

__device__ __forceinline__ void voxel_xyz(const Dims& d, int64_t i, int& x, int& y, int& z) {
    x = static_cast<int>(i % d.nx);
    const int64_t r = i / d.nx;
    y = static_cast<int>(r % d.ny);
    z = static_cast<int>(r / d.ny);
}

// deterministic block sum (fixed shuffle tree); valid in thread 0
template <int NT>
__device__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = 0.0;
    if (w == 0) {
        v = l < NT / 32 ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    __syncthreads();
    return v;
}

template <class T>
__device__ __forceinline__ T ld(const T* p, int64_t i) {
    return __ldg(p + i);
}

}  // namespace

// ---------------------------------------------------------------- staging
template <class T, class S>
__global__ void k_cast(const S* __restrict__ in, T* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
        out[i] = static_cast<T>(in[i]);
}

template <class T, class S>
void launch_cast(const Launch& L, const S* in, T* out, int64_t n) {
    k_cast<T, S><<<grid_for(n, 8192), kNT, 0, L.stream>>>(in, out, n);
    L.bump();
}

template <class T, class S>
__global__ void k_aos_to_soa(const S* __restrict__ aos, Planes3<T> out, int64_t n, int nd) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        for (int c = 0; c < 3; ++c)
            out.c[c][i] = c < nd ? static_cast<T>(aos[i * nd + c]) : T(0);
    }
}

template <class T, class S>
void launch_aos_to_soa(const Launch& L, const S* aos, Planes3<T> out, int64_t n, int nd) {
    k_aos_to_soa<T, S><<<grid_for(n, 8192), kNT, 0, L.stream>>>(aos, out, n, nd);
    L.bump();
}

template <class T, class S>
__global__ void k_soa_to_aos(CPlanes3<T> in, S* __restrict__ aos, int64_t n, int nd) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
        for (int c = 0; c < nd; ++c) aos[i * nd + c] = static_cast<S>(in.c[c][i]);
}

template <class T, class S>
void launch_soa_to_aos(const Launch& L, CPlanes3<T> in, S* aos, int64_t n, int nd) {
    k_soa_to_aos<T, S><<<grid_for(n, 8192), kNT, 0, L.stream>>>(in, aos, n, nd);
    L.bump();
}

template <class T>
__global__ void k_fill(T* p, int64_t n, T v) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
        p[i] = v;
}

template <class T>
void launch_fill(const Launch& L, T* p, int64_t n, T v) {
    k_fill<T><<<grid_for(n, 8192), kNT, 0, L.stream>>>(p, n, v);
    L.bump();
}

// ---------------------------------------------------------------- sampling
template <class T>
__global__ void k_sample_points(const T* __restrict__ img, Dims d, const double* __restrict__ pts,
                                int64_t np, double* vals, double* grads) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= np) return;
    const Cell3<T> c = locate3<T>(d, 0, 0, 0, static_cast<T>(pts[3 * i]),
                                  static_cast<T>(pts[3 * i + 1]),
                                  static_cast<T>(d.ndim == 3 ? pts[3 * i + 2] : 0.0));
    const Corners<T> k = fetch_corners<T>(img, c);
    vals[i] = static_cast<double>(lerp_value(c, k));
    if (grads) {
        T g[3];
        lerp_grad(c, k, d.ndim, g);
        for (int a = 0; a < 3; ++a) grads[3 * i + a] = static_cast<double>(g[a]);
    }
}

template <class T>
void launch_sample_points(const Launch& L, const T* img, Dims d, const double* pts, int64_t np,
                          double* vals, double* grads) {
    if (np <= 0) return;
    k_sample_points<T><<<grid_for(np), kNT, 0, L.stream>>>(img, d, pts, np, vals, grads);
    L.bump();
}

// warp_image (interp.cpp:229-246); the image may have its own grid (loss use)
template <class T>
__global__ void k_warp_image(const T* __restrict__ img, Dims dimg, CPlanes3<T> u, Dims d,
                             T* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int x, y, z;
    voxel_xyz(d, i, x, y, z);
    const Cell3<T> c = locate3<T>(dimg, x, y, z, ld(u.c[0], i), ld(u.c[1], i),
                                  d.ndim == 3 ? ld(u.c[2], i) : T(0));
    out[i] = lerp_value(c, fetch_corners<T>(img, c));
}

template <class T>
void launch_warp_image(const Launch& L, const T* img, Dims dimg, CPlanes3<T> u, Dims d, T* out) {
    k_warp_image<T><<<grid_for(d.n), kNT, 0, L.stream>>>(img, dimg, u, d, out);
    L.bump();
}

// warp_labels (interp.cpp:248-267): llround (half away from zero) + clamp
template <class T>
__global__ void k_warp_labels(const int32_t* __restrict__ lab, CPlanes3<T> u, Dims d,
                              int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int q[3];
    voxel_xyz(d, i, q[0], q[1], q[2]);
    const int n[3] = {d.nx, d.ny, d.nz};
    for (int c = 0; c < d.ndim; ++c) {
        long long r = llround(static_cast<double>(q[c]) + static_cast<double>(u.c[c][i]));
        r = r < 0 ? 0 : (r > n[c] - 1 ? n[c] - 1 : r);
        q[c] = static_cast<int>(r);
    }
    out[i] = lab[d.idx(q[0], q[1], q[2])];
}

template <class T>
void launch_warp_labels(const Launch& L, const int32_t* lab, CPlanes3<T> u, Dims d, int32_t* out) {
    k_warp_labels<T><<<grid_for(d.n), kNT, 0, L.stream>>>(lab, u, d, out);
    L.bump();
}

// compose (interp.cpp:269-289): out = psi + lerp(phi)(x + psi)
template <class T>
__global__ void k_compose(CPlanes3<T> phi, CPlanes3<T> psi, Dims d, Planes3<T> out) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int x, y, z;
    voxel_xyz(d, i, x, y, z);
    const T s[3] = {psi.c[0][i], psi.c[1][i], d.ndim == 3 ? psi.c[2][i] : T(0)};
    const Cell3<T> c = locate3<T>(d, x, y, z, s[0], s[1], s[2]);
    T v[3];
    lerp_field(c, phi.c[0], phi.c[1], phi.c[2], d.ndim, v);
    for (int k = 0; k < 3; ++k) out.c[k][i] = k < d.ndim ? s[k] + v[k] : T(0);
}

template <class T>
void launch_compose(const Launch& L, CPlanes3<T> phi, CPlanes3<T> psi, Dims d, Planes3<T> out) {
    k_compose<T><<<grid_for(d.n), kNT, 0, L.stream>>>(phi, psi, d, out);
    L.bump();
}

// jacobian_det (interp.cpp:330-349) + singularity count (analysis.cpp:160-167)
template <class T>
__global__ void k_jacobian_det(CPlanes3<T> u, Dims d, T* det, unsigned long long* nonpos) {
    // only the produced planes [zb, ze) of a slab view are evaluated
    const int x = blockIdx.x * kRX + threadIdx.x;
    const int zb = d.out_begin();
    const int rows = (d.out_end() - zb) * d.ny;
    // rows are uniform per warp (threadIdx.y): the ballot below sees whole warps
    for (int row0 = blockIdx.y * kRY; row0 < rows; row0 += gridDim.y * kRY) {
        const int row = row0 + threadIdx.y;
        int bad = 0;
        if (x < d.nx && row < rows) {
            const int y = row % d.ny, z = zb + row / d.ny;
            T J[9];
            T v;
            if (d.ndim == 3) {
                jacobian_at3(u, d, x, y, z, J);
                v = det_of(J, 3);
            } else {
                jacobian_at(u, d, x, y, z, J);
                v = det_of(J, d.ndim);
            }
            if (det) det[d.idx(x, y, z)] = v;
            bad = (v <= T(0));
        }
        if (nonpos) {
            const unsigned m = __ballot_sync(0xffffffffu, bad);
            if ((threadIdx.x & 31) == 0 && m) atomicAdd(nonpos, (unsigned long long)__popc(m));
        }
    }
}

template <class T>
void launch_jacobian_det(const Launch& L, CPlanes3<T> u, Dims d, T* det,
                         unsigned long long* nonpos) {
    const int64_t rows = static_cast<int64_t>(d.out_end() - d.out_begin()) * d.ny;
    k_jacobian_det<T><<<rows_grid(d.nx, rows), dim3(kRX, kRY), 0, L.stream>>>(u, d, det, nonpos);
    L.bump();
}

// eulerian_direction (diffeo.cpp:11-40)
template <class T>
__global__ void k_eulerian(CPlanes3<T> g, CPlanes3<T> u, Dims d, int use_jac, Planes3<T> out) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    if (!use_jac) {
        for (int c = 0; c < 3; ++c) out.c[c][i] = c < d.ndim ? -g.c[c][i] : T(0);
        return;
    }
    int x, y, z;
    voxel_xyz(d, i, x, y, z);
    T J[9];
    jacobian_at(u, d, x, y, z, J);
    for (int a = 0; a < 3; ++a) {
        T acc = T(0);
        if (a < d.ndim)
            for (int c = 0; c < d.ndim; ++c) acc += J[c * d.ndim + a] * g.c[c][i];
        out.c[a][i] = -acc;
    }
}

template <class T>
void launch_eulerian(const Launch& L, CPlanes3<T> g, CPlanes3<T> u, Dims d, int use_jac,
                     Planes3<T> out) {
    k_eulerian<T><<<grid_for(d.n), kNT, 0, L.stream>>>(g, u, d, use_jac, out);
    L.bump();
}

// adam_step (optim.cpp:22-42), standalone form for the per-call API
template <class T>
__global__ void k_adam(Planes3<T> m, Planes3<T> nu, CPlanes3<T> v, Planes3<T> dir, Dims d,
                       T b1, T omb1, T b2, T omb2, T c1, T c2, T eps) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    for (int c = 0; c < d.ndim; ++c) {
        const T vv = v.c[c][i];
        const T mm = b1 * m.c[c][i] + omb1 * vv;
        const T nn = b2 * nu.c[c][i] + omb2 * vv * vv;
        m.c[c][i] = mm;
        nu.c[c][i] = nn;
        dir.c[c][i] = (mm / c1) / (sqrt(nn / c2) + eps);
    }
}

template <class T>
void launch_adam(const Launch& L, Planes3<T> m, Planes3<T> nu, CPlanes3<T> v, Planes3<T> dir,
                 Dims d, double b1, double b2, double c1, double c2, double eps) {
    k_adam<T><<<grid_for(d.n), kNT, 0, L.stream>>>(m, nu, v, dir, d, T(b1), T(1.0 - b1), T(b2),
                                                   T(1.0 - b2), T(c1), T(c2), T(eps));
    L.bump();
}

// apply_update step (diffeo.cpp:47-59): clamp(eta*v, +-cap), non-finite flag
template <class T>
__global__ void k_clamp_step(CPlanes3<T> v, Planes3<T> step, Dims d, T eta, T cap, int* bad) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    for (int c = 0; c < 3; ++c) {
        if (c >= d.ndim) {
            step.c[c][i] = T(0);
            continue;
        }
        const T s = eta * v.c[c][i];
        if (!isfinite(s)) *bad = 1;
        step.c[c][i] = s < -cap ? -cap : (cap < s ? cap : s);
    }
}

template <class T>
void launch_clamp_step(const Launch& L, CPlanes3<T> v, Planes3<T> step, Dims d, double eta,
                       double cap, int* bad) {
    k_clamp_step<T><<<grid_for(d.n), kNT, 0, L.stream>>>(v, step, d, T(eta), T(cap), bad);
    L.bump();
}

// corner-aligned linear resample (interp.cpp:381-445, optim.cpp:59-85,
// core.cpp:78-90): dst(x) = mult_c * lerp(src_c)(x * (ns-1)/(nd-1)).
// The sample position is formed in double like the reference, the cell is
// decided in double, only the fraction is rounded to T.
template <class T>
struct ResampleArgs {  // up to 9 components (field + both Adam moments in one pass)
    const T* src[9];
    T* dst[9];
    double mult[9];
    double step[3];
};

__device__ __forceinline__ void locate_point(double p, int n, int& i0, double& f) {
    if (n == 1) {
        i0 = 0;
        f = 0.0;
        return;
    }
    const double hi = static_cast<double>(n - 1);
    p = p < 0.0 ? 0.0 : (hi < p ? hi : p);
    int i = static_cast<int>(floor(p));
    i = i < 0 ? 0 : (i > n - 2 ? n - 2 : i);
    i0 = i;
    f = p - static_cast<double>(i);
}

// NC > 0: the component count fixed at compile time, every component's 8
// corners loaded before the first blend (up to 72 independent loads in flight
// per thread; the full-size 1/2 -> 1 upsample of field and moments is 9
// components). NC == 0: runtime count, one component at a time. Same
// arithmetic either way.
template <class T, int NC>
__global__ void k_resample(ResampleArgs<T> a, Dims ds, Dims dd, int ncomp) {
    const int x = blockIdx.x * kRX + threadIdx.x;
    if (x >= dd.nx) return;
    const int rows = dd.ny * dd.nz;
    int ix;
    double fx;
    locate_point(x * a.step[0], ds.nx, ix, fx);
    for (int row = blockIdx.y * kRY + threadIdx.y; row < rows; row += gridDim.y * kRY) {
        const int y = row % dd.ny, z = row / dd.ny;
        int iy, iz;
        double fy, fz;
        locate_point(y * a.step[1], ds.ny, iy, fy);
        locate_point((z + dd.zoff) * a.step[2], ds.nz, iz, fz);  // dd may be a z-slab view
        Cell3<T> c;
        c.base = ds.idx(ix, iy, iz);
        c.sx = ds.nx > 1 ? 1 : 0;
        c.sy = ds.ny > 1 ? ds.nx : 0;
        c.three = ds.nz > 1;
        c.sz = c.three ? static_cast<int64_t>(ds.nx) * ds.ny : 0;
        c.fx = static_cast<T>(fx);
        c.fy = static_cast<T>(fy);
        c.fz = static_cast<T>(fz);
        c.clx = c.cly = c.clz = false;
        const int64_t i = dd.idx(x, y, z);
        if constexpr (NC > 0) {
            // 3-D source with every axis > 1 (launcher): the +x corner is the
            // next element, so each component needs four row pointers (base,
            // +y, +z, +y+z) and reads two neighbours from each
            const int64_t sy = ds.nx, sz = static_cast<int64_t>(ds.nx) * ds.ny;
            Corners<T> k[NC];
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const T* p0 = a.src[q] + c.base;
                const T* p1 = p0 + sy;
                const T* p2 = p0 + sz;
                const T* p3 = p2 + sy;
                k[q].v[0] = __ldg(p0);
                k[q].v[1] = __ldg(p0 + 1);
                k[q].v[2] = __ldg(p1);
                k[q].v[3] = __ldg(p1 + 1);
                k[q].v[4] = __ldg(p2);
                k[q].v[5] = __ldg(p2 + 1);
                k[q].v[6] = __ldg(p3);
                k[q].v[7] = __ldg(p3 + 1);
            }
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                const T v = lerp_value(c, k[q]);
                a.dst[q][i] = a.mult[q] == 1.0 ? v : static_cast<T>(v * a.mult[q]);
            }
        } else {
#pragma unroll 3
            for (int k = 0; k < ncomp; ++k) {
                const T v = lerp_value(c, fetch_corners<T>(a.src[k], c));
                a.dst[k][i] = a.mult[k] == 1.0 ? v : static_cast<T>(v * a.mult[k]);
            }
        }
    }
}

template <class T>
void launch_resample(const Launch& L, const T* const* src, Dims ds, T* const* dst, Dims dd,
                     int ncomp, const double* mult) {
    ResampleArgs<T> a;
    const int ns[3] = {ds.nx, ds.ny, ds.nz}, nd[3] = {dd.nx, dd.ny, dd.gz()};
    for (int k = 0; k < 9; ++k) {
        a.src[k] = k < ncomp ? src[k] : nullptr;
        a.dst[k] = k < ncomp ? dst[k] : nullptr;
        a.mult[k] = mult && k < ncomp ? mult[k] : 1.0;
    }
    for (int k = 0; k < 3; ++k)
        a.step[k] = nd[k] > 1 ? static_cast<double>(ns[k] - 1) / (nd[k] - 1) : 0.0;
    const dim3 grid = rows_grid(dd.nx, static_cast<int64_t>(dd.ny) * dd.nz), block(kRX, kRY);
    // fp64 keeps the runtime count: 9 fixed components take 182 registers there
    const bool solid = ds.nx > 1 && ds.ny > 1 && ds.nz > 1;
    switch (sizeof(T) == 4 && solid ? ncomp : 0) {
        case 3: k_resample<T, 3><<<grid, block, 0, L.stream>>>(a, ds, dd, ncomp); break;
        case 9: k_resample<T, 9><<<grid, block, 0, L.stream>>>(a, ds, dd, ncomp); break;
        default: k_resample<T, 0><<<grid, block, 0, L.stream>>>(a, ds, dd, ncomp); break;
    }
    L.bump();
}

// affine working field (affine.cpp:26-48): u = S^-1 (A S x + t) - x
template <class T>
struct AffineArgs {
    double A[9], t[3], S[3];
};

template <class T>
__global__ void k_affine_field(AffineArgs<T> a, Dims d, Planes3<T> out) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int q[3];
    voxel_xyz(d, i, q[0], q[1], q[2]);
    const int nd = d.ndim;
    for (int r = 0; r < 3; ++r) {
        if (r >= nd) {
            out.c[r][i] = T(0);
            continue;
        }
        double acc = a.t[r];
        for (int c = 0; c < nd; ++c) acc += a.A[r * nd + c] * a.S[c] * static_cast<double>(q[c]);
        out.c[r][i] = static_cast<T>(acc / a.S[r] - static_cast<double>(q[r]));
    }
}

template <class T>
void launch_affine_field(const Launch& L, const double* A, const double* t, const double* S,
                         Dims d, Planes3<T> out) {
    AffineArgs<T> a;
    for (int k = 0; k < 9; ++k) a.A[k] = A[k];
    for (int k = 0; k < 3; ++k) {
        a.t[k] = t[k];
        a.S[k] = S[k];
    }
    k_affine_field<T><<<grid_for(d.n), kNT, 0, L.stream>>>(a, d, out);
    L.bump();
}

// one axis of a separable truncated Gaussian with boundary renormalisation
// (interp.cpp:110-151): generic radius, used for the pyramid pre-blur and
// for sigmas beyond the fused kernels' kRMax.
template <class T>
__global__ void k_gauss_axis(const T* __restrict__ in, T* __restrict__ out, Dims d, int axis,
                             int R, const double* __restrict__ taps,
                             const double* __restrict__ norm, const LoopState* st) {
    if (st && st->done) return;
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int q[3];
    voxel_xyz(d, i, q[0], q[1], q[2]);
    const int n = axis == 0 ? d.nx : (axis == 1 ? d.ny : d.nz);
    const int64_t stride = axis == 0 ? 1 : (axis == 1 ? d.nx : static_cast<int64_t>(d.nx) * d.ny);
    const int p = q[axis];
    const int jlo = -R > -p ? -R : -p;
    const int jhi = R < n - 1 - p ? R : n - 1 - p;
    double acc = 0.0;
    for (int j = jlo; j <= jhi; ++j) acc += taps[j + R] * static_cast<double>(in[i + j * stride]);
    out[i] = static_cast<T>(acc * norm[p]);
}

template <class T>
void launch_gauss_axis(const Launch& L, const T* in, T* out, Dims d, int axis, int R,
                       const double* taps, const double* norm, const LoopState* st) {
    k_gauss_axis<T><<<grid_for(d.n), kNT, 0, L.stream>>>(in, out, d, axis, R, taps, norm, st);
    L.bump();
}

template <class T>
__global__ void k_range_check(const T* p, int64_t n, int* bad) {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
        const T v = p[i];
        if (!(v >= T(0) && v <= T(1))) *bad = 1;
    }
}

template <class T>
void launch_range_check(const Launch& L, const T* p, int64_t n, int* bad) {
    k_range_check<T><<<grid_for(n, 4096), kNT, 0, L.stream>>>(p, n, bad);
    L.bump();
}

// ---------------------------------------------------------------- losses
// ssd_eval (similarity.cpp:81-104): partial sums of (F-W)^2; grad = (W-F) G / N
template <class T>
__global__ void __launch_bounds__(kNT) k_ssd(const T* __restrict__ F, const T* __restrict__ M,
                                             Dims d, Dims dm, CPlanes3<T> u, Planes3<T> grad,
                                             double* partials, const LoopState* st,
                                             MonitorArgs mon) {
    __shared__ double sh[32];
    if (st && st->done) return;
    double acc = 0.0;
    const T nn = static_cast<T>(d.n);
    if (d.ndim == 3) {  // 3-D fast form: 32-bit gather, grad * (1/N) in fp32
        const T inv = sizeof(T) == 4 ? T(1) / nn : T(0);
        for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < d.n;
             i += (int64_t)gridDim.x * kNT) {
            int x, y, z;
            voxel_xyz(d, i, x, y, z);
            WG3<T> wg;
            wg3_fetch<T, false>(M, dm, x, y, z, ld(u.c[0], i), ld(u.c[1], i), ld(u.c[2], i), wg);
            const T w = wg3_value(wg);
            const T f = ld(F, i);
            const double r = static_cast<double>(f) - static_cast<double>(w);
            acc += r * r;
            if (grad.c[0]) {
                T g[3];
                wg3_grad(wg, g);
                const T rr = w - f;
                for (int a = 0; a < 3; ++a)
                    grad.c[a][i] = sizeof(T) == 4 ? rr * g[a] * inv : rr * g[a] / nn;
            }
        }
    } else {
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * kNT) {
        int x, y, z;
        voxel_xyz(d, i, x, y, z);
        const Cell3<T> c = locate3<T>(dm, x, y, z, ld(u.c[0], i), ld(u.c[1], i),
                                      d.ndim == 3 ? ld(u.c[2], i) : T(0));
        const Corners<T> k = fetch_corners<T>(M, c);
        const T w = lerp_value(c, k);
        const T f = ld(F, i);
        const double r = static_cast<double>(f) - static_cast<double>(w);
        acc += r * r;
        if (grad.c[0]) {
            T g[3];
            lerp_grad(c, k, d.ndim, g);
            const T rr = w - f;
            for (int a = 0; a < 3; ++a) grad.c[a][i] = rr * g[a] / nn;
        }
    }
    }
    const double s = block_sum<kNT>(acc, sh);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
    if (mon.st) {  // fused convergence monitor (value = +sum / N)
        __syncthreads();
        monitor_tail<kNT>(mon, partials, gridDim.x, static_cast<double>(d.n), sh, 1.0);
    }
}

template <class T>
int launch_ssd(const Launch& L, const T* F, const T* M, Dims d, Dims dm, CPlanes3<T> u,
               Planes3<T> grad, double* partials, const LoopState* st, const MonitorArgs* mon) {
    const int nb = grid_for(d.n, kRedBlocks);
    k_ssd<T><<<nb, kNT, 0, L.stream>>>(F, M, d, dm, u, grad, partials, st,
                                       mon ? *mon : MonitorArgs{nullptr, nullptr, nullptr, 0, 0.0});
    L.bump();
    return nb;
}

// dice_soft_eval (similarity.cpp:192-231): sums P=F*W, SF, SM
template <class T>
__global__ void __launch_bounds__(kNT) k_dice_sums(const T* __restrict__ F,
                                                   const T* __restrict__ M, Dims d, Dims dm,
                                                   CPlanes3<T> u, double* partials,
                                                   const LoopState* st) {
    __shared__ double sh[32];
    if (st && st->done) return;
    double p = 0.0, sf = 0.0, sm = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < d.n;
         i += (int64_t)gridDim.x * kNT) {
        int x, y, z;
        voxel_xyz(d, i, x, y, z);
        const Cell3<T> c = locate3<T>(dm, x, y, z, ld(u.c[0], i), ld(u.c[1], i),
                                      d.ndim == 3 ? ld(u.c[2], i) : T(0));
        const double w = static_cast<double>(lerp_value(c, fetch_corners<T>(M, c)));
        const double f = static_cast<double>(ld(F, i));
        p += f * w;
        sf += f;
        sm += w;
    }
    const double a = block_sum<kNT>(p, sh);
    const double b = block_sum<kNT>(sf, sh);
    const double e = block_sum<kNT>(sm, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = a;
        partials[gridDim.x + blockIdx.x] = b;
        partials[2 * gridDim.x + blockIdx.x] = e;
    }
}

template <class T>
int launch_dice_sums(const Launch& L, const T* F, const T* M, Dims d, Dims dm, CPlanes3<T> u,
                     double* partials, const LoopState* st) {
    const int nb = grid_for(d.n, kRedBlocks);
    k_dice_sums<T><<<nb, kNT, 0, L.stream>>>(F, M, d, dm, u, partials, st);
    L.bump();
    return nb;
}

template <class T>
__global__ void k_dice_grad(const T* __restrict__ F, const T* __restrict__ M, Dims d, Dims dm,
                            CPlanes3<T> u, Planes3<T> grad, const LoopState* st, double P,
                            double D) {
    if (st) {
        if (st->done) return;
        P = st->dice_p;
        D = st->dice_d;
    }
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int x, y, z;
    voxel_xyz(d, i, x, y, z);
    const Cell3<T> c = locate3<T>(dm, x, y, z, ld(u.c[0], i), ld(u.c[1], i),
                                  d.ndim == 3 ? ld(u.c[2], i) : T(0));
    T g[3];
    lerp_grad(c, fetch_corners<T>(M, c), d.ndim, g);
    const double dW = -2.0 * static_cast<double>(ld(F, i)) / D + 2.0 * P / (D * D);
    for (int a = 0; a < 3; ++a) grad.c[a][i] = static_cast<T>(dW * static_cast<double>(g[a]));
}

template <class T>
void launch_dice_grad(const Launch& L, const T* F, const T* M, Dims d, Dims dm, CPlanes3<T> u,
                      Planes3<T> grad, const LoopState* st, double P, double D) {
    k_dice_grad<T><<<grid_for(d.n), kNT, 0, L.stream>>>(F, M, d, dm, u, grad, st, P, D);
    L.bump();
}

// ---------------------------------------------------------------- loop control
__device__ double sum_partials(const double* p, int np, double* sh) {
    double acc = 0.0;
    for (int k = threadIdx.x; k < np; k += 1024) acc += p[k];
    return block_sum<1024>(acc, sh);
}

__device__ double loss_value(int kind, const double* partials, int np, double nvox, double* sh,
                             double* P_out, double* D_out) {
    if (kind == 2) {
        const double P = sum_partials(partials, np, sh);
        const double SF = sum_partials(partials + np, np, sh);
        const double SM = sum_partials(partials + 2 * np, np, sh);
        const double D = SF + SM + 1e-7;
        *P_out = P;
        *D_out = D;
        return 1.0 - 2.0 * P / D;
    }
    const double s = sum_partials(partials, np, sh);
    return kind == 1 ? -s / nvox : s / nvox;
}


// Finishes the loss of the current iteration and runs the convergence monitor
// (pipeline.cpp:157-179): non-finite -> error; converged -> record kept, the
// scale ends before the update.
__global__ void __launch_bounds__(1024) k_monitor(int kind, const double* partials, int np,
                                                  double nvox, LoopState* st, double* loss,
                                                  unsigned long long* stamp, int window,
                                                  double tol) {
    __shared__ double sh[32];
    if (st->done) return;
    double P = 0.0, D = 0.0;
    const double v = loss_value(kind, partials, np, nvox, sh, &P, &D);
    if (threadIdx.x != 0) return;
    monitor_commit(st, v, P, D, loss, stamp, window, tol);
}

void launch_monitor(const Launch& L, int kind, const double* partials, int np, double nvox,
                    LoopState* st, double* loss, unsigned long long* stamp, int window,
                    double tol) {
    k_monitor<<<1, 1024, 0, L.stream>>>(kind, partials, np, nvox, st, loss, stamp, window, tol);
    L.bump();
}

__global__ void __launch_bounds__(1024) k_reduce_value(int kind, const double* partials, int np,
                                                       double nvox, double* out) {
    __shared__ double sh[32];
    double P, D;
    const double v = loss_value(kind, partials, np, nvox, sh, &P, &D);
    if (threadIdx.x == 0) {
        out[0] = v;
        out[1] = P;
        out[2] = D;
    }
}

void launch_reduce_value(const Launch& L, int kind, const double* partials, int np, double nvox,
                         double* out) {
    k_reduce_value<<<1, 1024, 0, L.stream>>>(kind, partials, np, nvox, out);
    L.bump();
}

__global__ void k_stamp(unsigned long long* slot) { *slot = dfm_global_ns(); }

void launch_stamp(const Launch& L, unsigned long long* slot) {
    k_stamp<<<1, 1, 0, L.stream>>>(slot);
    L.bump();
}

// ---------------------------------------------------------------- C++ drop-in extras
// jacobian (interp.cpp:291-328): J = I + central differences (one-sided at the
// borders), ndim x ndim row-major per voxel (row = component), AoS
template <class T>
__global__ void k_jacobian_full(CPlanes3<T> u, Dims d, T* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    int x, y, z;
    voxel_xyz(d, i, x, y, z);
    T J[9];
    jacobian_at(u, d, x, y, z, J);
    const int nn = d.ndim * d.ndim;
    for (int k = 0; k < nn; ++k) out[i * nn + k] = J[k];
}

template <class T>
void launch_jacobian_full(const Launch& L, CPlanes3<T> u, Dims d, T* out) {
    k_jacobian_full<T><<<grid_for(d.n), kNT, 0, L.stream>>>(u, d, out);
    L.bump();
}

// Catmull-Rom weight (interp.cpp:59-67)
__device__ __forceinline__ double cubic_weight(double t) {
    t = fabs(t);
    if (t <= 1.0) return __dadd_rn(__dmul_rn(__dmul_rn(__dsub_rn(__dmul_rn(1.5, t), 2.5), t), t), 1.0);
    if (t < 2.0)
        return __dadd_rn(
            __dmul_rn(__dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(-0.5, t), 2.5), t), 4.0), t), 2.0);
    return 0.0;
}

// upsample_field with UpsampleMethod::cubic (interp.cpp:69-101, 408-445):
// corner-aligned Catmull-Rom resample of each component (clamped 4^d
// neighbourhood), then the per-axis displacement rescale.  The reference keeps
// it only for its folding demonstration; it is not on the registration path.
template <class T>
__global__ void k_upsample_cubic(CPlanes3<T> f, Dims ds, Planes3<T> out, Dims dd, double st0,
                                 double st1, double st2, double r0, double r1, double r2) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= dd.n) return;
    int x, y, z;
    voxel_xyz(dd, i, x, y, z);
    const double p[3] = {__dmul_rn(static_cast<double>(x), st0),
                         __dmul_rn(static_cast<double>(y), st1),
                         __dmul_rn(static_cast<double>(z), st2)};
    const int dims[3] = {ds.nx, ds.ny, ds.nz};
    int base[3];
    double frac[3];
    for (int a = 0; a < 3; ++a) {
        if (a >= ds.ndim || dims[a] == 1) {
            base[a] = 0;
            frac[a] = 0.0;
            continue;
        }
        const double q = fmin(fmax(p[a], 0.0), static_cast<double>(dims[a] - 1));
        int b = static_cast<int>(floor(q));
        b = min(max(b, 0), dims[a] - 2);
        base[a] = b;
        frac[a] = __dsub_rn(q, static_cast<double>(b));
    }
    const int na = (ds.ndim == 3 && ds.nz > 1) ? 4 : 1;
    const double rs[3] = {r0, r1, r2};
    for (int c = 0; c < ds.ndim; ++c) {
        double acc = 0.0;
        for (int kz = 0; kz < na; ++kz) {
            const double wz = na == 4 ? cubic_weight(__dsub_rn(frac[2], double(kz - 1))) : 1.0;
            const int zz = na == 4 ? min(max(base[2] + kz - 1, 0), ds.nz - 1) : 0;
            for (int ky = 0; ky < 4; ++ky) {
                const double wy = cubic_weight(__dsub_rn(frac[1], double(ky - 1)));
                const int yy = min(max(base[1] + ky - 1, 0), ds.ny - 1);
                for (int kx = 0; kx < 4; ++kx) {
                    const double wx = cubic_weight(__dsub_rn(frac[0], double(kx - 1)));
                    const int xx = min(max(base[0] + kx - 1, 0), ds.nx - 1);
                    const double v = static_cast<double>(f.c[c][ds.idx(xx, yy, zz)]);
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(wz, wy), wx), v));
                }
            }
        }
        out.c[c][i] = static_cast<T>(__dmul_rn(acc, rs[c]));
    }
}

template <class T>
void launch_upsample_cubic(const Launch& L, CPlanes3<T> f, Dims ds, Planes3<T> out, Dims dd,
                           const double step[3], const double rescale[3]) {
    k_upsample_cubic<T><<<grid_for(dd.n), kNT, 0, L.stream>>>(
        f, ds, out, dd, step[0], step[1], step[2], rescale[0], rescale[1], rescale[2]);
    L.bump();
}

// sgd_step (optim.cpp:44-57): mu <- momentum * mu + v
template <class T>
__global__ void k_sgd(Planes3<T> mu, CPlanes3<T> v, Dims d, T momentum) {
    const int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x;
    if (i >= d.n) return;
    for (int c = 0; c < d.ndim; ++c) mu.c[c][i] = momentum * mu.c[c][i] + v.c[c][i];
}

template <class T>
void launch_sgd(const Launch& L, Planes3<T> mu, CPlanes3<T> v, Dims d, double momentum) {
    k_sgd<T><<<grid_for(d.n), kNT, 0, L.stream>>>(mu, v, d, T(momentum));
    L.bump();
}

// the level loop alternates the field between two buffers; with an early stop
// the result may sit in the other one.  Without a host round trip the next
// level reads `dst`: copy src -> dst when (T_si - nupdates) is odd.
template <class T>
__global__ void k_parity_fix(const LoopState* __restrict__ st, int T_si, CPlanes3<T> src,
                             Planes3<T> dst, int64_t n, int ncomp) {
    if (((T_si - st->nupdates) & 1) == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kNT)
        for (int c = 0; c < ncomp; ++c) dst.c[c][i] = src.c[c][i];
}

template <class T>
void launch_parity_fix(const Launch& L, const LoopState* st, int T_si, CPlanes3<T> src,
                       Planes3<T> dst, int64_t n, int ncomp) {
    const int64_t b = (n + kNT - 1) / kNT;
    k_parity_fix<T><<<static_cast<unsigned>(b < 4096 ? b : 4096), kNT, 0, L.stream>>>(
        st, T_si, src, dst, n, ncomp);
    L.bump();
}

// ---------------------------------------------------------------- instantiations
#define DFM_INST_T(T)                                                                          \
    template void launch_aos_to_soa<T, double>(const Launch&, const double*, Planes3<T>,       \
                                               int64_t, int);                                  \
    template void launch_aos_to_soa<T, float>(const Launch&, const float*, Planes3<T>,         \
                                              int64_t, int);                                   \
    template void launch_soa_to_aos<T, double>(const Launch&, CPlanes3<T>, double*, int64_t,   \
                                               int);                                           \
    template void launch_soa_to_aos<T, float>(const Launch&, CPlanes3<T>, float*, int64_t,     \
                                              int);                                            \
    template void launch_fill<T>(const Launch&, T*, int64_t, T);                               \
    template void launch_sample_points<T>(const Launch&, const T*, Dims, const double*,        \
                                          int64_t, double*, double*);                          \
    template void launch_warp_image<T>(const Launch&, const T*, Dims, CPlanes3<T>, Dims, T*);  \
    template void launch_warp_labels<T>(const Launch&, const int32_t*, CPlanes3<T>, Dims,      \
                                        int32_t*);                                             \
    template void launch_compose<T>(const Launch&, CPlanes3<T>, CPlanes3<T>, Dims, Planes3<T>); \
    template void launch_jacobian_det<T>(const Launch&, CPlanes3<T>, Dims, T*,                 \
                                         unsigned long long*);                                 \
    template void launch_eulerian<T>(const Launch&, CPlanes3<T>, CPlanes3<T>, Dims, int,       \
                                     Planes3<T>);                                              \
    template void launch_adam<T>(const Launch&, Planes3<T>, Planes3<T>, CPlanes3<T>,           \
                                 Planes3<T>, Dims, double, double, double, double, double);    \
    template void launch_clamp_step<T>(const Launch&, CPlanes3<T>, Planes3<T>, Dims, double,   \
                                       double, int*);                                          \
    template void launch_resample<T>(const Launch&, const T* const*, Dims, T* const*, Dims,    \
                                     int, const double*);                                      \
    template void launch_affine_field<T>(const Launch&, const double*, const double*,          \
                                         const double*, Dims, Planes3<T>);                     \
    template void launch_gauss_axis<T>(const Launch&, const T*, T*, Dims, int, int,            \
                                       const double*, const double*, const LoopState*);        \
    template void launch_range_check<T>(const Launch&, const T*, int64_t, int*);               \
    template int launch_ssd<T>(const Launch&, const T*, const T*, Dims, Dims, CPlanes3<T>,     \
                               Planes3<T>, double*, const LoopState*, const MonitorArgs*);                         \
    template int launch_dice_sums<T>(const Launch&, const T*, const T*, Dims, Dims,            \
                                     CPlanes3<T>, double*, const LoopState*);                  \
    template void launch_dice_grad<T>(const Launch&, const T*, const T*, Dims, Dims,           \
                                      CPlanes3<T>, Planes3<T>, const LoopState*, double,       \
                                      double);                                                 \
    template void launch_jacobian_full<T>(const Launch&, CPlanes3<T>, Dims, T*);              \
    template void launch_upsample_cubic<T>(const Launch&, CPlanes3<T>, Dims, Planes3<T>, Dims, \
                                           const double*, const double*);                      \
    template void launch_sgd<T>(const Launch&, Planes3<T>, CPlanes3<T>, Dims, double);      \
    template void launch_parity_fix<T>(const Launch&, const LoopState*, int, CPlanes3<T>,      \
                                       Planes3<T>, int64_t, int);

DFM_INST_T(float)
DFM_INST_T(double)
template void launch_cast<float, float>(const Launch&, const float*, float*, int64_t);
template void launch_cast<float, double>(const Launch&, const double*, float*, int64_t);
template void launch_cast<double, float>(const Launch&, const float*, double*, int64_t);
template void launch_cast<double, double>(const Launch&, const double*, double*, int64_t);

}  // namespace dfm
