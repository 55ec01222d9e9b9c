// kernels_stencil.cu — the fused 2.5-D "z-march" stencil kernels of the hot
// loop.  One CTA owns a kTX x kTY column of the volume and a chunk of z; per
// z-plane it stages a haloed xy tile in shared memory (computing the plane's
// channels on the fly, e.g. the warped moving image), filters x then y in
// shared memory, and keeps the last 2R+1 xy-filtered planes in a register ring
// so the z filter needs no extra HBM pass.  Every intermediate of a separable
// (2R+1)^3 filter therefore stays on chip; HBM sees each input once (plus the
// halo re-reads, served by L2) and each output once.
//
// Ops (what is loaded / emitted per voxel):
//   LnccFwdOp     similarity.cpp:106-168  W = M(x+u); box sums of F, W, F^2,
//                 W^2, FW; per-window coefficients alpha/n, alpha muF/n,
//                 beta/n, beta muW/n; cc^2 partial sums (loss value).
//   LnccBwdOp     similarity.cpp:170-189  box sums of the 4 coefficients;
//                 dW; grad = dW * grad M(x+u) (interpolant recomputed).
//   SmoothAdamOp  pipeline.cpp:182-186 + diffeo.cpp:11-24 + optim.cpp:22-42 +
//                 diffeo.cpp:47-57: sigma_grad Gaussian of the gradient,
//                 v = -g (or -J^T g), Adam moments, capped step, max |step|,
//                 non-finite flag.
//   ComposeSmoothOp diffeo.cpp:60-62 + interp.cpp:269-289: u' = step +
//                 u(x+step), then the sigma_warp Gaussian.
//   GaussOp       interp.cpp:351-371 (API smoothing).
#include <cstdint>
#include <type_traits>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"

namespace dfm {

namespace {

constexpr int kNT = kTX * kTY;

struct Red {
    double sum;
    double mx;
};

template <int NT>
__device__ double block_sum_s(double v, double* sh) {
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

template <int NT>
__device__ double block_max_s(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = 0.0;
    if (w == 0) {
        v = l < NT / 32 ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;
}

struct ZGeom {
    Dims d;
    int zchunk;
    int tiles_x;
};

// ---------------------------------------------------------------------------
// the z-march driver
template <int R, class Op>
__global__ void __launch_bounds__(kNT) k_zmarch(const Op op, const ZGeom g) {
    using Acc = typename Op::Acc;
    constexpr int C = Op::C;
    constexpr int K = 2 * R + 1;
    constexpr int WI = kTX + 2 * R, HI = kTY + 2 * R;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Acc* s_in = reinterpret_cast<Acc*>(smem_raw);  // [C][HI][WI]
    Acc* s_x = s_in + C * HI * WI;                  // [C][HI][kTX]
    __shared__ double s_red[32];

    if (op.skip()) return;
    const Dims& d = g.d;
    const int tid = threadIdx.x;
    const int tx = tid % kTX, ty = tid / kTX;
    const int x0 = (blockIdx.x % g.tiles_x) * kTX;
    const int y0 = (blockIdx.x / g.tiles_x) * kTY;
    const int z0 = blockIdx.y * g.zchunk;
    const int z1 = min(z0 + g.zchunk, d.nz);
    const int x = x0 + tx, y = y0 + ty;
    const bool own = x < d.nx && y < d.ny;

    Acc ring[C][K];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < K; ++k) ring[c][k] = Acc(0);
    double rsum = 0.0, rmax = 0.0;

    for (int zi = z0 - R; zi < z1 + R; ++zi) {
        Acc v[C];
        if (zi >= 0 && zi < d.nz) {
            // stage the haloed plane tile
            for (int e = tid; e < HI * WI; e += kNT) {
                const int row = e / WI, col = e - row * WI;
                const int gx = x0 - R + col, gy = y0 - R + row;
                Acc t[C];
                if (gx >= 0 && gx < d.nx && gy >= 0 && gy < d.ny) {
                    op.load(gx, gy, zi, t);
                } else {
#pragma unroll
                    for (int c = 0; c < C; ++c) t[c] = Acc(0);
                }
#pragma unroll
                for (int c = 0; c < C; ++c) s_in[(c * HI + row) * WI + col] = t[c];
            }
            __syncthreads();
            // x pass
            for (int e = tid; e < HI * kTX; e += kNT) {
                const int row = e / kTX, col = e - row * kTX;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const Acc* src = s_in + (c * HI + row) * WI + col;
                    Acc a = Acc(0);
#pragma unroll
                    for (int j = 0; j < K; ++j) a += op.wgt(0, j) * src[j];
                    if (!Op::kBox && x0 + col < d.nx) a *= op.nrm(0, x0 + col);
                    s_x[(c * HI + row) * kTX + col] = a;
                }
            }
            __syncthreads();
            // y pass
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const Acc* src = s_x + (c * HI + ty) * kTX + tx;
                Acc a = Acc(0);
#pragma unroll
                for (int j = 0; j < K; ++j) a += op.wgt(1, j) * src[j * kTX];
                if (!Op::kBox && own) a *= op.nrm(1, y);
                v[c] = a;
            }
        } else {
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = Acc(0);
        }
        // z ring
#pragma unroll
        for (int c = 0; c < C; ++c) {
#pragma unroll
            for (int k = 0; k < K - 1; ++k) ring[c][k] = ring[c][k + 1];
            ring[c][K - 1] = v[c];
        }
        const int zo = zi - R;
        if (zo >= z0 && own) {
            Acc s[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                Acc a = Acc(0);
#pragma unroll
                for (int k = 0; k < K; ++k) a += op.wgt(2, k) * ring[c][k];
                if (!Op::kBox) a *= op.nrm(2, zo);
                s[c] = a;
            }
            const Red r = op.emit(x, y, zo, s);
            rsum += r.sum;
            rmax = fmax(rmax, r.mx);
        }
    }
    if (Op::kSum || Op::kMax) {
        const int blk = blockIdx.y * gridDim.x + blockIdx.x;
        const double bs = Op::kSum ? block_sum_s<kNT>(rsum, s_red) : 0.0;
        const double bm = Op::kMax ? block_max_s<kNT>(rmax, s_red) : 0.0;
        if (tid == 0) op.finish(blk, bs, bm);
    } else if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        op.finish(0, 0.0, 0.0);
    }
}

// ---------------------------------------------------------------------------
// ops

template <class T, int R>
struct LnccFwdOp {
    using Acc = double;
    static constexpr int C = 5;
    static constexpr bool kBox = true, kSum = true, kMax = false;
    const T* F;
    const T* M;
    CPlanes3<T> u;
    Dims d, dm;
    T* coef[4];  // coef[0] == nullptr: value only
    double* partials;
    const LoopState* st;

    __device__ bool skip() const { return st && st->done; }
    __device__ Acc wgt(int, int) const { return 1.0; }
    __device__ Acc nrm(int, int) const { return 1.0; }

    __device__ void load(int x, int y, int z, double v[5]) const {
        const int64_t i = d.idx(x, y, z);
        const double f = static_cast<double>(__ldg(F + i));
        const Cell3<T> c = locate3<T>(dm, x, y, z, __ldg(u.c[0] + i), __ldg(u.c[1] + i),
                                      d.ndim == 3 ? __ldg(u.c[2] + i) : T(0));
        const double w = static_cast<double>(lerp_value(c, fetch_corners<T>(M, c)));
        v[0] = f;
        v[1] = w;
        v[2] = f * f;
        v[3] = w * w;
        v[4] = f * w;
    }

    __device__ Red emit(int x, int y, int z, const double s[5]) const {
        const double n = static_cast<double>(box_len(x, d.nx, R) * box_len(y, d.ny, R) *
                                             (d.nz > 1 ? box_len(z, d.nz, R) : 1));
        const double muF = s[0] / n;
        const double muW = s[1] / n;
        double vF = s[2] / n - muF * muF;
        double vW = s[3] / n - muW * muW;
        vF = vF < 0.0 ? 0.0 : vF;
        vW = vW < 0.0 ? 0.0 : vW;
        const double cv = s[4] / n - muF * muW;
        double cc2 = 0.0, an = 0.0, amu = 0.0, bn = 0.0, bmu = 0.0;
        if (!(vF < 1e-5 || vW < 1e-5)) {  // similarity.cpp:13,151-154
            const double cc = cv / sqrt(vF * vW);
            cc2 = cc * cc;
            const double alpha = cv / (vF * vW);
            const double beta = cv * cv / (vF * vW * vW);
            an = alpha / n;
            amu = alpha * muF / n;
            bn = beta / n;
            bmu = beta * muW / n;
        }
        if (coef[0]) {
            const int64_t i = d.idx(x, y, z);
            coef[0][i] = static_cast<T>(an);
            coef[1][i] = static_cast<T>(amu);
            coef[2][i] = static_cast<T>(bn);
            coef[3][i] = static_cast<T>(bmu);
        }
        return {cc2, 0.0};
    }

    __device__ void finish(int blk, double s, double) const { partials[blk] = s; }
};

template <class T, int R>
struct LnccBwdOp {
    using Acc = double;
    static constexpr int C = 4;
    static constexpr bool kBox = true, kSum = false, kMax = false;
    const T* F;
    const T* M;
    CPlanes3<T> u;
    Dims d, dm;
    const T* coef[4];
    Planes3<T> grad;
    const LoopState* st;

    __device__ bool skip() const { return st && st->done; }
    __device__ Acc wgt(int, int) const { return 1.0; }
    __device__ Acc nrm(int, int) const { return 1.0; }

    __device__ void load(int x, int y, int z, double v[4]) const {
        const int64_t i = d.idx(x, y, z);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = static_cast<double>(__ldg(coef[k] + i));
    }

    __device__ Red emit(int x, int y, int z, const double s[4]) const {
        const int64_t i = d.idx(x, y, z);
        const Cell3<T> c = locate3<T>(dm, x, y, z, __ldg(u.c[0] + i), __ldg(u.c[1] + i),
                                      d.ndim == 3 ? __ldg(u.c[2] + i) : T(0));
        const Corners<T> k = fetch_corners<T>(M, c);
        const double w = static_cast<double>(lerp_value(c, k));
        T g[3];
        lerp_grad(c, k, d.ndim, g);
        const double f = static_cast<double>(__ldg(F + i));
        const double dW = -2.0 / static_cast<double>(d.n) * (f * s[0] - s[1] - w * s[2] + s[3]);
#pragma unroll
        for (int a = 0; a < 3; ++a) grad.c[a][i] = static_cast<T>(dW * static_cast<double>(g[a]));
        return {0.0, 0.0};
    }

    __device__ void finish(int, double, double) const {}
};

template <class T, int R>
struct SmoothAdamOp {
    using Acc = T;
    static constexpr int C = 3;
    static constexpr bool kBox = false, kSum = false, kMax = true;
    GaussW<T> w;
    CPlanes3<T> g;
    CPlanes3<T> u;
    Planes3<T> m, nu, step;
    Dims d;
    T b1, omb1, b2, omb2, eps, eta, cap;
    const double* corr1;
    const double* corr2;
    int use_jac;
    LoopState* st;
    unsigned long long* maxstep;

    __device__ bool skip() const { return st && st->done; }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const { return __ldg(w.norm[a] + i); }

    __device__ void load(int x, int y, int z, T v[3]) const {
        const int64_t i = d.idx(x, y, z);
        v[0] = __ldg(g.c[0] + i);
        v[1] = __ldg(g.c[1] + i);
        v[2] = d.ndim == 3 ? __ldg(g.c[2] + i) : T(0);
    }

    __device__ Red emit(int x, int y, int z, const T s[3]) const {
        const int64_t i = d.idx(x, y, z);
        T v[3];
        if (use_jac) {
            T J[9];
            jacobian_at(u, d, x, y, z, J);
            for (int a = 0; a < 3; ++a) {
                T acc = T(0);
                if (a < d.ndim)
                    for (int c = 0; c < d.ndim; ++c) acc += J[c * d.ndim + a] * s[c];
                v[a] = -acc;
            }
        } else {
            v[0] = -s[0];
            v[1] = -s[1];
            v[2] = -s[2];
        }
        const long long t = st ? st->t : 1;
        const T c1 = static_cast<T>(corr1[t]);
        const T c2 = static_cast<T>(corr2[t]);
        double mx = 0.0;
        bool bad = false;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (c >= d.ndim) {
                step.c[c][i] = T(0);
                continue;
            }
            const T mm = b1 * m.c[c][i] + omb1 * v[c];
            const T nn = b2 * nu.c[c][i] + omb2 * v[c] * v[c];
            m.c[c][i] = mm;
            nu.c[c][i] = nn;
            const T dir = (mm / c1) / (sqrt(nn / c2) + eps);
            const T sv = eta * dir;
            bad |= !isfinite(sv);
            const T cl = sv < -cap ? -cap : (cap < sv ? cap : sv);
            step.c[c][i] = cl;
            mx = fmax(mx, static_cast<double>(fabs(cl)));
        }
        if (bad && st) st->bad_step = 1;
        return {0.0, mx};
    }

    __device__ void finish(int, double, double mx) const {
        if (maxstep) atomic_max_nonneg(maxstep + (st ? st->slot : 0), mx);
    }
};

template <class T, int R>
struct ComposeSmoothOp {
    using Acc = T;
    static constexpr int C = 3;
    static constexpr bool kBox = false, kSum = false, kMax = false;
    GaussW<T> w;
    CPlanes3<T> step;
    CPlanes3<T> uin;
    Planes3<T> uout;
    Dims d;
    LoopState* st;

    __device__ bool skip() const {
        if (!st) return false;
        if (st->done) return true;
        if (st->bad_step) {  // diffeo.cpp:52-53: throw before composing
            if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
                st->err = 2;
                st->done = 1;
            }
            return true;
        }
        return false;
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const { return __ldg(w.norm[a] + i); }

    __device__ void load(int x, int y, int z, T v[3]) const {
        const int64_t i = d.idx(x, y, z);
        const T s0 = __ldg(step.c[0] + i), s1 = __ldg(step.c[1] + i);
        const T s2 = d.ndim == 3 ? __ldg(step.c[2] + i) : T(0);
        const Cell3<T> c = locate3<T>(d, x, y, z, s0, s1, s2);
        T q[3];
        lerp_field(c, uin.c[0], uin.c[1], uin.c[2], d.ndim, q);
        v[0] = s0 + q[0];
        v[1] = s1 + q[1];
        v[2] = d.ndim == 3 ? s2 + q[2] : T(0);
    }

    __device__ Red emit(int x, int y, int z, const T s[3]) const {
        const int64_t i = d.idx(x, y, z);
        uout.c[0][i] = s[0];
        uout.c[1][i] = s[1];
        uout.c[2][i] = s[2];
        return {0.0, 0.0};
    }

    __device__ void finish(int, double, double) const {
        if (st) st->nupdates += 1;
    }
};

template <class T, int R, int NC>
struct GaussOp {
    using Acc = T;
    static constexpr int C = NC;
    static constexpr bool kBox = false, kSum = false, kMax = false;
    GaussW<T> w;
    CPlanes3<T> in;
    Planes3<T> out;
    Dims d;

    __device__ bool skip() const { return false; }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const { return __ldg(w.norm[a] + i); }
    __device__ void load(int x, int y, int z, T v[NC]) const {
        const int64_t i = d.idx(x, y, z);
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = __ldg(in.c[c] + i);
    }
    __device__ Red emit(int x, int y, int z, const T s[NC]) const {
        const int64_t i = d.idx(x, y, z);
#pragma unroll
        for (int c = 0; c < NC; ++c) out.c[c][i] = s[c];
        return {0.0, 0.0};
    }
    __device__ void finish(int, double, double) const {}
};

// SVF update (pipeline.cpp:199-205): field + capped step, then sigma_warp
// smoothing; one counted update per iteration, nothing once the scale is done
template <class T, int R>
struct SvfUpdateOp {
    using Acc = T;
    static constexpr int C = 3;
    static constexpr bool kBox = false, kSum = false, kMax = false;
    GaussW<T> w;
    CPlanes3<T> v, step;
    Planes3<T> out;
    LoopState* st;
    Dims d;

    // diffeo-mode parity: a non-finite Adam step throws before the update
    // (pipeline.cpp:198-203 clamps NaN into the field; the next loss throws) —
    // here the update is skipped and the run fails with DFM_E_NUMERICAL
    __device__ bool skip() const {
        if (!st) return false;
        if (st->done) return true;
        if (st->bad_step) {
            if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
                st->err = 2;
                st->done = 1;
            }
            return true;
        }
        return false;
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const { return __ldg(w.norm[a] + i); }
    __device__ void load(int x, int y, int z, T s[3]) const {
        const int64_t i = d.idx(x, y, z);
#pragma unroll
        for (int c = 0; c < 3; ++c) s[c] = c < d.ndim ? v.c[c][i] + step.c[c][i] : T(0);
    }
    __device__ Red emit(int x, int y, int z, const T s[3]) const {
        const int64_t i = d.idx(x, y, z);
#pragma unroll
        for (int c = 0; c < 3; ++c) out.c[c][i] = s[c];
        return {0.0, 0.0};
    }
    __device__ void finish(int, double, double) const {
        if (st) st->nupdates += 1;
    }
};

// ---------------------------------------------------------------------------
// launch plumbing

template <int R, class Op>
size_t zmarch_smem() {
    using Acc = typename Op::Acc;
    const int WI = kTX + 2 * R, HI = kTY + 2 * R;
    return sizeof(Acc) * Op::C * (HI * WI + HI * kTX);
}

template <int R, class Op>
int run_zmarch(const Launch& L, const Op& op, Dims d) {
    ZGeom g;
    g.d = d;
    int tiles = 0;
    const int nchunks = zmarch_blocks(d, R, L.num_sms, &g.zchunk, &tiles);
    g.tiles_x = (d.nx + kTX - 1) / kTX;
    const size_t smem = zmarch_smem<R, Op>();
    kernel_setup(reinterpret_cast<const void*>(k_zmarch<R, Op>), kNT, smem);
    dim3 grid(tiles, nchunks);
    k_zmarch<R, Op><<<grid, kNT, smem, L.stream>>>(op, g);
    L.bump();
    return tiles * nchunks;
}

// radius dispatch: F(std::integral_constant<int,R>) for R in [RLO, kRMax]
template <int RLO, class F>
int with_radius(int R, F&& f) {
    switch (R) {
#define DFM_R(r)     \
    case r:          \
        if constexpr (r >= RLO) return f(std::integral_constant<int, r>{}); \
        break;
        DFM_R(0) DFM_R(1) DFM_R(2) DFM_R(3) DFM_R(4) DFM_R(5) DFM_R(6) DFM_R(7) DFM_R(8)
#undef DFM_R
    }
    return -1;
}

}  // namespace

int zmarch_blocks(Dims d, int R, int num_sms, int* zchunk, int* tiles) {
    const int tx = (d.nx + kTX - 1) / kTX, ty = (d.ny + kTY - 1) / kTY;
    *tiles = tx * ty;
    const int target = 3 * (num_sms > 0 ? num_sms : 148);
    int nchunks = (target + *tiles - 1) / *tiles;
    int minchunk = 4 > R ? 4 : R;
    if (minchunk > d.nz) minchunk = d.nz;
    int chunk = (d.nz + nchunks - 1) / nchunks;
    if (chunk < minchunk) chunk = minchunk;
    nchunks = (d.nz + chunk - 1) / chunk;
    *zchunk = chunk;
    return nchunks;
}

template <class T>
int launch_lncc_fwd(const Launch& L, int R, const T* F, const T* M, Dims d, Dims dm,
                    CPlanes3<T> u, T* const* coef, double* partials, const LoopState* st) {
    return with_radius<1>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        LnccFwdOp<T, RR> op;
        op.F = F;
        op.M = M;
        op.u = u;
        op.d = d;
        op.dm = dm;
        for (int k = 0; k < 4; ++k) op.coef[k] = coef ? coef[k] : nullptr;
        op.partials = partials;
        op.st = st;
        return run_zmarch<RR>(L, op, d);
    });
}

template <class T>
void launch_lncc_bwd(const Launch& L, int R, const T* F, const T* M, Dims d, Dims dm,
                     CPlanes3<T> u, const T* const* coef, Planes3<T> grad, const LoopState* st) {
    with_radius<1>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        LnccBwdOp<T, RR> op;
        op.F = F;
        op.M = M;
        op.u = u;
        op.d = d;
        op.dm = dm;
        for (int k = 0; k < 4; ++k) op.coef[k] = coef[k];
        op.grad = grad;
        op.st = st;
        return run_zmarch<RR>(L, op, d);
    });
}

template <class T>
void launch_smooth_adam(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> grad,
                        CPlanes3<T> u, Planes3<T> m, Planes3<T> nu, Planes3<T> step, Dims d,
                        AdamParams ap, LoopState* st, unsigned long long* maxstep_slots) {
    with_radius<0>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        SmoothAdamOp<T, RR> op;
        op.w = w;
        op.g = grad;
        op.u = u;
        op.m = m;
        op.nu = nu;
        op.step = step;
        op.d = d;
        op.b1 = T(ap.b1);
        op.omb1 = T(1.0 - ap.b1);
        op.b2 = T(ap.b2);
        op.omb2 = T(1.0 - ap.b2);
        op.eps = T(ap.eps);
        op.eta = T(ap.eta);
        op.cap = T(ap.cap);
        op.corr1 = ap.corr1;
        op.corr2 = ap.corr2;
        op.use_jac = ap.use_jac;
        op.st = st;
        op.maxstep = maxstep_slots;
        return run_zmarch<RR>(L, op, d);
    });
}

template <class T>
void launch_compose_smooth(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> step,
                           CPlanes3<T> u_in, Planes3<T> u_out, Dims d, LoopState* st) {
    with_radius<0>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        ComposeSmoothOp<T, RR> op;
        op.w = w;
        op.step = step;
        op.uin = u_in;
        op.uout = u_out;
        op.d = d;
        op.st = st;
        return run_zmarch<RR>(L, op, d);
    });
}

template <class T>
void launch_gauss_fused(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> in,
                        Planes3<T> out, int ncomp, Dims d) {
    with_radius<0>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        if (ncomp == 1) {
            GaussOp<T, RR, 1> op;
            op.w = w;
            op.in = in;
            op.out = out;
            op.d = d;
            return run_zmarch<RR>(L, op, d);
        }
        GaussOp<T, RR, 3> op;
        op.w = w;
        op.in = in;
        op.out = out;
        op.d = d;
        return run_zmarch<RR>(L, op, d);
    });
}

template <class T>
void launch_svf_update(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> v,
                       CPlanes3<T> step, Planes3<T> out, Dims d, LoopState* st) {
    with_radius<0>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        SvfUpdateOp<T, RR> op;
        op.w = w;
        op.v = v;
        op.step = step;
        op.out = out;
        op.st = st;
        op.d = d;
        return run_zmarch<RR>(L, op, d);
    });
}

#define DFM_INST_S(T)                                                                          \
    template int launch_lncc_fwd<T>(const Launch&, int, const T*, const T*, Dims, Dims,        \
                                    CPlanes3<T>, T* const*, double*, const LoopState*);        \
    template void launch_lncc_bwd<T>(const Launch&, int, const T*, const T*, Dims, Dims,       \
                                     CPlanes3<T>, const T* const*, Planes3<T>,                 \
                                     const LoopState*);                                        \
    template void launch_smooth_adam<T>(const Launch&, int, const GaussW<T>&, CPlanes3<T>,     \
                                        CPlanes3<T>, Planes3<T>, Planes3<T>, Planes3<T>, Dims, \
                                        AdamParams, LoopState*, unsigned long long*);          \
    template void launch_compose_smooth<T>(const Launch&, int, const GaussW<T>&, CPlanes3<T>,  \
                                           CPlanes3<T>, Planes3<T>, Dims, LoopState*);         \
    template void launch_gauss_fused<T>(const Launch&, int, const GaussW<T>&, CPlanes3<T>,     \
                                        Planes3<T>, int, Dims);                                \
    template void launch_svf_update<T>(const Launch&, int, const GaussW<T>&, CPlanes3<T>,      \
                                       CPlanes3<T>, Planes3<T>, Dims, LoopState*);

DFM_INST_S(float)
DFM_INST_S(double)

}  // namespace dfm
