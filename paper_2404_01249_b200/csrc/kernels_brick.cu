// kernels_brick.cu — brick-tiled stencil kernels of the hot loop for the
// small pyramid levels.
//
// The plane-streaming kernels (kernels_tma.cu) march each CTA through a long
// z-chunk, which is the right shape for a 160x192x224 volume but latency-bound
// on the 40x48x56 and 80x96x112 levels: there a CTA walks only a few planes,
// each a serial chain of TMA wait -> x pass -> barrier -> y pass -> z ring.
// Here a CTA owns an 8 x BY x 8 brick (BY = 4 by default) instead and does
// every pass for the whole brick in parallel:
//   1. stage the haloed brick (8+2R)^3 of the op's raw channels into shared
//      memory (all loads independent: one L2 round trip; zero outside the
//      volume, which together with the per-position renormalisation factors
//      reproduces the reference's clipped windows / truncated Gaussians);
//   2. x pass over (8+2R)^2 rows x 8 columns -> shared;
//   3. y pass over (8+2R) planes x 8 x 8 -> shared (reuses the staging buffer);
//   4. z pass + the op's per-voxel epilogue for the 512 voxels of the brick.
// Three barriers per launch, no serial plane loop.  The per-voxel arithmetic
// is loop_ops.cuh, shared with the plane-streaming kernels.
//
// Buffers the loop rewrites (W, G, coefficients, grad, step, u) are read with
// plain coherent loads, never ld.global.nc: the persistent solvers below read
// them within one launch, after a grid barrier (k_persist) or after an
// acquire on their neighbour bricks' phase counters (k_persist_nb, the
// default for the config-1 coarse level).
//
// Ops (same roles as in kernels_tma.cu):
//   LnccFwdB    F, W          -> 4 window coefficients, cc^2 partials (+ monitor)
//   LnccBwdB    coefficients  -> grad = dW * G
//   SmoothAdamB grad          -> m, nu, capped step, max |step|
//   ComposeB    step, u       -> u' = smooth(step + u(x+step)), W, G
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <type_traits>

#include <cooperative_groups.h>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"
#include "loop_ops.cuh"

namespace dfm {

namespace {

#ifndef DFM_BRICK_BY
#define DFM_BRICK_BY 4
#endif
#ifndef DFM_BRICK_NTB
#define DFM_BRICK_NTB 256
#endif
constexpr int NTB = DFM_BRICK_NTB;
constexpr int BX = 8, BY = DFM_BRICK_BY, BZ = 8;
constexpr size_t kBrickSmemMax = 227 * 1024;

struct BG {
    Dims d;
    int nbx, nby;
};

#ifndef DFM_BRICK_XQUAD
#define DFM_BRICK_XQUAD 1
#endif
#ifndef DFM_BRICK_YPAIR
#define DFM_BRICK_YPAIR 1
#endif

// ops whose stage is a plain load of NR planes of T (Op::vsrc(c), Op::vnc(c)
// = read-only) stage whole rows with 128-bit loads when the level allows it
template <class Op, class = void>
struct VecStageB {
    static constexpr bool value = false;
    using Src = typename Op::Raw;
};
template <class Op>
struct VecStageB<Op, std::void_t<decltype(&Op::vsrc)>> {
    static constexpr bool value = true;
    using Src = typename Op::Src;
};

constexpr int round_up_b(int v, int m) { return (v + m - 1) / m * m; }

template <class Op>
struct BrickLayout {
    using A = typename Op::Acc;
    using S = typename Op::Raw;
    using G = typename VecStageB<Op>::Src;
    static constexpr int R = Op::R, C = Op::C, NR = Op::NR;
    static constexpr int HX = BX + 2 * R, HY = BY + 2 * R, HZ = BZ + 2 * R;
    // Staged rows start PADL columns left of the brick (PADL >= R, a whole
    // number of 128-bit chunks of the global rows, so rows stage as aligned
    // vectors) and are padded to HXP.  Quad x pass (DFM_BRICK_XQUAD): a thread
    // filters 4 consecutive columns from one register window of 4 + 2R
    // staged values per channel, read with 128-bit loads from the aligned
    // position MIS values left of the window.
    static constexpr int VT = 16 / int(sizeof(G));  // global values per 128-bit load
    static constexpr int VEC = 16 / int(sizeof(S));  // staged values per 128-bit load
    static constexpr int W4 = 4 + 2 * R;
    // padded row length for a left pad PL: long enough for the stage and the
    // quad windows, a whole number of 128-bit chunks, and a row stride of 8 or
    // 24 words mod 32, so the 8 lanes of each 128-bit shared-load phase of the
    // quad x pass (4 rows x 2 quads) hit distinct banks
    static constexpr int hxp(int PL) {
        const int mis = (PL - R) % VEC, nv = (W4 + mis + VEC - 1) / VEC, q0 = PL - R - mis;
        const int n = PL + BX + R > q0 + (BX - 4) + nv * VEC ? PL + BX + R
                                                             : q0 + (BX - 4) + nv * VEC;
        const int step = VT > VEC ? VT : VEC;
        int h = round_up_b(n, step);
        for (int k = 0; k < 8; ++k) {
            const int w = (h * int(sizeof(S)) / 4) % 32;
            if (w == 8 || w == 24) break;
            h += step;
        }
        return h;
    }
    // the vector stage's aligned left pad for radii >= 3 (the sigma_grad
    // smooth+Adam: stage 3.3 -> 1.9 us per brick phase) where its staged rows
    // fit 48 KB; at radius 2 (LNCC, sigma_warp) the scalar stage measured as
    // fast or faster
    static constexpr bool kVec =
        DFM_BRICK_XQUAD != 0 && VecStageB<Op>::value && R >= 3 &&
        size_t(NR) * HY * HZ * hxp(round_up_b(R, VT)) * sizeof(S) <= 48 * 1024;
    static constexpr int PADL = kVec ? round_up_b(R, VT) : R;
    static constexpr int MIS = (PADL - R) % VEC;
    static constexpr int NV4 = (W4 + MIS + VEC - 1) / VEC;  // vector loads per window
    static constexpr int XQ0 = PADL - R - MIS;              // first quad's aligned start
    static constexpr int HXP = DFM_BRICK_XQUAD ? hxp(PADL) : HX;
    // 128-bit chunks per staged row (vector stage): the columns the x pass uses
    static constexpr int NCH = (PADL + BX + R + VT - 1) / VT;
    static constexpr int nS = HXP * HY * HZ;  // per staged channel (padded rows)
    static constexpr int nX = HZ * HY * BX;  // per channel, x-pass output
    static constexpr int nY = HZ * BY * BX;  // per channel, y-pass output
    static constexpr size_t bX = (static_cast<size_t>(C) * nX * sizeof(A) + 15) / 16 * 16;
    static constexpr size_t bS = static_cast<size_t>(NR) * nS * sizeof(S);
    static constexpr size_t bY = static_cast<size_t>(C) * nY * sizeof(A);
    static constexpr size_t bytes = bX + (bS > bY ? bS : bY);
};

__device__ __forceinline__ float4 ld_vec4(const float* p, bool nc) {
    return nc ? __ldg(reinterpret_cast<const float4*>(p)) : *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ double2 ld_vec4(const double* p, bool nc) {
    return nc ? __ldg(reinterpret_cast<const double2*>(p)) : *reinterpret_cast<const double2*>(p);
}

// ops with centre operands (Op::Center, Op::load_center) have them loaded
// before the stage, so their latency hides behind the stage round trip
struct NoCenterB {};
template <class Op, class = void>
struct CenterOfB {
    using type = NoCenterB;
    static constexpr bool value = false;
};
template <class Op>
struct CenterOfB<Op, std::void_t<typename Op::Center>> {
    using type = typename Op::Center;
    static constexpr bool value = true;
};

// One brick of one op: stage, x, y, z passes, per-voxel epilogue and the
// CTA reduction; op.finish(b, ...) records brick b's partial.  Ends with the
// CTA's threads synchronised (smem reusable).
#ifndef DFM_NB_TRACE
#define DFM_NB_TRACE -1
#endif
#if DFM_NB_TRACE >= 0
__device__ long long g_nb_bt[1024][4][6];  // brick_body stage clocks (trace builds)
#define DFM_BT(k)                                                               \
    do {                                                                        \
        if (trace >= 0 && threadIdx.x == 0 && blockIdx.x < 1024)                \
            g_nb_bt[blockIdx.x][trace][k] = clock64();                          \
    } while (0)
#else
#define DFM_BT(k) \
    do {          \
    } while (0)
#endif

struct NoPreStage {
    __device__ bool operator()() const { return true; }
};

// pre(): called by every thread after the centre loads are issued and before
// the stage (the persistent solver waits for its neighbours there, so the
// own-brick centre loads overlap the wait); false -> return false at once
template <class Op, int NTB, class Pre = NoPreStage>
__device__ __forceinline__ bool brick_body(const Op& op, const BG& g, int b, unsigned char* smem,
                                           double* s_red, const Pre& pre = Pre{},
                                           int trace = -1) {
    (void)trace;
    using Lay = BrickLayout<Op>;
    using A = typename Op::Acc;
    using S = typename Op::Raw;
    constexpr int R = Op::R, C = Op::C, NR = Op::NR, K = 2 * R + 1;
    constexpr int HX = Lay::HX, HY = Lay::HY, HXP = Lay::HXP;
    constexpr int nS = Lay::nS, nX = Lay::nX, nY = Lay::nY;
    constexpr int nE = HX * HY * Lay::HZ;  // staged elements per channel (scalar stage)
    A* sX = reinterpret_cast<A*>(smem);
    S* sS = reinterpret_cast<S*>(smem + Lay::bX);
    A* sY = reinterpret_cast<A*>(smem + Lay::bX);  // aliases sS after the x pass

    const Dims& d = g.d;
    const int tid = threadIdx.x;
    const int bid = b;
    const int x0 = (b % g.nbx) * BX;
    b /= g.nbx;
    const int y0 = (b % g.nby) * BY;
    const int z0 = (b / g.nby) * BZ;

    // 0. centre operands of this thread's output voxels
    constexpr int IZ = BZ * BY * BX / NTB;
    static_assert(IZ * NTB == BZ * BY * BX, "brick must be a multiple of the CTA size");
    using Cen = CenterOfB<Op>;
    typename Cen::type cen[IZ];
    if constexpr (Cen::value) {
#pragma unroll
        for (int k = 0; k < IZ; ++k) {
            const int e = tid + k * NTB;
            const int xl = e % BX, t = e / BX, yl = t % BY, zl = t / BY;
            const int gx = x0 + xl, gy = y0 + yl, gz = z0 + zl;
            if (gx < d.nx && gy < d.ny && gz < d.nz) op.load_center(gx, gy, gz, cen[k]);
        }
    }
    if (!pre()) return false;
    DFM_BT(0);
    // 1. stage: the loads of a batch of elements are all issued before any is
    // stored (one L2 round trip per batch instead of one per element)
    constexpr int PADL = Lay::PADL;
    bool vec = false;
    if constexpr (Lay::kVec) {
        // rows as aligned 128-bit chunks: chunk starts are multiples of VT and
        // so is nx, so a chunk is wholly inside or wholly outside the volume
        vec = d.nx % Lay::VT == 0;
#pragma unroll
        for (int c = 0; c < NR; ++c)
            vec = vec && (reinterpret_cast<uintptr_t>(op.vsrc(c)) & 15) == 0;
    }
    if (vec) {
        if constexpr (Lay::kVec) {
            using G = typename Lay::G;
            using GV = typename std::conditional<sizeof(G) == 4, float4, double2>::type;
            constexpr int VT = Lay::VT, NCH = Lay::NCH, NRW = HY * Lay::HZ;
            constexpr int NI = NR * NRW * NCH, II = (NI + NTB - 1) / NTB, SBV = 8;
            for (int b0 = 0; b0 < II; b0 += SBV) {
                GV v[SBV];
#pragma unroll
                for (int k = 0; k < SBV; ++k) {
                    const int e = tid + (b0 + k) * NTB;
                    const int ch = e % NCH, t = (e / NCH) % NRW, c = e / (NCH * NRW);
                    const int yl = t % HY, zl = t / HY;
                    const int gx = x0 - PADL + VT * ch, gy = y0 - R + yl, gz = z0 - R + zl;
                    if (b0 + k < II && e < NI && gx >= 0 && gx + VT <= d.nx && gy >= 0 &&
                        gy < d.ny && gz >= 0 && gz < d.nz) {
                        v[k] = ld_vec4(op.vsrc(c) + d.idx32(gx, gy, gz), Op::vnc(c));
                    } else {
                        v[k] = GV{};
                    }
                }
#pragma unroll
                for (int k = 0; k < SBV; ++k) {
                    const int e = tid + (b0 + k) * NTB;
                    if (b0 + k < II && e < NI) {
                        const int ch = e % NCH, t = (e / NCH) % NRW, c = e / (NCH * NRW);
                        S* o = sS + c * nS + t * HXP + VT * ch;
                        if constexpr (sizeof(G) == 4) {
                            const float4 f = v[k];
                            if constexpr (sizeof(S) == 4) {
                                *reinterpret_cast<float4*>(o) = f;
                            } else {
                                reinterpret_cast<double2*>(o)[0] =
                                    make_double2(static_cast<double>(f.x), static_cast<double>(f.y));
                                reinterpret_cast<double2*>(o)[1] =
                                    make_double2(static_cast<double>(f.z), static_cast<double>(f.w));
                            }
                        } else {
                            *reinterpret_cast<double2*>(o) = v[k];
                        }
                    }
                }
            }
        }
    } else {
        constexpr int HW = BX + 2 * R;  // the columns the x pass reads
        const bool inner = x0 - R >= 0 && x0 + BX + R <= d.nx && y0 - R >= 0 &&
                           y0 + BY + R <= d.ny && z0 - R >= 0 && z0 + BZ + R <= d.nz;
        constexpr int IS = (nE + NTB - 1) / NTB, SB = Op::kStageBatch;
        for (int b0 = 0; b0 < IS; b0 += SB) {
            S v[SB][NR];
#pragma unroll
            for (int k = 0; k < SB; ++k) {
                const int e = tid + (b0 + k) * NTB;
                const int xl = e % HW, t = e / HW, yl = t % HY, zl = t / HY;
                const int gx = x0 - R + xl, gy = y0 - R + yl, gz = z0 - R + zl;
                if (b0 + k < IS && e < nE &&
                    (inner || (gx >= 0 && gx < d.nx && gy >= 0 && gy < d.ny && gz >= 0 &&
                               gz < d.nz))) {
                    op.stage(gx, gy, gz, v[k]);
                } else {
#pragma unroll
                    for (int c = 0; c < NR; ++c) v[k][c] = S(0);
                }
            }
#pragma unroll
            for (int k = 0; k < SB; ++k) {
                const int e = tid + (b0 + k) * NTB;
                if (b0 + k < IS && e < nE) {
                    const int xl = e % HW, t = e / HW;
#pragma unroll
                    for (int c = 0; c < NR; ++c)
                        sS[c * nS + t * HXP + (PADL - R) + xl] = v[k][c];
                }
            }
        }
    }
    __syncthreads();
    DFM_BT(1);
    // 2. x pass
    if constexpr (DFM_BRICK_XQUAD != 0) {
        // the same op.xpass arithmetic per output, its operands from a
        // register window instead of 2R+1 shared loads per output
        constexpr int W4 = Lay::W4, NV4 = Lay::NV4, VEC = Lay::VEC, NQ = BX / 4;
        static_assert(BX % 4 == 0, "quad x pass: whole quads per brick row");
        constexpr int nQ = Lay::HZ * HY * NQ;
        constexpr int IQ = (nQ + NTB - 1) / NTB;
#pragma unroll
        for (int k = 0; k < IQ; ++k) {
            const int e = tid + k * NTB;
            if (e < nQ) {
                const int q = e % NQ, t = e / NQ;  // t = zl*HY + yl
                S wv[NR * NV4 * VEC];
#pragma unroll
                for (int c = 0; c < NR; ++c) {
                    const S* src = sS + c * nS + t * HXP + Lay::XQ0 + 4 * q;
#pragma unroll
                    for (int j = 0; j < NV4; ++j) {
                        if constexpr (sizeof(S) == 4) {
                            const float4 f = reinterpret_cast<const float4*>(src)[j];
                            S* o = wv + c * NV4 * VEC + 4 * j;
                            o[0] = f.x, o[1] = f.y, o[2] = f.z, o[3] = f.w;
                        } else {
                            const double2 f = reinterpret_cast<const double2*>(src)[j];
                            S* o = wv + c * NV4 * VEC + 2 * j;
                            o[0] = f.x, o[1] = f.y;
                        }
                    }
                }
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                    const int xl = 4 * q + o, gx = x0 + xl;
                    A v[C];
                    op.xpass(wv + Lay::MIS + o, NV4 * VEC, v);
                    const A nxv = gx < d.nx ? op.nrm(0, gx) : A(0);
#pragma unroll
                    for (int c = 0; c < C; ++c) sX[c * nX + t * BX + xl] = v[c] * nxv;
                }
            }
        }
        (void)W4;
    } else {
        constexpr int IX = (nX + NTB - 1) / NTB;
#pragma unroll
        for (int k = 0; k < IX; ++k) {
            const int e = tid + k * NTB;
            if (e < nX) {
                const int xl = e % BX, t = e / BX;  // t = zl*HY + yl
                const int gx = x0 + xl;
                A v[C];
                op.xpass(sS + t * HXP + (PADL - R) + xl, nS, v);
                const A nxv = gx < d.nx ? op.nrm(0, gx) : A(0);
#pragma unroll
                for (int c = 0; c < C; ++c) sX[c * nX + e] = v[c] * nxv;
            }
        }
    }
    __syncthreads();
    DFM_BT(2);
    // 3. y pass (into the dead staging buffer).  DFM_BRICK_YPAIR: a thread
    // filters two consecutive rows from K+1 loads per channel (one round of
    // items instead of 1.5-1.75 rounds), the same sums per output.  fp32
    // accumulators only (A 0.82 -> 0.71, C 0.72 -> 0.55 us per brick phase;
    // the fp64 passes measured slower: F 0.84 -> 0.90, B 1.15 -> 1.28)
    if constexpr (DFM_BRICK_YPAIR != 0 && BY % 2 == 0 && sizeof(A) == 4) {
        constexpr int nY2 = nY / 2, IY2 = (nY2 + NTB - 1) / NTB;
#pragma unroll
        for (int k = 0; k < IY2; ++k) {
            const int e = tid + k * NTB;
            if (e < nY2) {
                const int xl = e % BX, t = e / BX, yp = t % (BY / 2), zl = t / (BY / 2);
                const int yl = 2 * yp, gy = y0 + yl;
                const A ny0 = gy < d.ny ? op.nrm(1, gy) : A(0);
                const A ny1 = gy + 1 < d.ny ? op.nrm(1, gy + 1) : A(0);
                const A* src = sX + (zl * HY + yl) * BX + xl;
                const int o = (zl * BY + yl) * BX + xl;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    A v[K + 1];
#pragma unroll
                    for (int j = 0; j <= K; ++j) v[j] = src[c * nX + j * BX];
                    A a0 = A(0), a1 = A(0);
#pragma unroll
                    for (int j = 0; j < K; ++j) a0 += op.wgt(1, j) * v[j];
#pragma unroll
                    for (int j = 0; j < K; ++j) a1 += op.wgt(1, j) * v[j + 1];
                    sY[c * nY + o] = a0 * ny0;
                    sY[c * nY + o + BX] = a1 * ny1;
                }
            }
        }
    } else {
        constexpr int IY = (nY + NTB - 1) / NTB;
#pragma unroll
        for (int k = 0; k < IY; ++k) {
            const int e = tid + k * NTB;
            if (e < nY) {
                const int xl = e % BX, t = e / BX, yl = t % BY, zl = t / BY;
                const int gy = y0 + yl;
                const A nyv = gy < d.ny ? op.nrm(1, gy) : A(0);
                const A* src = sX + (zl * HY + yl) * BX + xl;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    A a = A(0);
#pragma unroll
                    for (int j = 0; j < K; ++j) a += op.wgt(1, j) * src[c * nX + j * BX];
                    sY[c * nY + e] = a * nyv;
                }
            }
        }
    }
    __syncthreads();
    DFM_BT(3);
    // 4. z pass + per-voxel epilogue (both voxels of a thread in flight together)
    const typename Op::Prol pr = op.prologue();
    double rsum = 0.0, rmax = 0.0;
#pragma unroll
    for (int k = 0; k < IZ; ++k) {
        const int e = tid + k * NTB;
        const int xl = e % BX, t = e / BX, yl = t % BY, zl = t / BY;
        const int gx = x0 + xl, gy = y0 + yl, gz = z0 + zl;
        if (gx < d.nx && gy < d.ny && gz < d.nz) {
            const A nzv = op.nrm(2, gz);
            const A* src = sY + e;
            A sv[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                A a = A(0);
#pragma unroll
                for (int j = 0; j < K; ++j) a += op.wgt(2, j) * src[c * nY + j * (BY * BX)];
                sv[c] = a * nzv;
            }
            Red2 r;
            if constexpr (Cen::value)
                r = op.emit(gx, gy, gz, sv, pr, cen[k]);
            else
                r = op.emit(gx, gy, gz, sv, pr);
            rsum += r.sum;
            rmax = fmax(rmax, r.mx);
        }
    }
    DFM_BT(4);
    if constexpr (Op::kSum || Op::kMax) {
        const double bs = Op::kSum ? bsum<NTB>(rsum, s_red) : 0.0;
        const double bm = Op::kMax ? bmax<NTB>(rmax, s_red) : 0.0;
        if (tid == 0) op.finish(bid, bs, bm, pr);
    } else {
        if (tid == 0 && bid == 0) op.finish(0, 0.0, 0.0, pr);
        __syncthreads();
    }
    DFM_BT(5);
    return true;
}

template <class Op>
__global__ void __launch_bounds__(NTB, 2) k_brick(const __grid_constant__ Op op, const BG g) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_red[32];
    pdl_wait();
    if (op.skip()) return;
    brick_body<Op, NTB>(op, g, blockIdx.x, smem, s_red);
    pdl_trigger();  // the successor may launch while the last bricks finish
    if constexpr (Op::kSum) {
        if (op.mon.st)
            monitor_tail<NTB>(op.mon, op.partials, gridDim.x,
                              static_cast<double>(g.d.nx) * g.d.ny * g.d.nz, s_red);
    }
}

struct NoProl {};

// similarity.cpp:122-168 — box moments (fp64) of F and W = M(x+u), the window
// coefficients and cc^2.  FS: the level's F statistics (muF, vF) come
// precomputed (FStatsB) and only the three W moments are summed.
template <class T, int R_, bool FS = false>
struct LnccFwdB {
    using Acc = double;
    using Raw = double;
    using Prol = NoProl;
    static constexpr int R = R_, C = FS ? 3 : 5, NR = 2, kStageBatch = 8;
    static constexpr bool kSum = true, kMax = false;
    const T* F;
    const T* W;
    const double* fstat;  // FS: 2 planes muF, vF
    T* coef;  // 4 planes; nullptr -> value only
    double* partials;
    const LoopState* st;
    MonitorArgs mon;
    Dims d;

    __device__ bool skip() const { return st && st->done; }
    __device__ void stage(int x, int y, int z, double v[2]) const {
        const int i = d.idx32(x, y, z);
        v[0] = static_cast<double>(__ldg(F + i));
        v[1] = static_cast<double>(W[i]);
    }
    using Src = T;  // vector stage: the same loads as stage()
    __device__ const T* vsrc(int c) const { return c == 0 ? F : W; }
    __device__ static constexpr bool vnc(int c) { return c == 0; }
    __device__ void xpass(const double* p, int cs, double v[C]) const {
        if constexpr (FS) {
            double a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) {
                const double f = p[j], w = p[cs + j];
                a0 += w;
                a1 += w * w;
                a2 += f * w;
            }
            v[0] = a0;
            v[1] = a1;
            v[2] = a2;
        } else {
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) {
                const double f = p[j], w = p[cs + j];
                a0 += f;
                a1 += w;
                a2 += f * f;
                a3 += w * w;
                a4 += f * w;
            }
            v[0] = a0;
            v[1] = a1;
            v[2] = a2;
            v[3] = a3;
            v[4] = a4;
        }
    }
    __device__ double wgt(int, int) const { return 1.0; }
    __device__ double nrm(int, int) const { return 1.0; }
    __device__ Prol prologue() const { return {}; }
    struct Center {
        double muF, vF;
    };
    __device__ void load_center(int x, int y, int z, Center& c) const {
        if constexpr (FS) {
            const int i = d.idx32(x, y, z);
            c.muF = __ldg(fstat + i);
            c.vF = __ldg(fstat + d.n + i);
        }
    }
    __device__ Red2 emit(int x, int y, int z, const double s[C], const Prol&,
                         const Center& c) const {
        const double inv_n = window_inv<R>(x, y, z, d);
        const int i = d.idx32(x, y, z);
        LnccCoef k;
        if constexpr (FS)
            k = lncc_coef_f(c.muF, c.vF, s[0], s[1], s[2], inv_n);
        else
            k = lncc_coef(s, inv_n);
        if (coef) {
            coef[i] = static_cast<T>(k.an);
            coef[d.n + i] = static_cast<T>(k.amu);
            coef[2 * d.n + i] = static_cast<T>(k.bn);
            coef[3 * d.n + i] = static_cast<T>(k.bmu);
        }
        return {k.cc2, 0.0};
    }
    __device__ void finish(int blk, double s, double, const Prol&) const { partials[blk] = s; }
};

// similarity.cpp:145-150, F half, once per level: muF and vF per voxel
template <class T, int R_>
struct FStatsB {
    using Acc = double;
    using Raw = double;
    using Prol = NoProl;
    static constexpr int R = R_, C = 2, NR = 1, kStageBatch = 8;
    static constexpr bool kSum = false, kMax = false;
    const T* F;
    double* fstat;
    Dims d;

    __device__ bool skip() const { return false; }
    __device__ void stage(int x, int y, int z, double v[1]) const {
        v[0] = static_cast<double>(__ldg(F + d.idx32(x, y, z)));
    }
    using Src = T;
    __device__ const T* vsrc(int) const { return F; }
    __device__ static constexpr bool vnc(int) { return true; }
    __device__ void xpass(const double* p, int, double v[2]) const {
        double a0 = 0, a1 = 0;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
            a0 += p[j];
            a1 += p[j] * p[j];
        }
        v[0] = a0;
        v[1] = a1;
    }
    __device__ double wgt(int, int) const { return 1.0; }
    __device__ double nrm(int, int) const { return 1.0; }
    __device__ Prol prologue() const { return {}; }
    __device__ Red2 emit(int x, int y, int z, const double s[2], const Prol&) const {
        const double inv_n = window_inv<R>(x, y, z, d);
        double muF, vF;
        lncc_fstats(s[0], s[1], inv_n, muF, vF);
        const int i = d.idx32(x, y, z);
        fstat[i] = muF;
        fstat[d.n + i] = vF;
        return {0.0, 0.0};
    }
    __device__ void finish(int, double, double, const Prol&) const {}
};

// similarity.cpp:170-189 — box sums of the 4 coefficients, dW, grad = dW * G
template <class T, int R_>
struct LnccBwdB {
    // coefficient box sums in fp64 unless DFM_BWD_ACC32 (as LnccBwd2)
    using Acc = typename std::conditional<(DFM_BWD_ACC32 != 0) && sizeof(T) == 4, float,
                                          double>::type;
    using Raw = Acc;
    using Prol = NoProl;
    static constexpr int R = R_, C = 4, NR = 4, kStageBatch = 8;
    static constexpr bool kSum = false, kMax = false;
    const T* coef;  // 4 planes
    const T* F;
    const T* W;
    const T* G;  // 3 planes
    T* grad;     // 3 planes
    double m2n;  // -2 / N
    const LoopState* st;
    Dims d;

    __device__ bool skip() const { return st && st->done; }
    __device__ void stage(int x, int y, int z, Acc v[4]) const {
        const int i = d.idx32(x, y, z);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = static_cast<Acc>(coef[k * d.n + i]);
    }
    using Src = T;
    __device__ const T* vsrc(int c) const { return coef + static_cast<size_t>(c) * d.n; }
    __device__ static constexpr bool vnc(int) { return false; }
    __device__ void xpass(const Acc* p, int cs, Acc v[4]) const {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            Acc a = Acc(0);
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) a += p[c * cs + j];
            v[c] = a;
        }
    }
    __device__ Acc wgt(int, int) const { return Acc(1); }
    __device__ Acc nrm(int, int) const { return Acc(1); }
    __device__ Prol prologue() const { return {}; }
    struct Center {
        T f, w, g[3];
    };
    __device__ void load_center(int x, int y, int z, Center& c) const {
        const int i = d.idx32(x, y, z);
        c.f = __ldg(F + i);
        c.w = W[i];
#pragma unroll
        for (int k = 0; k < 3; ++k) c.g[k] = G[k * d.n + i];
    }
    __device__ Red2 emit(int x, int y, int z, const Acc sa[4], const Prol&,
                         const Center& c) const {
        const double s[4] = {static_cast<double>(sa[0]), static_cast<double>(sa[1]),
                             static_cast<double>(sa[2]), static_cast<double>(sa[3])};
        const int i = d.idx32(x, y, z);
        const double f = static_cast<double>(c.f), w = static_cast<double>(c.w);
        const double dW = lncc_dw(m2n, f, w, s);
        grad[i] = static_cast<T>(dW * static_cast<double>(c.g[0]));
        grad[d.n + i] = static_cast<T>(dW * static_cast<double>(c.g[1]));
        grad[2 * d.n + i] = static_cast<T>(dW * static_cast<double>(c.g[2]));
        return {0.0, 0.0};
    }
    __device__ void finish(int, double, double, const Prol&) const {}
};

// Gaussian x pass shared by the smoothing ops (interp.cpp:110-151)
template <class T, int R>
__device__ __forceinline__ void gauss_xpass(const GaussW<T>& w, const T* p, int cs, T v[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const T* q = p + c * cs;
        T a0 = T(0), a1 = T(0);
#pragma unroll
        for (int j = 0; j < 2 * R + 1; j += 2) a0 += w.taps[0][j] * q[j];
#pragma unroll
        for (int j = 1; j < 2 * R + 1; j += 2) a1 += w.taps[0][j] * q[j];
        v[c] = a0 + a1;
    }
}

// pipeline.cpp:182-186 + optim.cpp:22-42 + diffeo.cpp:47-57: sigma_grad
// smoothing, v = -g, Adam, capped step, max |step|
template <class T, int R_, int CAPH_ = 0>
struct SmoothAdamB {
    using Acc = T;
    using Raw = T;
    static constexpr int R = R_, C = 3, NR = 3, kStageBatch = 8;
    static constexpr bool kSum = false, kMax = true;
    const T* grad;  // 3 planes
    GaussW<T> w;
    T* m;
    T* nu;
    T* step;        // CAPH_ > 0: receives the composed field c = step + u(x+step)
    const T* uin;   // CAPH_ > 0: the current field
    AdamK<T> ak;
    const double* corr1;
    const double* corr2;
    LoopState* st;
    unsigned long long* maxstep;
    Dims d;
    struct Prol {
        T ic1, ic2;
        int slot;
    };

    __device__ bool skip() const { return st && st->done; }
    __device__ void stage(int x, int y, int z, T v[3]) const {
        const int i = d.idx32(x, y, z);
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] = grad[k * d.n + i];
    }
    using Src = T;
    __device__ const T* vsrc(int c) const { return grad + static_cast<size_t>(c) * d.n; }
    __device__ static constexpr bool vnc(int) { return false; }
    __device__ void xpass(const T* p, int cs, T v[3]) const { gauss_xpass<T, R>(w, p, cs, v); }
    __device__ T wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ T nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const {
        Prol p;
        const long long t = st ? st->t : 1;
        p.ic1 = static_cast<T>(1.0 / corr1[t]);
        p.ic2 = static_cast<T>(1.0 / corr2[t]);
        p.slot = st ? st->slot : 0;
        return p;
    }
    struct Center {
        T m[3], nu[3];
    };
    __device__ void load_center(int x, int y, int z, Center& c) const {
        const int i = d.idx32(x, y, z);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c.m[k] = m[k * d.n + i];
            c.nu[k] = nu[k * d.n + i];
        }
    }
    __device__ Red2 emit(int x, int y, int z, const T s[3], const Prol& p,
                         const Center& c) const {
        const int i = d.idx32(x, y, z);
        T mx = T(0);
        bool bad = false;
        T cl[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            T mm = c.m[k], nn = c.nu[k];
            cl[k] = adam_component(ak, s[k], mm, nn, p.ic1, p.ic2, bad);
            m[k * d.n + i] = mm;
            nu[k * d.n + i] = nn;
            mx = fmax(mx, fabs(cl[k]));
        }
        if constexpr (CAPH_ > 0) {  // pointwise compose (interp.cpp:269-289)
            T cv[3];
            compose_at<T, CAPH_>(uin, d, x, y, z, cl, cv);
#pragma unroll
            for (int k = 0; k < 3; ++k) step[k * d.n + i] = cv[k];
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) step[k * d.n + i] = cl[k];
        }
        if (bad && st) st->bad_step = 1;
        return {0.0, static_cast<double>(mx)};
    }
    __device__ void finish(int, double, double mx, const Prol& p) const {
        if (maxstep) atomic_max_nonneg(maxstep + p.slot, mx);
    }
};

// diffeo.cpp:60-62 + interp.cpp:269-289: u' = step + u(x+step) (clamp-to-edge
// trilinear), sigma_warp smoothing, then W = M(x+u'), G = grad M(x+u')
// (similarity.cpp:25-45) for the next loss evaluation.  The u gather reads
// global memory (L1/L2), so any step cap is supported.
template <class T, int R_>
struct ComposeB {
    using Acc = T;
    using Raw = T;
    using Prol = NoProl;
    static constexpr int R = R_, C = 3, NR = 3, kStageBatch = 4;
    static constexpr bool kSum = false, kMax = false;
    const T* step;  // 3 planes
    const T* u;     // 3 planes
    GaussW<T> w;
    T* uout;
    const T* M;
    Dims dm;
    T* W;  // nullptr: no W / G
    T* G;
    LoopState* st;
    int count_update;
    Dims d;

    __device__ bool skip() const {
        if (!st) return false;
        if (st->done) return true;
        if (st->bad_step) {  // diffeo.cpp:52-53: throw before composing
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                st->err = 2;
                st->done = 1;
            }
            return true;
        }
        return false;
    }
    __device__ void stage(int x, int y, int z, T v[3]) const {
        const int i = d.idx32(x, y, z);
        const T s0 = step[i], s1 = step[d.n + i], s2 = step[2 * d.n + i];
        const Cell3<T> c = locate3<T>(d, x, y, z, s0, s1, s2);
        T o[3];
        lerp_field<T, false>(c, u, u + d.n, u + 2 * d.n, 3, o);
        v[0] = s0 + o[0];
        v[1] = s1 + o[1];
        v[2] = s2 + o[2];
    }
    __device__ void xpass(const T* p, int cs, T v[3]) const { gauss_xpass<T, R>(w, p, cs, v); }
    __device__ T wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ T nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const { return {}; }
    __device__ Red2 emit(int x, int y, int z, const T s[3], const Prol&) const {
        const int i = d.idx32(x, y, z);
        uout[i] = s[0];
        uout[d.n + i] = s[1];
        uout[2 * d.n + i] = s[2];
        if (W) {
            WG3<T> w;
            wg3_fetch<T>(M, dm, x, y, z, s[0], s[1], s[2], w);
            W[i] = wg3_value(w);
            T gr[3];
            wg3_grad(w, gr);
            G[i] = gr[0];
            G[d.n + i] = gr[1];
            G[2 * d.n + i] = gr[2];
        }
        return {0.0, 0.0};
    }
    __device__ void finish(int, double, double, const Prol&) const {
        if (st && count_update) st->nupdates += 1;
    }
};

// split update, second half: sigma_warp smoothing of the composed field c
// (SmoothAdamB<..., CAPH> wrote it) and the fused W/G epilogue
template <class T, int R_>
struct ComposeSB {
    using Acc = T;
    using Raw = T;
    using Prol = NoProl;
    static constexpr int R = R_, C = 3, NR = 3, kStageBatch = 8;
    static constexpr bool kSum = false, kMax = false;
    const T* c;  // 3 planes
    GaussW<T> w;
    T* uout;
    const T* M;
    Dims dm;
    T* W;
    T* G;
    LoopState* st;
    int count_update;
    Dims d;

    __device__ bool skip() const {
        if (!st) return false;
        if (st->done) return true;
        if (st->bad_step) {  // diffeo.cpp:52-53: throw before composing
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                st->err = 2;
                st->done = 1;
            }
            return true;
        }
        return false;
    }
    __device__ void stage(int x, int y, int z, T v[3]) const {
        const int i = d.idx32(x, y, z);
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] = c[k * d.n + i];
    }
    using Src = T;
    __device__ const T* vsrc(int k) const { return c + static_cast<size_t>(k) * d.n; }
    __device__ static constexpr bool vnc(int) { return false; }
    __device__ void xpass(const T* p, int cs, T v[3]) const { gauss_xpass<T, R>(w, p, cs, v); }
    __device__ T wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ T nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const { return {}; }
    __device__ Red2 emit(int x, int y, int z, const T s[3], const Prol&) const {
        const int i = d.idx32(x, y, z);
        uout[i] = s[0];
        uout[d.n + i] = s[1];
        uout[2 * d.n + i] = s[2];
        if (W) {
            WG3<T> wg;
            wg3_fetch<T>(M, dm, x, y, z, s[0], s[1], s[2], wg);
            W[i] = wg3_value(wg);
            T gr[3];
            wg3_grad(wg, gr);
            G[i] = gr[0];
            G[d.n + i] = gr[1];
            G[2 * d.n + i] = gr[2];
        }
        return {0.0, 0.0};
    }
    __device__ void finish(int, double, double, const Prol&) const {
        if (st && count_update) st->nupdates += 1;
    }
};

// ---------------------------------------------------------------------------
// Persistent scale solver: one cooperative launch runs every iteration of a
// (small) pyramid level.  Phases are the four brick ops over all bricks
// (grid-stride), separated by grid-wide barriers; the convergence monitor is
// evaluated redundantly by every CTA from the per-brick partials (same values,
// same order -> the same decision everywhere), CTA 0 keeps the device log.
// Replaces 4 kernel launches + 4 kernel boundaries per iteration by 4 grid
// barriers.  pipeline.cpp:157-205 semantics: loss -> converged? -> smooth ->
// Adam -> non-finite step check -> compose.
template <class T, int R, int RG, int RW>
struct PersistArgs {
    LnccFwdB<T, R> fwd;
    LnccBwdB<T, R> bwd;
    // the split update of the graph path: smooth+Adam composes c = step + u(x+step)
    // once per voxel (u alternates between the two fields), then sigma_warp + W/G
    SmoothAdamB<T, RG, 1> sa;
    ComposeSB<T, RW> co;  // c -> uout; uout alternates with sa.uin
    int iters;
    LoopState* st;
    double* loss;
    unsigned long long* stamp;
    int window;
    double tol;
};

constexpr int NTP = NTB;  // persistent solvers: 3 CTAs of 256 threads per SM (one brick each)

template <class T, int R, int RG, int RW>
__global__ void __launch_bounds__(NTP, 3)
    k_persist(const __grid_constant__ PersistArgs<T, R, RG, RW> a, const BG g, int nb) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_red[32];
    LoopState* st = a.st;
    const double nvox = static_cast<double>(g.d.nx) * g.d.ny * g.d.nz;
    int nupd = 0;
    for (int it = 0; it < a.iters; ++it) {
        // loss: fused LNCC forward over every brick
        for (int b = blockIdx.x; b < nb; b += gridDim.x) brick_body<decltype(a.fwd), NTP>(a.fwd, g, b, smem, s_red);
        grid.sync();
        double acc = 0.0;
        for (int k = threadIdx.x; k < nb; k += NTP) acc += __ldcg(a.fwd.partials + k);
        const double v = -bsum<NTP>(acc, s_red) / nvox;
        // the monitor's decision (monitor_commit), taken identically by all CTAs
        const int slot = it;
        bool stop = !isfinite(v);
        if (!stop && slot + 1 >= a.window + 1) {
            const double prev = __ldcg(a.loss + slot - a.window);
            const double den = fabs(prev) > 1e-30 ? fabs(prev) : 1e-30;
            stop = ((prev - v) / static_cast<double>(a.window)) / den < a.tol;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0)
            monitor_commit(st, v, 0.0, 0.0, a.loss, a.stamp, a.window, a.tol);
        if (stop) break;
        for (int b = blockIdx.x; b < nb; b += gridDim.x) brick_body<decltype(a.bwd), NTP>(a.bwd, g, b, smem, s_red);
        grid.sync();  // also publishes CTA 0's st->t / st->slot to the Adam prologue
        SmoothAdamB<T, RG, 1> sa = a.sa;
        ComposeSB<T, RW> co = a.co;
        if (it & 1) {  // ping-pong of the field
            sa.uin = a.co.uout;
            co.uout = const_cast<T*>(a.sa.uin);
        }
        for (int b = blockIdx.x; b < nb; b += gridDim.x) brick_body<decltype(sa), NTP>(sa, g, b, smem, s_red);
        grid.sync();
        if (*reinterpret_cast<volatile int*>(&st->bad_step)) {  // diffeo.cpp:52-53
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                st->err = 2;
                st->done = 1;
            }
            break;
        }
        for (int b = blockIdx.x; b < nb; b += gridDim.x) brick_body<decltype(co), NTP>(co, g, b, smem, s_red);
        ++nupd;
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st->nupdates += nupd;
}

// ---------------------------------------------------------------------------
// Neighbour-synchronised persistent solver.  Same phases and per-voxel
// arithmetic as k_persist, but no grid-wide barrier: a brick's phase p only
// reads (within its halo) what its 26 neighbour bricks wrote in phase p-1 or
// earlier, so before phase p each brick waits for its neighbours' phase
// counters to reach p-1 and publishes its own counter after the phase
// (release / acquire at gpu scope).  CTAs drift against each other and the
// fill/drain of a grid barrier (or of a kernel boundary) disappears.
//
// Hazards: a brick is at most one phase ahead of any neighbour, and no phase
// writes a buffer its predecessor phase reads (F: coef / B: grad / A: m, nu,
// c / C: u', W, G; u ping-pongs), so halo reads always see the intended
// version.  Halo reach: LNCC r, sigma_grad radius, sigma_warp radius and the
// compose gather (cap <= 1.5 -> 2 voxels) all stay within one brick
// (8 x BY x 8, BY >= 4) of the own brick.
//
// Loss and monitor (pipeline.cpp:157-179): the last brick to finish the
// forward of iteration i sums the iteration's partials (fixed order) and
// commits the record; nobody waits for it unless iteration i could stop the
// level (slot >= window), in which case every brick waits for the commit
// before its update.  Adam's step counter and record slot are t0 + i + 1 and
// it0 + i, exactly the values the monitor would have produced.  A non-finite
// loss, a non-finite step or convergence raises `abort`, which every wait
// polls; a wait that outlives kNbTimeoutNs raises err 4 instead of hanging.
struct NbSync {
    unsigned* flags;  // [2 nb] per brick: neighbour completions by phase parity (push)
                      // or the brick's own completed phases (poll)
    unsigned* fdone;  // [iters] bricks past the forward of iteration i
    unsigned* mseq;   // iterations whose record is committed
    unsigned* abort_;
};
constexpr unsigned long long kNbTimeoutNs = 4000000000ull;

// polls are relaxed (no L1 invalidation per poll: the other CTAs of the SM
// keep their cached halo lines); one acq_rel fence after a successful wait
// and one before a publication make the pattern an acquire / a release
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// raise abort (and err 4 on a stall); returns false
__device__ bool nb_fail(const NbSync& s, LoopState* st, bool stalled) {
    if (stalled && atomicCAS(&st->err, 0, 4) == 0) st->done = 1;
    atomicExch(s.abort_, 1u);
    return false;
}

#ifndef DFM_NB_PUSH
#define DFM_NB_PUSH 1
#endif
// DFM_NB_TRACE=i (debug builds): every brick CTA printfs, for iteration i,
// per phase the clock64 cycles spent waiting and in the body, and the
// globaltimer at its publication (NBTR), and brick_body's stage clocks (NBBT)
#if DFM_NB_TRACE >= 0
__device__ long long g_nb_tr_enter[1024][4], g_nb_tr_ready[1024][4], g_nb_tr_done[1024][4];
__device__ unsigned long long g_nb_tr_pub[1024][4];
#endif
// existing neighbour l (0..26, 13 = self excluded) of brick b, or -1
__device__ __forceinline__ int nb_neighbour(const BG& g, int nbz, int b, int l) {
    if (l >= 27 || l == 13) return -1;
    const int bx = b % g.nbx, t = b / g.nbx, by = t % g.nby, bz = t / g.nby;
    const int nx = bx + l % 3 - 1, ny = by + (l / 3) % 3 - 1, nz = bz + l / 9 - 1;
    if (nx < 0 || nx >= g.nbx || ny < 0 || ny >= g.nby || nz < 0 || nz >= nbz) return -1;
    return (nz * g.nby + ny) * g.nbx + nx;
}

// spin until *f >= target (or abort / stall); false when the level was aborted
__device__ bool nb_spin(const NbSync& s, LoopState* st, const unsigned* f, unsigned target) {
    if (ld_relaxed_u32(f) >= target) return true;
    const unsigned long long t0 = dfm_global_ns();
    while (ld_relaxed_u32(f) < target) {
        if (ld_relaxed_u32(s.abort_)) return false;
        if (dfm_global_ns() - t0 > kNbTimeoutNs) return nb_fail(s, st, true);
    }
    return true;
}

// wait until every existing neighbour of brick b has completed phase `target`.
// Push form (DFM_NB_PUSH): neighbours add to b's counter of their completed
// phases of b's parity class; a neighbour is at most one phase ahead of b, so
// counter[target & 1] == nneigh * ((target + 1) / 2) exactly when all of them
// completed `target` (one thread polls one word).  Poll form: warp 0 polls
// the 26 neighbours' own phase counters.
__device__ bool nb_wait(const NbSync& s, LoopState* st, const BG& g, int nbz, int b,
                        unsigned target, int* s_flag) {
#if DFM_NB_TRACE >= 0
    if (threadIdx.x == 0 && target / 4 == DFM_NB_TRACE && blockIdx.x < 1024)
        g_nb_tr_enter[blockIdx.x][target % 4] = clock64();
#endif
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        bool ok = true;
        if (target > 0) {
#if DFM_NB_PUSH
            const unsigned nn = __popc(__ballot_sync(0xffffffffu, nb_neighbour(g, nbz, b, l) >= 0));
            if (l == 0)
                ok = nb_spin(s, st, s.flags + 2 * b + (target & 1u), nn * ((target + 1u) / 2u));
#else
            const int n = nb_neighbour(g, nbz, b, l);
            if (n >= 0) ok = nb_spin(s, st, s.flags + n, target);
#endif
        }
        ok = __all_sync(0xffffffffu, ok);
        if (l == 0) {
            fence_acq_rel_gpu();  // acquire: the neighbours' phase outputs
            *s_flag = ok;
        }
    }
    __syncthreads();
#if DFM_NB_TRACE >= 0
    if (threadIdx.x == 0 && target / 4 == DFM_NB_TRACE && blockIdx.x < 1024)
        g_nb_tr_ready[blockIdx.x][target % 4] = clock64();
#endif
    return *s_flag != 0;
}

// publish: brick b completed phase p (the CTA's threads are synchronised)
__device__ __forceinline__ void nb_publish(const NbSync& s, const BG& g, int nbz, int b,
                                           unsigned p) {
#if DFM_NB_TRACE >= 0
    if (threadIdx.x == 0 && (p - 1) / 4 == DFM_NB_TRACE && blockIdx.x < 1024) {
        g_nb_tr_done[blockIdx.x][(p - 1) % 4] = clock64();
        g_nb_tr_pub[blockIdx.x][(p - 1) % 4] = dfm_global_ns();
    }
#endif
#if DFM_NB_PUSH
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) fence_acq_rel_gpu();  // release: the CTA's phase outputs
        __syncwarp();
        const int n = nb_neighbour(g, nbz, b, threadIdx.x);
        if (n >= 0)
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(s.flags + 2 * n + (p & 1u))
                         : "memory");
    }
#else
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();  // release: the CTA's phase outputs (ordered by the barrier)
        st_relaxed_u32(s.flags + b, p);
    }
#endif
}

template <class T, int R, int CAPH>
struct SmoothAdamNB : SmoothAdamB<T, R, CAPH> {
    using Base = SmoothAdamB<T, R, CAPH>;
    long long t;  // Adam step counter of this iteration (st->t after the commit)
    int slot;     // record slot of this iteration
    __device__ typename Base::Prol prologue() const {
        typename Base::Prol p;
        p.ic1 = static_cast<T>(1.0 / this->corr1[t]);
        p.ic2 = static_cast<T>(1.0 / this->corr2[t]);
        p.slot = slot;
        return p;
    }
};

template <class T, int R, int RG, int RW, int CAPH>
struct PersistNbArgs {
    LnccFwdB<T, R, true> fwd;  // partials: [iters][nb]
    LnccBwdB<T, R> bwd;
    SmoothAdamNB<T, RG, CAPH> sa;
    ComposeSB<T, RW> co;
    NbSync sync;
    int iters;
    LoopState* st;
    double* loss;
    unsigned long long* stamp;
    int window;
    double tol;
};

#ifndef DFM_NB_MINB
#define DFM_NB_MINB 3
#endif
template <class T, int R, int RG, int RW, int CAPH>
__global__ void __launch_bounds__(NTP, DFM_NB_MINB)
    k_persist_nb(const __grid_constant__ PersistNbArgs<T, R, RG, RW, CAPH> a, const BG g,
                 int nb) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_red[32];
    __shared__ int s_flag, s_done0, s_stop, s_bad;
    __shared__ long long s_t0;
    __shared__ int s_it0;
    LoopState* st = a.st;
    const NbSync& sy = a.sync;
    if (threadIdx.x == 0) {  // read before this CTA's first publication (see header)
        s_t0 = st->t;
        s_it0 = st->it;
        s_done0 = st->done;
    }
    __syncthreads();
    if (s_done0) return;  // an earlier level failed
    const long long t0 = s_t0;
    const int it0 = s_it0;
    const int nbz = (g.d.nz + BZ - 1) / BZ;
    const int nbc = gridDim.x - 1;  // brick CTAs; the last CTA is the monitor
    if (blockIdx.x == nbc) {
        // monitor (pipeline.cpp:157-179): per iteration, once every brick's
        // forward partial is in, the fixed-order sum and the record commit
        const double nvox = static_cast<double>(g.d.nx) * g.d.ny * g.d.nz;
        for (int it = 0; it < a.iters; ++it) {
            if (threadIdx.x == 0) {
                s_flag = nb_spin(sy, st, sy.fdone + it, static_cast<unsigned>(nb));
                fence_acq_rel_gpu();
            }
            __syncthreads();
            if (!s_flag) return;
            const double* part = a.fwd.partials + static_cast<size_t>(it) * nb;
            double acc = 0.0;
            for (int k = threadIdx.x; k < nb; k += NTP) acc += __ldcg(part + k);
            const double v = -bsum<NTP>(acc, s_red) / nvox;
            if (threadIdx.x == 0) {
                monitor_commit(st, v, 0.0, 0.0, a.loss, a.stamp, a.window, a.tol);
                s_stop = st->done;
                if (st->err) atomicExch(sy.abort_, 1u);  // non-finite loss
                fence_acq_rel_gpu();
                st_relaxed_u32(sy.mseq, static_cast<unsigned>(it + 1));
            }
            __syncthreads();
            if (s_stop) return;  // converged (every brick stops before this update)
        }
        return;
    }
    int nupd = 0;
    for (int it = 0; it < a.iters; ++it) {
        const unsigned p0 = 4u * static_cast<unsigned>(it);
        // F: loss forward; the partials go to the monitor CTA
        {
            auto fwd = a.fwd;
            fwd.partials = a.fwd.partials + static_cast<size_t>(it) * nb;
            for (int b = blockIdx.x; b < nb; b += nbc) {
                auto pre = [&] { return nb_wait(sy, st, g, nbz, b, p0, &s_flag); };
                if (!brick_body<decltype(fwd), NTP>(fwd, g, b, smem, s_red, pre,
                                                    it == DFM_NB_TRACE ? 0 : -1))
                    return;
                nb_publish(sy, g, nbz, b, p0 + 1);
                if (threadIdx.x == 0)  // the partial is released by nb_publish's fence
                    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(sy.fdone + it)
                                 : "memory");
            }
        }
        // B: LNCC backward
        for (int b = blockIdx.x; b < nb; b += nbc) {
            auto pre = [&] { return nb_wait(sy, st, g, nbz, b, p0 + 1, &s_flag); };
            if (!brick_body<decltype(a.bwd), NTP>(a.bwd, g, b, smem, s_red, pre,
                                                  it == DFM_NB_TRACE ? 1 : -1))
                return;
            nb_publish(sy, g, nbz, b, p0 + 2);
        }
        // the level may stop at this iteration: wait for its record (every
        // brick gets here: B(it) needs only F(it), which the commit follows)
        if (it0 + it >= a.window) {
            if (threadIdx.x == 0) {
                const bool ok = nb_spin(sy, st, sy.mseq, static_cast<unsigned>(it + 1));
                fence_acq_rel_gpu();
                s_stop = !ok || *reinterpret_cast<volatile int*>(&st->done);
            }
            __syncthreads();
            if (s_stop) break;
        }
        // A: smooth + Adam + pointwise compose into c
        SmoothAdamNB<T, RG, CAPH> sa = a.sa;
        ComposeSB<T, RW> co = a.co;
        if (it & 1) {  // ping-pong of the field
            sa.uin = a.co.uout;
            co.uout = const_cast<T*>(a.sa.uin);
        }
        sa.t = t0 + it + 1;
        sa.slot = it0 + it;
        for (int b = blockIdx.x; b < nb; b += nbc) {
            auto pre = [&] { return nb_wait(sy, st, g, nbz, b, p0 + 2, &s_flag); };
            if (!brick_body<decltype(sa), NTP>(sa, g, b, smem, s_red, pre,
                                               it == DFM_NB_TRACE ? 2 : -1))
                return;
            nb_publish(sy, g, nbz, b, p0 + 3);
        }
        // C: sigma_warp smoothing of c, W/G; a non-finite step stops first
        for (int b = blockIdx.x; b < nb; b += nbc) {
            if (!nb_wait(sy, st, g, nbz, b, p0 + 3, &s_flag)) return;
            if (threadIdx.x == 0) s_bad = *reinterpret_cast<volatile int*>(&st->bad_step);
            __syncthreads();
            if (s_bad) {  // diffeo.cpp:52-53
                if (threadIdx.x == 0) {
                    st->err = 2;
                    st->done = 1;
                    atomicExch(sy.abort_, 1u);
                }
                return;
            }
            brick_body<decltype(co), NTP>(co, g, b, smem, s_red, NoPreStage{},
                                          it == DFM_NB_TRACE ? 3 : -1);
            nb_publish(sy, g, nbz, b, p0 + 4);
        }
        ++nupd;
#if DFM_NB_TRACE >= 0
        if (it == DFM_NB_TRACE && threadIdx.x == 0 && blockIdx.x < 1024) {
            const int c = blockIdx.x;
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            printf("NBTR %d %d %lld %lld %lld %lld %lld %lld %lld %lld %llu %llu %llu %llu\n", c,
                   (int)smid,
                   g_nb_tr_ready[c][0] - g_nb_tr_enter[c][0], g_nb_tr_done[c][0] - g_nb_tr_ready[c][0],
                   g_nb_tr_ready[c][1] - g_nb_tr_enter[c][1], g_nb_tr_done[c][1] - g_nb_tr_ready[c][1],
                   g_nb_tr_ready[c][2] - g_nb_tr_enter[c][2], g_nb_tr_done[c][2] - g_nb_tr_ready[c][2],
                   g_nb_tr_ready[c][3] - g_nb_tr_enter[c][3], g_nb_tr_done[c][3] - g_nb_tr_ready[c][3],
                   g_nb_tr_pub[c][0], g_nb_tr_pub[c][1], g_nb_tr_pub[c][2], g_nb_tr_pub[c][3]);
            for (int k = 0; k < 4; ++k)
                printf("NBBT %d %d %lld %lld %lld %lld %lld\n", c, k,
                       g_nb_bt[c][k][1] - g_nb_bt[c][k][0], g_nb_bt[c][k][2] - g_nb_bt[c][k][1],
                       g_nb_bt[c][k][3] - g_nb_bt[c][k][2], g_nb_bt[c][k][4] - g_nb_bt[c][k][3],
                       g_nb_bt[c][k][5] - g_nb_bt[c][k][4]);
        }
#endif
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&st->nupdates, nupd);
}

template <class T, int R, int RG, int RW, int CAPH>
int run_persist_nb(const Launch& L, const PersistNbArgs<T, R, RG, RW, CAPH>& a, const Dims& d,
                   bool any_size) {
    using A = PersistNbArgs<T, R, RG, RW, CAPH>;
    constexpr size_t b1 = BrickLayout<decltype(A::fwd)>::bytes;
    constexpr size_t b2 = BrickLayout<decltype(A::bwd)>::bytes;
    constexpr size_t b3 = BrickLayout<decltype(A::sa)>::bytes;
    constexpr size_t b4 = BrickLayout<decltype(A::co)>::bytes;
    constexpr size_t m12 = b1 > b2 ? b1 : b2, m34 = b3 > b4 ? b3 : b4;
    constexpr size_t bytes = m12 > m34 ? m12 : m34;
    if constexpr (bytes > kBrickSmemMax) {
        return -2;
    } else {
        const void* fn = reinterpret_cast<const void*>(k_persist_nb<T, R, RG, RW, CAPH>);
        const int per_sm = kernel_setup(fn, NTP, bytes);
        if (per_sm < 1) return -3;
        BG g;
        g.d = d;
        g.nbx = (d.nx + BX - 1) / BX;
        g.nby = (d.ny + BY - 1) / BY;
        int nb = g.nbx * g.nby * ((d.nz + BZ - 1) / BZ);
        const int cap = per_sm * (L.num_sms > 0 ? L.num_sms : 148);
        if (cap < 2) return -3;
        // several bricks per CTA serialise their phase latencies (48x48x52:
        // 64 us per iteration vs 35 on the graph path): by default only levels
        // whose bricks each get a CTA run here
        if (nb > cap - 1 && !any_size) return -2;
        // and few bricks: a kernel boundary inside the graph (0.6-0.9 us) is
        // cheaper than a neighbour wait + release (16^3: 21.2 vs 26.0, 32^3:
        // 24.4 vs 27.6 us per iteration; 40x48x56, 420 bricks: 36.3 vs 34.2)
        const int sms = L.num_sms > 0 ? L.num_sms : 148;
        if (nb < 2 * sms && !any_size) return -2;
        const int grid = (nb < cap - 1 ? nb : cap - 1) + 1;  // + the monitor CTA
        void* args[] = {const_cast<A*>(&a), &g, &nb};
        // co-residency of every CTA is what makes the spin waits safe
        const cudaError_t e =
            cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(NTP), args, bytes, L.stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return -4;
        }
        L.bump();
        return grid;
    }
}

template <class T, int R, int RG, int RW>
int run_persist(const Launch& L, const PersistArgs<T, R, RG, RW>& a, const Dims& d) {
    using A = PersistArgs<T, R, RG, RW>;
    constexpr size_t b1 = BrickLayout<decltype(A::fwd)>::bytes;
    constexpr size_t b2 = BrickLayout<decltype(A::bwd)>::bytes;
    constexpr size_t b3 = BrickLayout<decltype(A::sa)>::bytes;
    constexpr size_t b4 = BrickLayout<decltype(A::co)>::bytes;
    constexpr size_t m12 = b1 > b2 ? b1 : b2, m34 = b3 > b4 ? b3 : b4;
    constexpr size_t bytes = m12 > m34 ? m12 : m34;
    if constexpr (bytes > kBrickSmemMax) {
        return -2;
    } else {
        const int per_sm =
            kernel_setup(reinterpret_cast<const void*>(k_persist<T, R, RG, RW>), NTP, bytes);
        if (per_sm < 1) return -3;
        BG g;
        g.d = d;
        g.nbx = (d.nx + BX - 1) / BX;
        g.nby = (d.ny + BY - 1) / BY;
        int nb = g.nbx * g.nby * ((d.nz + BZ - 1) / BZ);
        const int cap = per_sm * (L.num_sms > 0 ? L.num_sms : 148);
        const int grid = nb < cap ? nb : cap;
        void* args[] = {const_cast<A*>(&a), &g, &nb};
        const cudaError_t e = cudaLaunchCooperativeKernel(
            reinterpret_cast<const void*>(k_persist<T, R, RG, RW>), dim3(grid), dim3(NTP), args,
            bytes, L.stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return -4;
        }
        L.bump();
        return grid;
    }
}

template <class Op>
int run_brick(const Launch& L, const Op& op, const Dims& d) {
    using Lay = BrickLayout<Op>;
    if constexpr (Lay::bytes > kBrickSmemMax) {
        return -2;  // e.g. fp64 with a large Gaussian radius: caller falls back
    } else {
    kernel_setup(reinterpret_cast<const void*>(k_brick<Op>), NTB, Lay::bytes);
    BG g;
    g.d = d;
    g.nbx = (d.nx + BX - 1) / BX;
    g.nby = (d.ny + BY - 1) / BY;
    const int nb = g.nbx * g.nby * ((d.nz + BZ - 1) / BZ);
    launch_maybe_pdl(L, k_brick<Op>, dim3(nb), dim3(NTB), Lay::bytes, op, g);
    L.bump();
    return nb;
    }
}

template <int RLO, int RHI, class F>
int with_rb(int R, F&& f) {
    switch (R) {
#define DFM_RB(r)                                                                   \
    case r:                                                                         \
        if constexpr (r >= RLO && r <= RHI) return f(std::integral_constant<int, r>{}); \
        break;
        DFM_RB(0) DFM_RB(1) DFM_RB(2) DFM_RB(3) DFM_RB(4) DFM_RB(5) DFM_RB(6)
#undef DFM_RB
    }
    return -2;
}

}  // namespace

bool brick_supported(Dims d, int esz, int lncc_r, int rg, int rw) {
    // fp64 smoothing at radius 6 would need > 227 KB of shared memory
    const int rg_max = esz == 8 ? kBrickGaussRMax - 1 : kBrickGaussRMax;
    return d.ndim == 3 && d.nz > 1 && d.zoff == 0 && d.gnz == 0 && d.zb == 0 && d.ze == 0 &&
           lncc_r >= 1 && lncc_r <= kBrickLnccRMax && rg >= 0 && rg <= rg_max &&
           rw >= 0 && rw <= kBrickComposeRMax && d.n < (int64_t(1) << 31);
}

template <class T>
int launch_lncc_fwd_brick(const Launch& L, int R, const T* F, const T* W, Dims d, T* coef,
                          double* partials, const LoopState* st, const MonitorArgs* mon,
                          const double* fstat) {
    return with_rb<1, kBrickLnccRMax>(R, [&](auto rc) {
        auto go = [&](auto op) {
            op.F = F;
            op.W = W;
            op.fstat = fstat;
            op.coef = coef;
            op.partials = partials;
            op.st = st;
            op.mon = mon ? *mon : MonitorArgs{nullptr, nullptr, nullptr, 0, 0.0};
            op.d = d;
            return run_brick(L, op, d);
        };
        if (fstat) return go(LnccFwdB<T, decltype(rc)::value, true>{});
        return go(LnccFwdB<T, decltype(rc)::value, false>{});
    });
}

template <class T>
int launch_fstats_brick(const Launch& L, int R, const T* F, Dims d, double* fstat) {
    return with_rb<1, kBrickLnccRMax>(R, [&](auto rc) {
        FStatsB<T, decltype(rc)::value> op;
        op.F = F;
        op.fstat = fstat;
        op.d = d;
        return run_brick(L, op, d);
    });
}

template <class T>
int launch_lncc_bwd_brick(const Launch& L, int R, const T* coef, const T* F, const T* W,
                          const T* G, Dims d, T* grad, const LoopState* st) {
    return with_rb<1, kBrickLnccRMax>(R, [&](auto rc) {
        using Op = LnccBwdB<T, decltype(rc)::value>;
        Op op;
        op.coef = coef;
        op.F = F;
        op.W = W;
        op.G = G;
        op.grad = grad;
        op.m2n = -2.0 / static_cast<double>(d.n);
        op.st = st;
        op.d = d;
        return run_brick(L, op, d);
    });
}

template <class T>
int launch_smooth_adam_brick(const Launch& L, int R, const GaussW<T>& w, const T* grad, T* m,
                             T* nu, T* step, Dims d, AdamParams ap, LoopState* st,
                             unsigned long long* maxstep) {
    return with_rb<0, kBrickGaussRMax>(R, [&](auto rc) {
        using Op = SmoothAdamB<T, decltype(rc)::value>;
        Op op;
        op.grad = grad;
        op.w = w;
        op.m = m;
        op.nu = nu;
        op.step = step;
        op.ak = adam_k<T>(ap);
        op.corr1 = ap.corr1;
        op.corr2 = ap.corr2;
        op.st = st;
        op.maxstep = maxstep;
        op.d = d;
        return run_brick(L, op, d);
    });
}

template <class T>
int launch_compose_brick(const Launch& L, int R, const GaussW<T>& w, const T* step,
                         const T* uin, T* uout, const T* M, Dims dm, Dims d, T* W, T* G,
                         LoopState* st, bool count_update) {
    return with_rb<0, kBrickComposeRMax>(R, [&](auto rc) {
        using Op = ComposeB<T, decltype(rc)::value>;
        Op op;
        op.step = step;
        op.u = uin;
        op.w = w;
        op.uout = uout;
        op.M = M;
        op.dm = dm;
        op.W = W;
        op.G = G;
        op.st = st;
        op.count_update = count_update ? 1 : 0;
        op.d = d;
        return run_brick(L, op, d);
    });
}

// instantiated radius triples of the persistent solver (LNCC r, sigma_grad
// radius, sigma_warp radius): BASELINE's kernel 5 / 7 with sigma 1.0 / 0.5
template <class T>
int launch_persist_scale(const Launch& L, const PersistScale<T>& p) {
    auto go = [&](auto rr) -> int {
        constexpr int R = decltype(rr)::value;
        PersistArgs<T, R, 3, 2> a;
        a.fwd.F = p.F;
        a.fwd.W = p.W;
        a.fwd.fstat = nullptr;
        a.fwd.coef = p.coef;
        a.fwd.partials = p.partials;
        a.fwd.st = p.st;
        a.fwd.mon = MonitorArgs{nullptr, nullptr, nullptr, 0, 0.0};
        a.fwd.d = p.d;
        a.bwd.coef = p.coef;
        a.bwd.F = p.F;
        a.bwd.W = p.W;
        a.bwd.G = p.G;
        a.bwd.grad = p.grad;
        a.bwd.m2n = -2.0 / static_cast<double>(p.d.n);
        a.bwd.st = p.st;
        a.bwd.d = p.d;
        a.sa.grad = p.grad;
        a.sa.w = p.wg;
        a.sa.m = p.m;
        a.sa.nu = p.nu;
        a.sa.step = p.step;  // receives c
        a.sa.uin = p.u0;
        a.sa.ak = adam_k<T>(p.ap);
        a.sa.corr1 = p.ap.corr1;
        a.sa.corr2 = p.ap.corr2;
        a.sa.st = p.st;
        a.sa.maxstep = p.maxstep;
        a.sa.d = p.d;
        a.co.c = p.step;
        a.co.w = p.ww;
        a.co.uout = p.u1;
        a.co.M = p.M;
        a.co.dm = p.d;
        a.co.W = p.W;
        a.co.G = p.G;
        a.co.st = p.st;
        a.co.count_update = 0;
        a.co.d = p.d;
        a.iters = p.iters;
        a.st = p.st;
        a.loss = p.loss;
        a.stamp = p.stamp;
        a.window = p.window;
        a.tol = p.tol;
        return run_persist(L, a, p.d);
    };
    if (p.rg != 3 || p.rw != 2 || p.ap.cap > 0.5) return -2;
    switch (p.lncc_r) {
        case 1: return go(std::integral_constant<int, 1>{});
        case 2: return go(std::integral_constant<int, 2>{});
        case 3: return go(std::integral_constant<int, 3>{});
    }
    return -2;
}

// words of the neighbour-synchronised solver's sync workspace for a level:
// per-brick phase counters, per-iteration forward arrivals, commit sequence, abort
int persist_nb_sync_words(Dims d, int iters) {
    const int nb = ((d.nx + BX - 1) / BX) * ((d.ny + BY - 1) / BY) * ((d.nz + BZ - 1) / BZ);
    return 2 * nb + iters + 2;
}

// the neighbour-synchronised solver: LNCC r 1..3 with the level's F
// statistics, sigma_grad radius 3 (sigma 1.0), sigma_warp radius 2 (0.5),
// step cap <= 1.5 (compose gather within 2 voxels)
template <class T>
int launch_persist_nb_scale(const Launch& L, const PersistScale<T>& p) {
    if (!p.fstat || !p.sync || p.rg != 3 || p.rw != 2 || !(p.ap.cap <= 1.5)) return -2;
    const int nbx = (p.d.nx + BX - 1) / BX, nby = (p.d.ny + BY - 1) / BY;
    const int nb = nbx * nby * ((p.d.nz + BZ - 1) / BZ);
    auto go = [&](auto rr, auto cc) -> int {
        constexpr int R = decltype(rr)::value, CAPH = decltype(cc)::value;
        PersistNbArgs<T, R, 3, 2, CAPH> a;
        a.fwd.F = p.F;
        a.fwd.W = p.W;
        a.fwd.fstat = p.fstat;
        a.fwd.coef = p.coef;
        a.fwd.partials = p.partials;
        a.fwd.st = p.st;
        a.fwd.mon = MonitorArgs{nullptr, nullptr, nullptr, 0, 0.0};
        a.fwd.d = p.d;
        a.bwd.coef = p.coef;
        a.bwd.F = p.F;
        a.bwd.W = p.W;
        a.bwd.G = p.G;
        a.bwd.grad = p.grad;
        a.bwd.m2n = -2.0 / static_cast<double>(p.d.n);
        a.bwd.st = p.st;
        a.bwd.d = p.d;
        a.sa.grad = p.grad;
        a.sa.w = p.wg;
        a.sa.m = p.m;
        a.sa.nu = p.nu;
        a.sa.step = p.step;  // receives c
        a.sa.uin = p.u0;
        a.sa.ak = adam_k<T>(p.ap);
        a.sa.corr1 = p.ap.corr1;
        a.sa.corr2 = p.ap.corr2;
        a.sa.st = p.st;
        a.sa.maxstep = p.maxstep;
        a.sa.d = p.d;
        a.sa.t = 0;
        a.sa.slot = 0;
        a.co.c = p.step;
        a.co.w = p.ww;
        a.co.uout = p.u1;
        a.co.M = p.M;
        a.co.dm = p.d;
        a.co.W = p.W;
        a.co.G = p.G;
        a.co.st = p.st;
        a.co.count_update = 0;
        a.co.d = p.d;
        a.sync.flags = p.sync;
        a.sync.fdone = p.sync + 2 * nb;
        a.sync.mseq = p.sync + 2 * nb + p.iters;
        a.sync.abort_ = p.sync + 2 * nb + p.iters + 1;
        a.iters = p.iters;
        a.st = p.st;
        a.loss = p.loss;
        a.stamp = p.stamp;
        a.window = p.window;
        a.tol = p.tol;
        return run_persist_nb(L, a, p.d, p.nb_any_size);
    };
    auto by_cap = [&](auto rr) -> int {
        if (p.ap.cap <= 0.5) return go(rr, std::integral_constant<int, 1>{});
        return go(rr, std::integral_constant<int, 2>{});
    };
    switch (p.lncc_r) {
        case 1: return by_cap(std::integral_constant<int, 1>{});
        case 2: return by_cap(std::integral_constant<int, 2>{});
        case 3: return by_cap(std::integral_constant<int, 3>{});
    }
    return -2;
}

template <class T>
int launch_smooth_adam_compose_brick(const Launch& L, int R, const GaussW<T>& w, const T* grad,
                                     T* m, T* nu, const T* uin, T* cout, double cap, Dims d,
                                     AdamParams ap, LoopState* st, unsigned long long* maxstep) {
    return with_rb<0, kBrickGaussRMax>(R, [&](auto rc) {
        auto go = [&](auto op) {
            op.grad = grad;
            op.w = w;
            op.m = m;
            op.nu = nu;
            op.step = cout;
            op.uin = uin;
            op.ak = adam_k<T>(ap);
            op.corr1 = ap.corr1;
            op.corr2 = ap.corr2;
            op.st = st;
            op.maxstep = maxstep;
            op.d = d;
            return run_brick(L, op, d);
        };
        constexpr int RR = decltype(rc)::value;
        if (cap <= 0.5) return go(SmoothAdamB<T, RR, 1>{});
        if (cap <= 1.5) return go(SmoothAdamB<T, RR, 2>{});
        return go(SmoothAdamB<T, RR, 1 << 20>{});  // any cap: the clamped general form
    });
}

template <class T>
int launch_compose_smooth_brick(const Launch& L, int R, const GaussW<T>& w, const T* c, T* uout,
                                const T* M, Dims dm, Dims d, T* W, T* G, LoopState* st,
                                bool count_update) {
    return with_rb<0, kBrickComposeRMax>(R, [&](auto rc) {
        ComposeSB<T, decltype(rc)::value> op;
        op.c = c;
        op.w = w;
        op.uout = uout;
        op.M = M;
        op.dm = dm;
        op.W = W;
        op.G = G;
        op.st = st;
        op.count_update = count_update ? 1 : 0;
        op.d = d;
        return run_brick(L, op, d);
    });
}

#define DFM_INST_BRICK(T)                                                                      \
    template int launch_lncc_fwd_brick<T>(const Launch&, int, const T*, const T*, Dims, T*,    \
                                          double*, const LoopState*, const MonitorArgs*,       \
                                          const double*);                                      \
    template int launch_fstats_brick<T>(const Launch&, int, const T*, Dims, double*);         \
    template int launch_lncc_bwd_brick<T>(const Launch&, int, const T*, const T*, const T*,    \
                                          const T*, Dims, T*, const LoopState*);               \
    template int launch_smooth_adam_brick<T>(const Launch&, int, const GaussW<T>&, const T*,   \
                                             T*, T*, T*, Dims, AdamParams, LoopState*,         \
                                             unsigned long long*);                             \
    template int launch_compose_brick<T>(const Launch&, int, const GaussW<T>&, const T*,       \
                                         const T*, T*, const T*, Dims, Dims, T*, T*,           \
                                         LoopState*, bool);                                    \
    template int launch_persist_scale<T>(const Launch&, const PersistScale<T>&);              \
    template int launch_persist_nb_scale<T>(const Launch&, const PersistScale<T>&);           \
    template int launch_smooth_adam_compose_brick<T>(const Launch&, int, const GaussW<T>&,      \
                                                     const T*, T*, T*, const T*, T*, double,   \
                                                     Dims, AdamParams, LoopState*,             \
                                                     unsigned long long*);                     \
    template int launch_compose_smooth_brick<T>(const Launch&, int, const GaussW<T>&,           \
                                                const T*, T*, const T*, Dims, Dims, T*, T*,    \
                                                LoopState*, bool);

DFM_INST_BRICK(float)
DFM_INST_BRICK(double)

}  // namespace dfm
