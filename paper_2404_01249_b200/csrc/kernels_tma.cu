// kernels_tma.cu — plane-streaming stencil kernels of the hot loop (v2).
//
// Same 2.5-D z-march as kernels_stencil.cu (haloed xy tile per plane, x/y
// filters in shared memory, z filter in a register ring), but every input
// plane tile is fetched by TMA (cp.async.bulk.tensor, zero fill outside the
// volume) into an S-stage shared-memory ring guarded by mbarriers, one
// elected thread running S-1 planes ahead of the compute.  Memory latency is
// therefore off the critical path and the compute reads only shared memory.
//
// Data flow of one LNCC iteration with these kernels:
//   compose (previous iteration / warpgrad at scale start) -> u, W=M(x+u), G=grad M(x+u)
//   lncc_fwd   F, W (halo r)          -> 4 window coefficients + cc^2 partials
//   lncc_bwd   coefficients (halo r)  -> grad = dW * G            (center F, W, G)
//   smooth_adam grad (halo 3 sigma_g) -> m, nu, capped step       (center m, nu)
//   compose    step (halo 3 sigma_w), u (halo 3 sigma_w + cap)  -> u', W', G'
// The compose gathers u(x+step) from the shared-memory u tiles: with
// |step| <= cap <= 1.5 the 8 interpolation corners lie within 2 voxels.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>


#include "dfm_device.cuh"
#include "dfm_kernels.cuh"
#include "loop_ops.cuh"
#include "tma_util.cuh"

// This file is compiled twice: as itself (32-wide tiles, namespace dfm::tx32,
// plus the public dispatching launchers at the end) and through
// kernels_tma16.cu (16-wide tiles, dfm::tx16): a level whose last 32-wide x
// tile would be at most half full runs the narrow instantiation.
#ifndef DFM_TMA_TX  // x width of a z-march tile
#define DFM_TMA_TX kTX
#endif
#ifndef DFM_TMA_NS
#define DFM_TMA_NS tx32
#endif

namespace dfm {
namespace DFM_TMA_NS {

namespace {

constexpr int TX = DFM_TMA_TX;
// narrow tiles: the launch-bound minimum CTAs per SM of the 32-wide form (a
// 16-wide CTA has half the threads, so twice the register budget per CTA
// count): measured 91.2 vs 93.8 us per 80x96x112 iteration against scaling
// the minimum by 32/TX (same per-thread budget as the wide form)
#ifndef DFM_TMA_NARROW_MINB_SCALE
#define DFM_TMA_NARROW_MINB_SCALE 1
#endif
constexpr int kMinBScale = TX < 32 ? DFM_TMA_NARROW_MINB_SCALE : 1;

// TMA ring depths (planes in flight per CTA); overridable for tuning builds
#ifndef DFM_S_FWD
#define DFM_S_FWD 4
#endif
#ifndef DFM_S_BWD
#define DFM_S_BWD 4
#endif
#ifndef DFM_S_SA
#define DFM_S_SA 4
#endif
#ifndef DFM_S_CO_EXTRA
#define DFM_S_CO_EXTRA 0
#endif
// CTA tile heights (rows of 32 columns) per op; overridable for tuning builds
// minimum resident CTAs per SM requested from ptxas (register budget)
#ifndef DFM_MINB_FWD
#define DFM_MINB_FWD 3
#endif
#ifndef DFM_SINK
#define DFM_SINK 1
#endif
#ifndef DFM_CS_ASYNC
#define DFM_CS_ASYNC 1
#endif
#ifndef DFM_FWD3_WIDE_R
#define DFM_FWD3_WIDE_R 3
#endif
#ifndef DFM_SA_CASYNC
#define DFM_SA_CASYNC 0
#endif
#ifndef DFM_SA_CTMA
#define DFM_SA_CTMA 0
#endif
#ifndef DFM_FWD_QUAD
#define DFM_FWD_QUAD 1
#endif
#ifndef DFM_SA_QUAD1
#define DFM_SA_QUAD1 1
#endif
#ifndef DFM_SA_QUAD2
#define DFM_SA_QUAD2 0
#endif
#ifndef DFM_MINB_SA2
#define DFM_MINB_SA2 3
#endif
#ifndef DFM_SAC_ASYNC
#define DFM_SAC_ASYNC 0
#endif
#ifndef DFM_TY_SAC
#define DFM_TY_SAC 8
#endif
#ifndef DFM_MINB_SAC
#define DFM_MINB_SAC 2
#endif
#ifndef DFM_TY_CS
#define DFM_TY_CS 8
#endif
#ifndef DFM_CY_CS
#define DFM_CY_CS 1
#endif
#ifndef DFM_MINB_CS
#define DFM_MINB_CS 3
#endif
#ifndef DFM_CY_BWD64
#define DFM_CY_BWD64 2
#endif
// sliding box sums in the fp64 LNCC moment / coefficient passes: bit 0 the
// x (quad) and y (row pairs) sums, bit 1 a running z sum (more registers)
#ifndef DFM_SLIDE
#define DFM_SLIDE 1
#endif
// rows per thread of the fp32 LNCC forward (radius <= 2)
#ifndef DFM_CY_FWD3
#define DFM_CY_FWD3 1
#endif
#ifndef DFM_BWD_QUAD64
#define DFM_BWD_QUAD64 1
#endif
#ifndef DFM_BWD_QUAD64_RMAX
#define DFM_BWD_QUAD64_RMAX 3
#endif
#ifndef DFM_MINB_FWD3
#define DFM_MINB_FWD3 3
#endif
#ifndef DFM_MINB_BWD
#define DFM_MINB_BWD 4
#endif
#ifndef DFM_MINB_SA
#define DFM_MINB_SA 2
#endif
#ifndef DFM_MINB_CO
#define DFM_MINB_CO 3
#endif
// rows per thread (coarsening) per op
#ifndef DFM_CY_FWD
#define DFM_CY_FWD 1
#endif
#ifndef DFM_CY_BWD
#define DFM_CY_BWD 2
#endif
#ifndef DFM_CY_SA
#define DFM_CY_SA 1
#endif
#ifndef DFM_CY_CO
#define DFM_CY_CO 1
#endif
#ifndef DFM_TY_FWD
#define DFM_TY_FWD 8
#endif
#ifndef DFM_TY_BWD
#define DFM_TY_BWD 8
#endif
#ifndef DFM_TY_SA
#define DFM_TY_SA 16
#endif
#ifndef DFM_TY_CO
#define DFM_TY_CO 8
#endif

template <class T>
constexpr int round_bx(int w) {
    return (w + (16 / int(sizeof(T))) - 1) / (16 / int(sizeof(T))) * (16 / int(sizeof(T)));
}
constexpr int align128(int b) { return (b + 127) / 128 * 128; }

// xor of the 32-bit words of a padding-free value (a use of every word)
template <class V>
__device__ __forceinline__ unsigned fold_bits(const V& v) {
    static_assert(sizeof(V) % 4 == 0, "fold_bits: 4-byte granular values only");
    unsigned w[sizeof(V) / 4];
    memcpy(w, &v, sizeof(V));
    unsigned h = 0;
#pragma unroll
    for (int k = 0; k < int(sizeof(V) / 4); ++k) h ^= w[k];
    return h;
}

// dynamic shared memory of a z-march launch: [align pad][S stage ring]
// [staged input tile][2 x-filtered buffers][op extra (Op::kExtraBytes)]
template <class Op, class = void>
struct ExtraBytes {
    static constexpr int value = 0;
};
template <class Op>
struct ExtraBytes<Op, std::void_t<decltype(Op::kExtraBytes)>> {
    static constexpr int value = Op::kExtraBytes;
};
template <class Op>
__host__ __device__ constexpr int zm2_core_bytes() {
    using Acc = typename Op::Acc;
    constexpr int HI = Op::TYv + 2 * Op::R, WI = TX + 2 * Op::R;
    if constexpr (Op::kStaged && Op::R == 0)  // pointwise: no filter buffers
        return Op::S * Op::kStageBytes;
    return Op::S * Op::kStageBytes +
           (Op::kStaged ? int(sizeof(Acc)) * Op::C * HI * WI : 0) +
           2 * int(sizeof(Acc)) * Op::C * HI * TX;
}
__device__ __forceinline__ unsigned char* zm2_smem_base() {
    // TMA destinations need 128 B alignment; the dynamic window starts right
    // after the static shared variables, so align it here (+128 B reserved)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    return smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
}
// the op's own region (e.g. cp.async gather slots), 16 B aligned
template <class Op>
__device__ __forceinline__ unsigned char* zm2_extra() {
    return zm2_smem_base() + ((zm2_core_bytes<Op>() + 15) & ~15);
}

// x filter four columns per thread (Op::kXQuad, fp32 ops): 128-bit shared
// loads of the row window, one 128-bit store of the four results
template <class Op, class = void>
struct XQuad {
    static constexpr bool value = false;
};
template <class Op>
struct XQuad<Op, std::void_t<decltype(Op::kXQuad)>> {
    static constexpr bool value = Op::kXQuad;
};

// four consecutive box sums of 2R+1 values (e[0 .. 2R+4)): the first direct,
// the next three sliding (+ entering - leaving) when DFM_SLIDE
template <int R, class A>
__device__ __forceinline__ void box4(const A* e, A out[4]) {
    A a = A(0);
#pragma unroll
    for (int j = 0; j < 2 * R + 1; ++j) a += e[j];
    out[0] = a;
#pragma unroll
    for (int o = 1; o < 4; ++o) {
        if constexpr ((DFM_SLIDE & 1) != 0) {
            a = (a + e[o + 2 * R]) - e[o - 1];
        } else {
            a = A(0);
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) a += e[o + j];
        }
        out[o] = a;
    }
}

// the float4 chunks [col, col + 4 * NCH) of a stage row, col % 4 == 0
template <int NCH>
__device__ __forceinline__ void load_row4(const float* p, float w[4 * NCH]) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
        const float4 t = reinterpret_cast<const float4*>(p)[k];
        w[4 * k] = t.x;
        w[4 * k + 1] = t.y;
        w[4 * k + 2] = t.z;
        w[4 * k + 3] = t.w;
    }
}

// box-filter ops (unit taps, unit norms: the LNCC moments and coefficient
// sums) may compute their window sums by sliding: y rows of a thread from the
// previous row's sum (+ entering - leaving), z from a running sum of the ring
// (Op::kSlide).  fp64 accumulation keeps the rounding drift ~1e-16 relative.
template <class Op, class = void>
struct BoxSlide {
    static constexpr bool value = false;
};
template <class Op>
struct BoxSlide<Op, std::void_t<decltype(Op::kSlide)>> {
    static constexpr bool value = Op::kSlide;
};

// the op's centre operands of plane zo = q - R arrive by TMA with stage q
// (Op::kCenterTMA; read with Op::load_center_st): no per-voxel global loads
template <class Op, class = void>
struct CenterTMA {
    static constexpr bool value = false;
};
template <class Op>
struct CenterTMA<Op, std::void_t<decltype(Op::kCenterTMA)>> {
    static constexpr bool value = Op::kCenterTMA;
};

// the op's centre operands of plane zo + 1 are requested with cp.async during
// plane zo's epilogue (Op::kCenterAsync: center_async / load_center_async):
// a whole plane of latency hiding, no register scoreboard across the loop
template <class Op, class = void>
struct CenterAsync {
    static constexpr bool value = false;
};
template <class Op>
struct CenterAsync<Op, std::void_t<decltype(Op::kCenterAsync)>> {
    static constexpr bool value = Op::kCenterAsync;
};

// optional per-row carry initialisation (Op::init_carry(carry, row))
template <class Op, class C>
__device__ __forceinline__ auto carry_init(const Op& op, C& c, int r, int)
    -> decltype(op.init_carry(c, r), void()) {
    op.init_carry(c, r);
}
template <class Op, class C>
__device__ __forceinline__ void carry_init(const Op&, C&, int, long) {}

struct ZG2 {
    Dims d;
    int zchunk;
    int tiles_x;
};

// ---------------------------------------------------------------------------
// the streaming z-march driver.  A CTA is TX x (TYv / CY) threads; each thread
// owns CY output columns of its x (rows ty, ty + TYv/CY, ...): per-plane
// overheads (barrier, mbarrier wait, loop control, address math) are shared by
// CY voxels.  Per-thread constants (norm factors, the op's prologue such as
// Adam bias corrections) are computed once; Op::Carry lets an op defer work of
// plane zo into plane zo+1 (latency hiding).
template <class Op>
__global__ void __launch_bounds__(TX * Op::TYv / Op::kCY, Op::kMinB * kMinBScale)
    k_zm2(const __grid_constant__ Op op, const ZG2 g) {
    using Acc = typename Op::Acc;
    constexpr int TYv = Op::TYv, CY = Op::kCY, TYt = TYv / CY, NTh = TX * TYt;
    static_assert(TYt * CY == TYv, "tile rows must be a multiple of the coarsening");
    constexpr int R = Op::R, C = Op::C, S = Op::S, K = 2 * R + 1;
    constexpr int HI = TYv + 2 * R, WI = TX + 2 * R;
    constexpr int SB = Op::kStageBytes;
    unsigned char* const smem = zm2_smem_base();
    unsigned char* stages = smem;
    Acc* s_in = reinterpret_cast<Acc*>(smem + S * SB);
    Acc* s_x = s_in + (Op::kStaged ? C * HI * WI : 0);  // two buffers of C*HI*TX
    __shared__ __align__(8) uint64_t bars[S];
    __shared__ double s_red[32];

    pdl_wait();  // predecessor's outputs (and LoopState) are visible from here
    if (op.skip()) return;
    const Dims& d = g.d;
    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    const int x0 = (blockIdx.x % g.tiles_x) * TX;
    const int y0 = (blockIdx.x / g.tiles_x) * TYv;
    const int z0 = d.out_begin() + blockIdx.y * g.zchunk;
    const int z1 = min(z0 + g.zchunk, d.out_end());
    const int x = x0 + tx;
    const int q0 = z0 - R - Op::BACK;
    const int qend = z1 + R + Op::AHEAD;

    if (tid == 0) {
        op.prefetch_maps();
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int q = q0; q < qend && q < q0 + S; ++q)
            op.issue(stages + ((q - q0) % S) * SB, &bars[(q - q0) % S], x0, y0, q);

    const Acc nxv = x < d.nx ? op.nrm(0, x) : Acc(0);
    constexpr bool kQuad = XQuad<Op>::value;
    constexpr int NQ = TX / 4;  // quads per tile row
    static_assert(!kQuad || NTh % NQ == 0, "quad x pass: whole rows per thread group");
    const int xq = 4 * (tid % NQ);  // this thread's quad of tile columns
    Acc nx4[4];
#pragma unroll
    for (int o = 0; o < 4; ++o)
        nx4[o] = (kQuad && x0 + xq + o < d.nx) ? op.nrm(0, x0 + xq + o) : Acc(0);
    int yk[CY];
    bool own[CY];
    Acc nyv[CY];
#pragma unroll
    for (int k = 0; k < CY; ++k) {
        yk[k] = y0 + ty * CY + k;  // consecutive rows: their y windows share K-1 loads
        own[k] = x < d.nx && yk[k] < d.ny;
        nyv[k] = own[k] ? op.nrm(1, yk[k]) : Acc(0);
    }
    const typename Op::Prol pr = op.prologue();
    {
        // consume every pre-loop global load here.  ptxas shares its few
        // scoreboards between these loads and the plane loop's own loads
        // (the carried gathers, the centre loads); a first wait inside the
        // loop would then also wait for the in-flight gathers of the previous
        // plane on every plane, which is what the Carry exists to avoid
        __shared__ volatile unsigned s_sink;
        unsigned h = fold_bits(nxv);
        if constexpr (kQuad) h ^= fold_bits(nx4);
#pragma unroll
        for (int k = 0; k < CY; ++k) h ^= fold_bits(nyv[k]);
        if constexpr (!std::is_empty<typename Op::Prol>::value) h ^= pr.bits();
        if (DFM_SINK && h == 0x9e3779b9u) s_sink = h;  // any consumer will do; almost never runs
    }
    typename Op::Carry carry[CY] = {};
#pragma unroll
    for (int r = 0; r < CY; ++r) carry_init(op, carry[r], r, 0);
    if constexpr (CenterAsync<Op>::value) {  // the first emitted plane's centre operands
        if (z0 < z1) {
#pragma unroll
            for (int r = 0; r < CY; ++r)
                if (own[r]) op.center_async(x, yk[r], z0, r, 0);
        }
        cp_async_commit();
    }

    // register ring of the last K xy-filtered planes per owned row; it shifts
    // by register moves (C*(K-1) MOVs per plane and row) rather than unrolling
    // the plane loop by K: the unrolled body overflowed the instruction cache
    Acc ring[CY][C][K];
#pragma unroll
    for (int r = 0; r < CY; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
            for (int k = 0; k < K; ++k) ring[r][c][k] = Acc(0);
    constexpr bool kSlide = BoxSlide<Op>::value;
    constexpr bool kSlideZ = kSlide && (DFM_SLIDE & 2);  // running z sum (+registers)
    Acc zsum[kSlideZ ? CY : 1][kSlideZ ? C : 1];
#pragma unroll
    for (int r = 0; r < (kSlideZ ? CY : 1); ++r)
#pragma unroll
        for (int c = 0; c < (kSlideZ ? C : 1); ++c) zsum[r][c] = Acc(0);
    double rsum = 0.0, rmax = 0.0;
    int waited = q0 - 1;
    int buf = 0;
    const int zend = z1 + R;

    for (int zi = z0 - R; zi < zend; ++zi) {
        if constexpr (Op::kStaged && R == 0) {
            // pointwise staged op (e.g. the radius-0 compose of the split
            // update): the staged value is the output, no filter passes
            if constexpr (Op::AHEAD == 0) {  // exactly plane zi (ring position >= 0)
                const unsigned k = static_cast<unsigned>(zi - q0);
                mbar_wait(&bars[k % S], (k / S) & 1u);
            } else {
                while (waited < zi + Op::AHEAD) {
                    ++waited;
                    const unsigned k = static_cast<unsigned>(waited - q0);
                    mbar_wait(&bars[k % S], (k / S) & 1u);
                }
            }
            const typename Op::PlaneCtx pc = op.plane_ctx(stages, q0, zi);
            typename Op::Center cen{};
#pragma unroll
            for (int r = 0; r < CY; ++r) {
                if (!own[r]) continue;
                Acc v[C];
                op.stage_point(pc, x0, y0, zi, ty * CY + r, tx, v);
                const Red2 rr = op.emit(x, yk[r], zi, v, cen, pr, carry[r]);
                rsum += rr.sum;
                rmax = fmax(rmax, rr.mx);
            }
            __syncthreads();  // plane zi - BACK's slot is free for the next plane
            if (tid == 0) {
                const int qf = zi - Op::BACK + S;
                if (qf < qend) {
                    const unsigned k = static_cast<unsigned>(qf - q0);
                    op.issue(stages + (k % S) * SB, &bars[k % S], x0, y0, qf);
                }
            }
            continue;
        }
        constexpr int kk = K - 1;
        const int zo = zi - R;
        constexpr bool kCT = CenterTMA<Op>::value;
        constexpr bool kCA = CenterAsync<Op>::value;
        typename Op::Center cen[CY];
        if constexpr (!kCT && !kCA) {
#pragma unroll
            for (int r = 0; r < CY; ++r)
                if (zo >= z0 && own[r]) op.load_center(x, yk[r], zo, cen[r]);
        }
        if constexpr (Op::AHEAD == 0) {  // exactly plane zi (ring position >= 0)
            const unsigned k = static_cast<unsigned>(zi - q0);
            mbar_wait(&bars[k % S], (k / S) & 1u);
        } else {
            while (waited < zi + Op::AHEAD) {
                ++waited;
                const unsigned k = static_cast<unsigned>(waited - q0);
                mbar_wait(&bars[k % S], (k / S) & 1u);
            }
        }
        Acc* sx = s_x + buf * (C * HI * TX);
        if constexpr (Op::kStaged) {
            const typename Op::PlaneCtx pc = op.plane_ctx(stages, q0, zi);
            if (op.interior(x0, y0, zi)) {  // CTA-uniform: no clamping, no bounds
                for (int e = tid; e < HI * WI; e += NTh) {
                    const int row = e / WI, col = e - row * WI;
                    Acc v[C];
                    op.stage_fast(pc, x0, y0, zi, row, col, v);
#pragma unroll
                    for (int c = 0; c < C; ++c) s_in[(c * HI + row) * WI + col] = v[c];
                }
            } else {
                for (int e = tid; e < HI * WI; e += NTh) {
                    const int row = e / WI, col = e - row * WI;
                    Acc v[C];
                    op.stage(pc, x0, y0, zi, row, col, v);
#pragma unroll
                    for (int c = 0; c < C; ++c) s_in[(c * HI + row) * WI + col] = v[c];
                }
            }
            __syncthreads();
#pragma unroll
            for (int row = ty; row < HI; row += TYt) {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const Acc* src = s_in + (c * HI + row) * WI + tx;
                    Acc a = Acc(0);
#pragma unroll
                    for (int j = 0; j < K; ++j) a += op.wgt(0, j) * src[j];
                    sx[(c * HI + row) * TX + tx] = a * nxv;
                }
            }
        } else if constexpr (kQuad) {
            const unsigned char* st = stages + (static_cast<unsigned>(zi - q0) % S) * SB;
#pragma unroll
            for (int row = tid / NQ; row < HI; row += NTh / NQ) {
                Acc v[C][4];
                op.xpass4(st, row, xq, nx4, v);
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    Acc* o = sx + (c * HI + row) * TX + xq;
                    if constexpr (sizeof(Acc) == 4) {
                        *reinterpret_cast<float4*>(o) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
                    } else {
                        reinterpret_cast<double2*>(o)[0] = make_double2(v[c][0], v[c][1]);
                        reinterpret_cast<double2*>(o)[1] = make_double2(v[c][2], v[c][3]);
                    }
                }
            }
        } else {
            const unsigned char* st = stages + (static_cast<unsigned>(zi - q0) % S) * SB;
#pragma unroll
            for (int row = ty; row < HI; row += TYt) {
                Acc v[C];
                op.xpass(st, row, tx, nxv, v);
#pragma unroll
                for (int c = 0; c < C; ++c) sx[(c * HI + row) * TX + tx] = v[c];
            }
        }
        __syncthreads();
        if (tid == 0) {
            // the slot of plane zi - BACK is free once every thread passed the
            // x pass; with centre operands in the stage it is still read by
            // this plane's emit, so the previous plane's slot is refilled
            const int qf = kCT ? zi - 1 + S : zi - Op::BACK + S;
            if (qf < qend && (!kCT || zi > q0)) {
                const unsigned k = static_cast<unsigned>(qf - q0);
                op.issue(stages + (k % S) * SB, &bars[k % S], x0, y0, qf);
            }
        }
        // y pass of every owned row into ring slot kk (the newest plane) before
        // any emit: the rows' windows overlap and their loads are shared
        if constexpr (kSlide) {
            Acc yprev[C];
#pragma unroll
            for (int r = 0; r < CY; ++r) {
                const int row = ty * CY + r;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const Acc* src = sx + (c * HI + row) * TX + tx;
                    Acc a;
                    if (r == 0) {
                        a = Acc(0);
#pragma unroll
                        for (int j = 0; j < K; ++j) a += src[j * TX];
                    } else {  // the previous row's window, shifted by one row
                        a = (yprev[c] + src[(K - 1) * TX]) - src[-TX];
                    }
                    yprev[c] = a;
                    const Acc leaving = ring[r][c][0];
#pragma unroll
                    for (int k = 0; k < K - 1; ++k) ring[r][c][k] = ring[r][c][k + 1];
                    ring[r][c][kk] = a;
                    if constexpr (kSlideZ) zsum[r][c] = (zsum[r][c] + a) - leaving;
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < CY; ++r) {
                const int row = ty * CY + r;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const Acc* src = sx + (c * HI + row) * TX + tx;
                    Acc a = Acc(0);
#pragma unroll
                    for (int j = 0; j < K; ++j) a += op.wgt(1, j) * src[j * TX];
#pragma unroll
                    for (int k = 0; k < K - 1; ++k) ring[r][c][k] = ring[r][c][k + 1];
                    ring[r][c][kk] = a * nyv[r];
                }
            }
        }
        if constexpr (kCA) {
            if (zo >= z0) {  // request plane zo + 1, then wait for plane zo
                if (zo + 1 < z1) {
#pragma unroll
                    for (int r = 0; r < CY; ++r)
                        if (own[r]) op.center_async(x, yk[r], zo + 1, r, (zo + 1 - z0) & 1);
                }
                cp_async_commit();
                cp_async_wait_group<1>();
#pragma unroll
                for (int r = 0; r < CY; ++r)
                    if (own[r]) op.load_center_async(r, (zo - z0) & 1, cen[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < CY; ++r) {
            if (zo >= z0 && own[r]) {
                if constexpr (kCT)
                    op.load_center_st(stages + (static_cast<unsigned>(zi - q0) % S) * SB,
                                      ty * CY + r, tx, cen[r]);
                // oldest plane (zo - R) sits in slot 0 (slot (kk + 1) % K)
                const Acc nz = op.nrm(2, zo + d.zoff);
                Acc sv[C];
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    if constexpr (kSlideZ) {
                        sv[c] = zsum[r][c];
                    } else {
                        Acc a = Acc(0);
#pragma unroll
                        for (int j = 0; j < K; ++j)
                            a += op.wgt(2, j) * ring[r][c][(kk + 1 + j) % K];
                        sv[c] = a * nz;
                    }
                }
                const Red2 rr = op.emit(x, yk[r], zo, sv, cen[r], pr, carry[r]);
                rsum += rr.sum;
                rmax = fmax(rmax, rr.mx);
            }
        }
        buf ^= 1;
    }
    pdl_trigger();  // the successor may launch into our tail (PDL mode)
#pragma unroll
    for (int r = 0; r < CY; ++r) op.flush(carry[r]);
    if constexpr (Op::kSum || Op::kMax) {
        const int blk = blockIdx.y * gridDim.x + blockIdx.x;
        const double bs = Op::kSum ? bsum<NTh>(rsum, s_red) : 0.0;
        const double bm = Op::kMax ? bmax<NTh>(rmax, s_red) : 0.0;
        if (tid == 0) op.finish(blk, bs, bm, pr);
        if constexpr (Op::kSum) {
            if (op.mon.st)  // fused convergence monitor: the last CTA reduces
                monitor_tail<NTh>(op.mon, op.partials, gridDim.x * gridDim.y,
                                  static_cast<double>(d.nx) * d.ny * d.gz(), s_red);
        }
    } else {
        if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) op.finish(0, 0.0, 0.0, pr);
    }
}

// ---------------------------------------------------------------------------
// ops

struct NoCenter {};
struct NoProl {};
struct NoCarry {};

// similarity.cpp:122-168 — box moments of F and W = M(x+u), window coefficients
template <class T, int R_, int TY_ = DFM_TY_FWD>
struct LnccFwd2 {
    using Acc = double;
    using Center = NoCenter;
    using Prol = NoProl;
    using Carry = NoCarry;
    static constexpr int R = R_, C = 5, BACK = 0, AHEAD = 0, S = DFM_S_FWD, TYv = TY_;
    static constexpr int kMinB = DFM_MINB_FWD, kCY = DFM_CY_FWD;
    static constexpr bool kStaged = false, kSum = true, kMax = false;
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);  // TMA smem destinations 128 B aligned
    static constexpr int kStageBytes = 2 * kBox;
    CUtensorMap mF, mW;
    T* coef;  // 4 planes, coef[k*n + i]; nullptr -> value only
    double* partials;
    const LoopState* st;
    MonitorArgs mon;  // mon.st == nullptr: no fused monitor
    Dims d;

    __device__ bool skip() const { return st && st->done; }
    __device__ void prefetch_maps() const {
        prefetch_tmap(&mF);
        prefetch_tmap(&mW);
    }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 2 * kBytes);
        tma_load_4d(dst, &mF, bar, x0 - XA, y0 - R, q, 0);
        tma_load_4d(dst + kBox, &mW, bar, x0 - XA, y0 - R, q, 0);
    }
    __device__ Acc wgt(int, int) const { return 1.0; }
    __device__ Acc nrm(int, int) const { return 1.0; }
    __device__ Prol prologue() const { return {}; }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc, Acc v[5]) const {
        const T* F = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
        const T* W = F + kBox / int(sizeof(T));
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
            const double f = static_cast<double>(F[j]), w = static_cast<double>(W[j]);
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
    __device__ void load_center(int, int, int, Center&) const {}
    __device__ Red2 emit(int x, int y, int z, const double s[5], const Center&, const Prol&,
                         Carry&) const {
        // similarity.cpp:145-162 (loop_ops.cuh)
        const double inv_n = window_inv<R>(x, y, z, d);
        const LnccCoef k = lncc_coef(s, inv_n);
        if (coef) {
            const int64_t i = d.idx32(x, y, z);
            coef[i] = static_cast<T>(k.an);
            coef[d.n + i] = static_cast<T>(k.amu);
            coef[2 * d.n + i] = static_cast<T>(k.bn);
            coef[3 * d.n + i] = static_cast<T>(k.bmu);
        }
        return {k.cc2, 0.0};
    }
    __device__ void flush(Carry&) const {}
    __device__ void finish(int blk, double s, double, const Prol&) const { partials[blk] = s; }
};

// similarity.cpp:122-150, fixed-image half: per-voxel window mean and variance
// of F, once per pyramid level (F does not change between iterations)
template <class T, int R_, int TY_ = DFM_TY_FWD>
struct FStats2 {
    using Acc = double;
    using Center = NoCenter;
    using Prol = NoProl;
    using Carry = NoCarry;
    static constexpr int R = R_, C = 2, BACK = 0, AHEAD = 0, S = DFM_S_FWD, TYv = TY_;
    static constexpr int kMinB = DFM_MINB_FWD, kCY = 1;
    static constexpr bool kStaged = false, kSum = false, kMax = false;
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    static constexpr int kStageBytes = kBox;
    CUtensorMap mF;
    double* fstat;  // 2 planes: muF, vF
    Dims d;

    __device__ bool skip() const { return false; }
    __device__ void prefetch_maps() const { prefetch_tmap(&mF); }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, kBytes);
        tma_load_4d(dst, &mF, bar, x0 - XA, y0 - R, q, 0);
    }
    __device__ Acc wgt(int, int) const { return 1.0; }
    __device__ Acc nrm(int, int) const { return 1.0; }
    __device__ Prol prologue() const { return {}; }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc, Acc v[2]) const {
        const T* F = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
        double a0 = 0, a1 = 0;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
            const double f = static_cast<double>(F[j]);
            a0 += f;
            a1 += f * f;
        }
        v[0] = a0;
        v[1] = a1;
    }
    __device__ void load_center(int, int, int, Center&) const {}
    __device__ Red2 emit(int x, int y, int z, const double s[2], const Center&, const Prol&,
                         Carry&) const {
        const double inv_n = window_inv<R>(x, y, z, d);
        double muF, vF;
        lncc_fstats(s[0], s[1], inv_n, muF, vF);
        const int i = d.idx32(x, y, z);
        fstat[i] = muF;
        fstat[d.n + i] = vF;
        return {0.0, 0.0};
    }
    __device__ void flush(Carry&) const {}
    __device__ void finish(int, double, double, const Prol&) const {}
};

// similarity.cpp:122-168 with the F statistics precomputed (FStats2): three
// fp64 box moments of W per iteration instead of five
#ifndef DFM_FWD_WCARRY
#define DFM_FWD_WCARRY 1
#endif
// The clipped window's 1/n of a voxel column (x, y fixed per thread row): the
// x*y window length and the interior-plane quotient 1/(nxy K) are formed on
// the first plane and carried, so the per-voxel work is one uniform z test;
// only the 2R border planes divide.  Same n, same correctly rounded 1/n as
// window_inv (border tiles no longer divide on every voxel).
struct WinCarry {
    int nxy;     // 0: not yet formed
    double inv;  // 1 / (nxy K)
};
template <int R>
__device__ __forceinline__ double window_inv_carried(int x, int y, int z, const Dims& d,
                                                     WinCarry& c) {
    constexpr int K = 2 * R + 1;
    const int gz = d.gz(), zg = z + d.zoff;
    if (gz <= 1) return window_inv<R>(x, y, z, d);
    if (c.nxy == 0) {
        c.nxy = box_len(x, d.nx, R) * box_len(y, d.ny, R);
        c.inv = 1.0 / static_cast<double>(c.nxy * K);
    }
    if (static_cast<unsigned>(zg - R) < static_cast<unsigned>(max(gz - 2 * R, 0))) return c.inv;
    return 1.0 / static_cast<double>(c.nxy * box_len(zg, gz, R));
}

template <class T, int R_, int TY_ = DFM_TY_FWD>
struct LnccFwd3 {
    using Acc = double;
    using Prol = NoProl;
    using Carry = typename std::conditional<DFM_FWD_WCARRY != 0, WinCarry, NoCarry>::type;
    static constexpr int R = R_, C = 3, BACK = 0, AHEAD = 0, S = DFM_S_FWD, TYv = TY_;
    // radius >= 3 (LNCC window 7+) or fp64 needs more than the 80 registers of
    // 3 CTAs per SM: 2 CTAs, no spills
    static constexpr int kMinB = (R_ >= DFM_FWD3_WIDE_R || sizeof(T) == 8) ? 2 : DFM_MINB_FWD3,
                         kCY = (sizeof(T) == 4 && R_ <= 2) ? DFM_CY_FWD3 : 1;
    static constexpr bool kStaged = false, kSum = true, kMax = false;
    static constexpr bool kSlide = DFM_SLIDE != 0;  // box moments: sliding y/z sums
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    static constexpr int kStageBytes = 2 * kBox;
    CUtensorMap mF, mW;
    const double* fstat;
    T* coef[4];  // per-coefficient plane pointers
    double* partials;
    const LoopState* st;
    MonitorArgs mon;
    Dims d;
    struct Center {
        double muF, vF;
    };

    __device__ bool skip() const { return st && st->done; }
    __device__ void prefetch_maps() const {
        prefetch_tmap(&mF);
        prefetch_tmap(&mW);
    }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 2 * kBytes);
        tma_load_4d(dst, &mF, bar, x0 - XA, y0 - R, q, 0);
        tma_load_4d(dst + kBox, &mW, bar, x0 - XA, y0 - R, q, 0);
    }
    __device__ Acc wgt(int, int) const { return 1.0; }
    __device__ Acc nrm(int, int) const { return 1.0; }
    __device__ Prol prologue() const { return {}; }
    // four columns per thread: each element is widened and its W^2, FW
    // products formed once for the 4 windows that contain it
    static constexpr bool kXQuad = sizeof(T) == 4 && DFM_FWD_QUAD;
    __device__ void xpass4(const unsigned char* st_, int row, int col, const Acc*,
                           Acc v[3][4]) const {
        constexpr int NCH = (XA + R + 4 + 3) / 4, LO = XA - R, NE = 4 + 2 * R;
        float wf[4 * NCH], ff[4 * NCH];
        const float* base = reinterpret_cast<const float*>(st_) + row * BX + col;
        load_row4<NCH>(base + kBox / 4, wf);
        load_row4<NCH>(base, ff);
        double e[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) e[k] = static_cast<double>(wf[LO + k]);
        box4<R>(e, v[0]);
        double p[NE];
#pragma unroll
        for (int k = 0; k < NE; ++k) p[k] = __dmul_rn(e[k], e[k]);
        box4<R>(p, v[1]);
#pragma unroll
        for (int k = 0; k < NE; ++k) p[k] = __dmul_rn(static_cast<double>(ff[LO + k]), e[k]);
        box4<R>(p, v[2]);
    }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc, Acc v[3]) const {
        const T* F = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
        const T* W = F + kBox / int(sizeof(T));
        double a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
            const double w = static_cast<double>(W[j]);
            a0 += w;
            a1 += w * w;
            a2 += static_cast<double>(F[j]) * w;
        }
        v[0] = a0;
        v[1] = a1;
        v[2] = a2;
    }
    __device__ void load_center(int x, int y, int z, Center& c) const {
        const int i = d.idx32(x, y, z);
        c.muF = __ldg(fstat + i);
        c.vF = __ldg(fstat + d.n + i);
    }
    __device__ Red2 emit(int x, int y, int z, const double s[3], const Center& c, const Prol&,
                         Carry& cr) const {
        double inv_n;
        if constexpr (DFM_FWD_WCARRY != 0)
            inv_n = window_inv_carried<R>(x, y, z, d, cr);
        else
            inv_n = window_inv<R>(x, y, z, d);
        const LnccCoef k = lncc_coef_f(c.muF, c.vF, s[0], s[1], s[2], inv_n);
        const int i = d.idx32(x, y, z);
        coef[0][i] = static_cast<T>(k.an);
        coef[1][i] = static_cast<T>(k.amu);
        coef[2][i] = static_cast<T>(k.bn);
        coef[3][i] = static_cast<T>(k.bmu);
        return {k.cc2, 0.0};
    }
    __device__ void flush(Carry&) const {}
    __device__ void finish(int blk, double s, double, const Prol&) const { partials[blk] = s; }
};

// similarity.cpp:170-189 — box sums of the coefficients, dW, grad = dW * G
template <class T, int R_, int TY_ = DFM_TY_BWD>
struct LnccBwd2 {
    // box sums of the (fp32-stored) coefficients in fp64 (DFM_BWD_ACC32 = 0,
    // loop_ops.cuh): fp32 sums miss the per-kernel criterion at 160x192x224
    using Acc = typename std::conditional<(DFM_BWD_ACC32 != 0) && sizeof(T) == 4, float,
                                          double>::type;
    using Prol = NoProl;
    using Carry = NoCarry;
    static constexpr int R = R_, C = 4, BACK = 0, AHEAD = 0, S = DFM_S_BWD, TYv = TY_;
    // fp32 sums: two consecutive rows per thread (-20 us/iteration at 160x192x224)
    // fp64 sums at radius >= 3 need the 128-register budget of 2 CTAs per SM
    static constexpr int kMinB = (sizeof(Acc) == 8 && R_ >= 3) ? 2 : DFM_MINB_BWD,
                         kCY = sizeof(Acc) == 4 ? DFM_CY_BWD
                                              : (sizeof(T) == 4 && R_ <= 2 ? DFM_CY_BWD64 : 1);
    static constexpr bool kStaged = false, kSum = false, kMax = false;
    static constexpr bool kSlide = DFM_SLIDE != 0 && sizeof(Acc) == 8;  // fp64 sliding sums
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    static constexpr int kStageBytes = 4 * kBox;
    CUtensorMap mC;
    const T* F;
    const T* W;
    const T* G[3];  // per-component plane pointers (3-D only)
    T* grad[3];
    double m2n;  // -2 / N (similarity.cpp:182)
    const LoopState* st;
    Dims d;
    struct Center {
        T f, w, g0, g1, g2;
    };

    __device__ bool skip() const { return st && st->done; }
    __device__ void prefetch_maps() const { prefetch_tmap(&mC); }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 4 * kBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k) tma_load_4d(dst + k * kBox, &mC, bar, x0 - XA, y0 - R, q, k);
    }
    __device__ Acc wgt(int, int) const { return 1.0; }
    __device__ Acc nrm(int, int) const { return 1.0; }
    __device__ Prol prologue() const { return {}; }
    static constexpr bool kXQuad = sizeof(T) == 4 && (sizeof(Acc) == 4 || (DFM_BWD_QUAD64 && R_ <= DFM_BWD_QUAD64_RMAX));
    __device__ void xpass4(const unsigned char* st_, int row, int col, const Acc*,
                           Acc v[4][4]) const {
        constexpr int NCH = (XA + R + 4 + 3) / 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float wv[4 * NCH];
            load_row4<NCH>(reinterpret_cast<const float*>(st_) + c * (kBox / 4) + row * BX + col,
                           wv);
            if constexpr (kSlide) {
                double e[4 + 2 * R];
#pragma unroll
                for (int k = 0; k < 4 + 2 * R; ++k) e[k] = static_cast<double>(wv[(XA - R) + k]);
                box4<R>(e, v[c]);
            } else {
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                    Acc a = Acc(0);
#pragma unroll
                    for (int j = 0; j < 2 * R + 1; ++j) a += static_cast<Acc>(wv[o + (XA - R) + j]);
                    v[c][o] = a;
                }
            }
        }
    }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc, Acc v[4]) const {
        const T* p = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            Acc a = Acc(0);
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j)
                a += static_cast<Acc>(p[c * (kBox / int(sizeof(T))) + j]);
            v[c] = a;
        }
    }
    __device__ void load_center(int x, int y, int z, Center& c) const {
        const int i = d.idx32(x, y, z);
        c.f = __ldg(F + i);
        c.w = __ldg(W + i);
        c.g0 = __ldg(G[0] + i);
        c.g1 = __ldg(G[1] + i);
        c.g2 = __ldg(G[2] + i);
    }
    __device__ Red2 emit(int x, int y, int z, const Acc sa[4], const Center& c, const Prol&,
                         Carry&) const {
        const int i = d.idx32(x, y, z);
        const double f = static_cast<double>(c.f), w = static_cast<double>(c.w);
        const double s[4] = {static_cast<double>(sa[0]), static_cast<double>(sa[1]),
                             static_cast<double>(sa[2]), static_cast<double>(sa[3])};
        const double dW = lncc_dw(m2n, f, w, s);
        grad[0][i] = static_cast<T>(dW * static_cast<double>(c.g0));
        grad[1][i] = static_cast<T>(dW * static_cast<double>(c.g1));
        grad[2][i] = static_cast<T>(dW * static_cast<double>(c.g2));
        return {0.0, 0.0};
    }
    __device__ void flush(Carry&) const {}
    __device__ void finish(int, double, double, const Prol&) const {}
};

// pipeline.cpp:182-186 + optim.cpp:22-42 + diffeo.cpp:47-57
// CAPH_ > 0: the emit also composes, writing c = step + u(x + step) (the
// composed field ComposeS2 smooths) into `step` instead of the step itself
// JAC_: eulerian_direction(use_jac = true) (diffeo.cpp:25-39): the smoothed
// gradient is mapped by J(u)^T at the voxel before Adam (central differences of
// the current field, one-sided at the borders)
template <class T, int R_, int TY_ = DFM_TY_SA, int CY_ = DFM_CY_SA, int MINB_ = DFM_MINB_SA,
          int CAPH_ = 0, bool JAC_ = false>
struct SmoothAdam2 {
    using Acc = T;
    // the composing emit's gather: cp.async into shared memory (fp32, one row
    // per thread) or 24 loads carried in registers
    static constexpr bool kAsync = DFM_SAC_ASYNC && CAPH_ > 0 && sizeof(T) == 4 && CY_ == 1;
    using Carry = typename std::conditional<
        (CAPH_ > 0),
        typename std::conditional<kAsync, ComposeCarryA<T>, ComposeCarry<T>>::type,
        NoCarry>::type;
    static constexpr int R = R_, C = 3, BACK = 0, AHEAD = 0, S = DFM_S_SA, TYv = TY_;
    static constexpr int kMinB = MINB_, kCY = CY_;
    static constexpr int NTH = TX * TY_ / CY_;
    // two slots of the 24 gathered corners per thread: [slot][corner][thread]
    static constexpr int kGatherBytes = kAsync ? 2 * 24 * NTH * int(sizeof(T)) : 0;
    // m, nu of the next plane by cp.async (composing variant: its carried
    // gather already needs the registers): [slot][row][6][thread]
    static constexpr bool kCenterAsync = CAPH_ > 0 && DFM_SA_CASYNC != 0;
    static constexpr int kCenterBytes = kCenterAsync ? 2 * CY_ * 6 * NTH * int(sizeof(T)) : 0;
    static constexpr int kExtraBytes = kGatherBytes + kCenterBytes;
    __device__ static T* gather_buf(int slot) {
        return reinterpret_cast<T*>(zm2_extra<SmoothAdam2>()) + (slot * 24) * NTH + threadIdx.x;
    }
    __device__ static T* center_buf(int slot, int r) {
        return reinterpret_cast<T*>(zm2_extra<SmoothAdam2>() + kGatherBytes) +
               ((slot * CY_ + r) * 6) * NTH + threadIdx.x;
    }
    __device__ void center_async(int x, int y, int z, int r, int slot) const {
        const int i = d.idx32(x, y, z);
        T* b = center_buf(slot, r);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            cp_async<int(sizeof(T))>(b + k * NTH, m[k] + i);
            cp_async<int(sizeof(T))>(b + (3 + k) * NTH, nu[k] + i);
        }
    }
    template <class CC>  // CC = Center (declared below)
    __device__ void load_center_async(int r, int slot, CC& c) const {
        const T* b = center_buf(slot, r);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c.m[k] = b[k * NTH];
            c.nu[k] = b[(3 + k) * NTH];
        }
    }
    static constexpr bool kStaged = false, kSum = false, kMax = true;
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    // stage q: 3 gradient boxes of plane q, then m and nu tiles of plane q - R
    static constexpr bool kCenterTMA = DFM_SA_CTMA != 0;
    static constexpr int kCBytes = TX * TYv * int(sizeof(T));
    static constexpr int kCBox = align128(kCBytes);
    static constexpr int kStageBytes = 3 * kBox + (kCenterTMA ? 6 * kCBox : 0);
    CUtensorMap mG;
    CUtensorMap mM, mN;
    GaussW<T> w;
    // per-component plane pointers (3-D only: the TMA family): one 32-bit
    // index per voxel, no 64-bit component offsets
    T* m[3];
    T* nu[3];
    T* step[3];
    const T* uin;  // CAPH_ > 0: the current field (3 planes)
    const T* uin3[3];
    const T* ujac[3];  // JAC_: the current field u (3 planes) for J(u)^T
    AdamK<T> ak;
    const double* corr1;
    const double* corr2;
    LoopState* st;
    unsigned long long* maxstep;
    Dims d;
    struct Center {
        T m[3], nu[3];
    };
    struct Prol {  // per-launch constants, read once per thread
        T ic1, ic2;  // 1 / (1 - beta^t), optim.cpp:27-30
        int slot;
        // a use of every member (not of the padding: branching on its
        // indeterminate bits would let the optimiser drop the kernel body)
        __device__ unsigned bits() const { return fold_bits(ic1) ^ fold_bits(ic2) ^ unsigned(slot); }
    };

    __device__ bool skip() const { return st && st->done; }
    __device__ void prefetch_maps() const {
        prefetch_tmap(&mG);
        if constexpr (kCenterTMA) {
            prefetch_tmap(&mM);
            prefetch_tmap(&mN);
        }
    }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 3 * kBytes + (kCenterTMA ? 6 * kCBytes : 0));
#pragma unroll
        for (int k = 0; k < 3; ++k) tma_load_4d(dst + k * kBox, &mG, bar, x0 - XA, y0 - R, q, k);
        if constexpr (kCenterTMA) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                tma_load_4d(dst + 3 * kBox + k * kCBox, &mM, bar, x0, y0, q - R, k);
                tma_load_4d(dst + 3 * kBox + (3 + k) * kCBox, &mN, bar, x0, y0, q - R, k);
            }
        }
    }
    __device__ void load_center_st(const unsigned char* st, int row, int col, Center& c) const {
        const T* p = reinterpret_cast<const T*>(st + 3 * kBox) + row * TX + col;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c.m[k] = p[k * (kCBox / int(sizeof(T)))];
            c.nu[k] = p[(3 + k) * (kCBox / int(sizeof(T)))];
        }
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const {
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
    static constexpr bool kXQuad = sizeof(T) == 4 && (CY_ == 1 ? DFM_SA_QUAD1 : DFM_SA_QUAD2);
    __device__ void xpass4(const unsigned char* st_, int row, int col, const Acc nx[4],
                           Acc v[3][4]) const {
        constexpr int NCH = (XA + R + 4 + 3) / 4;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float wv[4 * NCH];
            load_row4<NCH>(reinterpret_cast<const float*>(st_) + c * (kBox / 4) + row * BX + col,
                           wv);
#pragma unroll
            for (int o = 0; o < 4; ++o) {  // the arithmetic of xpass, per column
                const float* q = wv + o + (XA - R);
                T a0 = T(0), a1 = T(0);
#pragma unroll
                for (int j = 0; j < 2 * R + 1; j += 2) a0 += w.taps[0][j] * q[j];
#pragma unroll
                for (int j = 1; j < 2 * R + 1; j += 2) a1 += w.taps[0][j] * q[j];
                v[c][o] = (a0 + a1) * nx[o];
            }
        }
    }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc nx, Acc v[3]) const {
        const T* p = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T* q = p + c * (kBox / int(sizeof(T)));
            T a0 = T(0), a1 = T(0);  // two chains: halves the FMA dependency depth
#pragma unroll
            for (int j = 0; j < 2 * R + 1; j += 2) a0 += w.taps[0][j] * q[j];
#pragma unroll
            for (int j = 1; j < 2 * R + 1; j += 2) a1 += w.taps[0][j] * q[j];
            v[c] = (a0 + a1) * nx;
        }
    }
    __device__ void load_center(int x, int y, int z, Center& c) const {
        const int i = d.idx32(x, y, z);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            c.m[k] = m[k][i];
            c.nu[k] = nu[k][i];
        }
    }
    __device__ void finish_c(const Carry& cr) const {
        if constexpr (kAsync) {
            cp_async_wait_all();
            T cv[3];
            compose_finish_async(cr, gather_buf(cr.slot), NTH, cv);
#pragma unroll
            for (int k = 0; k < 3; ++k) step[k][cr.i] = cv[k];
        } else if constexpr (CAPH_ > 0) {
            T cv[3];
            compose_finish(cr, cv);
#pragma unroll
            for (int k = 0; k < 3; ++k) step[k][cr.i] = cv[k];
        }
    }
    __device__ Red2 emit(int x, int y, int z, const T s[3], const Center& c, const Prol& p,
                         Carry& cr) const {
        const int i = d.idx32(x, y, z);
        T mx = T(0);
        bool bad = false;
        T cl[3];
        T g[3] = {s[0], s[1], s[2]};
        if constexpr (JAC_) {  // diffeo.cpp:30-37: acc_a = sum_c J[c][a] g_c, v = -acc
            T J[9];
            jacobian_at3(CPlanes3<T>{{ujac[0], ujac[1], ujac[2]}}, d, x, y, z, J);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                T acc = T(0);
#pragma unroll
                for (int k = 0; k < 3; ++k) acc += J[k * 3 + a] * s[k];
                g[a] = acc;
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            T mm = c.m[k], nn = c.nu[k];
            cl[k] = adam_component(ak, g[k], mm, nn, p.ic1, p.ic2, bad);
            m[k][i] = mm;
            nu[k][i] = nn;
            mx = fmax(mx, fabs(cl[k]));
        }
        if constexpr (CAPH_ > 0) {  // diffeo.cpp:60 compose, pointwise (interp.cpp:269-289)
            if (cr.valid) finish_c(cr);  // the previous plane's voxel
            if constexpr (kAsync) {
                cr.slot ^= 1;
                compose_fetch_async<T, CAPH_>(uin3, d, x, y, z + d.zoff, cl, i, cr,
                                              gather_buf(cr.slot), NTH);
            } else {
                compose_fetch<T, CAPH_>(uin, d, x, y, z + d.zoff, cl, i, cr);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) step[k][i] = cl[k];
        }
        if (bad && st) st->bad_step = 1;
        return {0.0, static_cast<double>(mx)};
    }
    __device__ void flush(Carry& cr) const {
        if constexpr (CAPH_ > 0) {
            if (cr.valid) finish_c(cr);
        }
    }
    __device__ void finish(int, double, double mx, const Prol& p) const {
        if (maxstep) atomic_max_nonneg(maxstep + p.slot, mx);
    }
};

// diffeo.cpp:60-62 + interp.cpp:269-289 — u' = step + u(x+step), sigma_warp
// Gaussian, then W = M(x+u') and G = grad M(x+u') for the next loss pass.  The
// M gather of plane zo is issued at its emit and consumed at the emit of plane
// zo+1 (Carry), so its latency hides behind a whole plane of work.
template <class T, int R_, int CAPH, int TY_ = DFM_TY_CO>
struct Compose2 {
    using Acc = T;
    using Center = NoCenter;
    using Prol = NoProl;
    static constexpr int kMinB = DFM_MINB_CO, kCY = R_ == 0 ? 2 : DFM_CY_CO;  // pointwise: 2 rows
    static constexpr int R = R_, C = 3, BACK = CAPH, AHEAD = CAPH,
                         S = 2 * CAPH + 2 + DFM_S_CO_EXTRA, TYv = TY_;
    static constexpr bool kStaged = true, kSum = false, kMax = false;
    static constexpr int HU = R + CAPH;  // u halo: Gaussian radius + gather reach
    static constexpr int XAS = round_bx<T>(R), BXS = round_bx<T>(TX + XAS + R), BYS = TYv + 2 * R;
    static constexpr int XAU = round_bx<T>(HU), BXU = round_bx<T>(TX + XAU + HU), BYU = TYv + 2 * HU;
    static constexpr int kBytesS = BXS * BYS * int(sizeof(T));
    static constexpr int kBytesU = BXU * BYU * int(sizeof(T));
    static constexpr int kBoxS = align128(kBytesS), kBoxU = align128(kBytesU);
    static constexpr int kStageBytes = 3 * kBoxS + 3 * kBoxU;
    static constexpr int PS = kBoxS / int(sizeof(T)), PU = kBoxU / int(sizeof(T));
    CUtensorMap mS, mU;
    GaussW<T> w;
    T* uout[3];  // per-component plane pointers (3-D only: the launcher)
    const T* M;
    Dims dm;
    T* W;     // nullptr: do not produce W/G
    T* G[3];
    LoopState* st;
    int count_update;  // 0 for all but one slab of an emulated decomposition
    Dims d;
    struct Carry {  // the M gather of the previous plane's voxel (3-D fast form)
        bool valid;
        int i;
        WG3<T> w;
    };

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
    __device__ void prefetch_maps() const {
        prefetch_tmap(&mS);
        prefetch_tmap(&mU);
    }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 3 * kBytesS + 3 * kBytesU);
#pragma unroll
        for (int k = 0; k < 3; ++k) tma_load_4d(dst + k * kBoxS, &mS, bar, x0 - XAS, y0 - R, q, k);
#pragma unroll
        for (int k = 0; k < 3; ++k)
            tma_load_4d(dst + 3 * kBoxS + k * kBoxU, &mU, bar, x0 - XAU, y0 - HU, q, k);
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const { return {}; }
    // stage pointers of the planes one composed plane needs (zi-CAPH .. zi+CAPH)
    struct PlaneCtx {
        const T* step;               // step box of plane zi
        const T* u[2 * CAPH + 1];    // u boxes of planes zi-CAPH .. zi+CAPH
    };
    __device__ PlaneCtx plane_ctx(const unsigned char* stages, int q0, int zi) const {
        PlaneCtx pc;
        pc.step = reinterpret_cast<const T*>(stages + (unsigned(zi - q0) % S) * kStageBytes);
#pragma unroll
        for (int k = 0; k < 2 * CAPH + 1; ++k) {
            const int q = zi - CAPH + k;
            pc.u[k] = reinterpret_cast<const T*>(stages + (unsigned(q - q0) % S) * kStageBytes +
                                                 3 * kBoxS);
        }
        return pc;
    }
    // every composed element of this CTA-plane (tile + Gaussian halo) has its
    // interpolation cell strictly inside the volume: no clamping is possible
    __device__ bool interior(int x0, int y0, int zi) const {
        const int zg = zi + d.zoff;
        return d.ndim == 3 && x0 - R - CAPH >= 0 && x0 + TX + R - 1 + CAPH <= d.nx - 1 &&
               y0 - R - CAPH >= 0 && y0 + TYv + R - 1 + CAPH <= d.ny - 1 && zg - CAPH >= 0 &&
               zg + CAPH <= d.gz() - 1;
    }
    __device__ __forceinline__ static void cell_fast(int g, float s, int& i0, float& f) {
        const float fl = floorf(s);
        f = s - fl;
        i0 = g + static_cast<int>(fl);
    }
    __device__ __forceinline__ static void cell_fast(int g, double s, int& i0, double& f) {
        const double p = static_cast<double>(g) + s;  // the reference's formulation
        const double fl = floor(p);
        f = p - fl;
        i0 = static_cast<int>(fl);
    }
    __device__ void stage_fast(const PlaneCtx& pc, int x0, int y0, int zi, int row, int col,
                               T v[3]) const {
        const int so = row * BXS + col + (XAS - R);
        const T s0 = pc.step[so], s1 = pc.step[PS + so], s2 = pc.step[2 * PS + so];
        int ix, iy, iz;
        T fx, fy, fz;
        cell_fast(x0 - R + col, s0, ix, fx);
        cell_fast(y0 - R + row, s1, iy, fy);
        cell_fast(zi + d.zoff, s2, iz, fz);
        iz -= d.zoff;
        const int o = (iy - (y0 - HU)) * BXU + (ix - (x0 - XAU));
        const T wx0 = T(1) - fx, wy0 = T(1) - fy, wz0 = T(1) - fz;
        const T w00 = wx0 * wy0, w10 = fx * wy0, w01 = wx0 * fy, w11 = fx * fy;
        const int dz = iz - zi;
        const T* u0 = pc.u[CAPH];
        const T* u1 = pc.u[CAPH];
#pragma unroll
        for (int k = 0; k < 2 * CAPH; ++k)
            if (dz == k - CAPH) {
                u0 = pc.u[k];
                u1 = pc.u[k + 1];
            }
        const T s[3] = {s0, s1, s2};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const T* a = u0 + k * PU + o;
            const T* b = u1 + k * PU + o;
            const T lo = bilerp4(w00, w10, w01, w11, a[0], a[1], a[BXU], a[BXU + 1]);
            const T hi = bilerp4(w00, w10, w01, w11, b[0], b[1], b[BXU], b[BXU + 1]);
            v[k] = s[k] + zlerp(wz0, lo, fz, hi);
        }
    }
    // the pointwise (radius-0) form for any voxel of the tile: the clamped cell
    // search of stage() (identical to stage_fast's cell where nothing clamps),
    // without its halo bounds and 2-D branches — border tiles no longer take
    // the general path (their clamped corners stay inside the staged tiles)
    __device__ void stage_point(const PlaneCtx& pc, int x0, int y0, int zi, int row, int col,
                                T v[3]) const {
        const int gx = x0 + col, gy = y0 + row, zg = zi + d.zoff;
        const int so = row * BXS + col + (XAS - R);
        const T s0 = pc.step[so], s1 = pc.step[PS + so], s2 = pc.step[2 * PS + so];
        AxisCell<T> ax, ay, az;
        locate_cells3<T>(gx, gy, zg, s0, s1, s2, d.nx, d.ny, d.gz(), ax, ay, az);
        const int o = (ay.i0 - (y0 - HU)) * BXU + (ax.i0 - (x0 - XAU));
        const T fx = ax.f, fy = ay.f, fz = az.f;
        const T wx0 = T(1) - fx, wy0 = T(1) - fy, wz0 = T(1) - fz;
        const T w00 = wx0 * wy0, w10 = fx * wy0, w01 = wx0 * fy, w11 = fx * fy;
        const int dz = az.i0 - zg;
        const T* u0 = pc.u[CAPH];
        const T* u1 = pc.u[CAPH];
#pragma unroll
        for (int k = 0; k < 2 * CAPH; ++k)
            if (dz == k - CAPH) {
                u0 = pc.u[k];
                u1 = pc.u[k + 1];
            }
        const T s[3] = {s0, s1, s2};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const T* a = u0 + k * PU + o;
            const T* b = u1 + k * PU + o;
            const T lo = bilerp4(w00, w10, w01, w11, a[0], a[1], a[BXU], a[BXU + 1]);
            const T hi = bilerp4(w00, w10, w01, w11, b[0], b[1], b[BXU], b[BXU + 1]);
            v[k] = s[k] + zlerp(wz0, lo, fz, hi);
        }
    }
    // composed value step + u(x + step) at halo element (row, col) of plane zi
    __device__ void stage(const PlaneCtx& pc, int x0, int y0, int zi, int row, int col,
                          T v[3]) const {
        const int gx = x0 - R + col, gy = y0 - R + row, zg = zi + d.zoff;
        if (gx < 0 || gx >= d.nx || gy < 0 || gy >= d.ny || zg < 0 || zg >= d.gz()) {
            v[0] = v[1] = v[2] = T(0);
            return;
        }
        const int so = row * BXS + col + (XAS - R);
        const T s0 = pc.step[so], s1 = pc.step[PS + so];
        const bool three = d.ndim == 3;
        const T s2 = three ? pc.step[2 * PS + so] : T(0);
        const AxisCell<T> ax = locate_axis(gx, s0, d.nx);
        const AxisCell<T> ay = locate_axis(gy, s1, d.ny);
        int dz = 0;  // lower z corner relative to zi, in [-CAPH, CAPH-1]
        T fz = T(0);
        if (three) {
            const AxisCell<T> az = locate_axis(zg, s2, d.gz());
            dz = az.i0 - zg;
            fz = az.f;
        }
        const int o = (ay.i0 - (y0 - HU)) * BXU + (ax.i0 - (x0 - XAU));
        // 8 corner weights, computed once for the 3 components
        const T wx0 = T(1) - ax.f, wx1 = ax.f, wy0 = T(1) - ay.f, wy1 = ay.f;
        const T w00 = wx0 * wy0, w10 = wx1 * wy0, w01 = wx0 * wy1, w11 = wx1 * wy1;
        const T wz0 = T(1) - fz, wz1 = fz;
        const T* u0 = pc.u[CAPH];
        const T* u1 = pc.u[CAPH];
#pragma unroll
        for (int k = 0; k < 2 * CAPH; ++k)
            if (dz == k - CAPH) {
                u0 = pc.u[k];
                u1 = pc.u[k + 1];
            }
        const T s[3] = {s0, s1, s2};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const T* a = u0 + k * PU + o;
            T acc = bilerp4(w00, w10, w01, w11, a[0], a[1], a[BXU], a[BXU + 1]);
            if (three) {
                const T* b = u1 + k * PU + o;
                const T up = bilerp4(w00, w10, w01, w11, b[0], b[1], b[BXU], b[BXU + 1]);
                acc = zlerp(wz0, acc, wz1, up);
            }
            v[k] = (k < d.ndim) ? s[k] + acc : T(0);
        }
    }
    __device__ void xpass(const unsigned char*, int, int, Acc, Acc*) const {}
    __device__ void load_center(int, int, int, Center&) const {}
    __device__ void finish_wg(const Carry& c) const {
        W[c.i] = wg3_value(c.w);
        T gr[3];
        wg3_grad(c.w, gr);
        G[0][c.i] = gr[0];
        G[1][c.i] = gr[1];
        G[2][c.i] = gr[2];
    }
    __device__ Red2 emit(int x, int y, int z, const T u[3], const Center&, const Prol&,
                         Carry& cr) const {
        const int i = d.idx32(x, y, z);
        uout[0][i] = u[0];
        uout[1][i] = u[1];
        uout[2][i] = u[2];
        if (W) {  // similarity.cpp:25-45 for the next loss evaluation (3-D only: launcher)
            if (cr.valid) finish_wg(cr);
            wg3_fetch<T>(M, dm, x, y, z + d.zoff, u[0], u[1], u[2], cr.w);
            cr.i = static_cast<int>(i);
            cr.valid = true;
        }
        return {0.0, 0.0};
    }
    __device__ void flush(Carry& cr) const {
        if (W && cr.valid) finish_wg(cr);
    }
    __device__ void finish(int, double, double, const Prol&) const {
        if (st && count_update) st->nupdates += 1;
    }
};

// interp.cpp:362-371 + similarity.cpp:25-45: sigma_warp smoothing of the
// composed field c (SmoothAdam2<..., CAPH> wrote it), u' = G * c, then the
// fused W = M(x+u'), G = grad M(x+u') epilogue (3-D fast gather, carried one
// plane).  With the pointwise compose in the Adam kernel this replaces
// Compose2, which recomposed every halo element of its tile (1.7x work).
template <class T, int R_, int TY_ = DFM_TY_CS, bool ASYNC_ = DFM_CS_ASYNC, bool FLAT_ = true>
struct ComposeS2 {
    using Acc = T;
    using Center = NoCenter;
    using Prol = NoProl;
    static constexpr int R = R_, C = 3, BACK = 0, AHEAD = 0, S = DFM_S_SA, TYv = TY_;
    static constexpr int kMinB = DFM_MINB_CS, kCY = DFM_CY_CS;
    static constexpr bool kStaged = false, kSum = false, kMax = false;
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    static constexpr int kStageBytes = 3 * kBox;
    CUtensorMap mC;
    GaussW<T> w;
    T* uout[3];  // per-component plane pointers (3-D only)
    const T* M;
    Dims dm;
    T* W;
    T* G[3];
    LoopState* st;
    int count_update;
    Dims d;
    struct Carry {
        bool valid;
        int slot;  // shared-memory slot of the gather in flight
        int i;
        WG3<T> w;
    };
    static constexpr int NTH = TX * TYv / kCY;
    // the 8 corners of the carried M gather land here (cp.async), two slots
    static constexpr bool kAsync = ASYNC_;
    // slots 2r, 2r+1 belong to the thread's row r
    static constexpr int kExtraBytes = kAsync ? 2 * kCY * 8 * NTH * int(sizeof(T)) : 0;
    __device__ static T* gather_buf(int slot) {
        return reinterpret_cast<T*>(zm2_extra<ComposeS2>()) + (slot * 8) * NTH + threadIdx.x;
    }
    __device__ void init_carry(Carry& c, int r) const { c.slot = 2 * r; }

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
    __device__ void prefetch_maps() const { prefetch_tmap(&mC); }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 3 * kBytes);
#pragma unroll
        for (int k = 0; k < 3; ++k) tma_load_4d(dst + k * kBox, &mC, bar, x0 - XA, y0 - R, q, k);
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const { return {}; }
    static constexpr bool kXQuad = sizeof(T) == 4;
    __device__ void xpass4(const unsigned char* st_, int row, int col, const Acc nx[4],
                           Acc v[3][4]) const {
        constexpr int NCH = (XA + R + 4 + 3) / 4;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float wv[4 * NCH];
            load_row4<NCH>(reinterpret_cast<const float*>(st_) + c * (kBox / 4) + row * BX + col,
                           wv);
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                const float* q = wv + o + (XA - R);
                T a = T(0);
#pragma unroll
                for (int j = 0; j < 2 * R + 1; ++j) a += w.taps[0][j] * q[j];
                v[c][o] = a * nx[o];
            }
        }
    }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc nx, Acc v[3]) const {
        const T* p = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T* q = p + c * (kBox / int(sizeof(T)));
            T a = T(0);
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) a += w.taps[0][j] * q[j];
            v[c] = a * nx;
        }
    }
    __device__ void load_center(int, int, int, Center&) const {}
    __device__ void finish_wg(const Carry& c) const {
        W[c.i] = wg3_value(c.w);
        T gr[3];
        wg3_grad(c.w, gr);
        G[0][c.i] = gr[0];
        G[1][c.i] = gr[1];
        G[2][c.i] = gr[2];
    }
    __device__ Red2 emit(int x, int y, int z, const T u[3], const Center&, const Prol&,
                         Carry& cr) const {
        const int i = d.idx32(x, y, z);
        uout[0][i] = u[0];
        uout[1][i] = u[1];
        uout[2][i] = u[2];
        if (W) {
            if constexpr (!kAsync) {
                if (cr.valid) finish_wg(cr);
                wg3_fetch<T, true, FLAT_>(M, dm, x, y, z + d.zoff, u[0], u[1], u[2], cr.w);
                cr.i = i;
                cr.valid = true;
                return {0.0, 0.0};
            }
            if (cr.valid) {
                cp_async_wait_all();
                wg3_load(cr.w, gather_buf(cr.slot), NTH);
                finish_wg(cr);
            }
            cr.slot ^= 1;
            wg3_fetch_async<T, FLAT_>(M, dm, x, y, z + d.zoff, u[0], u[1], u[2], cr.w,
                               gather_buf(cr.slot), NTH);
            cr.i = i;
            cr.valid = true;
        }
        return {0.0, 0.0};
    }
    __device__ void flush(Carry& cr) const {
        if (W && cr.valid) {
            if constexpr (kAsync) {
                cp_async_wait_all();
                wg3_load(cr.w, gather_buf(cr.slot), NTH);
            }
            finish_wg(cr);
        }
    }
    __device__ void finish(int, double, double, const Prol&) const {
        if (st && count_update) st->nupdates += 1;
    }
};

// interp.cpp:110-151 — one-component Gaussian smoothing (the pyramid's
// pre-blur before downsampling), same arithmetic as the generic z-march
// GaussOp of kernels_stencil.cu with TMA-fed planes and the quad x filter
template <class T, int R_, int TY_ = 8>
struct Gauss2 {
    using Acc = T;
    using Center = NoCenter;
    using Prol = NoProl;
    using Carry = NoCarry;
    static constexpr int R = R_, C = 1, BACK = 0, AHEAD = 0, S = 4, TYv = TY_;
    static constexpr int kMinB = 3, kCY = 1;
    static constexpr bool kStaged = false, kSum = false, kMax = false;
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    static constexpr int kStageBytes = kBox;
    CUtensorMap mI;
    GaussW<T> w;
    T* out;
    Dims d;

    __device__ bool skip() const { return false; }
    __device__ void prefetch_maps() const { prefetch_tmap(&mI); }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, kBytes);
        tma_load_4d(dst, &mI, bar, x0 - XA, y0 - R, q, 0);
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const { return {}; }
    static constexpr bool kXQuad = sizeof(T) == 4;
    __device__ void xpass4(const unsigned char* st_, int row, int col, const Acc nx[4],
                           Acc v[1][4]) const {
        constexpr int NCH = (XA + R + 4 + 3) / 4;
        float wv[4 * NCH];
        load_row4<NCH>(reinterpret_cast<const float*>(st_) + row * BX + col, wv);
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            T a = T(0);
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) a += w.taps[0][j] * wv[o + (XA - R) + j];
            v[0][o] = a * nx[o];
        }
    }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc nx, Acc v[1]) const {
        const T* q = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
        T a = T(0);
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) a += w.taps[0][j] * q[j];
        v[0] = a * nx;
    }
    __device__ void load_center(int, int, int, Center&) const {}
    __device__ Red2 emit(int x, int y, int z, const T s[1], const Center&, const Prol&,
                         Carry&) const {
        out[d.idx32(x, y, z)] = s[0];
        return {0.0, 0.0};
    }
    __device__ void flush(Carry&) const {}
    __device__ void finish(int, double, double, const Prol&) const {}
};

// pipeline.cpp:199-205 — the SVF update v' = G_sigma_warp * (v + step) (the
// generic z-march SvfUpdateOp's arithmetic: sum per element, then the three
// normalised passes) with TMA-fed planes; one counted update per launch
template <class T, int R_, int TY_ = 8>
struct SvfUpdate2 {
    using Acc = T;
    using Center = NoCenter;
    using Prol = NoProl;
    using Carry = NoCarry;
    static constexpr int R = R_, C = 3, BACK = 0, AHEAD = 0, S = 4, TYv = TY_;
    static constexpr int kMinB = 2, kCY = 1;
    static constexpr bool kStaged = false, kSum = false, kMax = false;
    static constexpr int XA = round_bx<T>(R), BX = round_bx<T>(TX + XA + R), BY = TYv + 2 * R;
    static constexpr int kBytes = BX * BY * int(sizeof(T));
    static constexpr int kBox = align128(kBytes);
    static constexpr int kStageBytes = 6 * kBox;  // v (3 components), step (3)
    CUtensorMap mV, mS;
    GaussW<T> w;
    T* out[3];
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
    __device__ void prefetch_maps() const {
        prefetch_tmap(&mV);
        prefetch_tmap(&mS);
    }
    __device__ void issue(unsigned char* dst, uint64_t* bar, int x0, int y0, int q) const {
        mbar_expect_tx(bar, 6 * kBytes);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            tma_load_4d(dst + k * kBox, &mV, bar, x0 - XA, y0 - R, q, k);
            tma_load_4d(dst + (3 + k) * kBox, &mS, bar, x0 - XA, y0 - R, q, k);
        }
    }
    __device__ Acc wgt(int a, int j) const { return w.taps[a][j]; }
    __device__ Acc nrm(int a, int i) const {
        return w.nrm(a, i, a == 0 ? d.nx : (a == 1 ? d.ny : d.gz()));
    }
    __device__ Prol prologue() const { return {}; }
    __device__ void xpass(const unsigned char* st_, int row, int col, Acc nx, Acc v[3]) const {
        const T* p = reinterpret_cast<const T*>(st_) + row * BX + col + (XA - R);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T* pv = p + c * (kBox / int(sizeof(T)));
            const T* ps = p + (3 + c) * (kBox / int(sizeof(T)));
            T a = T(0);
#pragma unroll
            for (int j = 0; j < 2 * R + 1; ++j) a += w.taps[0][j] * (pv[j] + ps[j]);
            v[c] = a * nx;
        }
    }
    __device__ void load_center(int, int, int, Center&) const {}
    __device__ Red2 emit(int x, int y, int z, const T s[3], const Center&, const Prol&,
                         Carry&) const {
        const int i = d.idx32(x, y, z);
#pragma unroll
        for (int c = 0; c < 3; ++c) out[c][i] = s[c];
        return {0.0, 0.0};
    }
    __device__ void flush(Carry&) const {}
    __device__ void finish(int, double, double, const Prol&) const {
        if (st) st->nupdates += 1;
    }
};

// W = M(x+u), G = grad M(x+u) (similarity.cpp:25-45) at scale start / epilogue
template <class T>
__global__ void k_warpgrad(const T* __restrict__ M, Dims dm, CPlanes3<T> u, Dims d,
                           T* __restrict__ W, T* __restrict__ G) {
    // (x, row) mapping, 32 x 8 blocks: no 64-bit index division per voxel
    const int x = blockIdx.x * 32 + threadIdx.x;
    if (x >= d.nx) return;
    const int rows = d.ny * d.nz;
    for (int row = blockIdx.y * 8 + threadIdx.y; row < rows; row += gridDim.y * 8) {
        const int y = row % d.ny, z = row / d.ny;
        const int64_t i = d.idx(x, y, z);
        if (d.ndim == 3 && dm.nx > 1 && dm.ny > 1 && dm.nz > 1 && dm.n < (int64_t(1) << 31)) {
            WG3<T> w;
            wg3_fetch<T>(M, dm, x, y, z + d.zoff, __ldg(u.c[0] + i), __ldg(u.c[1] + i),
                         __ldg(u.c[2] + i), w);
            W[i] = wg3_value(w);
            if (G) {
                T gr[3];
                wg3_grad(w, gr);
                G[i] = gr[0];
                G[d.n + i] = gr[1];
                G[2 * d.n + i] = gr[2];
            }
            continue;
        }
        const Cell3<T> c = locate3<T>(dm, x, y, z + d.zoff, __ldg(u.c[0] + i),
                                      __ldg(u.c[1] + i), d.ndim == 3 ? __ldg(u.c[2] + i) : T(0));
        const Corners<T> k = fetch_corners<T>(M, c);
        W[i] = lerp_value(c, k);
        if (G) {
            T gr[3];
            lerp_grad(c, k, d.ndim, gr);
            G[i] = gr[0];
            G[d.n + i] = gr[1];
            G[2 * d.n + i] = gr[2];
        }
    }
}

// ---------------------------------------------------------------------------
// host side: tensor maps and launches

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <class T>
bool make_map(CUtensorMap* m, const T* base, const Dims& d, int ncomp, int bx, int by) {
    auto enc = encoder();
    if (!enc) return false;
    const cuuint64_t esz = sizeof(T);
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(d.nx), static_cast<cuuint64_t>(d.ny),
                          static_cast<cuuint64_t>(d.nz), static_cast<cuuint64_t>(ncomp)};
    cuuint64_t strides[3] = {d.nx * esz, static_cast<cuuint64_t>(d.nx) * d.ny * esz,
                             static_cast<cuuint64_t>(d.n) * esz};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(bx), static_cast<cuuint32_t>(by), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = enc(m, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                           4, const_cast<T*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <class Op>
size_t zm2_smem() {
    return 128 + ((zm2_core_bytes<Op>() + 15) & ~15) + ExtraBytes<Op>::value;
}

// z-chunk length minimising the makespan: waves of resident CTAs x planes per
// CTA (chunk + halo planes), given the kernel's measured residency per SM.
inline int pick_chunks(const Dims& d, int tiles, int slots, int halo_planes, int* zchunk) {
    double best = 1e30;
    int best_n = 1, best_chunk = d.nz;
    for (int nch = 1; nch <= d.nz; ++nch) {
        const int chunk = (d.nz + nch - 1) / nch;
        const int nreal = (d.nz + chunk - 1) / chunk;
        if (nreal != nch || static_cast<int64_t>(tiles) * nch > 65536) continue;
        const int blocks = tiles * nch;
        const int waves = (blocks + slots - 1) / slots;
        // per-wave cost in plane-steps plus a small per-CTA fixed cost
        const double cost = static_cast<double>(waves) * (chunk + halo_planes + 2.0);
        if (cost < best - 1e-9) {
            best = cost;
            best_n = nch;
            best_chunk = chunk;
        }
    }
    *zchunk = best_chunk;
    return best_n;
}

template <class Op>
int run_zm2(const Launch& L, const Op& op, Dims d) {
    ZG2 g;
    g.d = d;
    const size_t smem = zm2_smem<Op>();
    int occ = kernel_setup(reinterpret_cast<const void*>(k_zm2<Op>), TX * Op::TYv / Op::kCY,
                           smem);  // resident CTAs per SM
    if (occ < 1) occ = 1;
    g.tiles_x = (d.nx + TX - 1) / TX;
    const int tiles = g.tiles_x * ((d.ny + Op::TYv - 1) / Op::TYv);
    // resident-CTA slots the chunking may plan for (DFM_SLOT_CAP caps CTAs per
    // SM: beyond ~2 the per-SM issue rate saturates and extra chunks only add
    // halo planes)
    static const int slot_cap = getenv("DFM_SLOT_CAP") ? atoi(getenv("DFM_SLOT_CAP")) : 0;
    const int per_sm = slot_cap > 0 && slot_cap < occ ? slot_cap : occ;
    const int slots = per_sm * (L.num_sms > 0 ? L.num_sms : 148);
    Dims dr = d;  // chunk the produced plane range only
    dr.nz = d.out_end() - d.out_begin();
    const int nchunks = pick_chunks(dr, tiles, slots, 2 * Op::R + Op::BACK + Op::AHEAD, &g.zchunk);
    launch_maybe_pdl(L, k_zm2<Op>, dim3(tiles, nchunks), dim3(TX * Op::TYv / Op::kCY), smem, op,
                     g);
    L.bump();
    return tiles * nchunks;
}

template <int RLO, int RHI, class F>
int with_r(int R, F&& f) {
    switch (R) {
#define DFM_R2(r)                                                                   \
    case r:                                                                         \
        if constexpr (r >= RLO && r <= RHI) return f(std::integral_constant<int, r>{}); \
        break;
        DFM_R2(0) DFM_R2(1) DFM_R2(2) DFM_R2(3) DFM_R2(4) DFM_R2(5) DFM_R2(6) DFM_R2(7) DFM_R2(8)
#undef DFM_R2
    }
    return -2;
}

}  // namespace

bool tma_supported_(Dims d, int esz) {
    return encoder() != nullptr && (static_cast<int64_t>(d.nx) * esz) % 16 == 0;
}

template <class T>
int launch_lncc_fwd_tma(const Launch& L, int R, const T* F, const T* W, Dims d, T* coef,
                        double* partials, const LoopState* st, const MonitorArgs* mon) {
    return with_r<1, 5>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        using Op = LnccFwd2<T, RR>;
        Op op;
        if (!make_map<T>(&op.mF, F, d, 1, Op::BX, Op::BY) ||
            !make_map<T>(&op.mW, W, d, 1, Op::BX, Op::BY))
            return -1;
        op.coef = coef;
        op.partials = partials;
        op.st = st;
        op.mon = mon ? *mon : MonitorArgs{nullptr, nullptr, nullptr, 0, 0.0};
        op.d = d;
        return run_zm2(L, op, d);
    });
}

template <class T>
int launch_fstats_tma(const Launch& L, int R, const T* F, Dims d, double* fstat) {
    return with_r<1, 5>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        using Op = FStats2<T, RR>;
        Op op;
        if (!make_map<T>(&op.mF, F, d, 1, Op::BX, Op::BY)) return -1;
        op.fstat = fstat;
        op.d = d;
        return run_zm2(L, op, d);
    });
}

template <class T>
int launch_lncc_fwd3_tma(const Launch& L, int R, const T* F, const T* W, const double* fstat,
                         Dims d, T* coef, double* partials, const LoopState* st,
                         const MonitorArgs* mon) {
    return with_r<1, 5>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        using Op = LnccFwd3<T, RR>;
        Op op;
        if (!make_map<T>(&op.mF, F, d, 1, Op::BX, Op::BY) ||
            !make_map<T>(&op.mW, W, d, 1, Op::BX, Op::BY))
            return -1;
        op.fstat = fstat;
        for (int k = 0; k < 4; ++k) op.coef[k] = coef + k * d.n;
        op.partials = partials;
        op.st = st;
        op.mon = mon ? *mon : MonitorArgs{nullptr, nullptr, nullptr, 0, 0.0};
        op.d = d;
        return run_zm2(L, op, d);
    });
}

template <class T>
int launch_lncc_bwd_tma(const Launch& L, int R, const T* coef, const T* F, const T* W,
                        const T* G, Dims d, T* grad, const LoopState* st) {
    if (d.ndim != 3) return -2;
    return with_r<1, 5>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        using Op = LnccBwd2<T, RR>;
        Op op;
        if (!make_map<T>(&op.mC, coef, d, 4, Op::BX, Op::BY)) return -1;
        op.F = F;
        op.W = W;
        for (int k = 0; k < 3; ++k) {
            op.G[k] = G + k * d.n;
            op.grad[k] = grad + k * d.n;
        }
        op.m2n = -2.0 / (static_cast<double>(d.nx) * d.ny * d.gz());  // global N
        op.st = st;
        op.d = d;
        return run_zm2(L, op, d);
    });
}

template <class T>
int launch_smooth_adam_tma(const Launch& L, int R, const GaussW<T>& w, const T* grad, T* m,
                           T* nu, T* step, Dims d, AdamParams ap, LoopState* st,
                           unsigned long long* maxstep, const T* ujac) {
    if (d.ndim != 3) return -2;
    if (ap.use_jac && !ujac) return -2;
    return with_r<0, 6>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        auto go = [&](auto op) {
            using Op = decltype(op);
            if (!make_map<T>(&op.mG, grad, d, 3, Op::BX, Op::BY)) return -1;
            if (Op::kCenterTMA && (!make_map<T>(&op.mM, m, d, 3, TX, Op::TYv) ||
                                   !make_map<T>(&op.mN, nu, d, 3, TX, Op::TYv)))
                return -1;
            op.w = w;
            for (int k = 0; k < 3; ++k) {
                op.m[k] = m + k * d.n;
                op.nu[k] = nu + k * d.n;
                op.step[k] = step + k * d.n;
            }
            for (int k = 0; k < 3; ++k) op.ujac[k] = ujac ? ujac + k * d.n : nullptr;
            op.ak = adam_k<T>(ap);
            op.corr1 = ap.corr1;
            op.corr2 = ap.corr2;
            op.st = st;
            op.maxstep = maxstep;
            op.d = d;
            return run_zm2(L, op, d);
        };
        if (ap.use_jac) return go(SmoothAdam2<T, RR, 8, 1, DFM_MINB_SA, 0, true>{});
        // large levels: two rows per thread (measured -8% at 160x192x224,
        // +8% at 80x96x112); fp64 keeps one row (register budget)
        // (register ring of 2 x 3 x (2R+1): only for the BASELINE sigma_grad 1.0;
        // at R = 5 it spills, 504 vs ~160 us)
        if constexpr (RR <= 3) {
            if (sizeof(T) == 4 && d.n >= L.large_min)
                return go(SmoothAdam2<T, RR, 16, 2, DFM_MINB_SA2>{});
        }
        // 512-thread CTAs (TY 16) get 64 registers at 2 CTAs per SM: the
        // gradient ring of radius >= 4 and every fp64 variant spill there
        if constexpr (RR >= 4 || sizeof(T) == 8) return go(SmoothAdam2<T, RR, 8>{});
        return go(SmoothAdam2<T, RR>{});
    });
}

template <class T>
int launch_compose_tma(const Launch& L, int R, double cap, const GaussW<T>& w, const T* step,
                       const T* uin, T* uout, const T* M, Dims dm, Dims d, T* W, T* G,
                       LoopState* st, bool count_update) {
    const int caph = cap <= 0.5 ? 1 : (cap <= 1.5 ? 2 : 0);
    if (caph == 0 || d.ndim != 3) return -2;  // 3-D plane pointers, fast M gather
    return with_r<0, 4>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        auto go = [&](auto ch) {
            constexpr int CH = decltype(ch)::value;
            using Op = Compose2<T, RR, CH>;
            Op op;
            if (!make_map<T>(&op.mS, step, d, 3, Op::BXS, Op::BYS) ||
                !make_map<T>(&op.mU, uin, d, 3, Op::BXU, Op::BYU))
                return -1;
            op.w = w;
            for (int k = 0; k < 3; ++k) {
                op.uout[k] = uout + k * d.n;
                op.G[k] = G ? G + k * d.n : nullptr;
            }
            op.M = M;
            op.dm = dm;
            op.W = W;
            op.st = st;
            op.count_update = count_update ? 1 : 0;
            op.d = d;
            return run_zm2(L, op, d);
        };
        return caph == 1 ? go(std::integral_constant<int, 1>{})
                         : go(std::integral_constant<int, 2>{});
    });
}

template <class T>
int launch_smooth_adam_compose_tma(const Launch& L, int R, const GaussW<T>& w, const T* grad,
                                   T* m, T* nu, const T* uin, T* cout, double cap, Dims d,
                                   AdamParams ap, LoopState* st, unsigned long long* maxstep) {
    const int caph = cap <= 0.5 ? 1 : (cap <= 1.5 ? 2 : 0);
    if (caph == 0 || d.ndim != 3) return -2;
    return with_r<0, 6>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        auto go = [&](auto op) {
            using Op = decltype(op);
            if (!make_map<T>(&op.mG, grad, d, 3, Op::BX, Op::BY)) return -1;
            if (Op::kCenterTMA && (!make_map<T>(&op.mM, m, d, 3, TX, Op::TYv) ||
                                   !make_map<T>(&op.mN, nu, d, 3, TX, Op::TYv)))
                return -1;
            op.w = w;
            for (int k = 0; k < 3; ++k) {
                op.m[k] = m + k * d.n;
                op.nu[k] = nu + k * d.n;
                op.step[k] = cout + k * d.n;
            }
            op.uin = uin;
            for (int k = 0; k < 3; ++k) op.uin3[k] = uin + k * d.n;
            op.ak = adam_k<T>(ap);
            op.corr1 = ap.corr1;
            op.corr2 = ap.corr2;
            op.st = st;
            op.maxstep = maxstep;
            op.d = d;
            return run_zm2(L, op, d);
        };
        auto pick = [&](auto ch) {  // the carried gather needs ~100 registers
            constexpr int CH = decltype(ch)::value;
            return go(SmoothAdam2<T, RR, DFM_TY_SAC, 1, DFM_MINB_SAC, CH>{});
        };
        return caph == 1 ? pick(std::integral_constant<int, 1>{})
                         : pick(std::integral_constant<int, 2>{});
    });
}

// pointwise compose c = step + u(x + step) (interp.cpp:269-289), one voxel
// per thread, for the split update on large levels: a light streaming kernel
// at full occupancy hides the 24 gathers better than the Adam epilogue can
template <class T, int CAPH>
__global__ void __launch_bounds__(256) k_compose_pw(const T* __restrict__ step,
                                                    const T* __restrict__ u, Dims d,
                                                    T* __restrict__ c, const LoopState* st) {
    if (st && (st->done || st->bad_step)) return;
    const int64_t i = blockIdx.x * 256ll + threadIdx.x;
    if (i >= d.n) return;
    const int x = static_cast<int>(i % d.nx);
    const int64_t r = i / d.nx;
    const int y = static_cast<int>(r % d.ny), z = static_cast<int>(r / d.ny);
    const T s[3] = {step[i], step[d.n + i], step[2 * d.n + i]};
    T cv[3];
    compose_at<T, CAPH>(u, d, x, y, z + d.zoff, s, cv);
    c[i] = cv[0];
    c[d.n + i] = cv[1];
    c[2 * d.n + i] = cv[2];
}

template <class T>
int launch_compose_pointwise(const Launch& L, const T* step, const T* u, double cap, Dims d,
                             T* c, const LoopState* st) {
    const unsigned nb = static_cast<unsigned>((d.n + 255) / 256);
    if (cap <= 0.5)
        k_compose_pw<T, 1><<<nb, 256, 0, L.stream>>>(step, u, d, c, st);
    else if (cap <= 1.5)
        k_compose_pw<T, 2><<<nb, 256, 0, L.stream>>>(step, u, d, c, st);
    else
        k_compose_pw<T, (1 << 20)><<<nb, 256, 0, L.stream>>>(step, u, d, c, st);
    L.bump();
    return static_cast<int>(nb);
}

template <class Op, class T>
int go_compose_smooth(const Launch& L, const GaussW<T>& w, const T* c, T* uout, const T* M,
                      Dims dm, Dims d, T* W, T* G, LoopState* st, bool count_update);

template <class T>
int launch_compose_smooth_tma(const Launch& L, int R, const GaussW<T>& w, const T* c, T* uout,
                              const T* M, Dims dm, Dims d, T* W, T* G, LoopState* st,
                              bool count_update) {
    if (d.ndim != 3) return -2;
    return with_r<0, 4>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        // the cp.async carried gather pays on large levels (-10 us/iteration at
        // 160x192x224), the register carry on mid ones (-1.6 us at 80x96x112)
        if (d.n >= L.large_min) {
            if (dm.nx > 1 && dm.ny > 1 && dm.nz > 1)  // no flat axis: no per-voxel check
                return go_compose_smooth<ComposeS2<T, RR, DFM_TY_CS, DFM_CS_ASYNC != 0, false>>(
                    L, w, c, uout, M, dm, d, W, G, st, count_update);
            return go_compose_smooth<ComposeS2<T, RR, DFM_TY_CS, DFM_CS_ASYNC != 0>>(
                L, w, c, uout, M, dm, d, W, G, st, count_update);
        }
        if (dm.nx > 1 && dm.ny > 1 && dm.nz > 1)
            return go_compose_smooth<ComposeS2<T, RR, DFM_TY_CS, false, false>>(
                L, w, c, uout, M, dm, d, W, G, st, count_update);
        return go_compose_smooth<ComposeS2<T, RR, DFM_TY_CS, false>>(L, w, c, uout, M, dm, d, W,
                                                                      G, st, count_update);
    });
}

template <class Op, class T>
int go_compose_smooth(const Launch& L, const GaussW<T>& w, const T* c, T* uout, const T* M,
                      Dims dm, Dims d, T* W, T* G, LoopState* st, bool count_update) {
    Op op;
    if (!make_map<T>(&op.mC, c, d, 3, Op::BX, Op::BY)) return -1;
    op.w = w;
    for (int k = 0; k < 3; ++k) {
        op.uout[k] = uout + k * d.n;
        op.G[k] = G ? G + k * d.n : nullptr;
    }
    op.M = M;
    op.dm = dm;
    op.W = W;
    op.st = st;
    op.count_update = count_update ? 1 : 0;
    op.d = d;
    return run_zm2(L, op, d);
}

template <class T>
int launch_svf_update_tma(const Launch& L, int R, const GaussW<T>& w, const T* v, const T* step,
                          T* out, Dims d, LoopState* st) {
    if (d.ndim != 3) return -2;
    return with_r<0, 4>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        using Op = SvfUpdate2<T, RR>;
        Op op;
        if (!make_map<T>(&op.mV, v, d, 3, Op::BX, Op::BY) ||
            !make_map<T>(&op.mS, step, d, 3, Op::BX, Op::BY))
            return -1;
        op.w = w;
        for (int k = 0; k < 3; ++k) op.out[k] = out + k * d.n;
        op.st = st;
        op.d = d;
        return run_zm2(L, op, d);
    });
}

template <class T>
int launch_gauss_tma(const Launch& L, int R, const GaussW<T>& w, const T* in, T* out, Dims d) {
    if (d.ndim != 3) return -2;
    return with_r<1, 6>(R, [&](auto rc) {
        constexpr int RR = decltype(rc)::value;
        using Op = Gauss2<T, RR>;
        Op op;
        if (!make_map<T>(&op.mI, in, d, 1, Op::BX, Op::BY)) return -1;
        op.w = w;
        op.out = out;
        op.d = d;
        return run_zm2(L, op, d);
    });
}

template <class T>
void launch_warpgrad(const Launch& L, const T* M, Dims dm, CPlanes3<T> u, Dims d, T* W, T* G) {
    const int64_t by = (static_cast<int64_t>(d.ny) * d.nz + 7) / 8;
    const dim3 grid((d.nx + 31) / 32, static_cast<unsigned>(by < 65535 ? by : 65535));
    k_warpgrad<T><<<grid, dim3(32, 8), 0, L.stream>>>(M, dm, u, d, W, G);
    L.bump();
}

#define DFM_INST_TMA(T)                                                                        \
    template int launch_lncc_fwd_tma<T>(const Launch&, int, const T*, const T*, Dims, T*,      \
                                        double*, const LoopState*, const MonitorArgs*);        \
    template int launch_lncc_bwd_tma<T>(const Launch&, int, const T*, const T*, const T*,      \
                                        const T*, Dims, T*, const LoopState*);                 \
    template int launch_fstats_tma<T>(const Launch&, int, const T*, Dims, double*);           \
    template int launch_lncc_fwd3_tma<T>(const Launch&, int, const T*, const T*,               \
                                         const double*, Dims, T*, double*, const LoopState*,   \
                                         const MonitorArgs*);                                  \
    template int launch_smooth_adam_tma<T>(const Launch&, int, const GaussW<T>&, const T*, T*, \
                                           T*, T*, Dims, AdamParams, LoopState*,               \
                                           unsigned long long*, const T*);                     \
    template int launch_compose_tma<T>(const Launch&, int, double, const GaussW<T>&, const T*, \
                                       const T*, T*, const T*, Dims, Dims, T*, T*,             \
                                       LoopState*, bool);                                      \
    template void launch_warpgrad<T>(const Launch&, const T*, Dims, CPlanes3<T>, Dims, T*, T*); \
    template int launch_gauss_tma<T>(const Launch&, int, const GaussW<T>&, const T*, T*, Dims); \
    template int launch_svf_update_tma<T>(const Launch&, int, const GaussW<T>&, const T*,       \
                                          const T*, T*, Dims, LoopState*);                      \
    template int launch_smooth_adam_compose_tma<T>(const Launch&, int, const GaussW<T>&,        \
                                                   const T*, T*, T*, const T*, T*, double,     \
                                                   Dims, AdamParams, LoopState*,               \
                                                   unsigned long long*);                       \
    template int launch_compose_pointwise<T>(const Launch&, const T*, const T*, double, Dims,   \
                                             T*, const LoopState*);                            \
    template int launch_compose_smooth_tma<T>(const Launch&, int, const GaussW<T>&, const T*,  \
                                              T*, const T*, Dims, Dims, T*, T*, LoopState*,    \
                                              bool);

DFM_INST_TMA(float)
DFM_INST_TMA(double)

}  // namespace DFM_TMA_NS

#ifndef DFM_TMA_NO_DISPATCH
// ---------------------------------------------------------------------------
// public launchers (dfm_kernels.cuh): 16-wide tiles where the last 32-wide x
// tile of a mid-size level would be at most half full (80 columns: 97.6 ->
// 93.7 us per iteration at 80x96x112; full-size and 32-multiple widths keep
// 32); DFM_OPT_NARROW 0 disables the choice
namespace tx16 {
template <class T>
int launch_lncc_fwd_tma(const Launch&, int, const T*, const T*, Dims, T*, double*,
                        const LoopState*, const MonitorArgs*);
template <class T>
int launch_lncc_bwd_tma(const Launch&, int, const T*, const T*, const T*, const T*, Dims, T*,
                        const LoopState*);
template <class T>
int launch_fstats_tma(const Launch&, int, const T*, Dims, double*);
template <class T>
int launch_lncc_fwd3_tma(const Launch&, int, const T*, const T*, const double*, Dims, T*,
                         double*, const LoopState*, const MonitorArgs*);
template <class T>
int launch_smooth_adam_tma(const Launch&, int, const GaussW<T>&, const T*, T*, T*, T*, Dims,
                           AdamParams, LoopState*, unsigned long long*, const T*);
template <class T>
int launch_compose_tma(const Launch&, int, double, const GaussW<T>&, const T*, const T*, T*,
                       const T*, Dims, Dims, T*, T*, LoopState*, bool);
template <class T>
int launch_gauss_tma(const Launch&, int, const GaussW<T>&, const T*, T*, Dims);
template <class T>
int launch_svf_update_tma(const Launch&, int, const GaussW<T>&, const T*, const T*, T*, Dims,
                          LoopState*);
template <class T>
int launch_smooth_adam_compose_tma(const Launch&, int, const GaussW<T>&, const T*, T*, T*,
                                   const T*, T*, double, Dims, AdamParams, LoopState*,
                                   unsigned long long*);
template <class T>
int launch_compose_smooth_tma(const Launch&, int, const GaussW<T>&, const T*, T*, const T*, Dims,
                              Dims, T*, T*, LoopState*, bool);
}  // namespace tx16

namespace {
bool narrow_tile(const Launch& L, const Dims& d) {
    const int rem = d.nx % kTX;
    return L.narrow && d.n < L.large_min && rem != 0 && rem <= kTX / 2 && d.nx >= kTX;
}
}  // namespace

bool tma_supported(Dims d, int esz) { return tx32::tma_supported_(d, esz); }

#define DFM_PICK(fn, ...) \
    (narrow_tile(L, d) ? tx16::fn<T>(__VA_ARGS__) : tx32::fn<T>(__VA_ARGS__))

template <class T>
int launch_lncc_fwd_tma(const Launch& L, int R, const T* F, const T* W, Dims d, T* coef,
                        double* partials, const LoopState* st, const MonitorArgs* mon) {
    return DFM_PICK(launch_lncc_fwd_tma, L, R, F, W, d, coef, partials, st, mon);
}
template <class T>
int launch_lncc_bwd_tma(const Launch& L, int R, const T* coef, const T* F, const T* W,
                        const T* G, Dims d, T* grad, const LoopState* st) {
    return DFM_PICK(launch_lncc_bwd_tma, L, R, coef, F, W, G, d, grad, st);
}
template <class T>
int launch_fstats_tma(const Launch& L, int R, const T* F, Dims d, double* fstat) {
    return DFM_PICK(launch_fstats_tma, L, R, F, d, fstat);
}
template <class T>
int launch_lncc_fwd3_tma(const Launch& L, int R, const T* F, const T* W, const double* fstat,
                         Dims d, T* coef, double* partials, const LoopState* st,
                         const MonitorArgs* mon) {
    return DFM_PICK(launch_lncc_fwd3_tma, L, R, F, W, fstat, d, coef, partials, st, mon);
}
template <class T>
int launch_smooth_adam_tma(const Launch& L, int R, const GaussW<T>& w, const T* grad, T* m,
                           T* nu, T* step, Dims d, AdamParams ap, LoopState* st,
                           unsigned long long* maxstep, const T* ujac) {
    return DFM_PICK(launch_smooth_adam_tma, L, R, w, grad, m, nu, step, d, ap, st, maxstep, ujac);
}
template <class T>
int launch_compose_tma(const Launch& L, int R, double cap, const GaussW<T>& w, const T* step,
                       const T* uin, T* uout, const T* M, Dims dm, Dims d, T* W, T* G,
                       LoopState* st, bool count_update) {
    return DFM_PICK(launch_compose_tma, L, R, cap, w, step, uin, uout, M, dm, d, W, G, st,
                    count_update);
}
template <class T>
int launch_gauss_tma(const Launch& L, int R, const GaussW<T>& w, const T* in, T* out, Dims d) {
    return DFM_PICK(launch_gauss_tma, L, R, w, in, out, d);
}
template <class T>
int launch_svf_update_tma(const Launch& L, int R, const GaussW<T>& w, const T* v, const T* step,
                          T* out, Dims d, LoopState* st) {
    return DFM_PICK(launch_svf_update_tma, L, R, w, v, step, out, d, st);
}
template <class T>
int launch_smooth_adam_compose_tma(const Launch& L, int R, const GaussW<T>& w, const T* grad,
                                   T* m, T* nu, const T* uin, T* cout, double cap, Dims d,
                                   AdamParams ap, LoopState* st, unsigned long long* maxstep) {
    return DFM_PICK(launch_smooth_adam_compose_tma, L, R, w, grad, m, nu, uin, cout, cap, d, ap,
                    st, maxstep);
}
template <class T>
int launch_compose_smooth_tma(const Launch& L, int R, const GaussW<T>& w, const T* c, T* uout,
                              const T* M, Dims dm, Dims d, T* W, T* G, LoopState* st,
                              bool count_update) {
    return DFM_PICK(launch_compose_smooth_tma, L, R, w, c, uout, M, dm, d, W, G, st,
                    count_update);
}
#undef DFM_PICK
template <class T>
int launch_compose_pointwise(const Launch& L, const T* step, const T* u, double cap, Dims d,
                             T* c, const LoopState* st) {
    return tx32::launch_compose_pointwise<T>(L, step, u, cap, d, c, st);
}
template <class T>
void launch_warpgrad(const Launch& L, const T* M, Dims dm, CPlanes3<T> u, Dims d, T* W, T* G) {
    tx32::launch_warpgrad<T>(L, M, dm, u, d, W, G);
}

DFM_INST_TMA(float)
DFM_INST_TMA(double)
#endif  // DFM_TMA_NO_DISPATCH

}  // namespace dfm
