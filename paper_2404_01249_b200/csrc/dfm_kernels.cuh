// dfm_kernels.cuh — host-callable launchers for every kernel of the path.
// Definitions live in kernels_*.cu with explicit float/double instantiations.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

#include "dfm_device.cuh"

namespace dfm {

// One-time setup of a kernel on the current device: opt in to `smem` bytes of
// dynamic shared memory and return its resident CTAs per SM (0 on failure).
// Function attributes belong to the device's context, so a process driving
// several GPUs (dfm_sweep over devices) configures each device once.
inline int kernel_setup(const void* kern, int block, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(dev, kern);
    const auto it = done.find(key);
    if (it != done.end()) return it->second;
    int occ = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem) != cudaSuccess) {
        cudaGetLastError();
        occ = 0;
    }
    done[key] = occ;
    return occ;
}

constexpr int kRMax = 8;          // largest radius of the fused z-march kernels
constexpr int kTX = 32, kTY = 8;  // z-march CTA tile (x, y)

// Device-resident loop bookkeeping for one registration (SURVEY §7 hard part 5:
// the convergence monitor runs on the device so the host never waits per
// iteration).
struct LoopState {
    int it;          // next record slot within the current scale
    int slot;        // slot of the iteration being processed
    int done;        // scale finished (converged) or failed
    int err;         // 0 ok, 2 numerical failure
    int converged;   // convergence monitor fired this scale
    int nupdates;    // updates applied this scale
    int bad_step;    // non-finite step seen (diffeo.cpp:52-59)
    unsigned int arrive;  // CTAs done in a fused loss+monitor launch (reset by the last)
    long long t;     // Adam step counter (optim.cpp:26), kept across scales
    double dice_p;   // dice: sum F*W
    double dice_d;   // dice: SF + SM + 1e-7
};

__device__ __forceinline__ unsigned long long dfm_global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Thread-0 part of the convergence monitor (pipeline.cpp:157-179): records the
// loss of the current iteration; non-finite -> error; converged -> the record
// is kept and the scale ends before the update; else the Adam step advances.
__device__ __forceinline__ void monitor_commit(LoopState* st, double v, double P, double D,
                                               double* loss, unsigned long long* stamp,
                                               int window, double tol) {
    const int slot = st->it;
    loss[slot] = v;
    stamp[slot] = dfm_global_ns();
    st->slot = slot;
    st->it = slot + 1;
    st->dice_p = P;
    st->dice_d = D;
    if (!isfinite(v)) {
        st->err = 2;
        st->done = 1;
        return;
    }
    const int n = slot + 1;
    if (n >= window + 1) {
        const double prev = loss[n - 1 - window];
        const double cur = loss[n - 1];
        const double den = fabs(prev) > 1e-30 ? fabs(prev) : 1e-30;
        const double rel = ((prev - cur) / static_cast<double>(window)) / den;
        if (rel < tol) {
            st->converged = 1;
            st->done = 1;
            return;
        }
    }
    st->t += 1;
}

// Kernel launch bookkeeping handed to every launcher.
struct Launch {
    cudaStream_t stream;
    int64_t* counter;  // incremented per kernel launch (host side)
    int num_sms;
    bool pdl = false;  // launch the loop kernels with programmatic dependent launch
    // levels with at least this many voxels take the large-level kernel variants
    // (two-row fp32 smooth+Adam, cp.async-carried compose-smooth gather);
    // DFM_OPT_LARGE_MIN lowers it so the tests reach those variants at any size
    int64_t large_min = 2000000;
    // mid-size levels whose last 32-wide x tile would be at most half full run
    // the 16-wide z-march instantiation (DFM_OPT_NARROW)
    bool narrow = true;
    void bump() const {
        if (counter) ++*counter;
    }
};

// Launches `kern` with programmatic stream serialization when L.pdl (the
// kernel must call pdl_wait() before touching its predecessor's outputs).
template <class Kern, class... Args>
inline cudaError_t launch_maybe_pdl(const Launch& L, Kern kern, dim3 grid, dim3 block,
                                    size_t smem, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = L.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = L.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Gaussian weights of one smoothing call (interp.cpp:114-123), per axis, padded
// with zero taps to a common radius; norm = 1 / (in-range tap sum) per position.
template <class A>
struct GaussW {
    A taps[3][2 * kRMax + 1];
    const A* norm[3];
    // positions ra <= i < n - ra see the whole window: their norm is the one
    // value norm_int (computed like the array's entries), no load needed
    A norm_int[3];
    int ra[3];
#ifdef __CUDACC__
    __device__ __forceinline__ A nrm(int a, int i, int n) const {
        return static_cast<unsigned>(i - ra[a]) < static_cast<unsigned>(max(n - 2 * ra[a], 0))
                   ? norm_int[a]
                   : __ldg(norm[a] + i);
    }
#endif
};

// -------- conversions / staging
template <class T, class S>
void launch_cast(const Launch& L, const S* in, T* out, int64_t n);
template <class T, class S>
void launch_aos_to_soa(const Launch& L, const S* aos, Planes3<T> out, int64_t n, int ndim);
template <class T, class S>
void launch_soa_to_aos(const Launch& L, CPlanes3<T> in, S* aos, int64_t n, int ndim);
template <class T>
void launch_fill(const Launch& L, T* p, int64_t n, T v);

// -------- pointwise / gather kernels
template <class T>
void launch_sample_points(const Launch& L, const T* img, Dims d, const double* pts, int64_t np,
                          double* vals, double* grads);
template <class T>
void launch_warp_image(const Launch& L, const T* img, Dims dimg, CPlanes3<T> u, Dims d, T* out);
template <class T>
void launch_warp_labels(const Launch& L, const int32_t* lab, CPlanes3<T> u, Dims d,
                        int32_t* out);
template <class T>
void launch_compose(const Launch& L, CPlanes3<T> phi, CPlanes3<T> psi, Dims d, Planes3<T> out);
template <class T>
void launch_jacobian_full(const Launch& L, CPlanes3<T> u, Dims d, T* out);
template <class T>
void launch_upsample_cubic(const Launch& L, CPlanes3<T> f, Dims ds, Planes3<T> out, Dims dd,
                           const double step[3], const double rescale[3]);
template <class T>
void launch_sgd(const Launch& L, Planes3<T> mu, CPlanes3<T> v, Dims d, double momentum);
template <class T>
void launch_jacobian_det(const Launch& L, CPlanes3<T> u, Dims d, T* det,
                         unsigned long long* nonpos);
template <class T>
void launch_eulerian(const Launch& L, CPlanes3<T> g, CPlanes3<T> u, Dims d, int use_jac,
                     Planes3<T> out);
template <class T>
void launch_adam(const Launch& L, Planes3<T> m, Planes3<T> nu, CPlanes3<T> v, Planes3<T> dir,
                 Dims d, double b1, double b2, double c1, double c2, double eps);
template <class T>
void launch_clamp_step(const Launch& L, CPlanes3<T> v, Planes3<T> step, Dims d, double eta,
                       double cap, int* bad);
template <class T>
void launch_resample(const Launch& L, const T* const* src, Dims ds, T* const* dst, Dims dd,
                     int ncomp, const double* mult);
template <class T>
void launch_affine_field(const Launch& L, const double* A, const double* t, const double* S,
                         Dims d, Planes3<T> out);
template <class T>
void launch_gauss_axis(const Launch& L, const T* in, T* out, Dims d, int axis, int R,
                       const double* taps, const double* norm, const LoopState* st = nullptr);
template <class T>
void launch_range_check(const Launch& L, const T* p, int64_t n, int* bad);

// -------- losses
// per-CTA partial sums (double) into `partials`; returns number of partials.
struct MonitorArgs;
template <class T>
int launch_ssd(const Launch& L, const T* F, const T* M, Dims d, Dims dm, CPlanes3<T> u,
               Planes3<T> grad, double* partials, const LoopState* st,
               const MonitorArgs* mon = nullptr);
template <class T>
int launch_dice_sums(const Launch& L, const T* F, const T* M, Dims d, Dims dm, CPlanes3<T> u,
                     double* partials, const LoopState* st);
template <class T>
void launch_dice_grad(const Launch& L, const T* F, const T* M, Dims d, Dims dm, CPlanes3<T> u,
                      Planes3<T> grad, const LoopState* st, double P, double D);
template <class T>
int launch_lncc_fwd(const Launch& L, int R, const T* F, const T* M, Dims d, Dims dm,
                    CPlanes3<T> u, T* const* coef, double* partials, const LoopState* st);
template <class T>
void launch_lncc_bwd(const Launch& L, int R, const T* F, const T* M, Dims d, Dims dm,
                     CPlanes3<T> u, const T* const* coef, Planes3<T> grad, const LoopState* st);

// -------- fused update kernels
struct AdamParams {
    double b1, b2, eps, eta, cap;
    const double* corr1;  // 1 - b1^t, indexed by t (host std::pow, optim.cpp:27-28)
    const double* corr2;
    int use_jac;
};
template <class T>
void launch_smooth_adam(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> grad,
                        CPlanes3<T> u, Planes3<T> m, Planes3<T> nu, Planes3<T> step, Dims d,
                        AdamParams ap, LoopState* st, unsigned long long* maxstep_slots);
template <class T>
void launch_compose_smooth(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> step,
                           CPlanes3<T> u_in, Planes3<T> u_out, Dims d, LoopState* st);
// plain fused Gaussian (gaussian_smooth / gaussian_smooth_field), ncomp 1..3
// SVF update v' = G * (v + step) on the TMA z-march (3-D; < 0: not eligible)
template <class T>
int launch_svf_update_tma(const Launch& L, int R, const GaussW<T>& w, const T* v, const T* step,
                          T* out, Dims d, LoopState* st);

// one-component Gaussian on the TMA z-march (3-D; < 0: not eligible)
template <class T>
int launch_gauss_tma(const Launch& L, int R, const GaussW<T>& w, const T* in, T* out, Dims d);

template <class T>
void launch_gauss_fused(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> in,
                        Planes3<T> out, int ncomp, Dims d);

// -------- plane-streaming (TMA) kernels, kernels_tma.cu.  Fields are passed as
// the base of their 3 (coef: 4) contiguous planes.  Launchers return < 0 when
// the shape/radius is not supported (caller falls back to the kernels above).
bool tma_supported(Dims d, int esz);
// With `mon` set, the last CTA to finish also reduces the partials (fixed
// order) and runs the convergence monitor: one launch instead of two.
struct MonitorArgs {
    LoopState* st;
    double* loss;
    unsigned long long* stamp;
    int window;
    double tol;
};
template <class T>
int launch_lncc_fwd_tma(const Launch& L, int R, const T* F, const T* W, Dims d, T* coef,
                        double* partials, const LoopState* st,
                        const MonitorArgs* mon = nullptr);
template <class T>
int launch_lncc_bwd_tma(const Launch& L, int R, const T* coef, const T* F, const T* W,
                        const T* G, Dims d, T* grad, const LoopState* st);
// per-level window statistics of F (fstat: 2 fp64 planes muF, vF), then the
// 3-moment forward that reads them — bit-identical to launch_lncc_fwd_tma
template <class T>
int launch_fstats_tma(const Launch& L, int R, const T* F, Dims d, double* fstat);
template <class T>
int launch_lncc_fwd3_tma(const Launch& L, int R, const T* F, const T* W, const double* fstat,
                         Dims d, T* coef, double* partials, const LoopState* st,
                         const MonitorArgs* mon = nullptr);
template <class T>
int launch_smooth_adam_tma(const Launch& L, int R, const GaussW<T>& w, const T* grad, T* m,
                           T* nu, T* step, Dims d, AdamParams ap, LoopState* st,
                           unsigned long long* maxstep, const T* ujac = nullptr);
template <class T>
int launch_compose_tma(const Launch& L, int R, double cap, const GaussW<T>& w, const T* step,
                       const T* uin, T* uout, const T* M, Dims dm, Dims d, T* W, T* G,
                       LoopState* st, bool count_update = true);
template <class T>
void launch_warpgrad(const Launch& L, const T* M, Dims dm, CPlanes3<T> u, Dims d, T* W, T* G);
// split update (3-D): smooth+Adam whose epilogue also composes, writing the
// composed field c = step + u(x+step) to `cout`; then the sigma_warp smoothing
// of c with the fused W/G gather.  Same values as launch_smooth_adam_tma +
// launch_compose_tma without recomposing halo elements.
template <class T>
int launch_smooth_adam_compose_tma(const Launch& L, int R, const GaussW<T>& w, const T* grad,
                                   T* m, T* nu, const T* uin, T* cout, double cap, Dims d,
                                   AdamParams ap, LoopState* st, unsigned long long* maxstep);
template <class T>
int launch_compose_pointwise(const Launch& L, const T* step, const T* u, double cap, Dims d,
                             T* c, const LoopState* st);
template <class T>
int launch_compose_smooth_tma(const Launch& L, int R, const GaussW<T>& w, const T* c, T* uout,
                              const T* M, Dims dm, Dims d, T* W, T* G, LoopState* st,
                              bool count_update = true);

// -------- brick kernels (kernels_brick.cu): 8x8x8 bricks, every pass in
// parallel; used on the small pyramid levels where the z-march is
// latency-bound.  Same contracts as the plane-streaming launchers; return < 0
// when the radius / precision combination is not instantiated.
constexpr int kBrickLnccRMax = 3, kBrickGaussRMax = 6, kBrickComposeRMax = 4;
bool brick_supported(Dims d, int esz, int lncc_r, int rg, int rw);
template <class T>
int launch_lncc_fwd_brick(const Launch& L, int R, const T* F, const T* W, Dims d, T* coef,
                          double* partials, const LoopState* st,
                          const MonitorArgs* mon = nullptr, const double* fstat = nullptr);
template <class T>
int launch_fstats_brick(const Launch& L, int R, const T* F, Dims d, double* fstat);
template <class T>
int launch_lncc_bwd_brick(const Launch& L, int R, const T* coef, const T* F, const T* W,
                          const T* G, Dims d, T* grad, const LoopState* st);
template <class T>
int launch_smooth_adam_brick(const Launch& L, int R, const GaussW<T>& w, const T* grad, T* m,
                             T* nu, T* step, Dims d, AdamParams ap, LoopState* st,
                             unsigned long long* maxstep);
template <class T>
int launch_compose_brick(const Launch& L, int R, const GaussW<T>& w, const T* step,
                         const T* uin, T* uout, const T* M, Dims dm, Dims d, T* W, T* G,
                         LoopState* st, bool count_update = true);

// brick forms of the split update (see launch_smooth_adam_compose_tma)
template <class T>
int launch_smooth_adam_compose_brick(const Launch& L, int R, const GaussW<T>& w, const T* grad,
                                     T* m, T* nu, const T* uin, T* cout, double cap, Dims d,
                                     AdamParams ap, LoopState* st, unsigned long long* maxstep);
template <class T>
int launch_compose_smooth_brick(const Launch& L, int R, const GaussW<T>& w, const T* c, T* uout,
                                const T* M, Dims dm, Dims d, T* W, T* G, LoopState* st,
                                bool count_update = true);

// Persistent scale solver (kernels_brick.cu): every iteration of one small
// LNCC pyramid level in ONE cooperative launch, grid barriers between the
// brick phases, device-side monitor.  u0 -> u1 on even iterations (ping-pong);
// on return LoopState holds it / t / nupdates / err like the graph path.
// Returns < 0 if the radius triple is not instantiated or co-residency fails.
template <class T>
struct PersistScale {
    Dims d;
    int lncc_r, rg, rw;
    const T* F;
    const T* M;
    T* W;
    T* G;
    T* coef;
    T* grad;
    T* m;
    T* nu;
    T* step;
    T* u0;
    T* u1;
    GaussW<T> wg, ww;
    AdamParams ap;
    LoopState* st;
    double* partials;
    double* loss;
    unsigned long long* stamp;
    unsigned long long* maxstep;
    int window;
    double tol;
    int iters;
    const double* fstat;  // neighbour-synchronised solver: the level's F statistics
    unsigned* sync;       // and its zeroed sync words (persist_nb_sync_words)
    bool nb_any_size;     // also levels with more bricks than CTA slots
};
template <class T>
int launch_persist_scale(const Launch& L, const PersistScale<T>& p);
template <class T>
int launch_persist_nb_scale(const Launch& L, const PersistScale<T>& p);
int persist_nb_sync_words(Dims d, int iters);

// -------- SVF mode (kernels_svf.cu): exp_map and the deterministic
// svf_pullback (stable-sorted gather in place of the reference's serial
// scatter).  Fields are packed 3-plane bases; levels = (M+1) packed fields.
template <class T>
struct SvfWork {
    T* wa;
    T* wb;              // 3n each: cotangent ping-pong
    int32_t* keys[2];   // 8n each
    int32_t* vals[2];   // 8n each
    int32_t* start;     // n+1
    T* wts;             // 8n: lerp weight of pair 8i+k (written with the keys)
    void* temp;
    size_t temp_bytes;  // >= svf_sort_temp_bytes(n)
};
size_t svf_sort_temp_bytes(int64_t n);
template <class T>
void launch_exp_map(const Launch& L, const T* v, Dims d, int M, T* levels,
                    const LoopState* st = nullptr);
template <class T>
void launch_svf_pullback(const Launch& L, const T* levels, Dims d, int M, const T* grad_phi,
                         T* out, const SvfWork<T>& ws, const LoopState* st = nullptr);
// SVF update (pipeline.cpp:199-205): out = G_sigma_warp * (v + step); skips
// when the scale is done, counts the update (kernels_stencil.cu)
template <class T>
void launch_svf_update(const Launch& L, int R, const GaussW<T>& w, CPlanes3<T> v,
                       CPlanes3<T> step, Planes3<T> out, Dims d, LoopState* st);

// -------- affine pre-alignment (kernels_affine.cu): the 12 parameter sums
// of affine_param_gradient; out12 = dA (row-major, ndim x ndim packed) then dt
// at [9..11]; partials needs affine_grad_partials() doubles.
struct AffineS {
    double S[3];
};
int affine_grad_partials();
template <class T>
void launch_affine_grad(const Launch& L, CPlanes3<T> g, Dims d, AffineS S, double* partials,
                        double* out12);

// -------- evaluation epilogue (kernels_eval.cu): label maxima and per-label
// counts (3 rows of maxl+1: |S_l|, |T_l|, |S_l n T_l|) for overlap_report
int launch_label_max(const Launch& L, const int32_t* a, const int32_t* b, int64_t n, int* out);
void launch_label_hist(const Launch& L, const int32_t* warped, const int32_t* fixed, int64_t n,
                       int maxl, unsigned long long* counts);

// -------- loop control
// kind: 0 ssd, 1 lncc, 2 dice (3 partial arrays of np each)
void launch_monitor(const Launch& L, int kind, const double* partials, int np, double nvox,
                    LoopState* st, double* loss, unsigned long long* stamp, int window,
                    double tol);
// value-only reduction (epilogue / per-call API): out = kind-specific value
void launch_reduce_value(const Launch& L, int kind, const double* partials, int np, double nvox,
                         double* out);
void launch_stamp(const Launch& L, unsigned long long* slot);
// copy src -> dst (ncomp planes of n) when (T_si - st->nupdates) is odd
template <class T>
void launch_parity_fix(const Launch& L, const LoopState* st, int T_si, CPlanes3<T> src,
                       Planes3<T> dst, int64_t n, int ncomp);

int zmarch_blocks(Dims d, int R, int num_sms, int* zchunk, int* tiles);

}  // namespace dfm
