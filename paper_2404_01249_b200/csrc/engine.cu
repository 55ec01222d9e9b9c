// engine.cu — the C-ABI (include/difform_gpu.h): context, staging, the
// per-function entry points and the device-resident register_images driver.
//
// Host side of the boundary: plain pointers in, status codes out.  Inside, a
// dfm_ctx owns a CUDA stream, a named workspace arena (grown on demand, reused
// across calls), two captured CUDA graphs per pyramid scale (ping-pong of the
// displacement buffers) and an event pool for optional per-kernel timing.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>
#include <cstddef>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/difform_gpu.h"
#include "dfm_device.cuh"
#include "dfm_kernels.cuh"

using namespace dfm;

namespace dfm {
// kernels_exact.cu: register_images with the reference's arithmetic (DFM_OPT_EXACT)
int exact_register_status(cudaStream_t stream, int64_t* launches, const dfm_grid* g,
                          const double* F, const double* M, const dfm_config* cfg,
                          const double* scales, const int32_t* iters, int ns,
                          const dfm_init* init, double* d_field_aos,
                          std::vector<dfm_iter_record>& recs, double* final_loss, double* sing,
                          std::string& msg);
}  // namespace dfm

namespace {


thread_local std::string g_err;

}  // namespace

// the thread's error message, for host modules built on the C-ABI (sweep.cu)
dfm_status dfm_internal_set_error(dfm_status code, const char* msg) {
    g_err = msg;
    return code;
}

namespace {

struct DfmError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw DfmError{code, buf};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(DFM_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(x) ck((x), #x)

template <class F>
dfm_status guarded(F&& fn) {
    try {
        fn();
        return DFM_OK;
    } catch (const DfmError& e) {
        g_err = e.msg;
        return static_cast<dfm_status>(e.code);
    } catch (const std::exception& e) {
        g_err = e.what();
        return DFM_E_CUDA;
    }
}

// NVTX ranges (SURVEY §5 tracing): registration, pyramid level, level loop,
// epilogue, slab level; header-only NVTX v3, inert unless a tool is attached
struct Nvtx {
    explicit Nvtx(const char* fmt, ...) {
        char buf[160];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        nvtxRangePushA(buf);
    }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

double now_ms() {
    using clk = std::chrono::steady_clock;
    return std::chrono::duration<double, std::milli>(clk::now().time_since_epoch()).count();
}

}  // namespace

// ---------------------------------------------------------------------------
// context

struct dfm_ctx {
    int device = 0;
    int prec = DFM_PREC_F32;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int64_t launches = 0;
    std::map<std::string, std::pair<void*, size_t>> bufs;
    bool profiling = false;
    bool force_legacy = getenv("DFM_FORCE_LEGACY") != nullptr;  // A/B the v1 kernels
    int tma_mask = getenv("DFM_TMA_MASK") ? atoi(getenv("DFM_TMA_MASK")) : 15;
    // pyramid levels up to this many voxels run the brick kernels
    int64_t brick_max = getenv("DFM_BRICK_MAX") ? atoll(getenv("DFM_BRICK_MAX")) : 200000;
    // brick levels of an LNCC registration run as one persistent launch per level
    // (1: grid barriers between phases, 2: neighbour-synchronised bricks where
    // that is faster (>= 2 bricks per SM, one CTA each), 3: at any size;
    // measured 35.0 -> 34.0 us per 40x48x56 iteration, config-1 pair -0.4 ms)
    int persist = getenv("DFM_PERSIST") ? atoi(getenv("DFM_PERSIST")) : 2;
    double kt_ms[DFM_NUM_KCLASS] = {};
    int64_t kt_n[DFM_NUM_KCLASS] = {};
    int64_t kt_vox[DFM_NUM_KCLASS] = {};

    LoopState* hstate = nullptr;  // 2 pinned slots for the chunked launch loop
    cudaEvent_t chunk_ev[2] = {nullptr, nullptr};

    bool pdl = getenv("DFM_PDL") ? atoi(getenv("DFM_PDL")) != 0 : false;
    // LNCC forward with per-level F statistics (3 fp64 moments per iteration)
    bool fwd3 = getenv("DFM_FWD3") ? atoi(getenv("DFM_FWD3")) != 0 : true;
    // split update: pointwise compose in the Adam epilogue + smoothing kernel
    bool split_compose = getenv("DFM_SPLIT") ? atoi(getenv("DFM_SPLIT")) != 0 : true;
    bool split3 = getenv("DFM_SPLIT3") ? atoi(getenv("DFM_SPLIT3")) != 0 : true;
    // levels below this size fold the compose into the Adam epilogue, larger
    // ones run it as its own radius-0 streaming kernel
    int64_t split_fold_max = getenv("DFM_SPLIT_FOLD_MAX") ? atoll(getenv("DFM_SPLIT_FOLD_MAX"))
                                                          : 2000000;
    // large-level kernel variants from this many voxels (DFM_OPT_LARGE_MIN)
    int64_t large_min = 2000000;
    // z-slab runs: pyramid levels up to this many voxels are replicated on every
    // rank instead of decomposed (DFM_OPT_SLAB_REPL_MAX)
    int64_t slab_repl_max = 4000000;
    // z-slab runs: overlap each stage's halo exchange with its interior planes
    // (-1 auto = multi-process NCCL only, 0 off, 1 on; DFM_OPT_SLAB_OVERLAP)
    int slab_overlap = -1;
    // register_images with the reference's arithmetic, bit-identical (fp64
    // contexts; DFM_OPT_EXACT)
    bool exact = false;
    // 16-wide z-march tiles on mid-size levels with a half-empty last x tile
    bool narrow = getenv("DFM_TMA_NARROW") ? atoi(getenv("DFM_TMA_NARROW")) != 0 : true;
    Launch L() {
        Launch l{stream, &launches, num_sms, pdl, large_min};
        l.narrow = narrow;
        return l;
    }

    LoopState* pinned_state() {
        if (!hstate) {
            CK(cudaMallocHost(&hstate, 2 * sizeof(LoopState)));
            for (int k = 0; k < 2; ++k)
                CK(cudaEventCreateWithFlags(&chunk_ev[k], cudaEventDisableTiming));
        }
        return hstate;
    }

    // per-(level, ping-pong variant) executable graphs kept across calls: a
    // re-capture is applied with cudaGraphExecUpdate (cheap) instead of a new
    // cudaGraphInstantiate (hundreds of us of host time the GPU waits for)
    // keyed by a signature of everything that shapes the captured kernels
    // (level dims, config, kernel family, options): an in-place update is only
    // attempted between captures of the same structure.  (An update from a
    // clustered plane-streaming launch of another level or config could
    // report success yet keep stale launch attributes.)
    std::map<uint64_t, cudaGraphExec_t> graph_cache;
    void trim_graphs() {  // bounded cache: a long sweep of shapes/configs (between levels)
        if (graph_cache.size() < 64) return;
        CK(cudaStreamSynchronize(stream));
        for (auto& kv : graph_cache) cudaGraphExecDestroy(kv.second);
        graph_cache.clear();
    }
    cudaGraphExec_t graph_exec(uint64_t key, cudaGraph_t graph) {
        auto it = graph_cache.find(key);
        if (it != graph_cache.end()) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(it->second, graph, &info) == cudaSuccess) return it->second;
            cudaGetLastError();  // topology changed: instantiate afresh
            CK(cudaGraphExecDestroy(it->second));
            graph_cache.erase(it);
        }
        cudaGraphExec_t e = nullptr;
        CK(cudaGraphInstantiate(&e, graph, 0));
        graph_cache[key] = e;
        return e;
    }

    std::map<std::string, std::pair<void*, size_t>> pinned;  // page-locked host staging
    void* get_pinned(const std::string& name, size_t bytes) {
        auto it = pinned.find(name);
        if (it != pinned.end() && it->second.second >= bytes) return it->second.first;
        if (it != pinned.end()) {
            CK(cudaStreamSynchronize(stream));
            CK(cudaFreeHost(it->second.first));
            pinned.erase(it);
        }
        void* p = nullptr;
        CK(cudaMallocHost(&p, bytes));
        pinned[name] = {p, bytes};
        return p;
    }

    // small host -> device uploads staged through pinned memory: from pageable
    // memory cudaMemcpyAsync first waits for the stream to drain, which would
    // stall the host (and then idle the GPU) at every pyramid level
    std::map<std::string, cudaEvent_t> up_ev;
    void upload(void* dev, const void* src, size_t bytes, const std::string& key) {
        auto it = up_ev.find(key);
        if (it == up_ev.end()) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            it = up_ev.emplace(key, e).first;
        } else {
            CK(cudaEventSynchronize(it->second));  // the previous copy out of it is done
        }
        void* h = get_pinned("@up:" + key, bytes);
        std::memcpy(h, src, bytes);
        CK(cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice, stream));
        CK(cudaEventRecord(it->second, stream));
    }

    void* get(const std::string& name, size_t bytes) {
        if (bytes == 0) bytes = 16;
        auto it = bufs.find(name);
        if (it != bufs.end() && it->second.second >= bytes) return it->second.first;
        if (it != bufs.end()) {
            CK(cudaStreamSynchronize(stream));
            CK(cudaFree(it->second.first));
            bufs.erase(it);
        }
        void* p = nullptr;
        CK(cudaMalloc(&p, bytes));
        bufs[name] = {p, bytes};
        return p;
    }
    template <class T>
    T* arr(const std::string& name, int64_t n) {
        return static_cast<T*>(get(name, sizeof(T) * static_cast<size_t>(n)));
    }
    void sync() { CK(cudaStreamSynchronize(stream)); }
    void check_launch() { CK(cudaGetLastError()); }
    // a second stream for copies that overlap the main stream's kernels (the
    // result download beside the registration epilogue)
    cudaStream_t side = nullptr;
    cudaEvent_t side_ev = nullptr;
    cudaStream_t side_stream() {
        if (!side) {
            CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&side_ev, cudaEventDisableTiming));
        }
        return side;
    }
};

namespace {

// ---------------------------------------------------------------------------
// validation (core.cpp:26-37 etc.)

void validate_grid(const dfm_grid* g) {
    if (!g) fail(DFM_E_INVALID, "grid is NULL");
    if (g->ndim != 2 && g->ndim != 3) fail(DFM_E_INVALID, "grid must have 2 or 3 axes");
    for (int a = 0; a < g->ndim; ++a) {
        if (g->dims[a] < 2) fail(DFM_E_INVALID, "grid dims must be >= 2 per axis");
        if (!(g->spacing[a] > 0.0) || !std::isfinite(g->spacing[a]))
            fail(DFM_E_INVALID, "grid spacing must be > 0");
    }
    if (g->ndim == 2 && g->dims[2] != 1) fail(DFM_E_INVALID, "2D grid must have dims[2] == 1");
    const double n = static_cast<double>(g->dims[0]) * g->dims[1] * g->dims[2];
    if (n >= 2147483647.0) fail(DFM_E_INVALID, "grid has more than 2^31-1 voxels");
}

Dims to_dims(const dfm_grid* g) {
    Dims d;
    d.nx = static_cast<int>(g->dims[0]);
    d.ny = static_cast<int>(g->dims[1]);
    d.nz = static_cast<int>(g->dims[2]);
    d.ndim = g->ndim;
    d.n = g->dims[0] * g->dims[1] * g->dims[2];
    return d;
}

bool same_grid(const dfm_grid* a, const dfm_grid* b) {
    return a->ndim == b->ndim && a->dims[0] == b->dims[0] && a->dims[1] == b->dims[1] &&
           a->dims[2] == b->dims[2];
}

bool dims_equal(const Dims& a, const Dims& b) {
    return a.nx == b.nx && a.ny == b.ny && a.nz == b.nz;
}

void downsample_grid(const dfm_grid* g, const double f[3], dfm_grid* out) {
    validate_grid(g);
    *out = *g;
    for (int a = 0; a < g->ndim; ++a) {
        if (!(f[a] >= 1.0)) fail(DFM_E_INVALID, "downsample factor must be >= 1");
        out->dims[a] = static_cast<int64_t>(std::ceil(static_cast<double>(g->dims[a]) / f[a]));
        if (out->dims[a] < 2) fail(DFM_E_INVALID, "downsample would leave < 2 samples on an axis");
        out->spacing[a] =
            g->spacing[a] * (static_cast<double>(g->dims[a]) / static_cast<double>(out->dims[a]));
    }
}

// ---------------------------------------------------------------------------
// Gaussian weights (interp.cpp:110-124)

struct HostGauss {
    int R = 0;                          // common radius over axes
    int Ra[3] = {0, 0, 0};
    std::vector<double> taps[3];        // 2*Ra+1 each, normalised
    std::vector<double> norm[3];        // 1 / in-range tap sum per position
};

HostGauss make_gauss(const Dims& d, const double sigma[3]) {
    HostGauss h;
    const int n[3] = {d.nx, d.ny, d.nz};
    for (int a = 0; a < 3; ++a) {
        const bool active = a < d.ndim && sigma[a] > 0.0 && n[a] > 1;
        const int R = active ? static_cast<int>(std::ceil(3.0 * sigma[a])) : 0;
        h.Ra[a] = R;
        h.taps[a].assign(2 * R + 1, 0.0);
        if (!active) {
            h.taps[a][0] = 1.0;
        } else {
            double s = 0.0;
            for (int j = -R; j <= R; ++j) {
                const double q = static_cast<double>(j) / sigma[a];
                h.taps[a][j + R] = std::exp(-0.5 * q * q);
                s += h.taps[a][j + R];
            }
            for (double& t : h.taps[a]) t /= s;
        }
        h.norm[a].assign(n[a], 1.0);
        if (active)
            for (int i = 0; i < n[a]; ++i) {
                const int jlo = -R > -i ? -R : -i;
                const int jhi = R < n[a] - 1 - i ? R : n[a] - 1 - i;
                double ws = 0.0;
                for (int j = jlo; j <= jhi; ++j) ws += h.taps[a][j + R];
                h.norm[a][i] = 1.0 / ws;
            }
        if (R > h.R) h.R = R;
    }
    return h;
}

template <class T>
GaussW<T> upload_gauss(dfm_ctx* ctx, const HostGauss& h, const Dims& d, const std::string& key) {
    GaussW<T> w{};
    const int n[3] = {d.nx, d.ny, d.nz};
    std::vector<T> host(static_cast<size_t>(n[0] + n[1] + n[2]));
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
        for (int j = 0; j < 2 * kRMax + 1; ++j) w.taps[a][j] = T(0);
        // center the axis taps inside the common radius
        if (h.R <= kRMax)
            for (int j = -h.Ra[a]; j <= h.Ra[a]; ++j)
                w.taps[a][j + h.R] = static_cast<T>(h.taps[a][j + h.Ra[a]]);
        for (int i = 0; i < n[a]; ++i) host[off + i] = static_cast<T>(h.norm[a][i]);
        off += n[a];
        // the interior entry of make_gauss (same summation order)
        double ws = 0.0;
        for (int j = 0; j < 2 * h.Ra[a] + 1; ++j) ws += h.taps[a][j];
        const bool active = h.Ra[a] > 0;
        w.norm_int[a] = static_cast<T>(active ? 1.0 / ws : 1.0);
        w.ra[a] = h.Ra[a];
    }
    T* dev = ctx->arr<T>("gauss_norm_" + key, static_cast<int64_t>(host.size()));
    ctx->upload(dev, host.data(), host.size() * sizeof(T), "gauss_norm_" + key);
    w.norm[0] = dev;
    w.norm[1] = dev + n[0];
    w.norm[2] = dev + n[0] + n[1];
    return w;
}

// per-axis generic path for radii above kRMax (pyramid pre-blur, large sigma)
struct DevAxisGauss {
    int Ra[3];
    const double* taps[3];
    const double* norm[3];
};

DevAxisGauss upload_axis_gauss(dfm_ctx* ctx, const HostGauss& h, const Dims& d,
                               const std::string& key) {
    DevAxisGauss g{};
    const int n[3] = {d.nx, d.ny, d.nz};
    std::vector<double> host;
    size_t offs[6];
    for (int a = 0; a < 3; ++a) {
        offs[2 * a] = host.size();
        host.insert(host.end(), h.taps[a].begin(), h.taps[a].end());
        offs[2 * a + 1] = host.size();
        host.insert(host.end(), h.norm[a].begin(), h.norm[a].end());
    }
    double* dev = ctx->arr<double>("axis_gauss_" + key, static_cast<int64_t>(host.size()));
    ctx->upload(dev, host.data(), host.size() * sizeof(double), "axis_gauss_" + key);
    for (int a = 0; a < 3; ++a) {
        g.Ra[a] = h.Ra[a];
        g.taps[a] = dev + offs[2 * a];
        g.norm[a] = dev + offs[2 * a + 1];
    }
    (void)n;
    return g;
}

// Gaussian of one plane through the generic per-axis kernel: src -> dst,
// `tmp` as the ping-pong partner; dst may equal src.
template <class T>
void axis_smooth_plane(dfm_ctx* ctx, const Dims& d, const DevAxisGauss& g, const T* src, T* dst,
                       T* tmp, const LoopState* st) {
    Launch L = ctx->L();
    const T* s = src;
    for (int a = 0; a < 3; ++a) {
        if (g.Ra[a] == 0) continue;
        T* o = (s == dst) ? tmp : dst;
        launch_gauss_axis<T>(L, s, o, d, a, g.Ra[a], g.taps[a], g.norm[a], st);
        s = o;
    }
    if (s != dst)
        CK(cudaMemcpyAsync(dst, s, sizeof(T) * d.n, cudaMemcpyDeviceToDevice, ctx->stream));
}

// smooth `ncomp` planes in -> out (fused z-march when the radius allows)
template <class T>
void smooth_planes(dfm_ctx* ctx, const Dims& d, const double sigma[3], CPlanes3<T> in,
                   Planes3<T> out, int ncomp, const std::string& key) {
    const HostGauss h = make_gauss(d, sigma);
    if (h.R <= kRMax) {
        const GaussW<T> w = upload_gauss<T>(ctx, h, d, key);
        launch_gauss_fused<T>(ctx->L(), h.R, w, in, out, ncomp, d);
        return;
    }
    const DevAxisGauss g = upload_axis_gauss(ctx, h, d, key);
    T* tmp = ctx->arr<T>("smooth_tmp_" + key, d.n);
    for (int c = 0; c < ncomp; ++c) axis_smooth_plane<T>(ctx, d, g, in.c[c], out.c[c], tmp, nullptr);
}

// ---------------------------------------------------------------------------
// staging helpers (host AoS doubles <-> device SoA T)

template <class T>
struct Field {
    T* p[3];
    Planes3<T> w() const { return {{p[0], p[1], p[2]}}; }
    CPlanes3<T> r() const { return {{p[0], p[1], p[2]}}; }
};

template <class T>
Field<T> dev_field(dfm_ctx* ctx, const std::string& name, int64_t n) {
    T* base = ctx->arr<T>(name, 3 * n);
    return Field<T>{{base, base + n, base + 2 * n}};
}

template <class T, class S>
void upload_image(dfm_ctx* ctx, const S* host, int64_t n, T* dst) {
    if (std::is_same<T, S>::value) {
        CK(cudaMemcpyAsync(dst, host, sizeof(S) * n, cudaMemcpyHostToDevice, ctx->stream));
        return;
    }
    S* stage = ctx->arr<S>(std::is_same<S, double>::value ? "stage_d" : "stage_f", n);
    CK(cudaMemcpyAsync(stage, host, sizeof(S) * n, cudaMemcpyHostToDevice, ctx->stream));
    launch_cast<T, S>(ctx->L(), stage, dst, n);
}

template <class T>
void upload_field(dfm_ctx* ctx, const double* host, int64_t n, int nd, const Field<T>& dst) {
    double* stage = ctx->arr<double>("stage_d", n * nd);
    CK(cudaMemcpyAsync(stage, host, sizeof(double) * n * nd, cudaMemcpyHostToDevice,
                       ctx->stream));
    launch_aos_to_soa<T, double>(ctx->L(), stage, dst.w(), n, nd);
}

template <class T, class S>
void download_image(dfm_ctx* ctx, const T* src, int64_t n, S* host) {
    if (std::is_same<T, S>::value) {
        CK(cudaMemcpyAsync(host, src, sizeof(S) * n, cudaMemcpyDeviceToHost, ctx->stream));
        return;
    }
    S* stage = ctx->arr<S>(std::is_same<S, double>::value ? "stage_d" : "stage_f", n);
    launch_cast<S, T>(ctx->L(), src, stage, n);
    CK(cudaMemcpyAsync(host, stage, sizeof(S) * n, cudaMemcpyDeviceToHost, ctx->stream));
}

template <class T, class S>
void download_field(dfm_ctx* ctx, CPlanes3<T> src, int64_t n, int nd, S* host) {
    S* stage = ctx->arr<S>(std::is_same<S, double>::value ? "stage_d" : "stage_f", n * nd);
    launch_soa_to_aos<T, S>(ctx->L(), src, stage, n, nd);
    CK(cudaMemcpyAsync(host, stage, sizeof(S) * n * nd, cudaMemcpyDeviceToHost, ctx->stream));
}

// ---------------------------------------------------------------------------
// per-function implementations (templated on the device precision)

template <class T>
struct Impl {
    dfm_ctx* ctx;

    void downsample_dev(const Dims& d, const T* img, const double f[3], const Dims& od,
                        T* out, const std::string& key) {
        // core.cpp:66-95: sigma = f/2 pre-blur on axes with f > 1, then the
        // corner-aligned resample; factor 1 everywhere -> bit copy.
        double sigma[3] = {0.0, 0.0, 0.0};
        bool blur = false;
        for (int a = 0; a < d.ndim; ++a)
            if (f[a] > 1.0) {
                sigma[a] = f[a] / 2.0;
                blur = true;
            }
        Launch L = ctx->L();
        if (dims_equal(d, od) && !blur) {
            CK(cudaMemcpyAsync(out, img, sizeof(T) * d.n, cudaMemcpyDeviceToDevice, ctx->stream));
            return;
        }
        const T* src = img;
        if (blur && make_gauss(d, sigma).R <= kRMax) {
            // one fused 3-axis pass (z-march, x/y in shared memory, z in registers)
            const HostGauss h = make_gauss(d, sigma);
            const GaussW<T> w = upload_gauss<T>(ctx, h, d, "down_" + key);
            T* b0 = ctx->arr<T>("down_tmp0", d.n);
            if (h.R < 1 || launch_gauss_tma<T>(L, h.R, w, img, b0, d) < 0)
                launch_gauss_fused<T>(L, h.R, w, CPlanes3<T>{{img, nullptr, nullptr}},
                                      Planes3<T>{{b0, nullptr, nullptr}}, 1, d);
            src = b0;
        } else if (blur) {
            const HostGauss h = make_gauss(d, sigma);
            const DevAxisGauss g = upload_axis_gauss(ctx, h, d, "down_" + key);
            T* b0 = ctx->arr<T>("down_tmp0", d.n);
            T* b1 = ctx->arr<T>("down_tmp1", d.n);
            T* bufs[2] = {b0, b1};
            int k = 0;
            for (int a = 0; a < d.ndim; ++a) {
                if (h.Ra[a] == 0) continue;
                launch_gauss_axis<T>(L, src, bufs[k], d, a, h.Ra[a], g.taps[a], g.norm[a]);
                src = bufs[k];
                k ^= 1;
            }
        }
        const T* s1[1] = {src};
        T* d1[1] = {out};
        launch_resample<T>(L, s1, d, d1, od, 1, nullptr);
    }
};

template <class T>
int loss_kind_launch_fwd(dfm_ctx* ctx, int loss, int R, const T* F, const T* M, const Dims& d,
                         const Dims& dm, CPlanes3<T> u, T* const* coef, Planes3<T> grad,
                         double* partials, const LoopState* st) {
    Launch L = ctx->L();
    if (loss == DFM_LOSS_SSD) return launch_ssd<T>(L, F, M, d, dm, u, grad, partials, st);
    if (loss == DFM_LOSS_DICE) return launch_dice_sums<T>(L, F, M, d, dm, u, partials, st);
    return launch_lncc_fwd<T>(L, R, F, M, d, dm, u, coef, partials, st);
}

int monitor_kind(int loss) { return loss == DFM_LOSS_SSD ? 0 : (loss == DFM_LOSS_LNCC ? 1 : 2); }

// one loss evaluation outside the loop (API lncc_eval / ssd_eval / dice, final loss)
template <class T>
double eval_loss_dev(dfm_ctx* ctx, int loss, int R, const T* F, const T* M, const Dims& d,
                     const Dims& dm, CPlanes3<T> u, bool want_grad, Planes3<T> grad) {
    Launch L = ctx->L();
    double* partials = ctx->arr<double>("partials", 1 << 17);
    double* val = ctx->arr<double>("value3", 4);
    if (loss == DFM_LOSS_LNCC && want_grad && R <= 5 && tma_supported(d, sizeof(T))) {
        // plane-streaming path (the one the registration loop runs):
        // W, G = M(x+u), grad M(x+u); TMA-fed box passes.  grad planes contiguous.
        T* W = ctx->arr<T>("api_W", d.n);
        T* G = ctx->arr<T>("api_G", 3 * d.n);
        T* cb = ctx->arr<T>("coef", 4 * d.n);
        launch_warpgrad<T>(L, M, dm, u, d, W, G);
        const int np = launch_lncc_fwd_tma<T>(L, R, F, W, d, cb, partials, nullptr);
        if (np > 0) {
            launch_reduce_value(L, 1, partials, np, static_cast<double>(d.n), val);
            if (launch_lncc_bwd_tma<T>(L, R, cb, F, W, G, d, grad.c[0], nullptr) < 0)
                fail(DFM_E_CUDA, "lncc_bwd_tma launch failed");
            double hv[3];
            CK(cudaMemcpyAsync(hv, val, sizeof(hv), cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            return hv[0];
        }
    }
    T* coef[4] = {nullptr, nullptr, nullptr, nullptr};
    if (loss == DFM_LOSS_LNCC && want_grad) {
        T* cb = ctx->arr<T>("coef", 4 * d.n);
        for (int k = 0; k < 4; ++k) coef[k] = cb + k * d.n;
    }
    Planes3<T> g = want_grad ? grad : Planes3<T>{{nullptr, nullptr, nullptr}};
    const int np =
        loss_kind_launch_fwd<T>(ctx, loss, R, F, M, d, dm, u, coef, g, partials, nullptr);
    launch_reduce_value(L, monitor_kind(loss), partials, np, static_cast<double>(d.n), val);
    double hv[3];
    CK(cudaMemcpyAsync(hv, val, sizeof(hv), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (want_grad) {
        if (loss == DFM_LOSS_LNCC) {
            const T* cc[4] = {coef[0], coef[1], coef[2], coef[3]};
            launch_lncc_bwd<T>(L, R, F, M, d, dm, u, cc, grad, nullptr);
        } else if (loss == DFM_LOSS_DICE) {
            launch_dice_grad<T>(L, F, M, d, dm, u, grad, nullptr, hv[1], hv[2]);
        }
    }
    return hv[0];
}

}  // namespace

// ===========================================================================
// C-ABI

extern "C" {

int dfm_abi_version(void) { return DFM_ABI_VERSION; }

void dfm_config_defaults(dfm_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->loss = DFM_LOSS_SSD;
    c->lncc_radius = 2;
    c->eta = 0.5;
    c->sigma_grad = 1.0;
    c->sigma_warp = 0.5;
    c->use_jac = 0;
    c->mode = DFM_MODE_DIRECT;
    c->svf_M = 6;
    c->beta1 = 0.9;
    c->beta2 = 0.999;
    c->eps_adam = 1e-8;
    c->step_cap = 0.5;
    c->conv_window = 10;
    c->conv_tol = 1e-5;
    c->seed = 0;
}

size_t dfm_last_error(char* buf, size_t cap) {
    if (buf && cap) {
        const size_t n = g_err.size() < cap - 1 ? g_err.size() : cap - 1;
        std::memcpy(buf, g_err.data(), n);
        buf[n] = 0;
    }
    return g_err.size();
}

dfm_status dfm_ctx_create(int device, int precision, dfm_ctx** out) {
    return guarded([&] {
        if (!out) fail(DFM_E_INVALID, "out is NULL");
        if (precision != DFM_PREC_F32 && precision != DFM_PREC_F64)
            fail(DFM_E_INVALID, "precision must be DFM_PREC_F32 or DFM_PREC_F64");
        int count = 0;
        CK(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(DFM_E_INVALID, "no CUDA device %d", device);
        CK(cudaSetDevice(device));
        auto* c = new dfm_ctx();
        c->device = device;
        c->prec = precision;
        // fp64: the folded compose's carried gather spills (128 registers);
        // the split update is faster there at every size (152.6 vs 169.5 us
        // per iteration on 80x96x112)
        if (precision == DFM_PREC_F64 && !getenv("DFM_SPLIT_FOLD_MAX")) c->split_fold_max = 0;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        *out = c;
    });
}

void dfm_ctx_destroy(dfm_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->bufs) cudaFree(kv.second.first);
    for (auto& kv : ctx->up_ev) cudaEventDestroy(kv.second);
    for (auto& kv : ctx->pinned) cudaFreeHost(kv.second.first);
    for (auto& kv : ctx->graph_cache) cudaGraphExecDestroy(kv.second);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
        cudaEventDestroy(ctx->side_ev);
    }
    if (ctx->hstate) cudaFreeHost(ctx->hstate);
    for (int k = 0; k < 2; ++k)
        if (ctx->chunk_ev[k]) cudaEventDestroy(ctx->chunk_ev[k]);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int dfm_ctx_precision(const dfm_ctx* ctx) { return ctx ? ctx->prec : -1; }
void* dfm_ctx_stream(dfm_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int64_t dfm_ctx_launch_count(const dfm_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"

// context plumbing for host modules (mhd_io.cu): precision + stream, named
// device ("name") or pinned host ("@pinned:name") buffers, launch counting
dfm_status dfm_internal_ctx_info(dfm_ctx* ctx, int* precision, cudaStream_t* stream) {
    if (!ctx) return DFM_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    *precision = ctx->prec;
    *stream = ctx->stream;
    return DFM_OK;
}
void* dfm_internal_ctx_buffer(dfm_ctx* ctx, const char* name, size_t bytes) {
    const std::string n(name);
    if (n.rfind("@pinned:", 0) == 0) return ctx->get_pinned(n, bytes);
    return ctx->get(n, bytes);
}
void dfm_internal_bump(dfm_ctx* ctx) { ++ctx->launches; }

extern "C" {

dfm_status dfm_ctx_set_profiling(dfm_ctx* ctx, int enable) {
    return guarded([&] {
        if (!ctx) fail(DFM_E_INVALID, "ctx is NULL");
        ctx->profiling = enable != 0;
    });
}

dfm_status dfm_ctx_set_option(dfm_ctx* ctx, int key, int64_t value) {
    return guarded([&] {
        if (!ctx) fail(DFM_E_INVALID, "ctx is NULL");
        if (key == DFM_OPT_BRICK_MAX) {
            if (value < 0) fail(DFM_E_INVALID, "brick_max must be >= 0");
            ctx->brick_max = value;
        } else if (key == DFM_OPT_FORCE_LEGACY) {
            ctx->force_legacy = value != 0;
        } else if (key == DFM_OPT_PERSIST) {
            if (value < 0 || value > 3) fail(DFM_E_INVALID, "persist must be 0..3");
            ctx->persist = static_cast<int>(value);
        } else if (key == DFM_OPT_PDL) {
            ctx->pdl = value != 0;
        } else if (key == DFM_OPT_SPLIT) {
            ctx->split_compose = value != 0;
        } else if (key == DFM_OPT_SPLIT_FOLD_MAX) {
            if (value < 0) fail(DFM_E_INVALID, "split_fold_max must be >= 0");
            ctx->split_fold_max = value;
        } else if (key == DFM_OPT_NARROW) {
            ctx->narrow = value != 0;
        } else if (key == DFM_OPT_EXACT) {
            if (value && ctx->prec != DFM_PREC_F64)
                fail(DFM_E_INVALID, "exact mode needs an fp64 context");
            ctx->exact = value != 0;
        } else if (key == DFM_OPT_SLAB_OVERLAP) {
            if (value < -1 || value > 1) fail(DFM_E_INVALID, "slab_overlap must be -1, 0 or 1");
            ctx->slab_overlap = static_cast<int>(value);
        } else if (key == DFM_OPT_SLAB_REPL_MAX) {
            if (value < 0) fail(DFM_E_INVALID, "slab_repl_max must be >= 0");
            ctx->slab_repl_max = value;
        } else if (key == DFM_OPT_LARGE_MIN) {
            if (value < 0) fail(DFM_E_INVALID, "large_min must be >= 0");
            ctx->large_min = value;
        } else {
            fail(DFM_E_INVALID, "unknown context option %d", key);
        }
    });
}

dfm_status dfm_ctx_debug_read(dfm_ctx* ctx, const char* name, size_t offset, size_t bytes,
                              void* host) {
    return guarded([&] {
        if (!ctx || !name || (!host && bytes)) fail(DFM_E_INVALID, "NULL argument");
        auto it = ctx->bufs.find(name);
        if (it == ctx->bufs.end()) fail(DFM_E_INVALID, "no workspace buffer '%s'", name);
        if (offset + bytes > it->second.second)
            fail(DFM_E_INVALID, "workspace buffer '%s' holds %zu bytes", name, it->second.second);
        CK(cudaSetDevice(ctx->device));
        ctx->sync();
        CK(cudaMemcpy(host, static_cast<char*>(it->second.first) + offset, bytes,
                      cudaMemcpyDeviceToHost));
    });
}

dfm_status dfm_ctx_kernel_times(const dfm_ctx* ctx, double* ms, int64_t* launches,
                                int64_t* voxels) {
    return guarded([&] {
        if (!ctx) fail(DFM_E_INVALID, "ctx is NULL");
        for (int k = 0; k < DFM_NUM_KCLASS; ++k) {
            if (ms) ms[k] = ctx->kt_ms[k];
            if (launches) launches[k] = ctx->kt_n[k];
            if (voxels) voxels[k] = ctx->kt_vox[k];
        }
    });
}

dfm_status dfm_validate_grid(const dfm_grid* g) {
    return guarded([&] { validate_grid(g); });
}

dfm_status dfm_validate_config(const dfm_config* c);
dfm_status dfm_validate_schedule(const double* scales, const int32_t* iterations,
                                 int32_t nscales);

dfm_status dfm_downsample_grid(const dfm_grid* g, const double factor[3], dfm_grid* out) {
    return guarded([&] { downsample_grid(g, factor, out); });
}

}  // extern "C"

// dispatch on the context precision
#define DFM_DISPATCH(ctx, ...)                               \
    do {                                                     \
        if (!(ctx)) fail(DFM_E_INVALID, "ctx is NULL");      \
        CK(cudaSetDevice((ctx)->device));                    \
        if ((ctx)->prec == DFM_PREC_F64) {                   \
            using T = double;                                \
            __VA_ARGS__;                                     \
        } else {                                             \
            using T = float;                                 \
            __VA_ARGS__;                                     \
        }                                                    \
        (ctx)->check_launch();                               \
    } while (0)

extern "C" {

dfm_status dfm_downsample_image(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                                const double factor[3], dfm_grid* out_grid, double* out) {
    return guarded([&] {
        dfm_grid og;
        downsample_grid(g, factor, &og);
        const Dims d = to_dims(g), od = to_dims(&og);
        DFM_DISPATCH(ctx, {
            T* in = ctx->arr<T>("api_img0", d.n);
            T* o = ctx->arr<T>("api_img1", od.n);
            upload_image<T, double>(ctx, img, d.n, in);
            Impl<T>{ctx}.downsample_dev(d, in, factor, od, o, "api");
            download_image<T, double>(ctx, o, od.n, out);
            ctx->sync();
        });
        *out_grid = og;
    });
}

dfm_status dfm_sample_linear_points(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                                    int64_t npts, const double* points, double* values,
                                    double* grads) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            T* im = ctx->arr<T>("api_img0", d.n);
            upload_image<T, double>(ctx, img, d.n, im);
            double* pts = ctx->arr<double>("api_pts", 3 * npts + 1);
            double* vals = ctx->arr<double>("api_vals", npts + 1);
            double* grs = ctx->arr<double>("api_grads", 3 * npts + 1);
            if (npts > 0) {
                CK(cudaMemcpyAsync(pts, points, sizeof(double) * 3 * npts, cudaMemcpyHostToDevice,
                                   ctx->stream));
                launch_sample_points<T>(ctx->L(), im, d, pts, npts, vals, grads ? grs : nullptr);
                CK(cudaMemcpyAsync(values, vals, sizeof(double) * npts, cudaMemcpyDeviceToHost,
                                   ctx->stream));
                if (grads)
                    CK(cudaMemcpyAsync(grads, grs, sizeof(double) * 3 * npts,
                                       cudaMemcpyDeviceToHost, ctx->stream));
            }
            ctx->sync();
        });
    });
}

dfm_status dfm_warp_image(dfm_ctx* ctx, const dfm_grid* g, const double* img, const double* phi,
                          double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            T* im = ctx->arr<T>("api_img0", d.n);
            T* o = ctx->arr<T>("api_img1", d.n);
            Field<T> u = dev_field<T>(ctx, "api_f0", d.n);
            upload_image<T, double>(ctx, img, d.n, im);
            upload_field<T>(ctx, phi, d.n, d.ndim, u);
            launch_warp_image<T>(ctx->L(), im, d, u.r(), d, o);
            download_image<T, double>(ctx, o, d.n, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_warp_labels(dfm_ctx* ctx, const dfm_grid* g, const int32_t* labels,
                           const double* phi, int32_t* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            int32_t* lab = ctx->arr<int32_t>("api_lab0", d.n);
            int32_t* o = ctx->arr<int32_t>("api_lab1", d.n);
            Field<T> u = dev_field<T>(ctx, "api_f0", d.n);
            CK(cudaMemcpyAsync(lab, labels, sizeof(int32_t) * d.n, cudaMemcpyHostToDevice,
                               ctx->stream));
            upload_field<T>(ctx, phi, d.n, d.ndim, u);
            launch_warp_labels<T>(ctx->L(), lab, u.r(), d, o);
            CK(cudaMemcpyAsync(out, o, sizeof(int32_t) * d.n, cudaMemcpyDeviceToHost,
                               ctx->stream));
            ctx->sync();
        });
    });
}

dfm_status dfm_compose(dfm_ctx* ctx, const dfm_grid* g, const double* phi, const double* psi,
                       double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> b = dev_field<T>(ctx, "api_f1", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f2", d.n);
            upload_field<T>(ctx, phi, d.n, d.ndim, a);
            upload_field<T>(ctx, psi, d.n, d.ndim, b);
            launch_compose<T>(ctx->L(), a.r(), b.r(), d, o.w());
            download_field<T, double>(ctx, o.r(), d.n, d.ndim, out);
            ctx->sync();
        });
    });
}

// ---------------------------------------------------------------------------
// affine pre-alignment (affine.cpp:50-183)

}  // extern "C"

static void check_lncc_window(int loss, int R, const Dims& d) {
    if (loss != DFM_LOSS_LNCC) return;
    if (R < 1) fail(DFM_E_INVALID, "lncc_eval: window_radius must be >= 1");
    const int n[3] = {d.nx, d.ny, d.nz};
    for (int a = 0; a < d.ndim; ++a)
        if (2 * static_cast<int64_t>(R) + 1 > n[a])
            fail(DFM_E_INVALID, "lncc_eval: window larger than image");
    if (R > kRMax) fail(DFM_E_INVALID, "lncc_eval: window_radius > %d unsupported", kRMax);
}

static void check_dice_masks(int loss, const double* fixed, const double* moving, int64_t n) {
    if (loss != DFM_LOSS_DICE) return;
    for (int64_t i = 0; i < n; ++i)
        if (!(fixed[i] >= 0.0 && fixed[i] <= 1.0))
            fail(DFM_E_INVALID, "dice_soft_eval: fixed mask values outside [0,1]");
    for (int64_t i = 0; i < n; ++i)
        if (!(moving[i] >= 0.0 && moving[i] <= 1.0))
            fail(DFM_E_INVALID, "dice_soft_eval: moving mask values outside [0,1]");
}

// affine.cpp:95-122 on device images of grid d: value, dA (packed), dt
template <class T>
static double affine_grad_dev(dfm_ctx* ctx, int loss, int R, const T* F, const T* M,
                              const Dims& d, const double A[9], const double t[3],
                              const double S[3], double dA[9], double dt[3]) {
    Launch L = ctx->L();
    Field<T> u = dev_field<T>(ctx, "aff_u", d.n);
    Field<T> gr = dev_field<T>(ctx, "aff_g", d.n);
    launch_affine_field<T>(L, A, t, S, d, u.w());
    const double value = eval_loss_dev<T>(ctx, loss, R, F, M, d, d, u.r(), true, gr.w());
    double* part = ctx->arr<double>("aff_partials", affine_grad_partials());
    double* out = ctx->arr<double>("aff_out", 12);
    AffineS s;
    for (int a = 0; a < 3; ++a) s.S[a] = S[a];
    launch_affine_grad<T>(L, gr.r(), d, s, part, out);
    double h[12];
    CK(cudaMemcpyAsync(h, out, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int k = 0; k < 9; ++k) dA[k] = 0.0;
    for (int k = 0; k < d.ndim * d.ndim; ++k) dA[k] = h[k];
    for (int k = 0; k < 3; ++k) dt[k] = k < d.ndim ? h[9 + k] : 0.0;
    return value;
}

extern "C" {

dfm_status dfm_affine_to_field(dfm_ctx* ctx, const dfm_grid* g, const double A[9],
                               const double t[3], double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        const double S[3] = {1.0, 1.0, 1.0};
        DFM_DISPATCH(ctx, {
            Field<T> o = dev_field<T>(ctx, "api_f2", d.n);
            launch_affine_field<T>(ctx->L(), A, t, S, d, o.w());
            download_field<T, double>(ctx, o.r(), d.n, d.ndim, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_affine_param_gradient(dfm_ctx* ctx, const dfm_grid* g, const double* fixed,
                                     const double* moving, int loss, const double A[9],
                                     const double t[3], const double S[3], int lncc_radius,
                                     double* value, double dA[9], double dt[3]) {
    return guarded([&] {
        validate_grid(g);
        if (loss < 0 || loss > 2) fail(DFM_E_INVALID, "unknown loss");
        const Dims d = to_dims(g);
        check_lncc_window(loss, lncc_radius, d);
        check_dice_masks(loss, fixed, moving, d.n);
        DFM_DISPATCH(ctx, {
            T* F = ctx->arr<T>("api_img0", d.n);
            T* M = ctx->arr<T>("api_img1", d.n);
            upload_image<T, double>(ctx, fixed, d.n, F);
            upload_image<T, double>(ctx, moving, d.n, M);
            *value = affine_grad_dev<T>(ctx, loss, lncc_radius, F, M, d, A, t, S, dA, dt);
        });
    });
}

dfm_status dfm_affine_register(dfm_ctx* ctx, const dfm_grid* g, const double* fixed,
                               const double* moving, int loss, const double* scales,
                               const int32_t* iters, int32_t nscales, double eta,
                               int lncc_radius, dfm_affine_result* out) {
    return guarded([&] {
        validate_grid(g);
        if (nscales < 1 || !scales || !iters) fail(DFM_E_INVALID, "affine_register: bad schedule");
        if (loss < 0 || loss > 2) fail(DFM_E_INVALID, "unknown loss");
        const Dims full = to_dims(g);
        const int nd = g->ndim, np = nd * nd + nd;
        check_dice_masks(loss, fixed, moving, full.n);
        DFM_DISPATCH(ctx, {
            T* F = ctx->arr<T>("aff_F", full.n);
            T* M = ctx->arr<T>("aff_M", full.n);
            T* Fw = ctx->arr<T>("aff_Fw", full.n);
            T* Mw = ctx->arr<T>("aff_Mw", full.n);
            upload_image<T, double>(ctx, fixed, full.n, F);
            upload_image<T, double>(ctx, moving, full.n, M);
            double A[9] = {0}, t[3] = {0}, bA[9], bt[3];
            for (int i = 0; i < nd; ++i) A[i * nd + i] = 1.0;
            std::memcpy(bA, A, sizeof(A));
            std::memcpy(bt, t, sizeof(t));
            double best = std::numeric_limits<double>::infinity();
            double am[12] = {0}, anu[12] = {0};
            int64_t ta = 0, total = 0;
            const double b1 = 0.9, b2 = 0.999, eps = 1e-8;  // affine.cpp:139
            bool diverged = false;
            for (int si = 0; si < nscales && !diverged; ++si) {
                const double fac[3] = {scales[si], scales[si], scales[si]};
                dfm_grid wgd;
                downsample_grid(g, fac, &wgd);
                const Dims d = to_dims(&wgd);
                check_lncc_window(loss, lncc_radius, d);
                Impl<T>{ctx}.downsample_dev(full, F, fac, d, Fw, "aff_pyr");
                Impl<T>{ctx}.downsample_dev(full, M, fac, d, Mw, "aff_pyr");
                double S[3] = {1.0, 1.0, 1.0};
                const int fd[3] = {full.nx, full.ny, full.nz}, wd[3] = {d.nx, d.ny, d.nz};
                for (int a = 0; a < nd; ++a)
                    S[a] = static_cast<double>(fd[a] - 1) / static_cast<double>(wd[a] - 1);
                for (int it = 0; it < iters[si]; ++it) {
                    double dA[9], dt[3];
                    const double value =
                        affine_grad_dev<T>(ctx, loss, lncc_radius, Fw, Mw, d, A, t, S, dA, dt);
                    ++total;
                    if (!std::isfinite(value)) {
                        diverged = true;
                        break;
                    }
                    if (value < best) {
                        best = value;
                        std::memcpy(bA, A, sizeof(A));
                        std::memcpy(bt, t, sizeof(t));
                    }
                    ++ta;
                    const double c1 = 1.0 - std::pow(b1, static_cast<double>(ta));
                    const double c2 = 1.0 - std::pow(b2, static_cast<double>(ta));
                    for (int p = 0; p < np; ++p) {
                        const double gp = p < nd * nd ? dA[p] : dt[p - nd * nd];
                        am[p] = b1 * am[p] + (1.0 - b1) * gp;
                        anu[p] = b2 * anu[p] + (1.0 - b2) * gp * gp;
                        const double dir = (am[p] / c1) / (std::sqrt(anu[p] / c2) + eps);
                        if (p < nd * nd)
                            A[p] -= eta * dir;
                        else
                            t[p - nd * nd] -= eta * dir;
                    }
                }
            }
            out->ndim = nd;
            std::memcpy(out->A, bA, sizeof(bA));
            std::memcpy(out->t, bt, sizeof(bt));
            out->loss = best;
            out->diverged = diverged ? 1 : 0;
            out->iterations = total;
            if (!diverged) {
                const double det = nd == 2 ? bA[0] * bA[3] - bA[1] * bA[2]
                                           : bA[0] * (bA[4] * bA[8] - bA[5] * bA[7]) -
                                                 bA[1] * (bA[3] * bA[8] - bA[5] * bA[6]) +
                                                 bA[2] * (bA[3] * bA[7] - bA[4] * bA[6]);
                if (std::fabs(det) < 1e-3)
                    fail(DFM_E_NUMERICAL, "affine_register: transform collapsed (|det A| < 1e-3)");
            }
        });
    });
}

// ---------------------------------------------------------------------------
// evaluation epilogue (analysis.cpp:169-283)

}  // extern "C"

// analysis.cpp:192-246 from the device label counts (integers: exact)
static void assemble_overlap(const std::vector<unsigned long long>& c, int maxl,
                             dfm_overlap_summary* rep, dfm_region_overlap* regions, int64_t cap) {
    const size_t L = static_cast<size_t>(maxl) + 1;
    *rep = dfm_overlap_summary{};
    int64_t ps = 0, pt = 0, pi = 0, pfn = 0, pfp = 0, nr = 0;
    int to_n = 0, fp_n = 0, vs_n = 0;
    for (size_t l = 1; l < L; ++l) {
        const int64_t S = static_cast<int64_t>(c[l]), T = static_cast<int64_t>(c[L + l]),
                      I = static_cast<int64_t>(c[2 * L + l]);
        if (S == 0 && T == 0) continue;
        dfm_region_overlap r{};
        r.label = static_cast<int32_t>(l);
        r.warped_count = S;
        r.fixed_count = T;
        r.intersection = I;
        const int64_t fn = T - I, fp = S - I;
        if (T > 0) {
            r.has_to = r.has_fn = 1;
            r.to = static_cast<double>(I) / static_cast<double>(T);
            r.fn = static_cast<double>(fn) / static_cast<double>(T);
            rep->to_mean += r.to;
            rep->fn_mean += r.fn;
            ++to_n;
        }
        if (S > 0) {
            r.has_fp = 1;
            r.fp = static_cast<double>(fp) / static_cast<double>(S);
            rep->fp_mean += r.fp;
            ++fp_n;
        }
        const int64_t den = S + T;
        r.mo = 2.0 * static_cast<double>(I) / static_cast<double>(den);
        r.vs = 2.0 * static_cast<double>(S - T) / static_cast<double>(den);
        rep->mo_mean += r.mo;
        rep->vs_mean += r.vs;
        ++vs_n;
        ps += S;
        pt += T;
        pi += I;
        pfn += fn;
        pfp += fp;
        if (regions && nr < cap) regions[nr] = r;
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
        rep->to_klein = static_cast<double>(pi) / static_cast<double>(pt);
        rep->fn_klein = static_cast<double>(pfn) / static_cast<double>(pt);
    }
    if (ps > 0) rep->fp_klein = static_cast<double>(pfp) / static_cast<double>(ps);
    if (ps + pt > 0) {
        rep->mo_klein = 2.0 * static_cast<double>(pi) / static_cast<double>(ps + pt);
        rep->vs_klein = 2.0 * static_cast<double>(ps - pt) / static_cast<double>(ps + pt);
    }
    rep->n_regions = nr;
}

static void overlap_dev(dfm_ctx* ctx, int64_t n, const int32_t* dw, const int32_t* df,
                        dfm_overlap_summary* out, dfm_region_overlap* regions, int64_t cap) {
    int* dmax = ctx->arr<int>("ev_max", 1);
    launch_label_max(ctx->L(), dw, df, n, dmax);
    int maxl = 0;
    CK(cudaMemcpyAsync(&maxl, dmax, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (maxl >= (1 << 24)) fail(DFM_E_INVALID, "overlap_report: label values >= 2^24 unsupported");
    const size_t L = static_cast<size_t>(maxl) + 1;
    auto* cnt = ctx->arr<unsigned long long>("ev_counts", static_cast<int64_t>(3 * L));
    launch_label_hist(ctx->L(), dw, df, n, maxl, cnt);
    std::vector<unsigned long long> h(3 * L);
    CK(cudaMemcpyAsync(h.data(), cnt, sizeof(unsigned long long) * 3 * L, cudaMemcpyDeviceToHost,
                       ctx->stream));
    ctx->sync();
    assemble_overlap(h, maxl, out, regions, cap);
}

extern "C" {

dfm_status dfm_overlap_report(dfm_ctx* ctx, const dfm_grid* gw, const int32_t* warped,
                              const dfm_grid* gf, const int32_t* fixed, dfm_overlap_summary* out,
                              dfm_region_overlap* regions, int64_t max_regions) {
    return guarded([&] {
        validate_grid(gw);
        validate_grid(gf);
        if (!same_grid(gw, gf)) fail(DFM_E_INVALID, "overlap_report: grid mismatch");
        const Dims d = to_dims(gw);
        int32_t* dw = ctx->arr<int32_t>("ev_w", d.n);
        int32_t* df = ctx->arr<int32_t>("ev_f", d.n);
        CK(cudaMemcpyAsync(dw, warped, sizeof(int32_t) * d.n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(df, fixed, sizeof(int32_t) * d.n, cudaMemcpyHostToDevice, ctx->stream));
        overlap_dev(ctx, d.n, dw, df, out, regions, max_regions);
    });
}

dfm_status dfm_dev_overlap_report(dfm_ctx* ctx, const dfm_grid* g, const int32_t* d_warped,
                                  const int32_t* d_fixed, dfm_overlap_summary* out,
                                  dfm_region_overlap* regions, int64_t max_regions) {
    return guarded([&] {
        validate_grid(g);
        overlap_dev(ctx, to_dims(g).n, d_warped, d_fixed, out, regions, max_regions);
    });
}

dfm_status dfm_dev_warp_labels(dfm_ctx* ctx, const dfm_grid* g, const int32_t* d_labels,
                               const void* d_field_soa, int32_t* d_out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            const T* u = static_cast<const T*>(d_field_soa);
            launch_warp_labels<T>(ctx->L(), d_labels, CPlanes3<T>{{u, u + d.n, u + 2 * d.n}}, d,
                                  d_out);
            ctx->sync();
        });
    });
}

dfm_status dfm_landmark_error(dfm_ctx* ctx, const dfm_grid* fg, const dfm_grid* mg,
                              const dfm_grid* pg, const double* phi, int64_t n,
                              const double* fixed_mm, const double* moving_mm, double* dist,
                              double* mean, double* mx) {
    return guarded([&] {
        validate_grid(fg);
        validate_grid(mg);
        validate_grid(pg);
        if (!same_grid(pg, fg))
            fail(DFM_E_INVALID, "landmark_error: field must live on the fixed grid");
        if (n < 0) fail(DFM_E_INVALID, "landmark_error: negative landmark count");
        *mean = 0.0;
        *mx = 0.0;
        if (n == 0) return;
        const Dims d = to_dims(pg);
        // fixed-space mm -> fixed voxel coordinates (analysis.cpp:262-266)
        std::vector<double> vox(3 * static_cast<size_t>(n), 0.0);
        for (int64_t i = 0; i < n; ++i)
            for (int a = 0; a < fg->ndim; ++a)
                vox[3 * i + a] = (fixed_mm[3 * i + a] - fg->origin[a]) / fg->spacing[a];
        std::vector<double> u(3 * static_cast<size_t>(n), 0.0);
        DFM_DISPATCH(ctx, {
            Field<T> f = dev_field<T>(ctx, "api_f0", d.n);
            upload_field<T>(ctx, phi, d.n, d.ndim, f);
            double* dp = ctx->arr<double>("lm_pts", 3 * n);
            double* dv = ctx->arr<double>("lm_vals", 3 * n);
            CK(cudaMemcpyAsync(dp, vox.data(), sizeof(double) * 3 * n, cudaMemcpyHostToDevice,
                               ctx->stream));
            for (int c = 0; c < d.ndim; ++c)  // sample_field = per-component lerp
                launch_sample_points<T>(ctx->L(), f.p[c], d, dp, n, dv + c * n, nullptr);
            std::vector<double> hv(3 * static_cast<size_t>(n));
            CK(cudaMemcpyAsync(hv.data(), dv, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost,
                               ctx->stream));
            ctx->sync();
            for (int64_t i = 0; i < n; ++i)
                for (int c = 0; c < d.ndim; ++c) u[3 * i + c] = hv[c * n + i];
        });
        for (int64_t i = 0; i < n; ++i) {  // analysis.cpp:267-279
            double d2 = 0.0;
            for (int a = 0; a < fg->ndim; ++a) {
                const double mapped = (vox[3 * i + a] + u[3 * i + a]) * mg->spacing[a] + mg->origin[a];
                const double diff = mapped - moving_mm[3 * i + a];
                d2 += diff * diff;
            }
            const double dd = std::sqrt(d2);
            dist[i] = dd;
            *mean += dd;
            *mx = std::max(*mx, dd);
        }
        *mean /= static_cast<double>(n);
    });
}

dfm_status dfm_exp_map(dfm_ctx* ctx, const dfm_grid* g, const double* v, int M, double* out) {
    return guarded([&] {
        if (M < 0) fail(DFM_E_INVALID, "exp_map: M must be >= 0");
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            upload_field<T>(ctx, v, d.n, d.ndim, a);
            T* lev = ctx->arr<T>("api_svf_levels", 3 * d.n * (M + 1));
            launch_exp_map<T>(ctx->L(), a.p[0], d, M, lev);
            const T* r = lev + 3 * d.n * M;
            download_field<T, double>(ctx, CPlanes3<T>{{r, r + d.n, r + 2 * d.n}}, d.n, d.ndim,
                                      out);
            ctx->sync();
        });
    });
}

dfm_status dfm_svf_pullback(dfm_ctx* ctx, const dfm_grid* g, const double* v,
                            const double* grad_phi, int M, double* out) {
    return guarded([&] {
        if (M < 0) fail(DFM_E_INVALID, "svf_pullback: M must be >= 0");
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> b = dev_field<T>(ctx, "api_f1", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f2", d.n);
            upload_field<T>(ctx, v, d.n, d.ndim, a);
            upload_field<T>(ctx, grad_phi, d.n, d.ndim, b);
            T* lev = ctx->arr<T>("api_svf_levels", 3 * d.n * (M + 1));
            launch_exp_map<T>(ctx->L(), a.p[0], d, M, lev);
            SvfWork<T> ws{};
            ws.wa = ctx->arr<T>("api_svf_wa", 3 * d.n);
            ws.wb = ctx->arr<T>("api_svf_wb", 3 * d.n);
            // one (cell base, voxel) pair per voxel, double-buffered for the sort
            int32_t* kv = ctx->arr<int32_t>("api_svf_kv", 4 * d.n);
            for (int k = 0; k < 2; ++k) {
                ws.keys[k] = kv + (2 * k) * d.n;
                ws.vals[k] = kv + (2 * k + 1) * d.n;
            }
            ws.start = ctx->arr<int32_t>("api_svf_start", d.n + 1);
            ws.wts = ctx->arr<T>("api_svf_wts", 8 * d.n);
            ws.temp_bytes = svf_sort_temp_bytes(d.n);
            ws.temp = ctx->get("api_svf_temp", ws.temp_bytes);
            launch_svf_pullback<T>(ctx->L(), lev, d, M, b.p[0], o.p[0], ws);
            download_field<T, double>(ctx, o.r(), d.n, d.ndim, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_jacobian_det(dfm_ctx* ctx, const dfm_grid* g, const double* phi, double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            T* o = ctx->arr<T>("api_img0", d.n);
            upload_field<T>(ctx, phi, d.n, d.ndim, a);
            launch_jacobian_det<T>(ctx->L(), a.r(), d, o, nullptr);
            download_image<T, double>(ctx, o, d.n, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_jacobian(dfm_ctx* ctx, const dfm_grid* g, const double* phi, double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        const int64_t nn = static_cast<int64_t>(d.ndim) * d.ndim;
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            T* o = ctx->arr<T>("api_jac", nn * d.n);
            upload_field<T>(ctx, phi, d.n, d.ndim, a);
            launch_jacobian_full<T>(ctx->L(), a.r(), d, o);
            download_image<T, double>(ctx, o, nn * d.n, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_upsample_field_cubic(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                                    const dfm_grid* ng, double* out) {
    return guarded([&] {
        validate_grid(g);
        validate_grid(ng);
        if (ng->ndim != g->ndim) fail(DFM_E_INVALID, "upsample_field: dimensionality mismatch");
        for (int a = 0; a < g->ndim; ++a)
            if (ng->dims[a] < g->dims[a]) fail(DFM_E_INVALID, "upsample_field: shrinking not allowed");
        const Dims d = to_dims(g), nd = to_dims(ng);
        if (dims_equal(d, nd)) {
            std::memmove(out, phi, sizeof(double) * d.n * d.ndim);
            return;
        }
        double step[3] = {0.0, 0.0, 0.0}, rescale[3] = {1.0, 1.0, 1.0};
        for (int a = 0; a < g->ndim; ++a) {
            step[a] = static_cast<double>(g->dims[a] - 1) / static_cast<double>(ng->dims[a] - 1);
            rescale[a] = static_cast<double>(ng->dims[a] - 1) / static_cast<double>(g->dims[a] - 1);
        }
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f1", nd.n);
            upload_field<T>(ctx, phi, d.n, d.ndim, a);
            launch_upsample_cubic<T>(ctx->L(), a.r(), d, o.w(), nd, step, rescale);
            download_field<T, double>(ctx, o.r(), nd.n, nd.ndim, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_sgd_step(dfm_ctx* ctx, const dfm_grid* g, double* mu, const double* v,
                        double momentum, double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        const size_t cnt = static_cast<size_t>(d.n) * d.ndim;
        if (momentum == 0.0) {  // optim.cpp:45-46: v unchanged, mu untouched
            std::memmove(out, v, sizeof(double) * cnt);
            return;
        }
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> b = dev_field<T>(ctx, "api_f1", d.n);
            upload_field<T>(ctx, mu, d.n, d.ndim, a);
            upload_field<T>(ctx, v, d.n, d.ndim, b);
            launch_sgd<T>(ctx->L(), a.w(), b.r(), d, momentum);
            download_field<T, double>(ctx, a.r(), d.n, d.ndim, mu);
            ctx->sync();
        });
        std::memcpy(out, mu, sizeof(double) * cnt);
    });
}

dfm_status dfm_sample_field_points(dfm_ctx* ctx, const dfm_grid* g, const double* field,
                                   int64_t npts, const double* points, double* values,
                                   double* jac) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        const int nd = d.ndim;
        DFM_DISPATCH(ctx, {
            Field<T> f = dev_field<T>(ctx, "api_f0", d.n);
            upload_field<T>(ctx, field, d.n, nd, f);
            double* pts = ctx->arr<double>("api_pts", 3 * npts + 1);
            double* vals = ctx->arr<double>("api_vals", 3 * npts + 1);
            double* grs = ctx->arr<double>("api_grads", 9 * npts + 1);
            std::vector<double> hv(3 * static_cast<size_t>(npts)), hg(9 * static_cast<size_t>(npts));
            if (npts > 0) {
                CK(cudaMemcpyAsync(pts, points, sizeof(double) * 3 * npts, cudaMemcpyHostToDevice,
                                   ctx->stream));
                // sample_field / sample_field_jacobian (interp.cpp:188-227): the
                // per-component lerp and its gradient
                for (int c = 0; c < nd; ++c)
                    launch_sample_points<T>(ctx->L(), f.p[c], d, pts, npts, vals + c * npts,
                                            jac ? grs + 3 * c * npts : nullptr);
                CK(cudaMemcpyAsync(hv.data(), vals, sizeof(double) * nd * npts,
                                   cudaMemcpyDeviceToHost, ctx->stream));
                if (jac)
                    CK(cudaMemcpyAsync(hg.data(), grs, sizeof(double) * 3 * nd * npts,
                                       cudaMemcpyDeviceToHost, ctx->stream));
            }
            ctx->sync();
            for (int64_t i = 0; i < npts; ++i)
                for (int c = 0; c < 3; ++c) {
                    values[3 * i + c] = c < nd ? hv[c * npts + i] : 0.0;
                    if (jac)
                        for (int a = 0; a < 3; ++a)
                            jac[9 * i + 3 * c + a] =
                                (c < nd && a < nd) ? hg[3 * c * npts + 3 * i + a] : 0.0;
                }
        });
    });
}

dfm_status dfm_singularity_fraction(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                                    double* fraction) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            auto* cnt = ctx->arr<unsigned long long>("api_count", 1);
            upload_field<T>(ctx, phi, d.n, d.ndim, a);
            CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
            launch_jacobian_det<T>(ctx->L(), a.r(), d, nullptr, cnt);
            unsigned long long h = 0;
            CK(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            *fraction = static_cast<double>(h) / static_cast<double>(d.n);
        });
    });
}

static dfm_status smooth_api(dfm_ctx* ctx, const dfm_grid* g, const double* in,
                             const double sigma[3], double* out, bool field) {
    return guarded([&] {
        validate_grid(g);
        for (int a = 0; a < g->ndim; ++a)
            if (sigma[a] < 0.0)
                fail(DFM_E_INVALID, field ? "gaussian_smooth_field: sigma must be >= 0"
                                          : "gaussian_smooth: sigma must be >= 0");
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f1", d.n);
            if (field)
                upload_field<T>(ctx, in, d.n, d.ndim, a);
            else
                upload_image<T, double>(ctx, in, d.n, a.p[0]);
            const int nc = field ? 3 : 1;
            smooth_planes<T>(ctx, d, sigma, a.r(), o.w(), nc, "api");
            if (field)
                download_field<T, double>(ctx, o.r(), d.n, d.ndim, out);
            else
                download_image<T, double>(ctx, o.p[0], d.n, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_gaussian_smooth(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                               const double sigma[3], double* out) {
    return smooth_api(ctx, g, img, sigma, out, false);
}

dfm_status dfm_gaussian_smooth_field(dfm_ctx* ctx, const dfm_grid* g, const double* f,
                                     const double sigma[3], double* out) {
    return smooth_api(ctx, g, f, sigma, out, true);
}

// resample kinds: 0 resample_field_linear, 1 upsample_field, 2 resample_displacement
static dfm_status resample_api(dfm_ctx* ctx, const dfm_grid* g, const double* f,
                               const dfm_grid* ng, double* out, int kind) {
    static const char* names[3] = {"resample_field_linear", "upsample_field",
                                   "resample_displacement"};
    return guarded([&] {
        validate_grid(g);
        validate_grid(ng);
        if (ng->ndim != g->ndim) fail(DFM_E_INVALID, "%s: dimensionality mismatch", names[kind]);
        if (kind == 1)
            for (int a = 0; a < g->ndim; ++a)
                if (ng->dims[a] < g->dims[a])
                    fail(DFM_E_INVALID, "upsample_field: shrinking not allowed");
        const Dims d = to_dims(g), nd = to_dims(ng);
        if (dims_equal(d, nd)) {  // returned unchanged (interp.cpp:386-387, 417-418, 452-453)
            std::memmove(out, f, sizeof(double) * d.n * d.ndim);
            return;
        }
        double mult[3] = {1.0, 1.0, 1.0};
        if (kind != 0)
            for (int a = 0; a < g->ndim; ++a)
                mult[a] = static_cast<double>(ng->dims[a] - 1) / static_cast<double>(g->dims[a] - 1);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f1", nd.n);
            upload_field<T>(ctx, f, d.n, d.ndim, a);
            const T* src[3] = {a.p[0], a.p[1], a.p[2]};
            T* dst[3] = {o.p[0], o.p[1], o.p[2]};
            launch_resample<T>(ctx->L(), src, d, dst, nd, d.ndim, mult);
            download_field<T, double>(ctx, o.r(), nd.n, nd.ndim, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_upsample_field(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                              const dfm_grid* new_grid, double* out) {
    return resample_api(ctx, g, phi, new_grid, out, 1);
}
dfm_status dfm_resample_field_linear(dfm_ctx* ctx, const dfm_grid* g, const double* f,
                                     const dfm_grid* new_grid, double* out) {
    return resample_api(ctx, g, f, new_grid, out, 0);
}
dfm_status dfm_resample_displacement(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                                     const dfm_grid* new_grid, double* out) {
    return resample_api(ctx, g, phi, new_grid, out, 2);
}

static dfm_status loss_api(dfm_ctx* ctx, int loss, const dfm_grid* fg, const double* fixed,
                           const dfm_grid* mg, const double* moving, const double* phi, int R,
                           double* value, double* grad) {
    static const char* names[3] = {"ssd_eval", "lncc_eval", "dice_soft_eval"};
    return guarded([&] {
        validate_grid(fg);
        validate_grid(mg);
        if (fg->ndim != mg->ndim) fail(DFM_E_INVALID, "%s: dimensionality mismatch", names[loss]);
        if (loss == DFM_LOSS_LNCC) {
            if (R < 1) fail(DFM_E_INVALID, "lncc_eval: window_radius must be >= 1");
            for (int a = 0; a < fg->ndim; ++a)
                if (2 * static_cast<int64_t>(R) + 1 > fg->dims[a])
                    fail(DFM_E_INVALID, "lncc_eval: window larger than image");
            if (R > kRMax) fail(DFM_E_INVALID, "lncc_eval: window_radius > %d unsupported", kRMax);
        }
        if (loss == DFM_LOSS_DICE) {
            const int64_t nf = fg->dims[0] * fg->dims[1] * fg->dims[2];
            const int64_t nm = mg->dims[0] * mg->dims[1] * mg->dims[2];
            for (int64_t i = 0; i < nf; ++i)
                if (!(fixed[i] >= 0.0 && fixed[i] <= 1.0))
                    fail(DFM_E_INVALID, "dice_soft_eval: fixed mask values outside [0,1]");
            for (int64_t i = 0; i < nm; ++i)
                if (!(moving[i] >= 0.0 && moving[i] <= 1.0))
                    fail(DFM_E_INVALID, "dice_soft_eval: moving mask values outside [0,1]");
        }
        const Dims d = to_dims(fg), dm = to_dims(mg);
        DFM_DISPATCH(ctx, {
            T* F = ctx->arr<T>("api_img0", d.n);
            T* M = ctx->arr<T>("api_img1", dm.n);
            Field<T> u = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> gr = dev_field<T>(ctx, "api_f1", d.n);
            upload_image<T, double>(ctx, fixed, d.n, F);
            upload_image<T, double>(ctx, moving, dm.n, M);
            upload_field<T>(ctx, phi, d.n, d.ndim, u);
            *value = eval_loss_dev<T>(ctx, loss, R, F, M, d, dm, u.r(), grad != nullptr, gr.w());
            if (grad) download_field<T, double>(ctx, gr.r(), d.n, d.ndim, grad);
            ctx->sync();
        });
    });
}

dfm_status dfm_ssd_eval(dfm_ctx* ctx, const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                        const double* moving, const double* phi, double* value, double* grad) {
    return loss_api(ctx, DFM_LOSS_SSD, fg, fixed, mg, moving, phi, 0, value, grad);
}
dfm_status dfm_lncc_eval(dfm_ctx* ctx, const dfm_grid* fg, const double* fixed,
                         const dfm_grid* mg, const double* moving, const double* phi, int r,
                         double* value, double* grad) {
    return loss_api(ctx, DFM_LOSS_LNCC, fg, fixed, mg, moving, phi, r, value, grad);
}
dfm_status dfm_dice_eval(dfm_ctx* ctx, const dfm_grid* fg, const double* fixed,
                         const dfm_grid* mg, const double* moving, const double* phi,
                         double* value, double* grad) {
    return loss_api(ctx, DFM_LOSS_DICE, fg, fixed, mg, moving, phi, 0, value, grad);
}

dfm_status dfm_adam_step(dfm_ctx* ctx, const dfm_grid* g, double* m, double* nu, int64_t* t,
                         double b1, double b2, double eps, const double* v, double* dir) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        *t += 1;
        const double c1 = 1.0 - std::pow(b1, static_cast<double>(*t));
        const double c2 = 1.0 - std::pow(b2, static_cast<double>(*t));
        DFM_DISPATCH(ctx, {
            Field<T> fm = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> fn = dev_field<T>(ctx, "api_f1", d.n);
            Field<T> fv = dev_field<T>(ctx, "api_f2", d.n);
            Field<T> fd = dev_field<T>(ctx, "api_f3", d.n);
            upload_field<T>(ctx, m, d.n, d.ndim, fm);
            upload_field<T>(ctx, nu, d.n, d.ndim, fn);
            upload_field<T>(ctx, v, d.n, d.ndim, fv);
            launch_adam<T>(ctx->L(), fm.w(), fn.w(), fv.r(), fd.w(), d, b1, b2, c1, c2, eps);
            download_field<T, double>(ctx, fm.r(), d.n, d.ndim, m);
            download_field<T, double>(ctx, fn.r(), d.n, d.ndim, nu);
            download_field<T, double>(ctx, fd.r(), d.n, d.ndim, dir);
            ctx->sync();
        });
    });
}

dfm_status dfm_upsample_state(dfm_ctx* ctx, const dfm_grid* g, const double* m, const double* nu,
                              const dfm_grid* ng, double* m_out, double* nu_out) {
    return guarded([&] {
        validate_grid(ng);
        for (int a = 0; a < ng->ndim; ++a)
            if (ng->dims[a] < g->dims[a])
                fail(DFM_E_INVALID, "upsample_state: shrinking not allowed");
        validate_grid(g);
        if (ng->ndim != g->ndim) fail(DFM_E_INVALID, "upsample_field: dimensionality mismatch");
        const Dims d = to_dims(g), nd = to_dims(ng);
        if (dims_equal(d, nd)) {
            std::memmove(m_out, m, sizeof(double) * d.n * d.ndim);
            std::memmove(nu_out, nu, sizeof(double) * d.n * d.ndim);
            return;
        }
        double mm[3] = {1.0, 1.0, 1.0}, mn[3] = {1.0, 1.0, 1.0};
        for (int a = 0; a < g->ndim; ++a) {
            const double r =
                static_cast<double>(ng->dims[a] - 1) / static_cast<double>(g->dims[a] - 1);
            mm[a] = r;
            mn[a] = r * r;
        }
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> b = dev_field<T>(ctx, "api_f1", d.n);
            Field<T> oa = dev_field<T>(ctx, "api_f2", nd.n);
            Field<T> ob = dev_field<T>(ctx, "api_f3", nd.n);
            upload_field<T>(ctx, m, d.n, d.ndim, a);
            upload_field<T>(ctx, nu, d.n, d.ndim, b);
            const T* sa[3] = {a.p[0], a.p[1], a.p[2]};
            T* da[3] = {oa.p[0], oa.p[1], oa.p[2]};
            const T* sb[3] = {b.p[0], b.p[1], b.p[2]};
            T* db[3] = {ob.p[0], ob.p[1], ob.p[2]};
            launch_resample<T>(ctx->L(), sa, d, da, nd, d.ndim, mm);
            launch_resample<T>(ctx->L(), sb, d, db, nd, d.ndim, mn);
            download_field<T, double>(ctx, oa.r(), nd.n, nd.ndim, m_out);
            download_field<T, double>(ctx, ob.r(), nd.n, nd.ndim, nu_out);
            ctx->sync();
        });
    });
}

dfm_status dfm_eulerian_direction(dfm_ctx* ctx, const dfm_grid* g, const double* grad,
                                  const double* phi, int use_jac, double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> b = dev_field<T>(ctx, "api_f1", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f2", d.n);
            upload_field<T>(ctx, grad, d.n, d.ndim, a);
            upload_field<T>(ctx, phi, d.n, d.ndim, b);
            launch_eulerian<T>(ctx->L(), a.r(), b.r(), d, use_jac, o.w());
            download_field<T, double>(ctx, o.r(), d.n, d.ndim, out);
            ctx->sync();
        });
    });
}

dfm_status dfm_apply_update(dfm_ctx* ctx, const dfm_grid* g, const double* phi, const double* v,
                            double eta, double sigma_warp, double cap, double* out) {
    return guarded([&] {
        validate_grid(g);
        const Dims d = to_dims(g);
        DFM_DISPATCH(ctx, {
            Field<T> a = dev_field<T>(ctx, "api_f0", d.n);
            Field<T> b = dev_field<T>(ctx, "api_f1", d.n);
            Field<T> s = dev_field<T>(ctx, "api_f2", d.n);
            Field<T> o = dev_field<T>(ctx, "api_f3", d.n);
            int* bad = ctx->arr<int>("api_flag", 1);
            upload_field<T>(ctx, phi, d.n, d.ndim, a);
            upload_field<T>(ctx, v, d.n, d.ndim, b);
            CK(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
            launch_clamp_step<T>(ctx->L(), b.r(), s.w(), d, eta, cap, bad);
            int hb = 0;
            CK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            if (hb) fail(DFM_E_NUMERICAL, "apply_update: non-finite step");
            const double sw[3] = {sigma_warp, sigma_warp, sigma_warp};
            const HostGauss h = make_gauss(d, sw);
            int done_tma = -1;
            if (h.R <= 4 && tma_supported(d, sizeof(T))) {
                const GaussW<T> w = upload_gauss<T>(ctx, h, d, "api_warp");
                done_tma = launch_compose_tma<T>(ctx->L(), h.R, cap, w, s.p[0], a.p[0], o.p[0],
                                                 nullptr, d, d, nullptr, nullptr, nullptr);
            }
            if (done_tma >= 0) {
                // plane-streaming compose + sigma_warp smoothing (the loop's kernel)
            } else if (sigma_warp > 0.0 && h.R <= kRMax) {
                const GaussW<T> w = upload_gauss<T>(ctx, h, d, "api_warp");
                launch_compose_smooth<T>(ctx->L(), h.R, w, s.r(), a.r(), o.w(), d, nullptr);
            } else {
                launch_compose<T>(ctx->L(), a.r(), s.r(), d, o.w());
                if (sigma_warp > 0.0) {
                    smooth_planes<T>(ctx, d, sw, o.r(), b.w(), 3, "api_warp2");
                    o = b;
                }
            }
            download_field<T, double>(ctx, o.r(), d.n, d.ndim, out);
            ctx->sync();
        });
    });
}

}  // extern "C"

// ===========================================================================
// register_images (pipeline.cpp:121-224), direct mode, fully device-resident

namespace {

struct RegOut {
    std::vector<dfm_iter_record> recs;
    double final_loss = 0.0, sing = 0.0, total_ms = 0.0;
};

void validate_config(const dfm_config* c) {
    if (!c) fail(DFM_E_INVALID, "config is NULL");
    if (!(c->eta > 0.0) || !std::isfinite(c->eta))
        fail(DFM_E_INVALID, "config: eta must be positive and finite");
    if (c->sigma_grad < 0.0 || c->sigma_warp < 0.0) fail(DFM_E_INVALID, "config: sigmas must be >= 0");
    if (c->lncc_radius < 1) fail(DFM_E_INVALID, "config: lncc_radius must be >= 1");
    if (c->svf_M < 0) fail(DFM_E_INVALID, "config: svf_M must be >= 0");
    if (!(c->beta1 >= 0.0 && c->beta1 < 1.0) || !(c->beta2 >= 0.0 && c->beta2 < 1.0))
        fail(DFM_E_INVALID, "config: betas must lie in [0, 1)");
    if (!(c->eps_adam > 0.0)) fail(DFM_E_INVALID, "config: eps_adam must be positive");
    if (!(c->step_cap > 0.0)) fail(DFM_E_INVALID, "config: step_cap must be positive");
    if (c->conv_window < 1) fail(DFM_E_INVALID, "config: conv_window must be >= 1");
    if (c->conv_tol < 0.0) fail(DFM_E_INVALID, "config: conv_tol must be >= 0");
    if (c->mode == DFM_MODE_SVF && c->loss == DFM_LOSS_DICE)
        fail(DFM_E_INVALID, "config: dice loss is not available in svf mode");
    if (c->mode != DFM_MODE_DIRECT && c->mode != DFM_MODE_SVF) fail(DFM_E_INVALID, "config: unknown mode");
    if (c->loss < 0 || c->loss > 2) fail(DFM_E_INVALID, "unknown loss");
    if (c->loss == DFM_LOSS_LNCC && c->lncc_radius > kRMax)
        fail(DFM_E_INVALID, "lncc_radius > %d unsupported on the device path", kRMax);
}

void validate_schedule(const double* s, const int32_t* it, int ns) {
    if (ns < 1 || !s || !it) fail(DFM_E_INVALID, "schedule: at least one scale required");
    for (int i = 0; i < ns; ++i) {
        if (!(s[i] >= 1.0) || !std::isfinite(s[i]))
            fail(DFM_E_INVALID, "schedule: scales must be finite and >= 1");
        if (i > 0 && !(s[i] < s[i - 1]))
            fail(DFM_E_INVALID, "schedule: scales must be strictly decreasing");
        if (it[i] < 0) fail(DFM_E_INVALID, "schedule: iterations must be >= 0");
    }
}

// kernel classes for the optional per-kernel timing
enum { KC_FWD = 0, KC_BWD = 1, KC_ADAM = 2, KC_COMPOSE = 3, KC_MON = 4, KC_PYR = 5, KC_EPI = 6 };

template <class T>
struct Registrar {
    // called once the full-resolution result field is final, before the
    // epilogue's loss and fold-check kernels (which only read it): the host
    // entry point starts the result download there, beside the epilogue
    std::function<void(CPlanes3<T>)> on_final;
    dfm_ctx* ctx;
    const dfm_grid* g;
    const dfm_config* cfg;
    Dims full;
    // workspace
    T* Fbuf;
    T* Mbuf;
    T* Fs;
    T* Ms;
    Field<T> u[2], m, nu, grad, step;
    T* coef[4];
    double* partials;
    LoopState* st;
    double* loss;
    unsigned long long* maxstep;
    unsigned long long* stamp;
    double* corr1;
    double* corr2;
    int cur = 0;
    GaussW<T> w_id{};          // identity (sigma 0) weights of the current level
    double* fstat = nullptr;   // per-level muF, vF (2 planes) for the 3-moment forward
    bool fstat_ready = false;  // this level's F statistics are current
    // the loop kept W = M(x+u) current for the field it ends with (and fstat
    // for the level's F), on a level of dims w_dims
    bool w_final = false;
    Dims w_dims{};
    T* Wb = nullptr;  // W = M(x+u) for the current u (TMA path)
    T* Gb = nullptr;  // grad M(x+u), 3 planes
    bool use_tma = false;    // fused W/G-carrying loop (plane-streaming and/or brick kernels)
    bool use_brick = false;  // this scale runs the brick kernels
    // SVF mode (pipeline.cpp:166-167, 189-206): exp_map levels + pullback work
    T* svf_levels = nullptr;
    T* svf_g = nullptr;  // pulled-back gradient (3 planes)
    SvfWork<T> svf{};
    // profiling
    std::vector<cudaEvent_t> evpool;
    std::vector<std::pair<int, int>> evuse;  // (class, pool index of start)

    void alloc(int64_t total_iters) {
        const int64_t n = full.n;
        Fbuf = Fs = ctx->arr<T>("reg_Fs", n);
        Mbuf = Ms = ctx->arr<T>("reg_Ms", n);
        u[0] = dev_field<T>(ctx, "reg_u0", n);
        u[1] = dev_field<T>(ctx, "reg_u1", n);
        m = dev_field<T>(ctx, "reg_m", n);
        nu = dev_field<T>(ctx, "reg_nu", n);
        grad = dev_field<T>(ctx, "reg_grad", n);
        step = dev_field<T>(ctx, "reg_step", n);
        T* cb = ctx->arr<T>("reg_coef", 4 * n);
        for (int k = 0; k < 4; ++k) coef[k] = cb + k * n;
        Wb = ctx->arr<T>("reg_W", n);
        Gb = ctx->arr<T>("reg_G", 3 * n);
        if (cfg->loss == DFM_LOSS_LNCC && ctx->fwd3) fstat = ctx->arr<double>("reg_fstat", 2 * n);
        if (cfg->mode == DFM_MODE_SVF) {
            const int M = cfg->svf_M;
            svf_levels = ctx->arr<T>("svf_levels", 3 * n * (M + 1));
            svf_g = ctx->arr<T>("svf_g", 3 * n);
            svf.wa = ctx->arr<T>("svf_wa", 3 * n);
            svf.wb = ctx->arr<T>("svf_wb", 3 * n);
            int32_t* kv = ctx->arr<int32_t>("svf_kv", 4 * n);  // keys/vals x 2 (sort)
            for (int k = 0; k < 2; ++k) {
                svf.keys[k] = kv + (2 * k) * n;
                svf.vals[k] = kv + (2 * k + 1) * n;
            }
            svf.start = ctx->arr<int32_t>("svf_start", n + 1);
            svf.wts = ctx->arr<T>("svf_wts", 8 * n);
            svf.temp_bytes = svf_sort_temp_bytes(n);
            svf.temp = ctx->get("svf_temp", svf.temp_bytes);
        }
        partials = ctx->arr<double>("reg_partials", 3 * 65536);
        st = ctx->arr<LoopState>("reg_state", 1);
        const int64_t cap = total_iters + 2;
        loss = ctx->arr<double>("reg_loss", cap);
        maxstep = ctx->arr<unsigned long long>("reg_maxstep", cap);
        stamp = ctx->arr<unsigned long long>("reg_stamp", cap);
        corr1 = ctx->arr<double>("reg_corr1", cap);
        corr2 = ctx->arr<double>("reg_corr2", cap);
        std::vector<double> h1(cap), h2(cap);
        for (int64_t t = 0; t < cap; ++t) {
            h1[t] = 1.0 - std::pow(cfg->beta1, static_cast<double>(t));
            h2[t] = 1.0 - std::pow(cfg->beta2, static_cast<double>(t));
        }
        ctx->upload(corr1, h1.data(), sizeof(double) * cap, "reg_corr1");
        ctx->upload(corr2, h2.data(), sizeof(double) * cap, "reg_corr2");
        CK(cudaMemsetAsync(st, 0, sizeof(LoopState), ctx->stream));
    }

    void zero_field(Field<T>& f, int64_t n) {
        CK(cudaMemsetAsync(f.p[0], 0, sizeof(T) * n, ctx->stream));
        CK(cudaMemsetAsync(f.p[1], 0, sizeof(T) * n, ctx->stream));
        CK(cudaMemsetAsync(f.p[2], 0, sizeof(T) * n, ctx->stream));
    }

    // profiling helpers
    void ev_begin(int cls) {
        if (!ctx->profiling) return;
        const size_t k = evpool.size();
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        evpool.push_back(a);
        evpool.push_back(b);
        evuse.push_back({cls, static_cast<int>(k)});
        CK(cudaEventRecord(a, ctx->stream));
    }
    void ev_end() {
        if (!ctx->profiling) return;
        CK(cudaEventRecord(evpool.back(), ctx->stream));
    }
    void ev_collect(const Dims& d) {
        if (!ctx->profiling) return;
        ctx->sync();
        for (auto& pr : evuse) {
            // loop classes are reported for the full-resolution scale only
            if (pr.first <= KC_MON && d.n != full.n) continue;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, evpool[pr.second], evpool[pr.second + 1]));
            ctx->kt_ms[pr.first] += ms;
            ctx->kt_n[pr.first] += 1;
            ctx->kt_vox[pr.first] += d.n;
        }
        for (auto e : evpool) cudaEventDestroy(e);
        evpool.clear();
        evuse.clear();
    }

    // can this scale run the plane-streaming (TMA) kernels?
    bool tma_eligible(const Dims& d, int Rg, int Rw, bool big) const {
        return !big && cfg->step_cap <= 1.5 && Rg <= 6 && Rw <= 4 &&
               d.ndim == 3 &&  // Compose2's fused W/G gather is 3-D only
               (cfg->loss != DFM_LOSS_LNCC || cfg->lncc_radius <= 5) &&
               tma_supported(d, sizeof(T));
    }

    // one iteration with the plane-streaming kernels: u[src] -> u[1-src]; W, G
    // (warped moving image and its interpolant gradient at u[src]) are kept
    // current by the compose of the previous iteration / warpgrad at scale start.
    void enqueue_iteration_tma(const Dims& d, int src, int Rg, int Rw, const GaussW<T>& wg,
                               const GaussW<T>& ww) {
        Launch L = ctx->L();
        const int loss_kind = cfg->loss;
        const CPlanes3<T> uin = u[src].r();
        const bool lncc = loss_kind == DFM_LOSS_LNCC;
        const int mask = ctx->tma_mask;  // A/B switch per kernel (DFM_TMA_MASK)
        int np;
        ev_begin(KC_FWD);
        const bool fused = lncc && (mask & 1);
        if (fused) {  // LNCC moments + window coefficients + loss + monitor, one launch
            const MonitorArgs mon{st, loss, stamp, cfg->conv_window, cfg->conv_tol};
            if (use_brick)
                np = launch_lncc_fwd_brick<T>(L, cfg->lncc_radius, Fs, Wb, d, coef[0], partials,
                                              st, &mon, fstat_ready ? fstat : nullptr);
            else if (fstat_ready)
                np = launch_lncc_fwd3_tma<T>(L, cfg->lncc_radius, Fs, Wb, fstat, d, coef[0],
                                             partials, st, &mon);
            else
                np = launch_lncc_fwd_tma<T>(L, cfg->lncc_radius, Fs, Wb, d, coef[0], partials,
                                            st, &mon);
        } else if (loss_kind == DFM_LOSS_SSD) {  // loss + grad + monitor, one launch
            const MonitorArgs mon{st, loss, stamp, cfg->conv_window, cfg->conv_tol};
            np = launch_ssd<T>(L, Fs, Ms, d, d, uin, grad.w(), partials, st, &mon);
        } else {
            np = loss_kind_launch_fwd<T>(ctx, loss_kind, cfg->lncc_radius, Fs, Ms, d, d, uin,
                                         coef, grad.w(), partials, st);
        }
        ev_end();
        if (!fused && loss_kind != DFM_LOSS_SSD) {
            ev_begin(KC_MON);
            launch_monitor(L, monitor_kind(loss_kind), partials, np, static_cast<double>(d.n),
                           st, loss, stamp, cfg->conv_window, cfg->conv_tol);
            ev_end();
        }
        if (lncc) {
            ev_begin(KC_BWD);
            if (use_brick) {
                launch_lncc_bwd_brick<T>(L, cfg->lncc_radius, coef[0], Fs, Wb, Gb, d, grad.p[0],
                                         st);
            } else if (mask & 2) {
                launch_lncc_bwd_tma<T>(L, cfg->lncc_radius, coef[0], Fs, Wb, Gb, d, grad.p[0], st);
            } else {
                const T* cc[4] = {coef[0], coef[1], coef[2], coef[3]};
                launch_lncc_bwd<T>(L, cfg->lncc_radius, Fs, Ms, d, d, uin, cc, grad.w(), st);
            }
            ev_end();
        } else if (loss_kind == DFM_LOSS_DICE) {
            ev_begin(KC_BWD);
            launch_dice_grad<T>(L, Fs, Ms, d, d, uin, grad.w(), st, 0.0, 1.0);
            ev_end();
        }
        AdamParams ap{cfg->beta1, cfg->beta2, cfg->eps_adam, cfg->eta, cfg->step_cap,
                      corr1, corr2, cfg->use_jac};
        // measured: the split wins on mid-size levels (80x96x112: 127 -> 115 us per
        // iteration) and loses on the full 160x192x224 level (610 -> 650 us)
        const bool split = !use_brick && ctx->split_compose && (mask & 4) && (mask & 8) &&
                           d.ndim == 3 && d.n < ctx->split_fold_max && !cfg->use_jac;
        if (use_brick && ctx->split_compose) {  // brick: compose once per voxel, not per halo
            ev_begin(KC_ADAM);
            const int r1 = launch_smooth_adam_compose_brick<T>(
                L, Rg, wg, grad.p[0], m.p[0], nu.p[0], u[src].p[0], step.p[0], cfg->step_cap, d,
                ap, st, maxstep);
            ev_end();
            ev_begin(KC_COMPOSE);
            const int r2 = launch_compose_smooth_brick<T>(L, Rw, ww, step.p[0], u[1 - src].p[0],
                                                          Ms, d, d, lncc ? Wb : nullptr,
                                                          lncc ? Gb : nullptr, st);
            ev_end();
            if (r1 < 0 || r2 < 0) fail(DFM_E_CUDA, "split update launch failed");
            return;
        }
        // large levels: plain smooth+Adam, a pointwise compose kernel, then the
        // smoothing + W/G kernel (compose once per voxel, at full occupancy)
        // use_jac (diffeo.cpp:25-39): J(u)^T in the plain smooth+Adam, so this path
        const bool split3 = !use_brick && (mask & 4) && (mask & 8) && d.ndim == 3 &&
                            ((ctx->split_compose && ctx->split3 && d.n >= ctx->split_fold_max) ||
                             cfg->use_jac);
        if (split3) {
            ev_begin(KC_ADAM);
            if (launch_smooth_adam_tma<T>(L, Rg, wg, grad.p[0], m.p[0], nu.p[0], step.p[0], d, ap,
                                          st, maxstep, cfg->use_jac ? u[src].p[0] : nullptr) < 0)
                fail(DFM_E_CUDA, "smooth+Adam launch failed");
            ev_end();
            ev_begin(KC_COMPOSE);
            T* cbuf = grad.p[0];  // grad is dead after smooth+Adam: it holds c
            // the plane-streaming compose at Gaussian radius 0: c = step + u(x+step)
            // from TMA-staged u tiles, no halo recomposition, no W/G, no count
            if (launch_compose_tma<T>(L, 0, cfg->step_cap, w_id, step.p[0], u[src].p[0], cbuf,
                                      Ms, d, d, nullptr, nullptr, st, false) < 0)
                launch_compose_pointwise<T>(L, step.p[0], u[src].p[0], cfg->step_cap, d, cbuf,
                                            st);
            const int r2 = launch_compose_smooth_tma<T>(L, Rw, ww, cbuf, u[1 - src].p[0], Ms, d,
                                                        d, lncc ? Wb : nullptr,
                                                        lncc ? Gb : nullptr, st);
            ev_end();
            if (r2 < 0) fail(DFM_E_CUDA, "split update launch failed");
            return;
        }
        if (split) {
            ev_begin(KC_ADAM);
            const int r1 = launch_smooth_adam_compose_tma<T>(L, Rg, wg, grad.p[0], m.p[0],
                                                             nu.p[0], u[src].p[0], step.p[0],
                                                             cfg->step_cap, d, ap, st, maxstep);
            ev_end();
            ev_begin(KC_COMPOSE);
            const int r2 = launch_compose_smooth_tma<T>(L, Rw, ww, step.p[0], u[1 - src].p[0],
                                                        Ms, d, d, lncc ? Wb : nullptr,
                                                        lncc ? Gb : nullptr, st);
            ev_end();
            if (r1 < 0 || r2 < 0) fail(DFM_E_CUDA, "split update launch failed");
            return;
        }
        ev_begin(KC_ADAM);
        if (use_brick)
            launch_smooth_adam_brick<T>(L, Rg, wg, grad.p[0], m.p[0], nu.p[0], step.p[0], d, ap,
                                        st, maxstep);
        else if (mask & 4)
            launch_smooth_adam_tma<T>(L, Rg, wg, grad.p[0], m.p[0], nu.p[0], step.p[0], d, ap, st,
                                      maxstep);
        else
            launch_smooth_adam<T>(L, Rg, wg, grad.r(), uin, m.w(), nu.w(), step.w(), d, ap, st,
                                  maxstep);
        ev_end();
        ev_begin(KC_COMPOSE);
        if (use_brick) {
            launch_compose_brick<T>(L, Rw, ww, step.p[0], u[src].p[0], u[1 - src].p[0], Ms, d, d,
                                    lncc ? Wb : nullptr, lncc ? Gb : nullptr, st);
        } else if (mask & 8) {
            launch_compose_tma<T>(L, Rw, cfg->step_cap, ww, step.p[0], u[src].p[0],
                                  u[1 - src].p[0], Ms, d, d, lncc ? Wb : nullptr,
                                  lncc ? Gb : nullptr, st);
        } else {
            launch_compose_smooth<T>(L, Rw, ww, step.r(), uin, u[1 - src].w(), d, st);
            if (lncc) launch_warpgrad<T>(L, Ms, d, u[1 - src].r(), d, Wb, Gb);
        }
        ev_end();
    }

    // one SVF iteration (pipeline.cpp:166-167, 189-206), v = u[src] -> u[1-src]:
    // phi = exp(v); loss + grad at phi; g = pullback; sigma_grad; -g; Adam;
    // v' = G_sigma_warp * (v + clamp(eta dir))
    void enqueue_iteration_svf(const Dims& d, int src, int Rg, int Rw, const GaussW<T>& wg,
                               const GaussW<T>& ww, const DevAxisGauss* big_g,
                               const DevAxisGauss* big_w) {
        Launch L = ctx->L();
        const int M = cfg->svf_M;
        const int64_t n = d.n;
        const int loss_kind = cfg->loss;
        ev_begin(KC_FWD);
        launch_exp_map<T>(L, u[src].p[0], d, M, svf_levels, st);
        const T* ph = svf_levels + 3 * n * M;
        const CPlanes3<T> phi{{ph, ph + n, ph + 2 * n}};
        // LNCC at phi = exp(v) through the plane-streaming kernels where they
        // apply: W, G = M(x + phi), then the moment/coefficient and the dW pass
        const bool tma = loss_kind == DFM_LOSS_LNCC && d.ndim == 3 && !ctx->force_legacy &&
                         cfg->lncc_radius >= 1 && cfg->lncc_radius <= 5 &&
                         tma_supported(d, sizeof(T));
        int np = -1;
        if (tma) {
            launch_warpgrad<T>(L, Ms, d, phi, d, Wb, Gb);
            np = launch_lncc_fwd_tma<T>(L, cfg->lncc_radius, Fs, Wb, d, coef[0], partials, st,
                                        nullptr);
        }
        const bool tma_fwd = np >= 0;
        if (!tma_fwd)
            np = loss_kind_launch_fwd<T>(ctx, loss_kind, cfg->lncc_radius, Fs, Ms, d, d, phi,
                                         coef, grad.w(), partials, st);
        ev_end();
        ev_begin(KC_MON);
        launch_monitor(L, monitor_kind(loss_kind), partials, np, static_cast<double>(n), st,
                       loss, stamp, cfg->conv_window, cfg->conv_tol);
        ev_end();
        if (loss_kind == DFM_LOSS_LNCC) {
            const T* cc[4] = {coef[0], coef[1], coef[2], coef[3]};
            ev_begin(KC_BWD);
            if (!tma_fwd ||
                launch_lncc_bwd_tma<T>(L, cfg->lncc_radius, coef[0], Fs, Wb, Gb, d, grad.p[0],
                                       st) < 0)
                launch_lncc_bwd<T>(L, cfg->lncc_radius, Fs, Ms, d, d, phi, cc, grad.w(), st);
            ev_end();
        }
        ev_begin(KC_ADAM);
        launch_svf_pullback<T>(L, svf_levels, d, M, grad.p[0], svf_g, svf, st);
        const CPlanes3<T> g{{svf_g, svf_g + n, svf_g + 2 * n}};
        if (big_g)
            for (int c = 0; c < 3; ++c)
                axis_smooth_plane<T>(ctx, d, *big_g, svf_g + c * n, svf_g + c * n, step.p[c], st);
        AdamParams ap{cfg->beta1, cfg->beta2, cfg->eps_adam, cfg->eta, cfg->step_cap,
                      corr1, corr2, 0};
        if (!tma || big_g ||
            launch_smooth_adam_tma<T>(L, Rg, wg, svf_g, m.p[0], nu.p[0], step.p[0], d, ap, st,
                                      maxstep) < 0)
            launch_smooth_adam<T>(L, big_g ? 0 : Rg, wg, g, u[src].r(), m.w(), nu.w(), step.w(),
                                  d, ap, st, maxstep);
        ev_end();
        ev_begin(KC_COMPOSE);
        if (!tma || big_w ||
            launch_svf_update_tma<T>(L, Rw, ww, u[src].p[0], step.p[0], u[1 - src].p[0], d, st) < 0)
            launch_svf_update<T>(L, big_w ? 0 : Rw, ww, u[src].r(), step.r(), u[1 - src].w(), d,
                                 st);
        if (big_w)
            for (int c = 0; c < 3; ++c)
                axis_smooth_plane<T>(ctx, d, *big_w, u[1 - src].p[c], u[1 - src].p[c], grad.p[c],
                                     st);
        ev_end();
    }

    // one iteration of the hot loop on grid d, u[src] -> u[1-src]
    void enqueue_iteration(const Dims& d, int src, int Rg, int Rw, const GaussW<T>& wg,
                           const GaussW<T>& ww, const DevAxisGauss* big_g,
                           const DevAxisGauss* big_w) {
        if (cfg->mode == DFM_MODE_SVF) {
            enqueue_iteration_svf(d, src, Rg, Rw, wg, ww, big_g, big_w);
            return;
        }
        if (use_tma) {
            enqueue_iteration_tma(d, src, Rg, Rw, wg, ww);
            return;
        }
        Launch L = ctx->L();
        const int loss_kind = cfg->loss;
        const CPlanes3<T> uin = u[src].r();
        ev_begin(KC_FWD);
        const int np = loss_kind_launch_fwd<T>(ctx, loss_kind, cfg->lncc_radius, Fs, Ms, d, d,
                                               uin, coef, grad.w(), partials, st);
        ev_end();
        ev_begin(KC_MON);
        launch_monitor(L, monitor_kind(loss_kind), partials, np, static_cast<double>(d.n), st,
                       loss, stamp, cfg->conv_window, cfg->conv_tol);
        ev_end();
        if (loss_kind == DFM_LOSS_LNCC) {
            const T* cc[4] = {coef[0], coef[1], coef[2], coef[3]};
            ev_begin(KC_BWD);
            launch_lncc_bwd<T>(L, cfg->lncc_radius, Fs, Ms, d, d, uin, cc, grad.w(), st);
            ev_end();
        } else if (loss_kind == DFM_LOSS_DICE) {
            ev_begin(KC_BWD);
            launch_dice_grad<T>(L, Fs, Ms, d, d, uin, grad.w(), st, 0.0, 1.0);
            ev_end();
        }
        AdamParams ap{cfg->beta1, cfg->beta2, cfg->eps_adam, cfg->eta, cfg->step_cap,
                      corr1, corr2, cfg->use_jac};
        ev_begin(KC_ADAM);
        if (big_g)  // sigma_grad beyond the fused radius: generic axis passes first
            for (int c = 0; c < 3; ++c)
                axis_smooth_plane<T>(ctx, d, *big_g, grad.p[c], grad.p[c], step.p[c], st);
        launch_smooth_adam<T>(L, big_g ? 0 : Rg, wg, grad.r(), uin, m.w(), nu.w(), step.w(), d,
                              ap, st, maxstep);
        ev_end();
        ev_begin(KC_COMPOSE);
        launch_compose_smooth<T>(L, big_w ? 0 : Rw, ww, step.r(), uin, u[1 - src].w(), d, st);
        if (big_w)
            for (int c = 0; c < 3; ++c)
                axis_smooth_plane<T>(ctx, d, *big_w, u[1 - src].p[c], u[1 - src].p[c], grad.p[c],
                                     st);
        ev_end();
    }

    void run(const T* F, const T* M, const double* scales, const int32_t* iters, int ns,
             const dfm_init* init, RegOut& out) {
        Nvtx range("register_images %s %dx%dx%d, %d levels", sizeof(T) == 4 ? "f32" : "f64",
                   full.nx, full.ny, full.nz, ns);
        const double t0 = now_ms();
        int64_t total = 0;
        for (int i = 0; i < ns; ++i) total += iters[i];
        alloc(total);
        Launch L = ctx->L();
        Dims cd{};  // current working grid
        bool have = false;
        int64_t global = 0;
        for (int si = 0; si < ns; ++si) {
            const double fac[3] = {scales[si], scales[si], scales[si]};
            dfm_grid wgd;
            downsample_grid(g, fac, &wgd);
            const Dims d = to_dims(&wgd);
            Nvtx lrange("level %d (scale %g): %dx%dx%d, %d iterations", si, scales[si], d.nx, d.ny,
                        d.nz, iters[si]);
            ev_begin(KC_PYR);
            bool blur = false;
            for (int a = 0; a < g->ndim; ++a) blur |= fac[a] > 1.0;
            const T* Fw = F;
            const T* Mw = M;
            if (blur || !dims_equal(d, full)) {
                Impl<T>{ctx}.downsample_dev(full, F, fac, d, Fbuf, "pyr");
                Impl<T>{ctx}.downsample_dev(full, M, fac, d, Mbuf, "pyr");
                Fw = Fbuf;
                Mw = Mbuf;
            }
            if (!have) {
                layout_all(d.n);
                init_field(d, init);
                zero_field(m, d.n);
                zero_field(nu, d.n);
                have = true;
            } else if (!dims_equal(cd, d)) {
                upsample_state(cd, d);
                layout_all(d.n);
            }
            ev_end();
            cd = d;
            const int T_si = iters[si];
            if (T_si == 0) continue;
            check_loss_inputs(Fw, Mw, &wgd);
            run_scale(d, Fw, Mw, si, scales[si], T_si, global, out);
        }
        // epilogue (pipeline.cpp:213-223)
        Nvtx erange("epilogue: full-resolution loss + fold check");
        ev_begin(KC_EPI);
        if (!dims_equal(cd, full)) {
            upsample_field_only(cd, full);
        }
        Dims d = full;
        if (cfg->mode == DFM_MODE_SVF) {  // pipeline.cpp:214-215: phi = exp(v)
            launch_exp_map<T>(L, u[cur].p[0], d, cfg->svf_M, svf_levels);
            relayout(u[1 - cur], d.n);
            CK(cudaMemcpyAsync(u[1 - cur].p[0], svf_levels + 3 * d.n * cfg->svf_M,
                               sizeof(T) * 3 * d.n, cudaMemcpyDeviceToDevice, ctx->stream));
            cur = 1 - cur;
        }
        if (on_final) on_final(u[cur].r());
        T* coef0[4] = {nullptr, nullptr, nullptr, nullptr};
        check_loss_inputs(F, M, g);
        int np = -1;
        if (w_final && dims_equal(w_dims, full) && dims_equal(cd, full) && d.ndim == 3 &&
            !use_brick && tma_supported(d, sizeof(T))) {
            // the last level ran at full resolution on the streaming loop: its W is
            // M(x+u) for the final field and fstat holds F's window statistics, so
            // the value is one 3-moment forward (same coefficients as the 5-moment
            // form, loop_ops.cuh)
            np = launch_lncc_fwd3_tma<T>(L, cfg->lncc_radius, F, Wb, fstat, d, coef[0], partials,
                                         nullptr, nullptr);
        }
        if (np < 0 && cfg->loss == DFM_LOSS_LNCC && cfg->lncc_radius <= 5 && d.ndim == 3 &&
            tma_supported(d, sizeof(T))) {
            // value only through the plane-streaming forward: W = M(x+u), then moments
            launch_warpgrad<T>(L, M, d, u[cur].r(), d, Wb, nullptr);
            np = launch_lncc_fwd_tma<T>(L, cfg->lncc_radius, F, Wb, d, nullptr, partials,
                                        nullptr);
        }
        if (np < 0)
            np = loss_kind_launch_fwd<T>(ctx, cfg->loss, cfg->lncc_radius, F, M, d, d,
                                         u[cur].r(), coef0,
                                         Planes3<T>{{nullptr, nullptr, nullptr}}, partials,
                                         nullptr);
        double* val = ctx->arr<double>("reg_value3", 4);
        launch_reduce_value(L, monitor_kind(cfg->loss), partials, np, static_cast<double>(d.n),
                            val);
        auto* cnt = ctx->arr<unsigned long long>("reg_count", 1);
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
        launch_jacobian_det<T>(L, u[cur].r(), d, nullptr, cnt);
        ev_end();
        double hv[3];
        unsigned long long hc = 0;
        CK(cudaMemcpyAsync(hv, val, sizeof(hv), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        ev_collect(full);
        consume_logs(global, out);
        out.final_loss = hv[0];
        out.sing = static_cast<double>(hc) / static_cast<double>(d.n);
        out.total_ms = now_ms() - t0;
    }

    // per-evaluation validation of lncc_eval / dice_soft_eval (similarity.cpp:108-114,194-200)
    void check_loss_inputs(const T* F, const T* M, const dfm_grid* wg) {
        if (cfg->loss == DFM_LOSS_LNCC)
            for (int a = 0; a < wg->ndim; ++a)
                if (2 * static_cast<int64_t>(cfg->lncc_radius) + 1 > wg->dims[a])
                    fail(DFM_E_INVALID, "lncc_eval: window larger than image");
        if (cfg->loss == DFM_LOSS_DICE) check_masks(F, M, to_dims(wg));
    }

    void check_masks(const T* F, const T* M, const Dims& d) {
        int* bad = ctx->arr<int>("reg_maskflag", 2);
        CK(cudaMemsetAsync(bad, 0, 2 * sizeof(int), ctx->stream));
        launch_range_check<T>(ctx->L(), F, d.n, bad);
        launch_range_check<T>(ctx->L(), M, d.n, bad + 1);
        int hb[2];
        CK(cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        if (hb[0]) fail(DFM_E_INVALID, "dice_soft_eval: fixed mask values outside [0,1]");
        if (hb[1]) fail(DFM_E_INVALID, "dice_soft_eval: moving mask values outside [0,1]");
    }

    // pipeline.cpp:57-79 initial_field on the coarsest grid
    void init_field(const Dims& d, const dfm_init* init) {
        cur = 0;
        if (!init || init->kind == DFM_INIT_NONE) {
            zero_field(u[0], d.n);
            return;
        }
        if (init->kind == DFM_INIT_AFFINE) {
            if (init->affine_ndim != d.ndim)
                fail(DFM_E_INVALID, "affine_to_working_field: dimensionality mismatch");
            double S[3] = {1.0, 1.0, 1.0};
            const int wd[3] = {d.nx, d.ny, d.nz};
            for (int a = 0; a < d.ndim; ++a) {
                const int den = wd[a] - 1 > 1 ? wd[a] - 1 : 1;
                S[a] = static_cast<double>(g->dims[a] - 1) / static_cast<double>(den);
            }
            launch_affine_field<T>(ctx->L(), init->A, init->t, S, d, u[0].w());
            return;
        }
        if (init->kind != DFM_INIT_FIELD) fail(DFM_E_INVALID, "unknown init kind");
        const dfm_grid* fg = &init->field_grid;
        if (fg->ndim != d.ndim)
            fail(DFM_E_INVALID, "register_images: init field dimensionality mismatch");
        const Dims id = to_dims(fg);
        if (dims_equal(id, d)) {
            upload_field<T>(ctx, init->field, d.n, d.ndim, u[0]);
            return;
        }
        if (!dims_equal(id, full))
            fail(DFM_E_INVALID, "register_images: init field must live on the full or coarsest grid");
        // resample_displacement from the full grid (interp.cpp:447-465)
        relayout(u[1], id.n);
        upload_field<T>(ctx, init->field, id.n, id.ndim, u[1]);
        double mult[3] = {1.0, 1.0, 1.0};
        const int nn[3] = {d.nx, d.ny, d.nz}, no[3] = {id.nx, id.ny, id.nz};
        for (int a = 0; a < d.ndim; ++a)
            mult[a] = static_cast<double>(nn[a] - 1) / static_cast<double>(no[a] - 1);
        const T* src[3] = {u[1].p[0], u[1].p[1], u[1].p[2]};
        T* dst[3] = {u[0].p[0], u[0].p[1], u[0].p[2]};
        launch_resample<T>(ctx->L(), src, id, dst, d, d.ndim, mult);
        relayout(u[1], d.n);
    }

    // Field planes are packed at the current scale's voxel count (the TMA maps
    // and the fused kernels address component k at base + k*n).
    static void relayout(Field<T>& f, int64_t n) {
        f.p[1] = f.p[0] + n;
        f.p[2] = f.p[0] + 2 * n;
    }
    // re-pack the buffers that carry no state across the scale change
    void layout_all(int64_t n) {
        relayout(u[1 - cur], n);
        relayout(grad, n);
        relayout(step, n);
        if (cur == 0 && u[0].p[1] != u[0].p[0] + n) relayout(u[0], n);
        if (m.p[1] != m.p[0] + n) relayout(m, n);
        if (nu.p[1] != nu.p[0] + n) relayout(nu, n);
        for (int k = 1; k < 4; ++k) coef[k] = coef[0] + k * n;
    }

    void upsample_field_only(const Dims& from, const Dims& to) {
        relayout(u[1 - cur], to.n);
        double mult[3] = {1.0, 1.0, 1.0};
        const int nn[3] = {to.nx, to.ny, to.nz}, no[3] = {from.nx, from.ny, from.nz};
        for (int a = 0; a < to.ndim; ++a)
            mult[a] = static_cast<double>(nn[a] - 1) / static_cast<double>(no[a] - 1);
        const T* src[3] = {u[cur].p[0], u[cur].p[1], u[cur].p[2]};
        T* dst[3] = {u[1 - cur].p[0], u[1 - cur].p[1], u[1 - cur].p[2]};
        launch_resample<T>(ctx->L(), src, from, dst, to, to.ndim, mult);
        cur = 1 - cur;
    }

    // upsample_field + upsample_state (pipeline.cpp:150-153, optim.cpp:59-85):
    // the field and both Adam moments in one resampling pass (one cell
    // location per voxel for 3 x ndim components)
    void upsample_state(const Dims& from, const Dims& to) {
        relayout(u[1 - cur], to.n);
        relayout(grad, to.n);
        relayout(step, to.n);
        double mu[3] = {1.0, 1.0, 1.0}, mm[3] = {1.0, 1.0, 1.0}, mn[3] = {1.0, 1.0, 1.0};
        const int nn[3] = {to.nx, to.ny, to.nz}, no[3] = {from.nx, from.ny, from.nz};
        for (int a = 0; a < to.ndim; ++a) {
            const double r = static_cast<double>(nn[a] - 1) / static_cast<double>(no[a] - 1);
            mu[a] = r;
            mm[a] = r;
            mn[a] = r * r;
        }
        const int nd = to.ndim;
        const T* src[9];
        T* dst[9];
        double mult[9];
        for (int a = 0; a < nd; ++a) {
            src[a] = u[cur].p[a];
            dst[a] = u[1 - cur].p[a];
            mult[a] = mu[a];
            src[nd + a] = m.p[a];
            dst[nd + a] = grad.p[a];
            mult[nd + a] = mm[a];
            src[2 * nd + a] = nu.p[a];
            dst[2 * nd + a] = step.p[a];
            mult[2 * nd + a] = mn[a];
        }
        launch_resample<T>(ctx->L(), src, from, dst, to, 3 * nd, mult);
        cur = 1 - cur;
        std::swap(m, grad);
        std::swap(nu, step);
    }

    void run_scale(const Dims& d, const T* Fw, const T* Mw, int si, double scale, int T_si,
                   int64_t& global, RegOut& out) {
        Nvtx range("loop: %d iterations at %dx%dx%d", T_si, d.nx, d.ny, d.nz);
        Fs = const_cast<T*>(Fw);
        Ms = const_cast<T*>(Mw);
        // per-scale reset of the loop state (t is kept)
        CK(cudaMemsetAsync(st, 0, offsetof(LoopState, t), ctx->stream));
        CK(cudaMemsetAsync(maxstep, 0, sizeof(unsigned long long) * (T_si + 1), ctx->stream));
        const double sg[3] = {cfg->sigma_grad, cfg->sigma_grad, cfg->sigma_grad};
        const double sw[3] = {cfg->sigma_warp, cfg->sigma_warp, cfg->sigma_warp};
        const HostGauss hg = make_gauss(d, sg), hw = make_gauss(d, sw);
        GaussW<T> wg = upload_gauss<T>(ctx, hg, d, "loop_g");
        GaussW<T> ww = upload_gauss<T>(ctx, hw, d, "loop_w");
        {
            const double zero[3] = {0, 0, 0};
            w_id = upload_gauss<T>(ctx, make_gauss(d, zero), d, "loop_id");
        }
        DevAxisGauss bg{}, bw{};
        const DevAxisGauss* pbg = nullptr;
        const DevAxisGauss* pbw = nullptr;
        if (hg.R > kRMax) {
            bg = upload_axis_gauss(ctx, hg, d, "loop_bg");
            pbg = &bg;
            const double zero[3] = {0, 0, 0};
            wg = upload_gauss<T>(ctx, make_gauss(d, zero), d, "loop_g0");
        }
        if (hw.R > kRMax) {
            bw = upload_axis_gauss(ctx, hw, d, "loop_bw");
            pbw = &bw;
            const double zero[3] = {0, 0, 0};
            ww = upload_gauss<T>(ctx, make_gauss(d, zero), d, "loop_w0");
        }
        const int Rg = hg.R > kRMax ? 0 : hg.R;
        const int Rw = hw.R > kRMax ? 0 : hw.R;
        const int start = cur;
        const bool big = pbg || pbw;
        const bool direct = cfg->mode == DFM_MODE_DIRECT;
        use_brick = direct && !ctx->force_legacy && !big && !cfg->use_jac && d.n <= ctx->brick_max &&
                    brick_supported(d, static_cast<int>(sizeof(T)),
                                    cfg->loss == DFM_LOSS_LNCC ? cfg->lncc_radius : 1, Rg, Rw);
        use_tma = use_brick || (direct && !ctx->force_legacy && tma_eligible(d, Rg, Rw, big));
        if (use_tma && cfg->loss == DFM_LOSS_LNCC)
            launch_warpgrad<T>(ctx->L(), Ms, d, u[cur].r(), d, Wb, Gb);
        fstat_ready = false;
        if (use_tma && fstat && (ctx->tma_mask & 1))
            fstat_ready = (use_brick ? launch_fstats_brick<T>(ctx->L(), cfg->lncc_radius, Fs, d,
                                                              fstat)
                                     : launch_fstats_tma<T>(ctx->L(), cfg->lncc_radius, Fs, d,
                                                            fstat)) >= 0;
        bool persisted = false;
        if (!ctx->profiling && ctx->persist && use_brick && cfg->loss == DFM_LOSS_LNCC) {
            PersistScale<T> ps{};
            ps.d = d;
            ps.lncc_r = cfg->lncc_radius;
            ps.rg = Rg;
            ps.rw = Rw;
            ps.F = Fs;
            ps.M = Ms;
            ps.W = Wb;
            ps.G = Gb;
            ps.coef = coef[0];
            ps.grad = grad.p[0];
            ps.m = m.p[0];
            ps.nu = nu.p[0];
            ps.step = step.p[0];
            ps.u0 = u[start].p[0];
            ps.u1 = u[1 - start].p[0];
            ps.wg = wg;
            ps.ww = ww;
            ps.ap = AdamParams{cfg->beta1, cfg->beta2, cfg->eps_adam, cfg->eta, cfg->step_cap,
                               corr1, corr2, cfg->use_jac};
            ps.st = st;
            ps.partials = partials;
            ps.loss = loss;
            ps.stamp = stamp;
            ps.maxstep = maxstep;
            ps.window = cfg->conv_window;
            ps.tol = cfg->conv_tol;
            ps.iters = T_si;
            if (ctx->persist >= 2 && fstat_ready) {
                ps.nb_any_size = ctx->persist == 3;
                const int words = persist_nb_sync_words(d, T_si);
                unsigned* sync = ctx->arr<unsigned>("nb_sync", words);
                CK(cudaMemsetAsync(sync, 0, sizeof(unsigned) * words, ctx->stream));
                ps.sync = sync;
                ps.fstat = fstat;
                ps.partials = ctx->arr<double>("nb_partials", int64_t(T_si) * words);
                persisted = launch_persist_nb_scale<T>(ctx->L(), ps) >= 0;
            } else {
                persisted = launch_persist_scale<T>(ctx->L(), ps) >= 0;
            }
            if (persisted) launch_stamp(ctx->L(), stamp + T_si);
        }
        if (persisted) {
        } else if (ctx->profiling) {
            for (int j = 0; j < T_si; ++j)
                enqueue_iteration(d, (start + j) % 2, Rg, Rw, wg, ww, pbg, pbw);
            launch_stamp(ctx->L(), stamp + T_si);
            ev_collect(d);
        } else {
            // capture the two ping-pong variants of one iteration as CUDA graphs,
            // and G consecutive iterations (G even, alternating variants) as one
            // graph: one graph launch per G iterations (the gap between graph
            // launches exceeds the gap between kernels inside a graph)
            static const int G = [] {
                const char* e = getenv("DFM_GRAPH_ITERS");
                const int g = e ? atoi(e) : 8;
                return g >= 2 ? g & ~1 : 0;
            }();
            ctx->trim_graphs();
            cudaGraphExec_t exec[2] = {nullptr, nullptr}, exec_g = nullptr;
            uint64_t sig = 1469598103934665603ull;  // FNV-1a over the level's structure
            auto mix = [&sig](const void* p, size_t nbytes) {
                const unsigned char* b = static_cast<const unsigned char*>(p);
                for (size_t k = 0; k < nbytes; ++k) sig = (sig ^ b[k]) * 1099511628211ull;
            };
            {
                const int64_t parts[] = {si, d.nx, d.ny, d.nz, d.ndim, Rg, Rw, use_brick, use_tma,
                                         fstat_ready, pbg != nullptr, pbw != nullptr, G,
                                         ctx->prec, ctx->brick_max, ctx->split_compose,
                                         ctx->split3, ctx->split_fold_max, ctx->large_min,
                                         ctx->pdl, ctx->tma_mask, ctx->fwd3,
                                         ctx->force_legacy, ctx->narrow};
                mix(parts, sizeof(parts));
                // config fields that select kernels (scalars such as eta or the
                // betas are kernel parameters: an update carries them)
                const int64_t cparts[] = {cfg->loss, cfg->lncc_radius, cfg->use_jac, cfg->mode,
                                          cfg->svf_M, cfg->step_cap <= 0.5 ? 1 : (cfg->step_cap <= 1.5 ? 2 : 3)};
                mix(cparts, sizeof(cparts));
            }
            int64_t nodes_per = 0;
            for (int v = 0; v < 3; ++v) {
                if (v == 2 && (G == 0 || T_si < G)) break;
                const int64_t before = ctx->launches;
                cudaGraph_t graph;
                CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
                if (v < 2) {
                    enqueue_iteration(d, (start + v) % 2, Rg, Rw, wg, ww, pbg, pbw);
                } else {
                    for (int k = 0; k < G; ++k)
                        enqueue_iteration(d, (start + k) % 2, Rg, Rw, wg, ww, pbg, pbw);
                }
                CK(cudaStreamEndCapture(ctx->stream, &graph));
                if (v < 2) {
                    exec[v] = ctx->graph_exec(sig * 4 + v, graph);
                    nodes_per = ctx->launches - before;
                } else {
                    exec_g = ctx->graph_exec(sig * 4 + 2, graph);
                }
                CK(cudaGraphDestroy(graph));
                ctx->launches = before;
            }
            // Launch in chunks, keeping at most two chunks in flight, and stop
            // once the device-side monitor reports the scale done (converged or
            // failed): no per-iteration host sync, bounded wasted launches.
            LoopState* hst = ctx->pinned_state();
            const int chunk = 16;
            int nchunk = 0;
            for (int j = 0; j < T_si;) {
                if (nchunk >= 2) {
                    const int w = (nchunk - 2) % 2;
                    CK(cudaEventSynchronize(ctx->chunk_ev[w]));
                    if (hst[w].done) break;
                }
                const int jend = j + chunk < T_si ? j + chunk : T_si;
                while (j < jend) {
                    if (exec_g && j % 2 == 0 && j + G <= T_si) {  // G even: parity kept
                        CK(cudaGraphLaunch(exec_g, ctx->stream));
                        ctx->launches += G * nodes_per;
                        j += G;
                    } else {
                        CK(cudaGraphLaunch(exec[j % 2], ctx->stream));
                        ctx->launches += nodes_per;
                        ++j;
                    }
                }
                const int w = nchunk % 2;
                CK(cudaMemcpyAsync(&hst[w], st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                                   ctx->stream));
                CK(cudaEventRecord(ctx->chunk_ev[w], ctx->stream));
                ++nchunk;
            }
            launch_stamp(ctx->L(), stamp + T_si);
            // no sync: the execs stay in ctx->graph_cache for the next call, the
            // scale's log leaves through pinned copies below
        }
        // the scale's log leaves through stream-ordered copies into pinned
        // per-level buffers and is read after the registration's last sync: no
        // host round trip between levels (the host prepares the next level while
        // the device finishes this one).  The field's buffer parity after an
        // early stop is settled on the device.
        LevelLog lg;
        lg.si = si;
        lg.scale = scale;
        lg.T_si = T_si;
        const std::string key = "lvl" + std::to_string(si) + "_";
        lg.hs = static_cast<LoopState*>(ctx->get_pinned(key + "st", sizeof(LoopState)));
        lg.hl = static_cast<double*>(ctx->get_pinned(key + "loss", sizeof(double) * (T_si + 1)));
        lg.hm = static_cast<unsigned long long*>(
            ctx->get_pinned(key + "max", sizeof(unsigned long long) * (T_si + 1)));
        lg.ht = static_cast<unsigned long long*>(
            ctx->get_pinned(key + "stamp", sizeof(unsigned long long) * (T_si + 1)));
        CK(cudaMemcpyAsync(lg.hs, st, sizeof(LoopState), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(lg.hl, loss, sizeof(double) * T_si, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaMemcpyAsync(lg.hm, maxstep, sizeof(unsigned long long) * T_si,
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(lg.ht, stamp, sizeof(unsigned long long) * (T_si + 1),
                           cudaMemcpyDeviceToHost, ctx->stream));
        pending.push_back(lg);
        w_final = use_tma && cfg->mode == DFM_MODE_DIRECT && cfg->loss == DFM_LOSS_LNCC &&
                  fstat_ready;
        w_dims = d;
        const int assumed = (start + T_si) % 2;  // no early stop: T_si updates
        launch_parity_fix<T>(ctx->L(), st, T_si, u[1 - assumed].r(), u[assumed].w(), d.n,
                             d.ndim);
        cur = assumed;
        if (ctx->profiling) {  // per-kernel timing: keep the scale's records in step
            ctx->sync();
            consume_logs(global, out);
        }
    }

    struct LevelLog {
        int si;
        double scale;
        int T_si;
        LoopState* hs;
        double* hl;
        unsigned long long* hm;
        unsigned long long* ht;
    };
    std::vector<LevelLog> pending;

    // records of the finished levels, in order (after a sync); a level's
    // numerical failure raises here, with the reference's messages
    void consume_logs(int64_t& global, RegOut& out) {
        std::vector<LevelLog> logs;
        logs.swap(pending);
        for (const LevelLog& lg : logs) {
            const LoopState& hs = *lg.hs;
            const int nrec = hs.it;
            for (int j = 0; j < nrec; ++j) {
                dfm_iter_record r{};
                r.scale_index = lg.si;
                r.scale = lg.scale;
                r.iter = j;
                r.global_iter = global++;
                r.loss = lg.hl[j];
                const bool conv_rec = hs.converged && j == nrec - 1;
                double ms;
                std::memcpy(&ms, &lg.hm[j], sizeof(double));
                r.max_step = conv_rec ? 0.0 : ms;
                const unsigned long long tn = (j + 1 < nrec) ? lg.ht[j + 1] : lg.ht[lg.T_si];
                r.wall_ms = tn > lg.ht[j] ? static_cast<double>(tn - lg.ht[j]) * 1e-6 : 0.0;
                if (hs.err && j == nrec - 1 && !std::isfinite(lg.hl[j])) break;  // not recorded
                out.recs.push_back(r);
            }
            if (hs.err == 4)  // a neighbour wait of the persistent solver timed out
                fail(DFM_E_CUDA, "register_images: persistent level solver stalled");
            if (hs.err) {
                if (nrec > 0 && !std::isfinite(lg.hl[nrec - 1]))
                    fail(DFM_E_NUMERICAL,
                         "register_images: non-finite loss at scale %f, iteration %d", lg.scale,
                         nrec - 1);
                fail(DFM_E_NUMERICAL, "apply_update: non-finite step");
            }
        }
    }
};

template <class T>
void register_dev(dfm_ctx* ctx, const dfm_grid* g, const T* F, const T* M, const dfm_config* cfg,
                  const double* scales, const int32_t* iters, int ns, const dfm_init* init,
                  RegOut& out, CPlanes3<T>* result,
                  std::function<void(CPlanes3<T>)> on_final = {}) {
    Registrar<T> R{};
    R.on_final = std::move(on_final);
    R.ctx = ctx;
    R.g = g;
    R.cfg = cfg;
    R.full = to_dims(g);
    R.run(F, M, scales, iters, ns, init, out);
    if (result) *result = R.u[R.cur].r();
}

// DFM_OPT_EXACT: register_images through kernels_exact.cu; F, M full-resolution
// device doubles; the AoS field stays in the context buffer "exact_field"
double* run_exact(dfm_ctx* ctx, const dfm_grid* g, const double* F, const double* M,
                  const dfm_config* cfg, const double* scales, const int32_t* iters, int ns,
                  const dfm_init* init, RegOut& out) {
    const double t0 = now_ms();
    for (int i = 0; i < ns; ++i) {  // core.cpp:58-74 grid checks, as the tuned path
        const double fac[3] = {scales[i], scales[i], scales[i]};
        dfm_grid wgd;
        downsample_grid(g, fac, &wgd);
    }
    const int64_t n = g->dims[0] * g->dims[1] * g->dims[2];
    double* field = ctx->arr<double>("exact_field", n * g->ndim);
    std::string msg;
    const int rc = exact_register_status(ctx->stream, &ctx->launches, g, F, M, cfg, scales, iters,
                                         ns, init, field, out.recs, &out.final_loss, &out.sing,
                                         msg);
    if (rc != DFM_OK) fail(rc, "%s", msg.c_str());
    out.total_ms = now_ms() - t0;
    return field;
}

void fill_log(const RegOut& o, dfm_iter_record* records, int64_t max_records, dfm_runlog* log) {
    const int64_t n = static_cast<int64_t>(o.recs.size());
    const int64_t k = n < max_records ? n : max_records;
    if (records && k > 0) std::memcpy(records, o.recs.data(), sizeof(dfm_iter_record) * k);
    if (log) {
        log->n_records = records ? k : 0;
        log->n_total = n;
        log->final_loss = o.final_loss;
        log->final_singularity_fraction = o.sing;
        log->total_ms = o.total_ms;
    }
}

}  // namespace

extern "C" {

dfm_status dfm_validate_config(const dfm_config* c) {
    return guarded([&] { validate_config(c); });
}

dfm_status dfm_validate_schedule(const double* scales, const int32_t* iterations,
                                 int32_t nscales) {
    return guarded([&] { validate_schedule(scales, iterations, nscales); });
}

dfm_status dfm_register(dfm_ctx* ctx, const dfm_grid* g, const void* fixed, const void* moving,
                        int image_dtype, const dfm_config* cfg, const double* scales,
                        const int32_t* iterations, int32_t nscales, const dfm_init* init,
                        void* out_field, int field_dtype, dfm_iter_record* records,
                        int64_t max_records, dfm_runlog* log) {
    return guarded([&] {
        const double t0 = now_ms();
        validate_grid(g);
        validate_config(cfg);
        validate_schedule(scales, iterations, nscales);
        if (image_dtype != DFM_HOST_F32 && image_dtype != DFM_HOST_F64)
            fail(DFM_E_INVALID, "image_dtype must be DFM_HOST_F32 or DFM_HOST_F64");
        const Dims d = to_dims(g);
        RegOut o;
        for (int k = 0; k < DFM_NUM_KCLASS; ++k) ctx->kt_ms[k] = 0, ctx->kt_n[k] = 0, ctx->kt_vox[k] = 0;
        if (ctx && ctx->exact) {
            CK(cudaSetDevice(ctx->device));
            double* F = ctx->arr<double>("host_F", d.n);
            double* M = ctx->arr<double>("host_M", d.n);
            if (image_dtype == DFM_HOST_F32) {
                upload_image<double, float>(ctx, static_cast<const float*>(fixed), d.n, F);
                upload_image<double, float>(ctx, static_cast<const float*>(moving), d.n, M);
            } else {
                upload_image<double, double>(ctx, static_cast<const double*>(fixed), d.n, F);
                upload_image<double, double>(ctx, static_cast<const double*>(moving), d.n, M);
            }
            double* fld = run_exact(ctx, g, F, M, cfg, scales, iterations, nscales, init, o);
            if (out_field) {
                if (field_dtype == DFM_HOST_F32)
                    download_image<double, float>(ctx, fld, d.n * d.ndim,
                                                  static_cast<float*>(out_field));
                else
                    download_image<double, double>(ctx, fld, d.n * d.ndim,
                                                   static_cast<double*>(out_field));
            }
            ctx->sync();
            o.total_ms = now_ms() - t0;
            fill_log(o, records, max_records, log);
            if (o.sing > 0.0)
                fail(DFM_E_NUMERICAL, "register_images: folded warp (det J <= 0 somewhere)");
            return;
        }
        DFM_DISPATCH(ctx, {
            T* F = ctx->arr<T>("host_F", d.n);
            T* M = ctx->arr<T>("host_M", d.n);
            if (image_dtype == DFM_HOST_F32) {
                upload_image<T, float>(ctx, static_cast<const float*>(fixed), d.n, F);
                upload_image<T, float>(ctx, static_cast<const float*>(moving), d.n, M);
            } else {
                upload_image<T, double>(ctx, static_cast<const double*>(fixed), d.n, F);
                upload_image<T, double>(ctx, static_cast<const double*>(moving), d.n, M);
            }
            CPlanes3<T> res;
            // the result leaves for the host on the side stream while the
            // epilogue (full-resolution loss, fold check) runs
            std::function<void(CPlanes3<T>)> hook;
            if (out_field)
                hook = [&](CPlanes3<T> r) {
                    cudaStream_t s2 = ctx->side_stream();
                    CK(cudaEventRecord(ctx->side_ev, ctx->stream));
                    CK(cudaStreamWaitEvent(s2, ctx->side_ev, 0));
                    cudaStream_t s1 = ctx->stream;
                    ctx->stream = s2;  // download_field enqueues on ctx->stream
                    if (field_dtype == DFM_HOST_F32)
                        download_field<T, float>(ctx, r, d.n, d.ndim,
                                                 static_cast<float*>(out_field));
                    else
                        download_field<T, double>(ctx, r, d.n, d.ndim,
                                                  static_cast<double*>(out_field));
                    ctx->stream = s1;
                };
            struct SideJoin {  // the download finishes before we return, error or not
                dfm_ctx* c;
                ~SideJoin() {
                    if (c->side) cudaStreamSynchronize(c->side);
                }
            } join{ctx};
            register_dev<T>(ctx, g, F, M, cfg, scales, iterations, nscales, init, o, &res, hook);
            if (out_field) CK(cudaStreamSynchronize(ctx->side_stream()));
            ctx->sync();
        });
        o.total_ms = now_ms() - t0;
        fill_log(o, records, max_records, log);
        if (cfg->mode == DFM_MODE_DIRECT && o.sing > 0.0)
            fail(DFM_E_NUMERICAL, "register_images: folded warp (det J <= 0 somewhere)");
    });
}

dfm_status dfm_dev_register(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                            const void* d_moving, const dfm_config* cfg, const double* scales,
                            const int32_t* iterations, int32_t nscales, void* d_out_soa_field,
                            dfm_iter_record* records, int64_t max_records, dfm_runlog* log) {
    return guarded([&] {
        validate_grid(g);
        validate_config(cfg);
        validate_schedule(scales, iterations, nscales);
        const Dims d = to_dims(g);
        RegOut o;
        for (int k = 0; k < DFM_NUM_KCLASS; ++k) ctx->kt_ms[k] = 0, ctx->kt_n[k] = 0, ctx->kt_vox[k] = 0;
        if (ctx && ctx->exact) {  // fp64 context: device doubles in, SoA doubles out
            CK(cudaSetDevice(ctx->device));
            double* fld = run_exact(ctx, g, static_cast<const double*>(d_fixed),
                                    static_cast<const double*>(d_moving), cfg, scales, iterations,
                                    nscales, nullptr, o);
            if (d_out_soa_field) {
                double* outp = static_cast<double*>(d_out_soa_field);
                launch_aos_to_soa<double, double>(
                    ctx->L(), fld, Planes3<double>{{outp, outp + d.n, outp + 2 * d.n}}, d.n,
                    d.ndim);
            }
            ctx->sync();
            fill_log(o, records, max_records, log);
            if (o.sing > 0.0)
                fail(DFM_E_NUMERICAL, "register_images: folded warp (det J <= 0 somewhere)");
            return;
        }
        DFM_DISPATCH(ctx, {
            CPlanes3<T> res;
            register_dev<T>(ctx, g, static_cast<const T*>(d_fixed), static_cast<const T*>(d_moving),
                            cfg, scales, iterations, nscales, nullptr, o, &res);
            if (d_out_soa_field) {
                T* outp = static_cast<T*>(d_out_soa_field);
                for (int c = 0; c < 3; ++c)
                    CK(cudaMemcpyAsync(outp + c * d.n, res.c[c], sizeof(T) * d.n,
                                       cudaMemcpyDeviceToDevice, ctx->stream));
            }
            ctx->sync();
        });
        fill_log(o, records, max_records, log);
        if (cfg->mode == DFM_MODE_DIRECT && o.sing > 0.0)
            fail(DFM_E_NUMERICAL, "register_images: folded warp (det J <= 0 somewhere)");
    });
}

}  // extern "C"

// ===========================================================================
// z-slab decomposition of register_images: each slab owns a
// contiguous range of z planes at every scale plus H halo planes on each
// side; the plane-streaming kernels run on slab views (Dims::zoff/gnz/zb/ze)
// and halo planes are exchanged after each producing stage — by device copies
// between emulated slabs on one GPU, or by NCCL send/recv between processes.

#include <dlfcn.h>
#include <nccl.h>

namespace {

// NCCL resolved at run time from the libnccl.so.2 already in the process (torch
// bundles one) or the system one; the library does not link NCCL.
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    void load() {
        if (h) return;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) fail(DFM_E_CUDA, "NCCL: cannot dlopen libnccl.so.2");
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) fail(DFM_E_CUDA, "NCCL: missing symbol %s", n);
            return p;
        };
        GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
        CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
        Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
        Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
        AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
        Broadcast = reinterpret_cast<decltype(Broadcast)>(sym("ncclBroadcast"));
        GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
        GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    }
    void ck(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess) fail(DFM_E_CUDA, "NCCL %s: %s", what, GetErrorString(r));
    }
};

NcclApi& nccl_api() {
    static NcclApi api;
    return api;
}

struct SlabBounds {
    int zlo, zhi, hlo, hhi;
    int owned() const { return zhi - zlo; }
    int z0g() const { return zlo - hlo; }
    int nzl() const { return hlo + owned() + hhi; }
};

SlabBounds slab_bounds(int nz, int part, int nparts, int H) {
    SlabBounds b;
    b.zlo = static_cast<int>(static_cast<int64_t>(part) * nz / nparts);
    b.zhi = static_cast<int>(static_cast<int64_t>(part + 1) * nz / nparts);
    b.hlo = std::min(H, b.zlo);
    b.hhi = std::min(H, nz - b.zhi);
    return b;
}

// halo depth: LNCC window r, sigma_grad radius, sigma_warp radius + gather
// reach of the capped compose (the u halo the compose kernel reads)
int slab_halo(const dfm_config* c) {
    const int rg = c->sigma_grad > 0 ? static_cast<int>(std::ceil(3.0 * c->sigma_grad)) : 0;
    const int rw = c->sigma_warp > 0 ? static_cast<int>(std::ceil(3.0 * c->sigma_warp)) : 0;
    const int caph = c->step_cap <= 0.5 ? 1 : 2;
    return std::max(std::max(c->lncc_radius, rg), rw + caph);
}

template <class T>
struct SlabRun;

// The slab loop's collective steps, behind one interface:
//   exchange  halo planes of a buffer with the z neighbours;
//   gather    every slab's owned planes of (u, m, nu) -> full volumes (scale
//             changes: the next level is resampled from them);
//   sum/max   global reductions of device scalars (loss partials, the
//             non-finite-step flag, the max-step log, the fold count).
// Three implementations: emulated slabs in one process (device copies),
// NCCL between processes (device-side, inside the captured graphs), and a
// caller transport (dfm_slab_transport: host-staged callbacks, eager loop).
template <class T>
struct SlabTransport {
    virtual ~SlabTransport() = default;
    // on stream s (the exchange stream: it overlaps the interior planes)
    virtual void exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t s) = 0;
    virtual void gather(SlabRun<T>& R, const Dims& ds) = 0;
    virtual void sum_f64(SlabRun<T>& R, double* dev, int n) = 0;
    virtual void sum_u64(SlabRun<T>& R, unsigned long long* dev, int n) = 0;
    virtual void max_u64(SlabRun<T>& R, unsigned long long* dev, int n) = 0;
    virtual void max_i32(SlabRun<T>& R, int* dev, int n) = 0;
    virtual bool capturable() const = 0;  // may be recorded into a CUDA graph
};

template <class T>
struct EmulatedTransport final : SlabTransport<T> {
    void exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t s) override;
    void gather(SlabRun<T>& R, const Dims& ds) override;
    void sum_f64(SlabRun<T>&, double*, int) override {}
    void sum_u64(SlabRun<T>&, unsigned long long*, int) override {}
    void max_u64(SlabRun<T>&, unsigned long long*, int) override {}
    void max_i32(SlabRun<T>&, int*, int) override {}
    bool capturable() const override { return true; }
};

template <class T>
struct NcclTransport final : SlabTransport<T> {
    const NcclApi* nc = nullptr;
    ncclComm_t comm = nullptr;
    void exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t s) override;
    void gather(SlabRun<T>& R, const Dims& ds) override;
    void sum_f64(SlabRun<T>& R, double* dev, int n) override;
    void sum_u64(SlabRun<T>& R, unsigned long long* dev, int n) override;
    void max_u64(SlabRun<T>& R, unsigned long long* dev, int n) override;
    void max_i32(SlabRun<T>& R, int* dev, int n) override;
    bool capturable() const override { return true; }
};

template <class T>
struct HostTransport final : SlabTransport<T> {
    const dfm_slab_transport* tp = nullptr;
    void exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t s) override;
    void gather(SlabRun<T>& R, const Dims& ds) override;
    void sum_f64(SlabRun<T>& R, double* dev, int n) override;
    void sum_u64(SlabRun<T>& R, unsigned long long* dev, int n) override;
    void max_u64(SlabRun<T>& R, unsigned long long* dev, int n) override;
    void max_i32(SlabRun<T>& R, int* dev, int n) override;
    bool capturable() const override { return false; }
    void ck(int rc, const char* what) const {
        if (rc != 0) fail(DFM_E_CUDA, "slab transport: %s failed (%d)", what, rc);
    }
};

template <class T>
struct SlabRun {
    dfm_ctx* ctx;
    const dfm_grid* g;
    const dfm_config* cfg;
    Dims full;
    int rank = 0, world = 1, E = 1;  // E local slabs (emulation) or 1 (one per process)
    SlabTransport<T>* tp = nullptr;
    int H = 0;
    // replicated levels: a small (coarse) level runs whole on every rank — one
    // local part, no halo exchange, no collective — until the first level with
    // more than repl_max voxels; from there on the levels are decomposed
    int64_t repl_max = 0;
    bool repl = false;
    int Ea = 1;  // active local parts (E, or 1 on a replicated level)
    int64_t cap = 0;  // elements per component buffer of a part

    struct Part {
        SlabBounds b;
        Dims dl;  // slab view at the current scale
        T* base[10];  // W G coef grad step u0 u1 m nu (F is a view of the pyramid)
        T* W() const { return base[0]; }
        T* G() const { return base[1]; }
        T* coef() const { return base[2]; }
        T* grad() const { return base[3]; }
        T* step() const { return base[4]; }
        T* u(int k) const { return base[5 + k]; }
        T* m() const { return base[7]; }
        T* nu() const { return base[8]; }
        double* fstat = nullptr;  // per-level muF, vF of the owned planes (FStats2)
    };
    std::vector<Part> parts;
    T* Fs = nullptr;
    T* Ms = nullptr;
    T* gath[3] = {nullptr, nullptr, nullptr};  // u, m, nu gathered at the previous scale
    LoopState* st = nullptr;
    double *loss = nullptr, *corr1 = nullptr, *corr2 = nullptr, *partials = nullptr,
           *red = nullptr;
    unsigned long long *maxstep = nullptr, *stamp = nullptr;
    int cur = 0;

    ~SlabRun() {
        if (xs) cudaStreamDestroy(xs);
        for (auto e : xev)
            if (e) cudaEventDestroy(e);
    }

    int nparts() const { return repl ? 1 : (world > 1 ? world : E); }
    int part_id(int j) const { return repl ? 0 : (world > 1 ? rank : j); }
    bool collective() const { return world > 1 && !repl; }
    struct Active {  // the active parts, for range-for
        Part* b;
        Part* e;
        Part* begin() const { return b; }
        Part* end() const { return e; }
    };
    Active active() { return {parts.data(), parts.data() + Ea}; }
    // plane size of the current slab views (the scale being processed)
    int64_t plane() const { return static_cast<int64_t>(parts.empty() ? full.nx * full.ny
                                                                       : parts[0].dl.nx * parts[0].dl.ny); }

    void alloc(int64_t total_iters, int64_t prev_n) {
        const int64_t pl = static_cast<int64_t>(full.nx) * full.ny;
        // local capacity: the largest owned range at full resolution + 2H
        int maxn = 0;
        for (int j = 0; j < E; ++j) {
            const SlabBounds b = slab_bounds(full.nz, part_id(j), nparts(), H);
            maxn = std::max(maxn, b.nzl());
        }
        cap = pl * maxn;
        parts.resize(E);
        const int comps[9] = {1, 3, 4, 3, 3, 3, 3, 3, 3};
        for (int j = 0; j < E; ++j) {
            for (int k = 0; k < 9; ++k)
                parts[j].base[k] = ctx->arr<T>("slab" + std::to_string(j) + "_" + std::to_string(k),
                                               comps[k] * cap);
            parts[j].fstat = ctx->arr<double>("slab" + std::to_string(j) + "_fstat", 2 * cap);
        }
        Fs = ctx->arr<T>("slab_Fs", full.n);
        Ms = ctx->arr<T>("slab_Ms", full.n);
        for (int k = 0; k < 3; ++k)  // u: also the final gathered field (full grid)
            gath[k] = ctx->arr<T>("slab_gath" + std::to_string(k), 3 * (k == 0 ? full.n : prev_n));
        st = ctx->arr<LoopState>("slab_state", 1);
        const int64_t ni = total_iters + 2;
        loss = ctx->arr<double>("slab_loss", ni);
        maxstep = ctx->arr<unsigned long long>("slab_maxstep", ni);
        stamp = ctx->arr<unsigned long long>("slab_stamp", ni);
        corr1 = ctx->arr<double>("slab_corr1", ni);
        corr2 = ctx->arr<double>("slab_corr2", ni);
        partials = ctx->arr<double>("slab_partials", 3 * 65536);
        red = ctx->arr<double>("slab_red", 4);
        std::vector<double> h1(ni), h2(ni);
        for (int64_t t = 0; t < ni; ++t) {
            h1[t] = 1.0 - std::pow(cfg->beta1, static_cast<double>(t));
            h2[t] = 1.0 - std::pow(cfg->beta2, static_cast<double>(t));
        }
        CK(cudaMemcpyAsync(corr1, h1.data(), sizeof(double) * ni, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(corr2, h2.data(), sizeof(double) * ni, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(st, 0, sizeof(LoopState), ctx->stream));
        ctx->sync();
    }

    // slab views of every part at scale grid ds
    void layout(const Dims& ds) {
        Ea = repl ? 1 : E;
        for (int j = 0; j < Ea; ++j) {
            Part& p = parts[j];
            p.b = slab_bounds(ds.nz, part_id(j), nparts(), H);
            if (p.b.owned() < H && nparts() > 1)
                fail(DFM_E_INVALID, "slab: %d slabs leave fewer than %d planes per slab at nz=%d",
                     nparts(), H, ds.nz);
            Dims& d = p.dl;
            d = ds;
            d.nz = p.b.nzl();
            d.n = static_cast<int64_t>(ds.nx) * ds.ny * d.nz;
            d.zoff = p.b.z0g();
            d.gnz = ds.nz;
            d.zb = p.b.hlo;
            d.ze = p.b.hlo + p.b.owned();
        }
    }

    void exchange(int which, int ncomp) {
        if (!repl) tp->exchange(*this, which, ncomp, ctx->stream);
    }

    // Halo-overlapped stage: `fn(part, j, view)` launches the stage's kernel on
    // a z sub-range of a part.  The planes the neighbours need (H next to each
    // internal face) go first; the exchange of `exch` (buffer index, component
    // count pairs) then runs on the exchange stream while the interior planes
    // are computed; the main stream joins it before the next stage.  Every
    // output plane's arithmetic is independent of the launch split.
    cudaStream_t xs = nullptr;
    cudaEvent_t xev[2] = {nullptr, nullptr};
    bool overlap = false;
    template <class Fn>
    void stage(Fn&& fn, std::initializer_list<std::pair<int, int>> exch) {
        const bool ov = overlap && !repl && tp->capturable() && xs != nullptr;
        int ib[64], ie[64];
        for (int j = 0; j < Ea; ++j) {
            Part& p = parts[j];
            const int lo = p.b.hlo, top = p.b.hlo + p.b.owned();
            ib[j] = lo;
            ie[j] = top;
            if (!ov) continue;
            if (p.b.hlo > 0) {  // a neighbour below reads our first H owned planes
                Dims d = p.dl;
                d.zb = lo;
                d.ze = std::min(lo + H, top);
                fn(p, j, d);
                ib[j] = d.ze;
            }
            if (p.b.hhi > 0 && ib[j] < top) {  // ... and one above our last H
                Dims d = p.dl;
                d.zb = std::max(top - H, ib[j]);
                d.ze = top;
                fn(p, j, d);
                ie[j] = d.zb;
            }
        }
        if (ov) {
            CK(cudaEventRecord(xev[0], ctx->stream));
            CK(cudaStreamWaitEvent(xs, xev[0], 0));
            for (const auto& e : exch) tp->exchange(*this, e.first, e.second, xs);
            CK(cudaEventRecord(xev[1], xs));
        }
        for (int j = 0; j < Ea; ++j) {
            if (ib[j] >= ie[j]) continue;
            Dims d = parts[j].dl;
            d.zb = ib[j];
            d.ze = ie[j];
            fn(parts[j], j, d);
        }
        if (ov) {
            CK(cudaStreamWaitEvent(ctx->stream, xev[1], 0));
        } else {
            for (const auto& e : exch) exchange(e.first, e.second);
        }
    }
    void gather(const Dims& ds) {
        if (repl) {  // every rank holds the whole level
            EmulatedTransport<T>().gather(*this, ds);
            return;
        }
        tp->gather(*this, ds);
    }

    // full volumes at grid from -> every slab's local planes at grid to
    void scatter_resample(const Dims& from, const Dims& to, bool with_state) {
        double mult[3] = {1, 1, 1}, sq[3] = {1, 1, 1};
        const int nn[3] = {to.nx, to.ny, to.nz}, no[3] = {from.nx, from.ny, from.nz};
        for (int a = 0; a < to.ndim; ++a) {
            mult[a] = static_cast<double>(nn[a] - 1) / static_cast<double>(no[a] - 1);
            sq[a] = mult[a] * mult[a];
        }
        for (int j = 0; j < Ea; ++j) {
            Part& p = parts[j];
            Dims dall = p.dl;  // every local plane, halos included
            dall.zb = 0;
            dall.ze = 0;
            const int tgt = 1 - cur;
            const T* su[3] = {gath[0], gath[0] + from.n, gath[0] + 2 * from.n};
            T* du[3] = {p.u(tgt), p.u(tgt) + p.dl.n, p.u(tgt) + 2 * p.dl.n};
            launch_resample<T>(ctx->L(), su, from, du, dall, to.ndim, mult);
            if (with_state) {
                const T* sm[3] = {gath[1], gath[1] + from.n, gath[1] + 2 * from.n};
                T* dm[3] = {p.m(), p.m() + p.dl.n, p.m() + 2 * p.dl.n};
                launch_resample<T>(ctx->L(), sm, from, dm, dall, to.ndim, mult);
                const T* sn[3] = {gath[2], gath[2] + from.n, gath[2] + 2 * from.n};
                T* dn[3] = {p.nu(), p.nu() + p.dl.n, p.nu() + 2 * p.dl.n};
                launch_resample<T>(ctx->L(), sn, from, dn, dall, to.ndim, sq);
            }
        }
        cur = 1 - cur;
    }

    double global_sum(const double* part_sums, int np) {
        // fixed-order device reduction, then (NCCL) a sum over ranks
        launch_reduce_value(ctx->L(), 0, part_sums, np, 1.0, red);
        if (collective()) tp->sum_f64(*this, red, 1);
        double h[3];
        CK(cudaMemcpyAsync(h, red, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        return h[0];
    }

    // one iteration on every local slab: the monolithic loop's large-level
    // kernels (3-moment LNCC forward on the level's F statistics, backward,
    // smooth+Adam, radius-0 compose, compose-smooth + W/G) with the halo of
    // each produced buffer exchanged before its consumer
    void enqueue_iteration(const Dims& ds, int src, int Rg, int Rw, const GaussW<T>& wg,
                           const GaussW<T>& ww, const GaussW<T>& wid) {
        Launch L = ctx->L();
        const int64_t pl = static_cast<int64_t>(ds.nx) * ds.ny;
        const double N = static_cast<double>(ds.n);
        int off = 0;
        stage([&](Part& p, int, const Dims& dv) {
            const int np = launch_lncc_fwd3_tma<T>(L, cfg->lncc_radius, Fs + p.b.z0g() * pl, p.W(),
                                                   p.fstat, dv, p.coef(), partials + off, st,
                                                   nullptr);
            if (np < 0) fail(DFM_E_CUDA, "slab: lncc forward launch failed");
            off += np;
        }, {{2, 4}});  // coefficients
        if (collective()) {
            launch_reduce_value(L, 0, partials, off, 1.0, red);
            tp->sum_f64(*this, red, 1);
            launch_monitor(L, 1, red, 1, N, st, loss, stamp, cfg->conv_window, cfg->conv_tol);
        } else {
            launch_monitor(L, 1, partials, off, N, st, loss, stamp, cfg->conv_window, cfg->conv_tol);
        }
        stage([&](Part& p, int, const Dims& dv) {
            if (launch_lncc_bwd_tma<T>(L, cfg->lncc_radius, p.coef(), Fs + p.b.z0g() * pl, p.W(),
                                       p.G(), dv, p.grad(), st) < 0)
                fail(DFM_E_CUDA, "slab: lncc backward launch failed");
        }, {{3, 3}});  // gradient
        AdamParams ap{cfg->beta1, cfg->beta2, cfg->eps_adam, cfg->eta, cfg->step_cap,
                      corr1, corr2, cfg->use_jac};
        for (Part& p : active())
            if (launch_smooth_adam_tma<T>(L, Rg, wg, p.grad(), p.m(), p.nu(), p.step(), p.dl, ap,
                                          st, maxstep) < 0)
                fail(DFM_E_CUDA, "slab: smooth+Adam launch failed");
        if (collective()) tp->max_i32(*this, &st->bad_step, 1);  // a non-finite step aborts everywhere
        // c = step + u(x + step) on the owned planes (the u halo covers the
        // gather reach), into the dead gradient buffer
        stage([&](Part& p, int, const Dims& dv) {
            if (launch_compose_tma<T>(L, 0, cfg->step_cap, wid, p.step(), p.u(src), p.grad(), Ms, ds,
                                      dv, nullptr, nullptr, st, false) < 0)
                fail(DFM_E_CUDA, "slab: compose launch failed");
        }, {{3, 3}});  // c
        bool counted = false;  // one counted update per iteration (emulated parts, split launches)
        stage([&](Part& p, int, const Dims& dv) {
            if (launch_compose_smooth_tma<T>(L, Rw, ww, p.grad(), p.u(1 - src), Ms, ds, dv, p.W(),
                                             p.G(), st, !counted) < 0)
                fail(DFM_E_CUDA, "slab: compose-smooth launch failed");
            counted = true;
        }, {{6 - src, 3}, {0, 1}});  // u (the buffer just written), W
    }

    void run(const T* F, const T* M, const double* scales, const int32_t* iters, int ns,
             RegOut& out, T* d_out, int64_t* ozlo, int64_t* ozhi) {
        Nvtx range("register_images slab %d/%d (%d local parts) %dx%dx%d", rank, world, E,
                   full.nx, full.ny, full.nz);
        const double t0 = now_ms();
        if (cfg->loss != DFM_LOSS_LNCC || cfg->use_jac || cfg->mode != DFM_MODE_DIRECT)
            fail(DFM_E_INVALID, "slab decomposition: direct mode, LNCC loss, use_jac off only");
        if (cfg->step_cap > 1.5)
            fail(DFM_E_INVALID, "slab decomposition: step_cap <= 1.5 only");
        if (!tma_supported(full, sizeof(T)))
            fail(DFM_E_INVALID, "slab decomposition: x extent must be a multiple of 16 bytes");
        if (full.ndim != 3) fail(DFM_E_INVALID, "slab decomposition: 3-D volumes only");
        H = slab_halo(cfg);
        if (overlap && tp->capturable() && !xs) {
            CK(cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking));
            for (auto& e : xev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        int64_t total = 0;
        for (int i = 0; i < ns; ++i) total += iters[i];
        // m and nu are gathered only when leaving a level that is not the full
        // grid: size their gather buffers for the largest such level
        int64_t prev_n = 1;
        for (int i = 0; i < ns; ++i) {
            const double fac[3] = {scales[i], scales[i], scales[i]};
            dfm_grid wgd;
            downsample_grid(g, fac, &wgd);
            const Dims di = to_dims(&wgd);
            if (!dims_equal(di, full)) prev_n = std::max(prev_n, di.n);
            if (!tma_supported(di, sizeof(T)))
                fail(DFM_E_INVALID,
                     "slab decomposition: the x extent of every pyramid level must be a multiple "
                     "of 16 bytes (level %d has %d voxels)", i, di.nx);
        }
        alloc(total, prev_n);
        Dims prev{};
        bool have = false;
        bool may_repl = true;  // replicated levels only precede the decomposed ones
        int64_t global = 0;
        const int64_t pl = static_cast<int64_t>(full.nx) * full.ny;  // epilogue (full grid)
        for (int si = 0; si < ns; ++si) {
            const double fac[3] = {scales[si], scales[si], scales[si]};
            dfm_grid wgd;
            downsample_grid(g, fac, &wgd);
            const Dims ds = to_dims(&wgd);
            if (2 * static_cast<int64_t>(cfg->lncc_radius) + 1 > ds.nx ||
                2 * static_cast<int64_t>(cfg->lncc_radius) + 1 > ds.ny ||
                2 * static_cast<int64_t>(cfg->lncc_radius) + 1 > ds.nz)
                fail(DFM_E_INVALID, "lncc_eval: window larger than image");
            Impl<T>{ctx}.downsample_dev(full, F, fac, ds, Fs, "spyr");
            Impl<T>{ctx}.downsample_dev(full, M, fac, ds, Ms, "spyr");
            Nvtx lrange("slab level %d (scale %g): %dx%dx%d, %d iterations", si, scales[si], ds.nx,
                        ds.ny, ds.nz, iters[si]);
            const bool want_repl = may_repl && ds.n <= repl_max && ds.n <= cap;
            may_repl = want_repl;
            if (!have) {
                repl = want_repl;
                layout(ds);
                for (Part& p : active())
                    for (int k : {5, 6, 7, 8})
                        CK(cudaMemsetAsync(p.base[k], 0, sizeof(T) * 3 * p.dl.n, ctx->stream));
                cur = 0;
                have = true;
            } else if (!dims_equal(prev, ds)) {
                gather(prev);  // in the previous level's mode
                repl = want_repl;
                layout(ds);
                scatter_resample(prev, ds, true);
            }
            prev = ds;
            const int T_si = iters[si];
            if (T_si == 0) continue;
            for (Part& p : active()) {
                launch_warpgrad<T>(ctx->L(), Ms, ds, CPlanes3<T>{{p.u(cur), p.u(cur) + p.dl.n,
                                                                  p.u(cur) + 2 * p.dl.n}},
                                   [&] { Dims a = p.dl; a.zb = a.ze = 0; return a; }(), p.W(), p.G());
                // the level's F window statistics of the owned planes
                if (launch_fstats_tma<T>(ctx->L(), cfg->lncc_radius, Fs + p.b.z0g() * plane(),
                                         p.dl, p.fstat) < 0)
                    fail(DFM_E_CUDA, "slab: F statistics launch failed");
            }
            CK(cudaMemsetAsync(st, 0, offsetof(LoopState, t), ctx->stream));
            CK(cudaMemsetAsync(maxstep, 0, sizeof(unsigned long long) * (T_si + 1), ctx->stream));
            const double sg[3] = {cfg->sigma_grad, cfg->sigma_grad, cfg->sigma_grad};
            const double sw[3] = {cfg->sigma_warp, cfg->sigma_warp, cfg->sigma_warp};
            const HostGauss hg = make_gauss(ds, sg), hw = make_gauss(ds, sw);
            if (hg.R > 6 || hw.R > 4)
                fail(DFM_E_INVALID, "slab decomposition: sigma_grad <= 2, sigma_warp <= 1.33 only");
            const GaussW<T> wg = upload_gauss<T>(ctx, hg, ds, "slab_g");
            const GaussW<T> ww = upload_gauss<T>(ctx, hw, ds, "slab_w");
            const double zero[3] = {0, 0, 0};
            const GaussW<T> wid = upload_gauss<T>(ctx, make_gauss(ds, zero), ds, "slab_id");
            const int start = cur;
            LoopState* hst = ctx->pinned_state();
            if (tp->capturable()) {
                cudaGraphExec_t exec[2] = {nullptr, nullptr};
                for (int v = 0; v < 2; ++v) {
                    cudaGraph_t graph;
                    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
                    enqueue_iteration(ds, (start + v) % 2, hg.R, hw.R, wg, ww, wid);
                    CK(cudaStreamEndCapture(ctx->stream, &graph));
                    CK(cudaGraphInstantiate(&exec[v], graph, 0));
                    CK(cudaGraphDestroy(graph));
                }
                // every rank launches the same number of graphs (global decisions)
                int nchunk = 0;
                for (int j = 0; j < T_si;) {
                    if (nchunk >= 2) {
                        const int w = (nchunk - 2) % 2;
                        CK(cudaEventSynchronize(ctx->chunk_ev[w]));
                        if (hst[w].done) break;
                    }
                    const int jend = std::min(j + 16, T_si);
                    for (; j < jend; ++j) CK(cudaGraphLaunch(exec[j % 2], ctx->stream));
                    const int w = nchunk % 2;
                    CK(cudaMemcpyAsync(&hst[w], st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                                       ctx->stream));
                    CK(cudaEventRecord(ctx->chunk_ev[w], ctx->stream));
                    ++nchunk;
                }
                ctx->sync();
                for (int v = 0; v < 2; ++v) CK(cudaGraphExecDestroy(exec[v]));
            } else {
                // host-staged transport: eager iterations (its collectives
                // synchronise); the global monitor decides on every rank alike
                for (int j = 0; j < T_si; ++j) {
                    enqueue_iteration(ds, (start + j) % 2, hg.R, hw.R, wg, ww, wid);
                    CK(cudaMemcpyAsync(&hst[0], st, sizeof(LoopState), cudaMemcpyDeviceToHost,
                                       ctx->stream));
                    ctx->sync();
                    if (hst[0].done) break;
                }
            }
            launch_stamp(ctx->L(), stamp + T_si);
            if (collective()) tp->max_u64(*this, maxstep, T_si);  // max |step| of the log over ranks
            ctx->sync();
            LoopState hs;
            std::vector<double> hl(T_si + 1);
            std::vector<unsigned long long> hm(T_si + 1), ht(T_si + 1);
            CK(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(hl.data(), loss, sizeof(double) * T_si, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(hm.data(), maxstep, sizeof(unsigned long long) * T_si,
                               cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(ht.data(), stamp, sizeof(unsigned long long) * (T_si + 1),
                               cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
            const int nrec = hs.it;
            for (int j = 0; j < nrec; ++j) {
                dfm_iter_record r{};
                r.scale_index = si;
                r.scale = scales[si];
                r.iter = j;
                r.global_iter = global++;
                r.loss = hl[j];
                double ms;
                std::memcpy(&ms, &hm[j], sizeof(double));
                r.max_step = (hs.converged && j == nrec - 1) ? 0.0 : ms;
                const unsigned long long tn = (j + 1 < nrec) ? ht[j + 1] : ht[T_si];
                r.wall_ms = tn > ht[j] ? static_cast<double>(tn - ht[j]) * 1e-6 : 0.0;
                if (hs.err && j == nrec - 1 && !std::isfinite(hl[j])) break;
                out.recs.push_back(r);
            }
            if (hs.err) {
                if (nrec > 0 && !std::isfinite(hl[nrec - 1]))
                    fail(DFM_E_NUMERICAL, "register_images: non-finite loss at scale %f, iteration %d",
                         scales[si], nrec - 1);
                fail(DFM_E_NUMERICAL, "apply_update: non-finite step");
            }
            cur = (start + hs.nupdates) % 2;
        }
        // epilogue at full resolution (pipeline.cpp:213-223)
        if (!dims_equal(prev, full)) {
            gather(prev);
            repl = may_repl && full.n <= repl_max && full.n <= cap;
            layout(full);
            scatter_resample(prev, full, false);
        }
        int off = 0;
        for (Part& p : active()) {
            Dims dall = p.dl;
            dall.zb = dall.ze = 0;
            launch_warpgrad<T>(ctx->L(), M, full,
                               CPlanes3<T>{{p.u(cur), p.u(cur) + p.dl.n, p.u(cur) + 2 * p.dl.n}},
                               dall, p.W(), nullptr);
            const int np = launch_lncc_fwd_tma<T>(ctx->L(), cfg->lncc_radius, F + p.b.z0g() * pl, p.W(),
                                                  p.dl, nullptr, partials + off, nullptr);
            off += np;
        }
        const double S = global_sum(partials, off);
        out.final_loss = -S / static_cast<double>(full.n);
        auto* cnt = ctx->arr<unsigned long long>("slab_count", 1);
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), ctx->stream));
        for (Part& p : active())
            launch_jacobian_det<T>(ctx->L(), CPlanes3<T>{{p.u(cur), p.u(cur) + p.dl.n,
                                                          p.u(cur) + 2 * p.dl.n}},
                                   p.dl, nullptr, cnt);
        if (collective()) tp->sum_u64(*this, cnt, 1);
        unsigned long long hc = 0;
        CK(cudaMemcpyAsync(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
        // result planes
        int64_t zlo = parts[0].b.zlo, zhi = parts[Ea - 1].b.zhi;
        const int64_t nout = (zhi - zlo) * pl;
        if (d_out)
            for (Part& p : active())
                for (int c = 0; c < 3; ++c)
                    CK(cudaMemcpyAsync(d_out + c * nout + (p.b.zlo - zlo) * pl,
                                       p.u(cur) + c * p.dl.n + p.b.hlo * pl,
                                       sizeof(T) * pl * p.b.owned(), cudaMemcpyDeviceToDevice,
                                       ctx->stream));
        ctx->sync();
        out.sing = static_cast<double>(hc) / static_cast<double>(full.n);
        out.total_ms = now_ms() - t0;
        if (ozlo) *ozlo = zlo;
        if (ozhi) *ozhi = zhi;
    }
};

// ---- emulated slabs: device copies between the parts of one process
template <class T>
void EmulatedTransport<T>::exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t s) {
    const int64_t pl = R.plane();
    for (int j = 0; j < R.Ea; ++j) {
        auto& p = R.parts[j];
        if (j > 0 && p.b.hlo > 0) {  // lower halo <- part j-1's top owned planes
            const auto& q = R.parts[j - 1];
            const int src_local = p.b.zlo - p.b.hlo - q.b.z0g();
            for (int c = 0; c < ncomp; ++c)
                CK(cudaMemcpyAsync(p.base[which] + c * p.dl.n,
                                   q.base[which] + c * q.dl.n + src_local * pl,
                                   sizeof(T) * pl * p.b.hlo, cudaMemcpyDeviceToDevice,
                                   s));
        }
        if (j + 1 < R.Ea && p.b.hhi > 0) {  // upper halo <- part j+1's bottom owned planes
            const auto& q = R.parts[j + 1];
            const int src_local = p.b.zhi - q.b.z0g();
            const int dst_local = p.b.hlo + p.b.owned();
            for (int c = 0; c < ncomp; ++c)
                CK(cudaMemcpyAsync(p.base[which] + c * p.dl.n + dst_local * pl,
                                   q.base[which] + c * q.dl.n + src_local * pl,
                                   sizeof(T) * pl * p.b.hhi, cudaMemcpyDeviceToDevice,
                                   s));
        }
    }
}

template <class T>
void EmulatedTransport<T>::gather(SlabRun<T>& R, const Dims& ds) {
    const int64_t pl = static_cast<int64_t>(ds.nx) * ds.ny;
    for (int j = 0; j < R.Ea; ++j) {
        const auto& p = R.parts[j];
        const T* srcs[3] = {p.u(R.cur), p.m(), p.nu()};
        for (int f = 0; f < 3; ++f)
            for (int c = 0; c < 3; ++c)
                CK(cudaMemcpyAsync(R.gath[f] + c * ds.n + static_cast<int64_t>(p.b.zlo) * pl,
                                   srcs[f] + c * p.dl.n + p.b.hlo * pl,
                                   sizeof(T) * pl * p.b.owned(), cudaMemcpyDeviceToDevice,
                                   R.ctx->stream));
    }
}

// ---- NCCL between processes (device-side, capturable)
template <class T>
void NcclTransport<T>::exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t s) {
    const int64_t pl = R.plane();
    const auto& p = R.parts[0];
    const ncclDataType_t dt = sizeof(T) == 4 ? ncclFloat32 : ncclFloat64;
    nc->ck(nc->GroupStart(), "group");
    for (int c = 0; c < ncomp; ++c) {
        T* buf = p.base[which] + c * p.dl.n;
        if (R.rank > 0) {  // exchange with the lower neighbour: H planes each way
            nc->ck(nc->Send(buf + p.b.hlo * pl, pl * p.b.hlo, dt, R.rank - 1, comm, s),
                   "send");
            nc->ck(nc->Recv(buf, pl * p.b.hlo, dt, R.rank - 1, comm, s), "recv");
        }
        if (R.rank + 1 < R.world) {
            const int top = p.b.hlo + p.b.owned();
            nc->ck(nc->Send(buf + (top - p.b.hhi) * pl, pl * p.b.hhi, dt, R.rank + 1, comm,
                            s), "send");
            nc->ck(nc->Recv(buf + top * pl, pl * p.b.hhi, dt, R.rank + 1, comm, s),
                   "recv");
        }
    }
    nc->ck(nc->GroupEnd(), "group");
}

template <class T>
void NcclTransport<T>::gather(SlabRun<T>& R, const Dims& ds) {
    const int64_t pl = static_cast<int64_t>(ds.nx) * ds.ny;
    const auto& p = R.parts[0];
    const T* srcs[3] = {p.u(R.cur), p.m(), p.nu()};
    const ncclDataType_t dt = sizeof(T) == 4 ? ncclFloat32 : ncclFloat64;
    nc->ck(nc->GroupStart(), "group");
    for (int r = 0; r < R.world; ++r) {  // every rank broadcasts its owned block to all
        const SlabBounds b = slab_bounds(ds.nz, r, R.world, R.H);
        for (int f = 0; f < 3; ++f)
            for (int c = 0; c < 3; ++c)
                nc->ck(nc->Broadcast(srcs[f] + c * p.dl.n + p.b.hlo * pl,
                                     R.gath[f] + c * ds.n + static_cast<int64_t>(b.zlo) * pl,
                                     pl * b.owned(), dt, r, comm, R.ctx->stream),
                       "broadcast");
    }
    nc->ck(nc->GroupEnd(), "group");
}

template <class T>
void NcclTransport<T>::sum_f64(SlabRun<T>& R, double* dev, int n) {
    nc->ck(nc->AllReduce(dev, dev, n, ncclFloat64, ncclSum, comm, R.ctx->stream), "allreduce");
}
template <class T>
void NcclTransport<T>::sum_u64(SlabRun<T>& R, unsigned long long* dev, int n) {
    nc->ck(nc->AllReduce(dev, dev, n, ncclUint64, ncclSum, comm, R.ctx->stream), "allreduce");
}
template <class T>
void NcclTransport<T>::max_u64(SlabRun<T>& R, unsigned long long* dev, int n) {
    nc->ck(nc->AllReduce(dev, dev, n, ncclUint64, ncclMax, comm, R.ctx->stream), "allreduce");
}
template <class T>
void NcclTransport<T>::max_i32(SlabRun<T>& R, int* dev, int n) {
    nc->ck(nc->AllReduce(dev, dev, n, ncclInt32, ncclMax, comm, R.ctx->stream), "allreduce");
}

// ---- caller transport: host-staged through pinned buffers (eager loop)
template <class T>
void HostTransport<T>::exchange(SlabRun<T>& R, int which, int ncomp, cudaStream_t) {
    const int64_t pl = R.plane();
    const auto& p = R.parts[0];
    const int top = p.b.hlo + p.b.owned();
    struct Side {
        int peer, n;       // neighbour rank, planes each way
        int send0, recv0;  // first local plane sent / received
        const char* name;
    };
    Side sides[2] = {{R.rank - 1, p.b.hlo, p.b.hlo, 0, "lo"},
                     {R.rank + 1, p.b.hhi, top - p.b.hhi, top, "hi"}};
    for (const Side& sd : sides) {
        if (sd.peer < 0 || sd.peer >= R.world || sd.n == 0) continue;
        const int64_t blk = pl * sd.n;  // elements per component
        const int64_t bytes = static_cast<int64_t>(sizeof(T)) * blk * ncomp;
        T* hs = static_cast<T*>(R.ctx->get_pinned(std::string("slab_tx_") + sd.name, bytes));
        T* hr = static_cast<T*>(R.ctx->get_pinned(std::string("slab_rx_") + sd.name, bytes));
        for (int c = 0; c < ncomp; ++c)
            CK(cudaMemcpyAsync(hs + c * blk, p.base[which] + c * p.dl.n + sd.send0 * pl,
                               sizeof(T) * blk, cudaMemcpyDeviceToHost, R.ctx->stream));
        R.ctx->sync();
        ck(tp->sendrecv(tp->user, sd.peer, hs, bytes, hr, bytes), "sendrecv");
        for (int c = 0; c < ncomp; ++c)
            CK(cudaMemcpyAsync(p.base[which] + c * p.dl.n + sd.recv0 * pl, hr + c * blk,
                               sizeof(T) * blk, cudaMemcpyHostToDevice, R.ctx->stream));
        R.ctx->sync();  // the staging buffers are reused by the next exchange
    }
}

template <class T>
void HostTransport<T>::gather(SlabRun<T>& R, const Dims& ds) {
    const int64_t pl = static_cast<int64_t>(ds.nx) * ds.ny;
    const auto& p = R.parts[0];
    const T* srcs[3] = {p.u(R.cur), p.m(), p.nu()};
    std::vector<int64_t> counts(R.world);
    int64_t total = 0;
    for (int r = 0; r < R.world; ++r) {
        counts[r] = static_cast<int64_t>(sizeof(T)) * 9 * pl * slab_bounds(ds.nz, r, R.world, R.H).owned();
        total += counts[r];
    }
    const int64_t mine = pl * p.b.owned();
    T* hs = static_cast<T*>(R.ctx->get_pinned("slab_gather_tx", counts[R.rank]));
    T* hr = static_cast<T*>(R.ctx->get_pinned("slab_gather_rx", total));
    for (int f = 0; f < 3; ++f)
        for (int c = 0; c < 3; ++c)
            CK(cudaMemcpyAsync(hs + (f * 3 + c) * mine, srcs[f] + c * p.dl.n + p.b.hlo * pl,
                               sizeof(T) * mine, cudaMemcpyDeviceToHost, R.ctx->stream));
    R.ctx->sync();
    ck(tp->allgather(tp->user, hs, counts[R.rank], hr, counts.data()), "allgather");
    const T* q = hr;
    for (int r = 0; r < R.world; ++r) {
        const SlabBounds b = slab_bounds(ds.nz, r, R.world, R.H);
        const int64_t own = pl * b.owned();
        for (int f = 0; f < 3; ++f)
            for (int c = 0; c < 3; ++c)
                CK(cudaMemcpyAsync(R.gath[f] + c * ds.n + static_cast<int64_t>(b.zlo) * pl,
                                   q + (f * 3 + c) * own, sizeof(T) * own, cudaMemcpyHostToDevice,
                                   R.ctx->stream));
        q += 9 * own;
    }
    R.ctx->sync();
}

template <class T>
void HostTransport<T>::sum_f64(SlabRun<T>& R, double* dev, int n) {
    std::vector<double> h(n);
    CK(cudaMemcpyAsync(h.data(), dev, sizeof(double) * n, cudaMemcpyDeviceToHost, R.ctx->stream));
    R.ctx->sync();
    ck(tp->allreduce_sum_f64(tp->user, h.data(), n), "allreduce_sum_f64");
    CK(cudaMemcpyAsync(dev, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, R.ctx->stream));
    R.ctx->sync();
}

template <class T>
void HostTransport<T>::max_u64(SlabRun<T>& R, unsigned long long* dev, int n) {
    std::vector<uint64_t> h(n);
    CK(cudaMemcpyAsync(h.data(), dev, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, R.ctx->stream));
    R.ctx->sync();
    ck(tp->allreduce_max_u64(tp->user, h.data(), n), "allreduce_max_u64");
    CK(cudaMemcpyAsync(dev, h.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, R.ctx->stream));
    R.ctx->sync();
}

template <class T>
void HostTransport<T>::sum_u64(SlabRun<T>& R, unsigned long long* dev, int n) {
    // counts (far below 2^53): summed exactly as doubles
    std::vector<uint64_t> h(n);
    CK(cudaMemcpyAsync(h.data(), dev, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, R.ctx->stream));
    R.ctx->sync();
    std::vector<double> d(h.begin(), h.end());
    ck(tp->allreduce_sum_f64(tp->user, d.data(), n), "allreduce_sum_f64");
    for (int k = 0; k < n; ++k) h[k] = static_cast<uint64_t>(d[k]);
    CK(cudaMemcpyAsync(dev, h.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, R.ctx->stream));
    R.ctx->sync();
}

template <class T>
void HostTransport<T>::max_i32(SlabRun<T>& R, int* dev, int n) {
    std::vector<int> h(n);
    CK(cudaMemcpyAsync(h.data(), dev, sizeof(int) * n, cudaMemcpyDeviceToHost, R.ctx->stream));
    R.ctx->sync();
    std::vector<uint64_t> u(n);
    for (int k = 0; k < n; ++k) u[k] = static_cast<uint64_t>(static_cast<int64_t>(h[k]) + (int64_t(1) << 31));
    ck(tp->allreduce_max_u64(tp->user, u.data(), n), "allreduce_max_u64");
    for (int k = 0; k < n; ++k) h[k] = static_cast<int>(static_cast<int64_t>(u[k]) - (int64_t(1) << 31));
    CK(cudaMemcpyAsync(dev, h.data(), sizeof(int) * n, cudaMemcpyHostToDevice, R.ctx->stream));
    R.ctx->sync();
}

}  // namespace

extern "C" {

dfm_status dfm_slab_bounds(int64_t nz, int part, int nparts, int halo, int64_t out[4]) {
    return guarded([&] {
        if (nz < 1 || nparts < 1 || part < 0 || part >= nparts || halo < 0)
            fail(DFM_E_INVALID, "slab_bounds: bad arguments");
        const SlabBounds b = slab_bounds(static_cast<int>(nz), part, nparts, halo);
        out[0] = b.zlo;
        out[1] = b.zhi;
        out[2] = b.hlo;
        out[3] = b.hhi;
    });
}

int dfm_slab_halo(const dfm_config* cfg, const dfm_grid*) { return cfg ? slab_halo(cfg) : -1; }

dfm_status dfm_slab_unique_id(unsigned char id[128]) {
    return guarded([&] {
        NcclApi& api = nccl_api();
        api.load();
        ncclUniqueId u;
        api.ck(api.GetUniqueId(&u), "get unique id");
        std::memcpy(id, u.internal, 128);
    });
}

}  // extern "C"

namespace {

dfm_status register_slab_impl(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                              const void* d_moving, const dfm_config* cfg, const double* scales,
                              const int32_t* iterations, int32_t nscales, int rank, int world,
                              const unsigned char* nccl_id, int emulate,
                              const dfm_slab_transport* tp, void* d_out_soa_field,
                              int64_t* out_zlo, int64_t* out_zhi, dfm_iter_record* records,
                              int64_t max_records, dfm_runlog* log) {
    return guarded([&] {
        validate_grid(g);
        validate_config(cfg);
        validate_schedule(scales, iterations, nscales);
        if (g->ndim != 3) fail(DFM_E_INVALID, "slab decomposition needs a 3-D grid");
        if (world < 1 || rank < 0 || rank >= world) fail(DFM_E_INVALID, "slab: bad rank/world");
        if (world > 1 && emulate > 1) fail(DFM_E_INVALID, "slab: emulate needs world == 1");
        if (emulate > 64) fail(DFM_E_INVALID, "slab: at most 64 emulated slabs");
        RegOut o;
        DFM_DISPATCH(ctx, {
            SlabRun<T> R;
            R.ctx = ctx;
            R.g = g;
            R.cfg = cfg;
            R.full = to_dims(g);
            R.rank = rank;
            R.world = world;
            R.E = world > 1 ? 1 : std::max(1, emulate);
            R.repl_max = ctx->slab_repl_max;
            // halo/interior overlap: across GPUs the exchange rides NVLink while
            // the interior planes compute; emulated slabs share one GPU's HBM
            // (measured slower there: 3.23 -> 3.39 s on config 4), so auto = NCCL only
            R.overlap = ctx->slab_overlap > 0 || (ctx->slab_overlap < 0 && world > 1 && !tp);
            EmulatedTransport<T> emu;
            NcclTransport<T> ncx;
            HostTransport<T> host;
            if (tp) {
                host.tp = tp;
                R.tp = &host;
            } else if (world > 1) {
                if (!nccl_id) fail(DFM_E_INVALID, "slab: nccl_id required when world > 1");
                NcclApi& api = nccl_api();
                api.load();
                ncclUniqueId u;
                std::memcpy(u.internal, nccl_id, 128);
                api.ck(api.CommInitRank(&ncx.comm, world, u, rank), "comm init");
                ncx.nc = &api;
                R.tp = &ncx;
            } else {
                R.tp = &emu;
            }
            try {
                R.run(static_cast<const T*>(d_fixed), static_cast<const T*>(d_moving), scales,
                      iterations, nscales, o, static_cast<T*>(d_out_soa_field), out_zlo, out_zhi);
            } catch (...) {
                if (ncx.comm) ncx.nc->CommDestroy(ncx.comm);
                throw;
            }
            if (ncx.comm) ncx.nc->CommDestroy(ncx.comm);
        });
        fill_log(o, records, max_records, log);
        if (o.sing > 0.0)
            fail(DFM_E_NUMERICAL, "register_images: folded warp (det J <= 0 somewhere)");
    });
}

}  // namespace

extern "C" {

dfm_status dfm_dev_register_slab(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                                 const void* d_moving, const dfm_config* cfg,
                                 const double* scales, const int32_t* iterations,
                                 int32_t nscales, int rank, int world,
                                 const unsigned char* nccl_id, int emulate,
                                 void* d_out_soa_field, int64_t* out_zlo, int64_t* out_zhi,
                                 dfm_iter_record* records, int64_t max_records, dfm_runlog* log) {
    return register_slab_impl(ctx, g, d_fixed, d_moving, cfg, scales, iterations, nscales, rank,
                              world, nccl_id, emulate, nullptr, d_out_soa_field, out_zlo, out_zhi,
                              records, max_records, log);
}

dfm_status dfm_dev_register_slab_tp(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                                    const void* d_moving, const dfm_config* cfg,
                                    const double* scales, const int32_t* iterations,
                                    int32_t nscales, int rank, int world,
                                    const dfm_slab_transport* tp, void* d_out_soa_field,
                                    int64_t* out_zlo, int64_t* out_zhi, dfm_iter_record* records,
                                    int64_t max_records, dfm_runlog* log) {
    if (!tp || !tp->sendrecv || !tp->allreduce_sum_f64 || !tp->allreduce_max_u64 ||
        !tp->allgather)
        return dfm_internal_set_error(DFM_E_INVALID, "slab transport: missing callback");
    return register_slab_impl(ctx, g, d_fixed, d_moving, cfg, scales, iterations, nscales, rank,
                              world, nullptr, 1, tp, d_out_soa_field, out_zlo, out_zhi, records,
                              max_records, log);
}

}  // extern "C"
