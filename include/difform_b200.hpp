// difform_b200.hpp — drop-in C++ face of the B200 path: the reference's
// difform:: registration API (/root/reference/proj/include/difform/*.hpp)
// implemented header-only on top of the C-ABI in difform_gpu.h.
//
// A caller of the reference (e.g. the `difform register` CLI, the sweep
// driver, the test suites) switches by including this header instead of the
// reference headers and linking libdifform_cuda.so.  Containers keep the
// reference's layout (x-fastest, AoS fields of doubles) so the call sites do
// not change; errors are thrown as the same exception classes
// (std::invalid_argument for validation, std::runtime_error for numerical
// failures).  Each host thread uses its own device context (re-entrant like
// the reference's sweep, pipeline.cpp:287-301).
//
// Precision: the default context computes in fp64 ("parity mode", the
// reference's arithmetic type); difform::gpu::set_precision(DFM_PREC_F32)
// selects the fp32 performance mode for the calling thread.
#pragma once

#include <array>
#include <algorithm>
#include <optional>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "difform_gpu.h"

namespace difform {

// ---- containers (core.hpp:13-87) -----------------------------------------
struct GridMeta {
    int ndim = 3;
    std::array<int64_t, 3> dims{1, 1, 1};
    std::array<double, 3> spacing{1.0, 1.0, 1.0};
    std::array<double, 3> origin{0.0, 0.0, 0.0};
    int64_t voxel_count() const { return dims[0] * dims[1] * dims[2]; }
    bool same_grid(const GridMeta& o) const { return ndim == o.ndim && dims == o.dims; }
};

inline GridMeta make_meta_2d(int64_t nx, int64_t ny, double sx = 1.0, double sy = 1.0) {
    GridMeta m;
    m.ndim = 2;
    m.dims = {nx, ny, 1};
    m.spacing = {sx, sy, 1.0};
    return m;
}
inline GridMeta make_meta_3d(int64_t nx, int64_t ny, int64_t nz, double sx = 1.0,
                             double sy = 1.0, double sz = 1.0) {
    GridMeta m;
    m.dims = {nx, ny, nz};
    m.spacing = {sx, sy, sz};
    return m;
}

struct ScalarImage {
    GridMeta meta;
    std::vector<double> data;
};
struct LabelImage {
    GridMeta meta;
    std::vector<int32_t> data;
};
struct VectorField {
    GridMeta meta;
    std::vector<double> data;  // voxel_count * ndim, interleaved
};
using DisplacementField = VectorField;

enum class LossKind { ssd = DFM_LOSS_SSD, lncc = DFM_LOSS_LNCC, dice = DFM_LOSS_DICE };
enum class RegMode { direct = DFM_MODE_DIRECT, svf = DFM_MODE_SVF };
enum class UpsampleMethod { linear, cubic };

struct AffineTransform {
    int ndim = 3;
    std::array<double, 9> A{1, 0, 0, 0, 1, 0, 0, 0, 1};
    std::array<double, 3> t{0, 0, 0};
};

struct LossEval {
    double value = 0.0;
    VectorField grad;
};

struct AdaptiveState {
    VectorField m, nu;
    int64_t t = 0;
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};

struct PyramidSchedule {
    std::vector<double> scales;
    std::vector<int> iterations;
    static PyramidSchedule defaults() { return {{4.0, 2.0, 1.0}, {50, 50, 50}}; }
};

struct RegistrationConfig {
    LossKind loss = LossKind::ssd;
    int lncc_radius = 2;
    double eta = 0.5;
    double sigma_grad = 1.0;
    double sigma_warp = 0.5;
    bool use_jac = false;
    RegMode mode = RegMode::direct;
    int svf_M = 6;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps_adam = 1e-8;
    double step_cap = 0.5;
    int conv_window = 10;
    double conv_tol = 1e-5;
    uint64_t seed = 0;
};

struct IterationRecord {
    int scale_index = 0;
    double scale = 1.0;
    int iter = 0;
    int64_t global_iter = 0;
    double loss = 0.0;
    double max_step = 0.0;
    double wall_ms = 0.0;
};

struct RunLog {
    std::vector<IterationRecord> iterations;
    double final_loss = 0.0;
    double final_singularity_fraction = 0.0;
    double total_ms = 0.0;
};

using RegInit = std::variant<std::monostate, AffineTransform, DisplacementField>;

// ---- device context plumbing ---------------------------------------------
namespace gpu {

inline int& thread_precision() {
    thread_local int p = DFM_PREC_F64;
    return p;
}

struct CtxDeleter {
    void operator()(dfm_ctx* c) const { dfm_ctx_destroy(c); }
};

inline void check(dfm_status s) {
    if (s == DFM_OK) return;
    char buf[512];
    dfm_last_error(buf, sizeof buf);
    if (s == DFM_E_INVALID) throw std::invalid_argument(buf);
    throw std::runtime_error(buf);  // numerical failure or device error
}

// The calling thread's context (created on first use on device 0).
inline dfm_ctx* ctx() {
    thread_local std::unique_ptr<dfm_ctx, CtxDeleter> c;
    thread_local int made_for = -1;
    if (!c || made_for != thread_precision()) {
        dfm_ctx* raw = nullptr;
        check(dfm_ctx_create(0, thread_precision(), &raw));
        c.reset(raw);
        made_for = thread_precision();
    }
    return c.get();
}

inline void set_precision(int precision) { thread_precision() = precision; }

inline dfm_grid grid(const GridMeta& m) {
    dfm_grid g{};
    g.ndim = m.ndim;
    for (int a = 0; a < 3; ++a) {
        g.dims[a] = m.dims[a];
        g.spacing[a] = m.spacing[a];
        g.origin[a] = m.origin[a];
    }
    return g;
}

inline GridMeta meta(const dfm_grid& g) {
    GridMeta m;
    m.ndim = g.ndim;
    for (int a = 0; a < 3; ++a) {
        m.dims[a] = g.dims[a];
        m.spacing[a] = g.spacing[a];
        m.origin[a] = g.origin[a];
    }
    return m;
}

inline dfm_config config(const RegistrationConfig& c) {
    dfm_config o{};
    o.loss = static_cast<int32_t>(c.loss);
    o.lncc_radius = c.lncc_radius;
    o.eta = c.eta;
    o.sigma_grad = c.sigma_grad;
    o.sigma_warp = c.sigma_warp;
    o.use_jac = c.use_jac ? 1 : 0;
    o.mode = static_cast<int32_t>(c.mode);
    o.svf_M = c.svf_M;
    o.beta1 = c.beta1;
    o.beta2 = c.beta2;
    o.eps_adam = c.eps_adam;
    o.step_cap = c.step_cap;
    o.conv_window = c.conv_window;
    o.conv_tol = c.conv_tol;
    o.seed = c.seed;
    return o;
}

inline VectorField field_like(const GridMeta& m) {
    return {m, std::vector<double>(static_cast<size_t>(m.voxel_count() * m.ndim))};
}

}  // namespace gpu

// ---- core.hpp ---------------------------------------------------------------
inline void validate_meta(const GridMeta& m) {
    const dfm_grid g = gpu::grid(m);
    gpu::check(dfm_validate_grid(&g));
}

inline ScalarImage downsample_image(const ScalarImage& img, const std::array<double, 3>& f) {
    const dfm_grid g = gpu::grid(img.meta);
    dfm_grid og{};
    gpu::check(dfm_downsample_grid(&g, f.data(), &og));
    ScalarImage out{gpu::meta(og), std::vector<double>(
                                       static_cast<size_t>(og.dims[0] * og.dims[1] * og.dims[2]))};
    gpu::check(dfm_downsample_image(gpu::ctx(), &g, img.data.data(), f.data(), &og,
                                    out.data.data()));
    return out;
}
inline ScalarImage downsample_image(const ScalarImage& img, double f) {
    return downsample_image(img, {f, f, f});
}

// ---- interp.hpp -------------------------------------------------------------
inline ScalarImage warp_image(const ScalarImage& img, const DisplacementField& phi) {
    if (!img.meta.same_grid(phi.meta)) throw std::invalid_argument("warp_image: grid dims mismatch");
    const dfm_grid g = gpu::grid(img.meta);
    ScalarImage out{img.meta, std::vector<double>(img.data.size())};
    gpu::check(dfm_warp_image(gpu::ctx(), &g, img.data.data(), phi.data.data(), out.data.data()));
    return out;
}

inline LabelImage warp_labels(const LabelImage& labels, const DisplacementField& phi) {
    if (!labels.meta.same_grid(phi.meta))
        throw std::invalid_argument("warp_labels: grid dims mismatch");
    const dfm_grid g = gpu::grid(labels.meta);
    LabelImage out{labels.meta, std::vector<int32_t>(labels.data.size())};
    gpu::check(dfm_warp_labels(gpu::ctx(), &g, labels.data.data(), phi.data.data(),
                               out.data.data()));
    return out;
}

inline DisplacementField compose(const DisplacementField& phi, const DisplacementField& psi) {
    if (!phi.meta.same_grid(psi.meta)) throw std::invalid_argument("compose: grid dims mismatch");
    const dfm_grid g = gpu::grid(phi.meta);
    VectorField out = gpu::field_like(phi.meta);
    gpu::check(dfm_compose(gpu::ctx(), &g, phi.data.data(), psi.data.data(), out.data.data()));
    return out;
}

inline ScalarImage jacobian_det(const DisplacementField& phi) {
    const dfm_grid g = gpu::grid(phi.meta);
    ScalarImage out{phi.meta, std::vector<double>(static_cast<size_t>(phi.meta.voxel_count()))};
    gpu::check(dfm_jacobian_det(gpu::ctx(), &g, phi.data.data(), out.data.data()));
    return out;
}

inline ScalarImage gaussian_smooth(const ScalarImage& img, const std::array<double, 3>& s) {
    const dfm_grid g = gpu::grid(img.meta);
    ScalarImage out{img.meta, std::vector<double>(img.data.size())};
    gpu::check(dfm_gaussian_smooth(gpu::ctx(), &g, img.data.data(), s.data(), out.data.data()));
    return out;
}
inline ScalarImage gaussian_smooth(const ScalarImage& img, double s) {
    return gaussian_smooth(img, {s, s, s});
}

inline VectorField gaussian_smooth_field(const VectorField& f, const std::array<double, 3>& s) {
    const dfm_grid g = gpu::grid(f.meta);
    VectorField out = gpu::field_like(f.meta);
    gpu::check(
        dfm_gaussian_smooth_field(gpu::ctx(), &g, f.data.data(), s.data(), out.data.data()));
    return out;
}
inline VectorField gaussian_smooth_field(const VectorField& f, double s) {
    return gaussian_smooth_field(f, {s, s, s});
}

inline DisplacementField upsample_field(const DisplacementField& phi, const GridMeta& nm,
                                        UpsampleMethod method = UpsampleMethod::linear) {
    if (method != UpsampleMethod::linear)
        throw std::invalid_argument("upsample_field: only the linear method is on the device path");
    const dfm_grid g = gpu::grid(phi.meta), ng = gpu::grid(nm);
    VectorField out = gpu::field_like(nm);
    gpu::check(dfm_upsample_field(gpu::ctx(), &g, phi.data.data(), &ng, out.data.data()));
    return out;
}

inline VectorField resample_field_linear(const VectorField& f, const GridMeta& nm) {
    const dfm_grid g = gpu::grid(f.meta), ng = gpu::grid(nm);
    VectorField out = gpu::field_like(nm);
    gpu::check(dfm_resample_field_linear(gpu::ctx(), &g, f.data.data(), &ng, out.data.data()));
    return out;
}

inline DisplacementField resample_displacement(const DisplacementField& phi, const GridMeta& nm) {
    const dfm_grid g = gpu::grid(phi.meta), ng = gpu::grid(nm);
    VectorField out = gpu::field_like(nm);
    gpu::check(dfm_resample_displacement(gpu::ctx(), &g, phi.data.data(), &ng, out.data.data()));
    return out;
}

// ---- similarity.hpp ---------------------------------------------------------
inline LossEval ssd_eval(const ScalarImage& f, const ScalarImage& m, const DisplacementField& phi) {
    const dfm_grid fg = gpu::grid(f.meta), mg = gpu::grid(m.meta);
    LossEval e{0.0, gpu::field_like(f.meta)};
    gpu::check(dfm_ssd_eval(gpu::ctx(), &fg, f.data.data(), &mg, m.data.data(), phi.data.data(),
                            &e.value, e.grad.data.data()));
    return e;
}

inline LossEval lncc_eval(const ScalarImage& f, const ScalarImage& m, const DisplacementField& phi,
                          int window_radius) {
    const dfm_grid fg = gpu::grid(f.meta), mg = gpu::grid(m.meta);
    LossEval e{0.0, gpu::field_like(f.meta)};
    gpu::check(dfm_lncc_eval(gpu::ctx(), &fg, f.data.data(), &mg, m.data.data(),
                             phi.data.data(), window_radius, &e.value, e.grad.data.data()));
    return e;
}

inline LossEval dice_soft_eval(const ScalarImage& f, const ScalarImage& m,
                               const DisplacementField& phi) {
    const dfm_grid fg = gpu::grid(f.meta), mg = gpu::grid(m.meta);
    LossEval e{0.0, gpu::field_like(f.meta)};
    gpu::check(dfm_dice_eval(gpu::ctx(), &fg, f.data.data(), &mg, m.data.data(), phi.data.data(),
                             &e.value, e.grad.data.data()));
    return e;
}

// ---- optim.hpp ----------------------------------------------------------------
inline AdaptiveState make_adaptive_state(const GridMeta& meta, double beta1 = 0.9,
                                         double beta2 = 0.999, double eps = 1e-8) {
    validate_meta(meta);
    AdaptiveState s;
    s.m = gpu::field_like(meta);
    s.nu = gpu::field_like(meta);
    s.beta1 = beta1;
    s.beta2 = beta2;
    s.eps = eps;
    return s;
}

inline VectorField adam_step(AdaptiveState& s, const VectorField& v) {
    if (!s.m.meta.same_grid(v.meta)) throw std::invalid_argument("adam_step: state/input grid mismatch");
    const dfm_grid g = gpu::grid(v.meta);
    VectorField dir = gpu::field_like(v.meta);
    gpu::check(dfm_adam_step(gpu::ctx(), &g, s.m.data.data(), s.nu.data.data(), &s.t, s.beta1,
                             s.beta2, s.eps, v.data.data(), dir.data.data()));
    return dir;
}

inline AdaptiveState upsample_state(const AdaptiveState& s, const GridMeta& nm) {
    const dfm_grid g = gpu::grid(s.m.meta), ng = gpu::grid(nm);
    AdaptiveState o = s;
    o.m = gpu::field_like(nm);
    o.nu = gpu::field_like(nm);
    gpu::check(dfm_upsample_state(gpu::ctx(), &g, s.m.data.data(), s.nu.data.data(), &ng,
                                  o.m.data.data(), o.nu.data.data()));
    return o;
}

// ---- diffeo.hpp ---------------------------------------------------------------
inline VectorField eulerian_direction(const VectorField& grad, const DisplacementField& phi,
                                      bool use_jac) {
    if (!grad.meta.same_grid(phi.meta)) throw std::invalid_argument("eulerian_direction: grid mismatch");
    const dfm_grid g = gpu::grid(grad.meta);
    VectorField out = gpu::field_like(grad.meta);
    gpu::check(dfm_eulerian_direction(gpu::ctx(), &g, grad.data.data(), phi.data.data(),
                                      use_jac ? 1 : 0, out.data.data()));
    return out;
}

inline DisplacementField apply_update(const DisplacementField& phi, const VectorField& v,
                                      double eta, double sigma_warp, double cap = 0.5) {
    if (!phi.meta.same_grid(v.meta)) throw std::invalid_argument("apply_update: grid mismatch");
    const dfm_grid g = gpu::grid(phi.meta);
    VectorField out = gpu::field_like(phi.meta);
    gpu::check(dfm_apply_update(gpu::ctx(), &g, phi.data.data(), v.data.data(), eta, sigma_warp,
                                cap, out.data.data()));
    return out;
}

// ---- analysis.hpp -------------------------------------------------------------
inline double singularity_fraction(const DisplacementField& phi) {
    const dfm_grid g = gpu::grid(phi.meta);
    double f = 0.0;
    gpu::check(dfm_singularity_fraction(gpu::ctx(), &g, phi.data.data(), &f));
    return f;
}

// ---- pipeline.hpp -------------------------------------------------------------
inline std::pair<DisplacementField, RunLog> register_images(
    const ScalarImage& fixed, const ScalarImage& moving, const RegistrationConfig& cfg,
    const PyramidSchedule& sched, const RegInit& init = std::monostate{}) {
    if (!fixed.meta.same_grid(moving.meta))
        throw std::invalid_argument("register_images: fixed/moving grids differ");
    if (sched.scales.size() != sched.iterations.size())
        throw std::invalid_argument("schedule: scales/iterations size mismatch");
    const dfm_grid g = gpu::grid(fixed.meta);
    const dfm_config c = gpu::config(cfg);
    dfm_init in{};
    in.kind = DFM_INIT_NONE;
    if (const auto* T = std::get_if<AffineTransform>(&init)) {
        in.kind = DFM_INIT_AFFINE;
        in.affine_ndim = T->ndim;
        for (int i = 0; i < 9; ++i) in.A[i] = T->A[static_cast<size_t>(i)];
        for (int i = 0; i < 3; ++i) in.t[i] = T->t[static_cast<size_t>(i)];
    } else if (const auto* u = std::get_if<DisplacementField>(&init)) {
        in.kind = DFM_INIT_FIELD;
        in.field_grid = gpu::grid(u->meta);
        in.field = u->data.data();
    }
    int64_t cap = 1;
    for (int it : sched.iterations) cap += it > 0 ? it : 0;
    std::vector<dfm_iter_record> recs(static_cast<size_t>(cap));
    std::vector<int32_t> iters(sched.iterations.begin(), sched.iterations.end());
    dfm_runlog rl{};
    DisplacementField phi = gpu::field_like(fixed.meta);
    gpu::check(dfm_register(gpu::ctx(), &g, fixed.data.data(), moving.data.data(), DFM_HOST_F64,
                            &c, sched.scales.data(), iters.data(),
                            static_cast<int32_t>(sched.scales.size()), &in, phi.data.data(),
                            DFM_HOST_F64, recs.data(), cap, &rl));
    RunLog log;
    log.final_loss = rl.final_loss;
    log.final_singularity_fraction = rl.final_singularity_fraction;
    log.total_ms = rl.total_ms;
    for (int64_t i = 0; i < rl.n_records; ++i) {
        const dfm_iter_record& r = recs[static_cast<size_t>(i)];
        log.iterations.push_back({r.scale_index, r.scale, r.iter, r.global_iter, r.loss,
                                  r.max_step, r.wall_ms});
    }
    return {std::move(phi), std::move(log)};
}

// ---- diffeo.hpp: SVF -----------------------------------------------------------
using VelocityField = VectorField;

inline DisplacementField exp_map(const VelocityField& v, int M) {
    const dfm_grid g = gpu::grid(v.meta);
    DisplacementField out = gpu::field_like(v.meta);
    gpu::check(dfm_exp_map(gpu::ctx(), &g, v.data.data(), M, out.data.data()));
    return out;
}

inline VectorField svf_pullback(const VelocityField& v, const VectorField& grad_phi, int M) {
    if (!v.meta.same_grid(grad_phi.meta))
        throw std::invalid_argument("svf_pullback: grid mismatch");
    const dfm_grid g = gpu::grid(v.meta);
    VectorField out = gpu::field_like(v.meta);
    gpu::check(dfm_svf_pullback(gpu::ctx(), &g, v.data.data(), grad_phi.data.data(), M,
                                out.data.data()));
    return out;
}

// ---- affine.hpp ----------------------------------------------------------------
struct AffineResult {
    AffineTransform transform;
    double loss = 0.0;
    bool diverged = false;
    int64_t iterations = 0;
};

struct AffineGrad {
    double value = 0.0;
    std::array<double, 9> dA{};
    std::array<double, 3> dt{};
};

inline AffineTransform identity_affine(int ndim) {
    AffineTransform T;
    T.ndim = ndim;
    T.A.fill(0.0);
    for (int i = 0; i < ndim; ++i) T.A[static_cast<size_t>(i * ndim + i)] = 1.0;
    T.t = {0.0, 0.0, 0.0};
    return T;
}

inline double affine_det(const AffineTransform& T) {
    const auto& a = T.A;
    if (T.ndim == 2) return a[0] * a[3] - a[1] * a[2];
    return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
           a[2] * (a[3] * a[7] - a[4] * a[6]);
}

inline DisplacementField affine_to_field(const AffineTransform& T, const GridMeta& meta) {
    if (T.ndim != meta.ndim)
        throw std::invalid_argument("affine_to_field: dimensionality mismatch");
    const dfm_grid g = gpu::grid(meta);
    DisplacementField out = gpu::field_like(meta);
    gpu::check(dfm_affine_to_field(gpu::ctx(), &g, T.A.data(), T.t.data(), out.data.data()));
    return out;
}

inline AffineGrad affine_param_gradient(const ScalarImage& fixed, const ScalarImage& moving,
                                        LossKind loss, const AffineTransform& T,
                                        const std::array<double, 3>& scale_to_full,
                                        int lncc_radius = 2) {
    const dfm_grid g = gpu::grid(fixed.meta);
    AffineGrad r;
    gpu::check(dfm_affine_param_gradient(gpu::ctx(), &g, fixed.data.data(), moving.data.data(),
                                         static_cast<int>(loss), T.A.data(), T.t.data(),
                                         scale_to_full.data(), lncc_radius, &r.value,
                                         r.dA.data(), r.dt.data()));
    return r;
}

inline AffineResult affine_register(const ScalarImage& fixed, const ScalarImage& moving,
                                    LossKind loss, const std::vector<double>& scales,
                                    const std::vector<int>& iters, double eta,
                                    int lncc_radius = 2) {
    if (!fixed.meta.same_grid(moving.meta))
        throw std::invalid_argument("affine_register: images must share a grid");
    if (scales.size() != iters.size() || scales.empty())
        throw std::invalid_argument("affine_register: bad schedule");
    const dfm_grid g = gpu::grid(fixed.meta);
    std::vector<int32_t> it(iters.begin(), iters.end());
    dfm_affine_result r{};
    gpu::check(dfm_affine_register(gpu::ctx(), &g, fixed.data.data(), moving.data.data(),
                                   static_cast<int>(loss), scales.data(), it.data(),
                                   static_cast<int32_t>(scales.size()), eta, lncc_radius, &r));
    AffineResult out;
    out.transform.ndim = r.ndim;
    for (int k = 0; k < 9; ++k) out.transform.A[static_cast<size_t>(k)] = r.A[k];
    for (int k = 0; k < 3; ++k) out.transform.t[static_cast<size_t>(k)] = r.t[k];
    out.loss = r.loss;
    out.diverged = r.diverged != 0;
    out.iterations = r.iterations;
    return out;
}

// ---- analysis.hpp: evaluation ------------------------------------------------------
struct RegionOverlap {
    int32_t label = 0;
    int64_t fixed_count = 0, warped_count = 0, intersection = 0;
    bool has_to = false;
    double to = 0.0, mo = 0.0;
    bool has_fn = false;
    double fn = 0.0;
    bool has_fp = false;
    double fp = 0.0, vs = 0.0;
};

struct OverlapReport {
    std::vector<RegionOverlap> regions;
    double to_mean = 0.0, mo_mean = 0.0, fn_mean = 0.0, fp_mean = 0.0, vs_mean = 0.0;
    double to_klein = 0.0, mo_klein = 0.0, fn_klein = 0.0, fp_klein = 0.0, vs_klein = 0.0;
};

inline OverlapReport overlap_report(const LabelImage& warped, const LabelImage& fixed) {
    const dfm_grid gw = gpu::grid(warped.meta), gf = gpu::grid(fixed.meta);
    dfm_overlap_summary s{};
    std::vector<dfm_region_overlap> regs(1024);
    for (;;) {
        gpu::check(dfm_overlap_report(gpu::ctx(), &gw, warped.data.data(), &gf,
                                      fixed.data.data(), &s, regs.data(),
                                      static_cast<int64_t>(regs.size())));
        if (s.n_regions <= static_cast<int64_t>(regs.size())) break;
        regs.resize(static_cast<size_t>(s.n_regions));
    }
    OverlapReport r;
    r.to_mean = s.to_mean;
    r.mo_mean = s.mo_mean;
    r.fn_mean = s.fn_mean;
    r.fp_mean = s.fp_mean;
    r.vs_mean = s.vs_mean;
    r.to_klein = s.to_klein;
    r.mo_klein = s.mo_klein;
    r.fn_klein = s.fn_klein;
    r.fp_klein = s.fp_klein;
    r.vs_klein = s.vs_klein;
    for (int64_t k = 0; k < s.n_regions; ++k) {
        const dfm_region_overlap& q = regs[static_cast<size_t>(k)];
        r.regions.push_back({q.label, q.fixed_count, q.warped_count, q.intersection,
                             q.has_to != 0, q.to, q.mo, q.has_fn != 0, q.fn, q.has_fp != 0,
                             q.fp, q.vs});
    }
    return r;
}

struct Landmark {
    std::array<double, 3> point_mm{0.0, 0.0, 0.0};
    std::string id;
};
using LandmarkSet = std::vector<Landmark>;

struct LandmarkErrors {
    std::vector<double> distances_mm;
    double mean = 0.0;
    double max = 0.0;
};

inline LandmarkErrors landmark_error(const LandmarkSet& fixed_pts, const LandmarkSet& moving_pts,
                                     const DisplacementField& phi, const GridMeta& fixed_meta,
                                     const GridMeta& moving_meta) {
    if (fixed_pts.size() != moving_pts.size())
        throw std::invalid_argument("landmark_error: landmark counts differ");
    const dfm_grid gf = gpu::grid(fixed_meta), gm = gpu::grid(moving_meta),
                   gp = gpu::grid(phi.meta);
    std::vector<double> a, b;
    for (size_t i = 0; i < fixed_pts.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            a.push_back(fixed_pts[i].point_mm[static_cast<size_t>(k)]);
            b.push_back(moving_pts[i].point_mm[static_cast<size_t>(k)]);
        }
    LandmarkErrors r;
    r.distances_mm.resize(fixed_pts.size());
    gpu::check(dfm_landmark_error(gpu::ctx(), &gf, &gm, &gp, phi.data.data(),
                                  static_cast<int64_t>(fixed_pts.size()), a.data(), b.data(),
                                  r.distances_mm.data(), &r.mean, &r.max));
    return r;
}

// ---- pipeline.hpp: sweep --------------------------------------------------------
enum class SweepMetric { loss, overlap };

struct SweepPair {
    ScalarImage fixed, moving;
    std::optional<LabelImage> fixed_labels, moving_labels;
    std::string name;
};

struct SweepRow {
    double eta = 0.0, sigma_warp = 0.0, sigma_grad = 0.0;
    double metric_mean = 0.0, metric_sd = 0.0;
    double wall_ms = 0.0;
    bool failed = false;
    std::string error;
};

struct SweepResult {
    std::vector<SweepRow> rows;
    std::vector<std::vector<std::vector<double>>> heatmaps;
    std::vector<double> etas, sigma_warps, sigma_grads;
};

// `workers` maps to worker contexts on the current device (the reference's
// worker threads); difform::gpu::set_sweep_devices() spreads them over GPUs.
inline std::vector<int>& sweep_devices() {
    static std::vector<int> d{0};
    return d;
}

inline SweepResult sweep(const std::vector<SweepPair>& pairs, const RegistrationConfig& base,
                         const PyramidSchedule& sched, const std::vector<double>& etas,
                         const std::vector<double>& sigma_warps,
                         const std::vector<double>& sigma_grads, SweepMetric metric,
                         int workers) {
    std::vector<dfm_grid> grids;
    grids.reserve(pairs.size());
    std::vector<dfm_sweep_pair> ps;
    for (const SweepPair& p : pairs) {
        grids.push_back(gpu::grid(p.fixed.meta));
        ps.push_back({&grids.back(), p.fixed.data.data(), p.moving.data.data(),
                      p.fixed_labels ? p.fixed_labels->data.data() : nullptr,
                      p.moving_labels ? p.moving_labels->data.data() : nullptr});
    }
    const dfm_config c = gpu::config(base);
    std::vector<int32_t> it(sched.iterations.begin(), sched.iterations.end());
    const size_t n_cfg = etas.size() * sigma_warps.size() * sigma_grads.size();
    std::vector<dfm_sweep_row> rows(n_cfg > 0 ? n_cfg : 1);
    const std::vector<int>& dev = sweep_devices();
    const int per_dev = std::max(1, workers / static_cast<int>(dev.size()));
    gpu::check(dfm_sweep(dev.data(), static_cast<int>(dev.size()), per_dev,
                         gpu::thread_precision(), ps.data(), static_cast<int>(ps.size()), &c,
                         sched.scales.data(), it.data(), static_cast<int32_t>(it.size()),
                         etas.data(), static_cast<int>(etas.size()), sigma_warps.data(),
                         static_cast<int>(sigma_warps.size()), sigma_grads.data(),
                         static_cast<int>(sigma_grads.size()),
                         metric == SweepMetric::overlap ? DFM_SWEEP_OVERLAP : DFM_SWEEP_LOSS, 0,
                         1, rows.data()));
    SweepResult r;
    r.etas = etas;
    r.sigma_warps = sigma_warps;
    r.sigma_grads = sigma_grads;
    r.heatmaps.assign(etas.size(), std::vector<std::vector<double>>(
                                       sigma_warps.size(),
                                       std::vector<double>(sigma_grads.size(), 0.0)));
    for (size_t k = 0; k < n_cfg; ++k) {
        const dfm_sweep_row& q = rows[k];
        r.rows.push_back({q.eta, q.sigma_warp, q.sigma_grad, q.metric_mean, q.metric_sd,
                          q.wall_ms, q.failed != 0, q.error});
        const size_t gi = k % sigma_grads.size();
        const size_t wi = (k / sigma_grads.size()) % sigma_warps.size();
        const size_t ei = k / (sigma_grads.size() * sigma_warps.size());
        r.heatmaps[ei][wi][gi] = q.metric_mean;
    }
    return r;
}

}  // namespace difform
