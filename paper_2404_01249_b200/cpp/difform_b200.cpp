// difform_b200.cpp — the reference's C++ API for the hot path, defined over
// the B200 C-ABI (include/difform_gpu.h) and compiled against the REFERENCE'S
// OWN headers (proj/include/difform/*.hpp): link-level drop-in.
//
// A caller of the reference keeps its #includes and object files and relinks:
// libdifform_b200.so replaces the reference's core.o, interp.o, similarity.o,
// optim.o, diffeo.o and pipeline.o, i.e. every function declared in
//   core.hpp:76-87      make_meta_*, validate_meta, make_image/labels/field,
//                       new_identity_field, downsample_image
//   interp.hpp:11-75    sample_linear[_gradient], sample_field[_jacobian],
//                       warp_image, warp_labels, compose, jacobian[_det],
//                       gaussian_smooth[_field], upsample_field,
//                       resample_field_linear, resample_displacement
//   similarity.hpp:17-28 ssd_eval, lncc_eval, dice_soft_eval
//   optim.hpp:18-31     make_adaptive_state, adam_step, sgd_step, upsample_state
//   diffeo.hpp:10-27    eulerian_direction, apply_update, exp_map, svf_pullback
//   pipeline.hpp:21-73  validate_schedule, validate_config, register_images, sweep
// The reference's off-path objects (affine.o, analysis.o, parallel.o, synth.o,
// toy.o, io.o) link unchanged on top and call into these definitions (e.g.
// analysis.cpp's singularity_fraction -> jacobian_det on the device).
//
// Containers keep the reference's layout (x-fastest, interleaved AoS doubles);
// every numeric function runs on the device through the C-ABI.  Errors map to
// the reference's exception classes: DFM_E_INVALID -> std::invalid_argument,
// DFM_E_NUMERICAL -> std::runtime_error (the message is the library's).
// Each host thread uses its own dfm_ctx (re-entrant like the reference's
// sweep workers, pipeline.cpp:287-301); precision defaults to fp64 (the
// reference's arithmetic type) and difform::gpu::set_precision selects fp32.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "difform/core.hpp"
#include "difform/diffeo.hpp"
#include "difform/interp.hpp"
#include "difform/optim.hpp"
#include "difform/pipeline.hpp"
#include "difform/similarity.hpp"
#include "difform_b200.hpp"
#include "difform_gpu.h"

namespace difform {
namespace gpu {

namespace {

int& thread_precision() {
    thread_local int p = DFM_PREC_F64;
    return p;
}

bool& thread_exact() {
    thread_local bool e = false;
    return e;
}

struct CtxDeleter {
    void operator()(dfm_ctx* c) const { dfm_ctx_destroy(c); }
};

std::vector<int>& sweep_device_list() {
    static std::vector<int> d{0};
    return d;
}

}  // namespace

void check(dfm_status s) {
    if (s == DFM_OK) return;
    char buf[512];
    dfm_last_error(buf, sizeof buf);
    if (s == DFM_E_INVALID) throw std::invalid_argument(buf);
    throw std::runtime_error(buf);  // numerical failure or device error
}

dfm_ctx* ctx() {
    thread_local std::unique_ptr<dfm_ctx, CtxDeleter> c;
    thread_local int made_for = -1;
    const int want = thread_precision() * 2 + (thread_exact() ? 1 : 0);
    if (!c || made_for != want) {
        dfm_ctx* raw = nullptr;
        check(dfm_ctx_create(0, thread_precision(), &raw));
        c.reset(raw);
        if (thread_exact()) check(dfm_ctx_set_option(raw, DFM_OPT_EXACT, 1));
        made_for = want;
    }
    return c.get();
}

void set_precision(int precision) {
    if (precision != DFM_PREC_F32 && precision != DFM_PREC_F64)
        throw std::invalid_argument("set_precision: DFM_PREC_F32 or DFM_PREC_F64");
    if (precision != DFM_PREC_F64 && thread_exact())
        throw std::invalid_argument("set_precision: the exact mode needs fp64 (set_exact(false) first)");
    thread_precision() = precision;
}
int precision() { return thread_precision(); }

void set_exact(bool on) {
    if (on && thread_precision() != DFM_PREC_F64)
        throw std::invalid_argument("set_exact: needs the fp64 precision");
    thread_exact() = on;
}

void set_sweep_devices(const std::vector<int>& devices) {
    if (devices.empty()) throw std::invalid_argument("set_sweep_devices: no devices");
    sweep_device_list() = devices;
}

}  // namespace gpu

namespace {

dfm_grid grid(const GridMeta& m) {
    dfm_grid g{};
    g.ndim = m.ndim;
    for (int a = 0; a < 3; ++a) {
        g.dims[a] = m.dims[static_cast<size_t>(a)];
        g.spacing[a] = m.spacing[static_cast<size_t>(a)];
        g.origin[a] = m.origin[static_cast<size_t>(a)];
    }
    return g;
}

GridMeta meta_of(const dfm_grid& g) {
    GridMeta m;
    m.ndim = g.ndim;
    for (int a = 0; a < 3; ++a) {
        m.dims[static_cast<size_t>(a)] = g.dims[a];
        m.spacing[static_cast<size_t>(a)] = g.spacing[a];
        m.origin[static_cast<size_t>(a)] = g.origin[a];
    }
    return m;
}

dfm_config config(const RegistrationConfig& c) {
    dfm_config o{};
    o.loss = static_cast<int32_t>(c.loss);  // LossKind {ssd, lncc, dice} = DFM_LOSS_*
    o.lncc_radius = c.lncc_radius;
    o.eta = c.eta;
    o.sigma_grad = c.sigma_grad;
    o.sigma_warp = c.sigma_warp;
    o.use_jac = c.use_jac ? 1 : 0;
    o.mode = c.mode == RegMode::svf ? DFM_MODE_SVF : DFM_MODE_DIRECT;
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

VectorField field_like(const GridMeta& m) {
    return {m, std::vector<double>(static_cast<size_t>(m.voxel_count() * m.ndim))};
}

ScalarImage image_like(const GridMeta& m) {
    return {m, std::vector<double>(static_cast<size_t>(m.voxel_count()))};
}

void same_grid_or_throw(const GridMeta& a, const GridMeta& b, const char* what) {
    if (!a.same_grid(b)) throw std::invalid_argument(std::string(what) + ": grid dims mismatch");
}

using gpu::check;
using gpu::ctx;

}  // namespace

// ---- core.hpp -----------------------------------------------------------------
GridMeta make_meta_2d(int64_t nx, int64_t ny, double sx, double sy) {
    GridMeta m;
    m.ndim = 2;
    m.dims = {nx, ny, 1};
    m.spacing = {sx, sy, 1.0};
    return m;
}

GridMeta make_meta_3d(int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz) {
    GridMeta m;
    m.ndim = 3;
    m.dims = {nx, ny, nz};
    m.spacing = {sx, sy, sz};
    return m;
}

void validate_meta(const GridMeta& m) {
    const dfm_grid g = grid(m);
    check(dfm_validate_grid(&g));
}

ScalarImage make_image(const GridMeta& m, double fill) {
    validate_meta(m);
    return {m, std::vector<double>(static_cast<size_t>(m.voxel_count()), fill)};
}

LabelImage make_labels(const GridMeta& m, int32_t fill) {
    validate_meta(m);
    return {m, std::vector<int32_t>(static_cast<size_t>(m.voxel_count()), fill)};
}

VectorField make_field(const GridMeta& m, double fill) {
    validate_meta(m);
    return {m, std::vector<double>(static_cast<size_t>(m.voxel_count() * m.ndim), fill)};
}

DisplacementField new_identity_field(const GridMeta& meta) { return make_field(meta, 0.0); }

ScalarImage downsample_image(const ScalarImage& img, const std::array<double, 3>& factor) {
    const dfm_grid g = grid(img.meta);
    dfm_grid og{};
    check(dfm_downsample_grid(&g, factor.data(), &og));
    ScalarImage out = image_like(meta_of(og));
    check(dfm_downsample_image(ctx(), &g, img.data.data(), factor.data(), &og, out.data.data()));
    return out;
}

ScalarImage downsample_image(const ScalarImage& img, double factor) {
    return downsample_image(img, {factor, factor, factor});
}

// ---- interp.hpp ---------------------------------------------------------------
double sample_linear(const ScalarImage& img, const std::array<double, 3>& point) {
    const dfm_grid g = grid(img.meta);
    double v = 0.0;
    check(dfm_sample_linear_points(ctx(), &g, img.data.data(), 1, point.data(), &v, nullptr));
    return v;
}

std::array<double, 3> sample_linear_gradient(const ScalarImage& img,
                                             const std::array<double, 3>& point) {
    const dfm_grid g = grid(img.meta);
    double v = 0.0;
    std::array<double, 3> gr{0.0, 0.0, 0.0};
    check(dfm_sample_linear_points(ctx(), &g, img.data.data(), 1, point.data(), &v, gr.data()));
    return gr;
}

std::array<double, 3> sample_field(const VectorField& f, const std::array<double, 3>& point) {
    const dfm_grid g = grid(f.meta);
    std::array<double, 3> v{0.0, 0.0, 0.0};
    check(dfm_sample_field_points(ctx(), &g, f.data.data(), 1, point.data(), v.data(), nullptr));
    return v;
}

std::array<std::array<double, 3>, 3> sample_field_jacobian(const VectorField& f,
                                                           const std::array<double, 3>& point) {
    const dfm_grid g = grid(f.meta);
    double v[3], j[9];
    check(dfm_sample_field_points(ctx(), &g, f.data.data(), 1, point.data(), v, j));
    std::array<std::array<double, 3>, 3> J{};
    for (int c = 0; c < 3; ++c)
        for (int a = 0; a < 3; ++a)
            J[static_cast<size_t>(c)][static_cast<size_t>(a)] = j[3 * c + a];
    return J;
}

ScalarImage warp_image(const ScalarImage& img, const DisplacementField& phi) {
    same_grid_or_throw(img.meta, phi.meta, "warp_image");
    const dfm_grid g = grid(img.meta);
    ScalarImage out = image_like(img.meta);
    check(dfm_warp_image(ctx(), &g, img.data.data(), phi.data.data(), out.data.data()));
    return out;
}

LabelImage warp_labels(const LabelImage& labels, const DisplacementField& phi) {
    same_grid_or_throw(labels.meta, phi.meta, "warp_labels");
    const dfm_grid g = grid(labels.meta);
    LabelImage out{labels.meta, std::vector<int32_t>(labels.data.size())};
    check(dfm_warp_labels(ctx(), &g, labels.data.data(), phi.data.data(), out.data.data()));
    return out;
}

DisplacementField compose(const DisplacementField& phi, const DisplacementField& psi) {
    same_grid_or_throw(phi.meta, psi.meta, "compose");
    const dfm_grid g = grid(phi.meta);
    VectorField out = field_like(phi.meta);
    check(dfm_compose(ctx(), &g, phi.data.data(), psi.data.data(), out.data.data()));
    return out;
}

JacobianImage jacobian(const DisplacementField& phi) {
    validate_meta(phi.meta);
    const dfm_grid g = grid(phi.meta);
    JacobianImage J;
    J.meta = phi.meta;
    J.data.resize(static_cast<size_t>(phi.meta.voxel_count() * phi.meta.ndim * phi.meta.ndim));
    check(dfm_jacobian(ctx(), &g, phi.data.data(), J.data.data()));
    return J;
}

ScalarImage jacobian_det(const DisplacementField& phi) {
    validate_meta(phi.meta);
    const dfm_grid g = grid(phi.meta);
    ScalarImage out = image_like(phi.meta);
    check(dfm_jacobian_det(ctx(), &g, phi.data.data(), out.data.data()));
    return out;
}

ScalarImage gaussian_smooth(const ScalarImage& img, const std::array<double, 3>& sigma) {
    const dfm_grid g = grid(img.meta);
    ScalarImage out = image_like(img.meta);
    check(dfm_gaussian_smooth(ctx(), &g, img.data.data(), sigma.data(), out.data.data()));
    return out;
}

VectorField gaussian_smooth_field(const VectorField& f, const std::array<double, 3>& sigma) {
    const dfm_grid g = grid(f.meta);
    VectorField out = field_like(f.meta);
    check(dfm_gaussian_smooth_field(ctx(), &g, f.data.data(), sigma.data(), out.data.data()));
    return out;
}

ScalarImage gaussian_smooth(const ScalarImage& img, double sigma) {
    return gaussian_smooth(img, {sigma, sigma, sigma});
}

VectorField gaussian_smooth_field(const VectorField& f, double sigma) {
    return gaussian_smooth_field(f, {sigma, sigma, sigma});
}

DisplacementField upsample_field(const DisplacementField& phi, const GridMeta& new_meta,
                                 UpsampleMethod method) {
    const dfm_grid g = grid(phi.meta), ng = grid(new_meta);
    VectorField out = field_like(new_meta);
    if (method == UpsampleMethod::cubic)
        check(dfm_upsample_field_cubic(ctx(), &g, phi.data.data(), &ng, out.data.data()));
    else
        check(dfm_upsample_field(ctx(), &g, phi.data.data(), &ng, out.data.data()));
    return out;
}

VectorField resample_field_linear(const VectorField& f, const GridMeta& new_meta) {
    const dfm_grid g = grid(f.meta), ng = grid(new_meta);
    VectorField out = field_like(new_meta);
    check(dfm_resample_field_linear(ctx(), &g, f.data.data(), &ng, out.data.data()));
    return out;
}

DisplacementField resample_displacement(const DisplacementField& phi, const GridMeta& new_meta) {
    const dfm_grid g = grid(phi.meta), ng = grid(new_meta);
    VectorField out = field_like(new_meta);
    check(dfm_resample_displacement(ctx(), &g, phi.data.data(), &ng, out.data.data()));
    return out;
}

// ---- similarity.hpp -------------------------------------------------------------
namespace {
void loss_grid_check(const ScalarImage& fixed, const ScalarImage& moving,
                     const DisplacementField& phi, const char* what) {
    if (!fixed.meta.same_grid(phi.meta))  // similarity.cpp:16-22
        throw std::invalid_argument(std::string(what) + ": fixed/phi grid mismatch");
    if (fixed.meta.ndim != moving.meta.ndim)
        throw std::invalid_argument(std::string(what) + ": dimensionality mismatch");
}
}  // namespace

LossEval ssd_eval(const ScalarImage& fixed, const ScalarImage& moving,
                  const DisplacementField& phi) {
    loss_grid_check(fixed, moving, phi, "ssd_eval");
    const dfm_grid fg = grid(fixed.meta), mg = grid(moving.meta);
    LossEval e{0.0, field_like(fixed.meta)};
    check(dfm_ssd_eval(ctx(), &fg, fixed.data.data(), &mg, moving.data.data(), phi.data.data(),
                       &e.value, e.grad.data.data()));
    return e;
}

LossEval lncc_eval(const ScalarImage& fixed, const ScalarImage& moving,
                   const DisplacementField& phi, int window_radius) {
    loss_grid_check(fixed, moving, phi, "lncc_eval");
    const dfm_grid fg = grid(fixed.meta), mg = grid(moving.meta);
    LossEval e{0.0, field_like(fixed.meta)};
    check(dfm_lncc_eval(ctx(), &fg, fixed.data.data(), &mg, moving.data.data(), phi.data.data(),
                        window_radius, &e.value, e.grad.data.data()));
    return e;
}

LossEval dice_soft_eval(const ScalarImage& fixed_mask, const ScalarImage& moving_mask,
                        const DisplacementField& phi) {
    loss_grid_check(fixed_mask, moving_mask, phi, "dice_soft_eval");
    const dfm_grid fg = grid(fixed_mask.meta), mg = grid(moving_mask.meta);
    LossEval e{0.0, field_like(fixed_mask.meta)};
    check(dfm_dice_eval(ctx(), &fg, fixed_mask.data.data(), &mg, moving_mask.data.data(),
                        phi.data.data(), &e.value, e.grad.data.data()));
    return e;
}

// ---- optim.hpp ------------------------------------------------------------------
AdaptiveState make_adaptive_state(const GridMeta& meta, double beta1, double beta2, double eps) {
    AdaptiveState s;
    s.m = make_field(meta);
    s.nu = make_field(meta);
    s.beta1 = beta1;
    s.beta2 = beta2;
    s.eps = eps;
    return s;
}

VectorField adam_step(AdaptiveState& state, const VectorField& v) {
    if (!state.m.meta.same_grid(v.meta))
        throw std::invalid_argument("adam_step: state/input grid mismatch");
    const dfm_grid g = grid(v.meta);
    VectorField dir = field_like(v.meta);
    check(dfm_adam_step(ctx(), &g, state.m.data.data(), state.nu.data.data(), &state.t,
                        state.beta1, state.beta2, state.eps, v.data.data(), dir.data.data()));
    return dir;
}

VectorField sgd_step(VectorField& mu, const VectorField& v, double momentum) {
    if (momentum == 0.0) return v;
    if (!mu.meta.same_grid(v.meta))
        throw std::invalid_argument("sgd_step: momentum/input grid mismatch");
    const dfm_grid g = grid(v.meta);
    VectorField out = field_like(v.meta);
    check(dfm_sgd_step(ctx(), &g, mu.data.data(), v.data.data(), momentum, out.data.data()));
    return out;
}

AdaptiveState upsample_state(const AdaptiveState& state, const GridMeta& new_meta) {
    const dfm_grid g = grid(state.m.meta), ng = grid(new_meta);
    AdaptiveState o = state;
    o.m = field_like(new_meta);
    o.nu = field_like(new_meta);
    check(dfm_upsample_state(ctx(), &g, state.m.data.data(), state.nu.data.data(), &ng,
                             o.m.data.data(), o.nu.data.data()));
    return o;
}

// ---- diffeo.hpp -----------------------------------------------------------------
VectorField eulerian_direction(const VectorField& grad, const DisplacementField& phi,
                               bool use_jac) {
    if (!grad.meta.same_grid(phi.meta))
        throw std::invalid_argument("eulerian_direction: grid mismatch");
    const dfm_grid g = grid(grad.meta);
    VectorField out = field_like(grad.meta);
    check(dfm_eulerian_direction(ctx(), &g, grad.data.data(), phi.data.data(), use_jac ? 1 : 0,
                                 out.data.data()));
    return out;
}

DisplacementField apply_update(const DisplacementField& phi, const VectorField& v, double eta,
                               double sigma_warp, double cap) {
    if (!phi.meta.same_grid(v.meta)) throw std::invalid_argument("apply_update: grid mismatch");
    const dfm_grid g = grid(phi.meta);
    VectorField out = field_like(phi.meta);
    check(dfm_apply_update(ctx(), &g, phi.data.data(), v.data.data(), eta, sigma_warp, cap,
                           out.data.data()));
    return out;
}

DisplacementField exp_map(const VelocityField& v, int M) {
    const dfm_grid g = grid(v.meta);
    DisplacementField out = field_like(v.meta);
    check(dfm_exp_map(ctx(), &g, v.data.data(), M, out.data.data()));
    return out;
}

VectorField svf_pullback(const VelocityField& v, const VectorField& grad_phi, int M) {
    if (!v.meta.same_grid(grad_phi.meta))
        throw std::invalid_argument("svf_pullback: grid mismatch");
    const dfm_grid g = grid(v.meta);
    VectorField out = field_like(v.meta);
    check(dfm_svf_pullback(ctx(), &g, v.data.data(), grad_phi.data.data(), M, out.data.data()));
    return out;
}

// ---- pipeline.hpp ---------------------------------------------------------------
void validate_schedule(const PyramidSchedule& s) {
    if (s.scales.size() != s.iterations.size() && !s.scales.empty())
        throw std::invalid_argument("schedule: scales/iterations size mismatch");
    std::vector<int32_t> it(s.iterations.begin(), s.iterations.end());
    check(dfm_validate_schedule(s.scales.data(), it.data(), static_cast<int32_t>(s.scales.size())));
}

void validate_config(const RegistrationConfig& c) {
    const dfm_config cc = config(c);
    check(dfm_validate_config(&cc));
}

std::pair<DisplacementField, RunLog> register_images(const ScalarImage& fixed,
                                                     const ScalarImage& moving,
                                                     const RegistrationConfig& cfg,
                                                     const PyramidSchedule& sched,
                                                     const RegInit& init) {
    validate_meta(fixed.meta);
    validate_meta(moving.meta);
    if (!fixed.meta.same_grid(moving.meta))
        throw std::invalid_argument("register_images: fixed/moving grids differ");
    validate_config(cfg);
    validate_schedule(sched);
    const dfm_grid g = grid(fixed.meta);
    const dfm_config c = config(cfg);
    dfm_init in{};
    in.kind = DFM_INIT_NONE;
    if (const auto* T = std::get_if<AffineTransform>(&init)) {
        in.kind = DFM_INIT_AFFINE;
        in.affine_ndim = T->ndim;
        for (int i = 0; i < 9; ++i) in.A[i] = T->A[static_cast<size_t>(i)];
        for (int i = 0; i < 3; ++i) in.t[i] = T->t[static_cast<size_t>(i)];
    } else if (const auto* u = std::get_if<DisplacementField>(&init)) {
        in.kind = DFM_INIT_FIELD;
        in.field_grid = grid(u->meta);
        in.field = u->data.data();
    }
    int64_t cap = 1;
    for (int it : sched.iterations) cap += it > 0 ? it : 0;
    std::vector<dfm_iter_record> recs(static_cast<size_t>(cap));
    std::vector<int32_t> iters(sched.iterations.begin(), sched.iterations.end());
    dfm_runlog rl{};
    DisplacementField phi = field_like(fixed.meta);
    check(dfm_register(ctx(), &g, fixed.data.data(), moving.data.data(), DFM_HOST_F64, &c,
                       sched.scales.data(), iters.data(), static_cast<int32_t>(sched.scales.size()),
                       &in, phi.data.data(), DFM_HOST_F64, recs.data(), cap, &rl));
    RunLog log;
    log.final_loss = rl.final_loss;
    log.final_singularity_fraction = rl.final_singularity_fraction;
    log.total_ms = rl.total_ms;
    for (int64_t i = 0; i < rl.n_records; ++i) {
        const dfm_iter_record& r = recs[static_cast<size_t>(i)];
        IterationRecord q;
        q.scale_index = r.scale_index;
        q.scale = r.scale;
        q.iter = r.iter;
        q.global_iter = r.global_iter;
        q.loss = r.loss;
        q.max_step = r.max_step;
        q.wall_ms = r.wall_ms;
        log.iterations.push_back(q);
    }
    return {std::move(phi), std::move(log)};
}

// `workers` maps to worker contexts on the sweep devices (the reference's
// worker threads; difform::gpu::set_sweep_devices spreads them over GPUs).
SweepResult sweep(const std::vector<SweepPair>& pairs, const RegistrationConfig& base,
                  const PyramidSchedule& sched, const std::vector<double>& etas,
                  const std::vector<double>& sigma_warps, const std::vector<double>& sigma_grads,
                  SweepMetric metric, int workers) {
    std::vector<dfm_grid> grids;
    grids.reserve(pairs.size());
    std::vector<dfm_sweep_pair> ps;
    for (const SweepPair& p : pairs) {
        grids.push_back(grid(p.fixed.meta));
        ps.push_back({&grids.back(), p.fixed.data.data(), p.moving.data.data(),
                      p.fixed_labels ? p.fixed_labels->data.data() : nullptr,
                      p.moving_labels ? p.moving_labels->data.data() : nullptr});
    }
    const dfm_config c = config(base);
    std::vector<int32_t> it(sched.iterations.begin(), sched.iterations.end());
    const size_t n_cfg = etas.size() * sigma_warps.size() * sigma_grads.size();
    std::vector<dfm_sweep_row> rows(n_cfg > 0 ? n_cfg : 1);
    const std::vector<int>& dev = gpu::sweep_device_list();
    const int per_dev = std::max(1, workers / static_cast<int>(dev.size()));
    check(dfm_sweep(dev.data(), static_cast<int>(dev.size()), per_dev, gpu::precision(),
                    ps.data(), static_cast<int>(ps.size()), &c, sched.scales.data(), it.data(),
                    static_cast<int32_t>(it.size()), etas.data(), static_cast<int>(etas.size()),
                    sigma_warps.data(), static_cast<int>(sigma_warps.size()), sigma_grads.data(),
                    static_cast<int>(sigma_grads.size()),
                    metric == SweepMetric::overlap ? DFM_SWEEP_OVERLAP : DFM_SWEEP_LOSS, 0, 1,
                    rows.data()));
    SweepResult r;
    r.etas = etas;
    r.sigma_warps = sigma_warps;
    r.sigma_grads = sigma_grads;
    r.heatmaps.assign(etas.size(), std::vector<std::vector<double>>(
                                       sigma_warps.size(),
                                       std::vector<double>(sigma_grads.size(), 0.0)));
    for (size_t k = 0; k < n_cfg; ++k) {
        const dfm_sweep_row& q = rows[k];
        SweepRow row;
        row.eta = q.eta;
        row.sigma_warp = q.sigma_warp;
        row.sigma_grad = q.sigma_grad;
        row.metric_mean = q.metric_mean;
        row.metric_sd = q.metric_sd;
        row.wall_ms = q.wall_ms;
        row.failed = q.failed != 0;
        row.error = q.error;
        r.rows.push_back(row);
        const size_t gi = k % sigma_grads.size();
        const size_t wi = (k / sigma_grads.size()) % sigma_warps.size();
        const size_t ei = k / (sigma_grads.size() * sigma_warps.size());
        r.heatmaps[ei][wi][gi] = q.metric_mean;
    }
    return r;
}

}  // namespace difform
