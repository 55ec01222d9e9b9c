// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI veneer over the UNMODIFIED reference library compiled in place from
// /root/reference/proj/src (see oracle/Makefile).  It lets the Python tests
// and bench.py's CPU-baseline leg drive the reference's own implementation of
// the hot path with the same argument conventions as include/difform_gpu.h
// (host AoS doubles, dfm_grid/dfm_config structs, 0/1/2 status codes).
//
// Nothing in the product (paper_2404_01249_b200/) links or loads this.
// Output goes to oracle/_ref/libdifform_ref.so (git-ignored, travels to the
// GPU box with the snapshot).
#include <cstring>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "difform/affine.hpp"
#include "difform/analysis.hpp"
#include "difform/core.hpp"
#include "difform/diffeo.hpp"
#include "difform/interp.hpp"
#include "difform/optim.hpp"
#include "difform/pipeline.hpp"
#include "difform/similarity.hpp"

#include "../include/difform_gpu.h"

using namespace difform;

namespace {

thread_local std::string g_err;

GridMeta to_meta(const dfm_grid* g) {
    GridMeta m;
    m.ndim = g->ndim;
    for (int a = 0; a < 3; ++a) {
        m.dims[a] = g->dims[a];
        m.spacing[a] = g->spacing[a];
        m.origin[a] = g->origin[a];
    }
    return m;
}

void from_meta(const GridMeta& m, dfm_grid* g) {
    g->ndim = m.ndim;
    for (int a = 0; a < 3; ++a) {
        g->dims[a] = m.dims[a];
        g->spacing[a] = m.spacing[a];
        g->origin[a] = m.origin[a];
    }
}

ScalarImage to_image(const dfm_grid* g, const double* p) {
    ScalarImage s;
    s.meta = to_meta(g);
    s.data.assign(p, p + s.meta.voxel_count());
    return s;
}

VectorField to_field(const dfm_grid* g, const double* p) {
    VectorField f;
    f.meta = to_meta(g);
    f.data.assign(p, p + f.meta.voxel_count() * f.meta.ndim);
    return f;
}

void put(const std::vector<double>& v, double* out) {
    if (out)
        std::memcpy(out, v.data(), v.size() * sizeof(double));
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

RegistrationConfig to_cfg(const dfm_config* c) {
    RegistrationConfig r;
    r.loss = static_cast<LossKind>(c->loss);
    r.lncc_radius = c->lncc_radius;
    r.eta = c->eta;
    r.sigma_grad = c->sigma_grad;
    r.sigma_warp = c->sigma_warp;
    r.use_jac = c->use_jac != 0;
    r.mode = static_cast<RegMode>(c->mode);
    r.svf_M = c->svf_M;
    r.beta1 = c->beta1;
    r.beta2 = c->beta2;
    r.eps_adam = c->eps_adam;
    r.step_cap = c->step_cap;
    r.conv_window = c->conv_window;
    r.conv_tol = c->conv_tol;
    r.seed = c->seed;
    return r;
}

}  // namespace

extern "C" {

size_t dfmref_last_error(char* buf, size_t cap) {
    if (buf && cap) {
        const size_t n = std::min(cap - 1, g_err.size());
        std::memcpy(buf, g_err.data(), n);
        buf[n] = 0;
    }
    return g_err.size();
}

int dfmref_downsample_image(const dfm_grid* g, const double* img, const double factor[3],
                            dfm_grid* out_grid, double* out) {
    return guarded([&] {
        const ScalarImage r =
            downsample_image(to_image(g, img), {factor[0], factor[1], factor[2]});
        from_meta(r.meta, out_grid);
        put(r.data, out);
    });
}

int dfmref_sample_linear_points(const dfm_grid* g, const double* img, int64_t npts,
                                const double* pts, double* values, double* grads) {
    return guarded([&] {
        const ScalarImage s = to_image(g, img);
        for (int64_t i = 0; i < npts; ++i) {
            const std::array<double, 3> p{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
            values[i] = sample_linear(s, p);
            if (grads) {
                const auto gr = sample_linear_gradient(s, p);
                for (int c = 0; c < 3; ++c)
                    grads[3 * i + c] = gr[c];
            }
        }
    });
}

int dfmref_warp_image(const dfm_grid* g, const double* img, const double* phi, double* out) {
    return guarded([&] { put(warp_image(to_image(g, img), to_field(g, phi)).data, out); });
}

int dfmref_warp_labels(const dfm_grid* g, const int32_t* labels, const double* phi,
                       int32_t* out) {
    return guarded([&] {
        LabelImage L;
        L.meta = to_meta(g);
        L.data.assign(labels, labels + L.meta.voxel_count());
        const LabelImage r = warp_labels(L, to_field(g, phi));
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(int32_t));
    });
}

int dfmref_compose(const dfm_grid* g, const double* phi, const double* psi, double* out) {
    return guarded([&] { put(compose(to_field(g, phi), to_field(g, psi)).data, out); });
}

static AffineTransform to_affine(int ndim, const double A[9], const double t[3]) {
    AffineTransform T;
    T.ndim = ndim;
    for (int k = 0; k < 9; ++k) T.A[k] = A[k];
    for (int k = 0; k < 3; ++k) T.t[k] = t[k];
    return T;
}

int dfmref_affine_to_field(const dfm_grid* g, const double A[9], const double t[3],
                           double* out) {
    return guarded([&] { put(affine_to_field(to_affine(g->ndim, A, t), to_meta(g)).data, out); });
}

int dfmref_affine_param_gradient(const dfm_grid* g, const double* fixed, const double* moving,
                                 int loss, const double A[9], const double t[3],
                                 const double S[3], int lncc_radius, double* value, double dA[9],
                                 double dt[3]) {
    return guarded([&] {
        const AffineGrad r = affine_param_gradient(
            to_image(g, fixed), to_image(g, moving), static_cast<LossKind>(loss),
            to_affine(g->ndim, A, t), {S[0], S[1], S[2]}, lncc_radius);
        *value = r.value;
        for (int k = 0; k < 9; ++k) dA[k] = r.dA[k];
        for (int k = 0; k < 3; ++k) dt[k] = r.dt[k];
    });
}

int dfmref_affine_register(const dfm_grid* g, const double* fixed, const double* moving,
                           int loss, const double* scales, const int32_t* iters,
                           int32_t nscales, double eta, int lncc_radius,
                           dfm_affine_result* out) {
    return guarded([&] {
        const AffineResult r = affine_register(
            to_image(g, fixed), to_image(g, moving), static_cast<LossKind>(loss),
            std::vector<double>(scales, scales + nscales), std::vector<int>(iters, iters + nscales),
            eta, lncc_radius);
        out->ndim = r.transform.ndim;
        for (int k = 0; k < 9; ++k) out->A[k] = r.transform.A[k];
        for (int k = 0; k < 3; ++k) out->t[k] = r.transform.t[k];
        out->loss = r.loss;
        out->diverged = r.diverged ? 1 : 0;
        out->iterations = r.iterations;
    });
}

int dfmref_exp_map(const dfm_grid* g, const double* v, int M, double* out) {
    return guarded([&] { put(exp_map(to_field(g, v), M).data, out); });
}

int dfmref_svf_pullback(const dfm_grid* g, const double* v, const double* grad_phi, int M,
                        double* out) {
    return guarded([&] { put(svf_pullback(to_field(g, v), to_field(g, grad_phi), M).data, out); });
}

int dfmref_jacobian_det(const dfm_grid* g, const double* phi, double* out) {
    return guarded([&] { put(jacobian_det(to_field(g, phi)).data, out); });
}

int dfmref_gaussian_smooth(const dfm_grid* g, const double* img, const double sigma[3],
                           double* out) {
    return guarded([&] {
        put(gaussian_smooth(to_image(g, img), {sigma[0], sigma[1], sigma[2]}).data, out);
    });
}

int dfmref_gaussian_smooth_field(const dfm_grid* g, const double* f, const double sigma[3],
                                 double* out) {
    return guarded([&] {
        put(gaussian_smooth_field(to_field(g, f), {sigma[0], sigma[1], sigma[2]}).data, out);
    });
}

int dfmref_upsample_field(const dfm_grid* g, const double* phi, const dfm_grid* ng,
                          double* out) {
    return guarded([&] {
        put(upsample_field(to_field(g, phi), to_meta(ng), UpsampleMethod::linear).data, out);
    });
}

int dfmref_resample_field_linear(const dfm_grid* g, const double* f, const dfm_grid* ng,
                                 double* out) {
    return guarded([&] { put(resample_field_linear(to_field(g, f), to_meta(ng)).data, out); });
}

int dfmref_resample_displacement(const dfm_grid* g, const double* phi, const dfm_grid* ng,
                                 double* out) {
    return guarded([&] { put(resample_displacement(to_field(g, phi), to_meta(ng)).data, out); });
}

int dfmref_ssd_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                    const double* moving, const double* phi, double* value, double* grad) {
    return guarded([&] {
        const LossEval ev = ssd_eval(to_image(fg, fixed), to_image(mg, moving), to_field(fg, phi));
        *value = ev.value;
        put(ev.grad.data, grad);
    });
}

int dfmref_lncc_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                     const double* moving, const double* phi, int r, double* value,
                     double* grad) {
    return guarded([&] {
        const LossEval ev =
            lncc_eval(to_image(fg, fixed), to_image(mg, moving), to_field(fg, phi), r);
        *value = ev.value;
        put(ev.grad.data, grad);
    });
}

int dfmref_dice_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                     const double* moving, const double* phi, double* value, double* grad) {
    return guarded([&] {
        const LossEval ev =
            dice_soft_eval(to_image(fg, fixed), to_image(mg, moving), to_field(fg, phi));
        *value = ev.value;
        put(ev.grad.data, grad);
    });
}

int dfmref_adam_step(const dfm_grid* g, double* m, double* nu, int64_t* t, double b1,
                     double b2, double eps, const double* v, double* dir) {
    return guarded([&] {
        AdaptiveState s;
        s.m = to_field(g, m);
        s.nu = to_field(g, nu);
        s.t = *t;
        s.beta1 = b1;
        s.beta2 = b2;
        s.eps = eps;
        const VectorField d = adam_step(s, to_field(g, v));
        put(s.m.data, m);
        put(s.nu.data, nu);
        *t = s.t;
        put(d.data, dir);
    });
}

int dfmref_upsample_state(const dfm_grid* g, const double* m, const double* nu,
                          const dfm_grid* ng, double* m_out, double* nu_out) {
    return guarded([&] {
        AdaptiveState s;
        s.m = to_field(g, m);
        s.nu = to_field(g, nu);
        const AdaptiveState r = upsample_state(s, to_meta(ng));
        put(r.m.data, m_out);
        put(r.nu.data, nu_out);
    });
}

int dfmref_eulerian_direction(const dfm_grid* g, const double* grad, const double* phi,
                              int use_jac, double* out) {
    return guarded([&] {
        put(eulerian_direction(to_field(g, grad), to_field(g, phi), use_jac != 0).data, out);
    });
}

int dfmref_apply_update(const dfm_grid* g, const double* phi, const double* v, double eta,
                        double sigma_warp, double cap, double* out) {
    return guarded([&] {
        put(apply_update(to_field(g, phi), to_field(g, v), eta, sigma_warp, cap).data, out);
    });
}

int dfmref_singularity_fraction(const dfm_grid* g, const double* phi, double* frac) {
    return guarded([&] { *frac = singularity_fraction(to_field(g, phi)); });
}

// register_images, images given as doubles; init none/affine/field.
int dfmref_register(const dfm_grid* g, const double* fixed, const double* moving,
                    const dfm_config* cfg, const double* scales, const int32_t* iters,
                    int32_t nscales, const dfm_init* init, double* out_field,
                    dfm_iter_record* records, int64_t max_records, dfm_runlog* log) {
    return guarded([&] {
        PyramidSchedule sched;
        for (int i = 0; i < nscales; ++i) {
            sched.scales.push_back(scales[i]);
            sched.iterations.push_back(iters[i]);
        }
        RegInit ri = std::monostate{};
        if (init && init->kind == DFM_INIT_AFFINE) {
            AffineTransform T;
            T.ndim = init->affine_ndim;
            for (int i = 0; i < 9; ++i)
                T.A[i] = init->A[i];
            for (int i = 0; i < 3; ++i)
                T.t[i] = init->t[i];
            ri = T;
        } else if (init && init->kind == DFM_INIT_FIELD) {
            ri = to_field(&init->field_grid, init->field);
        }
        auto [phi, rl] = register_images(to_image(g, fixed), to_image(g, moving), to_cfg(cfg),
                                         sched, ri);
        put(phi.data, out_field);
        const int64_t n = static_cast<int64_t>(rl.iterations.size());
        for (int64_t i = 0; i < n && i < max_records; ++i) {
            const IterationRecord& r = rl.iterations[static_cast<size_t>(i)];
            records[i].scale_index = r.scale_index;
            records[i].scale = r.scale;
            records[i].iter = r.iter;
            records[i].global_iter = r.global_iter;
            records[i].loss = r.loss;
            records[i].max_step = r.max_step;
            records[i].wall_ms = r.wall_ms;
        }
        log->n_records = std::min(n, max_records);
        log->n_total = n;
        log->final_loss = rl.final_loss;
        log->final_singularity_fraction = rl.final_singularity_fraction;
        log->total_ms = rl.total_ms;
    });
}

// overlap_report (analysis.cpp:169-247): MO (Dice) mean and Klein aggregate.
int dfmref_overlap_dice(const dfm_grid* g, const int32_t* warped, const int32_t* fixed,
                        double* mo_mean, double* mo_klein) {
    return guarded([&] {
        LabelImage W, F;
        W.meta = F.meta = to_meta(g);
        const int64_t n = W.meta.voxel_count();
        W.data.assign(warped, warped + n);
        F.data.assign(fixed, fixed + n);
        const OverlapReport r = overlap_report(W, F);
        *mo_mean = r.mo_mean;
        *mo_klein = r.mo_klein;
    });
}

int dfmref_sweep(const dfm_sweep_pair* pairs, int npairs, const dfm_config* base,
                 const double* scales, const int32_t* iters, int32_t nscales, const double* etas,
                 int n_eta, const double* sws, int n_sw, const double* sgs, int n_sg, int metric,
                 int workers, dfm_sweep_row* rows) {
    return guarded([&] {
        std::vector<SweepPair> ps(static_cast<size_t>(npairs));
        for (int p = 0; p < npairs; ++p) {
            ps[p].fixed = to_image(pairs[p].grid, pairs[p].fixed);
            ps[p].moving = to_image(pairs[p].grid, pairs[p].moving);
            const int64_t n = ps[p].fixed.meta.voxel_count();
            if (pairs[p].fixed_labels) {
                LabelImage L;
                L.meta = ps[p].fixed.meta;
                L.data.assign(pairs[p].fixed_labels, pairs[p].fixed_labels + n);
                ps[p].fixed_labels = L;
            }
            if (pairs[p].moving_labels) {
                LabelImage L;
                L.meta = ps[p].fixed.meta;
                L.data.assign(pairs[p].moving_labels, pairs[p].moving_labels + n);
                ps[p].moving_labels = L;
            }
        }
        PyramidSchedule sched;
        sched.scales.assign(scales, scales + nscales);
        sched.iterations.assign(iters, iters + nscales);
        const SweepResult r =
            sweep(ps, to_cfg(base), sched, std::vector<double>(etas, etas + n_eta),
                  std::vector<double>(sws, sws + n_sw), std::vector<double>(sgs, sgs + n_sg),
                  metric == DFM_SWEEP_OVERLAP ? SweepMetric::overlap : SweepMetric::loss, workers);
        for (size_t k = 0; k < r.rows.size(); ++k) {
            dfm_sweep_row& o = rows[k];
            std::memset(&o, 0, sizeof(o));
            const SweepRow& q = r.rows[k];
            o.eta = q.eta;
            o.sigma_warp = q.sigma_warp;
            o.sigma_grad = q.sigma_grad;
            o.metric_mean = q.metric_mean;
            o.metric_sd = q.metric_sd;
            o.wall_ms = q.wall_ms;
            o.failed = q.failed ? 1 : 0;
            o.computed = 1;
            std::strncpy(o.error, q.error.c_str(), sizeof(o.error) - 1);
        }
    });
}

int dfmref_overlap_report(const dfm_grid* gw, const int32_t* warped, const dfm_grid* gf,
                          const int32_t* fixed, dfm_overlap_summary* rep,
                          dfm_region_overlap* regions, int64_t cap) {
    return guarded([&] {
        LabelImage W, F;
        W.meta = to_meta(gw);
        F.meta = to_meta(gf);
        W.data.assign(warped, warped + W.meta.voxel_count());
        F.data.assign(fixed, fixed + F.meta.voxel_count());
        const OverlapReport r = overlap_report(W, F);
        rep->to_mean = r.to_mean;
        rep->mo_mean = r.mo_mean;
        rep->fn_mean = r.fn_mean;
        rep->fp_mean = r.fp_mean;
        rep->vs_mean = r.vs_mean;
        rep->to_klein = r.to_klein;
        rep->mo_klein = r.mo_klein;
        rep->fn_klein = r.fn_klein;
        rep->fp_klein = r.fp_klein;
        rep->vs_klein = r.vs_klein;
        rep->n_regions = static_cast<int64_t>(r.regions.size());
        for (size_t k = 0; k < r.regions.size() && static_cast<int64_t>(k) < cap; ++k) {
            const RegionOverlap& q = r.regions[k];
            dfm_region_overlap& o = regions[k];
            o.label = q.label;
            o.has_to = q.has_to;
            o.has_fn = q.has_fn;
            o.has_fp = q.has_fp;
            o.fixed_count = q.fixed_count;
            o.warped_count = q.warped_count;
            o.intersection = q.intersection;
            o.to = q.to;
            o.mo = q.mo;
            o.fn = q.fn;
            o.fp = q.fp;
            o.vs = q.vs;
        }
    });
}

int dfmref_landmark_error(const dfm_grid* fg, const dfm_grid* mg, const dfm_grid* pg,
                          const double* phi, int64_t n, const double* fixed_mm,
                          const double* moving_mm, double* dist, double* mean, double* mx) {
    return guarded([&] {
        LandmarkSet a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) {
                a[static_cast<size_t>(i)].point_mm[k] = fixed_mm[3 * i + k];
                b[static_cast<size_t>(i)].point_mm[k] = moving_mm[3 * i + k];
            }
        const LandmarkErrors r =
            landmark_error(a, b, to_field(pg, phi), to_meta(fg), to_meta(mg));
        for (int64_t i = 0; i < n; ++i) dist[i] = r.distances_mm[static_cast<size_t>(i)];
        *mean = r.mean;
        *mx = r.max;
    });
}

}  // extern "C"
