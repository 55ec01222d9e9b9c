// C++ drop-in test: reference-style call sites (difform::...) compiled against
// include/difform_b200.hpp and linked to libdifform_cuda.so.  Mirrors the
// reference's test_pipeline.cpp properties (record count of a self
// registration, error classes, fold detection).  Exit code = failures.
#include <cmath>
#include <cstdio>
#include <limits>
#include <stdexcept>

#include "difform_b200.hpp"

using namespace difform;

static int failures = 0;
#define EXPECT(c)                                                              \
    do {                                                                       \
        if (!(c)) {                                                            \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

static ScalarImage smooth(const GridMeta& m, double phase) {
    ScalarImage img{m, std::vector<double>(static_cast<size_t>(m.voxel_count()))};
    for (int64_t z = 0; z < m.dims[2]; ++z)
        for (int64_t y = 0; y < m.dims[1]; ++y)
            for (int64_t x = 0; x < m.dims[0]; ++x)
                img.data[static_cast<size_t>((z * m.dims[1] + y) * m.dims[0] + x)] =
                    0.5 + 0.2 * std::sin(0.4 * x + phase) * std::cos(0.3 * y) +
                    0.1 * std::sin(0.5 * z + 0.7 * x);
    return img;
}

int main() {
    for (int prec : {DFM_PREC_F64, DFM_PREC_F32}) {
        gpu::set_precision(prec);
        const GridMeta m = make_meta_3d(16, 16, 16);
        const ScalarImage F = smooth(m, 0.0);

        // self registration: zero loss, the monitor ends each scale after
        // conv_window + 1 records (test_pipeline.cpp:69-93)
        RegistrationConfig cfg;
        auto [phi, log] = register_images(F, F, cfg, PyramidSchedule::defaults());
        EXPECT(log.iterations.size() == 3u * (cfg.conv_window + 1));
        for (const auto& r : log.iterations) EXPECT(r.loss == 0.0);
        double worst = 0.0;
        for (double v : phi.data) worst = std::max(worst, std::abs(v));
        EXPECT(worst < 0.1);

        // a shifted pair registers and reduces the loss (LNCC)
        const ScalarImage M = smooth(m, 0.6);
        cfg.loss = LossKind::lncc;
        cfg.conv_window = 100;
        auto [phi2, log2] = register_images(F, M, cfg, {{2.0, 1.0}, {20, 20}});
        EXPECT(log2.iterations.size() == 40u);
        EXPECT(log2.final_loss < log2.iterations.front().loss);
        EXPECT(log2.final_singularity_fraction == 0.0);

        // apply the result with the warp operators
        const ScalarImage W = warp_image(M, phi2);
        EXPECT(W.data.size() == M.data.size());
        const double sf = singularity_fraction(phi2);
        EXPECT(sf == 0.0);

        // error classes (std::invalid_argument / std::runtime_error)
        bool threw = false;
        try {
            lncc_eval(F, M, phi2, 9);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
        ScalarImage bad = F;
        bad.data[7] = std::numeric_limits<double>::quiet_NaN();
        threw = false;
        try {
            register_images(bad, M, RegistrationConfig{}, {{1.0}, {3}});
        } catch (const std::runtime_error&) {
            threw = true;
        }
        EXPECT(threw);
        // SVF: exp_map of zero is zero; pullback of zero is zero; SVF registration runs
        VelocityField v0 = phi2;
        for (double& x : v0.data) x = 0.0;
        const DisplacementField e0 = exp_map(v0, 4);
        for (double x : e0.data) EXPECT(x == 0.0);
        const VectorField p0 = svf_pullback(phi2, v0, 4);
        for (double x : p0.data) EXPECT(x == 0.0);
        RegistrationConfig scfg = cfg;
        scfg.mode = RegMode::svf;
        scfg.svf_M = 4;
        auto [phis, logs] = register_images(F, M, scfg, {{2.0, 1.0}, {10, 10}});
        EXPECT(logs.iterations.size() == 20u);
        EXPECT(logs.final_loss < logs.iterations.front().loss);

        // affine: identity maps to a zero field; registration of a shifted copy
        const DisplacementField az = affine_to_field(identity_affine(3), m);
        for (double x : az.data) EXPECT(x == 0.0);
        const AffineResult ar = affine_register(F, M, LossKind::lncc, {2.0, 1.0}, {15, 10}, 0.01);
        EXPECT(!ar.diverged && ar.iterations == 25);
        EXPECT(std::abs(affine_det(ar.transform)) > 0.5);
        const AffineGrad ag =
            affine_param_gradient(F, M, LossKind::ssd, identity_affine(3), {1.0, 1.0, 1.0});
        EXPECT(std::isfinite(ag.value) && ag.value > 0.0);

        // evaluation: a label map against itself; landmarks through phi = 0
        LabelImage L{m, std::vector<int32_t>(static_cast<size_t>(m.voxel_count()), 0)};
        for (size_t i = 0; i < L.data.size(); ++i) L.data[i] = static_cast<int32_t>(i % 5);
        const OverlapReport ov = overlap_report(L, L);
        EXPECT(ov.regions.size() == 4u && ov.mo_mean == 1.0 && ov.vs_klein == 0.0);
        LandmarkSet a(3), b(3);
        for (int i = 0; i < 3; ++i) {
            a[static_cast<size_t>(i)].point_mm = {1.0 + i, 2.0, 3.0};
            b[static_cast<size_t>(i)].point_mm = {1.0 + i, 2.0, 3.0 + i};
        }
        const LandmarkErrors le = landmark_error(a, b, e0, m, m);
        EXPECT(std::abs(le.max - 2.0) < 1e-12 && std::abs(le.mean - 1.0) < 1e-12);

        // sweep over 2 x 1 x 1 configs on the pair (loss metric)
        std::vector<SweepPair> pairs(1);
        pairs[0].fixed = F;
        pairs[0].moving = M;
        const SweepResult sw = sweep(pairs, cfg, {{2.0, 1.0}, {5, 5}}, {0.3, 0.6}, {0.5}, {1.0},
                                     SweepMetric::loss, 2);
        EXPECT(sw.rows.size() == 2u && !sw.rows[0].failed && !sw.rows[1].failed);
        EXPECT(sw.heatmaps[1][0][0] == sw.rows[1].metric_mean);

        std::printf("precision %s: self records %zu, lncc loss %.5f -> %.5f\n",
                    prec == DFM_PREC_F64 ? "f64" : "f32", log.iterations.size(),
                    log2.iterations.front().loss, log2.final_loss);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures;
}
