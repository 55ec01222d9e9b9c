// Reference-style calls through the difform:: API, printing the numbers they
// return.  Built twice by oracle/Makefile `accept` — against the reference's
// own objects (dropin_numbers_ref) and against the B200 drop-in
// libdifform_b200.so (dropin_numbers_b200) — from this one source that
// includes only the reference's headers; tests/test_cpp_dropin.py compares
// the two outputs (fp64 on both sides).
#include <cmath>
#include <cstdio>
#include <random>

#include "difform/core.hpp"
#include "difform/diffeo.hpp"
#include "difform/interp.hpp"
#include "difform/optim.hpp"
#include "difform/pipeline.hpp"
#include "difform/similarity.hpp"

using namespace difform;

static ScalarImage blobs(const GridMeta& m, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    ScalarImage img = make_image(m);
    for (int b = 0; b < 6; ++b) {
        const double cx = u(rng) * m.dims[0], cy = u(rng) * m.dims[1], cz = u(rng) * m.dims[2];
        const double s = 2.0 + 3.0 * u(rng), a = 0.3 + 0.7 * u(rng);
        for (int64_t z = 0; z < m.dims[2]; ++z)
            for (int64_t y = 0; y < m.dims[1]; ++y)
                for (int64_t x = 0; x < m.dims[0]; ++x) {
                    const double d2 = (x - cx) * (x - cx) + (y - cy) * (y - cy) + (z - cz) * (z - cz);
                    img.at(x, y, z) += a * std::exp(-d2 / (2 * s * s));
                }
    }
    return img;
}

static double sum(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x;
    return s;
}
static double sumsq(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return s;
}

int main() {
    const GridMeta m = make_meta_3d(20, 18, 16);
    const ScalarImage F = blobs(m, 3), M = blobs(m, 4);
    DisplacementField u = new_identity_field(m);
    for (size_t i = 0; i < u.data.size(); ++i) u.data[i] = 0.3 * std::sin(0.37 * i);
    const LossEval l = lncc_eval(F, M, u, 2);
    std::printf("lncc_value %.17g\nlncc_grad_sumsq %.17g\n", l.value, sumsq(l.grad.data));
    const LossEval s = ssd_eval(F, M, u);
    std::printf("ssd_value %.17g\nssd_grad_sum %.17g\n", s.value, sum(s.grad.data));
    const VectorField g = gaussian_smooth_field(l.grad, 1.0);
    std::printf("smooth_sumsq %.17g\n", sumsq(g.data));
    AdaptiveState st = make_adaptive_state(m, 0.9, 0.99, 1e-8);
    const VectorField dir = adam_step(st, eulerian_direction(g, u, false));
    std::printf("adam_dir_sum %.17g\nadam_t %lld\n", sum(dir.data), static_cast<long long>(st.t));
    const DisplacementField up = apply_update(u, dir, 0.5, 0.5, 0.5);
    std::printf("apply_sumsq %.17g\n", sumsq(up.data));
    std::printf("compose_sum %.17g\n", sum(compose(u, up).data));
    std::printf("jacdet_sum %.17g\n", sum(jacobian_det(up).data));
    std::printf("warp_sum %.17g\n", sum(warp_image(M, up).data));
    const ScalarImage d2 = downsample_image(F, 2.0);
    std::printf("down2_sum %.17g\n", sum(d2.data));
    RegistrationConfig cfg;
    cfg.loss = LossKind::lncc;
    cfg.beta2 = 0.99;
    cfg.eta = 0.2;
    cfg.conv_window = 100;
    PyramidSchedule sched{{2.0, 1.0}, {20, 10}};
    const auto [phi, log] = register_images(F, M, cfg, sched);
    std::printf("register_records %zu\nregister_final_loss %.17g\nregister_field_sumsq %.17g\n",
                log.iterations.size(), log.final_loss, sumsq(phi.data));
    return 0;
}
