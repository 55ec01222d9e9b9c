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
        std::printf("precision %s: self records %zu, lncc loss %.5f -> %.5f\n",
                    prec == DFM_PREC_F64 ? "f64" : "f32", log.iterations.size(),
                    log2.iterations.front().loss, log2.final_loss);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures;
}
