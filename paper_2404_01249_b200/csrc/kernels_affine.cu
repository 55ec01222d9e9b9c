// kernels_affine.cu — parameter gradient of the affine pre-alignment
// (affine.cpp:95-122): dL/dA_rc = sum_x (g_r / S_r) S_c x_c and
// dL/dt_r = sum_x g_r / S_r over the loss gradient g of the working grid.
// Twelve fp64 sums in one pass over g; fixed grid, fixed per-CTA tree and a
// fixed-order final pass, so the result is bit-stable run to run.
#include <cstdint>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"
#include "loop_ops.cuh"

namespace dfm {

namespace {

constexpr int kNA = 256;
constexpr int kBlocksA = 592;  // 4 CTAs per SM on 148 SMs

template <class T>
__global__ void __launch_bounds__(kNA) k_affine_grad(CPlanes3<T> g, Dims d, AffineS S,
                                                     double* __restrict__ partials) {
    __shared__ double sh[32];
    const int nd = d.ndim;
    double acc[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) acc[k] = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kNA) + threadIdx.x; i < d.n;
         i += static_cast<int64_t>(gridDim.x) * kNA) {
        const int x = static_cast<int>(i % d.nx);
        const int64_t rr = i / d.nx;
        const double xw[3] = {static_cast<double>(x), static_cast<double>(rr % d.ny),
                              static_cast<double>(rr / d.ny)};
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            if (r >= nd) break;
            const double gr = static_cast<double>(g.c[r][i]) / S.S[r];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (c < nd) acc[r * nd + c] += gr * S.S[c] * xw[c];
            acc[9 + r] += gr;
        }
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const double v = bsum<kNA>(acc[k], sh);
        if (threadIdx.x == 0) partials[k * gridDim.x + blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(1024) k_affine_final(const double* __restrict__ partials,
                                                       int nb, double* __restrict__ out) {
    __shared__ double sh[32];
    for (int k = 0; k < 12; ++k) {
        double a = 0.0;
        for (int j = threadIdx.x; j < nb; j += 1024) a += partials[k * nb + j];
        const double v = bsum<1024>(a, sh);
        if (threadIdx.x == 0) out[k] = v;
    }
}

}  // namespace

template <class T>
void launch_affine_grad(const Launch& L, CPlanes3<T> g, Dims d, AffineS S, double* partials,
                        double* out12) {
    k_affine_grad<T><<<kBlocksA, kNA, 0, L.stream>>>(g, d, S, partials);
    L.bump();
    k_affine_final<<<1, 1024, 0, L.stream>>>(partials, kBlocksA, out12);
    L.bump();
}

int affine_grad_partials() { return 12 * kBlocksA; }

template void launch_affine_grad<float>(const Launch&, CPlanes3<float>, Dims, AffineS, double*,
                                        double*);
template void launch_affine_grad<double>(const Launch&, CPlanes3<double>, Dims, AffineS,
                                         double*, double*);

}  // namespace dfm
