// kernels_eval.cu — evaluation epilogue on the device (analysis.cpp:169-247):
// per-label voxel counts |S_r|, |T_r|, |S_r n T_r| of a warped and a fixed
// label map.  Integer counts (atomics on integers are order-independent), so
// the report the host assembles from them is exactly the reference's.
#include <cstdint>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"

namespace dfm {

namespace {

constexpr int kNE = 256;
constexpr int kSmemLabels = 4096;  // privatised shared-memory histogram up to this label

__global__ void k_label_max(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                            int64_t n, int* __restrict__ out) {
    int m = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kNE) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kNE)
        m = max(m, max(a[i], b[i]));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// counts[0][l] = |S_l| (warped), counts[1][l] = |T_l| (fixed), counts[2][l] = |S_l n T_l|
__global__ void k_label_hist(const int32_t* __restrict__ warped, const int32_t* __restrict__ fixed,
                             int64_t n, int maxl, unsigned long long* __restrict__ counts) {
    extern __shared__ unsigned int sh[];  // 3 * (maxl + 1) when small
    const bool priv = maxl < kSmemLabels;
    const int L = maxl + 1;
    if (priv)
        for (int k = threadIdx.x; k < 3 * L; k += kNE) sh[k] = 0u;
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kNE) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kNE) {
        const int32_t s = warped[i], t = fixed[i];
        if (priv) {
            if (s > 0) atomicAdd(&sh[s], 1u);
            if (t > 0) atomicAdd(&sh[L + t], 1u);
            if (s > 0 && s == t) atomicAdd(&sh[2 * L + s], 1u);
        } else {
            if (s > 0) atomicAdd(&counts[s], 1ull);
            if (t > 0) atomicAdd(&counts[L + t], 1ull);
            if (s > 0 && s == t) atomicAdd(&counts[2 * L + s], 1ull);
        }
    }
    if (priv) {
        __syncthreads();
        for (int k = threadIdx.x; k < 3 * L; k += kNE)
            if (sh[k]) atomicAdd(&counts[k], static_cast<unsigned long long>(sh[k]));
    }
}

}  // namespace

int launch_label_max(const Launch& L, const int32_t* a, const int32_t* b, int64_t n, int* out) {
    cudaMemsetAsync(out, 0, sizeof(int), L.stream);
    const int64_t want = (n + kNE - 1) / kNE;
    const int blocks = static_cast<int>(want < 1184 ? (want > 0 ? want : 1) : 1184);
    k_label_max<<<blocks, kNE, 0, L.stream>>>(a, b, n, out);
    L.bump();
    return blocks;
}

void launch_label_hist(const Launch& L, const int32_t* warped, const int32_t* fixed, int64_t n,
                       int maxl, unsigned long long* counts) {
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 3 * (static_cast<size_t>(maxl) + 1),
                    L.stream);
    const int64_t want = (n + kNE - 1) / kNE;
    const int blocks = static_cast<int>(want < 592 ? (want > 0 ? want : 1) : 592);
    const size_t smem = maxl < kSmemLabels ? sizeof(unsigned) * 3 * (maxl + 1) : 0;
    k_label_hist<<<blocks, kNE, smem, L.stream>>>(warped, fixed, n, maxl, counts);
    L.bump();
}

}  // namespace dfm
