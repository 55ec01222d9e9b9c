// Throughput of scalar FFMA vs packed FFMA2 (fma.rn.f32x2, sm_100a) and
// the bit-identity of the two forms.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(unsigned long long r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
constexpr int NCH = 8, ITERS = 4096;
__global__ void k1(float* out, float w) {
    float a[2 * NCH];
#pragma unroll
    for (int j = 0; j < 2 * NCH; ++j) a[j] = threadIdx.x * 1e-3f + j;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int j = 0; j < 2 * NCH; ++j) a[j] = fmaf(a[j], w, 0.5f);
    float s = 0;
#pragma unroll
    for (int j = 0; j < 2 * NCH; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, float w) {
    unsigned long long a[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) a[j] = pk(threadIdx.x * 1e-3f + 2 * j, threadIdx.x * 1e-3f + 2 * j + 1);
    const unsigned long long ww = pk(w, w), hh = pk(0.5f, 0.5f);
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int j = 0; j < NCH; ++j) a[j] = fma2(a[j], ww, hh);
    float s = 0;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
        float x, y;
        upk(a[j], x, y);
        s += x;
        s += y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* d;
    cudaMalloc(&d, 148 * 8 * 256 * sizeof(float) * 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float h1[256], h2[256];
    for (int rep = 0; rep < 2; ++rep)
        for (int v = 0; v < 2; ++v) {
            cudaEventRecord(e0);
            if (v == 0) k1<<<148 * 8, 256>>>(d, 0.999f);
            else k2<<<148 * 8, 256>>>(d + 148 * 8 * 256, 0.999f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double flop = 2.0 * 148 * 8 * 256 * 2.0 * NCH * ITERS;
            if (rep) printf("%s: %.3f ms  %.1f TFLOP/s\n", v ? "FFMA2" : "FFMA ", ms, flop / ms / 1e9);
        }
    cudaMemcpy(h1, d, sizeof h1, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, d + 148 * 8 * 256, sizeof h2, cudaMemcpyDeviceToHost);
    printf("bit-identical: %s\n", memcmp(h1, h2, sizeof h1) == 0 ? "yes" : "no");
    return 0;
}
