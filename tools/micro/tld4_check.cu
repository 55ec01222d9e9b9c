// tld4 (texture gather) on a 2-D layered fp32 texture: which texel lands in
// which component, and the bit-identity of the corner values with plain loads.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 gather_a2d(cudaTextureObject_t t, int layer, float x, float y) {
    float4 r;
    asm volatile("tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %7}];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(t), "r"(layer), "f"(x), "f"(y));
    return r;
}
__global__ void k(cudaTextureObject_t t, int nx, int ny, int nz, const float* M, int* bad, float4* probe) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int n = nx * ny * nz;
    if (i >= n) return;
    int x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
    if (x >= nx - 1 || y >= ny - 1) return;
    float4 g = gather_a2d(t, z, x + 1.0f, y + 1.0f);
    const float* p = M + (z * ny + y) * nx + x;
    // expected D3D/GL order: x=(i0,j1) y=(i1,j1) z=(i1,j0) w=(i0,j0)
    if (g.w != p[0] || g.z != p[1] || g.x != p[nx] || g.y != p[nx + 1]) atomicAdd(bad, 1);
    if (i == nx + 1) *probe = g;
}
int main() {
    const int nx = 37, ny = 29, nz = 11, n = nx * ny * nz;
    float* h = new float[n];
    for (int i = 0; i < n; ++i) h[i] = 0.001f * i + 1e-7f * (i % 13);
    float* dM; cudaMalloc(&dM, n * 4); cudaMemcpy(dM, h, n * 4, cudaMemcpyHostToDevice);
    cudaArray_t arr;
    cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
    cudaMalloc3DArray(&arr, &cd, make_cudaExtent(nx, ny, nz), cudaArrayLayered);
    cudaMemcpy3DParms cp = {};
    cp.srcPtr = make_cudaPitchedPtr(dM, nx * 4, nx, ny);
    cp.dstArray = arr;
    cp.extent = make_cudaExtent(nx, ny, nz);
    cp.kind = cudaMemcpyDeviceToDevice;
    printf("copy: %s\n", cudaGetErrorString(cudaMemcpy3D(&cp)));
    cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeArray; rd.res.array.array = arr;
    cudaTextureDesc td = {};
    td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint; td.readMode = cudaReadModeElementType; td.normalizedCoords = 0;
    cudaTextureObject_t t; printf("tex: %s\n", cudaGetErrorString(cudaCreateTextureObject(&t, &rd, &td, nullptr)));
    int* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
    float4* pr; cudaMalloc(&pr, 16);
    k<<<(n + 255) / 256, 256>>>(t, nx, ny, nz, dM, bad, pr);
    int hb; float4 hp; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&hp, pr, 16, cudaMemcpyDeviceToHost);
    printf("kernel: %s  mismatches %d\n", cudaGetErrorString(cudaGetLastError()), hb);
    const int i = nx + 1;
    printf("probe (x=1,y=1,z=0): %.7g %.7g %.7g %.7g | p00 %.7g p10 %.7g p01 %.7g p11 %.7g\n", hp.x, hp.y, hp.z, hp.w,
           h[i], h[i + 1], h[i + nx], h[i + nx + 1]);
    return 0;
}
