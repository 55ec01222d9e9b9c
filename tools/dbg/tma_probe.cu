// Minimal TMA probe: load one 36x12 tile (offset -2,-2) of a 64x17x5 float
// volume into shared memory and print a checksum.  Variants via argv[1].
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_2404_01249_b200/csrc/tma_util.cuh"
using namespace dfm;
struct P { CUtensorMap m; float* out; int variant; };
__global__ void k(const __grid_constant__ P p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    if (p.variant & 1) prefetch_tmap(&p.m);
    mbar_init(&bar, 1);
    if (p.variant & 2) fence_mbar_init(); else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 36 * 12 * 4);
    tma_load_4d(smem, &p.m, &bar, -2, -2, 1, 0);
  }
  mbar_wait(&bar, 0);
  const float* s = reinterpret_cast<const float*>(smem);
  float acc = 0; for (int i = threadIdx.x; i < 36 * 12; i += blockDim.x) acc += s[i];
  atomicAdd(p.out, acc);
  if (threadIdx.x == 0) p.out[1] = (float)(reinterpret_cast<uintptr_t>(smem) & 127);
}
int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  const int nx = 64, ny = 17, nz = 5;
  std::vector<float> h(nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0f;
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 8); cudaMemset(o, 0, 8);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  P p{}; p.out = o; p.variant = variant;
  cuuint64_t dims[4] = {nx, ny, nz, 1}; cuuint64_t str[3] = {nx * 4, nx * ny * 4, (cuuint64_t)nx * ny * nz * 4};
  cuuint32_t box[4] = {36, 12, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&p.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d\n", (int)r);
  k<<<1, 128, 4096>>>(p);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[2]; cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("variant %d: %s sum=%g (expect %d) smem%%128=%g\n", variant, cudaGetErrorString(e), ho[0], 34 * 10, ho[1]);
  return 0;
}
