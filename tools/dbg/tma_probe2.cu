#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_2404_01249_b200/csrc/tma_util.cuh"
using namespace dfm;
struct P { CUtensorMap m3; CUtensorMap m4; const CUtensorMap* g4; const CUtensorMap* g3; float* out; int variant; };
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__global__ void k(const __grid_constant__ P p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const int v = p.variant;
  if (threadIdx.x == 0) {
    if (v == 4) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&bar)) : "memory"); }
    else {
      mbar_expect_tx(&bar, 36 * 12 * 4);
      const CUtensorMap* m = (v == 0) ? &p.m4 : (v == 1) ? p.g4 : (v == 2) ? &p.m3 : p.g3;
      if (v == 0 || v == 1) tma_load_4d(smem, m, &bar, -2, -2, 1, 0); else tma_load_3d(smem, m, &bar, -2, -2, 1);
    }
  }
  mbar_wait(&bar, 0);
  const float* s = reinterpret_cast<const float*>(smem);
  float acc = 0; for (int i = threadIdx.x; i < 36 * 12; i += blockDim.x) acc += s[i];
  atomicAdd(p.out, acc);
}
int main(int argc, char** argv) {
  const int nx = 64, ny = 17, nz = 5;
  std::vector<float> h(nx * ny * nz, 1.0f);
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 8);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  P p{};
  cuuint64_t dims[4] = {nx, ny, nz, 1}; cuuint64_t str[3] = {nx * 4, nx * ny * 4, (cuuint64_t)nx * ny * nz * 4};
  cuuint32_t box[4] = {36, 12, 1, 1}, es[4] = {1, 1, 1, 1};
  int r4 = enc(&p.m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int r3 = enc(&p.m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* g; cudaMalloc(&g, 2 * sizeof(CUtensorMap));
  cudaMemcpy(g, &p.m4, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  cudaMemcpy(g + 1, &p.m3, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  p.g4 = g; p.g3 = g + 1; p.out = o;
  printf("encode r4=%d r3=%d driver q=%d\n", r4, r3, (int)q);
  int drv = 0; cudaDriverGetVersion(&drv); int rt = 0; cudaRuntimeGetVersion(&rt); printf("driver %d runtime %d\n", drv, rt);
  for (int v = 4; v >= 0; --v) {
    cudaMemset(o, 0, 8); p.variant = v;
    k<<<1, 128, 4096>>>(p);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[2]; cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
    printf("variant %d: %s sum=%g\n", v, cudaGetErrorString(e), ho[0]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
