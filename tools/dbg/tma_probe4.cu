#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2404_01249_b200/csrc/tma_util.cuh"
using namespace dfm;
struct P { CUtensorMap m; float* out; int v; const float* src; int cx, cy, cz; };
__global__ void k(const __grid_constant__ P p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const int v = p.v;
  int bytes = (v & 1) ? 32 * 8 * 4 : 36 * 12 * 4;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, bytes);
    if (v & 4) {  // plain bulk copy (UBLKCP)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(smem)), "l"(p.src), "r"(bytes), "r"(smem_u32(&bar)) : "memory");
    } else {
      const int c0 = p.cx, c1 = p.cy;
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(&p.m)), "r"(smem_u32(&bar)), "r"(c0), "r"(c1), "r"(p.cz) : "memory");
    }
  }
  mbar_wait(&bar, 0);
  const float* s = reinterpret_cast<const float*>(smem);
  float acc = 0; for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) acc += s[i];
  atomicAdd(p.out, acc);
}
int main(int argc, char** argv) {
  const int v = atoi(argv[1]);
  const int nx = 64, ny = 17, nz = 5;
  std::vector<float> h(nx * ny * nz, 1.0f);
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 8); cudaMemset(o, 0, 8);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  P p{}; p.out = o; p.v = v; p.src = d; p.cx = atoi(argv[2]); p.cy = atoi(argv[3]); p.cz = atoi(argv[4]);
  cuuint64_t dims[3] = {nx, ny, nz}; cuuint64_t str[2] = {nx * 4, nx * ny * 4};
  cuuint32_t box[3] = {(v & 1) ? 32u : 36u, (v & 1) ? 8u : 12u, 1}, es[3] = {1, 1, 1};
  int r = enc(&p.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaError_t e;
  if (v & 8) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 4096;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, p);
  } else { k<<<1, 128, 4096>>>(p); e = cudaGetLastError(); }
  cudaError_t e2 = cudaDeviceSynchronize();
  float ho[2]; cudaMemcpy(ho, o, 8, cudaMemcpyDeviceToHost);
  printf("c=(%d,%d,%d) variant %2d (box%s coords%s %s%s): enc=%d launch=%s sync=%s sum=%g\n", p.cx, p.cy, p.cz, v, (v&1)?"32x8":"36x12", (v&2)?"0":"-2",
     (v&4)?"BULK":"TENSOR", (v&8)?" cluster":"", r, cudaGetErrorString(e), cudaGetErrorString(e2), ho[0]);
  return 0;
}
