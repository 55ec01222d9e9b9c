// Per-kernel cost of dependent launches inside a CUDA graph on this GPU:
// N empty kernels (grid G x 256 threads, optional dynamic shared memory)
// captured back to back, the graph replayed; time per kernel node.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p, 1);
}
int main() {
    const int N = 32;
    int* d;
    cudaMalloc(&d, 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int grids[] = {148, 444, 840};
    const int smems[] = {0, 48 * 1024};
    for (int gi = 0; gi < 3; ++gi)
        for (int si = 0; si < 2; ++si) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
            for (int k = 0; k < N; ++k) k_empty<<<grids[gi], 256, smems[si], s>>>(d);
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t e;
            cudaGraphInstantiate(&e, g, 0);
            for (int w = 0; w < 5; ++w) cudaGraphLaunch(e, s);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, s);
            const int reps = 50;
            for (int r = 0; r < reps; ++r) cudaGraphLaunch(e, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("grid %4d x 256, smem %5d: %.2f us per kernel node\n", grids[gi], smems[si],
                   ms * 1e3 / (reps * N));
            cudaGraphExecDestroy(e);
            cudaGraphDestroy(g);
        }
    return 0;
}
