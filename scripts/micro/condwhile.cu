// Micro-benchmark: dependent kernels inside a CUDA-graph WHILE conditional node (device-driven
// loop, no host round trips).  Prints the time per body kernel for a few grid sizes.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void step(int* cnt) {
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(cnt + 1, 1);
}
__global__ void last(cudaGraphConditionalHandle h, int* cnt, int iters) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int c = ++cnt[0];
    if (c >= iters) cudaGraphSetConditional(h, 0);
  }
}
int main() {
  const int iters = 200, nk = 20;
  for (int grid : {1, 148, 296, 592}) {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t n; cudaGraphAddNode(&n, g, nullptr, 0, &cp);
    cudaGraph_t bg = cp.conditional.phGraph_out[0];
    cudaStream_t s; cudaStreamCreate(&s);
    int* cnt; cudaMalloc(&cnt, 8); cudaMemset(cnt, 0, 8);
    cudaStreamBeginCaptureToGraph(s, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    for (int k = 0; k < nk - 1; ++k) step<<<grid, 256, 0, s>>>(cnt);
    last<<<grid, 256, 0, s>>>(h, cnt, iters);
    cudaStreamEndCapture(s, &bg);
    cudaGraphExec_t ge;
    cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) { printf("inst %s\n", cudaGetErrorString(e)); return 1; }
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaMemset(cnt, 0, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int hc[2]; cudaMemcpy(hc, cnt, 8, cudaMemcpyDeviceToHost);
    printf("grid %d: %d iterations x %d kernels: %.3f us per kernel (%s, count %d/%d)\n", grid, iters, nk,
           1e3 * ms / (iters * nk), cudaGetErrorString(cudaGetLastError()), hc[0], hc[1]);
  }
}
