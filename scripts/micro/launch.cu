// Microbenchmark: per-kernel cost of dependent launches inside a CUDA graph, with and without
// programmatic dependent launch (PDL), for grids of 148..2368 CTAs.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_touch(double* buf, int n, int pdl) {
  if (pdl) cudaGridDependencySynchronize();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] += 1.0;
  if (pdl) cudaTriggerProgrammaticLaunchCompletion();
}

int main() {
  double* buf;
  const int n = 1 << 20;
  cudaMalloc(&buf, n * sizeof(double));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {148, 592, 2368}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      const int nk = 256;
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < nk; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_touch, buf, grid * 256, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphExec_t ge;
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %5d pdl %d: %.3f us per dependent kernel (%s)\n", grid, pdl,
             1e3 * ms / (10 * nk), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
