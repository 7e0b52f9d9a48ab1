// Micro-benchmark: dependent kernel launches inside a captured graph with small vs ~4 KB
// kernel parameter structs (the multigrid kernels' MgArgs).
#include <cuda_runtime.h>
#include <cstdio>
template <int N> struct Big { long long v[N]; };
template <int N>
__global__ void step(Big<N> b, int* cnt) {
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(cnt, (int)b.v[N - 1]);
}
template <int N>
float run(int grid, int nk) {
  cudaStream_t s; cudaStreamCreate(&s);
  int* cnt; cudaMalloc(&cnt, 4);
  Big<N> b{}; b.v[N - 1] = 1;
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < nk; ++k) step<N><<<grid, 256, 0, s>>>(b, cnt);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e, s); cudaStreamSynchronize(s);
  float ms; cudaEventElapsedTime(&ms, a, e);
  return 1e3f * ms / (10 * nk);
}
int main() {
  for (int grid : {8, 148, 592}) {
    printf("grid %4d: 16 B %.3f us, 1 KB %.3f us, 4 KB %.3f us, 8 KB %.3f us per kernel\n", grid,
           run<2>(grid, 200), run<128>(grid, 200), run<512>(grid, 200), run<1024>(grid, 200));
  }
}
