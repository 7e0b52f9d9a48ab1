// Microbenchmark: cost of a cooperative grid barrier on this GPU (cg::grid_group::sync vs a
// hand-rolled sense-reversing barrier), for several grid sizes.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cgsync(int n, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < n; ++i) { acc += i; g.sync(); }
  if (acc < 0) out[0] = acc;
}

__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;
__device__ __forceinline__ void my_sync(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int target = gen + 1;
    unsigned int arrived = atomicAdd(&g_count, 1);
    if (arrived == nblocks - 1) { g_count = 0; __threadfence(); g_gen = target; }
    else { while (g_gen != target) { __nanosleep(20); } }
    __threadfence();
  }
  gen += 1;
  __syncthreads();
}
__global__ void k_mysync(int n, double* out) {
  unsigned int gen = g_gen;
  double acc = 0;
  for (int i = 0; i < n; ++i) { acc += i; my_sync(gridDim.x, gen); }
  if (acc < 0) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int n = 2000;
  for (int grid : {16, 148, 296, 444, 592}) {
    for (int which = 0; which < 2; ++which) {
      void* args[] = {&n, &out};
      const void* fn = which ? (const void*)k_mysync : (const void*)k_cgsync;
      cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d %-8s %.3f us/sync  (%s)\n", grid, which ? "custom" : "cg", 1e3 * ms / n,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
