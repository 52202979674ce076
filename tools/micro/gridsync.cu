// Micro-benchmark: cost of cg::grid_group::sync() and of same-address atomics
// on this GPU (informs the solo/grid thresholds of k_simulate / k_cascade).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, unsigned* ctr) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}
__global__ void k_sync_atomic(int iters, unsigned* ctr) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if ((threadIdx.x & 31) == 0) atomicAdd(&ctr[i & 1], 32u);
    g.sync();
  }
}
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned* ctr;
  cudaMalloc(&ctr, 64);
  for (int bps : {1, 2, 3, 4}) {
    for (int which = 0; which < 2; ++which) {
      int iters = 2000;
      void* args[] = {&iters, &ctr};
      void* fn = which ? (void*)k_sync_atomic : (void*)k_sync;
      cudaLaunchCooperativeKernel(fn, dim3(sms * bps), dim3(256), args, 0, 0);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, dim3(sms * bps), dim3(256), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("blocks/SM %d %s: %.2f us per grid.sync\n", bps, which ? "+warp atomics" : "plain",
             ms * 1000 / iters);
    }
  }
  int iters = 1;
  void* args[] = {&iters, &ctr};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i)
    cudaLaunchCooperativeKernel((void*)k_sync, dim3(sms * 3), dim3(256), args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("cooperative launch + 1 sync: %.2f us per launch (back to back)\n", ms * 10);
  return 0;
}
