// Microbenchmark: cost of cooperative grid.sync() and of single-CTA serial phases on B200.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_syncs(int nsync, double* out) {
  cg::grid_group g = cg::this_grid();
  double v = threadIdx.x;
  for (int i = 0; i < nsync; ++i) { v += 1.0; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = v;
}

__global__ void k_empty(double* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1.0; }

__global__ void k_serial_div(int n, double* out) {
  // one warp: dependent chain of n fp64 divisions + sqrt (Cholesky-like latency chain)
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  double x = 1.0 + threadIdx.x;
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0) / (x * 0.5 + 1.0) + 1.0;
  out[threadIdx.x] = x;
}

int main() {
  double* d; cudaMalloc(&d, 1024 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int grid : {32, 64, 128, 148}) {
    for (int ns : {0, 1, 10, 100}) {
      void* args[] = {&ns, &d};
      for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel((void*)k_syncs, grid, 256, args, 0, 0);
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) cudaLaunchCooperativeKernel((void*)k_syncs, grid, 256, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("coop grid=%d syncs=%d: %.2f us per launch\n", grid, ns, ms * 1000 / 20);
    }
  }
  for (int w = 0; w < 3; ++w) k_empty<<<128, 256>>>(d);
  cudaEventRecord(a);
  for (int it = 0; it < 100; ++it) k_empty<<<128, 256>>>(d);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("plain empty launch (back-to-back): %.2f us\n", ms * 1000 / 100);
  for (int n : {18, 100, 1000}) {
    k_serial_div<<<1, 32>>>(n, d);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) k_serial_div<<<1, 32>>>(n, d);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("serial fp64 sqrt+div chain n=%d: %.2f us (%.1f ns/step)\n", n, ms * 1000 / 10, ms * 1e6 / 10 / n);
  }
  return 0;
}
