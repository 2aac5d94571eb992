// One block_jacobi solve for ncu: jacobi_prof m threads diag
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_jacobi.cuh"
using namespace megb200;
__global__ void __launch_bounds__(1024, 1) kj(const double* H, int m, double* th, double* S, double* info) {
  extern __shared__ double sm[];
  block_jacobi(H, m, m, th, S, sm, info);
}
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 108, thr = argc > 2 ? atoi(argv[2]) : 1024, diag = argc > 3 ? atoi(argv[3]) : 0;
  std::vector<double> h(m * m);
  srand(1);
  for (int i = 0; i < m; ++i) for (int j = 0; j <= i; ++j) { double v = ((rand() / (double)RAND_MAX) - 0.5) * (diag ? 1e-6 : 1.0); h[i*m+j] = h[j*m+i] = v; }
  for (int i = 0; i < m; ++i) h[i*m+i] += -13.6 + (diag ? 0.3 * i : 0.01 * i);
  double *dH, *dt, *dS, *di; cudaMalloc(&dH, m*m*8); cudaMalloc(&dt, m*8); cudaMalloc(&dS, m*m*8); cudaMalloc(&di, 64);
  cudaMemcpy(dH, h.data(), m*m*8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kj, cudaFuncAttributeMaxDynamicSharedMemorySize, 215*1024);
  kj<<<1, thr, jacobi_smem_doubles(m) * 8>>>(dH, m, dt, dS, di);
  cudaDeviceSynchronize();
  double info[3]; cudaMemcpy(info, di, 24, cudaMemcpyDeviceToHost);
  printf("%s sweeps=%g\n", cudaGetErrorString(cudaGetLastError()), info[0]);
}
