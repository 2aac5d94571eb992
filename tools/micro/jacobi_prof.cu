// One block_jacobi solve (m=108, 1024 threads) for ncu.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_jacobi.cuh"
using namespace megb200;
__global__ void kj(const double* H, int m, double* th, double* S, double* info) {
  extern __shared__ double sm[];
  block_jacobi(H, m, m, th, S, sm, info);
}
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 108, thr = argc > 2 ? atoi(argv[2]) : 1024;
  std::vector<double> h(m * m);
  srand(1);
  for (int i = 0; i < m; ++i) for (int j = 0; j <= i; ++j) { double v = (rand() / (double)RAND_MAX) - 0.5; h[i*m+j] = h[j*m+i] = v; }
  double *dH, *dt, *dS, *di; cudaMalloc(&dH, m*m*8); cudaMalloc(&dt, m*8); cudaMalloc(&dS, m*m*8); cudaMalloc(&di, 64);
  cudaMemcpy(dH, h.data(), m*m*8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kj, cudaFuncAttributeMaxDynamicSharedMemorySize, 215*1024);
  kj<<<1, thr, jacobi_smem_doubles(m) * 8>>>(dH, m, dt, dS, di);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
