// Standalone check of block_jacobi: eigen-decomposition accuracy vs sweeps.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_jacobi.cuh"
using namespace megb200;
__global__ void k(const double* H, int m, double* th, double* S, double* info) {
  extern __shared__ double sm[];
  block_jacobi(H, m, m, th, S, sm, info);
}
int main() {
  for (int m : {5, 18, 36, 72}) {
    std::vector<double> h(m * m);
    srand(1);
    for (int i = 0; i < m; ++i) for (int j = 0; j <= i; ++j) { double v = (rand() / (double)RAND_MAX) - 0.5; h[i*m+j] = h[j*m+i] = v; }
    for (int i = 0; i < m; ++i) h[i*m+i] += -13.6 + 0.01 * i;
    double *dH, *dt, *dS, *di; cudaMalloc(&dH, m*m*8); cudaMalloc(&dt, m*8); cudaMalloc(&dS, m*m*8); cudaMalloc(&di, 64);
    cudaMemcpy(dH, h.data(), m*m*8, cudaMemcpyHostToDevice);
    int smem = jacobi_smem_doubles(m) * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 215*1024);
    int thr = m <= 24 ? 64 : m <= 48 ? 256 : 512;
    k<<<1, thr, smem>>>(dH, m, dt, dS, di);
    cudaDeviceSynchronize();
    std::vector<double> th(m), S(m*m), info(8);
    cudaMemcpy(th.data(), dt, m*8, cudaMemcpyDeviceToHost); cudaMemcpy(S.data(), dS, m*m*8, cudaMemcpyDeviceToHost); cudaMemcpy(info.data(), di, 24, cudaMemcpyDeviceToHost);
    // residual max |H s - theta s|
    double res = 0, orth = 0;
    for (int j = 0; j < m; ++j) for (int i = 0; i < m; ++i) { double v = 0; for (int k2 = 0; k2 < m; ++k2) v += h[i*m+k2]*S[k2*m+j]; res = fmax(res, fabs(v - th[j]*S[i*m+j])); }
    for (int a = 0; a < m; ++a) for (int b = 0; b < m; ++b) { double v = 0; for (int i = 0; i < m; ++i) v += S[i*m+a]*S[i*m+b]; orth = fmax(orth, fabs(v - (a==b))); }
    printf("m=%d sweeps=%.0f off=%.3e fro=%.3e  max|Hs-ts|=%.3e  orth=%.3e %s\n", m, info[0], info[1], info[2], res, orth, cudaGetErrorString(cudaGetLastError()));
  }
}
