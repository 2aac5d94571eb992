// Timing of the single-CTA serial phases: block_jacobi (random / nearly diagonal H) by thread count.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_jacobi.cuh"
namespace oldj {
#include "jacobi_old.cuh"
}
using namespace megb200;
__global__ void __launch_bounds__(1024, 1) kj(const double* H, int m, double* th, double* S, double* info) {
  extern __shared__ double sm[];
  block_jacobi(H, m, m, th, S, sm, info);
}
__global__ void ko(const double* H, int m, double* th, double* S, double* info) {
  extern __shared__ double sm[];
  oldj::megb200::block_jacobi(H, m, m, th, S, sm, info);
}
__global__ void spin(double* p, int n) {
  double v = threadIdx.x;
  for (int i = 0; i < n; ++i) v = fma(v, 1.0000001, 0.5);
  if (v == -1.0) p[0] = v;
}
int main() {
  cudaFuncSetAttribute(kj, cudaFuncAttributeMaxDynamicSharedMemorySize, 215*1024);
  cudaFuncSetAttribute(ko, cudaFuncAttributeMaxDynamicSharedMemorySize, 215*1024);
  double* dummy; cudaMalloc(&dummy, 8);
  for (int i = 0; i < 50; ++i) spin<<<148 * 4, 256>>>(dummy, 200000);  // ramp clocks
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int diag : {0, 1}) for (int m : {18, 32, 64, 96, 108}) for (int thr : {64, 256, 1024}) for (int old : {0, 1}) {
    std::vector<double> h(m * m);
    srand(1);
    for (int i = 0; i < m; ++i) for (int j = 0; j <= i; ++j) { double v = ((rand() / (double)RAND_MAX) - 0.5) * (diag ? 1e-6 : 1.0); h[i*m+j] = h[j*m+i] = v; }
    for (int i = 0; i < m; ++i) h[i*m+i] += -13.6 + (diag ? 0.3 * i : 0.01 * i);
    double *dH, *dt, *dS, *di; cudaMalloc(&dH, m*m*8); cudaMalloc(&dt, m*8); cudaMalloc(&dS, m*m*8); cudaMalloc(&di, 64);
    cudaMemcpy(dH, h.data(), m*m*8, cudaMemcpyHostToDevice);
    const int mp = (m + 1) & ~1, half = mp / 2;
    if (half * half > 4 * thr || mp * half > 8 * thr) continue;
    int smem = jacobi_smem_doubles(m) * 8;
    if (old) ko<<<1, thr, smem>>>(dH, m, dt, dS, di); else kj<<<1, thr, smem>>>(dH, m, dt, dS, di);
    spin<<<148 * 4, 256>>>(dummy, 20000);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) { if (old) ko<<<1, thr, smem>>>(dH, m, dt, dS, di); else kj<<<1, thr, smem>>>(dH, m, dt, dS, di); }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double info[3]; cudaMemcpy(info, di, 24, cudaMemcpyDeviceToHost);
    // accuracy check
    std::vector<double> th(m), S(m*m);
    cudaMemcpy(th.data(), dt, m*8, cudaMemcpyDeviceToHost); cudaMemcpy(S.data(), dS, m*m*8, cudaMemcpyDeviceToHost);
    double res = 0; for (int j = 0; j < m; ++j) for (int i = 0; i < m; ++i) { double v = 0; for (int k2 = 0; k2 < m; ++k2) v += h[i*m+k2]*S[k2*m+j]; res = fmax(res, fabs(v - th[j]*S[i*m+j])); }
    printf("%s%s m=%3d threads=%4d: %8.1f us  sweeps=%.0f  (%.2f us/round) res=%.1e\n", old ? "OLD " : "NEW ", diag ? "near-diag" : "random   ", m, thr, ms * 100, info[0], ms * 100 / (info[0] * (m - 1 + (m & 1))), res);
    cudaFree(dH); cudaFree(dt); cudaFree(dS); cudaFree(di);
  }
}
