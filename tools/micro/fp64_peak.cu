// FP64 throughput on B200: DFMA (CUDA cores) vs DMMA (mma.sync.m8n8k4.f64 tensor path).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_k(double* out, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  if (s == -1.0) out[0] = s;
}
__global__ void dmma_k(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == -1.0) out[0] = s;
}
__global__ void spin(double* p, int n) { double v = threadIdx.x; for (int i = 0; i < n; ++i) v = fma(v, 1.0000001, 0.5); if (v == -1.0) p[0] = v; }
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 30; ++i) spin<<<148 * 4, 256>>>(d, 200000);
  for (int threads : {256, 512}) for (int blocks : {148, 296, 592}) {
    int iters = 20000;
    dfma_k<<<blocks, threads>>>(d, 100);
    cudaEventRecord(a); dfma_k<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 16 * iters * (double)threads * blocks;
    printf("DFMA blocks=%d threads=%d: %.1f TFLOP/s\n", blocks, threads, fl / ms / 1e9);
    dmma_k<<<blocks, threads>>>(d, 100);
    cudaEventRecord(a); dmma_k<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    fl = 2.0 * 256 * 8 * iters * (double)(threads / 32) * blocks;
    printf("DMMA blocks=%d threads=%d: %.1f TFLOP/s\n", blocks, threads, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
