// Legacy mma.sync TF32 (m16n8k8) and FFMA throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tf32_k(float* out, int iters) {
  float acc[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  unsigned a0 = 0x3f800000u + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 0x3f000000u, b1 = b0 + 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == -1.0f) out[0] = s;
}
__global__ void ffma_k(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 1.0000001f, 1e-9f);
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  if (s == -1.0f) out[0] = s;
}
__global__ void spin(float* p, int n) { float v = threadIdx.x; for (int i = 0; i < n; ++i) v = fmaf(v, 1.0000001f, 0.5f); if (v == -1.0f) p[0] = v; }
int main() {
  float* d; cudaMalloc(&d, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 30; ++i) spin<<<148 * 4, 256>>>(d, 400000);
  for (int threads : {256, 512}) for (int blocks : {148, 296}) {
    int iters = 20000; float ms;
    tf32_k<<<blocks, threads>>>(d, 100);
    cudaEventRecord(a); tf32_k<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("TF32 mma.sync blocks=%d threads=%d: %.1f TFLOP/s\n", blocks, threads, 2.0 * 16 * 8 * 8 * 8 * iters * (double)(threads / 32) * blocks / ms / 1e9);
    ffma_k<<<blocks, threads>>>(d, 100);
    cudaEventRecord(a); ffma_k<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("FFMA blocks=%d threads=%d: %.1f TFLOP/s\n", blocks, threads, 2.0 * 16 * iters * (double)threads * blocks / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
