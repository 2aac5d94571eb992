// Throughput of back-to-back tcgen05.mma kind::tf32 (K-major SW128 operands in smem) by N.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_umma.cuh"
using namespace megb200::umma;

template <int N, int NBUF, int TM>
__global__ void krate(int iters, unsigned long long* cyc, int noise, int tmema_unused) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - ((uintptr_t)sm & 1023)) & 1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < NBUF * (128 * 128 + N * 128) / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (noise && warp >= 1) {
    // concurrent LSU traffic: copy a 16 KB region back and forth
    float4* r0 = reinterpret_cast<float4*>(base + NBUF * (128 * 128 + N * 128));
    for (int it = 0; it < iters * noise; ++it)
      for (int v = t - 32; v < 1024; v += 96) { float4 x = r0[v]; x.x += 1.f; r0[(v + 512) & 1023] = x; }
  }
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    unsigned long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (!elect_one()) continue;
      const uint32_t sa = saddr(base) + (uint32_t)((it % NBUF) * (128 * 128 + N * 128)), sb = sa + 128 * 128;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t a = sdesc(sa + ks * 32), bdesc = sdesc(sb + ks * 32);
        if (TM) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tmem), "r"(tmem + 128u + (uint32_t)(8 * ks)), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
        } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(a), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
        }
      }
    }
    __syncwarp();
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long c1 = clock64();
    if (t == 0) cyc[0] = c1 - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

static int NOISE = 0;
static int TMA_MODE = 0;

template <int N, int NBUF = 1, int TM = 0>
void run(unsigned long long* d) {
  const int smem = 1024 + NBUF * (128 * 128 + N * 128) + 16384;
  cudaFuncSetAttribute(krate<N, NBUF, TM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  krate<N, NBUF, TM><<<1, 128, smem>>>(10, d, 0, TMA_MODE);
  cudaDeviceSynchronize();
  const int iters = 2000;
  krate<N, NBUF, TM><<<1, 128, smem>>>(iters, d, NOISE, TMA_MODE);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * 4);
  printf("NBUF=%d N=%3d: %s  %.1f cycles per 128x%dx8 MMA  -> %.0f flop/cycle/SM (%.0f TF/s at 148 SMs x 1.965 GHz)\n", N,
         NBUF, cudaGetErrorString(e), per, N, 2.0 * 128 * N * 8 / per, 2.0 * 128 * N * 8 / per * 148 * 1.965e9 / 1e12);
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  // spin to raise clocks
  run<64, 8>(d); run<128, 4>(d);
  printf("A operand in tensor memory:\n");
  run<64, 8, 1>(d); run<128, 4, 1>(d); run<256, 1, 1>(d);
}
