// Check tcgen05.mma kind::tf32 with the A operand in tensor memory (rows in lanes, k in columns),
// written by tcgen05.st from registers; B K-major SW128 in shared memory.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_umma.cuh"
using namespace megb200::umma;

__global__ void kt(const float* A, const float* B, float* out, int kstep, int acol) {
  __shared__ __align__(1024) float sb[64 * 32];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  for (int i = t; i < 64 * 32; i += 128) sb[i] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  // A row t (32 k values) -> TMEM lane t, columns acol .. acol + 31
  uint32_t r[32];
  for (int c = 0; c < 32; ++c) r[c] = __float_as_uint(A[t * 32 + c]);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)acol), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
               "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
               "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
               "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // N = 64, M = 128, A from TMEM (k-step kstep -> columns acol + 8 kstep), B K-major SW128 (+32 B per k-step)
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t bd = sdesc(saddr(sb) + kstep * 32);
    const uint32_t at = tmem + (uint32_t)acol + (uint32_t)(8 * kstep);
    const uint32_t dt = tmem + 64;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(dt), "r"(at), "l"(bd), "r"(idesc), "r"(0u) : "memory");
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int half = 0; half < 2; ++half) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(tmem + 64 + ((uint32_t)(warp * 32) << 16) + (uint32_t)(32 * half)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                 "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31]) :: "memory");
    for (int c = 0; c < 32; ++c) out[t * 64 + 32 * half + c] = __uint_as_float(r[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

int main() {
  static float a[128][32], b[64][32], hA[128 * 32], hB[64 * 32], hO[128 * 64];
  srand(2);
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) a[m][k] = (float)(rand() % 7 - 3);
  for (int n = 0; n < 64; ++n) for (int k = 0; k < 32; ++k) b[n][k] = (float)(rand() % 7 - 3);
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) hA[m * 32 + k] = a[m][k];
  for (int n = 0; n < 64; ++n) for (int k = 0; k < 32; ++k) {
    const int byte = (n / 8) * 1024 + (n % 8) * 128 + (((k / 4) ^ (n % 8)) * 16) + (k % 4) * 4;
    hB[byte / 4] = b[n][k];
  }
  float *dA, *dB, *dO; cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, sizeof hO);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int acol : {0, 128 - 64 - 32 >= 0 ? 0 : 0}) for (int ks = 0; ks < 4; ++ks) {
    kt<<<1, 128>>>(dA, dB, dO, ks, acol);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
    int bad = 0; double maxe = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 64; ++n) {
      double ref = 0; for (int k = 8 * ks; k < 8 * ks + 8; ++k) ref += a[m][k] * b[n][k];
      const double d = fabs(hO[m * 64 + n] - ref); maxe = fmax(maxe, d); bad += d > 1e-3;
    }
    printf("A in TMEM, k-step %d: %s mismatches %d maxerr %g (o00 %g)\n", ks, cudaGetErrorString(e), bad, maxe, hO[0]);
  }
  return 0;
}
