// Unit checks of the tcgen05 building blocks: TMEM st/ld round trip, one kind::tf32 MMA (K-major, no swizzle)
// and one MMA with MN-major 128B-swizzled operands (the layout the operand pass uses).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_umma.cuh"
using namespace megb200::umma;

__device__ uint64_t desc_any(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46) | ((uint64_t)layout << 61);
}

// mode 0: TMEM st/ld; mode 1: MMA K-major SWIZZLE_NONE; mode 2: MMA MN-major SW128
__global__ void kunit(int mode, const float* A, const float* B, float* out, uint32_t idesc, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  __shared__ __align__(1024) float sa[128 * 8 * 4];  // up to 128 x 32 floats (16 KB)
  __shared__ __align__(1024) float sb[32 * 32];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(saddr(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  uint32_t r[32];
  if (mode == 0) {
    for (int c = 0; c < 32; ++c) r[c] = __float_as_uint((float)(t * 100 + c));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(tmem + ((uint32_t)(warp * 32) << 16)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                 "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
                 "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                 "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else {
    // stage operands exactly as given (host prepared the layout)
    for (int i = t; i < 128 * 32; i += 128) sa[i] = A[i];
    for (int i = t; i < 32 * 32; i += 128) sb[i] = B[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t koff = mode >= 3 ? (uint32_t)(mode - 3) * 32u : 0u;
      const uint64_t da = desc_any(saddr(sa) + koff, lbo, sbo, lay), db = desc_any(saddr(sb) + koff, lbo, sbo, lay);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u) : "memory");
      mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
               "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
               "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
               "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
               "+r"(r[30]), "+r"(r[31]) :: "memory");
  for (int c = 0; c < 32; ++c) out[t * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main() {
  float *dA, *dB, *dO; cudaMalloc(&dA, 128 * 32 * 4); cudaMalloc(&dB, 32 * 32 * 4); cudaMalloc(&dO, 128 * 32 * 4);
  static float hA[128 * 32], hB[32 * 32], hO[128 * 32];
  // ---- mode 0
  kunit<<<1, 128>>>(0, dA, dB, dO, 0, 0, 0, 0);
  printf("mode0: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
  int bad = 0; for (int t = 0; t < 128; ++t) for (int c = 0; c < 32; ++c) bad += hO[t * 32 + c] != (float)(t * 100 + c);
  printf("  st/ld mismatches: %d (o[5][3]=%g)\n", bad, hO[5 * 32 + 3]);
  // logical operands: a[m][k] (128 x 8), b[n][k] (32 x 8), small integers (exact in tf32)
  static float a[128][8], b[32][8];
  srand(1);
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) a[m][k] = (float)(rand() % 7 - 3);
  for (int n = 0; n < 32; ++n) for (int k = 0; k < 8; ++k) b[n][k] = (float)(rand() % 7 - 3);
  auto check = [&](const char* name) {
    cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
    int bad = 0; double maxe = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) {
      double ref = 0; for (int k = 0; k < 8; ++k) ref += a[m][k] * b[n][k];
      double e = fabs(hO[m * 32 + n] - ref); maxe = fmax(maxe, e); bad += e > 1e-3;
    }
    printf("  %s: mismatches %d maxerr %g  (o[0][0]=%g ref %g, o[1][2]=%g)\n", name, bad, maxe, hO[0],
           (double)(a[0][0]*b[0][0]+a[0][1]*b[0][1]+a[0][2]*b[0][2]+a[0][3]*b[0][3]+a[0][4]*b[0][4]+a[0][5]*b[0][5]+a[0][6]*b[0][6]+a[0][7]*b[0][7]), hO[34]);
  };
  // ---- mode 1: K-major, no swizzle. core matrix = 8 rows x 4 k (16 B per row, 128 B); K=8 -> 2 core
  // matrices along K at LBO; rows in groups of 8 at SBO.  Layout: [m/8][k/4][m%8][k%4]
  const uint32_t LBO1 = 128, SBO1 = 256;  // k-core stride 128 B, 8-row group stride 256 B
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) hA[(m / 8) * 64 + (k / 4) * 32 + (m % 8) * 4 + (k % 4)] = a[m][k];
  for (int n = 0; n < 32; ++n) for (int k = 0; k < 8; ++k) hB[(n / 8) * 64 + (k / 4) * 32 + (n % 8) * 4 + (k % 4)] = b[n][k];
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  const uint32_t idK = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
  kunit<<<1, 128>>>(1, dA, dB, dO, idK, LBO1, SBO1, 0);
  printf("mode1: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  check("K-major/none");
  // ---- mode 2: MN-major SW128: row k (128 B) holds 32 MN elements; blocks of 32 MN at LBO; 8 k rows per atom.
  // element (mn, k) -> byte ((mn/32)*LBO + k*128 + (((mn%32)/4) ^ (k%8))*16 + (mn%4)*4)
  for (int i = 0; i < 128 * 32; ++i) hA[i] = 0;
  for (int i = 0; i < 32 * 32; ++i) hB[i] = 0;
  const uint32_t LBO2 = 1024, SBO2 = 1024;
  auto put = [&](float* buf, int mn, int k, float v) {
    const int byte = (mn / 32) * LBO2 + k * 128 + ((((mn % 32) / 4) ^ (k % 8)) * 16) + (mn % 4) * 4;
    buf[byte / 4] = v;
  };
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) put(hA, m, k, a[m][k]);
  for (int n = 0; n < 32; ++n) for (int k = 0; k < 8; ++k) put(hB, n, k, b[n][k]);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  const uint32_t idMN = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
  kunit<<<1, 128>>>(2, dA, dB, dO, idMN, LBO2, SBO2, 2);
  printf("mode2: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  check("MN-major/SW128");
  kunit<<<1, 128>>>(2, dA, dB, dO, idMN, SBO2, LBO2, 2);
  cudaDeviceSynchronize(); check("MN-major/SW128 lbo<->sbo (same values)");
  kunit<<<1, 128>>>(2, dA, dB, dO, idMN, 4096, 1024, 2);
  cudaDeviceSynchronize(); check("MN-major/SW128 lbo=4096");
  kunit<<<1, 128>>>(2, dA, dB, dO, idMN, 1024, 4096, 2);
  cudaDeviceSynchronize(); check("MN-major/SW128 sbo=4096");
  // ---- MN-major, no swizzle: core matrix = 8 k rows x 4 mn (16 B rows); mn groups of 4 at SBO, k groups of 8 at LBO
  for (int i = 0; i < 128 * 32; ++i) hA[i] = 0;
  for (int i = 0; i < 32 * 32; ++i) hB[i] = 0;
  const uint32_t SBO3 = 128, LBO3 = 128 * 32;
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) hA[((m / 4) * SBO3 + (k / 8) * LBO3) / 4 + (k % 8) * 4 + (m % 4)] = a[m][k];
  for (int n = 0; n < 32; ++n) for (int k = 0; k < 8; ++k) hB[((n / 4) * SBO3 + (k / 8) * LBO3) / 4 + (k % 8) * 4 + (n % 4)] = b[n][k];
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  kunit<<<1, 128>>>(2, dA, dB, dO, idMN, LBO3, SBO3, 0);
  cudaDeviceSynchronize(); check("MN-major/none (lbo=k-group, sbo=mn-group)");
  kunit<<<1, 128>>>(2, dA, dB, dO, idMN, SBO3, LBO3, 0);
  cudaDeviceSynchronize(); check("MN-major/none (swapped)");
  // ---- K-major SW128: row r (128 B) holds 32 k; atoms of 8 rows at SBO=1024; k-step s at +32 s bytes
  {
    static float a2[128][32], b2[32][32];
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) a2[m][k] = (float)(rand() % 7 - 3);
    for (int n = 0; n < 32; ++n) for (int k = 0; k < 32; ++k) b2[n][k] = (float)(rand() % 7 - 3);
    auto putk = [&](float* buf, int row, int k, float v) {
      const int byte = (row / 8) * 1024 + (row % 8) * 128 + (((k / 4) ^ (row % 8)) * 16) + (k % 4) * 4;
      buf[byte / 4] = v;
    };
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) putk(hA, m, k, a2[m][k]);
    for (int n = 0; n < 32; ++n) for (int k = 0; k < 32; ++k) putk(hB, n, k, b2[n][k]);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    for (int ks = 0; ks < 4; ++ks) {
      kunit<<<1, 128>>>(3 + ks, dA, dB, dO, idK, 16, 1024, 2);
      printf("mode K-SW128 ks=%d: %s\n", ks, cudaGetErrorString(cudaDeviceSynchronize()));
      cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
      int bad = 0; double maxe = 0;
      for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) {
        double ref = 0; for (int k = 8 * ks; k < 8 * ks + 8; ++k) ref += a2[m][k] * b2[n][k];
        double e = fabs(hO[m * 32 + n] - ref); maxe = fmax(maxe, e); bad += e > 1e-3;
      }
      printf("  K-major/SW128 k-step %d: mismatches %d maxerr %g\n", ks, bad, maxe);
    }
  }
  // ---- tf32 conversion of raw fp32 operands: truncation or rounding?  A = 1 + 3*2^-12 (0.75 tf32 ulp), B = 1
  {
    for (int i = 0; i < 128 * 32; ++i) hA[i] = 0;
    for (int i = 0; i < 32 * 32; ++i) hB[i] = 0;
    const float va = 1.0f + 3.0f / 4096.0f, vb = 1.0f;
    hA[(0 / 8) * 64 + (0 / 4) * 32 + (0 % 8) * 4 + 0] = va;   // a[0][0] (K-major, no swizzle layout of mode 1)
    hB[(0 / 8) * 64 + (0 / 4) * 32 + (0 % 8) * 4 + 0] = vb;   // b[0][0]
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    kunit<<<1, 128>>>(1, dA, dB, dO, idK, LBO1, SBO1, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
    printf("tf32 conversion: a=1+3*2^-12 -> D = %.9f (truncate: 1.0, round: %.9f)\n", hO[0], 1.0 + 1.0 / 1024.0);
    const float vn = -(1.0f + 3.0f / 4096.0f);
    hA[0] = vn;
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    kunit<<<1, 128>>>(1, dA, dB, dO, idK, LBO1, SBO1, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
    printf("negative: D = %.9f\n", hO[0]);
  }
  return 0;
}
