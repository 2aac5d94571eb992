// Standalone check of the tcgen05 3xTF32 operand pass (megb200_umma.cuh) against a float64 host product.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_2012_10469_b200/csrc/megb200_umma.cuh"
using namespace megb200;

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) { void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q); fn = (PFN_cuTensorMapEncodeTiled_v12000)p; }
  return fn;
}
static CUtensorMap map2d(const void* base, int64_t cols, int64_t rows, int64_t ld, uint32_t bc, uint32_t br) {
  CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {bc, br}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}
int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 512;
  const int b = argc > 2 ? atoi(argv[2]) : 32;
  const int G0 = argc > 3 ? atoi(argv[3]) : 148;
  srand(3);
  std::vector<float> M(n * n); std::vector<double> U(n * b);
  for (int64_t i = 0; i < n; ++i) for (int64_t j = 0; j <= i; ++j) M[i * n + j] = M[j * n + i] = (float)((rand() / (double)RAND_MAX) - 0.5);
  for (auto& v : U) v = (rand() / (double)RAND_MAX) - 0.5;
  float *dM, *dUh, *dUl; double *dU, *dP;
  cudaMalloc(&dM, n * n * 4); cudaMalloc(&dU, n * b * 8); cudaMalloc(&dUh, n * 64 * 4); dUl = nullptr;
  const int tiles = (int)((n + 127) / 128), kch = (int)((n + 31) / 32);
  const int64_t utot = (int64_t)tiles * kch;
  int grid = (int)std::min<int64_t>(G0, utot), smax = 1;
  for (;;) {
    auto cf = [&](int64_t x) { return (int)(((x + 1) * grid + utot - 1) / utot) - 1; };
    smax = 1;
    for (int t = 0; t < tiles; ++t) smax = std::max(smax, cf((int64_t)(t + 1) * kch - 1) - cf((int64_t)t * kch) + 1);
    if (smax <= 16 || grid == 1) break;
    grid = std::max(1, grid * 16 / (smax + 1));
  }
  cudaMalloc(&dP, (size_t)smax * n * b * 8);
  float* dD; cudaMalloc(&dD, 64 * 4); cudaMemset(dD, 0, 256);
  cudaMemcpy(dM, M.data(), n * n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), n * b * 8, cudaMemcpyHostToDevice);
  umma::k_split_u<<<(n + 31) / 32, 256>>>(n, b, dU, b, dUh, n);
  CUtensorMap tM = map2d(dM, n, n, n, 32, 128), tUh = map2d(dUh, n, 64, n, 32, 64);
  cudaFuncSetAttribute(umma::k_dense_pass_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)umma::smem_bytes());
  umma::k_dense_pass_umma<<<grid, umma::kThreads, umma::smem_bytes()>>>(tM, tUh, n, b, dP, tiles, kch, smax);
  cudaError_t e = cudaDeviceSynchronize();
  printf("n=%lld b=%d grid=%d smax=%d: %s\n", (long long)n, b, grid, smax, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<double> P((size_t)smax * n * b);
  cudaMemcpy(P.data(), dP, P.size() * 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int64_t i = 0; i < (n > 16384 ? 256 : n); ++i) for (int c = 0; c < b; ++c) {
    double ref = 0; for (int64_t k = 0; k < n; ++k) ref += (double)M[k * n + i] * U[k * b + c];
    double got = 0; for (int s = 0; s < smax; ++s) got += P[(size_t)s * n * b + i * b + c];
    maxerr = fmax(maxerr, fabs(got - ref)); maxref = fmax(maxref, fabs(ref));
  }
  printf("max abs err %.3e  max |ref| %.3e  rel %.3e\n", maxerr, maxref, maxerr / maxref);
  for (int64_t i = 0; i < 3; ++i) for (int c = 0; c < 3; ++c) {
    double ref = 0; for (int64_t k = 0; k < n; ++k) ref += (double)M[k * n + i] * U[k * b + c];
    double got = 0; for (int s = 0; s < smax; ++s) got += P[(size_t)s * n * b + i * b + c];
    double p0 = P[i * b + c];
    double r0 = 0; for (int64_t k = 0; k < 32; ++k) r0 += (double)M[k * n + i] * U[k * b + c];
    printf("  i=%lld c=%d ref %.6f got %.6f | slot0 %.6f ref(k<32) %.6f\n", (long long)i, c, ref, got, p0, r0);
  }
  // timing at this size
  cudaEvent_t a, z; cudaEventCreate(&a); cudaEventCreate(&z);
  for (int flags : {0}) {
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) umma::k_dense_pass_umma<<<grid, umma::kThreads, umma::smem_bytes()>>>(tM, tUh, n, b, dP, tiles, kch, smax);
    cudaEventRecord(z); cudaEventSynchronize(z);
    float ms; cudaEventElapsedTime(&ms, a, z);
    printf("flags %d (1=no mma 2=no split 4=3 products): avg %.1f us  (%.0f GB/s operand)\n", flags, ms * 1000 / 20, (double)n * n * 4 / (ms / 20 * 1e-3) / 1e9);
  }
#ifdef UMMA_PROFILE
  long long hp[8]; cudaMemcpyFromSymbol(hp, umma::g_uprof, sizeof hp);
  printf("split warp 0 per stage (cycles): wait abuf %.0f | wait full %.0f | load+split %.0f | st+wait+arrive %.0f (%lld stages)\n",
         (double)hp[0] / hp[4], (double)hp[1] / hp[4], (double)hp[2] / hp[4], (double)hp[3] / hp[4], hp[4]);
  printf("MMA warp: wait split %.0f cycles per stage | drain wait acc_full %.0f cycles per drain (%lld drains)\n",
         (double)hp[5] / hp[4], (double)hp[6] / hp[7], hp[7]);
#endif
  return 0;
}
