// Host side of the tcgen05 float32-operand pass (device code in megb200_umma.cuh).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "megb200_internal.h"
#include "megb200_umma.cuh"

namespace megb200 {

bool umma_pass_supported(int64_t n, int b, int64_t ldm, const void* M) {
  return b <= umma::kN && n % 4 == 0 && ldm % 4 == 0 && ((uintptr_t)M % 16) == 0 &&
         getenv("MEGB200_NO_UMMA") == nullptr;
}

int dense_pass_umma(const Launch& L, const float* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                    double* part, int64_t part_cap_slices, int sm_count, float* uscratch) {
  // stream-K over (128-row tile, 32-row k chunk), as the float64 DMMA pass
  const int tiles = (int)((n + umma::kRows - 1) / umma::kRows);
  const int kch = (int)((n + umma::kKC - 1) / umma::kKC);
  const int64_t utot = (int64_t)tiles * kch;
  const int cap = (int)std::max<int64_t>(1, std::min<int64_t>(part_cap_slices, 16));
  int grid = (int)std::min<int64_t>(sm_count, utot);
  int smax = 1;
  for (;;) {
    auto cfirst = [&](int64_t x) { return (int)(((x + 1) * grid + utot - 1) / utot) - 1; };
    smax = 1;
    for (int t = 0; t < tiles; ++t)
      smax = std::max(smax, cfirst((int64_t)(t + 1) * kch - 1) - cfirst((int64_t)t * kch) + 1);
    if (smax <= cap || grid == 1) break;
    grid = std::max(1, grid * cap / (smax + 1));
  }
  // [Uh | Ul]^T (64 x n float32) for this pass
  umma::k_split_u<<<(unsigned)((n + 31) / 32), 256, 0, L.stream>>>(n, b, U, ldu, uscratch, n);
  MEG_LAUNCHED();
  ++*L.counter;
  static char attr = 0;
  if (first_on_device(&attr)) {
    MEG_CUDA(cudaFuncSetAttribute(umma::k_dense_pass_umma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)umma::smem_bytes()));
  }
  const CUtensorMap tmM = make_map(M, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, n, n, ldm, umma::kKC, umma::kRows,
                                   CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tmU = make_map(uscratch, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, n, umma::kNM, n, umma::kKC,
                                   umma::kNM, CU_TENSOR_MAP_SWIZZLE_128B);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(umma::kThreads);
  cfg.dynamicSmemBytes = umma::smem_bytes();
  cfg.stream = L.stream;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  MEG_CUDA(cudaLaunchKernelEx(&cfg, umma::k_dense_pass_umma, tmM, tmU, n, b, part, tiles, kch, smax));
  ++*L.counter;
  return smax;
}

}  // namespace megb200
