// sm_100a kernels of the low-rank MEG hot path.
//
// Streaming kernels (the operand passes) are HBM-bound: the dense operand is
// read exactly once per pass with coalesced 16-byte streaming loads; the
// tall-skinny block U is staged through shared memory and broadcast.  The
// small dense work (Gram/projection reductions, Cholesky, Jacobi
// Rayleigh-Ritz) runs in float64 with fixed reduction orders so every result
// is bitwise reproducible run to run (SPEC.md:97 determinism).

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <string>

#include "megb200_internal.h"
#include "megb200_jacobi.cuh"
#include "megb200_tail.cuh"

namespace megb200 {
namespace {

constexpr double kTwoPi = 6.283185307179586;
constexpr double kInv53 = 1.0 / 9007199254740992.0;

__device__ __forceinline__ double gauss_dev(uint64_t key, uint64_t ctr) {
  const uint64_t b1 = mix64(key + (2 * ctr + 1) * kGolden);
  const uint64_t b2 = mix64(key + (2 * ctr + 2) * kGolden);
  const double u1 = ((double)(b1 >> 11) + 1.0) * kInv53;
  const double u2 = (double)(b2 >> 11) * kInv53;
  return sqrt(-2.0 * log(u1)) * cos(kTwoPi * u2);
}

__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ===========================================================================
// K1: dense streamed product, float64 operand.
//
// part[s][i][c] = sum_{k in slice s} M[k][i] * U[k][c]   (M symmetric: the
// k-th row of M supplies column i, so each warp reads 512 contiguous bytes
// of one operand row per k).  CTA = 8 warps over 64 output rows (2 per
// lane); warps interleave over k within the slice; U chunks of KC rows are
// staged in shared memory and read as broadcasts.
constexpr int kApplyThreads = 256;
constexpr int KC = 64;          // k rows per staged chunk
constexpr int kPerWarp = KC / 8; // k rows per warp per chunk

template <int BN, bool VEC>
__global__ void __launch_bounds__(kApplyThreads, 1)
    k_dense_apply_f64(const double* __restrict__ M, int64_t ldm, int64_t n, const double* __restrict__ U,
                      int64_t ldu, int b, double* __restrict__ part, int64_t kslice) {
  extern __shared__ __align__(16) double sm[];
  double* Us = sm;              // KC x BN
  double* red = sm + KC * BN;   // 4 x BN x 64
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * 64;
  const int64_t i = row0 + 2 * lane;
  const int64_t kbeg = (int64_t)blockIdx.y * kslice;
  const int64_t kend = min(n, kbeg + kslice);

  double a0[BN], a1[BN];
#pragma unroll
  for (int c = 0; c < BN; ++c) a0[c] = a1[c] = 0.0;

  for (int64_t kc = kbeg; kc < kend; kc += KC) {
    double m0[kPerWarp], m1[kPerWarp];
#pragma unroll
    for (int j = 0; j < kPerWarp; ++j) {
      const int64_t k = kc + warp + 8 * j;
      m0[j] = 0.0;
      m1[j] = 0.0;
      if (k < kend) {
        const double* p = M + k * ldm + i;
        if (VEC && i + 1 < n) {
          const double2 v = ld_stream2(p);
          m0[j] = v.x;
          m1[j] = v.y;
        } else {
          if (i < n) m0[j] = p[0];
          if (i + 1 < n) m1[j] = p[1];
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < KC * BN; idx += kApplyThreads) {
      const int r = idx / BN, c = idx - r * BN;
      const int64_t k = kc + r;
      Us[idx] = (k < kend && c < b) ? U[k * ldu + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPerWarp; ++j) {
      const double* u = Us + (warp + 8 * j) * BN;
#pragma unroll
      for (int c = 0; c < BN; c += 2) {
        const double2 uu = *reinterpret_cast<const double2*>(u + c);
        a0[c] = fma(m0[j], uu.x, a0[c]);
        a0[c + 1] = fma(m0[j], uu.y, a0[c + 1]);
        a1[c] = fma(m1[j], uu.x, a1[c]);
        a1[c + 1] = fma(m1[j], uu.y, a1[c + 1]);
      }
    }
  }
  // fixed-order tree over the 8 warps: (w, w+4) -> (w, w+2) -> (0, 1)
#pragma unroll
  for (int half = 4; half >= 1; half >>= 1) {
    __syncthreads();
    if (warp >= half && warp < 2 * half) {
      double* dst = red + (warp - half) * BN * 64;
#pragma unroll
      for (int c = 0; c < BN; ++c)
        *reinterpret_cast<double2*>(dst + c * 64 + 2 * lane) = make_double2(a0[c], a1[c]);
    }
    __syncthreads();
    if (warp < half) {
      const double* src = red + warp * BN * 64;
#pragma unroll
      for (int c = 0; c < BN; ++c) {
        const double2 v = *reinterpret_cast<const double2*>(src + c * 64 + 2 * lane);
        a0[c] += v.x;
        a1[c] += v.y;
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < BN; ++c) *reinterpret_cast<double2*>(red + c * 64 + 2 * lane) = make_double2(a0[c], a1[c]);
  }
  __syncthreads();
  double* out = part + (int64_t)blockIdx.y * n * b;
  const int rows = (int)min((int64_t)64, n - row0);
  for (int idx = threadIdx.x; idx < rows * b; idx += kApplyThreads) {
    const int r = idx / b, c = idx - r * b;
    out[(row0 + r) * b + c] = red[c * 64 + r];
  }
}

// K1 with a float32 operand: 4 rows per lane (16-byte streaming loads) and
// float32 FMA into per-lane accumulators over the CTA's k-slice (bounded to
// kF32Slice rows, so at most kF32Slice/8 terms per accumulator); the
// cross-warp tree and the cross-slice sum run in float64.
constexpr int kF32Slice = 4096;

template <int BN, bool VEC>
__global__ void __launch_bounds__(kApplyThreads, 1)
    k_dense_apply_f32(const float* __restrict__ M, int64_t ldm, int64_t n, const double* __restrict__ U,
                      int64_t ldu, int b, double* __restrict__ part, int64_t kslice) {
  extern __shared__ __align__(16) double sm[];
  float* Us = reinterpret_cast<float*>(sm);          // KC x BN floats
  double* red = sm + (KC * BN + 1) / 2;              // 4 x BN x 128 doubles
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * 128;
  const int64_t i = row0 + 4 * lane;
  const int64_t kbeg = (int64_t)blockIdx.y * kslice;
  const int64_t kend = min(n, kbeg + kslice);

  float s[4][BN];
#pragma unroll
  for (int c = 0; c < BN; ++c) s[0][c] = s[1][c] = s[2][c] = s[3][c] = 0.f;

  for (int64_t kc = kbeg; kc < kend; kc += KC) {
    float4 mv[kPerWarp];
#pragma unroll
    for (int j = 0; j < kPerWarp; ++j) {
      const int64_t k = kc + warp + 8 * j;
      mv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < kend) {
        const float* p = M + k * ldm + i;
        if (VEC && i + 3 < n) {
          mv[j] = ld_stream4(p);
        } else {
          if (i < n) mv[j].x = p[0];
          if (i + 1 < n) mv[j].y = p[1];
          if (i + 2 < n) mv[j].z = p[2];
          if (i + 3 < n) mv[j].w = p[3];
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < KC * BN; idx += kApplyThreads) {
      const int r = idx / BN, c = idx - r * BN;
      const int64_t k = kc + r;
      Us[idx] = (k < kend && c < b) ? __double2float_rn(U[k * ldu + c]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPerWarp; ++j) {
      const float* u = Us + (warp + 8 * j) * BN;
#pragma unroll
      for (int c = 0; c < BN; c += 4) {
        const float4 uu = *reinterpret_cast<const float4*>(u + c);
        s[0][c] = fmaf(mv[j].x, uu.x, s[0][c]);
        s[0][c + 1] = fmaf(mv[j].x, uu.y, s[0][c + 1]);
        s[0][c + 2] = fmaf(mv[j].x, uu.z, s[0][c + 2]);
        s[0][c + 3] = fmaf(mv[j].x, uu.w, s[0][c + 3]);
        s[1][c] = fmaf(mv[j].y, uu.x, s[1][c]);
        s[1][c + 1] = fmaf(mv[j].y, uu.y, s[1][c + 1]);
        s[1][c + 2] = fmaf(mv[j].y, uu.z, s[1][c + 2]);
        s[1][c + 3] = fmaf(mv[j].y, uu.w, s[1][c + 3]);
        s[2][c] = fmaf(mv[j].z, uu.x, s[2][c]);
        s[2][c + 1] = fmaf(mv[j].z, uu.y, s[2][c + 1]);
        s[2][c + 2] = fmaf(mv[j].z, uu.z, s[2][c + 2]);
        s[2][c + 3] = fmaf(mv[j].z, uu.w, s[2][c + 3]);
        s[3][c] = fmaf(mv[j].w, uu.x, s[3][c]);
        s[3][c + 1] = fmaf(mv[j].w, uu.y, s[3][c + 1]);
        s[3][c + 2] = fmaf(mv[j].w, uu.z, s[3][c + 2]);
        s[3][c + 3] = fmaf(mv[j].w, uu.w, s[3][c + 3]);
      }
    }
  }
  // float64 fixed-order tree over the 8 warps: w += w+4, then w += w+2, then 0 += 1
  __syncthreads();
  if (warp >= 4) {
    double* dst = red + (warp - 4) * BN * 128;
#pragma unroll
    for (int c = 0; c < BN; ++c) {
      *reinterpret_cast<double2*>(dst + c * 128 + 4 * lane) = make_double2(s[0][c], s[1][c]);
      *reinterpret_cast<double2*>(dst + c * 128 + 4 * lane + 2) = make_double2(s[2][c], s[3][c]);
    }
  }
  __syncthreads();
  if (warp < 4) {
    double* dst = red + warp * BN * 128;
#pragma unroll
    for (int c = 0; c < BN; ++c) {
      double2 v0 = *reinterpret_cast<const double2*>(dst + c * 128 + 4 * lane);
      double2 v1 = *reinterpret_cast<const double2*>(dst + c * 128 + 4 * lane + 2);
      v0.x = (double)s[0][c] + v0.x;
      v0.y = (double)s[1][c] + v0.y;
      v1.x = (double)s[2][c] + v1.x;
      v1.y = (double)s[3][c] + v1.y;
      *reinterpret_cast<double2*>(dst + c * 128 + 4 * lane) = v0;
      *reinterpret_cast<double2*>(dst + c * 128 + 4 * lane + 2) = v1;
    }
  }
#pragma unroll
  for (int half = 2; half >= 1; half >>= 1) {
    __syncthreads();
    if (warp < half) {
      double* dst = red + warp * BN * 128;
      const double* src = red + (warp + half) * BN * 128;
      for (int idx = lane; idx < BN * 128; idx += 32) dst[idx] += src[idx];
    }
  }
  __syncthreads();
  double* out = part + (int64_t)blockIdx.y * n * b;
  const int rows = (int)min((int64_t)128, n - row0);
  for (int idx = threadIdx.x; idx < rows * b; idx += kApplyThreads) {
    const int r = idx / b, c = idx - r * b;
    out[(row0 + r) * b + c] = red[c * 128 + r];
  }
}

// ===========================================================================
// K1 (pipelined): warp-specialised streamed pass.  One producer warp moves
// k-row segments of the operand tile and the matching rows of U into a ring
// of NST shared-memory stages with cp.async.bulk (the TMA engine, SASS
// UBLKCP), signalling an mbarrier per stage with the byte count; eight
// consumer warps wait on the stage, run the FMA block and release it.
// The grid is persistent: CTA c processes items c, c + grid, ... of the
// (k-slice, row-tile) work list, so the pipeline never drains between items.
namespace pipe {
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t* b, uint32_t bytes) {
  uint64_t st;
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 %0, [%1], %2;"
               : "=l"(st) : "r"(su32(b)), "r"(bytes) : "memory");
  (void)st;
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  uint64_t st;
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(su32(b)) : "memory");
  (void)st;
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(su32(dst)), "l"(map), "r"(x), "r"(y), "r"(su32(b)) : "memory");
}
// streaming variant: the operand is read once per pass, so its lines are marked
// evict-first in L2 (they must not displace the small, reused blocks)
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_2d_stream(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(su32(dst)), "l"(map), "r"(x), "r"(y), "r"(su32(b)), "l"(policy) : "memory");
}
}  // namespace pipe

constexpr int kPipeKC = 32;      // k rows per stage
constexpr int kPipeStages = 5;   // ring depth
constexpr int kPipeConsumers = 8;
constexpr int kPipeThreads = 32 * (kPipeConsumers + 1);

template <typename T>
struct PipeShape {
  static constexpr int RPL = sizeof(T) == 8 ? 2 : 4;  // output rows per lane (16-byte smem reads)
  static constexpr int BM = 32 * RPL;                 // output rows per item
};

template <typename T, int BN>
constexpr size_t pipe_smem_bytes() {
  return (size_t)kPipeStages * kPipeKC * PipeShape<T>::BM * sizeof(T) + (size_t)kPipeStages * kPipeKC * BN * 8 +
         (size_t)4 * BN * PipeShape<T>::BM * sizeof(T) + 2 * kPipeStages * 8;
}

template <typename T, int BN>
__global__ void __launch_bounds__(kPipeThreads, 1)
    k_dense_pass(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmU, int64_t n, int b,
                 double* __restrict__ part, int tiles, int64_t kslice, int items) {
  constexpr int RPL = PipeShape<T>::RPL, BM = PipeShape<T>::BM;
  extern __shared__ __align__(128) unsigned char smem[];
  T* Ms = reinterpret_cast<T*>(smem);
  double* Us = reinterpret_cast<double*>(smem + (size_t)kPipeStages * kPipeKC * BM * sizeof(T));
  T* red = reinterpret_cast<T*>(Us + (size_t)kPipeStages * kPipeKC * BN);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + (size_t)4 * BN * BM);
  uint64_t* empty = full + kPipeStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kPipeStages; ++st) {
      pipe::bar_init(full + st, 1);
      pipe::bar_init(empty + st, kPipeConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmM) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmU) : "memory");
  }
  __syncthreads();

  if (warp == kPipeConsumers) {
    // ---------------- producer warp: one elected lane issues two 2D TMA tiles per stage
    if (lane == 0) {
      const uint64_t pol = pipe::evict_first_policy();
      const uint32_t stage_bytes = (uint32_t)(kPipeKC * BM * sizeof(T) + kPipeKC * b * 8);
      int st = 0;
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int slice = item / tiles, tile = item - slice * tiles;
        const int64_t kbeg = (int64_t)slice * kslice, kend = min(n, kbeg + kslice);
        for (int64_t kc = kbeg; kc < kend; kc += kPipeKC) {
          pipe::bar_wait(empty + st, ph ^ 1u);
          pipe::bar_arrive_tx(full + st, stage_bytes);
          pipe::tma_2d_stream(Ms + (size_t)st * kPipeKC * BM, &tmM, tile * BM, (int)kc, full + st, pol);
          pipe::tma_2d(Us + (size_t)st * kPipeKC * BN, &tmU, 0, (int)kc, full + st);
          if (++st == kPipeStages) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  int st = 0;
  uint32_t ph = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int slice = item / tiles, tile = item - slice * tiles;
    const int64_t i0 = (int64_t)tile * BM;
    const int64_t kbeg = (int64_t)slice * kslice, kend = min(n, kbeg + kslice);
    T acc[RPL][BN];
#pragma unroll
    for (int q = 0; q < RPL; ++q)
#pragma unroll
      for (int c = 0; c < BN; ++c) acc[q][c] = (T)0;
    for (int64_t kc = kbeg; kc < kend; kc += kPipeKC) {
      const int nk = (int)min((int64_t)kPipeKC, kend - kc);
      pipe::bar_wait(full + st, ph);
      auto body = [&](int kk) {
        const T* mrow = Ms + ((size_t)st * kPipeKC + kk) * BM + RPL * lane;
        const double* urow = Us + (size_t)st * kPipeKC * BN + (size_t)kk * b;
        T mv[RPL];
        if constexpr (RPL == 2) {
          const double2 v = *reinterpret_cast<const double2*>(mrow);
          mv[0] = v.x;
          mv[1] = v.y;
        } else {
          const float4 v = *reinterpret_cast<const float4*>(mrow);
          mv[0] = v.x;
          mv[1] = v.y;
          mv[2] = v.z;
          mv[3] = v.w;
        }
#pragma unroll
        for (int c = 0; c < BN; c += 2) {
          const double2 uu = *reinterpret_cast<const double2*>(urow + c);
          const T u0 = (T)uu.x, u1 = (T)uu.y;
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            acc[q][c] = fma(mv[q], u0, acc[q][c]);
            acc[q][c + 1] = fma(mv[q], u1, acc[q][c + 1]);
          }
        }
      };
      if (nk == kPipeKC) {
#pragma unroll
        for (int j = 0; j < kPipeKC / kPipeConsumers; ++j) body(warp + kPipeConsumers * j);
      } else {
        for (int j = 0; j < kPipeKC / kPipeConsumers; ++j)
          if (warp + kPipeConsumers * j < nk) body(warp + kPipeConsumers * j);
      }
      __syncwarp();
      if (lane == 0) pipe::bar_arrive(empty + st);
      if (++st == kPipeStages) {
        st = 0;
        ph ^= 1u;
      }
    }
    // fixed-order tree over the consumer warps: w += w+4, w += w+2, 0 += 1
#pragma unroll
    for (int half = 4; half >= 1; half >>= 1) {
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kPipeConsumers) : "memory");
      if (warp >= half && warp < 2 * half) {
        T* dst = red + (size_t)(warp - half) * BN * BM;
#pragma unroll
        for (int c = 0; c < BN; ++c)
#pragma unroll
          for (int q = 0; q < RPL; ++q) dst[c * BM + RPL * lane + q] = acc[q][c];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kPipeConsumers) : "memory");
      if (warp < half) {
        const T* src = red + (size_t)warp * BN * BM;
#pragma unroll
        for (int c = 0; c < BN; ++c)
#pragma unroll
          for (int q = 0; q < RPL; ++q) acc[q][c] += src[c * BM + RPL * lane + q];
      }
    }
    if (warp == 0) {
#pragma unroll
      for (int c = 0; c < BN; ++c)
#pragma unroll
        for (int q = 0; q < RPL; ++q) red[c * BM + RPL * lane + q] = acc[q][c];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kPipeConsumers) : "memory");
    double* out = part + (int64_t)slice * n * b;
    const int rows = (int)min((int64_t)BM, n - i0);
    for (int idx = threadIdx.x; idx < rows * b; idx += 32 * kPipeConsumers) {
      const int r = idx / b, c = idx - r * b;
      out[(i0 + r) * b + c] = (double)red[c * BM + r];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kPipeConsumers) : "memory");
  }
}

// ===========================================================================
// K1 (float64, tensor path): same TMA/mbarrier producer as k_dense_pass, but
// the consumers run the FP64 tensor-core MMA (mma.sync.m8n8k4.f64, SASS
// DMMA.8x8x4): 256 FMAs per instruction instead of 32, so the FP64 pipe is fed
// without the issue/latency stalls of the DFMA loop.  Item = 128 output rows
// x one k-slice; consumer warp w owns rows [16w, 16w+16) (two 8-row m-tiles)
// x NT 8-column n-tiles over the whole k-slice, so no cross-warp reduction.
// U is staged as KC x (8 NT) with the columns beyond b zero-filled by TMA.
constexpr int kMmaRows = 128;

// U tile width in shared memory: >= the 8 NT + TAIL columns read, and = 2 (mod 8) so
// the B-fragment rows k, k+2, k+4, k+6 of a k group fall in disjoint bank quarters
template <int NT, int TAIL>
__host__ __device__ constexpr int mma_bnp() {
  return ((8 * NT + TAIL - 2 + 7) / 8) * 8 + 2;
}

template <int NT, int TAIL>
constexpr size_t mma_smem_bytes() {
  return 1024 + (size_t)kPipeStages * kPipeKC * kMmaRows * 8 + (size_t)kPipeStages * kPipeKC * mma_bnp<NT, TAIL>() * 8 +
         2 * kPipeStages * 8;
}

// Columns [0, 8 NT) of the block go through DMMA (tensor pipe); the TAIL (< 8)
// columns after them through DFMA on the FP64 pipe, which runs concurrently --
// so k = 18 costs 2 DMMA n-tiles + 2 DFMA columns instead of 3 padded n-tiles.
// CW consumer warps: 8 (warp w owns rows [16w, 16w+16), two m-tiles) or 16 (warp w owns one
// 8-row m-tile: rows [8w, 8w+8); twice the warps per SMSP to hide fragment-load latency)
//
// Stream-K: the (row tile, 32-row k chunk) space, tile-major, is cut into
// gridDim.x contiguous ranges of equal length (+-1 chunk), so every CTA
// streams the same number of operand bytes.  A CTA flushes one partial per
// tile segment it covers, into slot (its index - the index of the first CTA
// on that tile).  Pass only (STEP = false): the CTA that closes a tile zero-fills
// the tile's unused slots, so the consumer of `part` sums exactly smax slots per row.
// Fused step (STEP = true): every contributor bumps the tile's counter after its
// partial is visible; the last one records the tile in `fixlist` (it finishes the
// tile after its own range, k_dense_step_mma).  The producer warp falls through
// instead of returning when STEP, so the whole CTA can run the step tail.
__host__ __device__ __forceinline__ int sk_cfirst(int64_t x, int G, int64_t utot) {
  // the first CTA whose range contains unit x: the largest c with c * utot / G <= x
  return (int)(((x + 1) * G + utot - 1) / utot) - 1;
}

// STEP extras after the ring: U rows of the current tile (prefetched with cp.async when a tile
// segment starts) and the segment's W rows, for the segment's H partial U_tile^T W_segment
template <int NT, int TAIL>
__host__ __device__ constexpr size_t mma_step_extra_offset() {
  // the ring (operand + U stages) and its mbarriers, rounded up
  return (((size_t)kPipeStages * kPipeKC * kMmaRows * 8 + (size_t)kPipeStages * kPipeKC * mma_bnp<NT, TAIL>() * 8 +
           2 * kPipeStages * 8 + 127) / 128) * 128;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(pipe::su32(dst)), "l"(src) : "memory");
}

// diagnostics (MEGB200_PASS_STAMPS): %globaltimer per CTA at the pass's phase boundaries
// (0 CTA start, 1 dependency wait over, 2 first stage landed, 3 last stage consumed, 4 partials stored)
__device__ unsigned long long g_pass_ns[160 * 8];
__device__ __forceinline__ void pass_stamp(int on, int slot) {
  if (on) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_pass_ns[blockIdx.x * 8 + slot] = v;
  }
}

template <int NT, int TAIL, int CW, bool STEP>
__device__ __forceinline__ void dense_mma_body(const CUtensorMap* tmM, const CUtensorMap* tmU, int64_t n, int b,
                                               double* __restrict__ part, int tiles, int kch, int smax,
                                               unsigned char* base, unsigned* tilecnt, int* fixlist, int* nfix,
                                               const double* __restrict__ Ug = nullptr, int64_t ldu = 0,
                                               double* __restrict__ hpart = nullptr,
                                               const unsigned long long* wait_ctr = nullptr,
                                               unsigned long long wait_target = 0, int keep_q = 0, int keep_p = 1,
                                               int stamps = 0) {
  if (threadIdx.x == 0) pass_stamp(stamps, 0);
  const int64_t utot = (int64_t)tiles * kch;
  const int64_t ua = (int64_t)blockIdx.x * utot / gridDim.x, ub = (int64_t)(blockIdx.x + 1) * utot / gridDim.x;
  // Operand stage = 8 TMA boxes of 16 (i) x 32 (k) doubles with the 128-byte
  // swizzle (16-byte chunk index XOR row & 7), 4 KiB each; consumer warp w
  // reads box w.  Each 8-row k group feeds two MMAs, lane quad tq taking k rows
  // {2 tq} / {2 tq + 1}: under the swizzle the four rows of a half-warp land in
  // disjoint chunk pairs (A), and with a U row stride of 2 (mod 8) doubles in
  // disjoint bank quarters (B) -- both fragment loads at the 2-wavefront minimum.
  constexpr int BNP = mma_bnp<NT, TAIL>();
  constexpr int TL = TAIL > 0 ? TAIL : 1;
  double* Ms = reinterpret_cast<double*>(base);                      // stages x 8 boxes x 512 doubles
  double* Us = Ms + (size_t)kPipeStages * kPipeKC * kMmaRows;         // stages x KC x BNP
  uint64_t* full = reinterpret_cast<uint64_t*>(Us + (size_t)kPipeStages * kPipeKC * BNP);
  uint64_t* empty = full + kPipeStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kPipeStages; ++st) {
      pipe::bar_init(full + st, 1);
      pipe::bar_init(empty + st, CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmM) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmU) : "memory");
  }
  // launched programmatically dependent on the previous kernel: everything above
  // overlapped its tail; U and the partial buffer are touched only after it completed -- or,
  // after a k_fused_first_pass that released its Ritz rows early, once all of its CTAs counted
  // theirs (its last CTA may still be reducing residuals, in buffers this pass does not touch)
  if (wait_ctr) {
    if (threadIdx.x == 0) {
      unsigned long long v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(wait_ctr) : "memory");
        if (v >= wait_target) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
  } else {
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (threadIdx.x == 0) pass_stamp(stamps, 1);
  if (warp == CW) {
    if (lane == 0) {
      const uint32_t stage_bytes = (uint32_t)(kPipeKC * kMmaRows * 8 + kPipeKC * BNP * 8);
      // L2 residency: keep_q of every keep_p consecutive units are loaded evict-last (they stay in the
      // 126 MB L2 from pass to pass when the operand is not much larger than it), the rest evict-first;
      // interleaved by unit so every CTA's range holds the same mix
      const uint64_t pol_first = pipe::evict_first_policy();
      const uint64_t pol_last = keep_q > 0 ? pipe::evict_last_policy() : pol_first;
      int st = 0;
      uint32_t ph = 0;
      for (int64_t u = ua; u < ub; ++u) {
        const int tile = (int)(u / kch);
        const int64_t kc = (u - (int64_t)tile * kch) * kPipeKC;
        const uint64_t pol = (int)(u % keep_p) < keep_q ? pol_last : pol_first;
        {
          pipe::bar_wait(empty + st, ph ^ 1u);
          pipe::bar_arrive_tx(full + st, stage_bytes);
          double* mst = Ms + (size_t)st * kPipeKC * kMmaRows;
#pragma unroll
          for (int bx = 0; bx < kMmaRows / 16; ++bx)
            pipe::tma_2d_stream(mst + bx * 16 * kPipeKC, tmM, tile * kMmaRows + 16 * bx, (int)kc, full + st, pol);
          pipe::tma_2d(Us + (size_t)st * kPipeKC * BNP, tmU, 0, (int)kc, full + st);
          if (++st == kPipeStages) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
    }
    return;  // STEP: the caller's tail starts with a CTA barrier the producer warp joins
  }
  constexpr int MT = 16 / (CW / 8) / 8;  // m-tiles per warp: 2 (CW = 8) or 1 (CW = 16)
  const int mrow0 = (CW == 16) ? 8 * (warp & 1) : 0;  // first row of this warp within its box
  const int g = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  const int kperm = 2 * tq;  // {0,2,4,6}; +1 for the second MMA of a k group
  double* Usm = reinterpret_cast<double*>(base + mma_step_extra_offset<NT, TAIL>());  // 128 x b (STEP)
  double* Wsm = Usm + kMmaRows * b;                                                 // 128 x b (STEP)
  double hc[2] = {0.0, 0.0};  // STEP: this thread's entries o = tid, tid + 256 of sum_seg U_tile^T W_seg
  int st = 0;
  uint32_t ph = 0;
  for (int64_t u = ua; u < ub;) {
    const int tile = (int)(u / kch);
    const int64_t i0 = (int64_t)tile * kMmaRows;
    const int64_t uend = min(ub, (int64_t)(tile + 1) * kch);
    const bool closes = uend == (int64_t)(tile + 1) * kch;
    const int cfirst = sk_cfirst((int64_t)tile * kch, gridDim.x, utot);
    const int slot = (int)blockIdx.x - cfirst;
    const int trows = (int)min((int64_t)kMmaRows, n - i0);
    if constexpr (STEP) {
      // the tile's U rows, in flight while the segment streams (16-byte chunks)
      const int hb = b / 2;
      for (int q = threadIdx.x; q < trows * hb; q += 32 * CW) {
        const int rr = q / hb, cc = 2 * (q - rr * hb);
        cp_async16(Usm + rr * b + cc, Ug + (i0 + rr) * ldu + cc);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // two accumulator sets (even / odd k steps): dependent DMMAs on one accumulator
    // are 2 * 2 * NT instructions apart, which covers the DMMA latency
    double acc[2][MT][NT][2];
#pragma unroll
    for (int ps = 0; ps < 2; ++ps)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[ps][mt][nt][0] = acc[ps][mt][nt][1] = 0.0;
    double tl[MT][TL];  // DFMA tail: rows g (/ 8+g), this lane's k subset
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int tc = 0; tc < TL; ++tc) tl[mt][tc] = 0.0;
    for (; u < uend; ++u) {
      const int64_t kc = (u - (int64_t)tile * kch) * kPipeKC;
      const int nk = (int)min((int64_t)kPipeKC, n - kc);  // the last chunk of a row may be short
      pipe::bar_wait(full + st, ph);
      if (threadIdx.x == 0 && u == ua) pass_stamp(stamps, 2);
      const char* box = reinterpret_cast<const char*>(Ms + (size_t)st * kPipeKC * kMmaRows) + (warp / (CW / 8)) * 4096;
      const double* us = Us + (size_t)st * kPipeKC * BNP;
      auto mma_k = [&](int k, double (&ac)[MT][NT][2]) {  // one m8n8k4 step over k rows {k + kperm}
        const int kk = k + kperm;
        const bool valid = kk < nk;
        const int sw = kk & 7;
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int rib = mrow0 + 8 * mt + g;  // row within the 16-row box
          a[mt] = valid ? *reinterpret_cast<const double*>(box + kk * 128 + (((rib >> 1) ^ sw) << 4) + ((rib & 1) << 3))
                        : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double bv = valid ? us[kk * BNP + nt * 8 + g] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(ac[mt][nt][0]), "+d"(ac[mt][nt][1]) : "d"(a[mt]), "d"(bv));
        }
#pragma unroll
        for (int tc = 0; tc < TAIL; ++tc) {
          const double bt = valid ? us[kk * BNP + 8 * NT + tc] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) tl[mt][tc] = fma(a[mt], bt, tl[mt][tc]);
        }
      };
      // full chunks (all but possibly the last k chunk of a row): no bounds predicates; the
      // swizzled fragment addresses are per-lane bases plus immediates
      auto mma_full = [&](int k, double (&ac)[MT][NT][2]) {
        const int kk = k + kperm;
        const int sw = kk & 7;
        double a[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int rib = mrow0 + 8 * mt + g;
          a[mt] = *reinterpret_cast<const double*>(box + kk * 128 + (((rib >> 1) ^ sw) << 4) + ((rib & 1) << 3));
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double bv = us[kk * BNP + nt * 8 + g];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(ac[mt][nt][0]), "+d"(ac[mt][nt][1]) : "d"(a[mt]), "d"(bv));
        }
#pragma unroll
        for (int tc = 0; tc < TAIL; ++tc) {
          const double bt = us[kk * BNP + 8 * NT + tc];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) tl[mt][tc] = fma(a[mt], bt, tl[mt][tc]);
        }
      };
      if (nk == kPipeKC) {
#pragma unroll
        for (int k8 = 0; k8 < kPipeKC; k8 += 8) {
          mma_full(k8, acc[0]);
          mma_full(k8 + 1, acc[1]);
        }
      } else {
#pragma unroll
        for (int k8 = 0; k8 < kPipeKC; k8 += 8) {
          if (k8 < nk) {
            mma_k(k8, acc[0]);
            mma_k(k8 + 1, acc[1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) pipe::bar_arrive(empty + st);
      if (++st == kPipeStages) {
        st = 0;
        ph ^= 1u;
      }
    }
    if (threadIdx.x == 0 && u == ub) pass_stamp(stamps, 3);
    // C fragment: row g, columns 2*tq, 2*tq+1 of each 8x8 tile
    double* out = part + (int64_t)slot * n * b;
    const int rbase = (CW == 16) ? warp * 8 : warp * 16;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int64_t row = i0 + rbase + mt * 8 + g;
      if (row < n) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = nt * 8 + 2 * tq;
          if (c < b) out[row * b + c] = acc[0][mt][nt][0] + acc[1][mt][nt][0];
          if (c + 1 < b) out[row * b + c + 1] = acc[0][mt][nt][1] + acc[1][mt][nt][1];
        }
      }
    }
    // DFMA tail: sum the four k-subset lanes (tq) of each row, fixed xor order
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int tc = 0; tc < TAIL; ++tc) {
        double v = tl[mt][tc];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        const int64_t row = i0 + rbase + mt * 8 + g;
        if (tq == 0 && row < n) out[row * b + 8 * NT + tc] = v;
      }
    }
    if constexpr (STEP) {
      // the segment's W rows (pass part) to shared memory, next to the prefetched U rows
      const int rb = (CW == 16) ? warp * 8 : warp * 16;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int rr = rb + mt * 8 + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = nt * 8 + 2 * tq;
          if (c < b) Wsm[rr * b + c] = acc[0][mt][nt][0] + acc[1][mt][nt][0];
          if (c + 1 < b) Wsm[rr * b + c + 1] = acc[0][mt][nt][1] + acc[1][mt][nt][1];
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int tc = 0; tc < TAIL; ++tc) {
          double v = tl[mt][tc];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (tq == 0) Wsm[(rb + mt * 8 + g) * b + 8 * NT + tc] = v;
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      // the partial's global stores visible before the tile counter moves
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * CW) : "memory");
      // H partial of the segment: U_tile^T W_segment (upper triangle), accumulated in segment order
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int o = threadIdx.x + j * 32 * CW;
        if (o < b * b) {
          const int ia = o / b, c = o - ia * b;
          if (ia <= c) hc[j] += tile_dot(Usm, b, ia, Wsm, b, c, trows);
        }
      }
      if (threadIdx.x == 0) {
        // tile counter: the contributor that completes it finishes the tile (after its own range)
        const int clast = sk_cfirst((int64_t)(tile + 1) * kch - 1, gridDim.x, utot);
        const unsigned cnt = (unsigned)(clast - cfirst + 1);
        if (atomicAdd(tilecnt + tile, 1u) == cnt - 1) {
          atomicExch(tilecnt + tile, 0u);
          fixlist[(*nfix)++] = tile;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * CW) : "memory");  // Usm / Wsm free for the next segment
    } else if (closes) {
      // zero the tile's slots no CTA covers (rows of this warp)
      for (int sl = slot + 1; sl < smax; ++sl) {
        double* z = part + (int64_t)sl * n * b;
        for (int idx = lane; idx < 8 * MT * b; idx += 32) {
          const int64_t row = i0 + rbase + idx / b;
          if (row < n) z[row * b + idx % b] = 0.0;
        }
      }
    }
  }
  if constexpr (STEP) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int o = threadIdx.x + j * 32 * CW;
      if (o < b * b) hpart[(int64_t)blockIdx.x * kFusedStride + o] = hc[j];
    }
  }
  if (threadIdx.x == 0) pass_stamp(stamps, 4);
}

template <int NT, int TAIL, int CW>
__global__ void __launch_bounds__(32 * (CW + 1), 1)
    k_dense_pass_mma(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmU, int64_t n,
                     int b, double* __restrict__ part, int tiles, int kch, int smax,
                     const unsigned long long* wait_ctr, unsigned long long wait_target, int keep_q, int keep_p,
                     int stamps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* base = smem + ((1024 - ((uintptr_t)smem & 1023)) & 1023);
  dense_mma_body<NT, TAIL, CW, false>(&tmM, &tmU, n, b, part, tiles, kch, smax, base, nullptr, nullptr, nullptr,
                                      nullptr, 0, nullptr, wait_ctr, wait_target, keep_q, keep_p, stamps);
}

// ===========================================================================
// K1 + step tail in ONE launch (float64 dense operand, block b <= 32): the operand
// pass above, and -- as the tiles complete -- the whole first-pass finish of the MEG
// step (what k_fused_first_pass does after a separate pass):
//   fix-up (the last contributor of each 128-row tile): W = scale * sum_slots part +
//       L E + alpha U (E = diag(d) Eg, Eg = L^T U given), H_tile = U^T W (upper)
//   Rayleigh-Ritz (the CTA that fixes the last tile): H = sum over tiles in tile order,
//       near-diagonal / Jacobi solve (linalg.py:205-211), theta and S released by a flag;
//       the step epilogue (meg.py:347-356) after the release
//   phase 2 (CTA c takes tiles c, c + G, ...): Ritz block T = U S and V_next,
//       residuals ||W s_j - theta_j T_j|| (linalg.py:212-216), Gram of T, per tile
//   the last phase-2 arrival sums the tile partials in tile order and writes the
//       result pack (device + mapped host slot).
// Launched cooperatively (the flag spin needs every CTA resident).  Every reduction runs
// in a fixed order, so the result is bitwise reproducible; the Gram's tile partials use the
// same products as k_tile_gram, so L^T U of the next step taken from this Gram equals
// reducing it again.
namespace stepsync {  // word offsets in FusedPassArgs::sync
constexpr int kTileCnt = 256;  // per-tile contributor counters (<= kStepMaxTiles)
constexpr int kTicketA = 416;  // tiles finished (H partials ready)
constexpr int kTicketB = 417;  // phase-2 tiles done (+1 from the Rayleigh-Ritz CTA)
constexpr int kFlag = 418;     // theta / S released (epoch)
}  // namespace stepsync
constexpr int kStepMaxTiles = 148;
constexpr int kStepMaxFix = 16;
constexpr int kStepMaxTileSlots = 2;  // completed tiles whose U / W rows stay in shared memory
constexpr int kStepThreads = 32 * 9;

__device__ __forceinline__ void step_publish(unsigned* flag, unsigned epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release_u32(flag, epoch);
}

__device__ __forceinline__ void step_wait(const unsigned* flag, unsigned epoch) {
  if (threadIdx.x == 0)
    while (ld_acquire_u32(flag) != epoch) __nanosleep(32);
  __syncthreads();
}

// dA[r * wA + c] = sA[(r0 + r) * ldA + c] (and the same for B, wB = 0 for none), r < rows: eight
// loads of each source in flight per thread before the stores
__device__ __forceinline__ void step_stage2(double* dA, const double* __restrict__ sA, int64_t ldA, int wA, double* dB,
                                            const double* __restrict__ sB, int64_t ldB, int wB, int64_t r0,
                                            int rows) {
  const int ta = rows * wA, tb = rows * wB, nt = blockDim.x;
  for (int base = threadIdx.x; base < max(ta, tb); base += 8 * nt) {
    double va[8], vb[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = base + j * nt;
      const int ra = idx / max(wA, 1), ca = idx - ra * max(wA, 1);
      const int rb = idx / max(wB, 1), cb = idx - rb * max(wB, 1);
      va[j] = idx < ta ? __ldcg(sA + (r0 + ra) * ldA + ca) : 0.0;
      vb[j] = idx < tb ? __ldcg(sB + (r0 + rb) * ldB + cb) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = base + j * nt;
      if (idx < ta) dA[idx] = va[j];
      if (idx < tb) dB[idx] = vb[j];
    }
  }
}

__device__ __forceinline__ void step_stage(double* dst, const double* __restrict__ src, int64_t ld, int64_t r0,
                                           int rows, int w) {
  step_stage2(dst, src, ld, w, nullptr, nullptr, 0, 0, r0, rows);
}

// diagnostics (MEGB200_FUSED_STAMPS): %globaltimer maxima over CTAs at the tail's phase boundaries
__device__ __forceinline__ void step_stamp(unsigned long long* st, int slot) {
  if (st && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    atomicMax(st + slot, v);
  }
}

// the last arrival of phase 2: tile partials summed in tile order, result pack out
__device__ void step_finish_pack(const FusedPassArgs& a, int tiles) {
  step_stamp(a.stamps, 6);
  const int pw = a.nreq + a.gr * a.gr;
  for (int o = threadIdx.x; o < pw; o += blockDim.x) {
    const double s = tile_ordered_sum<32>(a.part2, tiles, kFusedStride, o);
    if (o < a.nreq)
      a.resid[o] = sqrt(s);
    else
      a.gram[o - a.nreq] = s;
  }
  __threadfence_block();
  __syncthreads();
  if (a.host_pack)
    for (int idx = threadIdx.x; idx < a.pack_count; idx += blockDim.x) a.host_pack[idx] = __ldcg(a.pack + idx);
  step_stamp(a.stamps, 7);
}

template <int NT, int TAIL>
__global__ void __launch_bounds__(kStepThreads, 1)
    k_dense_step_mma(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmU, int64_t n,
                     int b, double* __restrict__ part, int tiles, int kch, int smax,
                     const __grid_constant__ FusedPassArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* base = smem + ((1024 - ((uintptr_t)smem & 1023)) & 1023);
  __shared__ int s_fix[kStepMaxFix];
  __shared__ int s_nfix, s_flag;
  __shared__ double dsh[kFusedMaxL];
  __shared__ double thsh[64];
  if (threadIdx.x == 0) s_nfix = 0;  // ordered before the body's first CTA barrier
  dense_mma_body<NT, TAIL, 8, true>(&tmM, &tmU, n, b, part, tiles, kch, smax, base, a.sync + stepsync::kTileCnt,
                                    s_fix, &s_nfix, a.U, a.ldu, a.part1);
  step_stamp(a.stamps, 0);  // (per CTA) main loop and H partial done
  const int t = threadIdx.x, NTH = kStepThreads, l = a.l, rq = a.rq, G = gridDim.x;
  const int64_t utot = (int64_t)tiles * kch;
  // every CTA's H partial (sum over its segments of U_tile^T W_segment) is in a.part1: the last
  // CTA to get here forms H and solves the Rayleigh-Ritz problem while the others finish tiles
  __threadfence();
  __syncthreads();  // the ring is drained: its shared memory is reused below (the mbarriers are not touched)
  if (t == 0) {
    const unsigned old = atomicAdd(a.sync + stepsync::kTicketA, 1u);
    s_flag = old == (unsigned)G - 1;
    if (s_flag) atomicExch(a.sync + stepsync::kTicketA, 0u);
  }
  const int nfix = s_nfix;  // tiles this CTA completed (<= kStepMaxTileSlots)
  const bool rr_cta = s_flag != 0;  // (read after the barrier below)
  for (int k = t; k < l; k += NTH) {  // log-map coefficients: device kept weights (lc) or as given
    double v;
    if (a.lc.lam && k < a.lc.lr) {
      const double kept = a.lc.c1 * (a.lam_inline_n > 0 ? a.lam_inline[k] : __ldcg(a.lc.lam + k));
      v = (log(kept) - a.lc.log_tail) + (-a.lc.eta * (kept - a.lc.tail_g));
    } else {
      v = __ldcg(a.d + k);
    }
    dsh[k] = v;
  }
  __syncthreads();
  const bool is_rr = s_flag != 0;
  (void)rr_cta;
  if (nfix == 0 && !is_rr) return;
  const int lb = max(l, b);
  // shared memory: per completed tile its U and W rows (kept for phase 2), then L | T rows, E, S,
  // warp partials, H, Rayleigh-Ritz scratch (step_mma_tail_doubles)
  double* sm = reinterpret_cast<double*>(base);
  double* Ls = sm + 2 * (size_t)kStepMaxTileSlots * kMmaRows * b;  // 128 x l (fix-up) | T rows 128 x rq (phase 2)
  double* Ts = Ls;
  double* Es = Ls + kMmaRows * lb;     // l x b
  double* Ss = Es + max(l, 1) * b;     // b x rq
  double* red = Ss + b * rq;           // NTH
  double* Hs = red + NTH;              // b x b
  double* jac = Hs + b * b;            // Rayleigh-Ritz scratch
  auto Uf = [&](int f) { return sm + (size_t)f * 2 * kMmaRows * b; };
  auto Wf = [&](int f) { return sm + (size_t)f * 2 * kMmaRows * b + kMmaRows * b; };

  if (is_rr) {
    // ---- Rayleigh-Ritz: H = U^T W = scale sum_CTA H_partial + Eg^T diag(d) Eg + alpha U^T U
    // (W = scale M U + L diag(d) L^T U + alpha U), CTA partials in CTA order
    __threadfence();
    step_stamp(a.stamps, 2);
    for (int o = t; o < b * b; o += NTH) {
      const int ia = o / b, c = o - ia * b;
      double h = 0.0;
      if (ia <= c) {
        const double hm = tile_ordered_sum<32>(a.part1, G, kFusedStride, o);
        double lr = 0.0;
        for (int k = 0; k < l; ++k) lr = fma(__ldcg(a.Eg + k * a.ldg + ia) * dsh[k], __ldcg(a.Eg + k * a.ldg + c), lr);
        h = (a.scale * hm + lr) + a.alpha * __ldcg(a.Gu + ia * a.ldgu + c);
      }
      Hs[o] = h;
    }
    __syncthreads();
    if (!rr_small_neardiag<kStepThreads>(Hs, b, b, a.theta, a.Sout, jac, thsh, a.info)) {
      __syncthreads();
      jacobi_fallback(Hs, b, a.theta, a.Sout, jac, a.info);
      __syncthreads();
      for (int c = t; c < b; c += NTH) thsh[c] = a.theta[c];
      __syncthreads();
    }
    step_stamp(a.stamps, 3);
    step_publish(a.sync + stepsync::kFlag, a.epoch);
    for (int o = t; o < b * b; o += NTH) {  // H for a continued solve (read after the launch)
      const int ia = o / b, c = o - ia * b;
      if (ia <= c) a.H[ia * a.ldh + c] = Hs[o];
    }
    if (a.epi && t < 32) step_epilogue_warp(thsh, a.nreq, n, a.eps_next, a.epi);
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned old = atomicAdd(a.sync + stepsync::kTicketB, 1u);
      s_flag = old == (unsigned)tiles;
      if (s_flag) atomicExch(a.sync + stepsync::kTicketB, 0u);
    }
    __syncthreads();
    if (s_flag) {
      __threadfence();
      step_finish_pack(a, tiles);
    }
    if (nfix == 0) return;
  }

  // ---- fix-up: the W rows of each tile this CTA completed (kept in shared memory for phase 2)
  for (int idx = t; idx < l * b; idx += NTH) {
    const int k = idx / b, c = idx - k * b;
    Es[idx] = dsh[k] * __ldcg(a.Eg + k * a.ldg + c);
  }
  const int64_t slice = n * b;
  for (int f = 0; f < nfix; ++f) {
    const int tile = s_fix[f];
    const int64_t i0 = (int64_t)tile * kMmaRows;
    const int rows = (int)min((int64_t)kMmaRows, n - i0);
    double* Us = Uf(f);
    double* Ws = Wf(f);
    step_stage2(Us, a.U, a.ldu, b, Ls, a.L, a.ldl, l, i0, rows);
    __syncthreads();
    const int cf = sk_cfirst((int64_t)tile * kch, G, utot);
    const int cnt = sk_cfirst((int64_t)(tile + 1) * kch - 1, G, utot) - cf + 1;
    const int total = rows * b;
    // four outputs per thread per round, every slot load of the four in flight at once
    for (int base0 = t; base0 < total; base0 += 4 * NTH) {
      double pv[4][16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = base0 + q * NTH;
        const bool ok = idx < total;
        const double* pp = part + i0 * b + (ok ? idx : 0);
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) pv[q][s2] = (ok && s2 < cnt) ? __ldcg(pp + s2 * slice) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = base0 + q * NTH;
        if (idx < total) {
          const int rr = idx / b, c = idx - rr * b;
          double sum = 0.0;
#pragma unroll
          for (int s2 = 0; s2 < 16; ++s2) sum += pv[q][s2];  // slot order
          const double* Lr = Ls + rr * l;
          double v0 = a.scale * sum + a.alpha * Us[idx], v1 = 0.0;
          int k = 0;
          for (; k + 1 < l; k += 2) {
            v0 = fma(Lr[k], Es[k * b + c], v0);
            v1 = fma(Lr[k + 1], Es[(k + 1) * b + c], v1);
          }
          if (k < l) v0 = fma(Lr[k], Es[k * b + c], v0);
          const double wv = v0 + v1;
          Ws[idx] = wv;
          a.W[(i0 + rr) * a.ldw + c] = wv;
        }
      }
    }
    __syncthreads();  // Ls is restaged by the next tile
  }
  step_stamp(a.stamps, 1);  // fix-ups done

  // ---- phase 2 on the tiles this CTA completed (their U and W rows are still in shared memory):
  // Ritz block rows, residual and Gram partials
  step_wait(a.sync + stepsync::kFlag, a.epoch);
  step_stamp(a.stamps, 4);  // released (max over phase-2 CTAs)
  for (int idx = t; idx < b * rq; idx += NTH) {
    const int k = idx / rq, c = idx - k * rq;
    Ss[idx] = __ldcg(a.Sout + k * b + c);
  }
  for (int c = t; c < rq; c += NTH) thsh[c] = __ldcg(a.theta + c);
  __syncthreads();
  const int rpt = NTH / rq;  // rows in flight per column
  const int c = t % rq;
  const int rofs = t / rq;
  for (int f = 0; f < nfix; ++f) {
    const int tile = s_fix[f];
    const int64_t i0 = (int64_t)tile * kMmaRows;
    const int rows = (int)min((int64_t)kMmaRows, n - i0);
    const double* Us = Uf(f);
    const double* Ws = Wf(f);
    double sq = 0.0;
    if (rofs < rpt) {
      const double th = c < a.nreq ? thsh[c] : 0.0;
      const bool res = c < a.nreq;
      // four rows per round: independent chains x_q = U_row S_c, y_q = W_row S_c
      for (int r0 = rofs; r0 < rows; r0 += 4 * rpt) {
        double x[4] = {0.0, 0.0, 0.0, 0.0}, y[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = 0; k < b; ++k) {
          const double sk = Ss[k * rq + c];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int rr = min(r0 + q * rpt, rows - 1);
            x[q] = fma(Us[rr * b + k], sk, x[q]);
            if (res) y[q] = fma(Ws[rr * b + k], sk, y[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = r0 + q * rpt;
          if (rr < rows) {
            const int64_t i = i0 + rr;
            a.T[i * a.ldt + c] = x[q];
            Ts[rr * rq + c] = x[q];
            if (c < a.r2) a.V2[i * a.ld2 + c] = x[q];
            if (res) {
              const double d = y[q] - th * x[q];
              sq = fma(d, d, sq);
            }
          }
        }
      }
    }
    red[t] = sq;
    __syncthreads();  // also publishes Ts
    step_stamp(a.stamps, 5);  // Ritz rows written
    double* p2 = a.part2 + (int64_t)tile * kFusedStride;
    if (t < a.nreq) {
      double s2 = 0.0;
      for (int j = t; j < rpt * rq; j += rq) s2 += red[j];
      p2[t] = s2;
    }
    for (int o = t; o < a.gr * a.gr; o += NTH) {
      const int ia = o / a.gr, cc = o - ia * a.gr;
      p2[a.nreq + o] = tile_dot(Ts, rq, ia, Ts, rq, cc, rows);
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const unsigned old = atomicAdd(a.sync + stepsync::kTicketB, 1u);
      s_flag = old == (unsigned)tiles;
      if (s_flag) atomicExch(a.sync + stepsync::kTicketB, 0u);
    }
    __syncthreads();
    if (s_flag) {
      __threadfence();
      step_finish_pack(a, tiles);
    }
    __syncthreads();  // Ts and red are reused by the next tile
  }
}

// L^T U (l x b) and optionally L^T L (nvg x nvg) over 128-row tiles with the step tail's Gram
// products (tile_dot), the tile partials summed in tile order by the last CTA: the start of a
// step whose E is not carried over from the previous step's Ritz-block Gram (bit-identical to it).
__global__ void __launch_bounds__(256) k_tile_gram(int64_t n, const double* __restrict__ L, int64_t ldl, int l,
                                                   const double* __restrict__ U, int64_t ldu, int b, int nvg,
                                                   double* __restrict__ part, unsigned* ticket, double* __restrict__ E,
                                                   double* __restrict__ vgram, double* __restrict__ Gu) {
  extern __shared__ __align__(16) double gsm[];
  __shared__ int s_last;
  double* Ls = gsm;                  // 128 x l
  double* Us = Ls + kMmaRows * l;    // 128 x b
  const int tile = blockIdx.x, tiles = gridDim.x, t = threadIdx.x;
  const int64_t i0 = (int64_t)tile * kMmaRows;
  const int rows = (int)min((int64_t)kMmaRows, n - i0);
  step_stage2(Ls, L, ldl, l, Us, U, ldu, b, i0, rows);
  __syncthreads();
  double* p = part + (int64_t)tile * kFusedStride;
  for (int o = t; o < l * b; o += blockDim.x) p[o] = tile_dot(Ls, l, o / b, Us, b, o % b, rows);
  for (int o = t; o < nvg * nvg; o += blockDim.x) p[l * b + o] = tile_dot(Ls, l, o / nvg, Ls, l, o % nvg, rows);
  for (int o = t; o < b * b; o += blockDim.x) p[l * b + nvg * nvg + o] = tile_dot(Us, b, o / b, Us, b, o % b, rows);
  __threadfence();
  __syncthreads();
  if (t == 0) {
    s_last = atomicAdd(ticket, 1u) == (unsigned)tiles - 1;
    if (s_last) atomicExch(ticket, 0u);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int o = t; o < l * b + nvg * nvg + b * b; o += blockDim.x) {
    const double s = tile_ordered_sum<32>(part, tiles, kFusedStride, o);
    if (o < l * b)
      E[o] = s;
    else if (o < l * b + nvg * nvg)
      vgram[o - l * b] = s;
    else
      Gu[o - l * b - nvg * nvg] = s;
  }
}

// ===========================================================================
// K2: CSR product (sampled-entry gradient), one warp per row.  The warp loads 32
// (col, val) pairs with one coalesced access, then walks them two at a time: each
// half-warp takes one nonzero and reads that U row with consecutive lanes
// (columns hl and hl + 16), so a gathered row costs ~b*8/32 sectors instead of
// one sector per column.  Groups of UN steps are unrolled so their row loads are in
// flight together.  Fixed order: nonzeros in index order per half, halves
// combined at the end (bitwise reproducible).
template <int UN, int MINB>
__global__ void __launch_bounds__(256, MINB) k_csr_apply(const int32_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ col,
                                                      const double* __restrict__ val, int64_t n,
                                                      const double* __restrict__ U, int64_t ldu, int b,
                                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  double a0 = 0.0, a1 = 0.0;
  const int e0 = rowptr[row], e1 = rowptr[row + 1];
  const bool c0 = hl < b, c1 = hl + 16 < b;
  for (int base = e0; base < e1; base += 32) {
    const int e = base + lane;
    int j = 0;
    double g = 0.0;
    if (e < e1) {
      j = __ldg(col + e);
      g = __ldg(val + e);
    }
    // the batch's 16 pair-steps in groups of UN: UN row loads per lane in flight, fewer
    // registers (four CTAs per SM instead of one)
#pragma unroll
    for (int s0 = 0; s0 < 16; s0 += UN) {
      double u0[UN], u1[UN], gg[UN];
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        const int src = 2 * (s0 + q) + half;
        const int jj = __shfl_sync(0xffffffffu, j, src);
        gg[q] = __shfl_sync(0xffffffffu, g, src);
        const double* u = U + (int64_t)jj * ldu;
        u0[q] = c0 ? __ldg(u + hl) : 0.0;
        u1[q] = c1 ? __ldg(u + hl + 16) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < UN; ++q) {
        a0 = fma(gg[q], u0[q], a0);
        a1 = fma(gg[q], u1[q], a1);
      }
    }
  }
  a0 += __shfl_xor_sync(0xffffffffu, a0, 16);
  a1 += __shfl_xor_sync(0xffffffffu, a1, 16);
  if (half == 0) {
    if (c0) out[row * b + hl] = a0;
    if (c1) out[row * b + hl + 16] = a1;
  }
}

// ---------------------------------------------------------------------------
// Panel-tiled CSR pass (cfg3): the n columns are cut into P panels of pw columns whose U rows
// (pw x b doubles, <= ~200 KiB) fit shared memory.  CTA (row group g, panel p) stages panel p's rows
// of U once, then a warp per row walks that row's nonzeros inside the panel (pp: per-row panel
// pointers, columns are sorted within a row): the (column offset, value) pairs of 32 nonzeros are
// staged per warp in shared memory, each half-warp takes one nonzero per step (lane hl: block
// columns hl and hl + 16) with a broadcast read of the pair and a conflict-free read of the U row.
// Slice p of `out` (S = P slices, summed in order by the finish) holds panel p's contribution.
__global__ void __launch_bounds__(256) k_csr_panel_ptr(const int32_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ col, int64_t n, int P, int pw,
                                                       int32_t* __restrict__ pp) {
  const int64_t idx = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (idx >= n * (P + 1)) return;
  const int64_t row = idx / (P + 1);
  const int p = (int)(idx - row * (P + 1));
  int lo = rowptr[row], hi = rowptr[row + 1];
  if (p == 0) {
    hi = lo;
  } else if (p < P) {
    const int target = p * pw;  // first nonzero with column >= target
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(col + mid) < target) lo = mid + 1;
      else hi = mid;
    }
  } else {
    lo = hi;
  }
  pp[idx] = p == 0 ? hi : lo;
}

template <int NW>
__global__ void __launch_bounds__(32 * NW, 1) k_csr_apply_panel(const int32_t* __restrict__ rowptr,
                                                              const int32_t* __restrict__ col,
                                                              const double* __restrict__ val, int64_t n,
                                                              const double* __restrict__ U, int64_t ldu, int b,
                                                              double* __restrict__ out,
                                                              const int32_t* __restrict__ pp, int P, int pw,
                                                              int rpg) {
  extern __shared__ __align__(16) double csm[];
  struct Meta {
    int off, pad;
    double g;
  };
  constexpr int KB = 3;  // batches of 32 nonzeros prefetched per row (a longer panel row loops on)
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, half = lane >> 4, hl = lane & 15;
  const int p = blockIdx.x % P, grp = blockIdx.x / P;
  const int64_t c0 = (int64_t)p * pw;
  const int prow = (int)min((int64_t)pw, n - c0);
  Meta* meta = reinterpret_cast<Meta*>(csm) + warp * 32;
  double* Us = csm + (size_t)NW * 32 * 2;
  // stage the panel's rows of U: 16-byte asynchronous copies when the block is aligned (all in flight)
  if ((b & 1) == 0 && (ldu & 1) == 0 && (reinterpret_cast<uintptr_t>(U) & 15) == 0) {
    const int hb = b >> 1, total = prow * hb;
    for (int idx = t; idx < total; idx += 32 * NW) {
      const int r = idx / hb, c = 2 * (idx - r * hb);
      cp_async16(Us + r * b + c, U + (c0 + r) * ldu + c);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    const int total = prow * b;
    for (int idx = t; idx < total; idx += 32 * NW) {
      const int r = idx / b, c = idx - r * b;
      Us[idx] = __ldg(U + (c0 + r) * ldu + c);
    }
  }
  const bool ok0 = hl < b, ok1 = hl + 16 < b;
  const int64_t rbeg = (int64_t)grp * rpg, rend = min(n, (int64_t)(grp + 1) * rpg);
  const int nrw = rbeg + warp < rend ? (int)((rend - rbeg - warp + NW - 1) / NW) : 0;  // rows of this warp
  double* outp = out + (int64_t)p * n * b;
  auto load_row = [&](int e0, int e1, int (&jj)[KB], double (&gg)[KB]) {
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const int e = e0 + lane + 32 * k;
      const bool in = e < e1;
      jj[k] = in ? (__ldg(col + e) - (int)c0) * b : 0;
      gg[k] = in ? __ldg(val + e) : 0.0;
    }
  };
  // panel pointers of up to 32 of the warp's rows at a time (lane i: the chunk's i-th row), then per
  // row the first KB batches of (column, value) are prefetched while the previous row is multiplied
  int my_e0 = 0, my_e1 = 0;
  if (lane < min(nrw, 32)) {
    const int64_t r = rbeg + warp + (int64_t)NW * lane;
    my_e0 = __ldg(pp + r * (P + 1) + p);
    my_e1 = __ldg(pp + r * (P + 1) + p + 1);
  }
  int nj[KB];
  double ng[KB];
  int ne0 = __shfl_sync(0xffffffffu, my_e0, 0), ne1 = __shfl_sync(0xffffffffu, my_e1, 0);
  load_row(ne0, ne1, nj, ng);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  for (int i0 = 0; i0 < nrw; i0 += 32) {
    const int cnt = min(32, nrw - i0);
    if (i0 > 0) {
      my_e0 = my_e1 = 0;
      if (lane < cnt) {
        const int64_t r = rbeg + warp + (int64_t)NW * (i0 + lane);
        my_e0 = __ldg(pp + r * (P + 1) + p);
        my_e1 = __ldg(pp + r * (P + 1) + p + 1);
      }
      ne0 = __shfl_sync(0xffffffffu, my_e0, 0);
      ne1 = __shfl_sync(0xffffffffu, my_e1, 0);
      load_row(ne0, ne1, nj, ng);
    }
    for (int ii = 0; ii < cnt; ++ii) {
      const int e0 = ne0, e1 = ne1;
      int cj[KB];
      double cgv[KB];
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        cj[k] = nj[k];
        cgv[k] = ng[k];
      }
      if (ii + 1 < cnt) {
        ne0 = __shfl_sync(0xffffffffu, my_e0, ii + 1);
        ne1 = __shfl_sync(0xffffffffu, my_e1, ii + 1);
        load_row(ne0, ne1, nj, ng);
      }
      const int64_t row = rbeg + warp + (int64_t)NW * (i0 + ii);
      double a0 = 0.0, a1 = 0.0;
      auto batch = [&](int off, double g, int left) {
        Meta m;
        m.off = off;
        m.pad = 0;
        m.g = g;
        __syncwarp();
        meta[lane] = m;
        __syncwarp();
        const int steps = (min(32, left) + 1) >> 1;
#pragma unroll 4
        for (int q = 0; q < steps; ++q) {
          const Meta mm = meta[2 * q + half];
          const double* u = Us + mm.off;
          const double u0 = ok0 ? u[hl] : 0.0;
          const double u1 = ok1 ? u[hl + 16] : 0.0;
          a0 = fma(mm.g, u0, a0);
          a1 = fma(mm.g, u1, a1);
        }
      };
#pragma unroll
      for (int k = 0; k < KB; ++k)
        if (e0 + 32 * k < e1) batch(cj[k], cgv[k], e1 - (e0 + 32 * k));
      for (int base = e0 + 32 * KB; base < e1; base += 32) {  // long panel rows
        const int e = base + lane;
        const bool in = e < e1;
        batch(in ? (__ldg(col + e) - (int)c0) * b : 0, in ? __ldg(val + e) : 0.0, e1 - base);
      }
      a0 += __shfl_xor_sync(0xffffffffu, a0, 16);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 16);
      if (half == 0) {
        if (ok0) outp[row * b + hl] = a0;
        if (ok1) outp[row * b + hl + 16] = a1;
      }
    }
  }
}

// ===========================================================================
// Tall-skinny X^T Y partials: each CTA reduces a contiguous row range into
// one p x q partial; k_reduce_partials sums the partials in CTA order.
constexpr int kTnThreads = 512;
constexpr int kTnRows = 16;

template <int J>
__global__ void __launch_bounds__(kTnThreads) k_tn_partial(int64_t n, const double* __restrict__ X, int64_t ldx, int p,
                                                           const double* __restrict__ Y, int64_t ldy, int q,
                                                           double* __restrict__ part, int64_t rows_per_cta) {
  extern __shared__ double sm[];
  double* Xs = sm;                 // kTnRows x p
  double* Ys = sm + kTnRows * p;   // kTnRows x q
  const int pq = p * q;
  int oa[J], oc[J];
  double acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int o = threadIdx.x + j * kTnThreads;
    oa[j] = o < pq ? o / q : 0;
    oc[j] = o < pq ? o - (o / q) * q : 0;
    acc[j] = 0.0;
  }
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(n, r0 + rows_per_cta);
  for (int64_t rc = r0; rc < r1; rc += kTnRows) {
    const int rows = (int)min((int64_t)kTnRows, r1 - rc);
    __syncthreads();
    for (int idx = threadIdx.x; idx < kTnRows * p; idx += kTnThreads) {
      const int r = idx / p, a = idx - r * p;
      Xs[idx] = r < rows ? X[(rc + r) * ldx + a] : 0.0;
    }
    for (int idx = threadIdx.x; idx < kTnRows * q; idx += kTnThreads) {
      const int r = idx / q, c = idx - r * q;
      Ys[idx] = r < rows ? Y[(rc + r) * ldy + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < kTnRows; ++r) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(Xs[r * p + oa[j]], Ys[r * q + oc[j]], acc[j]);
    }
  }
  double* out = part + (int64_t)blockIdx.x * pq;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int o = threadIdx.x + j * kTnThreads;
    if (o < pq) out[o] = acc[j];
  }
}

// out[a * ldo + c] = rowscale[a] * sum_g part[g][a * q + c]; mode 1: sqrt
__global__ void k_reduce_partials(const double* __restrict__ part, int G, int p, int q, double* __restrict__ out,
                                  int64_t ldo, const double* __restrict__ rowscale, int mode) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  const int pq = p * q;
  if (o >= pq) return;
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += part[(int64_t)g * pq + o];
  const int a = o / q, c = o - a * q;
  if (rowscale) s *= rowscale[a];
  if (mode == 1) s = sqrt(s);
  out[(int64_t)a * ldo + c] = s;
}

// Y = beta Y + alpha X C   (C p x q in shared memory)
__global__ void k_nn(int64_t n, const double* __restrict__ X, int64_t ldx, int p, const double* __restrict__ C,
                     int64_t ldc, int q, double alpha, double beta, double* __restrict__ Y, int64_t ldy) {
  extern __shared__ double Cs[];
  for (int idx = threadIdx.x; idx < p * q; idx += blockDim.x) {
    const int k = idx / q, c = idx - k * q;
    Cs[idx] = C[(int64_t)k * ldc + c];
  }
  __syncthreads();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * q) return;
  const int64_t i = idx / q;
  const int c = (int)(idx - i * q);
  const double* xr = X + i * ldx;
  double s = 0.0;
  for (int k = 0; k < p; ++k) s = fma(xr[k], Cs[k * q + c], s);
  double* y = Y + i * ldy + c;
  *y = (beta == 0.0 ? 0.0 : beta * *y) + alpha * s;
}

__global__ void k_copy_block(int64_t n, int q, const double* __restrict__ src, int64_t lds, double* __restrict__ dst,
                             int64_t ldd) {
  // let a programmatically dependent launch (the operand pass) start its prologue now;
  // it waits for this grid's completion before touching memory
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * q) return;
  const int64_t i = idx / q;
  const int c = (int)(idx - i * q);
  dst[i * ldd + c] = src[i * lds + c];
}

__global__ void k_fill_gaussian(int64_t n, int q, uint64_t key, uint64_t base, double scale, int round_f32,
                                double* __restrict__ dst, int64_t ldd) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * q) return;
  const int64_t i = idx / q;
  const int c = (int)(idx - i * q);
  double v = scale * gauss_dev(key, base + (uint64_t)idx);
  if (round_f32) v = (double)__double2float_rn(v);
  dst[i * ldd + c] = v;
}

// sampled gradient values: one warp per row; optional per-row sum of squares
__global__ void __launch_bounds__(256) k_csr_values(int64_t n, const int32_t* __restrict__ rowptr,
                                                    const int32_t* __restrict__ col, const double* __restrict__ obs,
                                                    const double* __restrict__ V, int64_t ldv, int r,
                                                    const double* __restrict__ coeff, double tail,
                                                    double* __restrict__ g, double* __restrict__ sq_rows) {
  __shared__ double cf[64];
  if (threadIdx.x < r) cf[threadIdx.x] = coeff[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const double* vi = V + row * ldv;
  double s2 = 0.0;
  for (int e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) {
    const int64_t j = col[e];
    const double* vj = V + j * ldv;
    double x = 0.0;
    for (int k = 0; k < r; ++k) x = fma(vi[k] * vj[k], cf[k], x);
    if (j == row) x += tail;
    const double d = x - obs[e];
    if (g) g[e] = d;
    s2 = fma(d, d, s2);
  }
  if (sq_rows) {
    for (int off = 16; off >= 1; off >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    if (lane == 0) sq_rows[row] = s2;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_dense_stats(const T* __restrict__ M, int64_t ld, int64_t n,
                                                     double* __restrict__ part) {
  // part[2*blockIdx.x] = sum of squares over this CTA's rows, [2*blockIdx.x+1] = trace part
  __shared__ double red[2][8];
  double s = 0.0, tr = 0.0;
  const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const double v = (double)M[i * ld + j];
      s = fma(v, v, s);
      if (j == i) tr += v;
    }
  }
  for (int off = 16; off >= 1; off >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, off);
    tr += __shfl_xor_sync(0xffffffffu, tr, off);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s;
    red[1][threadIdx.x >> 5] = tr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// 1/2 ||X - M||_F^2 summed entry by entry (no cancellation between ||X||^2, <X, M>, ||M||^2):
// X_ij = sum_k (V_ik c_k) V_jk + tail [i == j] from the factors.  A CTA owns row blocks of RB rows
// (blk = blockIdx.x, + gridDim.x, ...); thread j streams M row entries coalesced and holds the
// RB values of X's column j in registers.  part[blockIdx.x] = the CTA's sum (fixed order).
template <typename T, int RB>
__global__ void __launch_bounds__(256) k_frob_direct(const T* __restrict__ M, int64_t ld, int64_t n,
                                                     const double* __restrict__ V, int64_t ldv, int r,
                                                     const double* __restrict__ coeff, double tail,
                                                     double* __restrict__ part) {
  __shared__ double vc[RB][64];
  __shared__ double red[8];
  double acc = 0.0;
  const int64_t nblk = (n + RB - 1) / RB;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t i0 = blk * RB;
    __syncthreads();
    for (int idx = threadIdx.x; idx < RB * r; idx += blockDim.x) {
      const int ii = idx / r, k = idx - ii * r;
      vc[ii][k] = i0 + ii < n ? V[(i0 + ii) * ldv + k] * coeff[k] : 0.0;
    }
    __syncthreads();
    const int rows = (int)min((int64_t)RB, n - i0);
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      double x[RB];
#pragma unroll
      for (int ii = 0; ii < RB; ++ii) x[ii] = 0.0;
      for (int k = 0; k < r; ++k) {
        const double v = V[j * ldv + k];
#pragma unroll
        for (int ii = 0; ii < RB; ++ii) x[ii] = fma(vc[ii][k], v, x[ii]);
      }
#pragma unroll
      for (int ii = 0; ii < RB; ++ii) {
        if (ii < rows) {
          const double d = (x[ii] + (i0 + ii == j ? tail : 0.0)) - (double)M[(i0 + ii) * ld + j];
          acc = fma(d, d, acc);
        }
      }
    }
  }
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < 8; ++w) a += red[w];
    part[blockIdx.x] = a;
  }
}

__device__ __forceinline__ double uniform_dev(uint64_t key, uint64_t ctr) {
  return (double)(mix64(key + (ctr + 1) * kGolden) >> 11) * kInv53;
}

// Config-3 sampling pattern (twin of oracle/inputs.sampled_instance): (i, j) is observed iff
// U[0,1) at the canonical counter min(i,j) * n + max(i,j) of stream 3 is < p -- a symmetric
// pattern.  One warp per row; columns ascend, so each CSR row comes out sorted.
__global__ void __launch_bounds__(256) k_sampled_count(int64_t n, uint64_t kmask, double p,
                                                       int32_t* __restrict__ counts) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  int c = 0;
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool hit = j < n && uniform_dev(kmask, (uint64_t)(min(i, j) * n + max(i, j))) < p;
    c += __popc(__ballot_sync(0xffffffffu, hit));
  }
  if (lane == 0) counts[i] = c;
}

// observed values (U diag(lam) U^T)_ij + obs_noise * N(0,1) at the same canonical counter (stream 4)
__global__ void __launch_bounds__(256) k_sampled_fill(int64_t n, uint64_t kmask, uint64_t knoise, double p,
                                                      const double* __restrict__ U, int r,
                                                      const double* __restrict__ lam, double obs_noise,
                                                      const int32_t* __restrict__ rowptr, int32_t* __restrict__ col,
                                                      double* __restrict__ val) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  int64_t pos = rowptr[i];
  for (int64_t j0 = 0; j0 < n; j0 += 32) {
    const int64_t j = j0 + lane;
    const uint64_t ctr = (uint64_t)(min(i, j) * n + max(i, j));
    const bool hit = j < n && uniform_dev(kmask, ctr) < p;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const int64_t at = pos + __popc(m & ((1u << lane) - 1u));
      double pl = 0.0;
      for (int k = 0; k < r; ++k) pl = fma(U[i * r + k] * U[j * r + k], lam[k], pl);
      col[at] = (int32_t)j;
      val[at] = pl + obs_noise * gauss_dev(knoise, ctr);
    }
    pos += __popc(m);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_gen_dense_target(const double* __restrict__ U, int r,
                                                          const double* __restrict__ lam, double sigma, uint64_t key,
                                                          T* __restrict__ M, int64_t ld, int64_t n) {
  __shared__ double lm[64];
  if (threadIdx.x < r) lm[threadIdx.x] = lam[threadIdx.x];
  __syncthreads();
  const int64_t i = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int k = 0; k < r; ++k) acc = fma(U[i * r + k] * U[j * r + k], lm[k], acc);
  if (sigma != 0.0) {
    const double g = gauss_dev(key, (uint64_t)i * n + j) + gauss_dev(key, (uint64_t)j * n + i);
    acc += sigma * ((0.5 / sqrt((double)n)) * g);
  }
  M[i * ld + j] = (T)acc;
}

__global__ void k_set_identity(int64_t n, double* __restrict__ Q, int64_t ldq) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  const int64_t i = idx / n, j = idx - i * n;
  Q[i * ldq + j] = i == j ? 1.0 : 0.0;
}

__global__ void k_set_diag(double* __restrict__ H, int cap, int k, const double* __restrict__ theta) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= cap * cap) return;
  const int i = idx / cap, j = idx - i * cap;
  H[idx] = (i == j && i < k) ? theta[i] : 0.0;
}

// Small problems solved on the identity basis (n <= the Rayleigh-Ritz limit): the operator itself,
// A = scale * M + L diag(d) L^T + alpha I, formed entry by entry into H (the Rayleigh-Ritz matrix) and
// AQ (the images A I) in one launch -- instead of n / 32 block passes over identity columns.
constexpr int kFormMaxLowrank = 160;
__global__ void __launch_bounds__(128) k_form_operator(int64_t n, const double* __restrict__ M, int64_t ldm, double scale,
                                                       const double* __restrict__ Lf, int64_t ldl, int l,
                                                       const double* __restrict__ d, LamCoef lc, double alpha,
                                                       double* __restrict__ AQ, int64_t ldq, double* __restrict__ H,
                                                       int64_t ldh) {
  __shared__ double dsh[kFormMaxLowrank];
  __shared__ double li[kFormMaxLowrank];
  const int i = blockIdx.x;
  for (int k = threadIdx.x; k < l; k += 128) {
    double v;
    if (lc.lam && k < lc.lr) {
      const double kept = lc.c1 * lc.lam[k];
      v = (log(kept) - lc.log_tail) + (-lc.eta * (kept - lc.tail_g));
    } else {
      v = d[k];
    }
    dsh[k] = v;
    li[k] = Lf[(int64_t)i * ldl + k] * v;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += 128) {
    double a0 = 0.0, a1 = 0.0;
    const double* lj = Lf + (int64_t)j * ldl;
    int k = 0;
    for (; k + 1 < l; k += 2) {
      a0 = fma(li[k], lj[k], a0);
      a1 = fma(li[k + 1], lj[k + 1], a1);
    }
    if (k < l) a0 = fma(li[k], lj[k], a0);
    // the pass reads rows of M where the product needs columns (M symmetric): M[j, i]
    const double v = (scale != 0.0 ? scale * M[(int64_t)j * ldm + i] : 0.0) + (a0 + a1) + (i == j ? alpha : 0.0);
    AQ[(int64_t)i * ldq + j] = v;
    H[(int64_t)i * ldh + j] = v;
  }
}

// Thick restart of the basis in ONE launch, in place: Q[:, 0:keep] = Q[:, 0:m] S_keep, the same for
// the images AQ, and the tq carried columns [m, m + tq) of both moved to [keep, keep + tq).  A CTA
// stages 32 rows of both arrays (m + tq columns) in shared memory next to S_keep (m x keep), so the
// rows are read once and written once (the seven launches this replaces re-read S per 256 outputs).
constexpr int kRestartRows = 32;
__global__ void __launch_bounds__(256) k_restart_basis(int64_t n, double* __restrict__ Q, double* __restrict__ AQ,
                                                       int64_t ldq, const double* __restrict__ S, int m, int keep,
                                                       int tq) {
  extern __shared__ double rsm[];
  const int W = m + tq, t = threadIdx.x;
  double* Ss = rsm;              // m x keep
  double* Xs = Ss + m * keep;    // 2 x kRestartRows x W
  for (int idx = t; idx < m * keep; idx += 256) {
    const int k = idx / keep, c = idx - k * keep;
    Ss[idx] = S[(int64_t)k * m + c];
  }
  const int64_t rows_per = ((n + gridDim.x - 1) / gridDim.x + kRestartRows - 1) / kRestartRows * kRestartRows;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(n, r0 + rows_per);
  for (int64_t rc = r0; rc < r1; rc += kRestartRows) {
    const int rows = (int)min((int64_t)kRestartRows, r1 - rc);
    __syncthreads();
    for (int idx = t; idx < rows * W; idx += 256) {
      const int r = idx / W, k = idx - r * W;
      Xs[idx] = Q[(rc + r) * ldq + k];
      Xs[kRestartRows * W + idx] = AQ[(rc + r) * ldq + k];
    }
    __syncthreads();
    // 2 rows x 4 columns per thread: six shared-memory loads per eight multiply-adds (one output per
    // thread loads two operands per multiply-add and is bound by shared-memory wavefronts)
    const int ncg = (keep + 3) / 4, nrg = (rows + 1) / 2;
    for (int o = t; o < 2 * nrg * ncg; o += 256) {
      const int mat = o / (nrg * ncg), rem = o - mat * nrg * ncg;
      const int r = 2 * (rem / ncg), c = 4 * (rem - (rem / ncg) * ncg);
      const double* x0 = Xs + mat * kRestartRows * W + r * W;
      const double* x1 = x0 + (r + 1 < rows ? W : 0);
      double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      for (int k = 0; k < m; ++k) {
        const double xa = x0[k], xb = x1[k];
        const double* sk = Ss + k * keep + c;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double sv = c + u < keep ? sk[u] : 0.0;
          acc[0][u] = fma(xa, sv, acc[0][u]);
          acc[1][u] = fma(xb, sv, acc[1][u]);
        }
      }
      double* dst = mat ? AQ : Q;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (c + u < keep) {
          dst[(rc + r) * ldq + c + u] = acc[0][u];
          if (r + 1 < rows) dst[(rc + r + 1) * ldq + c + u] = acc[1][u];
        }
      }
    }
    for (int o = t; o < 2 * rows * tq; o += 256) {
      const int mat = o / (rows * tq), rem = o - mat * rows * tq;
      const int r = rem / tq, j = rem - r * tq;
      (mat ? AQ : Q)[(rc + r) * ldq + keep + j] = Xs[mat * kRestartRows * W + r * W + m + j];
    }
  }
}

// one CTA: the new block's column block B = H[0:m+q, m:m+q] is staged in shared memory, H is
// cleared, then diag(theta), S_keep^T B[0:m] and the block's own diagonal block are written
__global__ void __launch_bounds__(1024) k_restart_h(double* __restrict__ H, int cap, const double* __restrict__ S, int m,
                                                    int keep, int q, const double* __restrict__ theta) {
  extern __shared__ double bs[];  // (m + q) x q, then S_keep (m x keep)
  double* Ss = bs + (m + q) * q;
  const int t = threadIdx.x, NT = blockDim.x;
  for (int idx = t; idx < (m + q) * q; idx += NT) {
    const int i = idx / q, j = idx - i * q;
    bs[idx] = H[(int64_t)i * cap + m + j];
  }
  for (int idx = t; idx < m * keep; idx += NT) {
    const int k = idx / keep, c = idx - k * keep;
    Ss[idx] = S[(int64_t)k * m + c];
  }
  __syncthreads();
  for (int idx = t; idx < cap * cap; idx += NT) H[idx] = 0.0;
  __syncthreads();
  for (int i = t; i < keep; i += NT) H[(int64_t)i * cap + i] = theta[i];
  for (int idx = t; idx < keep * q; idx += NT) {
    const int i = idx / q, j = idx - i * q;
    double a0 = 0.0, a1 = 0.0;
    int k = 0;
    for (; k + 1 < m; k += 2) {
      a0 = fma(Ss[k * keep + i], bs[k * q + j], a0);
      a1 = fma(Ss[(k + 1) * keep + i], bs[(k + 1) * q + j], a1);
    }
    if (k < m) a0 = fma(Ss[k * keep + i], bs[k * q + j], a0);
    H[(int64_t)i * cap + keep + j] = a0 + a1;
  }
  for (int idx = t; idx < q * q; idx += NT) {
    const int i = idx / q, j = idx - i * q;
    if (i <= j) H[(int64_t)(keep + i) * cap + keep + j] = bs[(m + i) * q + j];
  }
}

__global__ void k_reduce_sum(const double* __restrict__ part, int slots, int width, double* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= width) return;
  double s = 0.0;
  for (int g = 0; g < slots; ++g) s += part[(int64_t)g * width + c];
  out[c] = s;
}

template <int BN>
void launch_dense_f64(const Launch& L, const double* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                      double* part, int S, int64_t kslice, bool vec) {
  const size_t smem = (size_t)(KC * BN + 4 * BN * 64) * sizeof(double);
  dim3 grid(cdiv(n, 64), S);
  if (vec) {
    static char attr = 0;
    if (first_on_device(&attr)) {
      MEG_CUDA(cudaFuncSetAttribute(k_dense_apply_f64<BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k_dense_apply_f64<BN, true><<<grid, kApplyThreads, smem, L.stream>>>(M, ldm, n, U, ldu, b, part, kslice);
  } else {
    static char attr = 0;
    if (first_on_device(&attr)) {
      MEG_CUDA(cudaFuncSetAttribute(k_dense_apply_f64<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k_dense_apply_f64<BN, false><<<grid, kApplyThreads, smem, L.stream>>>(M, ldm, n, U, ldu, b, part, kslice);
  }
  MEG_LAUNCHED();
  ++*L.counter;
}

template <int BN>
void launch_dense_f32(const Launch& L, const float* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                      double* part, int S, int64_t kslice, bool vec) {
  const size_t smem = (size_t)((KC * BN + 1) / 2 + 4 * BN * 128) * sizeof(double);
  dim3 grid(cdiv(n, 128), S);
  if (vec) {
    static char attr = 0;
    if (first_on_device(&attr)) {
      MEG_CUDA(cudaFuncSetAttribute(k_dense_apply_f32<BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k_dense_apply_f32<BN, true><<<grid, kApplyThreads, smem, L.stream>>>(M, ldm, n, U, ldu, b, part, kslice);
  } else {
    static char attr = 0;
    if (first_on_device(&attr)) {
      MEG_CUDA(cudaFuncSetAttribute(k_dense_apply_f32<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k_dense_apply_f32<BN, false><<<grid, kApplyThreads, smem, L.stream>>>(M, ldm, n, U, ldu, b, part, kslice);
  }
  MEG_LAUNCHED();
  ++*L.counter;
}

}  // namespace

// ===========================================================================
// launch wrappers

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    MEG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(MEGB200_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D row-major tensor map: inner dimension `cols` (contiguous), outer `rows`, leading dimension `ld`
CUtensorMap encode_map(const void* base, CUtensorMapDataType dt, size_t es, int64_t cols, int64_t rows, int64_t ld,
                       uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(MEGB200_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return map;
}

// small direct-mapped cache of encoded tensor maps (the descriptors are pure
// functions of their arguments; re-encoding costs ~1 us of host time per launch)
CUtensorMap make_map(const void* base, CUtensorMapDataType dt, size_t es, int64_t cols, int64_t rows, int64_t ld,
                     uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  struct Key {
    const void* base;
    int dt;
    int64_t cols, rows, ld;
    uint32_t bc, br;
    int swz;
    bool operator==(const Key& o) const {
      return base == o.base && dt == o.dt && cols == o.cols && rows == o.rows && ld == o.ld && bc == o.bc &&
             br == o.br && swz == o.swz;
    }
  };
  struct Entry {
    Key key;
    CUtensorMap map;
    bool used;
  };
  static thread_local Entry cache[64] = {};
  const Key k{base, (int)dt, cols, rows, ld, box_cols, box_rows, (int)swz};
  const size_t h = (((uintptr_t)base >> 4) ^ (size_t)cols * 31 ^ (size_t)box_cols * 7 ^ (size_t)swz) & 63;
  Entry& e = cache[h];
  if (!(e.used && e.key == k)) {
    e.map = encode_map(base, dt, es, cols, rows, ld, box_cols, box_rows, swz);
    e.key = k;
    e.used = true;
  }
  return e.map;
}

template <typename T, int BN>
void launch_pipe(const Launch& L, const T* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                 double* part, int tiles, int64_t kslice, int items, int grid) {
  constexpr size_t smem = pipe_smem_bytes<T, BN>();
  static char attr = 0;
  if (first_on_device(&attr)) {
    MEG_CUDA(cudaFuncSetAttribute(k_dense_pass<T, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  const CUtensorMap tmM = make_map(M, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                   sizeof(T), n, n, ldm, PipeShape<T>::BM, kPipeKC);
  const CUtensorMap tmU = make_map(U, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, b, n, ldu, (uint32_t)b, kPipeKC);
  k_dense_pass<T, BN><<<grid, kPipeThreads, smem, L.stream>>>(tmM, tmU, n, b, part, tiles, kslice, items);
  MEG_LAUNCHED();
  ++*L.counter;
}

template <typename T>
void dispatch_pipe(const Launch& L, const T* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                   double* part, int tiles, int64_t kslice, int items, int grid) {
  switch ((b + 1) / 2) {
#define MEG_PIPE_CASE(h) \
  case h:                \
    launch_pipe<T, 2 * h>(L, M, ldm, n, U, ldu, b, part, tiles, kslice, items, grid); \
    break;
    MEG_PIPE_CASE(1) MEG_PIPE_CASE(2) MEG_PIPE_CASE(3) MEG_PIPE_CASE(4) MEG_PIPE_CASE(5) MEG_PIPE_CASE(6)
    MEG_PIPE_CASE(7) MEG_PIPE_CASE(8) MEG_PIPE_CASE(9) MEG_PIPE_CASE(10) MEG_PIPE_CASE(11) MEG_PIPE_CASE(12)
    MEG_PIPE_CASE(13) MEG_PIPE_CASE(14) MEG_PIPE_CASE(15) MEG_PIPE_CASE(16)
#undef MEG_PIPE_CASE
    default:
      throw Error(MEGB200_ERR_PARAM, "pipelined pass supports b <= 32");
  }
}

// 8 consumer warps (two m-tiles each); the 16-warp variant measured slower (47 vs 37 us at
// n = 4096, k = 18) and is kept only as a diagnostics option (MEGB200_MMA_WARPS=16)
int mma_consumer_warps() {
  static const int cw = [] {
    const char* e = getenv("MEGB200_MMA_WARPS");
    return (e && atoi(e) == 16) ? 16 : 8;
  }();
  return cw;
}

// Share of the operand's units loaded evict-last (L2-resident from pass to pass): none by default;
// MEGB200_L2_KEEP="q/p" (diagnostics) sets it
void l2_keep_fraction(int64_t operand_bytes, int* q, int* p) {
  static const int env_q = [] {
    const char* e = getenv("MEGB200_L2_KEEP");
    return e ? atoi(e) : -1;
  }();
  static const int env_p = [] {
    const char* e = getenv("MEGB200_L2_KEEP");
    const char* s = e ? strchr(e, '/') : nullptr;
    return s ? std::max(1, atoi(s + 1)) : 8;
  }();
  (void)operand_bytes;
  *q = 0;
  *p = 1;
  if (env_q >= 0) {
    *q = env_q;
    *p = env_p;
  }
}

template <int NT, int TAIL>
void launch_pipe_mma(const Launch& L, const double* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                     double* part, int tiles, int kch, int smax, int grid) {
  constexpr size_t smem = mma_smem_bytes<NT, TAIL>();
  const int cw = mma_consumer_warps();
  static char attr = 0;
  if (first_on_device(&attr)) {
    MEG_CUDA(cudaFuncSetAttribute(k_dense_pass_mma<NT, TAIL, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    MEG_CUDA(cudaFuncSetAttribute(k_dense_pass_mma<NT, TAIL, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  }
  const CUtensorMap tmM =
      make_map(M, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, n, n, ldm, 16, kPipeKC, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tmU =
      make_map(U, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, b, n, ldu, (uint32_t)mma_bnp<NT, TAIL>(), kPipeKC);
  // programmatic dependent launch: the CTA prologue (shared memory, mbarriers,
  // tensor-map prefetch) overlaps the preceding kernel
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32 * (cw + 1));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.stream;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  int keep_q = 0, keep_p = 1;
  l2_keep_fraction((int64_t)n * n * 8, &keep_q, &keep_p);
  static const int stamps = getenv("MEGB200_PASS_STAMPS") != nullptr;
  if (cw == 16)
    MEG_CUDA(cudaLaunchKernelEx(&cfg, k_dense_pass_mma<NT, TAIL, 16>, tmM, tmU, n, b, part, tiles, kch, smax,
                                L.wait_ctr, L.wait_target, keep_q, keep_p, stamps));
  else
    MEG_CUDA(cudaLaunchKernelEx(&cfg, k_dense_pass_mma<NT, TAIL, 8>, tmM, tmU, n, b, part, tiles, kch, smax,
                                L.wait_ctr, L.wait_target, keep_q, keep_p, stamps));
  MEG_LAUNCHED();
  ++*L.counter;
}

// Stream-K grid of the DMMA pass over (128-row tile, 32-row k chunk) units: one CTA per SM,
// shrunk until every tile is covered by at most min(cap, 16) CTAs (its partial slots).
void stream_k_grid(int64_t n, int sm_count, int64_t part_cap_slices, int* grid_out, int* smax_out) {
  const int tiles = cdiv(n, kMmaRows);
  const int kch = cdiv(n, kPipeKC);
  const int64_t utot = (int64_t)tiles * kch;
  const int cap = (int)std::max<int64_t>(1, std::min<int64_t>(part_cap_slices, 16));
  int grid = (int)std::min<int64_t>(sm_count, utot);
  int smax = 1;
  for (;;) {
    smax = 1;
    for (int t = 0; t < tiles; ++t)
      smax = std::max(smax, sk_cfirst((int64_t)(t + 1) * kch - 1, grid, utot) - sk_cfirst((int64_t)t * kch, grid, utot) + 1);
    if (smax <= cap || grid == 1) break;
    grid = std::max(1, grid * cap / (smax + 1));
  }
  *grid_out = grid;
  *smax_out = smax;
}

template <int NT, int TAIL>
void launch_step_mma(const Launch& L, const double* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                     double* part, int tiles, int kch, int smax, int grid, const FusedPassArgs& a) {
  constexpr size_t smem_ring = mma_smem_bytes<NT, TAIL>();
  const size_t smem = 1024 + mma_step_extra_offset<NT, TAIL>() + 2 * (size_t)kMmaRows * b * sizeof(double);
  (void)smem_ring;
  static char attr = 0;
  if (first_on_device(&attr))
    MEG_CUDA(cudaFuncSetAttribute(k_dense_step_mma<NT, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(1024 + mma_step_extra_offset<NT, TAIL>() +
                                        2 * kMmaRows * (8 * NT + TAIL) * sizeof(double))));
  const CUtensorMap tmM =
      make_map(M, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, n, n, ldm, 16, kPipeKC, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap tmU =
      make_map(U, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, b, n, ldu, (uint32_t)mma_bnp<NT, TAIL>(), kPipeKC);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  // the release flag needs every CTA resident: cooperative launch (driver-guaranteed co-residency)
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  MEG_CUDA(cudaLaunchKernelEx(&cfg, k_dense_step_mma<NT, TAIL>, tmM, tmU, n, b, part, tiles, kch, smax, a));
  MEG_LAUNCHED();
  ++*L.counter;
}

// Choose the number of k-slices S so that tiles * S fills whole waves of one
// CTA per SM (static round-robin of the persistent grid), preferring small S.
int choose_slices(int tiles, int64_t n, int sm_count, int s_min, int s_max) {
  int best = s_min;
  double best_eff = -1.0;
  for (int S = s_min; S <= s_max; ++S) {
    if ((int64_t)S * kPipeKC * 2 > n && S > s_min) break;
    const int items = tiles * S;
    const int waves = cdiv(items, sm_count);
    const double eff = (double)items / ((double)waves * sm_count);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = S;
    }
  }
  return best;
}

int dense_apply_partial(const Launch& L, const void* M, int dtype, int64_t ldm, int64_t n, const double* U,
                        int64_t ldu, int b, double* part, int64_t part_cap_slices, int sm_count, float* uscratch) {
  if (dtype == MEGB200_F32 && uscratch && umma_pass_supported(n, b, ldm, M))
    return dense_pass_umma(L, static_cast<const float*>(M), ldm, n, U, ldu, b, part, part_cap_slices, sm_count,
                           uscratch);
  {
    const size_t es = dtype == MEGB200_F64 ? 8 : 4;
    const bool aligned = b % 2 == 0 && b <= 32 && ldu % 2 == 0 && ((uintptr_t)U % 16 == 0) &&
                         (ldm * es) % 16 == 0 && ((uintptr_t)M % 16 == 0) && (n * es) % 16 == 0;
    if (aligned && dtype == MEGB200_F64 && getenv("MEGB200_NO_DMMA") == nullptr) {
      // stream-K over (row tile, k chunk): one CTA per SM, equal chunk counts; the grid
      // shrinks until every tile is covered by at most part_cap_slices CTAs
      const int tiles = cdiv(n, kMmaRows);
      const int kch = cdiv(n, kPipeKC);
      int grid = 0, smax = 0;
      // after an early-released fused first pass, one SM stays with its last CTA (the residual
      // reduction): the pass takes the others, so none of its CTAs queues behind that one.  Always
      // one SM less, whether or not this launch follows a fused pass: the stream-K partition (hence
      // every bit of the result) must not depend on what ran before
      stream_k_grid(n, std::max(1, sm_count - 1), part_cap_slices, &grid, &smax);
      const double* m = static_cast<const double*>(M);
      // DMMA n-tiles for the multiple-of-8 head of the block, DFMA for the (even) rest
#define MEG_MMA(nt, tail) launch_pipe_mma<nt, tail>(L, m, ldm, n, U, ldu, b, part, tiles, kch, smax, grid)
      static const bool pad = getenv("MEGB200_MMA_PAD") != nullptr;  // diagnostics: DMMA-only (padded) n-tiles
      switch (b < 8 ? 0 : (pad && b % 8 ? (b + 7) / 8 * 8 : b)) {
        case 0: MEG_MMA(1, 0); break;
        case 8: MEG_MMA(1, 0); break;
        case 10: MEG_MMA(1, 2); break;
        case 12: MEG_MMA(1, 4); break;
        case 14: MEG_MMA(1, 6); break;
        case 16: MEG_MMA(2, 0); break;
        case 18: MEG_MMA(2, 2); break;
        case 20: MEG_MMA(2, 4); break;
        case 22: MEG_MMA(2, 6); break;
        case 24: MEG_MMA(3, 0); break;
        case 26: MEG_MMA(3, 2); break;
        case 28: MEG_MMA(3, 4); break;
        case 30: MEG_MMA(3, 6); break;
        default: MEG_MMA(4, 0); break;
      }
#undef MEG_MMA
      return smax;
    }
    if (aligned) {
      const int BM = dtype == MEGB200_F64 ? 64 : 128;
      const int tiles = cdiv(n, BM);
      int s_min = dtype == MEGB200_F64 ? 1 : std::max(1, cdiv(n, kF32Slice));
      int s_max = std::max(s_min, (int)std::min<int64_t>(part_cap_slices, 16));
      s_min = std::min(s_min, (int)part_cap_slices);
      int S = choose_slices(tiles, n, sm_count, s_min, s_max);
      int64_t kslice = (int64_t)cdiv(cdiv(n, S), kPipeKC) * kPipeKC;
      S = cdiv(n, kslice);
      const int items = tiles * S;
      const int grid = std::min(items, sm_count);
      if (dtype == MEGB200_F64)
        dispatch_pipe<double>(L, static_cast<const double*>(M), ldm, n, U, ldu, b, part, tiles, kslice, items, grid);
      else
        dispatch_pipe<float>(L, static_cast<const float*>(M), ldm, n, U, ldu, b, part, tiles, kslice, items, grid);
      return S;
    }
  }
  const int rows = dtype == MEGB200_F64 ? 64 : 128;
  const int tiles = cdiv(n, rows);
  int S = std::max(1, cdiv(sm_count, tiles));
  if (dtype != MEGB200_F64) S = std::max(S, cdiv(n, kF32Slice));
  S = std::min<int>((int)part_cap_slices, S);
  int64_t kslice = (int64_t)cdiv(cdiv(n, S), KC) * KC;
  S = cdiv(n, kslice);
  if (dtype == MEGB200_F64) {
    const bool vec = (ldm % 2 == 0) && ((uintptr_t)M % 16 == 0);
    const double* m = static_cast<const double*>(M);
    if (b <= 8)
      launch_dense_f64<8>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
    else if (b <= 16)
      launch_dense_f64<16>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
    else if (b <= 24)
      launch_dense_f64<24>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
    else
      launch_dense_f64<32>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
  } else {
    const bool vec = (ldm % 4 == 0) && ((uintptr_t)M % 16 == 0);
    const float* m = static_cast<const float*>(M);
    if (b <= 8)
      launch_dense_f32<8>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
    else if (b <= 16)
      launch_dense_f32<16>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
    else if (b <= 24)
      launch_dense_f32<24>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
    else
      launch_dense_f32<32>(L, m, ldm, n, U, ldu, b, part, S, kslice, vec);
  }
  return S;
}

// panel geometry of the tiled CSR pass: the widest panel whose U rows (pw x b doubles) fit ~200 KiB
constexpr size_t kCsrPanelSmem = 200 * 1024;
constexpr int kCsrPanelWarps = 16;

int csr_apply_partial(const Launch& L, const int32_t* rowptr, const int32_t* col, const double* val, int64_t n,
                      const double* U, int64_t ldu, int b, double* part, int64_t part_cap_slices, int32_t* pp,
                      bool* pp_valid, int sm_count) {
  if (b > 32) throw Error(MEGB200_ERR_PARAM, "CSR pass supports b <= 32");
  static const bool no_panel = getenv("MEGB200_NO_CSR_PANEL") != nullptr;  // diagnostics: the L2-gather kernel
  const size_t meta = (size_t)kCsrPanelWarps * 32 * 16;
  const int64_t cap_rows = (int64_t)((kCsrPanelSmem - meta) / ((size_t)b * 8));
  const int P = (int)cdiv(n, cap_rows);
  if (!no_panel && pp && pp_valid && P <= kCsrMaxPanels && P <= part_cap_slices && n >= 1024) {
    const int pw = (int)cdiv(n, P);
    if (!*pp_valid) {
      k_csr_panel_ptr<<<cdiv(n * (P + 1), 256), 256, 0, L.stream>>>(rowptr, col, n, P, pw, pp);
      MEG_LAUNCHED();
      ++*L.counter;
      *pp_valid = true;
    }
    // row groups: the grid covers the SMs about once (one CTA per SM: the panel takes the shared memory)
    const int RG = std::max(1, sm_count / P);
    const int rpg = (int)cdiv(n, RG);
    const int rgs = (int)cdiv(n, rpg);
    const size_t smem = (size_t)pw * b * 8 + meta;
    static char attr = 0;
    if (first_on_device(&attr))
      MEG_CUDA(cudaFuncSetAttribute(k_csr_apply_panel<kCsrPanelWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kCsrPanelSmem));
    k_csr_apply_panel<kCsrPanelWarps><<<P * rgs, 32 * kCsrPanelWarps, smem, L.stream>>>(rowptr, col, val, n, U, ldu, b,
                                                                                       part, pp, P, pw, rpg);
    MEG_LAUNCHED();
    ++*L.counter;
    return P;
  }
  // four row loads in flight per lane at four CTAs per SM (cfg3 pass+finish 107 us) beat eight at
  // three CTAs (112 us) and sixteen at one (139 us): the gathers need warps more than depth
  k_csr_apply<4, 4><<<cdiv(n, 8), 256, 0, L.stream>>>(rowptr, col, val, n, U, ldu, b, part);
  MEG_LAUNCHED();
  ++*L.counter;
  return 1;
}

void tn(const Launch& L, int64_t n, const double* X, int64_t ldx, int p, const double* Y, int64_t ldy, int q,
        double* C, int64_t ldc, const double* rowscale, double* part, int64_t part_cap, int sm_count) {
  const int pq = p * q;
  int G = std::max(1, std::min(sm_count, cdiv(n, 128)));
  while ((int64_t)G * pq > part_cap && G > 1) G = (G + 1) / 2;
  const int64_t rows_per = (int64_t)cdiv(cdiv(n, G), kTnRows) * kTnRows;
  G = cdiv(n, rows_per);
  const size_t smem = (size_t)kTnRows * (p + q) * sizeof(double);
  const int J = cdiv(pq, kTnThreads);
  static char attr = 0;
  if (first_on_device(&attr)) {
    MEG_CUDA(cudaFuncSetAttribute(k_tn_partial<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    MEG_CUDA(cudaFuncSetAttribute(k_tn_partial<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    MEG_CUDA(cudaFuncSetAttribute(k_tn_partial<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    MEG_CUDA(cudaFuncSetAttribute(k_tn_partial<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    MEG_CUDA(cudaFuncSetAttribute(k_tn_partial<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  }
  if (J <= 1)
    k_tn_partial<1><<<G, kTnThreads, smem, L.stream>>>(n, X, ldx, p, Y, ldy, q, part, rows_per);
  else if (J <= 4)
    k_tn_partial<4><<<G, kTnThreads, smem, L.stream>>>(n, X, ldx, p, Y, ldy, q, part, rows_per);
  else if (J <= 8)
    k_tn_partial<8><<<G, kTnThreads, smem, L.stream>>>(n, X, ldx, p, Y, ldy, q, part, rows_per);
  else if (J <= 16)
    k_tn_partial<16><<<G, kTnThreads, smem, L.stream>>>(n, X, ldx, p, Y, ldy, q, part, rows_per);
  else if (J <= 24)
    k_tn_partial<24><<<G, kTnThreads, smem, L.stream>>>(n, X, ldx, p, Y, ldy, q, part, rows_per);
  else
    throw Error(MEGB200_ERR_PARAM, "tn: p*q too large");
  MEG_LAUNCHED();
  k_reduce_partials<<<cdiv(pq, 256), 256, 0, L.stream>>>(part, G, p, q, C, ldc, rowscale, 0);
  MEG_LAUNCHED();
  *L.counter += 2;
}

void nn(const Launch& L, int64_t n, const double* X, int64_t ldx, int p, const double* C, int64_t ldc, int q,
        double alpha, double beta, double* Y, int64_t ldy) {
  const size_t smem = (size_t)std::max(1, p * q) * sizeof(double);
  static char attr = 0;
  if (first_on_device(&attr)) {
    MEG_CUDA(cudaFuncSetAttribute(k_nn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  k_nn<<<cdiv(n * q, 256), 256, smem, L.stream>>>(n, X, ldx, p, C, ldc, q, alpha, beta, Y, ldy);
  MEG_LAUNCHED();
  ++*L.counter;
}

size_t step_mma_tail_doubles(int b, int l) {
  const size_t jac = std::max((size_t)jacobi_smem_doubles(b), (size_t)5 * b * b + 128);
  return 2 * (size_t)kStepMaxTileSlots * kMmaRows * b + (size_t)kMmaRows * std::max(l, b) +
         (size_t)std::max(l, 1) * b + 2 * (size_t)b * b + kStepThreads + jac;
}

bool dense_step_mma_supported(const void* M, int dtype, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                              int l, int64_t part_cap_slices, int sm_count) {
  // opt-in (MEGB200_STEP_MMA=1) until its tail beats the separate pass + k_fused_first_pass
  static const bool on = getenv("MEGB200_STEP_MMA") != nullptr && getenv("MEGB200_STEP_MMA")[0] == '1';
  if (!on) return false;
  if (dtype != MEGB200_F64 || b < 8 || b > 32 || b % 2 != 0 || l < 0 || l > kFusedMaxL) return false;
  if (!(ldu % 2 == 0 && ((uintptr_t)U % 16 == 0) && (ldm * 8) % 16 == 0 && ((uintptr_t)M % 16 == 0) && (n * 8) % 16 == 0))
    return false;
  const int tiles = cdiv(n, kMmaRows);
  if (tiles > kStepMaxTiles || b * b > kFusedStride || l * b > kFusedStride) return false;
  int grid = 0, smax = 0;
  stream_k_grid(n, sm_count, part_cap_slices, &grid, &smax);
  const int64_t units_per_cta = cdiv((int64_t)tiles * cdiv(n, kPipeKC), grid);
  // a CTA completes at most kStepMaxTileSlots tiles (its range spans <= 2 tiles when tiles <= grid)
  if (tiles > grid || cdiv(units_per_cta, cdiv(n, kPipeKC)) + 1 > kStepMaxTileSlots) return false;
  // the tail's shared memory stays below the operand ring (the mbarriers after it are not reused);
  // ring + the U / W segment rows fit one SM (b <= 18 with the 5-stage ring)
  if (b * b > 2 * 32 * 8) return false;  // two H entries per consumer thread
  const int bnp = ((b - 2 + 7) / 8) * 8 + 2;  // mma_bnp<b / 8, b % 8>()
  const size_t dyn = 1024 + (size_t)kPipeStages * kPipeKC * kMmaRows * 8 + 2 * (size_t)kMmaRows * b * 8 + 256 +
                     (size_t)kPipeStages * kPipeKC * bnp * 8;
  return dyn + 2048 <= 227 * 1024 &&
         step_mma_tail_doubles(b, l) * sizeof(double) <= (size_t)kPipeStages * kPipeKC * kMmaRows * 8;
}

void dense_step_mma(const Launch& L, const double* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                    double* part, int64_t part_cap_slices, int sm_count, const FusedPassArgs& a) {
  const int tiles = cdiv(n, kMmaRows);
  const int kch = cdiv(n, kPipeKC);
  int grid = 0, smax = 0;
  stream_k_grid(n, sm_count, part_cap_slices, &grid, &smax);
#define MEG_STEP(nt, tail) launch_step_mma<nt, tail>(L, M, ldm, n, U, ldu, b, part, tiles, kch, smax, grid, a)
  switch (b) {
    case 8: MEG_STEP(1, 0); break;
    case 10: MEG_STEP(1, 2); break;
    case 12: MEG_STEP(1, 4); break;
    case 14: MEG_STEP(1, 6); break;
    case 16: MEG_STEP(2, 0); break;
    case 18: MEG_STEP(2, 2); break;
    case 20: MEG_STEP(2, 4); break;
    case 22: MEG_STEP(2, 6); break;
    case 24: MEG_STEP(3, 0); break;
    case 26: MEG_STEP(3, 2); break;
    case 28: MEG_STEP(3, 4); break;
    case 30: MEG_STEP(3, 6); break;
    default: MEG_STEP(4, 0); break;
  }
#undef MEG_STEP
}

void tile_gram(const Launch& L, int64_t n, const double* Lm, int64_t ldl, int l, const double* U, int64_t ldu, int b,
               int nvg, double* part, unsigned* ticket, double* E, double* vgram, double* Gu) {
  const size_t smem = (size_t)kMmaRows * (l + b) * sizeof(double);
  static char attr = 0;
  if (first_on_device(&attr))
    MEG_CUDA(cudaFuncSetAttribute(k_tile_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  k_tile_gram<<<cdiv(n, kMmaRows), 256, smem, L.stream>>>(n, Lm, ldl, l, U, ldu, b, nvg, part, ticket, E, vgram, Gu);
  MEG_LAUNCHED();
  ++*L.counter;
}

void copy_block(const Launch& L, int64_t n, int q, const double* src, int64_t lds, double* dst, int64_t ldd) {
  if (n * q == 0) return;
  k_copy_block<<<cdiv(n * q, 256), 256, 0, L.stream>>>(n, q, src, lds, dst, ldd);
  MEG_LAUNCHED();
  ++*L.counter;
}

void fill_gaussian(const Launch& L, int64_t n, int q, uint64_t key, uint64_t base, double scale, bool round_f32,
                   double* dst, int64_t ldd) {
  if (n * q == 0) return;
  k_fill_gaussian<<<cdiv(n * q, 256), 256, 0, L.stream>>>(n, q, key, base, scale, round_f32 ? 1 : 0, dst, ldd);
  MEG_LAUNCHED();
  ++*L.counter;
}

void csr_values(const Launch& L, int64_t n, const int32_t* rowptr, const int32_t* col, const double* obs,
                const double* V, int64_t ldv, int r, const double* coeff, double tail, double* g, double* sq_rows,
                int) {
  k_csr_values<<<cdiv(n, 8), 256, 0, L.stream>>>(n, rowptr, col, obs, V, ldv, r, coeff, tail, g, sq_rows);
  MEG_LAUNCHED();
  ++*L.counter;
}

void dense_stats(const Launch& L, const void* M, int dtype, int64_t ld, int64_t n, double* part, int slots) {
  if (dtype == MEGB200_F64)
    k_dense_stats<double><<<slots, 256, 0, L.stream>>>(static_cast<const double*>(M), ld, n, part);
  else
    k_dense_stats<float><<<slots, 256, 0, L.stream>>>(static_cast<const float*>(M), ld, n, part);
  MEG_LAUNCHED();
  ++*L.counter;
}

void frob_direct(const Launch& L, const void* M, int dtype, int64_t ld, int64_t n, const double* V, int64_t ldv, int r,
                 const double* coeff, double tail, double* part, int slots) {
  if (dtype == MEGB200_F64)
    k_frob_direct<double, 8><<<slots, 256, 0, L.stream>>>(static_cast<const double*>(M), ld, n, V, ldv, r, coeff, tail,
                                                           part);
  else
    k_frob_direct<float, 8><<<slots, 256, 0, L.stream>>>(static_cast<const float*>(M), ld, n, V, ldv, r, coeff, tail,
                                                          part);
  MEG_LAUNCHED();
  ++*L.counter;
}

void sampled_count(const Launch& L, int64_t n, uint64_t kmask, double p, int32_t* counts) {
  k_sampled_count<<<cdiv(n * 32, 256), 256, 0, L.stream>>>(n, kmask, p, counts);
  MEG_LAUNCHED();
  ++*L.counter;
}

void sampled_fill(const Launch& L, int64_t n, uint64_t kmask, uint64_t knoise, double p, const double* U, int r,
                  const double* lam, double obs_noise, const int32_t* rowptr, int32_t* col, double* val) {
  k_sampled_fill<<<cdiv(n * 32, 256), 256, 0, L.stream>>>(n, kmask, knoise, p, U, r, lam, obs_noise, rowptr, col, val);
  MEG_LAUNCHED();
  ++*L.counter;
}

void gen_dense_target(const Launch& L, const double* U, int64_t r, const double* lam, double sigma, uint64_t key,
                      void* M, int dtype, int64_t ld, int64_t n) {
  dim3 grid(cdiv(n, 256), (unsigned)n);
  if (dtype == MEGB200_F64)
    k_gen_dense_target<double><<<grid, 256, 0, L.stream>>>(U, (int)r, lam, sigma, key, static_cast<double*>(M), ld, n);
  else
    k_gen_dense_target<float><<<grid, 256, 0, L.stream>>>(U, (int)r, lam, sigma, key, static_cast<float*>(M), ld, n);
  MEG_LAUNCHED();
  ++*L.counter;
}

void set_identity(const Launch& L, int64_t n, double* Q, int64_t ldq) {
  k_set_identity<<<cdiv(n * n, 256), 256, 0, L.stream>>>(n, Q, ldq);
  MEG_LAUNCHED();
  ++*L.counter;
}

void set_diag(const Launch& L, double* H, int cap, int k, const double* theta) {
  k_set_diag<<<cdiv((int64_t)cap * cap, 256), 256, 0, L.stream>>>(H, cap, k, theta);
  MEG_LAUNCHED();
  ++*L.counter;
}

void form_operator(const Launch& L, int64_t n, const double* M, int64_t ldm, double scale, const double* Lf, int64_t ldl,
                   int l, const double* d, LamCoef lc, double alpha, double* AQ, int64_t ldq, double* H, int64_t ldh) {
  if (l > kFormMaxLowrank) throw Error(MEGB200_ERR_PARAM, "form_operator: low-rank width out of range");
  k_form_operator<<<(unsigned)n, 128, 0, L.stream>>>(n, M, ldm, scale, Lf, ldl, l, d, lc, alpha, AQ, ldq, H, ldh);
  MEG_LAUNCHED();
  ++*L.counter;
}

void restart_basis(const Launch& L, int64_t n, double* Q, double* AQ, int64_t ldq, const double* S, int m, int keep,
                   int tq, int sm_count) {
  const size_t smem = ((size_t)m * keep + 2 * (size_t)kRestartRows * (m + tq)) * sizeof(double);
  if (keep + tq > m || smem > 200 * 1024) throw Error(MEGB200_ERR_PARAM, "restart_basis: shape out of range");
  static char attr = 0;
  if (first_on_device(&attr))
    MEG_CUDA(cudaFuncSetAttribute(k_restart_basis, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count, cdiv(n, kRestartRows)));
  k_restart_basis<<<grid, 256, smem, L.stream>>>(n, Q, AQ, ldq, S, m, keep, tq);
  MEG_LAUNCHED();
  ++*L.counter;
}

void restart_h(const Launch& L, double* H, int cap, const double* S, int m, int keep, int q, const double* theta) {
  const size_t smem = ((size_t)(m + q) * q + (size_t)m * keep) * sizeof(double);
  if (keep + q > m || m + q > cap || smem > 160 * 1024) throw Error(MEGB200_ERR_PARAM, "restart_h: shape out of range");
  static char attr = 0;
  if (first_on_device(&attr))
    MEG_CUDA(cudaFuncSetAttribute(k_restart_h, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  k_restart_h<<<1, 1024, smem, L.stream>>>(H, cap, S, m, keep, q, theta);
  MEG_LAUNCHED();
  ++*L.counter;
}

void reduce_sum(const Launch& L, const double* part, int slots, int width, double* out) {
  k_reduce_sum<<<1, 64, 0, L.stream>>>(part, slots, width, out);
  MEG_LAUNCHED();
  ++*L.counter;
}

}  // namespace megb200

// Diagnostics: per-CTA phase timestamps of the last float64 DMMA pass (MEGB200_PASS_STAMPS=1)
extern "C" int megb200_debug_pass_ns(unsigned long long* out, int count) {
  if (!out || count < 1 || count > 160 * 8) return MEGB200_ERR_PARAM;
  return cudaMemcpyFromSymbol(out, megb200::g_pass_ns, sizeof(unsigned long long) * count) == cudaSuccess
             ? MEGB200_OK
             : MEGB200_ERR_CUDA;
}
