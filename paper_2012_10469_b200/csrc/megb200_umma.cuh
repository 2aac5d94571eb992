// K1 (float32 operands): streamed operand pass on the 5th-generation tensor
// cores.  W_s[i, c] = sum_{k in segment s} M[k, i] U[k, c] for a 128-row tile
// of i, with M float32 (cfg 4/5) and U float64, computed as split TF32
// TF32: M = Mh + Ml, U = Uh + Ul with Mh, Uh rounded to TF32, and
//   W = Mh Uh + Mh Ul + Ml Uh + Ml Ul
// accumulated in float32 in tensor memory over sub-segments of kSub k chunks,
// each drained into float64 registers (so the float32 accumulation error does
// not grow with n).
//
// Roles (192 threads): warps 0-3 (thread t = tile row t) read row t of each
// landed M tile, split it into Mh / Ml in registers and store both into a
// tensor-memory operand buffer (tcgen05.st: lane t, one column per k), and drain
// the accumulators (tcgen05.ld -> float64 partial rows); warp 4 lane 0 is the
// TMA producer; warp 5 lane 0 issues tcgen05.mma (kind::tf32, M=128, N=64,
// K=8, A from tensor memory, B = [Uh | Ul]^T K-major 128-byte-swizzled in shared
// memory) and commits stage / operand-buffer releases and accumulator-ready
// to mbarriers.  Keeping the split operand out of shared memory leaves shared
// memory to the TMA stream and the small U tile.
// K-major A is M's rows i with k contiguous -- the symmetry of M (M[k][i] =
// M[i][k]) makes the tile a plain 128 x 32 box of M; K-major B is the
// transposed split copy of U (Uh^T, Ul^T: 32 x n, k contiguous).
// Work split: stream-K over (row tile, 32-row k chunk), identical to the DMMA
// pass (megb200_kernels.cu), so the partial-slot contract is the same.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace megb200 {
namespace umma {

constexpr int kKC = 32;      // k rows per stage (4 MMA k-steps of 8)
constexpr int kStages = 8;   // ring depth
constexpr int kRows = 128;   // UMMA M: tile rows (i)
constexpr int kN = 32;       // U columns per half (zero-padded to 32)
constexpr int kNM = 2 * kN;  // UMMA N: [Uh | Ul] side by side
constexpr int kThreads = 192;
constexpr int kSplitWarps = 4;
constexpr int kABytes = kRows * kKC * 4;              // 16 KiB: 128 rows i x 32 k (one TMA box)
constexpr int kBBytes = kNM * kKC * 4;                // 8 KiB: [Uh | Ul]^T, 64 rows x 32 k
constexpr int kStageBytes = kABytes + kBBytes;  // M tile | [Uh | Ul]^T tile (TMA-landed)
constexpr int kTmaBytes = kABytes + kBBytes;
constexpr int kABufs = 6;                        // split-operand buffers in tensor memory (columns 0..383)
constexpr int kABufCols = 2 * kKC;               // Mh (32 columns) | Ml (32 columns)
constexpr int kAccCol = 384;                     // accumulators: columns 384 + 64 a
constexpr int kTmemCols = 512;
constexpr int kSub = 8;  // k chunks (256 k) per float32 accumulator before it is drained into float64

__host__ __device__ constexpr size_t smem_bytes() { return 1024 + (size_t)kStages * kStageBytes + 512; }

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  uint64_t st;
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(saddr(b)) : "memory");
  (void)st;
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  uint64_t st;
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 %0, [%1], %2;"
               : "=l"(st) : "r"(saddr(b)), "r"(bytes) : "memory");
  (void)st;
}
// bounded wait: a protocol bug traps (launch error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t it = 0; !done; ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(saddr(b)), "r"(parity) : "memory");
    if (it > (1u << 28)) __trap();
  }
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(saddr(dst)), "l"(map), "r"(x), "r"(y), "r"(saddr(b)), "l"(pol) : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B canonical layout: rows of
// 128 B (32 tf32 along K), 8-row swizzle atoms 1024 B apart (SBO); a K=8 step
// advances the start address by 32 B inside the row.  Version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(16 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D f32, A/B tf32, both K-major, N = kNM, M = kRows
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kNM >> 3) << 17) |
                            ((uint32_t)(kRows >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((uint64_t)saddr(b)) : "memory");
}

// Stream-K range of this CTA and the first CTA on a tile (same arithmetic as the DMMA pass)
__device__ __forceinline__ int first_cta(int64_t x, int64_t utot) {
  return (int)(((x + 1) * gridDim.x + utot - 1) / utot) - 1;
}

#ifdef UMMA_PROFILE
__device__ long long g_uprof[8];
#endif

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

// A operand from tensor memory: D[tmem] (+)= A[tmem] . B[smem desc]
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(b), "r"(kIdesc), "r"(accumulate) : "memory");
}

#define MEG_R32(r)                                                                                          \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), \
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), \
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),  \
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])

// 32 consecutive columns of this warp's 32 TMEM lanes <- r[0..31] (thread = lane)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr), MEG_R32(r) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    k_dense_pass_umma(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmU,
                      int64_t n, int b, double* __restrict__ part, int tiles, int kch, int smax) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - ((uintptr_t)smem_raw & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)kStages * kStageBytes);
  uint64_t* full = bars;                  // [kStages] TMA landed (1 arrival + tx)
  uint64_t* split = full + kStages;       // [kStages] operand buffer written (128 arrivals)
  uint64_t* empty = split + kStages;      // [kStages] stage's MMAs done (tcgen05.commit)
  uint64_t* abuf_free = empty + kStages;  // [kABufs] operand buffer's MMAs done (tcgen05.commit)
  uint64_t* acc_full = abuf_free + kABufs;  // [2] accumulator complete (tcgen05.commit)
  uint64_t* acc_empty = acc_full + 2;       // [2] accumulator read out (128 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(split + s, 32 * kSplitWarps);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < kABufs; ++a) mbar_init(abuf_free + a, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + a, 1);
      mbar_init(acc_empty + a, 32 * kSplitWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmM) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmU) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                 "n"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int64_t utot = (int64_t)tiles * kch;
  const int64_t ua = (int64_t)blockIdx.x * utot / gridDim.x, ub = (int64_t)(blockIdx.x + 1) * utot / gridDim.x;

  if (warp == kSplitWarps) {
    // ---------------- TMA producer
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      uint64_t keep;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
      int st = 0;
      uint32_t ph = 0;
      for (int64_t u = ua; u < ub; ++u) {
        const int tile = (int)(u / kch);
        const int kc = (int)((u - (int64_t)tile * kch) * kKC);
        mbar_wait(empty + st, ph ^ 1u);
        mbar_arrive_tx(full + st, kTmaBytes);
        unsigned char* sb = base + (size_t)st * kStageBytes;
        tma_2d(sb, &tmM, kc, tile * kRows, full + st, pol);  // rows i of M, k contiguous (M symmetric)
        tma_2d(sb + kABytes, &tmU, kc, 0, full + st, keep);
        if (++st == kStages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == kSplitWarps + 1) {
    // ---------------- MMA issuer: one accumulator per sub-segment of <= kSub chunks.  The
    // whole warp runs the loop (warp-uniform control flow keeps descriptors and TMEM
    // addresses in uniform registers) and one elected lane issues: small MMAs are
    // issue-bound, so descriptors advance by adding to the start-address field.
    {
      int st = 0;
      uint32_t ph = 0;
      int abuf = 0;
      int g = 0;
      const uint64_t bdesc0 = sdesc(saddr(base + kABytes));
      for (int64_t u = ua; u < ub; ++g) {
        const int tile = (int)(u / kch);
        const int64_t uend = min(min(ub, (int64_t)(tile + 1) * kch), u + kSub);
        const int ab = g & 1;
        // the drain must have emptied this accumulator (used two sub-segments ago)
        if (g >= 2) mbar_wait(acc_empty + ab, ((g >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(kAccCol + ab * kNM);
        uint32_t acc0 = 0u;
        for (; u < uend; ++u) {
#ifdef UMMA_PROFILE
          long long m0 = clock64();
#endif
          mbar_wait(split + st, ph);  // operand buffer written (implies the stage landed)
#ifdef UMMA_PROFILE
          if (blockIdx.x == 0 && lane == 0) g_uprof[5] += clock64() - m0;
#endif
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t ah = tmem + (uint32_t)(abuf * kABufCols), al = ah + kKC;
          const uint64_t bd = bdesc0 + (uint64_t)((st * kStageBytes) >> 4);
          if (elect_one()) {
            // D[:, 0:32] += Mh Uh + Ml Uh,  D[:, 32:64] += Mh Ul + Ml Ul
            mma_tf32_ta(d, ah, bd, acc0);
            mma_tf32_ta(d, al, bd, 1u);
            mma_tf32_ta(d, ah + 8, bd + 2, 1u);
            mma_tf32_ta(d, al + 8, bd + 2, 1u);
            mma_tf32_ta(d, ah + 16, bd + 4, 1u);
            mma_tf32_ta(d, al + 16, bd + 4, 1u);
            mma_tf32_ta(d, ah + 24, bd + 6, 1u);
            mma_tf32_ta(d, al + 24, bd + 6, 1u);
            mma_commit(empty + st);        // shared-memory stage free once these MMAs have read U
            mma_commit(abuf_free + abuf);  // operand buffer free likewise
          }
          __syncwarp();
          acc0 = 1u;
          if (++abuf == kABufs) abuf = 0;
          if (++st == kStages) {
            st = 0;
            ph ^= 1u;
          }
        }
        if (elect_one()) mma_commit(acc_full + ab);  // accumulator complete
        __syncwarp();
      }
    }
  } else {
    // ---------------- split warps (0-3): row t of each tile -> Mh, Ml in tensor memory; drains
    int st = 0;
    uint32_t ph = 0;
    int abuf = 0;          // operand buffer of the next stage
    uint32_t aph = 0;      // its use parity
    bool awrapped = false;  // every buffer used once already
    int g = 0;
    const int t = threadIdx.x;  // 0..127: tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    double acc[kN];
    auto drain = [&](int gd) {
      const int ab = gd & 1;
#ifdef UMMA_PROFILE
      long long d0 = clock64();
#endif
      mbar_wait(acc_full + ab, (gd >> 1) & 1);
#ifdef UMMA_PROFILE
      if (blockIdx.x == 0 && threadIdx.x == 0) { g_uprof[6] += clock64() - d0; g_uprof[7] += 1; }
#endif
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + lane_base + (uint32_t)(kAccCol + ab * kNM);
      uint32_t r[32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr + (uint32_t)(half * kN)));
        // the loaded registers are valid only after wait::ld: tie them to it so no use is hoisted above
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                       "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                       "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                       "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                       "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                     :
                     : "memory");
#pragma unroll
        for (int c = 0; c < kN; ++c) acc[c] += (double)__uint_as_float(r[c]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(acc_empty + ab);
    };
    for (int64_t u = ua; u < ub;) {
      const int tile = (int)(u / kch);
      const int64_t send = min(ub, (int64_t)(tile + 1) * kch);
      const bool closes = send == (int64_t)(tile + 1) * kch;
      const int slot = (int)blockIdx.x - first_cta((int64_t)tile * kch, utot);
#pragma unroll
      for (int c = 0; c < kN; ++c) acc[c] = 0.0;
      int pending = -1;  // sub-segment of this tile split but not yet drained
      while (u < send) {
        const int64_t uend = min(send, u + kSub);
        for (; u < uend; ++u) {
#ifdef UMMA_PROFILE
          long long c0 = clock64();
#endif
          if (awrapped) mbar_wait(abuf_free + abuf, aph ^ 1u);  // the MMAs of this buffer's last use are done
#ifdef UMMA_PROFILE
          long long c1 = clock64();
#endif
          mbar_wait(full + st, ph);
#ifdef UMMA_PROFILE
          long long c2 = clock64();
#endif
          // row t (128 B, 128-byte swizzle: chunk j at (j ^ (t & 7)) * 16) -> Mh rounded to TF32, Ml = M - Mh
          const unsigned char* row = base + (size_t)st * kStageBytes + t * 128;
          uint32_t h[32], l[32];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 x = *reinterpret_cast<const float4*>(row + ((j ^ (t & 7)) << 4));
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t hb = (__float_as_uint(xs[e]) + 0x1000u) & 0xFFFFE000u;
              h[4 * j + e] = hb;
              l[4 * j + e] = __float_as_uint(xs[e] - __uint_as_float(hb));
            }
          }
          const uint32_t ta = tmem + lane_base + (uint32_t)(abuf * kABufCols);
#ifdef UMMA_PROFILE
          long long c3 = clock64();
#endif
          tmem_st32(ta, h);
          tmem_st32(ta + kKC, l);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(split + st);
          if (++abuf == kABufs) {
            abuf = 0;
            aph ^= 1u;
            awrapped = true;
          }
#ifdef UMMA_PROFILE
          long long c4 = clock64();
          if (blockIdx.x == 0 && t == 0) {
            g_uprof[0] += c1 - c0;
            g_uprof[1] += c2 - c1;
            g_uprof[2] += c3 - c2;
            g_uprof[3] += c4 - c3;
            g_uprof[4] += 1;
          }
#endif
          if (++st == kStages) {
            st = 0;
            ph ^= 1u;
          }
        }
        // the previous sub-segment's accumulator drains while the MMAs of this one run
        if (pending >= 0) drain(pending);
        pending = g++;
      }
      drain(pending);
      const int64_t row = (int64_t)tile * kRows + t;
      if (row < n) {
        double* out = part + (int64_t)slot * n * b + row * b;
#pragma unroll
        for (int c = 0; c < kN; ++c)
          if (c < b) out[c] = acc[c];
        if (closes)
          for (int sl = slot + 1; sl < smax; ++sl) {
            double* z = part + (int64_t)sl * n * b + row * b;
            for (int c = 0; c < b; ++c) z[c] = 0.0;
          }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
  }
}

// U (float64, n x b, ld) -> [Uh | Ul]^T (float32, 64 x ldt, k contiguous; rows c < 32 hold Uh^T,
// rows 32 + c hold Ul^T; columns >= b zero): Uh = U rounded to TF32, Ul = float32(U - Uh), so
// Uh + Ul carries U to ~2^-24 relative.  32 x 32 tiles transposed through shared memory.
__global__ void __launch_bounds__(256) k_split_u(int64_t n, int b, const double* __restrict__ U, int64_t ldu,
                                                 float* __restrict__ UT, int64_t ldt) {
  __shared__ float th[32][33], tl[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t k = k0 + r;
    float h = 0.f, l = 0.f;
    if (k < n && tx < b) {
      const double x = U[k * ldu + tx];
      h = __uint_as_float((__float_as_uint((float)x) + 0x1000u) & 0xFFFFE000u);
      l = (float)(x - (double)h);
    }
    th[r][tx] = h;
    tl[r][tx] = l;
  }
  __syncthreads();
  for (int c = ty; c < 32; c += 8) {
    const int64_t k = k0 + tx;
    if (k < ldt) {
      UT[c * ldt + k] = th[tx][c];
      UT[(32 + c) * ldt + k] = tl[tx][c];
    }
  }
}

}  // namespace umma
}  // namespace megb200
