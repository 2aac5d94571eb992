// First-pass finish + Rayleigh-Ritz + Ritz block + residuals + step epilogue
// in ONE launch (the steady-state MEG step is: operand pass, this kernel).
//
// Replaces, for the first pass of a solve (block of bw <= 32 columns), the pair
// k_coop_finish + k_coop_rr and their three grid barriers.  G <= #SMs CTAs of
// 256 threads each own a contiguous row range, staged once in shared memory;
// the cross-CTA steps use "last CTA" tickets instead of grid barriers: every
// CTA writes its partial, the CTA that arrives last reduces all partials in a
// FIXED CTA order (warp xor-trees: bitwise reproducible whichever CTA is last),
// runs the serial part and publishes it with a release flag the others spin on
// (all CTAs are co-resident: G <= #SMs, one CTA per SM at most).
//
//   phase 0  (only without a precomputed L^T U)  E = diag(d) L^T U
//   phase 1  W = scale * sum_s part[s] + L E + alpha U   (rows, -> AQ)
//            H = U^T W (upper triangle) -> last CTA: Jacobi Rayleigh-Ritz
//            (linalg.py:205-211) + step epilogue (meg.py:347-356)
//   phase 2  T = U S (Ritz block, V_next), residuals ||W s_j - theta_j T_j||
//            (linalg.py:212-216), Gram of T -> last CTA: reduce, write the
//            result pack to device memory and to the caller's pinned host slot.
//
// The phase-0 partial of L^T U and the phase-2 Gram partial use the same
// per-row fma order and the same cross-CTA tree, so a pipelined step that takes
// E from the previous step's Ritz-block Gram is bit-identical to one that
// reduces L^T U again (L = V_next = first r Ritz vectors, U = the Ritz block).

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "megb200_internal.h"

namespace cg = cooperative_groups;

#define JACOBI_MARK(slot)
#include "megb200_jacobi.cuh"
#include "megb200_tail.cuh"

namespace megb200 {
namespace {


// sum_{j < cnt} part[(g0 + j) * stride + o] in index order by ONE thread: the loads are
// issued eight at a time before they are added, neighbouring threads take neighbouring o
__device__ __forceinline__ double ordered_sum(const double* part, int g0, int cnt, int64_t stride, int o) {
  double s = 0.0;
  for (int j0 = 0; j0 < cnt; j0 += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = j0 + j < cnt ? __ldcg(part + (int64_t)(g0 + j0 + j) * stride + o) : 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  return s;
}

// Every thread's partial-sum stores are fenced, then one atomic ticket per CTA;
// returns true (in all threads) in the CTA that arrived last of `expected`, which
// re-arms the ticket.
__device__ __forceinline__ bool arrive_last(unsigned* ticket, unsigned expected, int* s_flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    const bool last = (t == expected - 1);
    if (last) atomicExch(ticket, 0u);
    *s_flag = last;
  }
  __syncthreads();
  const bool last = *s_flag != 0;
  if (last) __threadfence();
  return last;
}

// Two-level fixed-order reduction of the per-CTA partials part[g * stride + o], o < count:
// groups of kGroup consecutive CTAs (the last CTA of a group sums its group in CTA order
// into gpart), then the last group finisher sums the group partials in group order into
// res.  Returns true in the one CTA that wrote res (whichever CTAs arrive last, the
// association -- hence every bit of res -- is the same).  tick: 1 + #groups tickets.
constexpr int kGroup = 8;
template <int NT, bool CL>
__device__ __forceinline__ bool tree_reduce(const double* part, double* gpart, double* res, int count,
                                            int64_t stride, unsigned* tick, int* s_flag) {
  const int G = gridDim.x, NG = (G + kGroup - 1) / kGroup, grp = blockIdx.x / kGroup;
  const int g0 = grp * kGroup, gn = min(kGroup, G - g0);
  if constexpr (CL) {
    // launched as clusters of kGroup CTAs (cluster = group): the hardware cluster barrier
    // (release / acquire at cluster scope) replaces the group ticket; rank 0 sums the group
    __threadfence_block();
    cg::this_cluster().sync();
    if (cg::this_cluster().block_rank() != 0) return false;
  } else {
    if (!arrive_last(tick + 1 + grp, (unsigned)gn, s_flag)) return false;
  }
  for (int o = threadIdx.x; o < count; o += NT) gpart[grp * stride + o] = ordered_sum(part, g0, gn, stride, o);
  if (!arrive_last(tick, (unsigned)NG, s_flag)) return false;
  for (int o = threadIdx.x; o < count; o += NT) res[o] = ordered_sum(gpart, 0, NG, stride, o);
  __threadfence_block();
  __syncthreads();
  return true;
}

__device__ __forceinline__ void publish(unsigned* flag, unsigned epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release_u32(flag, epoch);
}

__device__ __forceinline__ void wait_published(const unsigned* flag, unsigned epoch) {
  if (threadIdx.x == 0)
    while (ld_acquire_u32(flag) != epoch) __nanosleep(40);  // back off: keep the flag's L2 line quiet
  __syncthreads();
}

// acc = sum over the CTA's rows of X[r, a] * Y[r, c]: even and odd rows in two chains,
// added at the end (shared by the L^T U partial and the Gram partial: same products,
// same order)
__device__ __forceinline__ double rows_dot(const double* X, int ldx, int a, const double* Y, int ldy, int c,
                                           int rows) {
  return tile_dot(X, ldx, a, Y, ldy, c, rows);  // four chains (rows mod 4): megb200_tail.cuh
}

// diagnostics: %globaltimer at phase boundaries (a.stamps, MEGB200_FUSED_STAMPS=1)
__device__ __forceinline__ void stamp(unsigned long long* st, int slot) {
  if (st && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    st[slot] = v;
  }
}

// dst[r * w + c] = src[(r0 + r) * ld + c] for r < rows, c < w: eight independent loads in
// flight per thread before the shared-memory stores
template <int NT>
__device__ __forceinline__ void stage_rows(double* dst, const double* __restrict__ src, int64_t ld, int64_t r0,
                                           int rows, int w) {
  const int total = rows * w;
  for (int base = threadIdx.x; base < total; base += 8 * NT) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = base + j * NT;
      const int r = idx / w, c = idx - r * w;
      v[j] = idx < total ? src[(r0 + r) * ld + c] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = base + j * NT;
      if (idx < total) dst[idx] = v[j];
    }
  }
}

template <int NT, bool CL>
__global__ void __launch_bounds__(NT, 1) k_fused_first_pass(const FusedPassArgs a) {
  // programmatic dependent launch after the operand pass: nothing is read before it completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.prev_epoch && a.done_flag) {
    // the previous launch's last CTA may still be reducing into the buffers reused below
    if (threadIdx.x == 0)
      while (ld_acquire_u32(a.done_flag) != a.prev_epoch) __nanosleep(32);
    __syncthreads();
  }
  unsigned long long* st0 = blockIdx.x == 0 ? a.stamps : nullptr;
  stamp(st0, 0);
  extern __shared__ __align__(16) double sm[];
  __shared__ double dsh[kFusedMaxL];
  __shared__ double thsh[64];
  __shared__ int s_flag;
  const int t = threadIdx.x, g = blockIdx.x, G = gridDim.x;
  const int b = a.b, l = a.l, rq = a.rq, R = a.R;
  const int64_t r0 = min(a.n, (int64_t)g * R);
  const int rows = (int)(min(a.n, r0 + (int64_t)R) - r0);
  double* Us = sm;            // R x b
  double* Ws = Us + R * b;    // R x b
  double* Ss = Ws + R * b;    // b x rq
  double* red = Ss + b * rq;  // NT
  double* Hs = red + NT;     // b x b: the reduced H (last CTA of phase 1)
  double* Ls = Hs + b * b;    // R x l      } phases 0-1 (L rows staged unless shared memory is short,
  const bool stL = a.stage_l;  //           } then read from global: cfg5-sized row ranges)
  double* Es = stL ? Ls + R * l : Ls;  // l x b
  const double* Lb = stL ? Ls : a.L + r0 * a.ldl;
  const int ldL = stL ? l : (int)a.ldl;
  double* jac = Es + l * b;   // Jacobi scratch (the last CTA of phase 1)
  double* Ts = Ls;            // R x rq: phase 2 (reuses the phase 0-1 region)

  // log-map coefficients: from the device-resident kept weights (lc) or as given
  for (int k = t; k < l; k += NT) {
    double v;
    if (a.lc.lam && k < a.lc.lr) {
      const double kept = a.lc.c1 * (a.lam_inline_n > 0 ? a.lam_inline[k] : a.lc.lam[k]);
      v = (log(kept) - a.lc.log_tail) + (-a.lc.eta * (kept - a.lc.tail_g));
    } else {
      v = a.d[k];
    }
    dsh[k] = v;
  }
  stage_rows<NT>(Us, a.U, a.ldu, r0, rows, b);
  if (l > 0 && stL) stage_rows<NT>(Ls, a.L, a.ldl, r0, rows, l);
  __syncthreads();
  stamp(st0, 1);

  // ---- phase 0: E = diag(d) L^T U
  if (l > 0) {
    if (a.Eg) {
      for (int idx = t; idx < l * b; idx += NT) {
        const int k = idx / b, c = idx - k * b;
        Es[idx] = dsh[k] * a.Eg[k * a.ldg + c];
      }
    } else {
      double* p0 = a.part0 + (int64_t)g * kFusedStride;
      for (int o = t; o < l * b; o += NT) {
        const int k = o / b, c = o - k * b;
        p0[o] = rows_dot(Lb, ldL, k, Us, b, c, rows);
      }
      // optional: the Gram of the first nvg factor columns (LowRankIterate validation, meg.py:69-71)
      const int nvg = a.vgram ? a.nvg : 0;
      for (int o = t; o < nvg * nvg; o += NT) {
        const int k = o / nvg, c = o - k * nvg;
        p0[l * b + o] = rows_dot(Lb, ldL, k, Lb, ldL, c, rows);
      }
      if (tree_reduce<NT, CL>(a.part0, a.part0 + (int64_t)G * kFusedStride, a.Ews, l * b + nvg * nvg, kFusedStride,
                              a.sync, &s_flag)) {
        for (int o = t; o < nvg * nvg; o += NT) a.vgram[o] = a.Ews[l * b + o];
        publish(a.sync + kFusedFlags, a.epoch);
      } else {
        wait_published(a.sync + kFusedFlags, a.epoch);
      }
      for (int idx = t; idx < l * b; idx += NT) Es[idx] = dsh[idx / b] * __ldcg(a.Ews + idx);
    }
  }
  __syncthreads();

  stamp(st0, 2);
  // ---- phase 1: W rows, H = U^T W
  {
    const int64_t slice = a.n * b;
    const int nw = rows * b;
    // four W elements per thread per round (large row ranges, e.g. cfg5's 256 rows): the first
    // eight slices of all four in flight together; per element the same slice-ordered sum and
    // the same two-chain L E product as one element at a time
    for (int base = t; base < nw; base += 4 * NT) {
      double pv[4][8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = base + q * NT;
        const bool ok = idx < nw;
        const double* pp = a.part + r0 * b + (ok ? idx : 0);
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) pv[q][tt] = (ok && tt < a.S) ? pp[tt * slice] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = base + q * NT;
        if (idx >= nw) break;
        const int rr = idx / b, c = idx - rr * b;
        const int64_t i = r0 + rr;
        const double* pp = a.part + i * b + c;
        double s = 0.0;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) s += pv[q][tt];
#pragma unroll
        for (int tt = 8; tt < 16; ++tt) s += tt < a.S ? pp[tt * slice] : 0.0;
        for (int tt = 16; tt < a.S; ++tt) s += pp[tt * slice];
        const double* Lr = Lb + rr * ldL;
        double v0 = a.scale * s + a.alpha * Us[idx], v1 = 0.0;
        int k = 0;
        for (; k + 1 < l; k += 2) {
          v0 = fma(Lr[k], Es[k * b + c], v0);
          v1 = fma(Lr[k + 1], Es[(k + 1) * b + c], v1);
        }
        if (k < l) v0 = fma(Lr[k], Es[k * b + c], v0);
        const double wv = v0 + v1;
        Ws[idx] = wv;
        a.W[i * a.ldw + c] = wv;
      }
    }
    __syncthreads();
    stamp(st0, 15);
    double* p1 = a.part1 + (int64_t)g * kFusedStride;
    for (int o = t; o < b * b; o += NT) {
      const int ia = o / b, c = o - ia * b;
      p1[o] = ia <= c ? rows_dot(Us, b, ia, Ws, b, c, rows) : 0.0;
    }
  }
  stamp(st0, 3);
  bool rr_cta = false;  // this CTA solved the Rayleigh-Ritz problem (its H write and epilogue are deferred)
  if (tree_reduce<NT, CL>(a.part1, a.part1 + (int64_t)G * kFusedStride, Hs, b * b, kFusedStride, a.sync + 32, &s_flag)) {
    stamp(a.stamps, 4);
    stamp(a.stamps, 5);
    if (!rr_small_neardiag<NT>(Hs, b, b, a.theta, a.Sout, jac, thsh, a.info)) {
      __syncthreads();
      jacobi_fallback(Hs, b, a.theta, a.Sout, jac, a.info);
      __syncthreads();
      for (int c = t; c < b; c += NT) thsh[c] = a.theta[c];
      __syncthreads();
    }
    stamp(a.stamps, 6);
    // the other CTAs need theta and S only; H (for a continued solve) and the step epilogue are
    // written after this CTA's own Ritz rows are out (rr_cta below): the next operand pass waits for
    // the Ritz rows of ALL CTAs, so anything this CTA does before them delays it
    publish(a.sync + kFusedFlags + 1, a.epoch);
    rr_cta = true;
    stamp(a.stamps, 7);
  } else {
    wait_published(a.sync + kFusedFlags + 1, a.epoch);
  }
  stamp(st0, 8);

  // ---- phase 2: Ritz block, residuals, Gram
  for (int idx = t; idx < b * rq; idx += NT) {
    const int k = idx / rq, c = idx - k * rq;
    Ss[idx] = __ldcg(a.Sout + k * b + c);
  }
  for (int c = t; c < rq; c += NT) thsh[c] = __ldcg(a.theta + c);
  __syncthreads();
  stamp(st0, 13);
  const int rpt = NT / rq;
  const int c = t % rq;
  const int rofs = t / rq;
  double sq = 0.0;
  if (rofs < rpt) {
    const double th = c < a.nreq ? thsh[c] : 0.0;
    const bool res = c < a.nreq;
    // four rows per round (independent chains; the S entry is loaded once for the four), each
    // row's products in the same two-chain order as one row at a time; residual squares in row order
    for (int rb = rofs; rb < rows; rb += 4 * rpt) {
      double x0[4], x1[4], y0[4], y1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) x0[q] = x1[q] = y0[q] = y1[q] = 0.0;
      int k = 0;
      for (; k + 1 < b; k += 2) {
        const double s0 = Ss[k * rq + c], s1 = Ss[(k + 1) * rq + c];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = min(rb + q * rpt, rows - 1);
          x0[q] = fma(Us[rr * b + k], s0, x0[q]);
          x1[q] = fma(Us[rr * b + k + 1], s1, x1[q]);
          if (res) {
            y0[q] = fma(Ws[rr * b + k], s0, y0[q]);
            y1[q] = fma(Ws[rr * b + k + 1], s1, y1[q]);
          }
        }
      }
      if (k < b) {
        const double s0 = Ss[k * rq + c];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rr = min(rb + q * rpt, rows - 1);
          x0[q] = fma(Us[rr * b + k], s0, x0[q]);
          if (res) y0[q] = fma(Ws[rr * b + k], s0, y0[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = rb + q * rpt;
        if (rr < rows) {
          const double x = x0[q] + x1[q];
          const int64_t i = r0 + rr;
          a.T[i * a.ldt + c] = x;
          Ts[rr * rq + c] = x;
          if (c < a.r2) a.V2[i * a.ld2 + c] = x;
          if (res) {
            const double d = (y0[q] + y1[q]) - th * x;
            sq = fma(d, d, sq);
          }
        }
      }
    }
  }
  red[t] = sq;
  __syncthreads();  // also publishes Ts
  stamp(st0, 14);
  const int pw = a.nreq + a.gr * a.gr;
  double* p2 = a.part2 + (int64_t)g * kFusedStride;
  if (t < a.nreq) {
    double s2 = 0.0;
    for (int j = t; j < rpt * rq; j += rq) s2 += red[j];
    p2[t] = s2;
  }
  if (a.gr > 0) {
    // same product order as the phase-0 partial
    for (int o = t; o < a.gr * a.gr; o += NT) {
      const int ia = o / a.gr, cc = o - ia * a.gr;
      p2[a.nreq + o] = rows_dot(Ts, rq, ia, Ts, rq, cc, rows);
    }
  }
  stamp(st0, 9);
  if (a.rows_ctr) {
    // this CTA's Ritz rows (T, V_next) are final: count them and let the next operand pass launch
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(a.rows_ctr, 1ull);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (rr_cta) {
    // (Hs and the theta copy in thsh are untouched by phase 2; the epilogue lands in the pack before
    // this CTA's ticket below, whose fence publishes it to the CTA that writes the pack out)
    for (int o = t; o < b * b; o += NT) {
      const int ia = o / b, cc = o - ia * b;
      if (ia <= cc) a.H[ia * a.ldh + cc] = Hs[o];
    }
    if (a.epi && t < 32) step_epilogue_warp(thsh, a.nreq, a.n, a.eps_next, a.epi);
  }
  double* res2 = a.part2 + (int64_t)(G + (G + kGroup - 1) / kGroup) * kFusedStride;
  if (tree_reduce<NT, CL>(a.part2, a.part2 + (int64_t)G * kFusedStride, res2, pw, kFusedStride, a.sync + 64, &s_flag)) {
    stamp(a.stamps, 10);
    for (int o = t; o < pw; o += NT) {
      const double v = res2[o];
      if (o < a.nreq)
        a.resid[o] = sqrt(v);
      else
        a.gram[o - a.nreq] = v;
    }
    __threadfence_block();
    __syncthreads();
    stamp(a.stamps, 11);
    if (a.host_pack) {
      // the result pack straight into the caller's pinned host slot (no separate read-back copy)
      for (int idx = t; idx < a.pack_count; idx += NT) a.host_pack[idx] = __ldcg(a.pack + idx);
    }
    stamp(a.stamps, 12);
    if (a.done_flag) {
      __threadfence_system();
      __syncthreads();
      if (t == 0) {
        if (a.host_pack) *reinterpret_cast<volatile double*>(a.host_pack + a.pack_count) = (double)a.epoch;
        __threadfence_system();
        st_release_u32(a.done_flag, a.epoch);
      }
    }
  }
}

}  // namespace

// launch shape: threads per CTA and target rows per CTA (diagnostics overrides
// MEGB200_FUSED_NT = 256 | 512 | 1024, MEGB200_FUSED_ROWS)
int fused_nt() {
  static const int nt = [] {
    const char* e = getenv("MEGB200_FUSED_NT");
    const int v = e ? atoi(e) : 512;
    return (v == 512 || v == 1024) ? v : 256;
  }();
  return nt;
}

int fused_pass_rows(int64_t n, int sm_count) {
  static const int target = [] {
    const char* e = getenv("MEGB200_FUSED_ROWS");
    return e ? std::max(1, atoi(e)) : 32;
  }();
  int G = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count, (n + target - 1) / target));
  if (G >= kGroup) G -= G % kGroup;  // whole clusters of kGroup CTAs
  return (int)((n + G - 1) / G);
}

// dynamic shared memory of the fused kernel: up to 224 KiB (its static arrays take ~1 KiB of the
// 227 KiB per CTA), so cfg5-sized row ranges (R = 256, b = 32, l = 20) still stage their L rows
constexpr size_t kFusedSmemMax = 224 * 1024;

// shared memory of the fused kernel; L rows are staged when they fit (stage_l), else read from global
size_t fused_pass_smem(int64_t n, int b, int l, int rq, int sm_count, bool* stage_l = nullptr) {
  const int R = fused_pass_rows(n, sm_count);
  const size_t jac = std::max((size_t)jacobi_smem_doubles(b), (size_t)5 * b * b + 128);
  const size_t head = (size_t)2 * R * b + (size_t)b * rq + fused_nt() + (size_t)b * b;
  const size_t with_l = (head + std::max((size_t)R * l + (size_t)l * b + jac, (size_t)R * rq)) * sizeof(double);
  const size_t without = (head + std::max((size_t)l * b + jac, (size_t)R * rq)) * sizeof(double);
  const bool st = with_l <= kFusedSmemMax;
  if (stage_l) *stage_l = st;
  return st ? with_l : without;
}

bool fused_pass_supported(int64_t n, int b, int l, int nreq, int sm_count) {
  return b >= 2 && b <= 32 && nreq <= b && l >= 0 && l <= kFusedMaxL && n >= b &&
         fused_pass_smem(n, b, l, b, sm_count) <= kFusedSmemMax;
}

template <int NT, bool CL>
void launch_fused(const Launch& L, const FusedPassArgs& a, int G, size_t smem) {
  static char attr = 0;
  if (first_on_device(&attr)) {
    MEG_CUDA(cudaFuncSetAttribute(k_fused_first_pass<NT, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kFusedSmemMax));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = L.stream;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  int na = 1;
  if (a.cooperative) {
    // the driver guarantees that all CTAs are co-resident (the tickets and release flags rely on
    // it) also against fused kernels of other solver handles that may run on other streams
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  if (CL) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = kGroup;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  MEG_CUDA(cudaLaunchKernelEx(&cfg, k_fused_first_pass<NT, CL>, a));
  MEG_LAUNCHED();
  ++*L.counter;
}

// clusters of kGroup CTAs when every cluster of the grid can be resident at once (the release
// flags need co-residency); otherwise the ticket version
template <int NT>
bool cluster_fits(int G, size_t smem) {
  static int max_clusters_dev[64];  // per device (the attribute and occupancy are per device)
  int dev = 0;
  MEG_CUDA(cudaGetDevice(&dev));
  int& max_clusters = max_clusters_dev[dev & 63];
  if (first_on_device(max_clusters_dev)) {
    MEG_CUDA(cudaFuncSetAttribute(k_fused_first_pass<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kFusedSmemMax));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = kFusedSmemMax;  // worst case of the supported shapes
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kGroup;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_fused_first_pass<NT, true>, &cfg) != cudaSuccess) nc = 0;
    cudaGetLastError();
    max_clusters = nc;
  }
  (void)smem;
  return G % kGroup == 0 && G / kGroup <= max_clusters;
}

int fused_first_pass(const Launch& L, FusedPassArgs a, int sm_count) {
  // clusters of 8 replace the group tickets with the hardware cluster barrier; measured ~1.5 us
  // faster per step but with sporadic 2x slow runs (cluster placement under the pass's tail), so
  // they are a diagnostics option (MEGB200_CLUSTER=1), not the default
  static const bool no_cluster = getenv("MEGB200_CLUSTER") == nullptr;
  a.R = fused_pass_rows(a.n, sm_count);
  int G = (int)((a.n + a.R - 1) / a.R);
  bool stage_l = true;
  const size_t smem = fused_pass_smem(a.n, a.b, a.l, a.rq, sm_count, &stage_l);
  a.stage_l = stage_l;
  if (!(a.b >= 2 && a.b <= 32 && a.rq <= a.b && a.nreq <= a.rq && a.gr <= a.rq && a.l <= kFusedMaxL) ||
      smem > kFusedSmemMax || G > sm_count)
    throw Error(MEGB200_ERR_PARAM, "fused first pass: unsupported shape");
  const int nt = fused_nt();
  const bool cl = !no_cluster && G % kGroup == 0 &&
                  (nt == 1024 ? cluster_fits<1024>(G, smem) : nt == 512 ? cluster_fits<512>(G, smem)
                                                                        : cluster_fits<256>(G, smem));
  switch (nt) {
    case 1024: cl ? launch_fused<1024, true>(L, a, G, smem) : launch_fused<1024, false>(L, a, G, smem); break;
    case 512: cl ? launch_fused<512, true>(L, a, G, smem) : launch_fused<512, false>(L, a, G, smem); break;
    default: cl ? launch_fused<256, true>(L, a, G, smem) : launch_fused<256, false>(L, a, G, smem); break;
  }
  return G;
}

}  // namespace megb200
