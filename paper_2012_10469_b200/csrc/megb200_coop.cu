// Cooperative tall-skinny kernels (K4, K5, K7 of SURVEY.md section 2).
//
// Each kernel is one cooperative launch over G <= #SMs CTAs: every CTA
// reduces its contiguous row range into a partial, grid.sync(), every CTA
// finishes a slice of the outputs by summing the G partials in CTA order
// (fixed order -> bitwise reproducible), and -- where the algorithm needs it
// -- a further grid.sync() lets the same launch apply the result to its rows.
// This turns a CGS round, a CholQR round or a Ritz/residual evaluation into a
// single launch instead of 3-5 dependent ones.

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "megb200_internal.h"

namespace cg = cooperative_groups;

namespace megb200 {

// Optional phase timestamps (compile with -DMEG_PHASE_TIMING): CTA 0 thread 0
// records %globaltimer at phase boundaries of the cooperative kernels.
__device__ unsigned long long g_phase_ns[64];
#ifdef MEG_PHASE_TIMING
#define PIPCLK(i_) if (blockIdx.x == 0 && threadIdx.x == 0) g_phase_ns[32 + (i_)] = clock64();
#else
#define PIPCLK(i_)
#endif
__device__ __forceinline__ void phase_mark(int slot) {
#ifdef MEG_PHASE_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase_ns[slot] = t;
  }
#else
  (void)slot;
#endif
}

}  // namespace megb200

#define JACOBI_MARK(slot) phase_mark(slot)
#include "megb200_jacobi.cuh"

namespace megb200 {

namespace {

constexpr int kCT = 256;     // threads per CTA
constexpr int kRC = 32;      // rows staged per chunk
constexpr int kMaxLowrank = 160;  // widest low-rank factor of an operator (solver max_lowrank)
constexpr double kInv53c = 1.0 / 9007199254740992.0;

__device__ __forceinline__ double gauss_c(uint64_t key, uint64_t ctr) {
  const uint64_t b1 = mix64(key + (2 * ctr + 1) * kGolden);
  const uint64_t b2 = mix64(key + (2 * ctr + 2) * kGolden);
  const double u1 = ((double)(b1 >> 11) + 1.0) * kInv53c;
  const double u2 = (double)(b2 >> 11) * kInv53c;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__device__ __forceinline__ void cta_rows(int64_t n, int64_t& r0, int64_t& r1) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  r0 = min(n, (int64_t)blockIdx.x * per);
  r1 = min(n, r0 + per);
}

// acc[j] += sum_{rows in [r0,r1)} X[r, a_j] * Y[r, c_j]   for outputs o_j = tid + j*kCT < p*q
template <int J>
__device__ __forceinline__ void xty_rows(int64_t r0, int64_t r1, const double* __restrict__ X, int64_t ldx, int p,
                                         const double* __restrict__ Y, int64_t ldy, int q, double* sm,
                                         double (&acc)[J], bool gram = false) {
  // gram: the output has q more rows, Y^T Y, after the p rows of X^T Y (the staged Y rows serve as both)
  double* Xs = sm;
  double* Ys = sm + kRC * p;
  const int pq = (gram ? p + q : p) * q;
  int oa[J], oc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int o = threadIdx.x + j * kCT;
    oa[j] = o < pq ? o / q : 0;
    oc[j] = o < pq ? o - (o / q) * q : 0;
    acc[j] = 0.0;
  }
  for (int64_t rc = r0; rc < r1; rc += kRC) {
    const int rows = (int)min((int64_t)kRC, r1 - rc);
    __syncthreads();
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * p; idx += kCT) {
      const int r = idx / p, a = idx - r * p;
      Xs[idx] = X[(rc + r) * ldx + a];
    }
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      Ys[idx] = Y[(rc + r) * ldy + c];
    }
    __syncthreads();
    #pragma unroll 1
    for (int r = 0; r < rows; ++r) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const double xv = oa[j] < p ? Xs[r * p + oa[j]] : Ys[r * q + (oa[j] - p)];
        acc[j] = fma(xv, Ys[r * q + oc[j]], acc[j]);
      }
    }
  }
}
// Register-tiled X^T Y over a CTA's rows (optionally with the q rows Y^T Y after the p rows of X^T Y):
// a thread owns NT tiles of TA output rows x 4 consecutive output columns, so a staged row costs
// TA + 4 shared-memory loads per 4 TA multiply-adds (the one-output-per-slot form above loads two
// operands per multiply-add and is bound by shared-memory wavefronts: 30 us for cfg4's L^T U).
// The partials land at their linear index a * q + c, as store_partial would put them.
template <int TA, int NT>
__device__ __forceinline__ void xty_rows_tiled_store(int64_t r0, int64_t r1, const double* __restrict__ X, int64_t ldx,
                                                     int p, const double* __restrict__ Y, int64_t ldy, int q,
                                                     double* sm, bool gram, double* __restrict__ part) {
  double* Xs = sm;
  double* Ys = sm + kRC * p;
  const int pe = gram ? p + q : p;
  const int ncg = (q + 3) / 4, nag = (pe + TA - 1) / TA, tiles = nag * ncg;
  int ta[NT], tc[NT];
  double acc[NT][TA][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int tt = threadIdx.x + i * kCT;
    ta[i] = tt < tiles ? (tt / ncg) * TA : -1;
    tc[i] = tt < tiles ? (tt - (tt / ncg) * ncg) * 4 : 0;
#pragma unroll
    for (int v = 0; v < TA; ++v)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[i][v][u] = 0.0;
  }
  for (int64_t rc = r0; rc < r1; rc += kRC) {
    const int rows = (int)min((int64_t)kRC, r1 - rc);
    __syncthreads();
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * p; idx += kCT) {
      const int r = idx / p, a = idx - r * p;
      Xs[idx] = X[(rc + r) * ldx + a];
    }
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      Ys[idx] = Y[(rc + r) * ldy + c];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      if (ta[i] < 0) continue;
      #pragma unroll 2
      for (int r = 0; r < rows; ++r) {
        double y[4], xv[TA];
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = tc[i] + u < q ? Ys[r * q + tc[i] + u] : 0.0;
#pragma unroll
        for (int v = 0; v < TA; ++v) {
          const int a = ta[i] + v;
          xv[v] = a < p ? Xs[r * p + a] : (a < pe ? Ys[r * q + (a - p)] : 0.0);
        }
#pragma unroll
        for (int v = 0; v < TA; ++v)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[i][v][u] = fma(xv[v], y[u], acc[i][v][u]);
      }
    }
  }
  double* out = part + (int64_t)blockIdx.x * pe * q;
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    if (ta[i] < 0) continue;
#pragma unroll
    for (int v = 0; v < TA; ++v)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int a = ta[i] + v, c = tc[i] + u;
        if (a < pe && c < q) out[a * q + c] = acc[i][v][u];
      }
  }
}
template <int J>
__device__ __forceinline__ void store_partial(double* __restrict__ part, int pq, const double (&acc)[J]) {
  double* out = part + (int64_t)blockIdx.x * pq;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int o = threadIdx.x + j * kCT;
    if (o < pq) out[o] = acc[j];
  }
}

// Distributed final reduction, one warp per output: lanes load partials
// g = lane, lane + 32, ... in parallel (independent L2 loads) and combine with a
// fixed xor-shuffle tree, so the result is reproducible and the latency is one
// round trip instead of G dependent ones.
__device__ __forceinline__ double warp_min_f64(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

__device__ __forceinline__ double warp_sum_partials(const double* __restrict__ part, int G, int64_t stride, int o) {
  const int lane = threadIdx.x & 31;
  double v[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {  // G <= 160 in one round of independent loads
    const int g = lane + 32 * k;
    v[k] = g < G ? part[(int64_t)g * stride + o] : 0.0;
  }
  double s = (v[0] + v[1]) + (v[2] + v[3]) + v[4];
#pragma unroll 1
  for (int g = lane + 160; g < G; g += 32) s += part[(int64_t)g * stride + o];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// Small grids (n <= 16 kRC rows): a thread per output sums the G partials with the xor tree
// warp_sum_partials applies across lanes (lanes >= G hold zeros), so the sum is the same; a warp
// per output leaves only G * 8 warps for up to 3.6k outputs there, a chain of dependent
// global-load round trips (80 us of k_coop_orth's CGS reduction at n = 100)
constexpr int kThreadSumG = 16;

__device__ __forceinline__ double thread_sum_partials(const double* __restrict__ part, int G, int64_t stride, int o) {
  double w[kThreadSumG];
#pragma unroll
  for (int g = 0; g < kThreadSumG; ++g) w[g] = g < G ? part[(int64_t)g * stride + o] : 0.0;
#pragma unroll
  for (int off = kThreadSumG / 2; off >= 1; off >>= 1)
#pragma unroll
    for (int i = 0; i < off; ++i) w[i] += w[i + off];
  return w[0];
}

struct PartRef {
  const double* p;
  int64_t stride;
  int o;
};

// emit(o, sum over the grid's partials of output o) for o in [0, nout); ref(o) locates the partials
template <typename Ref, typename Emit>
__device__ __forceinline__ void grid_reduce_outputs(int nout, Ref&& ref, Emit&& emit) {
  const int G = gridDim.x;
  if (G <= kThreadSumG) {
    #pragma unroll 1
    for (int o = blockIdx.x * kCT + threadIdx.x; o < nout; o += G * kCT) {
      const PartRef r = ref(o);
      emit(o, thread_sum_partials(r.p, G, r.stride, r.o));
    }
  } else {
    const int wpb = kCT / 32;
    #pragma unroll 1
    for (int o = blockIdx.x * wpb + (threadIdx.x >> 5); o < nout; o += G * wpb) {
      const PartRef r = ref(o);
      const double v = warp_sum_partials(r.p, G, r.stride, r.o);
      if ((threadIdx.x & 31) == 0) emit(o, v);
    }
  }
}

__device__ __forceinline__ void reduce_partials(const double* __restrict__ part, int pq, int q,
                                                double* __restrict__ C, int64_t ldc,
                                                const double* __restrict__ rowscale, double scale) {
  grid_reduce_outputs(
      pq, [&](int o) { return PartRef{part, pq, o}; },
      [&](int o, double s) {
        const int a = o / q, c = o - a * q;
        if (rowscale) s *= rowscale[a];
        C[(int64_t)a * ldc + c] = scale * s;
      });
}

// ---------------------------------------------------------------------------
// Cholesky of a q x q SPD Gram (q <= 64) by one CTA (all threads),
// column-equilibrated, with breakdown detection (pivot <= thresh^2 absolute or
// 1e-20 relative -> flagged column).  Writes Rrel (zero rows for flagged
// columns), Rinv (by a row-parallel backward sweep, reciprocal multiplies
// only), mask; optionally Rtot = Rrel * Rprev.
__device__ void block_cholesky(const double* __restrict__ Gg, int q, double thresh, double* sm,
                               double* __restrict__ Rrel, double* __restrict__ Rinv, int* __restrict__ mask,
                               const double* __restrict__ Rprev, double* __restrict__ Rtot,
                               double* pivot_min = nullptr) {
  const int t = threadIdx.x, nth = blockDim.x;
  const int ld = q + 1;
  PIPCLK(8)
  double pmin = 1.0;  // smallest equilibrated pivot (every thread tracks it from shared memory)
  double* A = sm;             // q x ld   (factorised in place: upper triangle -> Rs)
  double* X = sm + q * ld;    // q x ld   (Rs^-1)
  double* D = X + q * ld;     // q
  double* rd = D + q;         // q  (1 / Rs_ii)
  int* bad = reinterpret_cast<int*>(rd + q);
  for (int idx = t; idx < q * q; idx += nth) {
    const int i = idx / q, j = idx - i * q;
    A[i * ld + j] = Gg[(i <= j) ? i * q + j : j * q + i];
    X[i * ld + j] = 0.0;
  }
  __syncthreads();
  for (int i = t; i < q; i += nth) {
    const double g = A[i * ld + i];
    bad[i] = !(g > thresh * thresh);
    D[i] = bad[i] ? 1.0 : sqrt(g);
    X[i * ld + q] = 1.0 / D[i];  // padding column of X: used for R^-1's row scaling at the end
  }
  __syncthreads();
  for (int idx = t; idx < q * q; idx += nth) {
    const int i = idx / q, j = idx - i * q;
    A[i * ld + j] = (bad[i] || bad[j]) ? (i == j ? 1.0 : 0.0) : A[i * ld + j] / (D[i] * D[j]);
  }
  __syncthreads();
  // right-looking factorisation and R^-1 by ONE warp with warp barriers only (q <= 64 columns: a
  // column step is a few hundred cycles, which CTA-wide barriers and a one-thread pivot dominated --
  // 22 us at q = 18).  Every lane forms the pivot (reciprocal square root, r = d * rsqrt(d)); lane l
  // owns column l of the trailing update and of R^-1 (no barrier inside a column's back substitution).
  PIPCLK(9)
  if (t < 32) {
    const int lane = t;
    // left-looking by rows of R: in step k every lane l >= k forms s_l = A[k][l] - sum_{i<k} R[i][k] R[i][l]
    // (a dot product over finished entries: its loads pipeline, nothing is read back after a store
    // inside the loop -- the right-looking update's read-modify-write chains cost ~2000 cycles per
    // column), the pivot s_k is broadcast, R[k][l] = s_l / sqrt(s_k).  Same subtraction order per entry
    // as the right-looking form.  One warp barrier per step.
    double pm = 1.0;
    for (int k = 0; k < q; ++k) {
      double sv[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = lane + 32 * h;
        if (l >= k && l < q) {
          // two chains (even / odd i): the float64 multiply-add latency, not its rate, bounds this loop
          double s0 = A[k * ld + l], s1 = 0.0;
          int i = 0;
#pragma unroll 4
          for (; i + 1 < k; i += 2) {
            s0 = fma(-A[i * ld + k], A[i * ld + l], s0);
            s1 = fma(-A[(i + 1) * ld + k], A[(i + 1) * ld + l], s1);
          }
          if (i < k) s0 = fma(-A[i * ld + k], A[i * ld + l], s0);
          sv[h] = s0 + s1;
        }
      }
      const double d = __shfl_sync(0xffffffffu, (k >> 5) ? sv[1] : sv[0], k & 31);
      const bool bj = bad[k] || !(d > 1e-20);
      pm = bj ? 0.0 : fmin(pm, d);
      // (the step is a ~800-cycle chain of dependent float64 operations -- dot, broadcast, reciprocal
      // square root, scale, store -- whichever reciprocal square root is used)
      const double ir = bj ? 1.0 : rsqrt(d);
      const double r = bj ? 1.0 : d * ir;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = lane + 32 * h;
        if (l == k) {
          A[k * ld + k] = r;
          rd[k] = ir;
          bad[k] = bj;
        } else if (l > k && l < q) {
          A[k * ld + l] = bj ? 0.0 : sv[h] * ir;
        }
      }
      __syncwarp();
    }
    if (lane == 0) A[q] = pm;  // smallest pivot, in the padding column of row 0
    PIPCLK(10)
    // Rs^-1 by columns: X[i][c] = -rd_i * sum_{k=i+1..c} Rs[i][k] X[k][c], X[c][c] = rd_c
    for (int c = lane; c < q; c += 32) {
      X[c * ld + c] = rd[c];
      for (int i = c - 1; i >= 0; --i) {
        double s0 = 0.0, s1 = 0.0;
        int k = i + 1;
#pragma unroll 4
        for (; k + 1 <= c; k += 2) {
          s0 = fma(A[i * ld + k], X[k * ld + c], s0);
          s1 = fma(A[i * ld + k + 1], X[(k + 1) * ld + c], s1);
        }
        if (k <= c) s0 = fma(A[i * ld + k], X[k * ld + c], s0);
        X[i * ld + c] = -(s0 + s1) * rd[i];
      }
    }
  }
  PIPCLK(11)
  __syncthreads();
  pmin = A[q];
  for (int idx = t; idx < q * q; idx += nth) {
    const int i = idx / q, j = idx - i * q;
    Rinv[idx] = (i <= j) ? X[i * ld + j] * X[i * ld + q] : 0.0;  // 1 / D_i from the padding column
    Rrel[idx] = (bad[i] || j < i) ? 0.0 : A[i * ld + j] * D[j];
  }
  for (int i = t; i < q; i += nth) mask[i] = bad[i];
  PIPCLK(12)
  if (pivot_min) *pivot_min = pmin;
  if (Rtot) {
    for (int idx = t; idx < q * q; idx += nth) {
      const int i = idx / q, j = idx - i * q;
      double s = 0.0;
      if (!bad[i])
        for (int k = i; k < q; ++k) s += A[i * ld + k] * D[k] * Rprev[k * q + j];
      Rtot[idx] = s;
    }
  }
}

// ===========================================================================
// C = diag(rowscale) * scale * X^T Y    (one launch)
template <int J>
__global__ void __launch_bounds__(kCT) k_coop_tn(int64_t n, const double* __restrict__ X, int64_t ldx, int p,
                                                  const double* __restrict__ Y, int64_t ldy, int q,
                                                  double* __restrict__ C, int64_t ldc,
                                                  const double* __restrict__ rowscale, double scale,
                                                  double* __restrict__ part) {
  extern __shared__ double sm[];
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  double acc[J];
  xty_rows<J>(r0, r1, X, ldx, p, Y, ldy, q, sm, acc);
  store_partial<J>(part, p * q, acc);
  cg::this_grid().sync();
  reduce_partials(part, p * q, q, C, ldc, rowscale, scale);
}

// One classical Gram-Schmidt round: C = Q^T W (optionally saved to Cout), W -= Q C.
template <int J>
__global__ void __launch_bounds__(kCT) k_coop_cgs(int64_t n, const double* __restrict__ Q, int64_t ldq, int cols,
                                                   double* __restrict__ W, int64_t ldw, int q, double* __restrict__ Cws,
                                                   double* __restrict__ part) {
  extern __shared__ double sm[];
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  double acc[J];
  xty_rows<J>(r0, r1, Q, ldq, cols, W, ldw, q, sm, acc);
  store_partial<J>(part, cols * q, acc);
  cg::grid_group grid = cg::this_grid();
  grid.sync();
  reduce_partials(part, cols * q, q, Cws, q, nullptr, 1.0);
  grid.sync();
  // W[r, c] -= sum_k Q[r, k] C[k, c]   (C in shared memory)
  double* Cs = sm;
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < cols * q; idx += kCT) Cs[idx] = Cws[idx];
  __syncthreads();
  #pragma unroll 1
  for (int64_t idx = threadIdx.x; idx < (r1 - r0) * q; idx += kCT) {
    const int64_t r = r0 + idx / q;
    const int c = (int)(idx % q);
    const double* qr = Q + r * ldq;
    double s = 0.0;
    #pragma unroll 1
    for (int k = 0; k < cols; ++k) s = fma(qr[k], Cs[k * q + c], s);
    W[r * ldw + c] -= s;
  }
}

// One CholQR round: G = W^T W, R = chol(G) (CTA 0, one warp), W = W R^-1 with
// breakdown columns replaced by seeded random normals.
template <int J>
__global__ void __launch_bounds__(kCT) k_coop_cholqr(int64_t n, const double* __restrict__ Wsrc, int64_t lds, double* __restrict__ W, int64_t ldw, int q,
                                                      double thresh, double* __restrict__ Gws,
                                                      double* __restrict__ Rrel, double* __restrict__ Rinv,
                                                      int* __restrict__ mask, const double* __restrict__ Rprev,
                                                      double* __restrict__ Rtot, uint64_t key, uint64_t base,
                                                      double* __restrict__ part) {
  extern __shared__ double sm[];
  phase_mark(0);
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  double acc[J];
  xty_rows<J>(r0, r1, Wsrc, lds, q, Wsrc, lds, q, sm, acc);
  store_partial<J>(part, q * q, acc);
  phase_mark(1);
  cg::grid_group grid = cg::this_grid();
  grid.sync();
  phase_mark(2);
  reduce_partials(part, q * q, q, Gws, q, nullptr, 1.0);
  grid.sync();
  phase_mark(3);
  if (blockIdx.x == 0) block_cholesky(Gws, q, thresh, sm, Rrel, Rinv, mask, Rprev, Rtot);
  phase_mark(4);
  grid.sync();
  phase_mark(5);
  double* Ri = sm;
  int* bad = reinterpret_cast<int*>(sm + q * q);
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < q * q; idx += kCT) Ri[idx] = Rinv[idx];
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < q; idx += kCT) bad[idx] = mask[idx];
  __syncthreads();
  // rows of this CTA: W[r, :] <- W[r, :] Rinv  (row staged in registers through shared memory)
  double* Ws = sm + q * q + 64;
  for (int64_t rc = r0; rc < r1; rc += kRC) {
    const int rows = (int)min((int64_t)kRC, r1 - rc);
    __syncthreads();
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      Ws[idx] = Wsrc[(rc + r) * lds + c];
    }
    __syncthreads();
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      double v;
      if (bad[c]) {
        v = gauss_c(key, base + (uint64_t)(rc + r) * q + c);
      } else {
        v = 0.0;
        #pragma unroll 1
        for (int k = 0; k <= c; ++k) v = fma(Ws[r * q + k], Ri[k * q + c], v);
      }
      W[(rc + r) * ldw + c] = v;
    }
  }
  phase_mark(6);
}

// Operator epilogue: E = diag(d) L^T U (reduced across the grid), then
// W = scale * sum_s part[s] + L E + alpha U.
template <int J, int J2>
__global__ void __launch_bounds__(kCT) k_coop_finish(int64_t n, int b, int S, const double* __restrict__ spart,
                                                      double scale, const double* __restrict__ Lf, int64_t ldl, int l,
                                                      const double* __restrict__ d, double alpha,
                                                      const double* __restrict__ U, int64_t ldu,
                                                      double* __restrict__ W, int64_t ldw, double* __restrict__ Ews,
                                                      double* __restrict__ part, const double* __restrict__ Qh,
                                                      int64_t ldq, int hp, double* __restrict__ Hout, int64_t ldh,
                                                      LamCoef lc, const double* __restrict__ Eg, int64_t ldg,
                                                      double* __restrict__ Gout) {
  extern __shared__ double sm[];
  __shared__ double dsh[kMaxLowrank];
  phase_mark(20);
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  if (lc.lam) {
    // coefficients from device-resident kept weights (first lr), the rest as given
    #pragma unroll 1
    for (int k = threadIdx.x; k < l; k += kCT) {
      double v;
      if (k < lc.lr) {
        const double kept = lc.c1 * lc.lam[k];
        v = (log(kept) - lc.log_tail) + (-lc.eta * (kept - lc.tail_g));
      } else {
        v = d[k];
      }
      dsh[k] = v;
    }
    d = dsh;  // read after the barrier below
  }
  if (Eg) {
    __syncthreads();  // E = diag(d) L^T U from the caller's L^T U (no grid reduction)
  } else if (l > 0) {
    if constexpr (J > 16) xty_rows_tiled_store<4, 2>(r0, r1, Lf, ldl, l, U, ldu, b, sm, false, part);
    else xty_rows_tiled_store<2, 2>(r0, r1, Lf, ldl, l, U, ldu, b, sm, false, part);
    cg::grid_group grid = cg::this_grid();
    grid.sync();
    phase_mark(21);
    reduce_partials(part, l * b, b, Ews, b, d, 1.0);
    grid.sync();
  }
  phase_mark(22);
  double* Es = sm;
  double* Ls = sm + l * b;  // this chunk's rows of L (kRC x l)
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < l * b; idx += kCT) {
    const int k = idx / b, c = idx - k * b;
    Es[idx] = Eg ? d[k] * Eg[k * ldg + c] : Ews[idx];
  }
  for (int64_t rc = r0; rc < r1; rc += kRC) {
    const int rows = (int)min((int64_t)kRC, r1 - rc);
    __syncthreads();
    // stage the chunk's L rows (independent coalesced loads) so the L E products read shared memory
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * l; idx += kCT) {
      const int r = idx / l, k = idx - r * l;
      Ls[idx] = Lf[(rc + r) * ldl + k];
    }
    __syncthreads();
    #pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * b; idx += kCT) {
      const int rr = idx / b, c = idx - rr * b;
      const int64_t i = rc + rr;
      double pv[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) pv[t] = t < S ? spart[(int64_t)t * n * b + i * b + c] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < 16; ++t) s += pv[t];
      const double* Lr = Ls + rr * l;
      double v0 = scale * s + alpha * U[i * ldu + c], v1 = 0.0;
      int k = 0;
      #pragma unroll 1
      for (; k + 1 < l; k += 2) {
        v0 = fma(Lr[k], Es[k * b + c], v0);
        v1 = fma(Lr[k + 1], Es[(k + 1) * b + c], v1);
      }
      if (k < l) v0 = fma(Lr[k], Es[k * b + c], v0);
      W[i * ldw + c] = v0 + v1;
    }
  }
  phase_mark(23);
  if (Hout) {
    // H[0:hp, :] = Q[:, 0:hp]^T W over this CTA's rows (W just written), reduced across the grid
    __syncthreads();
    // (Gout: W^T W rides along as b more rows of the same reduction -- with H's rows, which are
    // Q^T W, it is what the first Pythagorean round of the next block's orthonormalisation needs)
    const int hpe = Gout ? hp + b : hp;
    // (E partials were consumed before the previous grid.sync)
    if constexpr (J2 > 16) xty_rows_tiled_store<4, 2>(r0, r1, Qh, ldq, hp, W, ldw, b, sm, Gout != nullptr, part);
    else xty_rows_tiled_store<2, 2>(r0, r1, Qh, ldq, hp, W, ldw, b, sm, Gout != nullptr, part);
    cg::grid_group grid = cg::this_grid();
    phase_mark(24);
    grid.sync();
    phase_mark(25);
    grid_reduce_outputs(
        hpe * b, [&](int o) { return PartRef{part, hpe * b, o}; },
        [&](int o, double v) {
          const int a = o / b, c = o - a * b;
          if (a < hp) Hout[(int64_t)a * ldh + c] = v;
          else Gout[(a - hp) * b + c] = v;
        });
  }
  phase_mark(26);
}


// ===========================================================================
// Whole block orthonormalisation in one cooperative launch (the sequence of
// orthonormalize(): CGS, CGS, CholQR (breakdown threshold), CGS, CholQR), the
// CTA's rows of the basis Q and of the block W staged ONCE in shared memory.
// Each CGS / Gram reduction is one grid barrier + a fixed-order warp reduction
// + one grid barrier; the q x q Cholesky and R^-1 run in CTA 0 (block_cholesky).
// Same rules as k_coop_cgs / k_coop_cholqr:
// column equilibration, breakdown pivots (<= thresh^2 absolute, 1e-20 relative)
// flagged and refilled with the seeded normals of the same counters.

__global__ void __launch_bounds__(kCT, 1) k_coop_orth(int64_t n, const double* __restrict__ Q, int64_t ldq, int cols,
                                                     const double* Wsrc, int64_t lds, double* W, int64_t ldw, int q,
                                                     double thresh1,
                                                     uint64_t key, uint64_t base, double* __restrict__ part,
                                                     double* __restrict__ Cws, double* __restrict__ Gws,
                                                     double* __restrict__ Rinv, int* __restrict__ mask,
                                                     double* __restrict__ Rrel, int cgs_rounds, int pip,
                                                     const double* __restrict__ Cpre, int64_t ldcp,
                                                     const double* __restrict__ Gpre) {
  extern __shared__ double sm[];
  phase_mark(50);
  cg::grid_group grid = cg::this_grid();
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  const int rows = (int)(r1 - r0);
  const int R = (int)((n + gridDim.x - 1) / gridDim.x);
  double* Qs = sm;               // R x cols
  double* Ws = Qs + R * cols;    // R x q
  double* W2 = Ws + R * q;       // R x q
  double* Cs = W2 + R * q;       // cols x q, later R^-1 (q x q)
  int* bad = reinterpret_cast<int*>(Cs + max(cols * q, q * q));
  double* chol_sm = Cs + max(cols * q, q * q) + 32;  // CTA 0: Cholesky scratch
  const int t = threadIdx.x;
  for (int idx = t; idx < rows * cols; idx += kCT) {
    const int r = idx / cols, k = idx - r * cols;
    Qs[idx] = Q[(r0 + r) * ldq + k];
  }
  // the block is read from Wsrc (the image block A Q_j of the previous pass) and the orthonormal
  // block is written to W (its place in the basis): no copy launch in between
  for (int idx = t; idx < rows * q; idx += kCT) {
    const int r = idx / q, c = idx - r * q;
    Ws[idx] = Wsrc[(r0 + r) * lds + c];
  }
  __syncthreads();
  phase_mark(51);
  int pm = 52;
  auto cgs = [&]() {
    const int pq = cols * q;
    // C partial = Qs^T Ws: a thread owns four basis columns a0..a0+3 of one block column c
    // (four independent row-ordered chains, one Ws load per four FMAs)
    const int na4 = (cols + 3) / 4;
    for (int item = t; item < na4 * q; item += kCT) {
      const int a0 = (item / q) * 4, c = item - (item / q) * q;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = 0; r < rows; ++r) {
        const double wv = Ws[r * q + c];
        const double* qr = Qs + r * cols + a0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (a0 + u < cols) acc[u] = fma(qr[u], wv, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (a0 + u < cols) part[(int64_t)blockIdx.x * pq + (a0 + u) * q + c] = acc[u];
    }
    phase_mark(pm++);
    grid.sync();
    grid_reduce_outputs(pq, [&](int o) { return PartRef{part, pq, o}; }, [&](int o, double v) { Cws[o] = v; });
    grid.sync();
    phase_mark(pm++);
    for (int o = t; o < pq; o += kCT) Cs[o] = Cws[o];
    __syncthreads();
    // Ws -= Qs C: a thread owns four block columns c0..c0+3 of one row (one Qs load per four FMAs)
    const int nc4 = (q + 3) / 4;
    for (int item = t; item < rows * nc4; item += kCT) {
      const int r = item / nc4, c0 = (item - r * nc4) * 4;
      const double* qr = Qs + r * cols;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < cols; ++k) {
        const double qk = qr[k];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < q) acc[u] = fma(qk, Cs[k * q + c0 + u], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u < q) Ws[r * q + c0 + u] -= acc[u];
    }
    __syncthreads();
    phase_mark(pm++);
  };
  auto cholqr = [&](double thresh, uint64_t bs) {
    const int qq = q * q;
    const int nq4 = (q + 3) / 4;
    for (int item = t; item < nq4 * q; item += kCT) {
      const int a0 = (item / q) * 4, c = item - (item / q) * q;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = 0; r < rows; ++r) {
        const double wc = Ws[r * q + c];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (a0 + u < q) acc[u] = fma(Ws[r * q + a0 + u], wc, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (a0 + u < q) part[(int64_t)blockIdx.x * qq + (a0 + u) * q + c] = acc[u];
    }
    phase_mark(pm++);
    grid.sync();
    grid_reduce_outputs(qq, [&](int o) { return PartRef{part, qq, o}; }, [&](int o, double v) { Gws[o] = v; });
    grid.sync();
    phase_mark(pm++);
    if (blockIdx.x == 0) block_cholesky(Gws, q, thresh, chol_sm, Rrel, Rinv, mask, nullptr, nullptr);
    __syncthreads();
    phase_mark(pm++);
    grid.sync();
    double* Ri = Cs;  // q x q (C is consumed)
    for (int o = t; o < qq; o += kCT) Ri[o] = Rinv[o];
    for (int c = t; c < q; c += kCT) bad[c] = mask[c];
    __syncthreads();
    for (int idx = t; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      double v;
      if (bad[c]) {
        v = gauss_c(key, bs + (uint64_t)(r0 + r) * q + c);
      } else {
        v = 0.0;
        for (int k = 0; k <= c; ++k) v = fma(Ws[r * q + k], Ri[k * q + c], v);
      }
      W2[idx] = v;
    }
    __syncthreads();
    for (int idx = t; idx < rows * q; idx += kCT) Ws[idx] = W2[idx];
    __syncthreads();
    phase_mark(pm++);
  };
  // ---- fast path: two rounds of block Gram-Schmidt with the Pythagorean inner product (BCGS-PIP2).
  // One grid reduction per round yields C = Q^T W and G = W^T W together; the Gram of the projected
  // block is G' = G - C^T C, factorised redundantly by every CTA (no broadcast barrier), and
  // W <- (W - Q C) R^-1 in one sweep: 4 grid barriers instead of 12.  G' is formed by subtraction, so
  // a round is only taken when (kept share of each column's squared norm) x (smallest equilibrated
  // pivot) >= 1e-12 (the round's error ~ eps / that <= 1e-4, which the second round removes);
  // otherwise -- near-breakdown blocks, refills -- the five-phase sequence below runs from the same W.
  double* Gs = chol_sm + (2 * q * (q + 1) + 2 * q + 1) + 64;  // q x q: G, then G'
  double* Rinv_s = Gs + q * q;                                // q x q
  double* Rrel_s = Rinv_s + q * q;                            // q x q (unused factor output)
  int* mask_s = reinterpret_cast<int*>(Rrel_s + q * q);       // q
  auto pip_round = [&](double thresh, bool pre) -> bool {
    const int pq = cols * q, qq = q * q, tot = pq + qq;
    const int na4 = (cols + 3) / 4, nq4 = (q + 3) / 4;
    double* mypart = part + (int64_t)blockIdx.x * tot;
    // pre: C = Q^T W and G = W^T W were already reduced (by the finish of the pass that produced W)
    if (pre) {
      for (int o = t; o < pq; o += kCT) Cs[o] = __ldcg(Cpre + (int64_t)(o / q) * ldcp + (o - (o / q) * q));
      for (int o = t; o < qq; o += kCT) Gs[o] = __ldcg(Gpre + o);
      pm += 2;
    } else {
    for (int item = t; item < (na4 + nq4) * q; item += kCT) {
      const int grp4 = item / q, c = item - grp4 * q;
      const bool isq = grp4 < na4;
      const int a0 = (isq ? grp4 : grp4 - na4) * 4;
      const int lim = isq ? cols : q;
      const double* X = isq ? Qs : Ws;
      const int ldx = isq ? cols : q;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = 0; r < rows; ++r) {
        const double wv = Ws[r * q + c];
        const double* xr = X + r * ldx + a0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (a0 + u < lim) acc[u] = fma(xr[u], wv, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (a0 + u < lim) mypart[(isq ? 0 : pq) + (a0 + u) * q + c] = acc[u];
    }
    phase_mark(pm++);
    grid.sync();
    grid_reduce_outputs(tot, [&](int o) { return PartRef{part, tot, o}; },
                        [&](int o, double v) {
                          if (o < pq) Cws[o] = v;
                          else Gws[o - pq] = v;
                        });
    grid.sync();
    phase_mark(pm++);
    for (int o = t; o < pq; o += kCT) Cs[o] = __ldcg(Cws + o);
    for (int o = t; o < qq; o += kCT) Gs[o] = __ldcg(Gws + o);
    }
    __syncthreads();
    PIPCLK(0)
    // G' = G - C^T C (upper triangle; the lower is mirrored by block_cholesky) and the kept share of
    // every column's squared norm
    double keep_min = 1.0;
    for (int o = t; o < qq; o += kCT) {
      const int i = o / q, j = o - i * q;
      if (i <= j) {
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
        for (; k + 1 < cols; k += 2) {
          s0 = fma(Cs[k * q + i], Cs[k * q + j], s0);
          s1 = fma(Cs[(k + 1) * q + i], Cs[(k + 1) * q + j], s1);
        }
        if (k < cols) s0 = fma(Cs[k * q + i], Cs[k * q + j], s0);
        const double g = Gs[o];
        const double gp = g - (s0 + s1);
        if (i == j) keep_min = (g > 0.0 && gp > thresh * thresh) ? fmin(keep_min, gp / g) : 0.0;
        Rrel_s[o] = gp;
      }
    }
    __syncthreads();
    PIPCLK(1)
    for (int o = t; o < qq; o += kCT) {
      const int i = o / q, j = o - i * q;
      if (i <= j) Gs[o] = Rrel_s[o];
    }
    // CTA-wide minimum of keep_min (bad[0..] as scratch is not enough: use the warp partials in Rrel_s tail)
    keep_min = warp_min_f64(keep_min);
    __syncthreads();
    if ((t & 31) == 0) Rinv_s[t >> 5] = keep_min;
    __syncthreads();
    double km = 1.0;
    for (int wv = 0; wv < kCT / 32; ++wv) km = fmin(km, Rinv_s[wv]);
    __syncthreads();
    if (!(km >= 1e-11)) {  // uniform: every CTA reduced the same G and C
      if (blockIdx.x == 0 && t == 0) {  // diagnostics: rejected rounds and why (megb200_debug_phase_ns 56-59)
        g_phase_ns[56] += 1;
        g_phase_ns[58] = (unsigned long long)(km * 1e18);
      }
      return false;
    }
    PIPCLK(2)
    double pmin = 1.0;
    block_cholesky(Gs, q, thresh, chol_sm, Rrel_s, Rinv_s, mask_s, nullptr, nullptr, &pmin);
    __syncthreads();
    PIPCLK(3)
    bool okc = km * pmin >= 1e-12;  // error of the round ~ eps / (kept share x smallest pivot) <= 1e-4
    for (int c = 0; c < q; ++c) okc = okc && !mask_s[c];
    if (blockIdx.x == 0 && t == 0) {
      if (okc) g_phase_ns[55] += 1;
      else {
        g_phase_ns[57] += 1;
        g_phase_ns[59] = (unsigned long long)(km * pmin * 1e18);
      }
    }
    if (!okc) return false;  // uniform
    // W <- (W - Q C) R^-1: the projection into W2, then the triangular solve back into Ws
    const int nc4 = (q + 3) / 4;
    for (int item = t; item < rows * nc4; item += kCT) {
      const int r = item / nc4, c0 = (item - r * nc4) * 4;
      const double* qr = Qs + r * cols;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < cols; ++k) {
        const double qk = qr[k];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < q) acc[u] = fma(qk, Cs[k * q + c0 + u], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u < q) W2[r * q + c0 + u] = Ws[r * q + c0 + u] - acc[u];
    }
    __syncthreads();
    PIPCLK(4)
    for (int idx = t; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      double v = 0.0;
      for (int k = 0; k <= c; ++k) v = fma(W2[r * q + k], Rinv_s[k * q + c], v);
      Ws[idx] = v;
    }
    __syncthreads();
    phase_mark(pm++);
    return true;
  };
  bool done = false;
  if (pip && cols > 0 && cgs_rounds == 2) {
    if (pip_round(thresh1, Cpre != nullptr && Gpre != nullptr)) {
      done = pip_round(0.0, false);
    } else {
      // the round's C = Q^T W is the first CGS projection: apply it (Cs holds it), no second reduction
      const int nc4 = (q + 3) / 4;
      for (int item = t; item < rows * nc4; item += kCT) {
        const int r = item / nc4, c0 = (item - r * nc4) * 4;
        const double* qr = Qs + r * cols;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = 0; k < cols; ++k) {
          const double qk = qr[k];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c0 + u < q) acc[u] = fma(qk, Cs[k * q + c0 + u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < q) Ws[r * q + c0 + u] -= acc[u];
      }
      __syncthreads();
    }
    if (!done) cgs_rounds = 1;  // W is projected once: one more CGS before the CholQR rounds
  }
  if (!done) {
    for (int round = 0; round < cgs_rounds && cols > 0; ++round) cgs();
    cholqr(thresh1, base);
    if (cols > 0) cgs();
    cholqr(0.0, base + (uint64_t)n * q);
  }
  for (int idx = t; idx < rows * q; idx += kCT) {
    const int r = idx / q, c = idx - r * q;
    W[(r0 + r) * ldw + c] = Ws[idx];
  }
  phase_mark(pm < 63 ? pm : 63);
  if (threadIdx.x == 0 && blockIdx.x == 0) g_phase_ns[49] = pm;
}

int coop_grid(int64_t n, int sm_count) {
  const int64_t want = (n + kRC - 1) / kRC;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, sm_count));
}

template <typename K, typename... Args>
void coop_launch(const Launch& L, K kernel, int grid, size_t smem, Args... args) {
  void* argv[] = {(void*)&args...};
  MEG_CUDA(cudaLaunchCooperativeKernel((const void*)kernel, dim3(grid), dim3(kCT), argv, smem, L.stream));
  ++*L.counter;
}

template <typename K>
void raise_smem(K kernel, size_t bytes) {
  MEG_CUDA(cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

int pick_j(int pq) {
  const int j = (pq + kCT - 1) / kCT;
  if (j <= 1) return 1;
  if (j <= 2) return 2;
  if (j <= 4) return 4;
  if (j <= 8) return 8;
  if (j <= 16) return 16;
  if (j <= 24) return 24;
  throw Error(MEGB200_ERR_PARAM, "tall-skinny product too wide");
}

#define MEG_J_DISPATCH(jv, MACRO) \
  switch (jv) {                   \
    case 1: MACRO(1); break;      \
    case 2: MACRO(2); break;      \
    case 4: MACRO(4); break;      \
    case 8: MACRO(8); break;      \
    case 16: MACRO(16); break;    \
    default: MACRO(24); break;    \
  }

constexpr size_t kCoopSmem = 120 * 1024;

}  // namespace

// ---------------------------------------------------------------------------

void coop_tn(const Launch& L, int64_t n, const double* X, int64_t ldx, int p, const double* Y, int64_t ldy, int q,
             double* C, int64_t ldc, const double* rowscale, double scale, double* part, int sm_count) {
  const int G = coop_grid(n, sm_count);
  const size_t smem = (size_t)kRC * (p + q) * sizeof(double);
  const int J = pick_j(p * q);
#define MEG_TN(jj)                                                                                      \
  {                                                                                                     \
    static char a = 0;                                                                              \
    if (first_on_device(&a)) raise_smem(k_coop_tn<jj>, kCoopSmem);                                         \
    coop_launch(L, k_coop_tn<jj>, G, smem, n, X, ldx, p, Y, ldy, q, C, ldc, rowscale, scale, part);     \
  }
  MEG_J_DISPATCH(J, MEG_TN)
#undef MEG_TN
}

void coop_cgs(const Launch& L, int64_t n, const double* Q, int64_t ldq, int cols, double* W, int64_t ldw, int q,
              double* Cws, double* part, int sm_count) {
  const int G = coop_grid(n, sm_count);
  const size_t smem = std::max((size_t)kRC * (cols + q), (size_t)cols * q) * sizeof(double);
  const int J = pick_j(cols * q);
#define MEG_CGS(jj)                                                                              \
  {                                                                                              \
    static char a = 0;                                                                       \
    if (first_on_device(&a)) raise_smem(k_coop_cgs<jj>, kCoopSmem);                                 \
    coop_launch(L, k_coop_cgs<jj>, G, smem, n, Q, ldq, cols, W, ldw, q, Cws, part);              \
  }
  MEG_J_DISPATCH(J, MEG_CGS)
#undef MEG_CGS
}

void coop_cholqr(const Launch& L, int64_t n, const double* Wsrc, int64_t lds, double* W, int64_t ldw, int q,
                 double thresh, double* Gws, double* Rrel, double* Rinv, int* mask, const double* Rprev, double* Rtot,
                 uint64_t key, uint64_t base, double* part, int sm_count) {
  const int G = coop_grid(n, sm_count);
  const size_t chol_smem = (size_t)(2 * q * (q + 1) + 2 * q + 1) * sizeof(double) + 64 * sizeof(int);
  const size_t smem = std::max({(size_t)kRC * 2 * q * sizeof(double), chol_smem,
                                (size_t)(q * q + 64 + kRC * q) * sizeof(double)});
  const int J = pick_j(q * q);
#define MEG_CQR(jj)                                                                                          \
  {                                                                                                          \
    static char a = 0;                                                                                   \
    if (first_on_device(&a)) raise_smem(k_coop_cholqr<jj>, kCoopSmem);                                          \
    coop_launch(L, k_coop_cholqr<jj>, G, smem, n, Wsrc, lds, W, ldw, q, thresh, Gws, Rrel, Rinv, mask, Rprev, Rtot, key, \
                base, part);                                                                                 \
  }
  MEG_J_DISPATCH(J, MEG_CQR)
#undef MEG_CQR
}


bool coop_orth(const Launch& L, int64_t n, const double* Q, int64_t ldq, int cols, double* W, int64_t ldw, int q,
               double thresh1, uint64_t key, uint64_t base, double* part, double* Cws, double* Gws, double* Rinv,
               int* mask, double* Rrel, int sm_count, int cgs_rounds, const double* Wsrc, int64_t lds,
               const double* Cpre, int64_t ldcp, const double* Gpre) {
  if (!Wsrc) {
    Wsrc = W;
    lds = ldw;
  }
  static const bool off = getenv("MEGB200_NO_ORTH_FUSED") != nullptr;  // diagnostics: the five-launch path
  const int G = coop_grid(n, sm_count);
  const int R = (int)((n + G - 1) / G);
  const size_t chol_smem = (size_t)(2 * q * (q + 1) + 2 * q + 1) + 64;
  const size_t pip_smem = 3 * (size_t)q * q + 64;  // G / G', R^-1, factor scratch, mask of the PIP rounds
  const size_t smem = ((size_t)R * cols + 2 * (size_t)R * q + (size_t)std::max(cols * q, q * q) + 32 + chol_smem +
                       pip_smem) * sizeof(double);
  if (off || q > 32 || q < 1 || smem > 200 * 1024) return false;
  static const int pip = getenv("MEGB200_NO_ORTH_PIP") == nullptr;  // diagnostics: the five-phase sequence only
  static char a = 0;
  if (first_on_device(&a)) {
    raise_smem(k_coop_orth, 200 * 1024);
  }
  coop_launch(L, k_coop_orth, G, smem, n, Q, ldq, cols, Wsrc, lds, W, ldw, q, thresh1, key, base, part, Cws, Gws, Rinv,
              mask, Rrel, cgs_rounds, pip, Cpre, ldcp, Gpre);
  return true;
}

void coop_finish(const Launch& L, int64_t n, int b, int S, const double* spart, double scale, const double* Lf,
                 int64_t ldl, int l, const double* d, double alpha, const double* U, int64_t ldu, double* W,
                 int64_t ldw, double* Ews, double* part, int sm_count, const double* Qh, int64_t ldq, int hp,
                 double* Hout, int64_t ldh, LamCoef lc, const double* Eg, int64_t ldg, double* Gout) {
  if (!Hout) Gout = nullptr;
  if (lc.lam && (l > kMaxLowrank || lc.lr > l)) throw Error(MEGB200_ERR_PARAM, "finish: coefficient width out of range");
  const int G = coop_grid(n, sm_count);
  const size_t smem = std::max({(size_t)kRC * (l + b), (size_t)std::max(1, l * b) + (size_t)kRC * l,
                                (size_t)kRC * (hp + b)}) * sizeof(double);
  const int J = pick_j(std::max(1, l * b));
  const int J2 = Hout ? pick_j((hp + (Gout ? b : 0)) * b) : 1;
#define MEG_FIN2(jj, j2)                                                                                        \
  {                                                                                                             \
    static char a = 0;                                                                                      \
    if (first_on_device(&a)) raise_smem(k_coop_finish<jj, j2>, kCoopSmem);                                         \
    coop_launch(L, k_coop_finish<jj, j2>, G, smem, n, b, S, spart, scale, Lf, ldl, l, d, alpha, U, ldu, W, ldw,  \
                Ews, part, Qh, ldq, hp, Hout, ldh, lc, Eg, ldg, Gout);                                          \
  }
#define MEG_FIN(jj)                                            \
  switch (J2) {                                                \
    case 1: MEG_FIN2(jj, 1); break;                            \
    case 2: MEG_FIN2(jj, 2); break;                            \
    case 4: MEG_FIN2(jj, 4); break;                            \
    case 8: MEG_FIN2(jj, 8); break;                            \
    case 16: MEG_FIN2(jj, 16); break;                          \
    default: MEG_FIN2(jj, 24); break;                          \
  }
  MEG_J_DISPATCH(J, MEG_FIN)
#undef MEG_FIN
#undef MEG_FIN2
}

// ===========================================================================
// Rayleigh-Ritz + Ritz vectors + residuals (+ optional V_next Gram and MEG
// step epilogue) in one cooperative launch: CTA 0 runs the Jacobi
// eigensolver while the grid waits, then every CTA forms its rows of the
// Ritz block and the squared residuals.
template <int JG>
__global__ void __launch_bounds__(kCT, 1) k_coop_rr(const double* __restrict__ H, int64_t ldh, int m,
                                                   double* __restrict__ theta, double* __restrict__ S,
                                                   double* __restrict__ info, int64_t n, const double* __restrict__ Q,
                                                   const double* __restrict__ AQ, int64_t ldq, int rq, int nreq,
                                                   double* __restrict__ T, int64_t ldt, double* __restrict__ resid,
                                                   double* __restrict__ part, int gr, double* __restrict__ Gout,
                                                   double eps_next, double* __restrict__ epi,
                                                   double* __restrict__ V2, int64_t ld2, int r2) {
  extern __shared__ double sm[];
  cg::grid_group grid = cg::this_grid();
  phase_mark(10);
  // small Rayleigh-Ritz problems are solved here by CTA 0; large ones (m > 48)
  // arrive pre-solved from k_rr_wide (megb200_rr.cu, 1024 threads) -- flagged by info == nullptr
  const int cols = m;
  double* Ss = sm;
  double* Qs = sm + cols * rq;    // chunk rows of Q (kRC x cols)
  double* As = Qs + kRC * cols;   // chunk rows of AQ
  double* red = As + kRC * cols;  // kCT
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  // a CTA whose rows fit one chunk stages them while CTA 0 solves the Rayleigh-Ritz problem
  const bool prestaged = (r1 - r0) <= kRC && (blockIdx.x != 0 || !info);
  if (prestaged) {
    const int rows = (int)(r1 - r0);
#pragma unroll 1
    for (int idx = threadIdx.x; idx < rows * cols; idx += kCT) {
      const int r = idx / cols, k = idx - r * cols;
      Qs[idx] = Q[(r0 + r) * ldq + k];
      As[idx] = AQ[(r0 + r) * ldq + k];
    }
  }
  if (blockIdx.x == 0 && info) block_jacobi(H, ldh, m, theta, S, sm, info);
  phase_mark(11);
  grid.sync();
  phase_mark(12);
  #pragma unroll 1
  for (int idx = threadIdx.x; idx < cols * rq; idx += kCT) {
    const int k = idx / rq, c = idx - k * rq;
    Ss[idx] = S[k * m + c];
  }
  const int rpt = kCT / rq;
  const int c = threadIdx.x % rq;
  const int rofs = threadIdx.x / rq;
  const double th = (rofs < rpt && c < nreq) ? theta[c] : 0.0;
  double sq = 0.0;
  for (int64_t rc = r0; rc < r1; rc += kRC) {
    const int rows = (int)min((int64_t)kRC, r1 - rc);
    __syncthreads();
    if (!prestaged) {
      // stage the chunk's rows of Q and AQ with independent coalesced loads
#pragma unroll 1
      for (int idx = threadIdx.x; idx < rows * cols; idx += kCT) {
        const int r = idx / cols, k = idx - r * cols;
        Qs[idx] = Q[(rc + r) * ldq + k];
        As[idx] = AQ[(rc + r) * ldq + k];
      }
      __syncthreads();
    }
    if (rofs < rpt) {
      #pragma unroll 1
      for (int rr = rofs; rr < rows; rr += rpt) {
        const double* qr = Qs + rr * cols;
        double x0 = 0.0, x1 = 0.0;
        int k = 0;
        #pragma unroll 1
        for (; k + 1 < cols; k += 2) {
          x0 = fma(qr[k], Ss[k * rq + c], x0);
          x1 = fma(qr[k + 1], Ss[(k + 1) * rq + c], x1);
        }
        if (k < cols) x0 = fma(qr[k], Ss[k * rq + c], x0);
        const double x = x0 + x1;
        T[(rc + rr) * ldt + c] = x;
        if (c < r2) V2[(rc + rr) * ld2 + c] = x;
        if (c < nreq) {
          const double* ar = As + rr * cols;
          double a0 = 0.0, a1 = 0.0;
          k = 0;
          #pragma unroll 1
          for (; k + 1 < cols; k += 2) {
            a0 = fma(ar[k], Ss[k * rq + c], a0);
            a1 = fma(ar[k + 1], Ss[(k + 1) * rq + c], a1);
          }
          if (k < cols) a0 = fma(ar[k], Ss[k * rq + c], a0);
          const double d = (a0 + a1) - th * x;
          sq = fma(d, d, sq);
        }
      }
    }
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  double* rpart = part;                                   // G x nreq
  double* gpart = part + (int64_t)gridDim.x * nreq;       // G x gr*gr
  if (threadIdx.x < nreq) {
    double s2 = 0.0;
    #pragma unroll 1
    for (int t = threadIdx.x; t < rpt * rq; t += rq) s2 += red[t];
    rpart[(int64_t)blockIdx.x * nreq + threadIdx.x] = s2;
  }
  if (gr > 0) {
    __syncthreads();
    double acc[JG];
    xty_rows<JG>(r0, r1, T, ldt, gr, T, ldt, gr, red + kCT, acc);
    double* out = gpart + (int64_t)blockIdx.x * gr * gr;
#pragma unroll
    for (int j = 0; j < JG; ++j) {
      const int o = threadIdx.x + j * kCT;
      if (o < gr * gr) out[o] = acc[j];
    }
  }
  phase_mark(13);
  grid.sync();
  phase_mark(14);
  {
    // grid reduction of the residual squares and the Gram
    grid_reduce_outputs(
        nreq + gr * gr,
        [&](int o) { return o < nreq ? PartRef{rpart, nreq, o} : PartRef{gpart, gr * gr, o - nreq}; },
        [&](int o, double v) {
          if (o < nreq)
            resid[o] = sqrt(v);
          else
            Gout[o - nreq] = v;
        });
  }
  phase_mark(15);
  if (blockIdx.x == 0 && threadIdx.x < 32 && epi) {
    // step epilogue (meg.py:347-356) by one warp, lane k (and k + 32) owning pair k:
    // y = exp(mu - mu_1), lam = y[:r] / sum renormalised, lambda_{r+1}, b_{r+1}, cheap certificate
    const int lane = threadIdx.x;
    const int r = nreq - 1;
    const double shift = theta[0];
    double y[2], lam[2];
    double kept = 0.0, b = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = lane + 32 * h;
      y[h] = k <= r ? exp(theta[k] - shift) : 0.0;
      if (k <= r) epi[k] = y[h];
      kept += k < r ? y[h] : 0.0;
      b += y[h];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      kept += __shfl_xor_sync(0xffffffffu, kept, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    double lsum = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      lam[h] = (lane + 32 * h) < r ? y[h] / kept : 0.0;
      lsum += lam[h];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (lane + 32 * h < r) epi[r + 1 + lane + 32 * h] = lam[h] / lsum;
    // y_{r+1} from the lane that owns pair r (register shuffle: no read of another lane's store)
    const double lam_rp1 = __shfl_sync(0xffffffffu, (r >> 5) ? y[1] : y[0], r & 31);
    if (lane == 0) {
      double status = !(kept > 1e-290) ? 4.0 : 0.0;
      double lhs;
      if (!(b > 0.0) || lam_rp1 < 0.0) {
        status = 1.0;
        lhs = 0.0;
      } else if (lam_rp1 == 0.0) {
        lhs = -INFINITY;
      } else {
        lhs = log((double)(n - r) * lam_rp1 / (eps_next * b));
      }
      double* tail = epi + 2 * r + 1;
      tail[0] = lam_rp1;
      tail[1] = b;
      tail[2] = shift;
      tail[3] = lhs;
      tail[4] = (lhs <= 2.0 * eps_next) ? 1.0 : 0.0;
      tail[5] = 2.0 * eps_next;
      tail[6] = status;
    }
  }
}

void coop_rr(const Launch& L, const double* H, int64_t ldh, int m, double* theta, double* S, double* info, int64_t n,
             const double* Q, const double* AQ, int64_t ldq, int rq, int nreq, double* T, int64_t ldt, double* resid,
             double* part, int sm_count, int gr, double* Gout, double eps_next, double* epi, double* V2, int64_t ld2,
             int r2, int nvec, bool presolved) {
  if (!V2) r2 = 0;
  if (nreq > 64 || rq > 64) throw Error(MEGB200_ERR_PARAM, "rr: at most 64 Ritz vectors");
  const int G = coop_grid(n, sm_count);
  const bool fused = m <= 48;
  // presolved: the caller already ran the wide solver (on its side stream, overlapped)
  if (presolved && fused) throw Error(MEGB200_ERR_PARAM, "rr: presolved needs the wide solver (m > 48)");
  if (!fused && !presolved) rr_wide(L, H, ldh, m, theta, S, info, nvec > 0 ? std::max(nvec, rq) : 0);
  const size_t smem = std::max(fused ? (size_t)jacobi_smem_doubles(m) : (size_t)0,
                               (size_t)(m * rq + 2 * kRC * m + kCT + kRC * 2 * std::max(gr, 1))) * sizeof(double);
  double* info_arg = fused ? info : nullptr;
  const int JG = pick_j(std::max(1, gr * gr));
#define MEG_RR(jj)                                                                                              \
  {                                                                                                             \
    static char a = 0;                                                                                      \
    if (first_on_device(&a)) raise_smem(k_coop_rr<jj>, 215 * 1024);                                                \
    coop_launch(L, k_coop_rr<jj>, G, smem, H, ldh, m, theta, S, info_arg, n, Q, AQ, ldq, rq, nreq, T, ldt, resid, \
                part, gr, Gout, eps_next, epi, V2, ld2, r2);                                                    \
  }
  MEG_J_DISPATCH(JG, MEG_RR)
#undef MEG_RR
}

}  // namespace megb200

// Diagnostics: copy the phase timestamps of the last cooperative launches (-DMEG_PHASE_TIMING builds).
extern "C" int megb200_debug_phase_ns(unsigned long long* out, int count) {
  if (!out || count < 1 || count > 64) return MEGB200_ERR_PARAM;
  return cudaMemcpyFromSymbol(out, megb200::g_phase_ns, sizeof(unsigned long long) * count) == cudaSuccess
             ? MEGB200_OK
             : MEGB200_ERR_CUDA;
}
