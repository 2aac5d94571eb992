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
namespace {

constexpr int kCT = 256;     // threads per CTA
constexpr int kRC = 32;      // rows staged per chunk
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
                                         double (&acc)[J]) {
  double* Xs = sm;
  double* Ys = sm + kRC * p;
  const int pq = p * q;
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
    for (int idx = threadIdx.x; idx < rows * p; idx += kCT) {
      const int r = idx / p, a = idx - r * p;
      Xs[idx] = X[(rc + r) * ldx + a];
    }
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      Ys[idx] = Y[(rc + r) * ldy + c];
    }
    __syncthreads();
    for (int r = 0; r < rows; ++r) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(Xs[r * p + oa[j]], Ys[r * q + oc[j]], acc[j]);
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

// distributed final reduction: CTA g handles outputs o = g*kCT + tid + k*G*kCT
__device__ __forceinline__ void reduce_partials(const double* __restrict__ part, int pq, int q,
                                                double* __restrict__ C, int64_t ldc,
                                                const double* __restrict__ rowscale, double scale) {
  const int G = gridDim.x;
  for (int o = blockIdx.x * kCT + threadIdx.x; o < pq; o += G * kCT) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += part[(int64_t)g * pq + o];
    const int a = o / q, c = o - a * q;
    if (rowscale) s *= rowscale[a];
    C[(int64_t)a * ldc + c] = scale * s;
  }
}

// ---------------------------------------------------------------------------
// Cholesky of a q x q SPD Gram (q <= 64) in one warp, column-equilibrated,
// breakdown (pivot <= thresh^2 absolute or 1e-20 relative) -> flagged column.
// Writes Rrel (zero rows for flagged columns), Rinv, mask; optionally
// Rtot = Rrel * Rprev.
__device__ void warp_cholesky(const double* __restrict__ Gg, int q, double thresh, double* sm,
                              double* __restrict__ Rrel, double* __restrict__ Rinv, int* __restrict__ mask,
                              const double* __restrict__ Rprev, double* __restrict__ Rtot) {
  const int lane = threadIdx.x & 31;
  const int ld = q + 1;
  double* A = sm;            // q x ld
  double* R = sm + q * ld;   // q x ld
  double* D = R + q * ld;    // q
  int* bad = reinterpret_cast<int*>(D + q);
  for (int idx = lane; idx < q * q; idx += 32) {
    const int i = idx / q, j = idx - i * q;
    A[i * ld + j] = Gg[(i <= j) ? i * q + j : j * q + i];
    R[i * ld + j] = 0.0;
  }
  __syncwarp();
  for (int t = lane; t < q; t += 32) {
    const double g = A[t * ld + t];
    bad[t] = !(g > thresh * thresh);
    D[t] = bad[t] ? 1.0 : sqrt(g);
  }
  __syncwarp();
  for (int idx = lane; idx < q * q; idx += 32) {
    const int i = idx / q, j = idx - i * q;
    A[i * ld + j] = (bad[i] || bad[j]) ? (i == j ? 1.0 : 0.0) : A[i * ld + j] / (D[i] * D[j]);
  }
  __syncwarp();
  for (int j = 0; j < q; ++j) {
    const double d = A[j * ld + j];
    const bool bj = bad[j] || !(d > 1e-20);
    const double rjj = bj ? 1.0 : sqrt(d);
    __syncwarp();
    if (lane == 0) {
      bad[j] = bj;
      R[j * ld + j] = rjj;
    }
    for (int k = j + 1 + lane; k < q; k += 32) R[j * ld + k] = bj ? 0.0 : A[j * ld + k] / rjj;
    __syncwarp();
    const int m = q - j - 1;
    for (int idx = lane; idx < m * m; idx += 32) {
      const int k = j + 1 + idx / m, l = j + 1 + idx % m;
      A[k * ld + l] -= R[j * ld + k] * R[j * ld + l];
    }
    __syncwarp();
  }
  // Rinv = D^-1 Rs^-1 : lane c owns column c (q <= 64 -> two passes)
  for (int c = lane; c < q; c += 32) {
    double x[64];
    x[c] = 1.0 / R[c * ld + c];
    for (int i = c - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= c; ++k) s += R[i * ld + k] * x[k];
      x[i] = -s / R[i * ld + i];
    }
    for (int i = 0; i < q; ++i) Rinv[i * q + c] = (i <= c) ? x[i] / D[i] : 0.0;
  }
  for (int idx = lane; idx < q * q; idx += 32) {
    const int i = idx / q, j = idx - i * q;
    Rrel[idx] = (bad[i] || j < i) ? 0.0 : R[i * ld + j] * D[j];
  }
  for (int t = lane; t < q; t += 32) mask[t] = bad[t];
  __syncwarp();
  if (Rtot) {
    for (int idx = lane; idx < q * q; idx += 32) {
      const int i = idx / q, j = idx - i * q;
      double s = 0.0;
      if (!bad[i])
        for (int k = i; k < q; ++k) s += R[i * ld + k] * D[k] * Rprev[k * q + j];
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
  for (int idx = threadIdx.x; idx < cols * q; idx += kCT) Cs[idx] = Cws[idx];
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (r1 - r0) * q; idx += kCT) {
    const int64_t r = r0 + idx / q;
    const int c = (int)(idx % q);
    const double* qr = Q + r * ldq;
    double s = 0.0;
    for (int k = 0; k < cols; ++k) s = fma(qr[k], Cs[k * q + c], s);
    W[r * ldw + c] -= s;
  }
}

// One CholQR round: G = W^T W, R = chol(G) (CTA 0, one warp), W = W R^-1 with
// breakdown columns replaced by seeded random normals.
template <int J>
__global__ void __launch_bounds__(kCT) k_coop_cholqr(int64_t n, double* __restrict__ W, int64_t ldw, int q,
                                                      double thresh, double* __restrict__ Gws,
                                                      double* __restrict__ Rrel, double* __restrict__ Rinv,
                                                      int* __restrict__ mask, const double* __restrict__ Rprev,
                                                      double* __restrict__ Rtot, uint64_t key, uint64_t base,
                                                      double* __restrict__ part) {
  extern __shared__ double sm[];
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  double acc[J];
  xty_rows<J>(r0, r1, W, ldw, q, W, ldw, q, sm, acc);
  store_partial<J>(part, q * q, acc);
  cg::grid_group grid = cg::this_grid();
  grid.sync();
  reduce_partials(part, q * q, q, Gws, q, nullptr, 1.0);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x < 32) warp_cholesky(Gws, q, thresh, sm, Rrel, Rinv, mask, Rprev, Rtot);
  grid.sync();
  double* Ri = sm;
  int* bad = reinterpret_cast<int*>(sm + q * q);
  for (int idx = threadIdx.x; idx < q * q; idx += kCT) Ri[idx] = Rinv[idx];
  for (int idx = threadIdx.x; idx < q; idx += kCT) bad[idx] = mask[idx];
  __syncthreads();
  // rows of this CTA: W[r, :] <- W[r, :] Rinv  (row staged in registers through shared memory)
  double* Ws = sm + q * q + 64;
  for (int64_t rc = r0; rc < r1; rc += kRC) {
    const int rows = (int)min((int64_t)kRC, r1 - rc);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      Ws[idx] = W[(rc + r) * ldw + c];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * q; idx += kCT) {
      const int r = idx / q, c = idx - r * q;
      double v;
      if (bad[c]) {
        v = gauss_c(key, base + (uint64_t)(rc + r) * q + c);
      } else {
        v = 0.0;
        for (int k = 0; k <= c; ++k) v = fma(Ws[r * q + k], Ri[k * q + c], v);
      }
      W[(rc + r) * ldw + c] = v;
    }
  }
}

// Ritz vectors and residuals: T[:, 0:rq] = Q S[:, 0:rq]; AX = AQ S[:, 0:nreq];
// resid[j] = ||AX_j - theta_j X_j|| (j < nreq).  S is cols x ldS row-major.
// Thread t owns column c = t % rq of rows t / rq, t / rq + rpt, ... so each
// thread accumulates one column's squared residual in a register.
__global__ void __launch_bounds__(kCT) k_coop_ritz(int64_t n, const double* __restrict__ Q,
                                                   const double* __restrict__ AQ, int64_t ldq, int cols,
                                                   const double* __restrict__ S, int ldS, int rq, int nreq,
                                                   const double* __restrict__ theta, double* __restrict__ T,
                                                   int64_t ldt, double* __restrict__ resid,
                                                   double* __restrict__ part) {
  extern __shared__ double sm[];
  double* Ss = sm;               // cols x rq
  double* red = sm + cols * rq;  // kCT
  for (int idx = threadIdx.x; idx < cols * rq; idx += kCT) {
    const int k = idx / rq, c = idx - k * rq;
    Ss[idx] = S[k * ldS + c];
  }
  __syncthreads();
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  const int rpt = kCT / rq;  // rows in flight per sweep
  const int c = threadIdx.x % rq;
  const int rofs = threadIdx.x / rq;
  double sq = 0.0;
  if (rofs < rpt) {
    const double th = c < nreq ? theta[c] : 0.0;
    for (int64_t r = r0 + rofs; r < r1; r += rpt) {
      const double* qr = Q + r * ldq;
      double x = 0.0;
      for (int k = 0; k < cols; ++k) x = fma(qr[k], Ss[k * rq + c], x);
      T[r * ldt + c] = x;
      if (c < nreq) {
        const double* ar = AQ + r * ldq;
        double ax = 0.0;
        for (int k = 0; k < cols; ++k) ax = fma(ar[k], Ss[k * rq + c], ax);
        const double d = ax - th * x;
        sq = fma(d, d, sq);
      }
    }
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  if (threadIdx.x < nreq) {
    double s = 0.0;
    for (int t = threadIdx.x; t < rpt * rq; t += rq) s += red[t];
    part[(int64_t)blockIdx.x * nreq + threadIdx.x] = s;
  }
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x < nreq) {
    double s = 0.0;
    for (int g = 0; g < (int)gridDim.x; ++g) s += part[(int64_t)g * nreq + threadIdx.x];
    resid[threadIdx.x] = sqrt(s);
  }
}

// Operator epilogue: E = diag(d) L^T U (reduced across the grid), then
// W = scale * sum_s part[s] + L E + alpha U.
template <int J>
__global__ void __launch_bounds__(kCT) k_coop_finish(int64_t n, int b, int S, const double* __restrict__ spart,
                                                      double scale, const double* __restrict__ Lf, int64_t ldl, int l,
                                                      const double* __restrict__ d, double alpha,
                                                      const double* __restrict__ U, int64_t ldu,
                                                      double* __restrict__ W, int64_t ldw, double* __restrict__ Ews,
                                                      double* __restrict__ part) {
  extern __shared__ double sm[];
  int64_t r0, r1;
  cta_rows(n, r0, r1);
  if (l > 0) {
    double acc[J];
    xty_rows<J>(r0, r1, Lf, ldl, l, U, ldu, b, sm, acc);
    store_partial<J>(part, l * b, acc);
    cg::grid_group grid = cg::this_grid();
    grid.sync();
    reduce_partials(part, l * b, b, Ews, b, d, 1.0);
    grid.sync();
  }
  double* Es = sm;
  for (int idx = threadIdx.x; idx < l * b; idx += kCT) Es[idx] = Ews[idx];
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (r1 - r0) * b; idx += kCT) {
    const int64_t i = r0 + idx / b;
    const int c = (int)(idx % b);
    double s = 0.0;
    for (int t = 0; t < S; ++t) s += spart[(int64_t)t * n * b + i * b + c];
    double v = scale * s + alpha * U[i * ldu + c];
    const double* Lr = Lf + i * ldl;
    for (int k = 0; k < l; ++k) v = fma(Lr[k], Es[k * b + c], v);
    W[i * ldw + c] = v;
  }
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
    static bool a = false;                                                                              \
    if (!a) { raise_smem(k_coop_tn<jj>, kCoopSmem); a = true; }                                         \
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
    static bool a = false;                                                                       \
    if (!a) { raise_smem(k_coop_cgs<jj>, kCoopSmem); a = true; }                                 \
    coop_launch(L, k_coop_cgs<jj>, G, smem, n, Q, ldq, cols, W, ldw, q, Cws, part);              \
  }
  MEG_J_DISPATCH(J, MEG_CGS)
#undef MEG_CGS
}

void coop_cholqr(const Launch& L, int64_t n, double* W, int64_t ldw, int q, double thresh, double* Gws, double* Rrel,
                 double* Rinv, int* mask, const double* Rprev, double* Rtot, uint64_t key, uint64_t base, double* part,
                 int sm_count) {
  const int G = coop_grid(n, sm_count);
  const size_t chol_smem = (size_t)(2 * q * (q + 1) + q + 1) * sizeof(double) + 64 * sizeof(int);
  const size_t smem = std::max({(size_t)kRC * 2 * q * sizeof(double), chol_smem,
                                (size_t)(q * q + 64 + kRC * q) * sizeof(double)});
  const int J = pick_j(q * q);
#define MEG_CQR(jj)                                                                                          \
  {                                                                                                          \
    static bool a = false;                                                                                   \
    if (!a) { raise_smem(k_coop_cholqr<jj>, kCoopSmem); a = true; }                                          \
    coop_launch(L, k_coop_cholqr<jj>, G, smem, n, W, ldw, q, thresh, Gws, Rrel, Rinv, mask, Rprev, Rtot, key, \
                base, part);                                                                                 \
  }
  MEG_J_DISPATCH(J, MEG_CQR)
#undef MEG_CQR
}

void coop_ritz(const Launch& L, int64_t n, const double* Q, const double* AQ, int64_t ldq, int cols, const double* S,
               int ldS, int rq, int nreq, const double* theta, double* T, int64_t ldt, double* resid, double* part,
               int sm_count) {
  if (nreq > 64 || rq > 64) throw Error(MEGB200_ERR_PARAM, "ritz: at most 64 vectors");
  const int G = coop_grid(n, sm_count);
  const size_t smem = (size_t)(cols * rq + kCT) * sizeof(double);
  static bool a = false;
  if (!a) {
    raise_smem(k_coop_ritz, kCoopSmem);
    a = true;
  }
  coop_launch(L, k_coop_ritz, G, smem, n, Q, AQ, ldq, cols, S, ldS, rq, nreq, theta, T, ldt, resid, part);
}

void coop_finish(const Launch& L, int64_t n, int b, int S, const double* spart, double scale, const double* Lf,
                 int64_t ldl, int l, const double* d, double alpha, const double* U, int64_t ldu, double* W,
                 int64_t ldw, double* Ews, double* part, int sm_count) {
  const int G = coop_grid(n, sm_count);
  const size_t smem = std::max((size_t)kRC * (l + b), (size_t)std::max(1, l * b)) * sizeof(double);
  const int J = pick_j(std::max(1, l * b));
#define MEG_FIN(jj)                                                                                            \
  {                                                                                                            \
    static bool a = false;                                                                                     \
    if (!a) { raise_smem(k_coop_finish<jj>, kCoopSmem); a = true; }                                            \
    coop_launch(L, k_coop_finish<jj>, G, smem, n, b, S, spart, scale, Lf, ldl, l, d, alpha, U, ldu, W, ldw, Ews, \
                part);                                                                                         \
  }
  MEG_J_DISPATCH(J, MEG_FIN)
#undef MEG_FIN
}

}  // namespace megb200
