// Quadratic-measurement objective (the paper's experiment; reference
// objectives.py:111-228): f(tau X) = 1/2 sum_i (a_i^T (tau X) b_i - y_i)^2 over
// m measurement pairs (a_i, b_i) of unit vectors in R^n.
//
//   k_qm_residuals   res_i = tau ((1 - eps) sum_k (a_i.v_k) lam_k (v_k.b_i)
//                              + tail (a_i.b_i - sum_k (a_i.v_k)(v_k.b_i))) - y_i
//                    (_measure_structured, objectives.py:111-118): a warp per
//                    measurement row, coalesced reads of a_i and b_i, fixed
//                    lane-strided sums + xor trees;
//   k_qm_grad_part   C_c = a[chunk]^T diag(res[chunk]) b[chunk] per m-chunk and
//                    64 x 64 output tile (split-K over the measurements, or over a
//                    mini-batch of measurement indices: StochasticOracle, :235-283);
//   k_qm_grad_reduce G = weight * (C + C^T) / 2, chunks summed in order
//                    (tau * _dense_measurement_gradient, objectives.py:155-156,
//                    the reference's own path for n <= dense_cap = 1024);
//   k_qm_sumsq       1/2 ||res||^2 (qm_value), one CTA, fixed order.
//
// The materialised gradient then drives the step through the dense operator
// pass like any fixed dense gradient.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "megb200_internal.h"

namespace megb200 {
namespace {

constexpr int kQmTile = 64;    // output tile of the gradient
constexpr int kQmSub = 32;     // measurement rows staged per sub-block
constexpr int kQmChunkMax = 512;  // measurement rows per split-K chunk (fewer when the grid would be small)

template <int RB>
__global__ void __launch_bounds__(256) k_qm_residuals(const double* __restrict__ a, const double* __restrict__ b,
                                                      const double* __restrict__ y, int64_t m, int64_t n,
                                                      const double* __restrict__ V, int64_t ldv, int r, QmCoef qc,
                                                      double* __restrict__ res) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= m) return;
  const double* ai = a + i * n;
  const double* bi = b + i * n;
  double av[RB], bv[RB], ab = 0.0;
#pragma unroll
  for (int k = 0; k < RB; ++k) av[k] = bv[k] = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    const double x = ai[j], z = bi[j];
    ab = fma(x, z, ab);
    const double* vj = V + j * ldv;
#pragma unroll
    for (int k = 0; k < RB; ++k) {
      if (k < r) {
        const double vk = __ldg(vj + k);
        av[k] = fma(x, vk, av[k]);
        bv[k] = fma(z, vk, bv[k]);
      }
    }
  }
  auto wsum = [](double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
  ab = wsum(ab);
  double kept = 0.0, cross = 0.0;
#pragma unroll
  for (int k = 0; k < RB; ++k) {
    if (k < r) {
      const double x = wsum(av[k]), z = wsum(bv[k]);
      kept = fma(x * qc.lam[k], z, kept);
      cross = fma(x, z, cross);
    }
  }
  if (lane == 0) res[i] = qc.tau * ((1.0 - qc.eps) * kept + qc.tail * (ab - cross)) - y[i];
}

// C_c[p][q] = sum_{l in chunk c} a[l][i0 + p] res[l] b[l][j0 + q]
// rows are the measurements idx[0 .. m) when idx is given (a mini-batch, with repeats), else 0 .. m.
// 64 x 64 output tile per CTA, a 4 x 4 register tile per thread (rows tp + 16 a, columns tq + 16 u):
// per staged measurement row a thread reads 4 + 4 shared values for 16 FMAs (conflict-free: the
// half-warps read the same 16 consecutive B values); each output sums its chunk's rows in order
__global__ void __launch_bounds__(256) k_qm_grad_part(const double* __restrict__ a, const double* __restrict__ b,
                                                      const double* __restrict__ res, int64_t m, int64_t n,
                                                      const int64_t* __restrict__ idx, int chunk,
                                                      double* __restrict__ part) {
  __shared__ double As[kQmSub][kQmTile + 1];
  __shared__ double Bs[kQmSub][kQmTile + 1];
  const int i0 = blockIdx.x * kQmTile, j0 = blockIdx.y * kQmTile;
  const int64_t l0 = (int64_t)blockIdx.z * chunk;
  const int64_t l1 = min(m, l0 + chunk);
  const int t = threadIdx.x;
  const int tp = t >> 4, tq = t & 15;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[x][u] = 0.0;
  for (int64_t ls = l0; ls < l1; ls += kQmSub) {
    const int rows = (int)min((int64_t)kQmSub, l1 - ls);
    __syncthreads();
    for (int e = t; e < kQmSub * kQmTile; e += 256) {
      const int rr = e / kQmTile, c = e % kQmTile;
      const bool ok = rr < rows;
      const int64_t l = ok ? (idx ? idx[ls + rr] : ls + rr) : 0;
      As[rr][c] = (ok && i0 + c < n) ? a[l * n + i0 + c] : 0.0;
      Bs[rr][c] = (ok && j0 + c < n) ? res[l] * b[l * n + j0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < kQmSub; ++rr) {
      double x[4], z[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x[k] = As[rr][tp + 16 * k];
        z[k] = Bs[rr][tq + 16 * k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[k][u] = fma(x[k], z[u], acc[k][u]);
    }
  }
  double* out = part + (int64_t)blockIdx.z * n * n;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = i0 + tp + 16 * k, q = j0 + tq + 16 * u;
      if (p < n && q < n) out[(int64_t)p * n + q] = acc[k][u];
    }
}

__global__ void k_qm_grad_reduce(const double* __restrict__ part, int chunks, int64_t n, double weight,
                                 double* __restrict__ G, int64_t ldg) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  const int64_t p = idx / n, q = idx - p * n;
  double s = 0.0, st = 0.0;
  for (int c = 0; c < chunks; ++c) {
    s += part[(int64_t)c * n * n + p * n + q];
    st += part[(int64_t)c * n * n + q * n + p];
  }
  G[p * ldg + q] = weight * 0.5 * (s + st);
}

__global__ void __launch_bounds__(1024) k_qm_sumsq(const double* __restrict__ res, int64_t m, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += 1024) s = fma(res[i], res[i], s);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 32; ++w) tot += red[w];
    *out = 0.5 * tot;
  }
}

// ---------------------------------------------------------------------------
// Matrix-free block application (reference _apply_measurement_gradient,
// objectives.py:152-158, the path RecoveryObjective takes above dense_cap, :214-221):
//     W = weight / 2 (a^T diag(res) (b U) + b^T diag(res) (a U)),  U n x k, k <= 32
// in two streaming passes over a and b (4 m n 8 bytes per application, like the
// reference's four products), never forming the n x n gradient:
//   k_qm_fwd   PQ[i] = res_i [b_i U | a_i U]  (m x 2 KB): a warp per MW measurements, lanes
//              stride the coalesced rows a_i, b_i; each lane's U row (KB doubles, L1/L2
//              resident) feeds 4 MW FMAs per load; fixed xor trees
//   k_qm_bwd   W_c[j] = sum_{i in chunk c} a_i[j] PQ[i][0:KB] + b_i[j] PQ[i][KB:2KB]: a thread
//              per two columns j (coalesced rows again), the chunk's PQ rows staged in shared
//              memory, split over (column block, measurement chunk)
//   k_qm_bwd_reduce  W = weight / 2 * sum_c W_c in chunk order (bitwise reproducible).
constexpr int kQmBwdRows = 64;    // measurements staged per round of k_qm_bwd
constexpr int kQmBwdCols = 512;   // columns per CTA of k_qm_bwd (two per thread)

template <int KB, int MW>
__global__ void __launch_bounds__(256) k_qm_fwd(const double* __restrict__ a, const double* __restrict__ b,
                                                const double* __restrict__ res, const int64_t* __restrict__ idx,
                                                int64_t m, int64_t n, const double* __restrict__ U, int64_t ldu,
                                                int k, double* __restrict__ PQ) {
  const int lane = threadIdx.x & 31;
  const int64_t i0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * MW;
  if (i0 >= m) return;
  double p[MW][KB], q[MW][KB];
#pragma unroll
  for (int w = 0; w < MW; ++w)
#pragma unroll
    for (int c = 0; c < KB; ++c) p[w][c] = q[w][c] = 0.0;
  const double* ar[MW];
  const double* br[MW];
  int64_t li[MW];  // measurement of batch position i0 + w
#pragma unroll
  for (int w = 0; w < MW; ++w) {
    const int64_t i = min(i0 + w, m - 1);
    li[w] = idx ? idx[i] : i;
    ar[w] = a + li[w] * n;
    br[w] = b + li[w] * n;
  }
  for (int64_t j = lane; j < n; j += 32) {
    double x[MW], z[MW];
#pragma unroll
    for (int w = 0; w < MW; ++w) {
      x[w] = __ldcs(ar[w] + j);  // streamed once per pass
      z[w] = __ldcs(br[w] + j);
    }
    const double* uj = U + j * ldu;
#pragma unroll
    for (int c = 0; c < KB; ++c) {
      if (c < k) {
        const double u = __ldg(uj + c);
#pragma unroll
        for (int w = 0; w < MW; ++w) {
          p[w][c] = fma(z[w], u, p[w][c]);  // b_i U
          q[w][c] = fma(x[w], u, q[w][c]);  // a_i U
        }
      }
    }
  }
#pragma unroll
  for (int w = 0; w < MW; ++w) {
    if (i0 + w < m) {
      const double rs = res[li[w]];
      double* out = PQ + (i0 + w) * (2 * KB);
#pragma unroll
      for (int c = 0; c < KB; ++c) {
        double pv = p[w][c], qv = q[w][c];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          pv += __shfl_xor_sync(0xffffffffu, pv, off);
          qv += __shfl_xor_sync(0xffffffffu, qv, off);
        }
        if (lane == 0) {
          out[c] = c < k ? rs * pv : 0.0;
          out[KB + c] = c < k ? rs * qv : 0.0;
        }
      }
    }
  }
}

template <int KB>
__global__ void __launch_bounds__(256) k_qm_bwd(const double* __restrict__ a, const double* __restrict__ b,
                                                const double* __restrict__ PQ, const int64_t* __restrict__ idx,
                                                int64_t m, int64_t n, int chunk, int k,
                                                double* __restrict__ part) {
  __shared__ double pq[kQmBwdRows][2 * KB];
  __shared__ int64_t lrow[kQmBwdRows];
  const int64_t j0 = (int64_t)blockIdx.x * kQmBwdCols + threadIdx.x;
  const int64_t j1 = j0 + 256;
  const int64_t l0 = (int64_t)blockIdx.y * chunk;
  const int64_t l1 = min(m, l0 + chunk);
  double w0[KB], w1[KB];
#pragma unroll
  for (int c = 0; c < KB; ++c) w0[c] = w1[c] = 0.0;
  const bool ok0 = j0 < n, ok1 = j1 < n;
  for (int64_t ls = l0; ls < l1; ls += kQmBwdRows) {
    const int rows = (int)min((int64_t)kQmBwdRows, l1 - ls);
    __syncthreads();
    for (int e = threadIdx.x; e < rows * 2 * KB; e += 256) (&pq[0][0])[e] = PQ[ls * (2 * KB) + e];
    if (threadIdx.x < rows) lrow[threadIdx.x] = idx ? idx[ls + threadIdx.x] : ls + threadIdx.x;
    __syncthreads();
#pragma unroll 2
    for (int rr = 0; rr < rows; ++rr) {
      const int64_t i = lrow[rr];
      const double x0 = ok0 ? __ldcs(a + i * n + j0) : 0.0, z0 = ok0 ? __ldcs(b + i * n + j0) : 0.0;
      const double x1 = ok1 ? __ldcs(a + i * n + j1) : 0.0, z1 = ok1 ? __ldcs(b + i * n + j1) : 0.0;
#pragma unroll
      for (int c = 0; c < KB; ++c) {
        const double pv = pq[rr][c], qv = pq[rr][KB + c];
        w0[c] = fma(x0, pv, w0[c]);
        w0[c] = fma(z0, qv, w0[c]);
        w1[c] = fma(x1, pv, w1[c]);
        w1[c] = fma(z1, qv, w1[c]);
      }
    }
  }
  double* out = part + (int64_t)blockIdx.y * n * k;
#pragma unroll
  for (int c = 0; c < KB; ++c) {
    if (c < k) {
      if (ok0) out[j0 * k + c] = w0[c];
      if (ok1) out[j1 * k + c] = w1[c];
    }
  }
}

__global__ void k_qm_bwd_reduce(const double* __restrict__ part, int chunks, int64_t nk, double weight,
                                double* __restrict__ W) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nk) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(int64_t)c * nk + idx];
  W[idx] = 0.5 * weight * s;
}

}  // namespace

// split of the backward pass: measurement chunks so that (column blocks x chunks) covers ~2 waves
int qm_apply_chunk(int64_t m, int64_t n, int sm_count) {
  const int64_t cb = (n + kQmBwdCols - 1) / kQmBwdCols;
  int64_t chunks = std::max<int64_t>(1, (2 * (int64_t)sm_count + cb - 1) / cb);
  int64_t chunk = (m + chunks - 1) / chunks;
  chunk = ((chunk + kQmBwdRows - 1) / kQmBwdRows) * kQmBwdRows;
  return (int)std::max<int64_t>(kQmBwdRows, chunk);
}

int qm_apply_kb(int k) { return k <= 8 ? 8 : (k <= 16 ? 16 : 32); }

// scratch: PQ (m x 2 KB) followed by the chunk partials (chunks x n x k)
int64_t qm_apply_scratch_doubles(int64_t m, int64_t n, int k, int sm_count) {
  const int chunk = qm_apply_chunk(m, n, sm_count);
  return m * 2 * qm_apply_kb(k) + ((m + chunk - 1) / chunk) * n * k;
}

void qm_apply(const Launch& L, const double* a, const double* b, const double* res, const int64_t* idx, int64_t m,
              int64_t n, double weight, const double* U, int64_t ldu, int k, double* W, double* scratch, int sm_count) {
  if (k < 1 || k > 32) throw Error(MEGB200_ERR_PARAM, "quadratic-measurement block application supports 1 <= k <= 32");
  const int KB = qm_apply_kb(k);
  double* PQ = scratch;
  double* part = scratch + m * 2 * KB;
  const int chunk = qm_apply_chunk(m, n, sm_count);
  const int chunks = (int)((m + chunk - 1) / chunk);
  const dim3 gb((unsigned)((n + kQmBwdCols - 1) / kQmBwdCols), (unsigned)chunks);
  if (KB == 8) {
    k_qm_fwd<8, 2><<<(unsigned)((m + 15) / 16), 256, 0, L.stream>>>(a, b, res, idx, m, n, U, ldu, k, PQ);
    MEG_LAUNCHED();
    k_qm_bwd<8><<<gb, 256, 0, L.stream>>>(a, b, PQ, idx, m, n, chunk, k, part);
  } else if (KB == 16) {
    k_qm_fwd<16, 2><<<(unsigned)((m + 15) / 16), 256, 0, L.stream>>>(a, b, res, idx, m, n, U, ldu, k, PQ);
    MEG_LAUNCHED();
    k_qm_bwd<16><<<gb, 256, 0, L.stream>>>(a, b, PQ, idx, m, n, chunk, k, part);
  } else {
    k_qm_fwd<32, 1><<<(unsigned)((m + 7) / 8), 256, 0, L.stream>>>(a, b, res, idx, m, n, U, ldu, k, PQ);
    MEG_LAUNCHED();
    k_qm_bwd<32><<<gb, 256, 0, L.stream>>>(a, b, PQ, idx, m, n, chunk, k, part);
  }
  MEG_LAUNCHED();
  k_qm_bwd_reduce<<<(unsigned)((n * k + 255) / 256), 256, 0, L.stream>>>(part, chunks, n * k, weight, W);
  MEG_LAUNCHED();
  *L.counter += 3;
}

void qm_residuals(const Launch& L, const double* a, const double* b, const double* y, int64_t m, int64_t n,
                  const double* V, int64_t ldv, int r, const QmCoef& qc, double* res) {
  if (r < 1 || r > 32) throw Error(MEGB200_ERR_PARAM, "quadratic-measurement residuals support 1 <= r <= 32");
  const unsigned grid = (unsigned)((m + 7) / 8);
  if (r <= 8)
    k_qm_residuals<8><<<grid, 256, 0, L.stream>>>(a, b, y, m, n, V, ldv, r, qc, res);
  else if (r <= 16)
    k_qm_residuals<16><<<grid, 256, 0, L.stream>>>(a, b, y, m, n, V, ldv, r, qc, res);
  else
    k_qm_residuals<32><<<grid, 256, 0, L.stream>>>(a, b, y, m, n, V, ldv, r, qc, res);
  MEG_LAUNCHED();
  ++*L.counter;
}

// split-K chunk: 512 measurements, halved (down to 64) until the grid covers ~2 waves of 148 SMs
int qm_chunk(int64_t m, int64_t n) {
  const int64_t tiles = ((n + kQmTile - 1) / kQmTile) * ((n + kQmTile - 1) / kQmTile);
  int chunk = kQmChunkMax;
  while (chunk > 64 && tiles * ((m + chunk - 1) / chunk) < 296) chunk /= 2;
  return chunk;
}

int64_t qm_grad_part_doubles(int64_t m, int64_t n) {
  const int chunk = qm_chunk(m, n);
  return ((m + chunk - 1) / chunk) * n * n;
}

void qm_gradient(const Launch& L, const double* a, const double* b, const double* res, int64_t m, int64_t n,
                 double weight, double* G, int64_t ldg, double* part, const int64_t* idx) {
  const int chunk = qm_chunk(m, n);
  const int chunks = (int)((m + chunk - 1) / chunk);
  const dim3 grid((unsigned)((n + kQmTile - 1) / kQmTile), (unsigned)((n + kQmTile - 1) / kQmTile), (unsigned)chunks);
  k_qm_grad_part<<<grid, 256, 0, L.stream>>>(a, b, res, m, n, idx, chunk, part);
  MEG_LAUNCHED();
  k_qm_grad_reduce<<<(unsigned)((n * n + 255) / 256), 256, 0, L.stream>>>(part, chunks, n, weight, G, ldg);
  MEG_LAUNCHED();
  *L.counter += 2;
}

void qm_sumsq(const Launch& L, const double* res, int64_t m, double* out) {
  k_qm_sumsq<<<1, 1024, 0, L.stream>>>(res, m, out);
  MEG_LAUNCHED();
  ++*L.counter;
}

}  // namespace megb200
