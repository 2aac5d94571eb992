// Device pieces shared by the kernels that finish a block pass on the device (the fused
// first pass, megb200_step.cu, and the fused pass + step tail, megb200_kernels.cu): the
// near-diagonal Rayleigh-Ritz solve, the step epilogue, the fixed-order row dot products and
// the release / acquire flag primitives.  Include after megb200_jacobi.cuh.
#pragma once

namespace megb200 {
namespace {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// Near-diagonal Rayleigh-Ritz for m <= 32 (the warm-started first pass) by the whole
// CTA with few barriers: up to three first-order Jacobi pre-steps, the scheme of
// block_jacobi (megb200_jacobi.cuh): Y = I + X, X_ij = h_ij / (h_jj - h_ii) (pairs with
// |h_ij| > 0.1 |gap| excluded), one Newton-Schulz step Z = Y (3I - Y^T Y) / 2 when
// |X| >= 1e-8, H <- Z^T H Z, V <- V Z.  Same stopping rule (off(H) <= 1e-15 ||H||_F).
// Returns false, having written nothing, when the rule is not met (H not near-diagonal
// or the pre-steps stagnate): the caller then runs the sweeping block_jacobi.
// Outputs: theta (non-increasing, stable by index) to theta_g and ths (shared), S to Sout
// (m x m row-major, column j = eigenvector j).  sm: 5 m^2 + 128 doubles.
template <int NT>
__device__ bool rr_small_neardiag(const double* __restrict__ Hg, int64_t ldh, int m, double* __restrict__ theta_g,
                                  double* __restrict__ Sout, double* sm, double* ths, double* __restrict__ info) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int mm = m * m;
  double* H = sm;
  double* V = H + mm;
  double* Y = V + mm;
  double* Tm = Y + mm;
  double* Z = Tm + mm;
  double* wred = Z + mm;          // 3 x 32 warp partials
  int* rk = reinterpret_cast<int*>(wred + 96);  // ranks (m ints)
  auto warp_sum = [](double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
  double f = 0.0, o = 0.0;
  for (int idx = t; idx < mm; idx += NT) {
    const int i = idx / m, j = idx - i * m;
    const double h = i <= j ? Hg[i * ldh + j] : Hg[j * ldh + i];
    H[idx] = h;
    V[idx] = i == j ? 1.0 : 0.0;
    f += h * h;
    if (i != j) o += h * h;
  }
  f = warp_sum(f);
  o = warp_sum(o);
  if (lane == 0) {
    wred[w] = f;
    wred[32 + w] = o;
  }
  __syncthreads();
  double fro2 = 0.0, off2 = 0.0;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) {
    fro2 += wred[k];
    off2 += wred[32 + k];
  }
  const double stop2 = fro2 * 1e-30;
  bool done = off2 <= stop2;
  if (!done && !(off2 <= 1e-6 * fro2)) return false;
  int npre = 0, nns = 0;  // diagnostics: pre-steps and Newton-Schulz steps taken
  for (int pre = 0; pre < 3 && !done; ++pre) {
    ++npre;
    // Y = I + X
    double xm = 0.0;
    for (int idx = t; idx < mm; idx += NT) {
      const int i = idx / m, j = idx - i * m;
      double y = 1.0;
      if (i != j) {
        const double h = H[idx], d = H[j * m + j] - H[i * m + i];
        y = (h != 0.0 && fabs(h) <= 0.1 * fabs(d)) ? h / d : 0.0;
        xm = fmax(xm, fabs(y));
      }
      Y[idx] = y;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) xm = fmax(xm, __shfl_xor_sync(0xffffffffu, xm, off));
    if (lane == 0) wred[64 + w] = xm;
    __syncthreads();
    double xmax = 0.0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) xmax = fmax(xmax, wred[64 + k]);
    double* Zp = Y;
    if (xmax >= 1e-8) {
      ++nns;
      // Newton-Schulz: Tm = (3I - Y^T Y) / 2, Z = Y Tm
      for (int idx = t; idx < mm; idx += NT) {
        const int i = idx / m, j = idx - i * m;
        Tm[idx] = 0.5 * ((i == j ? 3.0 : 0.0) - jdot(Y, i, m, Y, j, m, m));
      }
      __syncthreads();
      for (int idx = t; idx < mm; idx += NT) {
        const int i = idx / m, j = idx - i * m;
        Z[idx] = jdot(Y, i * m, 1, Tm, j, m, m);
      }
      __syncthreads();
      Zp = Z;
    }
    double* Vn = (Zp == Y) ? Z : Y;
    // Tm = H Zp, Vn = V Zp (V is still the identity in the first pre-step: Vn = Zp)
    for (int idx = t; idx < mm; idx += NT) {
      const int i = idx / m, j = idx - i * m;
      Tm[idx] = jdot(H, i * m, 1, Zp, j, m, m);
      Vn[idx] = pre == 0 ? Zp[idx] : jdot(V, i * m, 1, Zp, j, m, m);
    }
    __syncthreads();
    // H <- Zp^T Tm (upper triangle, mirrored)
    double lo = 0.0;
    for (int idx = t; idx < mm; idx += NT) {
      const int i = idx / m, j = idx - i * m;
      if (i <= j) {
        const double v = jdot(Zp, i, m, Tm, j, m, m);
        H[i * m + j] = v;
        H[j * m + i] = v;
        if (i != j) lo += 2.0 * v * v;
      }
    }
    lo = warp_sum(lo);
    if (lane == 0) wred[32 + w] = lo;
    // V <- Vn (pointer swap: the old V buffer becomes scratch)
    double* oldV = V;
    V = Vn;
    if (Vn == Y) Y = oldV;
    else Z = oldV;
    __syncthreads();
    const double prev = off2;
    off2 = 0.0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) off2 += wred[32 + k];
    done = off2 <= stop2;
    if (!done && !(off2 < 0.25 * prev)) return false;
  }
  if (!done) return false;
  // theta non-increasing, stable by index; S columns follow
  for (int i = t; i < m; i += NT) {
    const double di = H[i * m + i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = H[j * m + j];
      rank += (dj > di) || (dj == di && j < i);
    }
    rk[i] = rank;
    ths[rank] = di;
    theta_g[rank] = di;
  }
  __syncthreads();
  for (int idx = t; idx < mm; idx += NT) {
    const int k = idx / m, i = idx - k * m;
    Sout[k * m + rk[i]] = V[idx];
  }
  if (t == 0 && info) {
    info[0] = -(double)(npre + 10 * nns);  // fast path: -(pre-steps + 10 x Newton-Schulz steps)
    info[1] = sqrt(off2);
    info[2] = sqrt(fro2);
  }
  __syncthreads();
  return true;
}

// the sweeping Jacobi is a rare fallback here: kept out of line so the fused kernel's hot path
// stays small in the instruction cache
__device__ __noinline__ void jacobi_fallback(const double* H, int m, double* theta, double* S, double* sm,
                                             double* info) {
  block_jacobi(H, m, m, theta, S, sm, info);
}


// Step epilogue (meg.py:347-356) by one warp (lanes 0..31 of the calling CTA), lane k (and k + 32)
// owning pair k: y = exp(mu - mu_1), lam = y[:r] / sum renormalised, lambda_{r+1}, b_{r+1}, cheap
// certificate (meg.py:222-239); epi = [y (r+1) | lam (r) | lambda_{r+1}, b_{r+1}, shift, lhs, holds,
// threshold, status].  theta: the nreq = r + 1 Ritz values, non-increasing.
__device__ __forceinline__ void step_epilogue_warp(const double* theta, int nreq, int64_t n, double eps_next,
                                                   double* epi) {
  const int lane = threadIdx.x & 31;
  const int r = nreq - 1;
  const double shift = theta[0];
  double y[2], lam[2];
  double kept = 0.0, bsum = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = lane + 32 * h;
    y[h] = k <= r ? exp(theta[k] - shift) : 0.0;
    if (k <= r) epi[k] = y[h];
    kept += k < r ? y[h] : 0.0;
    bsum += y[h];
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    kept += __shfl_xor_sync(0xffffffffu, kept, off);
    bsum += __shfl_xor_sync(0xffffffffu, bsum, off);
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
  // y_{r+1} from the lane that owns pair r
  const double lam_rp1 = __shfl_sync(0xffffffffu, (r >> 5) ? y[1] : y[0], r & 31);
  if (lane == 0) {
    double status = !(kept > 1e-290) ? 4.0 : 0.0;
    double lhs;
    if (!(bsum > 0.0) || lam_rp1 < 0.0) {
      status = 1.0;
      lhs = 0.0;
    } else if (lam_rp1 == 0.0) {
      lhs = -INFINITY;
    } else {
      lhs = log((double)(n - r) * lam_rp1 / (eps_next * bsum));
    }
    double* tail = epi + 2 * r + 1;
    tail[0] = lam_rp1;
    tail[1] = bsum;
    tail[2] = shift;
    tail[3] = lhs;
    tail[4] = (lhs <= 2.0 * eps_next) ? 1.0 : 0.0;
    tail[5] = 2.0 * eps_next;
    tail[6] = status;
  }
}

// sum over rows of X[row, a] * Y[row, c]: rows r = 4q + j accumulate in chain j, the four chains
// added as (0 + 1) + (2 + 3).  The one product order of every Gram-type partial that must reproduce
// bit for bit in another kernel (L^T U of a step's start block == rows of the previous step's
// Ritz-block Gram, k_tile_gram vs k_dense_step_mma)
__device__ __forceinline__ double tile_dot(const double* X, int ldx, int a, const double* Y, int ldy, int c,
                                           int rows) {
  double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
  int r = 0;
#pragma unroll 2
  for (; r + 3 < rows; r += 4) {
    e0 = fma(X[r * ldx + a], Y[r * ldy + c], e0);
    e1 = fma(X[(r + 1) * ldx + a], Y[(r + 1) * ldy + c], e1);
    e2 = fma(X[(r + 2) * ldx + a], Y[(r + 2) * ldy + c], e2);
    e3 = fma(X[(r + 3) * ldx + a], Y[(r + 3) * ldy + c], e3);
  }
  for (; r < rows; ++r) e0 = fma(X[r * ldx + a], Y[r * ldy + c], e0);
  return (e0 + e1) + (e2 + e3);
}

// sum_{t < cnt} part[t * stride + o] in index order (the one association every caller reproduces),
// the loads issued B at a time before they are added
template <int B = 8>
__device__ __forceinline__ double tile_ordered_sum(const double* part, int cnt, int64_t stride, int o) {
  double s = 0.0;
  for (int j0 = 0; j0 < cnt; j0 += B) {
    double v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) v[j] = j0 + j < cnt ? __ldcg(part + (int64_t)(j0 + j) * stride + o) : 0.0;
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (j0 + j < cnt) s += v[j];
  }
  return s;
}

}  // namespace
}  // namespace megb200
