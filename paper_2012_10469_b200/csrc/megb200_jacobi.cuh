// K6: Rayleigh-Ritz eigensolver for the small projected matrix H (m <= 112):
// parallel cyclic Jacobi with round-robin pair ordering, run by one CTA with
// H and the accumulated rotations in shared memory (float64).  Each round
// applies m/2 disjoint rotations J^T H J as independent 2x2 block updates, so
// a round costs two __syncthreads; sweeps stop when off(H) <= 1e-15 ||H||_F or
// stagnates.  Output: theta non-increasing (stable by index), S (m x m
// row-major, column j = eigenvector j).
//
// Near-diagonal pre-step (m <= 64, off(H) <= 1e-3 ||H||_F -- the Rayleigh-Ritz
// matrix of a warm-started step): all pair rotations at once to first order,
// Y = I + X with X_ij = h_ij / (h_jj - h_ii) (pairs with |h_ij| > 0.1 |gap|
// are left to the sweeps), orthonormalised by one Newton-Schulz step
// S = Y (3I - Y^T Y) / 2 (orthogonal to O(|X|^4)), and H <- S^T H S, V <- V S.
// Each pre-step takes off(H) to O(off^2 / gap); up to three run while they
// keep converging, after which the sweeps (same rule, same outputs) usually
// have nothing left to do, so a warm step's Rayleigh-Ritz costs a few
// parallel m x m products instead of a sweep of m - 1 serialised rounds.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#ifndef JACOBI_MARK
#define JACOBI_MARK(slot)
#endif

namespace megb200 {

__host__ __device__ constexpr int jacobi_pad(int m) { return (m + 1) & ~1; }
// shared-memory doubles needed by block_jacobi for size m
__host__ __device__ constexpr int jacobi_base_doubles(int m) { return 2 * jacobi_pad(m) * jacobi_pad(m) + 64 * 4 + 40; }
constexpr int kJacobiPreMax = 64;  // largest m with the near-diagonal pre-step (third m x m buffer)
__host__ __device__ constexpr int jacobi_smem_doubles(int m) {
  return jacobi_base_doubles(m) + (m <= kJacobiPreMax ? 3 * jacobi_pad(m) * jacobi_pad(m) : 0);
}

// sum_k A[ia + k * sa] * B[ib + k * sb] for k < len, four independent accumulators
// (short dependent chains: these products are latency-bound on one SM)
__device__ __forceinline__ double jdot(const double* A, int ia, int sa, const double* B, int ib, int sb, int len) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int k = 0;
#pragma unroll 1
  for (; k + 3 < len; k += 4) {
    a0 = fma(A[ia + k * sa], B[ib + k * sb], a0);
    a1 = fma(A[ia + (k + 1) * sa], B[ib + (k + 1) * sb], a1);
    a2 = fma(A[ia + (k + 2) * sa], B[ib + (k + 2) * sb], a2);
    a3 = fma(A[ia + (k + 3) * sa], B[ib + (k + 3) * sb], a3);
  }
#pragma unroll 1
  for (; k < len; ++k) a0 = fma(A[ia + k * sa], B[ib + k * sb], a0);
  return (a0 + a1) + (a2 + a3);
}

__device__ inline void block_jacobi(const double* __restrict__ Hg, int64_t ldh, int m, double* __restrict__ theta,
                                    double* __restrict__ Sout, double* sm, double* __restrict__ info) {
  const int mp = jacobi_pad(m);
  double* H = sm;
  double* V = H + mp * mp;
  double* cs = V + mp * mp;
  double* sn = cs + 64;
  int* pp = reinterpret_cast<int*>(sn + 64);
  int* qq = pp + 64;
  double* red = sn + 64 + 64;  // 32 doubles after the two int arrays (64 ints = 32 doubles each)
  int* done = reinterpret_cast<int*>(red + 32);
  const int t = threadIdx.x;
  const int nth = blockDim.x;
  const int half = mp / 2;
  for (int idx = t; idx < mp * mp; idx += nth) {
    const int i = idx / mp, j = idx - i * mp;
    double h = 0.0;
    if (i < m && j < m) h = (i <= j) ? Hg[i * ldh + j] : Hg[j * ldh + i];
    H[idx] = h;
    V[idx] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  JACOBI_MARK(40);
  auto block_sum = [&](double v) -> double {
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
#pragma unroll 1
      for (int w = 0; w < (nth >> 5); ++w) s += red[w];
      red[0] = s;
    }
    __syncthreads();
    return red[0];
  };
  double local = 0.0, loff = 0.0;
  for (int idx = t; idx < mp * mp; idx += nth) {
    const int i = idx / mp, j = idx - i * mp;
    local += H[idx] * H[idx];
    if (i != j) loff += H[idx] * H[idx];
  }
  const double fro2 = block_sum(local);
  const double stop2 = fro2 * 1e-30;  // off(H) <= 1e-15 ||H||_F
  double off2 = block_sum(loff), prev = INFINITY;
  JACOBI_MARK(41);
  double* Vs = V;  // accumulated rotations (pointer rotates through the scratch buffers)
  for (int pre = 0; pre < 3 && m <= kJacobiPreMax && !(off2 <= stop2) && off2 <= 1e-6 * fro2 && off2 < 0.25 * prev;
       ++pre) {
    const int mm = mp * mp;
    double* Y = sm + jacobi_base_doubles(m);
    double* Tm = Y + mm;
    double* Z = Tm + mm;
    if (Vs != V) {  // Vs occupies one of the scratch buffers: use V's home as scratch instead
      if (Vs == Y) Y = V;
      else if (Vs == Tm) Tm = V;
      else Z = V;
    }
    // Y = I + X
    double xmax = 0.0;
#pragma unroll 1
    for (int idx = t; idx < mm; idx += nth) {
      const int i = idx / mp, j = idx - i * mp;
      double y = 1.0;
      if (i != j) {
        const double h = H[idx], d = H[j * mp + j] - H[i * mp + i];
        y = (h != 0.0 && fabs(h) <= 0.1 * fabs(d)) ? h / d : 0.0;
        xmax = fmax(xmax, fabs(y));
      }
      Y[idx] = y;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, off));
    if ((t & 31) == 0) red[32 + (t >> 5)] = xmax;
    __syncthreads();
    xmax = 0.0;
#pragma unroll 1
    for (int w = 0; w < (nth >> 5); ++w) xmax = fmax(xmax, red[32 + w]);
    if (xmax < 1e-8) {
      // Y^T Y = I + O(|X|^2) < 1e-16 off the identity: the Newton-Schulz step would not change S
#pragma unroll 1
      for (int idx = t; idx < mm; idx += nth) Z[idx] = Y[idx];
    } else {
      // Tm = (3I - Y^T Y) / 2
#pragma unroll 1
      for (int idx = t; idx < mm; idx += nth) {
        const int i = idx / mp, j = idx - i * mp;
        Tm[idx] = 0.5 * ((i == j ? 3.0 : 0.0) - jdot(Y, i, mp, Y, j, mp, mp));
      }
      __syncthreads();
      // Z = S = Y Tm
#pragma unroll 1
      for (int idx = t; idx < mm; idx += nth) {
        const int i = idx / mp, j = idx - i * mp;
        Z[idx] = jdot(Y, i * mp, 1, Tm, j, mp, mp);
      }
    }
    __syncthreads();
    // Tm = H S;  Y = Vs S (the new accumulated rotations)
#pragma unroll 1
    for (int idx = t; idx < mm; idx += nth) {
      const int i = idx / mp, j = idx - i * mp;
      Tm[idx] = jdot(H, i * mp, 1, Z, j, mp, mp);
      Y[idx] = jdot(Vs, i * mp, 1, Z, j, mp, mp);
    }
    __syncthreads();
    Vs = Y;
    // H <- S^T (H S), symmetric by construction (upper triangle mirrored)
    double lo2 = 0.0;
#pragma unroll 1
    for (int idx = t; idx < mm; idx += nth) {
      const int i = idx / mp, j = idx - i * mp;
      if (i <= j) {
        const double a = jdot(Z, i, mp, Tm, j, mp, mp);
        H[i * mp + j] = a;
        H[j * mp + i] = a;
        if (i != j) lo2 += 2.0 * a * a;
      }
    }
    prev = off2;
    off2 = block_sum(lo2);  // its barriers also publish H
    JACOBI_MARK(42 + pre);
  }
  if (Vs != V) {
    for (int idx = t; idx < mp * mp; idx += nth) V[idx] = Vs[idx];
    __syncthreads();
  }
  JACOBI_MARK(45);
  prev = INFINITY;
  int sweep = 0;
  // fixed thread -> work mapping for the whole solve (no divisions in the rounds)
  const int rot_pair = t < half ? t : -1;
  for (sweep = 0; sweep < 40 && !(off2 <= stop2); ++sweep) {
    int p = 0, q = 1;
    for (int round = 0; round < mp - 1; ++round) {
      if (rot_pair >= 0) {
        // round-robin schedule: player 0 fixed, players 1..mp-1 rotate
        if (rot_pair == 0) {
          p = 0;
          q = 1 + round;
        } else {
          int a = round + rot_pair, b = round - rot_pair + (mp - 1);
          a = a >= mp - 1 ? a - (mp - 1) : a;
          b = b >= mp - 1 ? b - (mp - 1) : b;
          p = 1 + a;
          q = 1 + b;
        }
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        const double apq = H[p * mp + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          // rotation angle in float32 (MUFU rcp/rsqrt instead of float64 div/sqrt
          // latency chains), (c, s) re-normalised in float64 by two Newton steps so
          // the rotation is orthogonal to working precision; the approximate angle
          // leaves a tiny a_pq that the next sweep annihilates
          const float tau = (float)(H[q * mp + q] - H[p * mp + p]) * (0.5f / (float)apq);
          const float at = fabsf(tau);
          float tt = at > 1e15f ? 0.5f / at : 1.0f / (at + sqrtf(1.0f + tau * tau));
          if (tau < 0.f) tt = -tt;
          const float cf = rsqrtf(1.0f + tt * tt);
          c = (double)cf;
          s = (double)tt * (double)cf;
#pragma unroll
          for (int it = 0; it < 2; ++it) {
            const double g = 1.5 - 0.5 * (c * c + s * s);
            c *= g;
            s *= g;
          }
        }
        pp[rot_pair] = p;
        qq[rot_pair] = q;
        cs[rot_pair] = c;
        sn[rot_pair] = s;
      }
      __syncthreads();
      // two independent items per iteration (ILP: both items' loads issue before either's math)
      auto hblock = [&](int idx) {
        const int aa = idx / half, bb = idx - aa * half;
        const int pa = pp[aa], qa = qq[aa], pb = pp[bb], qb = qq[bb];
        const double ca = cs[aa], sa = sn[aa], cb = cs[bb], sb = sn[bb];
        const double h00 = H[pa * mp + pb], h01 = H[pa * mp + qb];
        const double h10 = H[qa * mp + pb], h11 = H[qa * mp + qb];
        const double t00 = ca * h00 - sa * h10, t01 = ca * h01 - sa * h11;
        const double t10 = sa * h00 + ca * h10, t11 = sa * h01 + ca * h11;
        double n00 = t00 * cb - t01 * sb, n01 = t00 * sb + t01 * cb;
        double n10 = t10 * cb - t11 * sb, n11 = t10 * sb + t11 * cb;
        if (aa == bb) {
          const double avg = 0.5 * (n01 + n10);
          n01 = avg;
          n10 = avg;
        }
        H[pa * mp + pb] = n00;
        H[pa * mp + qb] = n01;
        H[qa * mp + pb] = n10;
        H[qa * mp + qb] = n11;
      };
      auto vrot = [&](int idx) {
        const int i = idx / half, aa = idx - i * half;
        const int pa = pp[aa], qa = qq[aa];
        const double ca = cs[aa], sa = sn[aa];
        const double vp = V[i * mp + pa], vq = V[i * mp + qa];
        V[i * mp + pa] = ca * vp - sa * vq;
        V[i * mp + qa] = sa * vp + ca * vq;
      };
      const int nhb = half * half, nvr = mp * half;
      for (int idx = t; idx < nhb; idx += 2 * nth) {
        hblock(idx);
        if (idx + nth < nhb) hblock(idx + nth);
      }
      for (int idx = t; idx < nvr; idx += 2 * nth) {
        vrot(idx);
        if (idx + nth < nvr) vrot(idx + nth);
      }
      __syncthreads();
    }
    double lo = 0.0;
    for (int idx = t; idx < mp * mp; idx += nth) {
      const int i = idx / mp, j = idx - i * mp;
      if (i != j) lo += H[idx] * H[idx];
    }
    off2 = block_sum(lo);
    if (t == 0) *done = (off2 > 0.25 * prev && off2 <= fro2 * 1e-26);
    __syncthreads();
    prev = off2;
    if (*done) {
      ++sweep;
      break;
    }
  }
  JACOBI_MARK(46);
  for (int i = t; i < m; i += nth) {
    const double di = H[i * mp + i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = H[j * mp + j];
      rank += (dj > di) || (dj == di && j < i);
    }
    theta[rank] = di;
    for (int k = 0; k < m; ++k) Sout[(int64_t)k * m + rank] = V[k * mp + i];
  }
  if (t == 0 && info) {
    info[0] = sweep;
    info[1] = sqrt(off2);
    info[2] = sqrt(fro2);
  }
  JACOBI_MARK(47);
}

// Single-warp variant for m <= 32: warp-synchronous rounds (only __syncwarp),
// the round-robin schedule tabulated once in shared memory, and each lane's
// 2x2-block and rotation work lists fixed for the whole solve.  Same numerics
// and outputs as block_jacobi; call with the whole warp (lanes 0..31).
__host__ __device__ constexpr int warp_jacobi_smem_doubles(int m) {
  return 2 * jacobi_pad(m) * jacobi_pad(m) + 32 * 16 + 64;
}

__device__ inline void warp_jacobi(const double* __restrict__ Hg, int64_t ldh, int m, double* __restrict__ theta,
                                   double* __restrict__ Sout, double* sm, double* __restrict__ info) {
  const int lane = threadIdx.x & 31;
  const int mp = jacobi_pad(m);
  const int half = mp / 2;
  double* H = sm;
  double* V = H + mp * mp;
  short2* sched = reinterpret_cast<short2*>(V + mp * mp);  // (mp-1) x half pairs (<= 31 x 16)
  double* cs = reinterpret_cast<double*>(sched + 32 * 16);
  double* sn = cs + 16;
  int* pp = reinterpret_cast<int*>(sn + 16);
  int* qq = pp + 16;
  for (int idx = lane; idx < mp * mp; idx += 32) {
    const int i = idx / mp, j = idx - i * mp;
    double h = 0.0;
    if (i < m && j < m) h = (i <= j) ? Hg[i * ldh + j] : Hg[j * ldh + i];
    H[idx] = h;
    V[idx] = (i == j) ? 1.0 : 0.0;
  }
  for (int idx = lane; idx < (mp - 1) * half; idx += 32) {
    const int round = idx / half, k = idx - round * half;
    int p, q;
    if (k == 0) {
      p = 0;
      q = 1 + round;
    } else {
      p = 1 + (round + k) % (mp - 1);
      q = 1 + (round - k + (mp - 1)) % (mp - 1);
    }
    sched[idx] = make_short2((short)min(p, q), (short)max(p, q));
  }
  __syncwarp();
  auto warp_sum = [&](double v) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
  double fl = 0.0, ol = 0.0;
  for (int idx = lane; idx < mp * mp; idx += 32) {
    const double h = H[idx];
    fl += h * h;
    if (idx / mp != idx % mp) ol += h * h;
  }
  const double fro2 = warp_sum(fl);
  const double stop2 = fro2 * 1e-30;
  double off2 = warp_sum(ol), prev = INFINITY;
  const int nblk = half * half, nv = mp * half;
  int sweep = 0;
  for (sweep = 0; sweep < 40 && !(off2 <= stop2); ++sweep) {
    for (int round = 0; round < mp - 1; ++round) {
      if (lane < half) {
        const short2 pq = sched[round * half + lane];
        const int p = pq.x, q = pq.y;
        const double apq = H[p * mp + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const float tau = (float)(H[q * mp + q] - H[p * mp + p]) * (0.5f / (float)apq);
          const float at = fabsf(tau);
          float tt = at > 1e15f ? 0.5f / at : 1.0f / (at + sqrtf(1.0f + tau * tau));
          if (tau < 0.f) tt = -tt;
          const float cf = rsqrtf(1.0f + tt * tt);
          c = (double)cf;
          s = (double)tt * (double)cf;
#pragma unroll
          for (int it = 0; it < 2; ++it) {
            const double g = 1.5 - 0.5 * (c * c + s * s);
            c *= g;
            s *= g;
          }
        }
        pp[lane] = p;
        qq[lane] = q;
        cs[lane] = c;
        sn[lane] = s;
      }
      __syncwarp();
      for (int b = lane; b < nblk; b += 32) {
        const int a = b / half, bb = b - a * half;
        const int pa = pp[a], qa = qq[a], pb = pp[bb], qb = qq[bb];
        const double ca = cs[a], sa = sn[a], cb = cs[bb], sb = sn[bb];
        const double h00 = H[pa * mp + pb], h01 = H[pa * mp + qb];
        const double h10 = H[qa * mp + pb], h11 = H[qa * mp + qb];
        const double t00 = ca * h00 - sa * h10, t01 = ca * h01 - sa * h11;
        const double t10 = sa * h00 + ca * h10, t11 = sa * h01 + ca * h11;
        double n00 = t00 * cb - t01 * sb, n01 = t00 * sb + t01 * cb;
        double n10 = t10 * cb - t11 * sb, n11 = t10 * sb + t11 * cb;
        if (a == bb) {
          const double avg = 0.5 * (n01 + n10);
          n01 = avg;
          n10 = avg;
        }
        H[pa * mp + pb] = n00;
        H[pa * mp + qb] = n01;
        H[qa * mp + pb] = n10;
        H[qa * mp + qb] = n11;
      }
      for (int v = lane; v < nv; v += 32) {
        const int i = v / half, a = v - i * half;
        const int pa = pp[a], qa = qq[a];
        const double ca = cs[a], sa = sn[a];
        const double vp = V[i * mp + pa], vq = V[i * mp + qa];
        V[i * mp + pa] = ca * vp - sa * vq;
        V[i * mp + qa] = sa * vp + ca * vq;
      }
      __syncwarp();
    }
    double lo = 0.0;
    for (int idx = lane; idx < mp * mp; idx += 32)
      if (idx / mp != idx % mp) lo += H[idx] * H[idx];
    off2 = warp_sum(lo);
    const bool stag = (off2 > 0.25 * prev && off2 <= fro2 * 1e-26);
    prev = off2;
    if (stag) {
      ++sweep;
      break;
    }
  }
  for (int i = lane; i < m; i += 32) {
    const double di = H[i * mp + i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double dj = H[j * mp + j];
      rank += (dj > di) || (dj == di && j < i);
    }
    theta[rank] = di;
    for (int k = 0; k < m; ++k) Sout[(int64_t)k * m + rank] = V[k * mp + i];
  }
  if (lane == 0 && info) {
    info[0] = sweep;
    info[1] = sqrt(off2);
    info[2] = sqrt(fro2);
  }
}

}  // namespace megb200
