// K6: Rayleigh-Ritz eigensolver for the small projected matrix H (m <= 112):
// parallel cyclic Jacobi with round-robin pair ordering, run by one CTA with
// H and the accumulated rotations in shared memory (float64).  Each round
// applies m/2 disjoint rotations J^T H J as independent 2x2 block updates, so
// a round costs two __syncthreads; sweeps stop when off(H) <= 1e-15 ||H||_F or
// stagnates.  Output: theta non-increasing (stable by index), S (m x m
// row-major, column j = eigenvector j).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace megb200 {

__host__ __device__ constexpr int jacobi_pad(int m) { return (m + 1) & ~1; }
// shared-memory doubles needed by block_jacobi for size m
__host__ __device__ constexpr int jacobi_smem_doubles(int m) { return 2 * jacobi_pad(m) * jacobi_pad(m) + 64 * 4 + 40; }

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
  auto block_sum = [&](double v) -> double {
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
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
      for (int idx = t; idx < half * half; idx += nth) {
        const int a = idx / half, bb = idx - a * half;
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
      for (int idx = t; idx < mp * half; idx += nth) {
        const int i = idx / half, a = idx - i * half;
        const int pa = pp[a], qa = qq[a];
        const double ca = cs[a], sa = sn[a];
        const double vp = V[i * mp + pa], vq = V[i * mp + qa];
        V[i * mp + pa] = ca * vp - sa * vq;
        V[i * mp + qa] = sa * vp + ca * vq;
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
}

}  // namespace megb200
