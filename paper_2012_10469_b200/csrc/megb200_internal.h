// Internal declarations shared by the kernel and runtime translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/megb200.h"

namespace megb200 {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define MEG_CUDA(call)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw ::megb200::Error(MEGB200_ERR_CUDA, std::string(#call " failed: ") + cudaGetErrorString(e_)); \
  } while (0)

#define MEG_LAUNCHED()                                                                              \
  do {                                                                                              \
    cudaError_t e_ = cudaGetLastError();                                                            \
    if (e_ != cudaSuccess)                                                                          \
      throw ::megb200::Error(MEGB200_ERR_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// counter-based Gaussian generator shared with oracle/inputs.py
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * kGolden + stream * kMix2);
}

// Random-stream ids (oracle/inputs.py uses 1..5 and 7 for inputs).
constexpr int kStreamStart = 11;   // solver start block
constexpr int kStreamRefill = 12;  // breakdown replacement directions

// ---------------------------------------------------------------------------
// launch wrappers (megb200_kernels.cu).  All tall-skinny arrays are float64
// row-major with explicit leading dimensions.

// True the first time it is called for (current device, tag), thread-safe: per-device one-time
// setup such as cudaFuncSetAttribute(MaxDynamicSharedMemorySize), which is a per-device function
// attribute (a process-wide flag would skip it on a second device).
bool first_on_device(const void* tag);

struct Launch {
  cudaStream_t stream;
  int64_t* counter;  // kernels launched (telemetry for bench.py)
  // float64 DMMA pass only: wait until *wait_ctr >= wait_target instead of for the preceding grid's
  // completion (the preceding k_fused_first_pass released its Ritz rows early, see FusedPassArgs)
  const unsigned long long* wait_ctr = nullptr;
  unsigned long long wait_target = 0;
};

// Streamed operator product: part[s] (S x n x b, dense row-major ld b) =
// Op restricted to k-slice s times U.  Returns the number of k-slices S used.
int dense_apply_partial(const Launch& L, const void* M, int dtype, int64_t ldm, int64_t n, const double* U,
                        int64_t ldu, int b, double* part, int64_t part_cap_slices, int sm_count, float* uscratch = nullptr);
// 2D row-major tensor map (cached): inner dimension `cols`, outer `rows`, leading dimension `ld` elements
CUtensorMap make_map(const void* base, CUtensorMapDataType dt, size_t es, int64_t cols, int64_t rows, int64_t ld,
                     uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE);
// tcgen05 split-TF32 pass for float32 operands (megb200_umma.cu); uscratch: 64 x n floats
bool umma_pass_supported(int64_t n, int b, int64_t ldm, const void* M);
int dense_pass_umma(const Launch& L, const float* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                    double* part, int64_t part_cap_slices, int sm_count, float* uscratch);
// Sampled-entry (CSR) pass.  With a panel-pointer scratch (pp: n x (P + 1) int32, P <= 16 column panels)
// and enough partial slices the panel-tiled kernel runs: CTA (row group, column panel) stages the
// panel's rows of U in shared memory and gathers from there; slice p holds panel p's contribution.
// pp_valid: the scratch already holds this pattern's panel pointers (set on return).  Returns the
// number of slices written (1 for the warp-per-row kernel that gathers U rows through L2).
int csr_apply_partial(const Launch& L, const int32_t* rowptr, const int32_t* col, const double* val, int64_t n,
                      const double* U, int64_t ldu, int b, double* part, int64_t part_cap_slices = 1,
                      int32_t* pp = nullptr, bool* pp_valid = nullptr, int sm_count = 148);
constexpr int kCsrMaxPanels = 16;

// C (p x q, ld ldc) = diag(rowscale) * X^T Y  (+ beta C if accumulate).  rowscale may be null.
void tn(const Launch& Lc, int64_t n, const double* X, int64_t ldx, int p, const double* Y, int64_t ldy, int q,
        double* C, int64_t ldc, const double* rowscale, double* part, int64_t part_cap, int sm_count);
// Y (n x q) = beta * Y + alpha * X C   (X n x p, C p x q dense ld ldc).  Z == Y allowed only if beta path.
void nn(const Launch& L, int64_t n, const double* X, int64_t ldx, int p, const double* C, int64_t ldc, int q,
        double alpha, double beta, double* Y, int64_t ldy);
// Wide Rayleigh-Ritz (m <= 112, one CTA): Householder tridiagonalisation + multisection +
// twisted-factorisation eigenvectors, verified, with a cyclic-Jacobi fallback (megb200_rr.cu)
// (only the top nvec eigenpairs and the smallest eigenvalue are computed when nvec < m; the
// other theta entries are reported as the smallest, the other S columns as zero)
void rr_wide(const Launch& L, const double* H, int64_t ldh, int m, double* theta, double* S, double* info,
             int nvec = 0);
void copy_block(const Launch& L, int64_t n, int q, const double* src, int64_t lds, double* dst, int64_t ldd);
void fill_gaussian(const Launch& L, int64_t n, int q, uint64_t key, uint64_t base, double scale, bool round_f32,
                   double* dst, int64_t ldd);
// sampled gradient values g_e = X_ij - obs_e from factors; optional partial sum of squares
void csr_values(const Launch& L, int64_t n, const int32_t* rowptr, const int32_t* col, const double* obs,
                const double* V, int64_t ldv, int r, const double* coeff, double tail, double* g, double* sq_part,
                int sq_slots);
void dense_stats(const Launch& L, const void* M, int dtype, int64_t ld, int64_t n, double* part, int slots);
void gen_dense_target(const Launch& L, const double* U, int64_t r, const double* lam, double sigma, uint64_t key,
                      void* M, int dtype, int64_t ld, int64_t n);
void reduce_sum(const Launch& L, const double* part, int slots, int width, double* out);
// config-3 synthetic sampled instance (twin of oracle/inputs.sampled_instance)
void sampled_count(const Launch& L, int64_t n, uint64_t kmask, double p, int32_t* counts);
void sampled_fill(const Launch& L, int64_t n, uint64_t kmask, uint64_t knoise, double p, const double* U, int r,
                  const double* lam, double obs_noise, const int32_t* rowptr, int32_t* col, double* val);
// part[g] (g < slots) = partial sums of (X_ij - M_ij)^2, X from (V, coeff, tail); r <= 64
void frob_direct(const Launch& L, const void* M, int dtype, int64_t ld, int64_t n, const double* V, int64_t ldv, int r,
                 const double* coeff, double tail, double* part, int slots);
// Q[0:n, 0:n] = I (leading dimension ldq)
void set_identity(const Launch& L, int64_t n, double* Q, int64_t ldq);
// H[0:cap, 0:cap] = 0 except H[j][j] = theta[j] for j < k
void set_diag(const Launch& L, double* H, int cap, int k, const double* theta);
// Thick restart of H when the next block's column block H[0:m+q, m:m+q] is already there (the overlapped
// Rayleigh-Ritz of top_eigs): H <- [diag(theta[0:keep]), S[:, 0:keep]^T H[0:m, m:m+q]; ., H[m:m+q, m:m+q]]
// (upper triangle), everything else zero.  S is m x m row-major (column k = Ritz vector k).
// Thick restart of the basis, in place, in one launch: Q[:, 0:keep] = Q[:, 0:m] S[:, 0:keep], the same for
// AQ, and the tq columns [m, m + tq) of both moved to [keep, keep + tq) (keep + tq <= m)
void restart_basis(const Launch& L, int64_t n, double* Q, double* AQ, int64_t ldq, const double* S, int m, int keep,
                   int tq, int sm_count);
void restart_h(const Launch& L, double* H, int cap, const double* S, int m, int keep, int q, const double* theta);

// cooperative tall-skinny kernels (megb200_coop.cu): one launch each
void coop_tn(const Launch& L, int64_t n, const double* X, int64_t ldx, int p, const double* Y, int64_t ldy, int q,
             double* C, int64_t ldc, const double* rowscale, double scale, double* part, int sm_count);
void coop_cgs(const Launch& L, int64_t n, const double* Q, int64_t ldq, int cols, double* W, int64_t ldw, int q,
              double* Cws, double* part, int sm_count);
void coop_cholqr(const Launch& L, int64_t n, const double* Wsrc, int64_t lds, double* W, int64_t ldw, int q,
                 double thresh, double* Gws, double* Rrel, double* Rinv, int* mask, const double* Rprev, double* Rtot,
                 uint64_t key, uint64_t base, double* part, int sm_count);
// The whole orthonormalize() sequence (CGS x cgs_rounds, CholQR(thresh1), CGS, CholQR(0)) of
// W (n x q) against Q[:, 0:cols] in one cooperative launch; false when the shape does not fit
// (q > 32 or the staged rows exceed shared memory): the caller then runs the separate launches.
bool coop_orth(const Launch& L, int64_t n, const double* Q, int64_t ldq, int cols, double* W, int64_t ldw, int q,
               double thresh1, uint64_t key, uint64_t base, double* part, double* Cws, double* Gws, double* Rinv,
               int* mask, double* Rrel, int sm_count, int cgs_rounds, const double* Wsrc = nullptr, int64_t lds = 0,
               const double* Cpre = nullptr, int64_t ldcp = 0, const double* Gpre = nullptr);
// Log-map coefficients of a factored iterate computed on the device (so a step
// can consume the kept weights lam another launch left in device memory):
// d[k] = log(c1 lam[k]) - log_tail - eta (c1 lam[k] - tail_g) for k < lr.
struct LamCoef {
  const double* lam = nullptr;
  int lr = 0;
  double c1 = 0.0, log_tail = 0.0, eta = 0.0, tail_g = 0.0;
};
// The operator itself into AQ (n x n, ld ldq) and H (ld ldh): A = scale * M + L diag(d) L^T + alpha I (identity-basis
// solves of small problems; M float64 symmetric, may be null with scale 0)
void form_operator(const Launch& L, int64_t n, const double* M, int64_t ldm, double scale, const double* Lf, int64_t ldl,
                   int l, const double* d, LamCoef lc, double alpha, double* AQ, int64_t ldq, double* H, int64_t ldh);
void coop_finish(const Launch& L, int64_t n, int b, int S, const double* spart, double scale, const double* Lf,
                 int64_t ldl, int l, const double* d, double alpha, const double* U, int64_t ldu, double* W,
                 int64_t ldw, double* Ews, double* part, int sm_count, const double* Qh = nullptr, int64_t ldq = 0,
                 int hp = 0, double* Hout = nullptr, int64_t ldh = 0, LamCoef lc = LamCoef(),
                 const double* Eg = nullptr, int64_t ldg = 0,  // Eg: precomputed L^T U (skips its reduction)
                 double* Gout = nullptr);  // with Hout: also W^T W (b x b, ld b), in the same reduction
// Jacobi RR + Ritz block + residuals (+ Gram of the first gr Ritz vectors, + MEG epilogue into epi);
// the first r2 Ritz vectors are also written to V2
void coop_rr(const Launch& L, const double* H, int64_t ldh, int m, double* theta, double* S, double* info, int64_t n,
             const double* Q, const double* AQ, int64_t ldq, int rq, int nreq, double* T, int64_t ldt, double* resid,
             double* part, int sm_count, int gr, double* Gout, double eps_next, double* epi, double* V2 = nullptr,
             int64_t ld2 = 0, int r2 = 0, int nvec = 0, bool presolved = false);

// First pass of a solve fused with its finish and Rayleigh-Ritz (megb200_step.cu):
// W = scale * sum_s part[s] + L E + alpha U, H = U^T W, Jacobi RR, Ritz block T,
// residuals, Gram of T, step epilogue, result pack (device + optional host slot),
// in one launch.  Cross-CTA reductions by last-CTA tickets in fixed CTA order.
constexpr int kFusedMaxL = 64;
constexpr int kFusedStride = 2048;  // doubles per CTA partial (>= l*b, b*b, nreq + gr*gr)
constexpr int kFusedFlags = 96;    // sync[0..95]: tickets of the three reductions, then release flags
struct FusedPassArgs {
  int64_t n = 0;
  int b = 0, R = 0;
  const double* part = nullptr;  // S x n x b pass partials
  int S = 0;
  double scale = 0.0, alpha = 0.0;
  const double* L = nullptr;
  int64_t ldl = 0;
  int l = 0;
  const double* d = nullptr;  // host-provided coefficients (device), or from lc
  LamCoef lc;
  const double* Eg = nullptr;  // precomputed L^T U (l x b, ld ldg) or null
  int64_t ldg = 0;
  const double* Gu = nullptr;  // U^T U (b x b, ld ldgu): k_dense_step_mma forms H = U^T W from it
  int64_t ldgu = 0;
  const double* U = nullptr;
  int64_t ldu = 0;
  double* W = nullptr;
  int64_t ldw = 0;
  double* H = nullptr;
  int64_t ldh = 0;
  double *theta = nullptr, *Sout = nullptr, *info = nullptr;
  double* T = nullptr;
  int64_t ldt = 0;
  double* V2 = nullptr;
  int64_t ld2 = 0;
  int r2 = 0;
  double *resid = nullptr, *gram = nullptr;
  int gr = 0, nreq = 0, rq = 0;
  double* epi = nullptr;
  double eps_next = 0.0;
  double *part0 = nullptr, *part1 = nullptr, *part2 = nullptr, *Ews = nullptr;
  unsigned* sync = nullptr;  // tickets [0..95] (32 per reduction), flags [96..97]
  unsigned epoch = 0;
  const double* pack = nullptr;  // device result pack, copied to host_pack[0:pack_count] at the end
  double* host_pack = nullptr;
  int pack_count = 0;
  unsigned long long* stamps = nullptr;  // diagnostics: phase timestamps (or null)
  double* vgram = nullptr;  // optional out: Gram of the first nvg columns of L (phase 0 only)
  int nvg = 0;
  bool stage_l = true;  // set by fused_first_pass: L rows staged in shared memory
  bool cooperative = false;  // launch cooperatively (more than one solver handle alive)
  int lam_inline_n = 0;   // > 0: lc's kept weights passed by value (lam_inline), lc.lam not read
  double lam_inline[64] = {};
  // overlap with the next step's operand pass: every CTA bumps rows_ctr once its Ritz rows are
  // written and lets the dependent launch start (the pass waits on the counter, not on this grid's
  // completion); the CTA that writes the result pack then stores `epoch` into done_flag (and into
  // host_pack[pack_count], the host's completion marker).  A launch first waits until done_flag
  // holds prev_epoch (the previous launch's reduction buffers are free); prev_epoch 0: no wait.
  unsigned long long* rows_ctr = nullptr;
  unsigned* done_flag = nullptr;
  unsigned prev_epoch = 0;
};
bool fused_pass_supported(int64_t n, int b, int l, int nreq, int sm_count);
int fused_first_pass(const Launch& L, FusedPassArgs a, int sm_count);  // returns the grid size

// The float64 dense pass and the step tail above in ONE cooperative launch (megb200_kernels.cu,
// k_dense_step_mma); needs a.Eg when a.l > 0, a.rq == b, a.gr <= b, no vgram, a.sync with >= 512
// zeroed words.  part: the pass's partial slots (part_cap_slices x n x b).
bool dense_step_mma_supported(const void* M, int dtype, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                              int l, int64_t part_cap_slices, int sm_count);
void dense_step_mma(const Launch& L, const double* M, int64_t ldm, int64_t n, const double* U, int64_t ldu, int b,
                    double* part, int64_t part_cap_slices, int sm_count, const FusedPassArgs& a);
// E = L^T U (l x b, ld b), vgram = L^T L (nvg x nvg) and Gu = U^T U (b x b) over 128-row tiles, the
// step tail's Gram product order; part: tiles x kFusedStride doubles; ticket: one zeroed word
void tile_gram(const Launch& L, int64_t n, const double* Lm, int64_t ldl, int l, const double* U, int64_t ldu, int b,
               int nvg, double* part, unsigned* ticket, double* E, double* vgram, double* Gu);

// quadratic-measurement objective (megb200_qm.cu)
struct QmCoef {
  double tau = 0.0, eps = 0.0, tail = 0.0;
  double lam[32] = {};
};
void qm_residuals(const Launch& L, const double* a, const double* b, const double* y, int64_t m, int64_t n,
                  const double* V, int64_t ldv, int r, const QmCoef& qc, double* res);
int64_t qm_grad_part_doubles(int64_t m, int64_t n);
void qm_gradient(const Launch& L, const double* a, const double* b, const double* res, int64_t m, int64_t n,
                 double weight, double* G, int64_t ldg, double* part, const int64_t* idx = nullptr);
void qm_sumsq(const Launch& L, const double* res, int64_t m, double* out);
// matrix-free block application W = weight / 2 (a^T diag(res) b + b^T diag(res) a) U  (n x k, ld k)
int64_t qm_apply_scratch_doubles(int64_t m, int64_t n, int k, int sm_count);
void qm_apply(const Launch& L, const double* a, const double* b, const double* res, const int64_t* idx, int64_t m,
              int64_t n, double weight, const double* U, int64_t ldu, int k, double* W, double* scratch, int sm_count);

}  // namespace megb200
