/*
 * megb200.h -- C ABI of the B200 (sm_100a) low-rank MEG hot path.
 *
 * Drop-in boundary for the per-iteration path of the reference `specmeg`
 * package (arXiv 2012.10469).  The reference is pure Python/numpy, so the
 * FFI a maintainer would bind is ctypes; each entry
 * point below names the reference function it replaces.
 *
 * Conventions
 *   - All pointers marked (device) are CUDA device pointers on the current
 *     device; (host) pointers are plain host memory.  Nothing is freed by the
 *     library that it did not allocate.
 *   - Tall-skinny blocks (V, U, W, Ritz vectors) are float64, row-major:
 *     element (i, c) at ptr[i * ld + c]  (a C-contiguous numpy (n, k) array
 *     has ld = k).
 *   - Dense operands (M or a dense gradient G) are symmetric n x n row-major
 *     with leading dimension ld, float64 or float32.
 *   - Every function returns an int status; on non-zero,
 *     megb200_last_error() describes it (thread-local).  No C++ exception
 *     crosses the ABI.  Parameter errors are detected before any launch.
 *   - Work is enqueued on the stream given to megb200_solver_set_stream
 *     (default: the legacy default stream); functions that return host
 *     results synchronise that stream.
 */
#ifndef MEGB200_H
#define MEGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEGB200_ABI_VERSION 1

/* status codes ------------------------------------------------------------ */
enum {
  MEGB200_OK = 0,
  MEGB200_ERR_PARAM = 1,     /* -> specmeg.linalg.ParameterError (linalg.py:23-24)     */
  MEGB200_ERR_LANCZOS = 2,   /* -> specmeg.linalg.LanczosError   (linalg.py:43-52)     */
  MEGB200_ERR_CUDA = 3,      /* CUDA runtime / launch failure                           */
  MEGB200_ERR_KEPT_MASS = 4, /* -> AssertionError "kept mass vanished" (meg.py:350)     */
  MEGB200_ERR_NO_DEVICE = 5, /* no sm_100 device visible                                */
  MEGB200_ERR_CALLBACK = 6   /* a caller-supplied apply callback returned non-zero      */
};

enum { MEGB200_F64 = 0, MEGB200_F32 = 1 };

/* A symmetric linear operator on R^n, applied to n x k blocks:
 *     A u = scale * Op(u) + L diag(d) L^T u + alpha u
 * Op is a dense symmetric matrix, a CSR matrix with float64 values, or
 * absent.  This is the device form of specmeg.linalg.SymmetricOperator
 * (linalg.py:81-103) for the operators the hot path builds. */
enum { MEGB200_OP_NONE = 0, MEGB200_OP_DENSE = 1, MEGB200_OP_CSR = 2, MEGB200_OP_CALLBACK = 3,
       MEGB200_OP_QUADMEAS = 4 };

/* Matrix-free quadratic-measurement gradient: Op U = weight / 2 (a^T diag(res) (b U) + b^T diag(res)
 * (a U)) over m measurement pairs -- the reference's _apply_measurement_gradient (objectives.py:152-158),
 * the operator RecoveryObjective builds above dense_cap (objectives.py:214-221).  a, b (m x n row-major,
 * ld n), res (one per measurement) and scratch are device pointers; scratch holds at least
 * megb200_qm_apply_scratch(s, m, 32) doubles.  Passed through `apply_ctx` of an operator / gradient of
 * kind QUADMEAS (`apply` unused). */
typedef struct megb200_qm_data {
  const double* a;
  const double* b;
  const double* res;
  int64_t m;          /* rows applied: the measurements, or the mini-batch length when idx is given */
  const int64_t* idx; /* (device, optional) mini-batch of measurement indices, repeats allowed
                         (StochasticOracle.grad_operator, objectives.py:255-269; weight carries tau m / L) */
  double weight;
  double* scratch;
  int64_t scratch_len;
} megb200_qm_data;

/* Caller-supplied block application W = Op U: the C form of the reference's Python callables
 * (SymmetricOperator(dim, apply_fn), linalg.py:81-94; grad_apply, meg.py:327-335).  U (n x k, ld
 * ldu) and W (n x k, ld ldw) are device pointers; the callback must enqueue its work on `stream`
 * (or finish it before returning) and return 0, non-zero on failure (-> MEGB200_ERR_CALLBACK).
 * The solver calls it once per block pass from the calling thread, k <= 64 columns at a time. */
typedef int (*megb200_apply_fn)(void* ctx, const double* U, int64_t ldu, int32_t k, double* W, int64_t ldw,
                                void* stream);

typedef struct megb200_operator {
  int32_t kind;          /* MEGB200_OP_*                                      */
  int32_t dtype;         /* dense only: MEGB200_F64 | MEGB200_F32             */
  int64_t n;
  const void* dense;     /* (device) n x n row-major, symmetric               */
  int64_t ld;            /* leading dimension of dense (elements)             */
  const int32_t* rowptr; /* (device) CSR row pointers, n + 1                  */
  const int32_t* col;    /* (device) CSR column indices, nnz                  */
  const double* val;     /* (device) CSR values, nnz                          */
  int64_t nnz;
  double scale;
  const double* L;       /* (device) n x l row-major low-rank factor, or NULL */
  int64_t l;
  int64_t ldl;
  const double* d;       /* (host) l coefficients                             */
  double alpha;
  megb200_apply_fn apply; /* CALLBACK: Op U (scaled by `scale`)               */
  void* apply_ctx;
} megb200_operator;

/* The gradient a step consumes: the device form of the reference's
 * `grad_apply` callable (meg.py:327-335).  grad f is evaluated at the
 * iterate X_g = (1 - g_eps) Vg diag(g_lam) Vg^T + g_eps/(n - r)(I - Vg Vg^T).
 *   DENSE       grad u = G u                        (test_meg.py:153 `g @ u`)
 *   FROBENIUS   grad u = X_g u - M u                (1/2||X - M||_F^2)
 *   SAMPLED     grad u = P_Omega(X_g - Mobs) u      (1/2 sum_Omega (X_ij - M_ij)^2)
 *   STOCHASTIC  grad u = X_g u - M u + sigma (A A^T u / b - u / n)
 *   ZERO        grad u = 0 */
enum {
  MEGB200_GRAD_ZERO = 0,
  MEGB200_GRAD_DENSE = 1,
  MEGB200_GRAD_FROBENIUS = 2,
  MEGB200_GRAD_SAMPLED = 3,
  MEGB200_GRAD_STOCHASTIC = 4,
  MEGB200_GRAD_CALLBACK = 5, /* grad u computed by `apply` (the reference's callable grad_apply) */
  MEGB200_GRAD_QUADMEAS = 6  /* grad u = matrix-free quadratic-measurement gradient, apply_ctx -> megb200_qm_data */
};

typedef struct megb200_gradient {
  int32_t kind;          /* MEGB200_GRAD_*                                    */
  int32_t dtype;         /* dtype of `dense`                                  */
  int64_t n;
  const void* dense;     /* (device) G (DENSE) or M (FROBENIUS, STOCHASTIC)   */
  int64_t ld;
  const int32_t* rowptr; /* (device) SAMPLED: Omega pattern (symmetric)       */
  const int32_t* col;
  const double* obs;     /* (device) SAMPLED: observed M_ij on Omega          */
  int64_t nnz;
  const double* gV;      /* (device) X_g factor, n x g_r row-major (ld g_ldv) */
  int64_t g_r;
  int64_t g_ldv;
  const double* g_lam;   /* (host) g_r weights                                */
  double g_eps;
  const double* A;       /* (device) STOCHASTIC: n x bsz row-major (ld lda)   */
  int64_t bsz;
  int64_t lda;
  double sigma;
  megb200_apply_fn apply; /* CALLBACK */
  void* apply_ctx;
} megb200_gradient;

/* Structured iterate (meg.py:47-92): V (device) n x r, lam (host) r, eps. */
typedef struct megb200_iterate {
  int64_t n;
  int64_t r;
  const double* V;
  int64_t ldv;
  const double* lam;
  double eps;
} megb200_iterate;

/* Eigensolver options: lanczos_top_r(op, r, tol, max_iter, seed, subspace,
 * restarts) (linalg.py:130-138) plus the block parameters of the device
 * solver.  Zero / NULL fields take defaults. */
typedef struct megb200_eig_opts {
  double tol;            /* residual rule tol * max(1, max|theta|) (linalg.py:214-215); 0 -> 1e-10 */
  int32_t max_passes;    /* budget in operator passes; 0 -> restarts * basis        */
  int32_t restarts;      /* 0 -> 12 (linalg.py:137)                                  */
  int32_t block;         /* block width k; 0 -> solver default                       */
  int32_t basis;         /* Krylov basis size (svd_subspace); 0 -> solver default    */
  int32_t keep;          /* thick-restart size; 0 -> basis / 2                       */
  uint64_t seed;         /* svd_seed: random start / refill directions               */
  const double* warm;    /* (device) optional warm-start block, n x warm_cols        */
  int64_t warm_cols;
  int64_t ld_warm;
  int32_t warm_orthonormal; /* warm block verified orthonormal (<= 1e-13): skip its CholQR */
} megb200_eig_opts;

typedef struct megb200_eig_result {
  double* eigenvalues;    /* (host, r)   theta, non-increasing                       */
  double* residual_norms; /* (host, r)   ||A x - theta x|| per pair                  */
  double* eigenvectors;   /* (device)    n x r row-major, ld = ld_vec (NULL: skip)   */
  int64_t ld_vec;
  double* ritz_block;     /* (device)    n x block top Ritz vectors for warm start    */
  int64_t ld_ritz;        /*             (NULL: skip)                                */
  int32_t passes;         /* out: operator passes executed                           */
  int32_t restarts;       /* out: thick restarts                                     */
  double norm_est;        /* out: max(1, max|theta_all|)                             */
  int32_t ritz_cols;      /* out: columns written to ritz_block (<= 64)              */
} megb200_eig_result;

/* Result of one MEG step (LowRankStepResult, meg.py:310-324).
 * Aliasing: V_next and ritz_block may overlap the iterate's V, the gradient's factor or the
 * warm block (opts->warm) -- the step then writes them only after the solve has converged
 * (through solver scratch), never while an operand is still being read. */
typedef struct megb200_step_result {
  double* V_next;         /* (device) n x r, ld = ld_next (caller-allocated)        */
  int64_t ld_next;
  double* lam_next;       /* (host, r)                                              */
  double* y;              /* (host, r+1) exp(mu - mu_1) = top_eigenvalues           */
  double* mu;             /* (host, r+1) Ritz values of log X - eta grad            */
  double* residual_norms; /* (host, r+1)                                            */
  double* ritz_block;     /* (device, optional) n x block warm block for next step  */
  int64_t ld_ritz;
  double lambda_r_plus_1; /* y[r]                                                   */
  double b_r_plus_1;      /* sum(y)                                                 */
  double shift;           /* mu_1                                                   */
  double lhs_cheap;       /* certificate (meg.py:222-239)                           */
  int32_t holds_cheap;
  double threshold;
  double gram_err;        /* max |V^T V - I| of V_next                              */
  int32_t passes;
  int32_t restarts;
  int32_t ritz_cols;      /* columns written to ritz_block (<= 64)                  */
  double ritz_orth_err;   /* max |B^T B - I| of the returned Ritz block B           */
} megb200_step_result;

typedef struct megb200_solver megb200_solver;

/* library ------------------------------------------------------------------ */
int megb200_abi_version(void);
const char* megb200_last_error(void);
/* 0 if a CUDA device of compute capability 10.x is current, else an error. */
int megb200_device_check(int* sm_count);

/* solver handle: owns the device workspace for dimension n and block/basis
 * limits (max_block <= 64, max_basis <= 112).  One stream per handle. */
int megb200_solver_create(int64_t n, int32_t max_block, int32_t max_basis, int64_t max_lowrank,
                          int64_t max_nnz, megb200_solver** out);
void megb200_solver_destroy(megb200_solver* s);
int megb200_solver_set_stream(megb200_solver* s, void* cuda_stream);
/* bytes of device workspace held by the handle */
int64_t megb200_solver_workspace_bytes(const megb200_solver* s);

/* operator application W = A U (SymmetricOperator.apply, linalg.py:93-94;
 * logmap_operator(...).apply, meg.py:299-305).  U, W: (device) n x k. */
int megb200_operator_apply(megb200_solver* s, const megb200_operator* op, const double* U, int64_t ldu,
                           int32_t k, double* W, int64_t ldw);

/* logmap_operator(x, grad_apply, eta).apply (meg.py:287-307): W = (log X - eta grad) U.
 * The low-rank factors are gathered into the handle's workspace. */
int megb200_logmap_apply(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g, double eta,
                         const double* U, int64_t ldu, int32_t k, double* W, int64_t ldw);

/* All eigenpairs of a small dense symmetric matrix A (m <= 112, device, row-major, ld lda):
 * w (device, m) non-increasing, V (device, m x m row-major, column j = eigenvector j).  The
 * Rayleigh-Ritz solver of the block Krylov method (tridiagonalisation + multisection + twisted
 * factorisation, verified to 1e-12 ||A||_F, Jacobi fallback) used directly; the dense-shadow
 * diagnostics (exact MEG, meg.py:269-284; Bregman distances, entropy.py:76-96) call it. */
int megb200_sym_eigh(megb200_solver* s, const double* A, int64_t lda, int32_t m, double* w, double* V);

/* grad f(X_g) U for any gradient descriptor (the device form of calling the reference's
 * grad_apply(u), meg.py:327-335): W (n x k, ld ldw) = G U.  Makes the descriptors callables. */
int megb200_gradient_apply(megb200_solver* s, const megb200_gradient* g, const double* U, int64_t ldu, int32_t k,
                           double* W, int64_t ldw);

/* lanczos_top_r (linalg.py:130-241): the r algebraically largest eigenpairs. */
int megb200_top_r(megb200_solver* s, const megb200_operator* op, int32_t r, const megb200_eig_opts* opts,
                  megb200_eig_result* out);

/* lowrank_meg_step (meg.py:327-364): one low-rank MEG update + cheap certificate. */
int megb200_lowrank_meg_step(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g, double eta,
                             double eps_next, const megb200_eig_opts* opts, megb200_step_result* out);

/* The step for a caller whose iterate factor lives in HOST memory: x->V and
 * V_next_host are host pointers (pinned memory makes the copies asynchronous).
 * In one call the factor is uploaded, validated (V^T V = I to 1e-10,
 * meg.py:69-71, before the step: MEGB200_ERR_PARAM otherwise), stepped, and
 * V_next read back.  A Frobenius / stochastic / sampled gradient with gV == NULL
 * is evaluated at the uploaded iterate.  out->V_next is not used. */
int megb200_lowrank_meg_step_host(megb200_solver* s, const megb200_iterate* x_host, const megb200_gradient* g,
                                  double eta, double eps_next, const megb200_eig_opts* opts, double* V_next_host,
                                  int64_t ld_next_host, megb200_step_result* out);

/* Run loop: T low-rank MEG steps from x0 without returning between steps --
 * the driver of test_meg.py:150-156 / the harness loop of SPEC.md:433-450,
 * absent from the reference code.  Step t = t0 + i uses eta_t, eps_next =
 * eps_{t+1} and svd_seed = t; the gradient is evaluated at the current iterate
 * (g's gV / g_lam / g_eps are ignored; STOCHASTIC regenerates A_t per step
 * into g->A).  flush_bytes > 0 writes that much scratch between steps,
 * outside the per-step events, to evict the operand from L2. */
enum {
  MEGB200_EPS_EXPERIMENT = 0,        /* 0.6/(t+c+1)^2                 meg.py:182-190 */
  MEGB200_EPS_CUBIC_DET = 1,         /* eps0/(2 max(G^2,1))/(t+1+c)^3 */
  MEGB200_EPS_CUBIC_DET_GENERAL = 2, /* 3 eps0/(2 max(G^2,1))/(t+c+1)^3 */
  MEGB200_EPS_QUADRATIC_STOCH = 3,   /* (9/32) eps0/(t+c+1)^2        */
  MEGB200_EPS_CONSTANT = 4           /* eps0_tilde                    */
};
enum { MEGB200_ETA_CONSTANT = 0, MEGB200_ETA_INV_SQRT = 1 /* eta0 / sqrt(t + 1) */ };

typedef struct megb200_schedule {
  int32_t eps_kind;
  double eps0_tilde, G, c;
  int32_t eta_kind;
  double eta0;
  uint64_t minibatch_seed;     /* STOCHASTIC: A_t = N(0,1/n) at stream 5, counter (t n + i) b + j */
  int32_t minibatch_round_f32; /* round A_t through float32 (f32 configs)                         */
  int32_t cert_every;          /* > 0: dual-gap certificate of X_{t+1} after every step t with      */
                               /* (t + 1) % cert_every == 0 (_dual_gap_core objectives.py:332-335;  */
                               /* FROBENIUS only), warm-started from the previous certificate      */
} megb200_schedule;

typedef struct megb200_run_record { /* host arrays, any may be NULL; row i = step t0 + i */
  double* shift;   /* T           */
  double* y;       /* T x (r + 1) */
  double* lam;     /* T x r       */
  double* eps;     /* T           */
  double* lhs;     /* T           */
  int32_t* holds;  /* T           */
  int32_t* passes; /* T           */
  double* step_ms; /* T: device time per step: previous step end -> this step end, minus the flush */
  /* final warm Ritz block (device, n x ritz_cap, leading dim ld_ritz) so a later run or step
   * continues warm: ritz_cols and ritz_orth_err are written when ritz_block is set */
  double* ritz_block;
  int64_t ld_ritz;
  int64_t ritz_cap;
  int64_t ritz_cols;
  double ritz_orth_err;
  /* optional sub-range timing: when timed_count > 0, CUDA events on the solver stream bracket
   * steps [timed_from, timed_from + timed_count) inside the loop (the device time of exactly those
   * steps in the pipelined steady state, the earlier steps being the warm-up);
   * timed_ms and timed_launches (kernels enqueued for those steps) are written back */
  int64_t timed_from;
  int64_t timed_count;
  double timed_ms;
  int64_t timed_launches;
  double* gap;  /* T: dual gap of X_{t+1} at certificate steps, NaN elsewhere (sch->cert_every)       */
  double* lmin; /* T: lambda_min(grad f(X_{t+1})) at certificate steps, NaN elsewhere                */
} megb200_run_record;

int megb200_meg_run(megb200_solver* s, const megb200_iterate* x0, const megb200_gradient* g,
                    const megb200_schedule* sch, int64_t t0, int64_t T, const megb200_eig_opts* opts,
                    uint64_t flush_bytes, double* V_out, int64_t ld_out, double* lam_out, double* eps_out,
                    megb200_run_record* rec);

/* certificate_cheap arithmetic (meg.py:222-239), host-only. */
int megb200_certificate_cheap(double lambda_r_plus_1, double b_r_plus_1, double eps, int64_t n, int64_t r,
                              double* lhs, int32_t* holds, double* threshold);

/* Objective evaluation from factors:
 *   FROBENIUS / STOCHASTIC: 1/2 ||X - M||_F^2  (needs ||M||_F^2 and Tr M:
 *                           pass NaN to have them computed and cached)
 *   SAMPLED:                1/2 sum_Omega (X_ij - Mobs_ij)^2
 * X is the gradient's (gV, g_lam, g_eps). */
int megb200_objective_value(megb200_solver* s, const megb200_gradient* g, double m_norm2, double m_trace,
                            double* value);

/* The same value summed entry by entry, 1/2 sum_ij (X_ij - M_ij)^2 with X_ij from the factors
 * (one pass over M, r FMAs per entry; no cancellation when X -> M, so the value compares
 * RELATIVELY).  SAMPLED descriptors take the entry sum above.  r <= 64. */
int megb200_objective_value_direct(megb200_solver* s, const megb200_gradient* g, double* value);

/* ||M||_F^2 and Tr M of a dense symmetric operand. */
int megb200_dense_stats(megb200_solver* s, const void* M, int32_t dtype, int64_t ld, double* norm2, double* trace);

/* Dual-gap certificate (_dual_gap_core, objectives.py:332-335) for the
 * Frobenius objective: Tr(X grad) - lambda_min(grad), grad = X - M, with
 * lambda_min from the block solver on M - X.  Also returns lambda_min. */
int megb200_dual_gap(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts, double m_trace,
                     double* gap, double* lambda_min);
/* The same certificate, also returning the solve's final Ritz block (device, n x *ritz_cols, ld
 * ld_ritz >= max_block) so the next certificate can start from it (opts->warm): the gradient
 * moves little between certificates, and a cold solve near the bulk edge takes ~200 passes. */
int megb200_dual_gap_warm(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts,
                          double m_trace, double* gap, double* lambda_min, double* ritz_out, int64_t ld_ritz,
                          int32_t* ritz_cols);

/* Quadratic-measurement objective (the paper's experiment; SURVEY.md 8f row 1,
 * reference objectives.py:111-228): f(tau X) = 1/2 sum_i (a_i^T (tau X) b_i - y_i)^2
 * over m unit-vector pairs a, b (m x n row-major, device, ld n).
 *   residuals: res_i = tau ((1-eps) sum_k (a_i.v_k) lam_k (v_k.b_i)
 *              + eps/(n-r) (a_i.b_i - sum_k (a_i.v_k)(v_k.b_i))) - y_i   (replaces
 *              _measure_structured / qm_residuals, objectives.py:111-130; 1 <= r <= 32)
 *   gradient:  G = weight * sym(a^T diag(res) b), n x n, ld ldg (replaces
 *              _dense_measurement_gradient, objectives.py:155-156; with weight = tau it is
 *              RecoveryObjective.grad_operator's tau * grad f(tau X), :211-223)
 *   value:     1/2 ||res||^2 (qm_value, objectives.py:133-136), host out.
 * eps = 0 evaluates X = V diag(lam) V^T for any V (spectral_init's probe, objectives.py:293-316).
 * Device pointers; n must equal the solver's dimension. */
int megb200_qm_residuals(megb200_solver* s, const double* a, const double* b, const double* y, int64_t m,
                         const double* V, int64_t ldv, int32_t r, const double* lam_host, double eps, double tau,
                         double* res);
int megb200_qm_gradient(megb200_solver* s, const double* a, const double* b, const double* res, int64_t m,
                        double weight, double* G, int64_t ldg);
int megb200_qm_value(megb200_solver* s, const double* res, int64_t m, double* value);
/* Mini-batch estimate (StochasticOracle.grad_operator, objectives.py:235-273): G = weight *
 * sym(a[idx]^T diag(res[idx]) b[idx]) over the L measurement indices idx (device int64, repeats
 * allowed; the caller folds tau * m / L into weight). */
int megb200_qm_gradient_batch(megb200_solver* s, const double* a, const double* b, const double* res,
                              const int64_t* idx, int64_t L, double weight, double* G, int64_t ldg);

/* Matrix-free block application of the measurement gradient (k <= 32): W (n x k, ld ldw) = Op U for the
 * QUADMEAS operator above; and the scratch it needs, in doubles. */
int64_t megb200_qm_apply_scratch(megb200_solver* s, int64_t m, int32_t k);
int megb200_qm_apply(megb200_solver* s, const megb200_qm_data* q, const double* U, int64_t ldu, int32_t k,
                     double* W, int64_t ldw);

/* Synthetic config-3 instance (seeded counter-based twin of oracle/inputs.sampled_instance):
 * pattern = symmetric Bernoulli(p) over i <= j at counter min*n + max of stream 3, mirrored;
 * _pattern writes rowptr (n + 1, device int32) and the nonzero count, _values fills col (sorted
 * per row) and val = (U diag(lam) U^T)_ij + obs_noise N(0,1) (stream 4, same counter). */
int megb200_gen_sampled_pattern(megb200_solver* s, uint64_t seed, double p, int32_t* rowptr, int64_t* nnz);
int megb200_gen_sampled_values(megb200_solver* s, uint64_t seed, double p, const double* U, int64_t r,
                               const double* lam_host, double obs_noise, const int32_t* rowptr, int32_t* col,
                               double* val);

/* Seeded synthetic inputs (oracle/inputs.py twins):
 *   M_ij = sum_k U_ik lam_k U_jk + sigma (g_ij + g_ji) / (2 sqrt(n)),
 *   g_ij = N(0,1) at counter i*n + j of stream `stream` (float64 or float32 output). */
int megb200_gen_dense_target(megb200_solver* s, const double* U, int64_t r, const double* lam_host, double sigma,
                             uint64_t seed, int32_t stream, void* M, int32_t dtype, int64_t ld);
/* out_ij = scale * N(0,1) at counter base + i*k + j (n x k row-major, ld).  If
 * round_f32 != 0 the values are rounded through float32. */
int megb200_gen_gaussian(megb200_solver* s, uint64_t seed, int32_t stream, uint64_t base, int64_t n, int64_t k,
                         double scale, int32_t round_f32, double* out, int64_t ld);

/* max |V^T V - I| of an n x r block (LowRankIterate validation, meg.py:69-71). */
int megb200_gram_error(megb200_solver* s, const double* V, int64_t ldv, int32_t r, double* err);

/* Live pass profiling (bench.py roofline): when enabled, every k-th streamed
 * operand pass kernel (dense or CSR product) is bracketed by CUDA events on the
 * solver stream.  read() synchronises, returns the summed time (ms) of the
 * bracketed passes, their number and their algorithmic bytes (operand + U read
 * + partial write), and resets the counters. */
int megb200_profile_enable(megb200_solver* s, int32_t enable); /* enable = k > 0: every k-th pass; 0: off */
int megb200_profile_read(megb200_solver* s, double* pass_ms, int64_t* passes, double* bytes);

/* Phase tracer (diagnostics): CUDA events at solver phase boundaries; the
 * report lists the average device time per phase tag. */
int megb200_trace_enable(megb200_solver* s, int32_t enable);
int megb200_trace_report(megb200_solver* s, char* buf, int64_t len);

/* counters of the last call (for benchmarks): kernels launched. */
int64_t megb200_kernel_launches(const megb200_solver* s);

#ifdef __cplusplus
}
#endif
#endif /* MEGB200_H */
