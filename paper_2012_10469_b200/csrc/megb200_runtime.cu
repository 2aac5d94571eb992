// Host runtime of the B200 low-rank MEG path: solver handle / workspace arena,
// the block thick-restart Lanczos eigensolver (replaces lanczos_top_r,
// linalg.py:130-241), the MEG step (replaces lowrank_meg_step,
// meg.py:327-364), objective values and the dual-gap certificate, and the
// extern "C" entry points declared in include/megb200.h.

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <functional>
#include <string>
#include <vector>

#include "megb200_internal.h"

#include <mutex>
#include <set>

namespace megb200 {
bool first_on_device(const void* tag) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  MEG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  return done.insert({dev, tag}).second;
}
}  // namespace megb200

using namespace megb200;

namespace {

thread_local std::string g_last_error;
// live solver handles (telemetry)
std::atomic<int> g_live_solvers{0};

constexpr int kMaxBlock = 64;
constexpr int kMaxBasis = 112;  // Jacobi Rayleigh-Ritz keeps H and S in shared memory

inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct megb200_solver {
  int64_t n = 0;
  int max_block = 0, max_basis = 0, cap = 0;
  int64_t max_lowrank = 0, max_nnz = 0;
  int sm_count = 148;
  // grid limit of the multi-pass solver's cooperative kernels: sm_count, or sm_count - 1 while a solve
  // overlaps its wide Rayleigh-Ritz (one CTA on the side stream) with the next block's work
  int coop_sm = 148;
  // Q^T W (a column block of H) and W^T W left by the finish of the last block pass, for the
  // orthonormalisation of W as the next Krylov block (block_pass / orthonormalize)
  bool pre_valid = false;
  const double *pre_src = nullptr, *pre_c = nullptr, *pre_g = nullptr;
  int pre_cols = 0, pre_q = 0;
  cudaStream_t stream = nullptr;
  // side stream of the overlapped wide Rayleigh-Ritz (top_eigs), forked / joined with events
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t launches = 0;
  // panel pointers of the tiled CSR pass (n x 17 int32, allocated on first use) and their key
  int32_t* csr_pp = nullptr;
  bool csr_pp_valid = false, in_solve = false;
  const int32_t *csr_pp_rowptr = nullptr, *csr_pp_col = nullptr;
  int csr_pp_b = 0;

  char* arena = nullptr;
  int64_t arena_bytes = 0;
  // tall-skinny (row-major, ld = cap)
  double *Q = nullptr, *AQ = nullptr, *T = nullptr;
  int64_t ldq = 0;
  double* W = nullptr;      // n x max_block
  double* part = nullptr;   // apply partial slices
  int64_t part_slices = 0;
  double* red = nullptr;    // reduction partials
  int64_t red_cap = 0;
  double* L = nullptr;      // n x max_lowrank
  double* E = nullptr;      // max_lowrank x max_block
  double* dvec = nullptr;   // max_lowrank
  double* dlam = nullptr;   // 64: kept weights of the current iterate (device copy)
  double* uT = nullptr;     // float32 operand-pass scratch (64 x n floats)
  double* host_io = nullptr;  // 2 x n x 64: device copies of a host caller's V / V_next
  double* H = nullptr;      // cap x cap
  double* C = nullptr;      // cap x max_block
  double* C2 = nullptr;
  double *G = nullptr, *R1 = nullptr, *R2 = nullptr, *Rinv = nullptr, *Rn = nullptr, *Rtmp = nullptr;
  int* mask = nullptr;
  double *theta = nullptr, *S = nullptr, *est = nullptr, *info = nullptr, *resid = nullptr;
  double* small = nullptr;  // misc device scalars
  // per-pass result pack, read back with ONE device-to-host copy:
  // [theta (cap) | resid (64) | step epilogue (136) | Ritz-block Gram (<= 64 x 64)]
  double* pack = nullptr;
  int64_t pack_resid = 0, pack_epi = 0, pack_gram = 0, pack_len = 0;
  double* csr_g = nullptr;  // max_nnz
  double* rowsq = nullptr;  // n
  double* h_buf = nullptr;  // pinned host staging
  double* h_buf_dev = nullptr;  // its device alias (mapped pinned memory), or null
  int64_t h_buf_len = 0;
  unsigned* fsync = nullptr;  // tickets / flags of the fused first-pass kernel (zeroed)
  unsigned epoch = 0;
  // early release of a fused first pass's Ritz rows to the next operand pass (FusedPassArgs):
  // cumulative count of fused CTAs launched, the last fused launch's epoch, and the launch counter
  // right after it (a pass launched with nothing in between waits on the counter)
  unsigned long long rows_target = 0;
  unsigned last_fused_epoch = 0;
  int64_t launches_after_fused = -1;
  int last_pack_count = 0;
  bool last_pack_host = false;
  int want_vgram = 0;      // host-buffer step: fused phase 0 also reduces the factor Gram (r x r)
  // kept weights of the current iterate, uploaded lazily: the fused first pass takes them as
  // kernel arguments, other consumers flush them to dlam first
  double dlam_host[64] = {};
  int dlam_n = 0;
  bool dlam_dirty = false;
  void flush_dlam() {
    if (dlam_dirty) {
      h2d(dlam, dlam_host, dlam_n);
      dlam_dirty = false;
    }
  }
  bool vgram_done = false;
  int64_t pack_vgram = 0;  // its offset in the result pack
  double* qm_part = nullptr;  // quadratic-measurement gradient split-K partials (grown on demand)
  int64_t qm_part_len = 0;
  int rr_nvec = 0;  // Ritz pairs a wide Rayleigh-Ritz must return (0: all); set by top_eigs
  double m_norm2_cache = NAN, m_trace_cache = NAN;
  const void* m_cache_ptr = nullptr;
  // run-loop buffers (allocated on first megb200_meg_run)
  double* run_buf = nullptr;  // 2 x n x 64 (V ping-pong) + 2 x n x 64 (warm ping-pong)
  void* flush_buf = nullptr;
  uint64_t flush_len = 0;
  // live pass profiling
  int prof = 0;              // profile every prof-th streamed pass (0 = off)
  int64_t prof_seen = 0;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_pending;
  int ev_next = 0;
  double prof_bytes = 0.0;
  int64_t prof_passes = 0;
  // phase tracer: (tag, event) marks; segment time is attributed to the tag of its end mark
  bool trace = false;
  std::vector<std::pair<const char*, cudaEvent_t>> marks;
  std::vector<cudaEvent_t> trace_pool;
  size_t trace_next = 0;
  std::vector<std::pair<std::string, std::pair<double, int64_t>>> trace_acc;
  std::vector<std::pair<std::string, std::pair<double, int64_t>>> trace_stat;  // (name, (sum, count))
  void stat(const std::string& name, double v) {
    for (auto& kv : trace_stat)
      if (kv.first == name) {
        kv.second.first += v;
        kv.second.second += 1;
        return;
      }
    trace_stat.push_back({name, {v, 1}});
  }
  void mark(const char* tag) {
    if (!trace) return;
    if (trace_next == trace_pool.size()) {
      cudaEvent_t e;
      MEG_CUDA(cudaEventCreate(&e));
      trace_pool.push_back(e);
    }
    cudaEvent_t e = trace_pool[trace_next++];
    MEG_CUDA(cudaEventRecord(e, stream));
    marks.emplace_back(tag, e);
  }
  void trace_collect() {
    if (marks.size() >= 2) {
      MEG_CUDA(cudaEventSynchronize(marks.back().second));
      for (size_t i = 1; i < marks.size(); ++i) {
        float ms = 0.f;
        MEG_CUDA(cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second));
        const std::string tag = marks[i].first;
        bool found = false;
        for (auto& kv : trace_acc)
          if (kv.first == tag) {
            kv.second.first += ms;
            kv.second.second += 1;
            found = true;
          }
        if (!found) trace_acc.push_back({tag, {ms, 1}});
      }
    }
    marks.clear();
    trace_next = 0;
  }
  cudaEvent_t next_event() {
    if (ev_next == (int)ev_pool.size()) {
      cudaEvent_t e;
      MEG_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }

  // pinned upload ring for the small per-step host->device copies (coefficients):
  // truly asynchronous, reset at every stream synchronisation
  double* h_up = nullptr;
  int64_t h_up_len = 0, h_up_cur = 0;

  Launch launch() { return Launch{stream, &launches}; }
  void sync() {
    MEG_CUDA(cudaStreamSynchronize(stream));
    h_up_cur = 0;
  }
  void d2h(double* host, const double* dev, int64_t count) {
    if (count <= 0) return;
    MEG_CUDA(cudaMemcpyAsync(host, dev, count * sizeof(double), cudaMemcpyDeviceToHost, stream));
  }
  void h2d(double* dev, const double* host, int64_t count) {
    if (count <= 0) return;
    if (count > h_up_len) {
      MEG_CUDA(cudaMemcpyAsync(dev, host, count * sizeof(double), cudaMemcpyHostToDevice, stream));
      return;
    }
    if (h_up_cur + count > h_up_len) sync();
    double* stage = h_up + h_up_cur;
    std::copy(host, host + count, stage);
    h_up_cur += count;
    MEG_CUDA(cudaMemcpyAsync(dev, stage, count * sizeof(double), cudaMemcpyHostToDevice, stream));
  }
};

namespace {

// ---------------------------------------------------------------------------
// operators

struct OpDev {
  int kind = MEGB200_OP_NONE;
  int dtype = MEGB200_F64;
  const void* dense = nullptr;
  int64_t ld = 0;
  const int32_t* rowptr = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
  int64_t nnz = 0;
  double scale = 0.0;
  const double* L = nullptr;
  int64_t ldl = 0;
  int l = 0;
  const double* d_dev = nullptr;  // device coefficients (length l)
  LamCoef lc;                     // or the first lc.lr of them from device-resident kept weights
  double alpha = 0.0;
  const double* Eg = nullptr;     // device L^T U when the caller already has it (else reduced per pass)
  int64_t ldg = 0;
  const double* Gu = nullptr;     // device U^T U when the caller already has it (with Eg)
  int64_t ldgu = 0;
  megb200_apply_fn apply = nullptr;  // CALLBACK: the caller's block application
  void* apply_ctx = nullptr;
};

constexpr int kRowsCtrWord = 512;     // u64 at words 512..513: fused CTAs whose Ritz rows are final
constexpr int kDoneFlagWord = 520;    // epoch of the last fused launch whose result pack is written

// Live pass profiling (megb200_profile_enable): every prof-th streamed pass kernel is bracketed
// by events on the solver stream; prof_end books its algorithmic bytes (operand as stored + the
// n x k float64 block read and written).
int prof_begin(megb200_solver* s) {
  if (!(s->prof > 0 && (s->prof_seen++ % s->prof) == 0)) return -1;
  const int ev0 = s->ev_next;
  MEG_CUDA(cudaEventRecord(s->next_event(), s->stream));
  return ev0;
}

void prof_end(megb200_solver* s, int ev0, const OpDev& op, int k) {
  if (ev0 < 0) return;
  const int64_t n = s->n;
  const int ev1 = s->ev_next;
  MEG_CUDA(cudaEventRecord(s->next_event(), s->stream));
  s->ev_pending.emplace_back(ev0, ev1);
  const double es = op.kind == MEGB200_OP_DENSE ? (op.dtype == MEGB200_F64 ? 8.0 : 4.0) : 0.0;
  double b = 2.0 * (double)n * k * 8.0;  // read U, write W (float64)
  if (op.kind == MEGB200_OP_DENSE) b += (double)n * (double)n * es;
  if (op.kind == MEGB200_OP_CSR) b += (double)op.nnz * 12.0 + (double)(n + 1) * 4.0;
  s->prof_bytes += b;
  s->prof_passes++;
}

void check_qm_data(const megb200_qm_data* q) {
  if (!q || !q->a || !q->b || !q->res || q->m < 1 || !q->scratch)
    throw Error(MEGB200_ERR_PARAM, "quadratic-measurement operator data missing");
}

// Streamed operand pass alone: partial slices of Op U into s->part; returns the slice count.
int pass_launch(megb200_solver* s, const OpDev& op, const double* U, int64_t ldu, int k) {
  Launch L = s->launch();
  static const bool no_rows_wait = getenv("MEGB200_NO_ROWS_WAIT") != nullptr;  // diagnostics
  if (!no_rows_wait && s->launches == s->launches_after_fused) {
    // directly after a fused first pass: wait for its Ritz rows, not for its residual reduction
    L.wait_ctr = reinterpret_cast<const unsigned long long*>(s->fsync + kRowsCtrWord);
    L.wait_target = s->rows_target;
  }
  const int64_t n = s->n;
  int S = 0;
  const bool streamed = (op.kind == MEGB200_OP_DENSE || op.kind == MEGB200_OP_CSR) && op.scale != 0.0;
  if (op.kind == MEGB200_OP_CALLBACK && op.scale != 0.0) {
    // the caller's application writes the one partial slice (n x k, ld k) on the solver stream
    const int rc = op.apply(op.apply_ctx, U, ldu, k, s->part, k, (void*)s->stream);
    if (rc != 0) throw Error(MEGB200_ERR_CALLBACK, "apply callback failed (returned " + std::to_string(rc) + ")");
    // the callback's last stream operation may be a copy: the programmatically dependent launches
    // that follow only order against kernels, so its completion is waited for here
    s->sync();
    return 1;
  }
  if (op.kind == MEGB200_OP_QUADMEAS && op.scale != 0.0) {
    // matrix-free quadratic-measurement gradient: two streaming passes over a and b write the one slice
    const megb200_qm_data* q = static_cast<const megb200_qm_data*>(op.apply_ctx);
    if (q->scratch_len < qm_apply_scratch_doubles(q->m, n, k, s->sm_count))
      throw Error(MEGB200_ERR_PARAM, "quadratic-measurement scratch too small (megb200_qm_apply_scratch)");
    qm_apply(L, q->a, q->b, q->res, q->idx, q->m, n, q->weight, U, ldu, k, s->part, q->scratch, s->sm_count);
    return 1;
  }
  // live profiling brackets the streamed operand kernel only (the roofline's dominant kernel)
  const int ev0 = streamed ? prof_begin(s) : -1;
  if (op.kind == MEGB200_OP_DENSE && op.scale != 0.0) {
    S = dense_apply_partial(L, op.dense, op.dtype, op.ld, n, U, ldu, k, s->part, s->part_slices, s->sm_count,
                            reinterpret_cast<float*>(s->uT));
  } else if (op.kind == MEGB200_OP_CSR && op.scale != 0.0) {
    // panel pointers are computed once per solve (the pattern cannot change inside top_eigs), per
    // pass outside one
    const bool same = s->in_solve && s->csr_pp_rowptr == op.rowptr && s->csr_pp_col == op.col && s->csr_pp_b == k;
    if (!same) s->csr_pp_valid = false;
    if (!s->csr_pp) {
      if (cudaMalloc(&s->csr_pp, (size_t)n * (kCsrMaxPanels + 1) * sizeof(int32_t)) != cudaSuccess) {
        cudaGetLastError();
        s->csr_pp = nullptr;
      }
    }
    S = csr_apply_partial(L, op.rowptr, op.col, op.val, n, U, ldu, k, s->part, s->part_slices, s->csr_pp,
                          &s->csr_pp_valid, s->sm_count);
    s->csr_pp_rowptr = op.rowptr;
    s->csr_pp_col = op.col;
    s->csr_pp_b = k;
  }
  prof_end(s, ev0, op, k);
  return S;
}

void apply_op(megb200_solver* s, const OpDev& op, const double* U, int64_t ldu, int k, double* W, int64_t ldw,
              int hp = 0, double* Hout = nullptr, double* Gout = nullptr) {
  Launch L = s->launch();
  const int S = pass_launch(s, op, U, ldu, k);
  if (op.lc.lam == s->dlam) s->flush_dlam();
  coop_finish(L, s->n, k, S, s->part, op.scale, op.L, op.ldl, op.l, op.d_dev, op.alpha, U, ldu, W, ldw, s->E, s->red,
              s->coop_sm, Hout ? s->Q : nullptr, s->ldq, hp, Hout, s->cap, op.lc, op.Eg, op.ldg, Gout);
}

// columns k > 64 are applied in chunks (re-streams the operand; not used by the configs)
void apply_op_wide(megb200_solver* s, const OpDev& op, const double* U, int64_t ldu, int k, double* W, int64_t ldw) {
  const int chunk = std::min(32, s->max_block);
  for (int c0 = 0; c0 < k; c0 += chunk) {
    const int kc = std::min(chunk, k - c0);
    apply_op(s, op, U + c0, ldu, kc, W + c0, ldw);
  }
}

OpDev op_from_public(megb200_solver* s, const megb200_operator* op) {
  if (!op) throw Error(MEGB200_ERR_PARAM, "operator is NULL");
  if (op->n != s->n) throw Error(MEGB200_ERR_PARAM, "operator dimension does not match the solver");
  OpDev o;
  o.kind = op->kind;
  o.dtype = op->dtype;
  o.dense = op->dense;
  o.ld = op->ld;
  o.rowptr = op->rowptr;
  o.col = op->col;
  o.val = op->val;
  o.nnz = op->nnz;
  o.scale = op->scale;
  o.alpha = op->alpha;
  o.apply = op->apply;
  o.apply_ctx = op->apply_ctx;
  if (o.kind == MEGB200_OP_CALLBACK && !o.apply) throw Error(MEGB200_ERR_PARAM, "callback operator without apply");
  if (o.kind == MEGB200_OP_QUADMEAS) check_qm_data(static_cast<const megb200_qm_data*>(o.apply_ctx));
  if (o.kind == MEGB200_OP_DENSE && (!o.dense || o.ld < s->n)) throw Error(MEGB200_ERR_PARAM, "dense operand missing");
  if (o.kind == MEGB200_OP_CSR && (!o.rowptr || !o.col || !o.val)) throw Error(MEGB200_ERR_PARAM, "CSR operand missing");
  if (op->l > 0) {
    if (op->l > s->max_lowrank) throw Error(MEGB200_ERR_PARAM, "low-rank width exceeds the solver's max_lowrank");
    if (!op->L || !op->d) throw Error(MEGB200_ERR_PARAM, "low-rank factor or coefficients missing");
    o.L = op->L;
    o.ldl = op->ldl;
    o.l = (int)op->l;
    s->h2d(s->dvec, op->d, op->l);
    o.d_dev = s->dvec;
  }
  return o;
}

// ---------------------------------------------------------------------------
// block orthonormalisation: W (n x q, ld ldw) against Q[:, 0:cols] with two
// cooperative CGS rounds, then two cooperative CholQR rounds (breakdown ->
// seeded random refill, the rule of linalg.py:193-199).  With want_relation
// the relation factor Rn = R2 R1 (W_in - Q C = W_out Rn) is formed.

void orthonormalize(megb200_solver* s, double* W, int64_t ldw, int q, int cols, double scale, uint64_t key,
                    uint64_t& refill_ctr, bool want_relation, int cgs_rounds = 2, const double* src = nullptr,
                    int64_t lds = 0) {
  Launch L = s->launch();
  const int64_t n = s->n;
  // src: the block to orthonormalise lives elsewhere (the image block of the previous pass); the fused
  // kernel reads it there and writes W, the fallback copies it first
  // the finish of the pass that produced src already reduced Q^T src and src^T src (block_pass)
  const bool pre = s->pre_valid && src && src == s->pre_src && cols == s->pre_cols && q == s->pre_q && lds == s->ldq;
  s->pre_valid = false;
  if (!want_relation && coop_orth(L, n, s->Q, s->ldq, cols, W, ldw, q, 1e-13 * scale, key, refill_ctr, s->red, s->C2,
                                  s->G, s->Rinv, s->mask, s->Rtmp, s->coop_sm, cgs_rounds, src, lds,
                                  pre ? s->pre_c : nullptr, s->cap, pre ? s->pre_g : nullptr)) {
    refill_ctr += 2 * (uint64_t)n * q;
    return;
  }
  if (src) copy_block(L, n, q, src, lds, W, ldw);
  for (int round = 0; round < cgs_rounds && cols > 0; ++round)
    coop_cgs(L, n, s->Q, s->ldq, cols, W, ldw, q, s->C2, s->red, s->coop_sm);
  coop_cholqr(L, n, W, ldw, W, ldw, q, 1e-13 * scale, s->G, s->R1, s->Rinv, s->mask, nullptr, nullptr, key,
              refill_ctr, s->red, s->coop_sm);
  refill_ctr += (uint64_t)n * q;
  if (cols > 0) coop_cgs(L, n, s->Q, s->ldq, cols, W, ldw, q, s->C2, s->red, s->coop_sm);
  coop_cholqr(L, n, W, ldw, W, ldw, q, 0.0, s->G, s->R2, s->Rinv, s->mask, want_relation ? s->R1 : nullptr,
              want_relation ? s->Rn : nullptr, key, refill_ctr, s->red, s->coop_sm);
  refill_ctr += (uint64_t)n * q;
}

// ---------------------------------------------------------------------------
// block thick-restart Lanczos (device Krylov-Schur) for the nreq algebraically
// largest eigenpairs.

struct EigRun {
  std::vector<double> theta, resid;
  int passes = 0, restarts = 0;
  double norm_est = 1.0;
  bool converged = false;
};

struct EigParams {
  double tol = 1e-10;
  int max_passes = 0;
  int restarts = 12;
  int block = 0, basis = 0, keep = 0;
  uint64_t seed = 0;
  const double* warm = nullptr;
  int64_t warm_cols = 0, ld_warm = 0;
  bool warm_orthonormal = false;
};

EigParams params_from_opts(const megb200_eig_opts* o) {
  EigParams p;
  if (!o) return p;
  if (o->tol > 0) p.tol = o->tol;
  p.max_passes = o->max_passes;
  if (o->restarts > 0) p.restarts = o->restarts;
  p.block = o->block;
  p.basis = o->basis;
  p.keep = o->keep;
  p.seed = o->seed;
  p.warm = o->warm;
  p.warm_cols = o->warm ? o->warm_cols : 0;
  p.ld_warm = o->ld_warm;
  p.warm_orthonormal = o->warm && o->warm_orthonormal != 0;
  return p;
}

// Speculative per-pass MEG epilogue: computed with the Rayleigh-Ritz launch and
// read back with the convergence data, so a converged step costs one sync.
struct EpiSpec {
  int r = 0;             // > 0: run the step epilogue for r kept pairs (nreq = r + 1)
  double eps_next = 0.0;
  int gr = 0;                // out: order of the returned Ritz-block Gram
  std::vector<double> host;  // out: epilogue block (2r + 8 doubles) + Gram (gr x gr)
  double* v_next = nullptr;  // in: V_next = first r Ritz vectors, written with the outputs
  int64_t ld_next = 0;
  double* v_host = nullptr;  // in: host copy of V_next read back with the pack (host-buffer step)
  int64_t ld_host = 0;
  bool v_host_done = false;  // out: v_host holds the converged V_next
};

// Block sizes of a solve: block width bw, basis limit mmax, thick-restart keep.
struct EigShape {
  int bw = 1, mmax = 1, keep = 1, max_passes = 1;
  bool exhaust = false;
  // n <= the Rayleigh-Ritz limit with a basis allowed to span R^n: the basis IS the identity (no
  // start block, no orthonormalisation), A I in passes of <= 32 columns, one Rayleigh-Ritz on all of
  // A returning only the Ritz pairs the step needs (linalg.py:215's basis.shape[1] >= n exit)
  bool identity = false;
};

EigShape eig_shape(const megb200_solver* s, int nreq, const EigParams& P) {
  const int64_t n = s->n;
  if (!(1 <= nreq && nreq < n)) throw Error(MEGB200_ERR_PARAM, "need 1 <= r < n, got r=" + std::to_string(nreq) + ", n=" + std::to_string(n));
  int bw = P.block > 0 ? P.block : std::min(s->max_block, nreq + 7);
  // basis: the reference's `subspace` (basis size of its single-vector Lanczos)
  // is honoured as a lower bound; a block method needs several blocks per cycle,
  // so the default is 6 blocks (<= 112, the Rayleigh-Ritz limit)
  if (P.basis > 0 && P.block <= 0) bw = std::max(1, std::min(bw, P.basis / 2));
  static const int blocks_per_basis = [] {  // diagnostics override (MEGB200_BASIS_BLOCKS), default 6
    const char* e = getenv("MEGB200_BASIS_BLOCKS");
    return e ? std::max(2, atoi(e)) : 6;
  }();
  int mmax = std::max({P.basis > 0 ? P.basis : 0, blocks_per_basis * bw, 2 * nreq + 10, 30});
  bw = std::max(1, std::min<int>(bw, s->max_block));
  mmax = std::min<int>(mmax, s->max_basis);
  mmax = std::max(mmax, std::min<int>(nreq + bw, s->max_basis));
  bool exhaust = false;
  if (n <= s->max_basis && n <= 64 && (P.basis <= 0 || P.basis >= n)) {  // tiny problems: span R^n exactly (basis.shape[1] >= n rule, linalg.py:215)
    bw = (int)std::min<int64_t>(n, s->max_block);
    mmax = (int)n;
    exhaust = true;
  }
  // small problems (n <= the Rayleigh-Ritz limit): let the basis grow to span R^n instead of
  // restarting -- a full basis converges by the basis.shape[1] >= n rule (linalg.py:215) with one
  // wide Rayleigh-Ritz, where restarted cycles near the bulk edge take tens of passes
  if (!exhaust && n <= s->max_basis && P.basis <= 0) {
    mmax = (int)n;
    // and a wider default block: four passes span R^n (each pass is latency-bound at this size)
    if (P.block <= 0) bw = std::min<int>(std::max<int>(bw, (int)((n + 3) / 4)), std::min(32, s->max_block));
  }
  mmax = (int)std::min<int64_t>(mmax, n);
  // even block widths and column offsets keep every block 16-byte aligned for the TMA pass
  if (!exhaust && (bw & 1) && bw < s->max_block && bw + 1 + nreq <= mmax) bw += 1;
  if (bw > mmax) bw = mmax;
  static const int keep_env = [] {  // diagnostics override of the default thick-restart size
    const char* e = getenv("MEGB200_KEEP");
    return e ? atoi(e) : 0;
  }();
  // default thick restart keeps a third of the basis (cfg3, n = 8192: 45.6 it/s vs 39.9 keeping half,
  // 42.7 keeping a quarter; the single-pass configs do not restart)
  int keep = P.keep > 0 ? P.keep : (keep_env > 0 ? std::max(nreq, keep_env) : std::max(nreq + 2, mmax / 3));
  keep = std::min(keep, mmax - bw);
  if (!exhaust && (keep & 1) && (bw & 1) == 0) keep = (keep + 1 <= mmax - bw) ? keep + 1 : (keep - 1 >= nreq ? keep - 1 : keep);
  if (!exhaust && keep < nreq) throw Error(MEGB200_ERR_PARAM, "basis too small for the requested eigenpairs");
  EigShape sh;
  static const bool no_identity = getenv("MEGB200_NO_IDENTITY_BASIS") != nullptr;  // diagnostics
  sh.identity = !no_identity && n <= s->max_basis && n <= s->cap && (P.basis <= 0 || P.basis >= n);
  if (sh.identity) {
    exhaust = true;
    mmax = (int)n;
    bw = (int)std::min<int64_t>(std::max(bw, std::min(nreq, 32)), std::min<int64_t>(32, n));
    keep = std::min(keep, mmax);
  }
  sh.bw = bw;
  sh.mmax = mmax;
  sh.keep = keep;
  sh.exhaust = exhaust;
  sh.max_passes = P.max_passes > 0 ? P.max_passes : P.restarts * mmax;
  return sh;
}

// One operator pass on the block Q[:, cols:cols+cur] into AQ, and its column of H = Q^T A Q.
void block_pass(megb200_solver* s, const OpDev& op, int cols, int cur) {
  Launch L = s->launch();
  s->pre_valid = false;
  if (cur <= 32) {
    // pass + epilogue; the epilogue launch also reduces the H column Q^T (A Q_j) and, in the same
    // reduction, the image block's Gram: together the first Pythagorean round of the orthonormalisation
    // of the next Krylov block (which is this image block) needs no reduction of its own
    double* gpre = s->small + 2048;  // 32 x 32
    apply_op(s, op, s->Q + cols, s->ldq, cur, s->AQ + cols, s->ldq, cols + cur, s->H + cols, gpre);
    s->pre_valid = true;
    s->pre_src = s->AQ + cols;
    s->pre_c = s->H + cols;
    s->pre_g = gpre;
    s->pre_cols = cols + cur;
    s->pre_q = cur;
  } else {
    apply_op_wide(s, op, s->Q + cols, s->ldq, cur, s->AQ + cols, s->ldq);
    coop_tn(L, s->n, s->Q, s->ldq, cols + cur, s->AQ + cols, s->ldq, cur, s->H + cols, s->cap, nullptr, 1.0, s->red,
            s->coop_sm);
  }
}

// Rayleigh-Ritz on H[0:newcols, 0:newcols] + Ritz block T + explicit residuals
// from the cached images (linalg.py:205-211) (+ speculative step epilogue and
// the Ritz-block Gram) in one launch, then one asynchronous read-back of the
// pack [theta | resid | epilogue | Gram] into dst (pinned).  Returns the Gram order.
int rr_readback(megb200_solver* s, int newcols, int nreq, int bw, const EpiSpec* epi, double* dst,
                double* tdst = nullptr, int64_t ldt = 0, double* v2 = nullptr, int64_t ld2 = 0, int r2 = 0,
                bool presolved = false) {
  Launch L = s->launch();
  const int rq = std::min(newcols, std::max(nreq, bw));
  const int gr = epi ? rq : 0;  // Gram of the whole Ritz block (V_next = its first r columns)
  if (!tdst) {
    tdst = s->T;
    ldt = s->ldq;
  }
  static const bool twice = getenv("MEGB200_DEBUG_RR_TWICE") != nullptr;  // diagnostics: warm i-cache timing
  for (int rep = 0; rep < (twice ? 2 : 1); ++rep)
    coop_rr(L, s->H, s->cap, newcols, s->theta, s->S, s->info, s->n, s->Q, s->AQ, s->ldq, rq, nreq, tdst, ldt,
            s->resid, s->red, s->coop_sm, gr, s->pack + s->pack_gram, epi ? epi->eps_next : 0.0,
            epi ? s->pack + s->pack_epi : nullptr, v2, ld2, r2, s->rr_nvec, presolved);
  s->d2h(dst, s->pack, s->pack_gram + (int64_t)gr * gr);
  return gr;
}

// The first pass of a solve through the fused kernel (megb200_step.cu): pass, then
// finish + H + Rayleigh-Ritz + Ritz block + residuals + Gram (+ epilogue) in one
// launch whose result pack lands in dst (pinned; written by the kernel itself when
// the staging buffer is mapped).  Same outputs as block_pass + rr_readback.
// per reduction: G partials + ceil(G / 8) group partials + the result, kFusedStride doubles each
constexpr int kTileGramTicket = 420;  // word of s->fsync (k_dense_step_mma uses words 256..418)
constexpr int64_t kFusedPart1 = (148 + 19 + 1) * (int64_t)kFusedStride;  // offsets in s->red
constexpr int64_t kFusedPart2 = 2 * kFusedPart1;
constexpr int64_t kFusedRed = 3 * kFusedPart1;

bool fused_ok(const megb200_solver* s, const OpDev& op, int bw, int nreq) {
  static const bool off = getenv("MEGB200_NO_FUSED") != nullptr;  // diagnostics: the two-kernel path
  return !off && s->sm_count <= 148 && s->red_cap >= kFusedRed && op.l <= kFusedMaxL && op.l <= s->max_lowrank &&
         nreq <= bw && fused_pass_supported(s->n, bw, op.l, nreq, s->sm_count);
}

// the pass + step tail in one launch applies (float64 dense operand, b <= 32, ...)
bool step_mma_ok(const megb200_solver* s, const OpDev& op, const double* U, int64_t ldu, int bw) {
  return op.kind == MEGB200_OP_DENSE && op.scale != 0.0 &&
         dense_step_mma_supported(op.dense, op.dtype, op.ld, s->n, U, ldu, bw, op.L ? op.l : 0, s->part_slices,
                                  s->sm_count);
}

int fused_pass(megb200_solver* s, const OpDev& op, const double* U, int64_t ldu, int bw, int nreq, const EpiSpec* epi,
               double* tdst, int64_t ldt, double* v2, int64_t ld2, int r2, double* dst) {
  Launch L = s->launch();
  const bool one_launch = step_mma_ok(s, op, U, ldu, bw);
  const int S = one_launch ? 0 : pass_launch(s, op, U, ldu, bw);
  FusedPassArgs a;
  a.n = s->n;
  a.b = bw;
  a.part = s->part;
  a.S = S;
  a.scale = op.scale;
  a.alpha = op.alpha;
  a.L = op.L;
  a.ldl = op.ldl;
  a.l = op.L ? op.l : 0;
  a.d = op.d_dev;
  a.lc = op.lc;
  if (op.lc.lam == s->dlam && s->dlam_dirty) {  // the iterate's weights as kernel arguments
    std::copy(s->dlam_host, s->dlam_host + s->dlam_n, a.lam_inline);
    a.lam_inline_n = s->dlam_n;
  }
  a.Eg = op.Eg;
  a.ldg = op.ldg;
  a.U = U;
  a.ldu = ldu;
  a.W = s->AQ;
  a.ldw = s->ldq;
  a.H = s->H;
  a.ldh = s->cap;
  a.theta = s->theta;
  a.Sout = s->S;
  a.info = s->info;
  a.T = tdst ? tdst : s->T;
  a.ldt = tdst ? ldt : s->ldq;
  a.V2 = v2;
  a.ld2 = ld2;
  a.r2 = v2 ? r2 : 0;
  a.resid = s->resid;
  a.rq = bw;
  a.gr = epi ? bw : 0;
  a.gram = s->pack + s->pack_gram;
  a.nreq = nreq;
  a.epi = epi ? s->pack + s->pack_epi : nullptr;
  a.eps_next = epi ? epi->eps_next : 0.0;
  a.part0 = s->red;
  a.part1 = s->red + kFusedPart1;
  a.part2 = s->red + kFusedPart2;
  a.Ews = s->E;
  a.sync = s->fsync;
  // always a cooperative launch: the release flags and last-CTA tickets need every CTA resident,
  // which only the driver's cooperative-launch guarantee provides against concurrent work (other
  // solver handles or streams, NCCL, MPS neighbours)
  a.cooperative = true;
  if (++s->epoch == 0) ++s->epoch;
  a.epoch = s->epoch;
  a.pack = s->pack;
  a.pack_count = (int)(s->pack_gram + (int64_t)a.gr * a.gr);
  if (!one_launch && s->want_vgram > 0 && !op.Eg && a.L && a.l >= s->want_vgram && s->want_vgram <= 32 &&
      a.l * bw + s->want_vgram * s->want_vgram <= kFusedStride) {
    a.vgram = s->pack + s->pack_vgram;
    a.nvg = s->want_vgram;
    a.pack_count = (int)(s->pack_vgram + (int64_t)a.nvg * a.nvg);
    s->vgram_done = true;
  }
  if (!one_launch) s->want_vgram = 0;
  a.host_pack = s->h_buf_dev ? s->h_buf_dev + (dst - s->h_buf) : nullptr;
  if (one_launch) {
    // E = diag(d) L^T U needs L^T U before the launch: carried over from the previous step's
    // Ritz-block Gram (op.Eg), else reduced here with the same products (k_tile_gram), which also
    // yields the Gram of the iterate's factor when the host-buffer step asked for it
    a.vgram = nullptr;
    a.pack_count = (int)(s->pack_gram + (int64_t)a.gr * a.gr);
    // H = U^T W is formed from U^T U too: the previous step's Ritz-block Gram when carried over
    // (pipelined: Eg is its first rows), else reduced with L^T U
    if (a.Eg && op.Gu) {
      a.Gu = op.Gu;
      a.ldgu = op.ldgu;
    } else {
      const int nvg = (s->want_vgram > 0 && s->want_vgram <= a.l && s->want_vgram <= 32) ? s->want_vgram : 0;
      tile_gram(L, s->n, a.L, a.ldl, a.l, U, ldu, bw, nvg, s->red, s->fsync + kTileGramTicket, s->E,
                nvg ? s->pack + s->pack_vgram : nullptr, s->E + (int64_t)a.l * bw);
      if (nvg) {
        a.pack_count = (int)(s->pack_vgram + (int64_t)nvg * nvg);
        s->vgram_done = true;
      }
      a.Eg = s->E;
      a.ldg = bw;
      a.Gu = s->E + (int64_t)a.l * bw;
      a.ldgu = bw;
    }
    s->want_vgram = 0;
    static const bool step_stamps = getenv("MEGB200_FUSED_STAMPS") != nullptr;
    if (step_stamps) {  // diagnostics: phase timestamps (maxima over CTAs), reset per launch
      a.stamps = reinterpret_cast<unsigned long long*>(s->fsync + 128);
      MEG_CUDA(cudaMemsetAsync(a.stamps, 0, 16 * sizeof(unsigned long long), s->stream));
    }
    const int ev0 = prof_begin(s);
    dense_step_mma(L, static_cast<const double*>(op.dense), op.ld, s->n, U, ldu, bw, s->part, s->part_slices,
                   s->sm_count, a);
    prof_end(s, ev0, op, bw);
    if (!a.host_pack) s->d2h(dst, s->pack, a.pack_count);
    return a.gr;
  }
  static const bool stamps = getenv("MEGB200_FUSED_STAMPS") != nullptr;
  if (stamps) a.stamps = reinterpret_cast<unsigned long long*>(s->fsync + 128);
  static const bool no_release = getenv("MEGB200_NO_EARLY_RELEASE") != nullptr;  // diagnostics
  if (!no_release) {
    a.rows_ctr = reinterpret_cast<unsigned long long*>(s->fsync + kRowsCtrWord);
    a.done_flag = s->fsync + kDoneFlagWord;
    a.prev_epoch = s->last_fused_epoch;
  }
  const int G = fused_first_pass(L, a, s->sm_count);
  if (!no_release) {
    s->rows_target += (unsigned long long)G;
    s->last_fused_epoch = a.epoch;
    s->launches_after_fused = s->launches;
  }
  s->last_pack_count = a.pack_count;
  s->last_pack_host = a.host_pack != nullptr && !no_release;
  if (!a.host_pack) s->d2h(dst, s->pack, a.pack_count);
  return a.gr;
}

// Convergence decision on a read-back pack (linalg.py:212-216): every wanted
// residual <= tol * max(1, max |theta|), or the basis spans R^n.
struct RRDecision {
  bool ok = false;
  double scale = 1.0, rmax = 0.0;
};

RRDecision rr_decide(const megb200_solver* s, const double* pk, int newcols, int nreq, double tol) {
  RRDecision d;
  double tmax = 0.0;
  for (int j = 0; j < newcols; ++j) tmax = std::max(tmax, fabs(pk[j]));
  d.scale = std::max(1.0, tmax);  // norm estimate max(1, max|theta_all|) (linalg.py:214)
  bool ok = true;
  for (int j = 0; j < nreq; ++j) {
    const double rj = pk[s->pack_resid + j];
    ok = ok && (rj <= tol * d.scale);
    d.rmax = std::max(d.rmax, rj);
  }
  d.ok = ok || (newcols >= s->n);
  return d;
}

// Outputs: eigenvectors (nreq) -> vec_out, top `bw` Ritz vectors -> ritz_out.
EigRun top_eigs(megb200_solver* s, const OpDev& op, int nreq, const EigParams& P, double* vec_out, int64_t ld_vec,
                double* ritz_out, int64_t ld_ritz, int* ritz_cols_out, EpiSpec* epi = nullptr) {
  const int64_t n = s->n;
  Launch L = s->launch();
  const EigShape sh = eig_shape(s, nreq, P);
  const int bw = sh.bw, mmax = sh.mmax, keep = sh.keep, max_passes = sh.max_passes;
  // a wide Rayleigh-Ritz needs the Ritz pairs a thick restart keeps (and the Ritz block)
  // identity basis: no later pass uses a Ritz block (no warm start, no restart), so only the nreq
  // wanted Ritz pairs are formed (eigenvectors, back-transform and Newton-Schulz of the wide solver
  // scale with that count) and the Ritz block returned is nreq wide
  const int rbw = sh.identity ? std::min(bw, nreq) : bw;
  s->rr_nvec = sh.identity ? nreq : sh.exhaust ? 0 : std::max(keep, nreq);
  struct NvecReset {
    megb200_solver* s;
    ~NvecReset() { s->rr_nvec = 0; }
  } nvec_reset{s};
  // Overlapped restarts: at a full basis the wide Rayleigh-Ritz (one CTA, ~0.5 ms) runs on the side
  // stream while the solver stream orthonormalises the next Krylov block against the full basis and
  // runs its operator pass (neither depends on the Ritz pairs); the restart then carries that block's
  // image and its column of H over (restart_h).  Same subspaces as the serial order.  The cooperative
  // kernels of such a solve leave one SM to the Rayleigh-Ritz CTA.
  static const bool no_overlap = getenv("MEGB200_NO_RR_OVERLAP") != nullptr;  // diagnostics
  const bool overlap = !no_overlap && s->side && !sh.identity && !sh.exhaust && mmax > 48 && s->sm_count > 8;
  struct CoopSmReset {
    megb200_solver* s;
    ~CoopSmReset() {
      s->coop_sm = s->sm_count;
      s->in_solve = false;
    }
  } coop_reset{s};
  s->in_solve = true;  // the operator is fixed for the solve: per-pattern scratch (CSR panel pointers) is reused
  s->csr_pp_valid = false;
  if (overlap) s->coop_sm = s->sm_count - 1;
  static const int rr_lag = [] {  // blocks run ahead of an overlapped Rayleigh-Ritz (diagnostics override)
    const char* e = getenv("MEGB200_RR_LAG");
    return e ? std::max(1, std::min(4, atoi(e))) : 1;
  }();
  const double tol = P.tol;
  const uint64_t key_start = stream_key(P.seed, kStreamStart);
  const uint64_t key_refill = stream_key(P.seed, kStreamRefill);
  uint64_t refill_ctr = 0;

  s->mark("begin");
  // ---- start block: warm columns + seeded random fill.  A verified-orthonormal warm block of
  // exactly bw columns is read in place by the fused first pass; it is copied into the basis only
  // if the solve continues past that pass (deferred_warm)
  const int wc = sh.identity ? 0 : (int)std::min<int64_t>(P.warm_cols, bw);
  bool deferred_warm = !sh.identity && wc == bw && P.warm_orthonormal && ((uintptr_t)P.warm % 16) == 0 &&
                       (P.ld_warm % 2) == 0 && fused_ok(s, op, bw, nreq) &&
                       getenv("MEGB200_NO_INPLACE_WARM") == nullptr;
  if (wc > 0 && !deferred_warm) copy_block(L, n, wc, P.warm, P.ld_warm, s->Q, s->ldq);
  if (sh.identity) {
    set_identity(L, n, s->Q, s->ldq);
  } else if (bw > wc) {
    fill_gaussian(L, n, bw - wc, key_start, 0, 1.0, false, s->Q + wc, s->ldq);
  }
  if (sh.identity) {
    // the identity is orthonormal
  } else if (wc == bw && P.warm_orthonormal) {
    // verified-orthonormal warm Ritz block (its Gram came back with the previous step): use as is
  } else if (wc == bw) {
    // a warm Ritz block needs one CholQR round
    coop_cholqr(L, n, s->Q, s->ldq, s->Q, s->ldq, bw, 1e-13, s->G, s->R1, s->Rinv, s->mask, nullptr, nullptr,
                key_refill, refill_ctr, s->red, s->sm_count);
    refill_ctr += (uint64_t)n * bw;
  } else {
    orthonormalize(s, s->Q, s->ldq, bw, 0, 1.0, key_refill, refill_ctr, false);
  }

  s->mark("start_block");
  EigRun run;
  std::vector<double> best(nreq, INFINITY);
  int cols = 0, cur = bw;
  double scale = 1.0;
  bool pass_done = false;  // the current block's pass already ran (overlapped with the last Rayleigh-Ritz)
  double first_ratio = 0.0;  // worst residual / tolerance after the first pass
  // identity basis with a float64 dense (or no) streamed operand: A I is the operator itself, formed
  // entry by entry in one launch (H and the images) instead of ceil(n / 32) block passes
  static const bool no_form = getenv("MEGB200_NO_FORM_OPERATOR") != nullptr;  // diagnostics
  if (sh.identity && !no_form && op.l <= 160 && (op.l == 0 || op.L) &&
      ((op.kind == MEGB200_OP_DENSE && op.dtype == MEGB200_F64) || op.scale == 0.0 || op.kind == MEGB200_OP_NONE)) {
    if (op.lc.lam == s->dlam) s->flush_dlam();
    const bool dense = op.kind == MEGB200_OP_DENSE && op.scale != 0.0;
    form_operator(L, n, dense ? static_cast<const double*>(op.dense) : nullptr, op.ld, dense ? op.scale : 0.0, op.L,
                  op.ldl, op.L ? op.l : 0, op.d_dev, op.lc, op.alpha, s->AQ, s->ldq, s->H, s->cap);
    run.passes = 1;
    cur = (int)n;
    pass_done = true;
    s->mark("pass+finish");
  }
  for (;;) {
    // operator pass on the current block, then its column of H = Q^T A Q; the first pass
    // of a solve runs fused with its Rayleigh-Ritz (one launch after the pass)
    const bool fuse = !sh.identity && cols == 0 && cur == bw && fused_ok(s, op, bw, nreq);
    if (!pass_done) {
      if (!fuse) block_pass(s, op, cols, cur);
      run.passes++;
      s->mark("pass+finish");
    }
    pass_done = false;
    const int newcols = cols + cur;
    const int nxt = (int)std::min<int64_t>(bw, n - newcols);
    const bool full = (nxt <= 0) || (newcols + nxt > mmax);
    // Rayleigh-Ritz only where its result is used: the first pass of a solve
    // (warm-started steps converge there), a full basis (restart), the budget end
    const bool do_rr = sh.identity ? (nxt <= 0 || run.passes >= max_passes)
                                   : ((cols == 0) || full || (run.passes >= max_passes));
    if (do_rr) {
      double* pk = s->h_buf;
      // outputs written by the Rayleigh-Ritz launch itself, before the wait: if it
      // converged nothing is left to launch after it (otherwise they are rewritten)
      double* v2 = vec_out ? vec_out : (epi ? epi->v_next : nullptr);
      const int64_t ld2 = vec_out ? ld_vec : (epi ? epi->ld_next : 0);
      const int r2 = vec_out ? nreq : (epi ? epi->r : 0);
      // overlapped restart: the wide solve on the side stream, the next `lag` blocks' orthonormalisation
      // and passes on the solver stream, joined before the Ritz block / residual launch
      // (from the second full basis of a solve on, or from the first when the first pass left the
      // residuals more than 1e5 x the tolerance away: a solve that converges at its first full basis --
      // cfg4's six-pass steps, ~1e4 x after the first pass -- would only pay for the speculation)
      int lag = 0;
      if (overlap && !fuse && full && cols > 0 && (run.restarts >= 1 || first_ratio > 1e5) && nxt == cur && cur == bw &&
          newcols > 48) {
        lag = rr_lag;
        while (lag > 0 && !(run.passes + lag <= max_passes && newcols + lag * bw <= std::min<int64_t>(s->cap, n) &&
                            keep + lag * bw <= newcols &&
                            ((size_t)(newcols + lag * bw) * (lag * bw) + (size_t)newcols * keep) * sizeof(double) <=
                                160 * 1024))
          --lag;
      }
      const bool spec = lag > 0;
      if (spec) {
        MEG_CUDA(cudaEventRecord(s->ev_fork, s->stream));
        MEG_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
        Launch Ls{s->side, &s->launches};
        const int rq_ = std::min(newcols, std::max(nreq, bw));
        rr_wide(Ls, s->H, s->cap, newcols, s->theta, s->S, s->info, s->rr_nvec > 0 ? std::max(s->rr_nvec, rq_) : 0);
        MEG_CUDA(cudaEventRecord(s->ev_join, s->side));
        for (int l = 0; l < lag; ++l) {
          const int cl = cols + l * bw;  // the block whose image seeds the next one
          orthonormalize(s, s->Q + cl + bw, s->ldq, bw, cl + bw, scale, key_refill, refill_ctr, false, 2, s->AQ + cl,
                         s->ldq);
          block_pass(s, op, cl + bw, bw);
        }
        s->mark("spec orth+pass");
        static const bool dbg_basis = getenv("MEGB200_DEBUG_BASIS") != nullptr;  // diagnostics: basis consistency
        if (dbg_basis) {
          const int nc = newcols + lag * bw;
          std::vector<double> g((size_t)nc * s->cap), hc((size_t)nc * s->cap), hh((size_t)nc * s->cap);
          for (int c0 = 0; c0 < nc; c0 += 32) {
            const int w = std::min(32, nc - c0);
            coop_tn(L, n, s->Q, s->ldq, nc, s->Q + c0, s->ldq, w, s->G + c0, s->cap, nullptr, 1.0, s->red, s->coop_sm);
          }
          s->sync();
          MEG_CUDA(cudaMemcpy(g.data(), s->G, g.size() * sizeof(double), cudaMemcpyDeviceToHost));
          for (int c0 = 0; c0 < nc; c0 += 32) {
            const int w = std::min(32, nc - c0);
            coop_tn(L, n, s->Q, s->ldq, nc, s->AQ + c0, s->ldq, w, s->G + c0, s->cap, nullptr, 1.0, s->red, s->coop_sm);
          }
          s->sync();
          MEG_CUDA(cudaMemcpy(hc.data(), s->G, hc.size() * sizeof(double), cudaMemcpyDeviceToHost));
          MEG_CUDA(cudaMemcpy(hh.data(), s->H, hh.size() * sizeof(double), cudaMemcpyDeviceToHost));
          double eg = 0.0, eh = 0.0;
          int gi = 0, gj = 0, hi = 0, hj = 0;
          for (int i = 0; i < nc; ++i)
            for (int j = i; j < nc; ++j) {
              const double dg = fabs(g[(size_t)i * s->cap + j] - (i == j ? 1.0 : 0.0));
              const double dh = fabs(hc[(size_t)i * s->cap + j] - hh[(size_t)i * s->cap + j]);
              if (dg > eg) { eg = dg; gi = i; gj = j; }
              if (dh > eh) { eh = dh; hi = i; hj = j; }
            }
          fprintf(stderr, "basis check nc %d: |Q^T Q - I| %.2e at (%d,%d), |Q^T AQ - H| %.2e at (%d,%d)\n", nc, eg, gi, gj,
                  eh, hi, hj);
        }
        MEG_CUDA(cudaStreamWaitEvent(s->stream, s->ev_join, 0));
      }
      const int gr = fuse ? fused_pass(s, op, deferred_warm ? P.warm : s->Q, deferred_warm ? P.ld_warm : s->ldq, bw,
                                       nreq, epi, ritz_out, ld_ritz, v2, ld2, r2, pk)
                          : rr_readback(s, newcols, nreq, rbw, epi, pk, ritz_out, ld_ritz, v2, ld2, r2, spec);
      const int rq = std::min(newcols, std::max(nreq, rbw));
      // host-buffer step: V_next travels back with the pack (one wait when this RR converges)
      if (epi && epi->v_host && epi->v_next && epi->ld_next == epi->r && epi->ld_host == epi->r)
        MEG_CUDA(cudaMemcpyAsync(epi->v_host, epi->v_next, (size_t)n * epi->r * sizeof(double),
                                 cudaMemcpyDeviceToHost, s->stream));
      s->mark("rr+ritz");
      s->sync();
      s->mark("host_decide");
      if (s->trace) {  // diagnostics only: Jacobi sweeps of this Rayleigh-Ritz solve
        double inf[3];
        MEG_CUDA(cudaMemcpy(inf, s->info, sizeof inf, cudaMemcpyDeviceToHost));
        s->stat("jacobi_sweeps m=" + std::to_string(newcols), inf[0]);
        // shape of the Rayleigh-Ritz matrix: off(H)/||H||, worst coupling/gap ratio
        if (newcols <= 64) {
          std::vector<double> h((size_t)newcols * s->cap);
          MEG_CUDA(cudaMemcpy(h.data(), s->H, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
          double f2 = 0.0, o2 = 0.0, worst = 0.0;
          for (int i = 0; i < newcols; ++i)
            for (int j = 0; j < newcols; ++j) {
              const double v = (i <= j) ? h[(size_t)i * s->cap + j] : h[(size_t)j * s->cap + i];
              f2 += v * v;
              if (i != j) {
                o2 += v * v;
                const double gap = fabs(h[(size_t)i * s->cap + i] - h[(size_t)j * s->cap + j]);
                worst = std::max(worst, fabs(v) / std::max(gap, 1e-300));
              }
            }
          s->stat("rr_off_rel_log10 m=" + std::to_string(newcols), 0.5 * log10(std::max(o2, 1e-300) / f2));
          s->stat("rr_coupling/gap_max_log10", log10(std::max(worst, 1e-300)));
        }
      }
      const RRDecision dec = rr_decide(s, pk, newcols, nreq, tol);
      if (cols == 0) first_ratio = dec.rmax / (tol * dec.scale);
      static const bool dbg_rr = getenv("MEGB200_DEBUG_RR") != nullptr;  // diagnostics
      if (dbg_rr)
        fprintf(stderr, "rr pass %d cols %d newcols %d full %d rmax %.3e theta0 %.6f scale %.3f\n", run.passes, cols,
                newcols, (int)full, dec.rmax, pk[0], dec.scale);
      scale = dec.scale;
      double best_max = 0.0;
      for (double v : best) best_max = std::max(best_max, v);
      if (dec.rmax < best_max)
        for (int j = 0; j < nreq; ++j) best[j] = pk[s->pack_resid + j];
      if (dec.ok) {
        run.theta.assign(pk, pk + nreq);
        run.resid.assign(pk + s->pack_resid, pk + s->pack_resid + nreq);
        run.norm_est = scale;
        run.converged = true;
        if (epi) {
          epi->v_host_done = epi->v_host && epi->v_next && epi->ld_next == epi->r && epi->ld_host == epi->r;
          const int epi_len = 2 * epi->r + 8;
          epi->host.assign(pk + s->pack_epi, pk + s->pack_epi + epi_len);
          epi->host.insert(epi->host.end(), pk + s->pack_gram, pk + s->pack_gram + (int64_t)gr * gr);
          epi->gr = gr;
        }
        if (ritz_cols_out) *ritz_cols_out = rq;
        return run;
      }
      if (run.passes >= max_passes) break;
      if (spec) {
        // not converged: the speculative passes are the next blocks' passes.  Thick restart keeping the
        // leading `keep` Ritz pairs, the new blocks (orthogonal to all of Q) and their images behind them
        const int tq = lag * bw;
        run.passes += lag;
        restart_basis(L, n, s->Q, s->AQ, s->ldq, s->S, newcols, keep, tq, s->sm_count);
        restart_h(L, s->H, s->cap, s->S, newcols, keep, tq, s->theta);
        s->mark("restart");
        run.restarts++;
        cols = keep + tq - bw;  // the last carried block is the current one, its pass done
        cur = bw;
        pass_done = true;
        continue;
      }
    }
    if (nxt <= 0) break;
    if (sh.identity) {  // the next identity columns are already in place
      cols = newcols;
      cur = nxt;
      continue;
    }
    if (deferred_warm) {  // the solve continues: the first block joins the basis
      copy_block(L, n, bw, P.warm, P.ld_warm, s->Q, s->ldq);
      deferred_warm = false;
    }
    // next Krylov block: the image block orthogonalised against the basis
    if (nxt == cur) {
      // the image block, read in place by the orthonormalisation kernel
      orthonormalize(s, s->Q + newcols, s->ldq, nxt, newcols, scale, key_refill, refill_ctr, false, 2, s->AQ + cols,
                     s->ldq);
    } else {
      fill_gaussian(L, n, nxt, key_refill, refill_ctr, 1.0, false, s->Q + newcols, s->ldq);
      refill_ctr += (uint64_t)n * nxt;
      orthonormalize(s, s->Q + newcols, s->ldq, nxt, newcols, scale, key_refill, refill_ctr, false);
    }
    s->mark("orth_next");
    cols = newcols;
    if (full) {
      // thick restart: keep the leading `keep` Ritz pairs, continue from the next block
      if (keep + nxt <= cols && cols + nxt <= s->cap) {
        // one launch (the carried AQ columns are not images yet: the next pass overwrites them)
        restart_basis(L, n, s->Q, s->AQ, s->ldq, s->S, cols, keep, nxt, s->sm_count);
      } else {
        nn(L, n, s->Q, s->ldq, cols, s->S, cols, keep, 1.0, 0.0, s->T, s->ldq);
        copy_block(L, n, keep, s->T, s->ldq, s->Q, s->ldq);
        nn(L, n, s->AQ, s->ldq, cols, s->S, cols, keep, 1.0, 0.0, s->T, s->ldq);
        copy_block(L, n, keep, s->T, s->ldq, s->AQ, s->ldq);
        copy_block(L, n, nxt, s->Q + cols, s->ldq, s->Q + keep, s->ldq);
      }
      set_diag(L, s->H, s->cap, keep, s->theta);  // H = diag(theta_keep); couplings arrive with the next pass
      s->mark("restart");
      cols = keep;
      run.restarts++;
    }
    cur = nxt;
  }
  run.resid = best;
  run.theta.clear();
  run.norm_est = scale;
  return run;
}

std::string fmt_resid(const std::vector<double>& r) {
  std::string out = "[";
  char buf[32];
  for (size_t i = 0; i < r.size(); ++i) {
    snprintf(buf, sizeof buf, "%s%.3e", i ? " " : "", r[i]);
    out += buf;
  }
  return out + "]";
}

[[noreturn]] void throw_lanczos(const EigRun& run, double tol) {
  char buf[128];
  snprintf(buf, sizeof buf, "residual tolerance %g not reached after %d block passes (best residuals ", tol,
           run.passes);
  throw Error(MEGB200_ERR_LANCZOS, std::string(buf) + fmt_resid(run.resid) + ")");
}

// ---------------------------------------------------------------------------
// MEG step operator: A = log X - eta grad  (logmap_operator, meg.py:287-307)

struct StepOperator {
  OpDev op;
  std::vector<double> d;  // host coefficients of the gathered low-rank factor
};

void check_iterate(megb200_solver* s, const megb200_iterate* x) {
  if (!x) throw Error(MEGB200_ERR_PARAM, "iterate is NULL");
  if (x->n != s->n) throw Error(MEGB200_ERR_PARAM, "iterate dimension does not match the solver");
  if (!(1 <= x->r && x->r < x->n)) throw Error(MEGB200_ERR_PARAM, "need 1 <= r < n");
  if (!x->V || !x->lam) throw Error(MEGB200_ERR_PARAM, "iterate factors missing");
  if (!(x->eps > 0.0 && x->eps <= 0.75)) throw Error(MEGB200_ERR_PARAM, "eps must lie in (0, 3/4]");
  for (int64_t k = 0; k < x->r; ++k)
    if (!(x->lam[k] > 0.0)) throw Error(MEGB200_ERR_PARAM, "lam must be strictly positive");
}

void check_gradient(megb200_solver* s, const megb200_gradient* g) {
  if (!g) throw Error(MEGB200_ERR_PARAM, "gradient is NULL");
  if (g->n != s->n) throw Error(MEGB200_ERR_PARAM, "gradient dimension does not match the solver");
  switch (g->kind) {
    case MEGB200_GRAD_ZERO:
      break;
    case MEGB200_GRAD_DENSE:
      if (!g->dense || g->ld < g->n) throw Error(MEGB200_ERR_PARAM, "dense gradient operand missing");
      break;
    case MEGB200_GRAD_FROBENIUS:
    case MEGB200_GRAD_STOCHASTIC:
      if (!g->dense || g->ld < g->n) throw Error(MEGB200_ERR_PARAM, "target matrix M missing");
      if (!g->gV || !g->g_lam || g->g_r < 1) throw Error(MEGB200_ERR_PARAM, "gradient iterate factors missing");
      if (g->kind == MEGB200_GRAD_STOCHASTIC && (!g->A || g->bsz < 1))
        throw Error(MEGB200_ERR_PARAM, "stochastic minibatch missing");
      break;
    case MEGB200_GRAD_CALLBACK:
      if (!g->apply) throw Error(MEGB200_ERR_PARAM, "callback gradient without apply");
      break;
    case MEGB200_GRAD_QUADMEAS:
      check_qm_data(static_cast<const megb200_qm_data*>(g->apply_ctx));
      break;
    case MEGB200_GRAD_SAMPLED:
      if (!g->rowptr || !g->col || !g->obs) throw Error(MEGB200_ERR_PARAM, "sampled pattern missing");
      if (g->nnz > s->max_nnz) throw Error(MEGB200_ERR_PARAM, "nnz exceeds the solver's max_nnz");
      if (!g->gV || !g->g_lam || g->g_r < 1) throw Error(MEGB200_ERR_PARAM, "gradient iterate factors missing");
      break;
    default:
      throw Error(MEGB200_ERR_PARAM, "unknown gradient kind");
  }
  if (g->gV && (g->g_r >= g->n || !(g->g_eps > 0.0)) && g->kind != MEGB200_GRAD_ZERO && g->kind != MEGB200_GRAD_DENSE &&
      g->kind != MEGB200_GRAD_CALLBACK && g->kind != MEGB200_GRAD_QUADMEAS)
    throw Error(MEGB200_ERR_PARAM, "invalid gradient iterate");
}

// X_g coefficients: c_k = (1 - eps) lam_k - tail, tail = eps / (n - r)
void x_coeffs(int64_t n, int64_t r, const double* lam, double eps, std::vector<double>& c, double& tail) {
  tail = eps / (double)(n - r);
  c.resize(r);
  for (int64_t k = 0; k < r; ++k) c[k] = (1.0 - eps) * lam[k] - tail;
}

// The step operator of a Frobenius objective whose gradient iterate is the
// iterate itself: eta M + V diag(d) V^T + alpha I with
// d = log((1-eps) lam) - log tail - eta ((1-eps) lam - tail), alpha = log tail - eta tail,
// tail = eps / (n - r) (meg.py:287-307 + objectives.py X_g).  The kept weights
// lam are read on the device (lam_dev), so the operator of step t+1 can be
// enqueued before step t's results reach the host.
OpDev frob_merged_op(const megb200_gradient* g, const double* V, int64_t ldv, int64_t n, int r, double eps, double eta,
                     const double* lam_dev) {
  OpDev op;
  op.kind = MEGB200_OP_DENSE;
  op.dtype = g->dtype;
  op.dense = g->dense;
  op.ld = g->ld;
  op.scale = eta;
  const double tail = eps / (double)(n - r);
  const double log_tail = log(tail);
  op.alpha = log_tail;
  op.alpha += -eta * tail;
  op.L = V;
  op.ldl = ldv;
  op.l = r;
  op.d_dev = nullptr;
  op.lc.lam = lam_dev;
  op.lc.lr = r;
  op.lc.c1 = 1.0 - eps;
  op.lc.log_tail = log_tail;
  op.lc.eta = eta;
  op.lc.tail_g = tail;
  return op;
}

StepOperator build_step_operator(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g,
                                 double eta) {
  Launch L = s->launch();
  const int64_t n = s->n, r = x->r;
  StepOperator so;
  if (g->kind == MEGB200_GRAD_FROBENIUS && g->gV == x->V && g->g_r == r && g->g_ldv == x->ldv && g->g_eps == x->eps &&
      r <= 64 && std::equal(x->lam, x->lam + r, g->g_lam)) {
    std::copy(x->lam, x->lam + r, s->dlam_host);
    s->dlam_n = (int)r;
    s->dlam_dirty = true;  // uploaded only if a consumer other than the fused first pass needs it
    so.op = frob_merged_op(g, x->V, x->ldv, n, (int)r, x->eps, eta, s->dlam);
    return so;
  }
  OpDev& op = so.op;
  // log X = V diag(log_kept - log_tail) V^T + log_tail I
  const double tail_x = x->eps / (double)(n - r);
  const double log_tail = log(tail_x);
  std::vector<double> dx(r);
  for (int64_t k = 0; k < r; ++k) dx[k] = log((1.0 - x->eps) * x->lam[k]) - log_tail;
  op.alpha = log_tail;
  bool merged = false;
  std::vector<double> cg;
  double tail_g = 0.0;
  if (g->kind == MEGB200_GRAD_FROBENIUS || g->kind == MEGB200_GRAD_STOCHASTIC || g->kind == MEGB200_GRAD_SAMPLED)
    x_coeffs(n, g->g_r, g->g_lam, g->g_eps, cg, tail_g);
  switch (g->kind) {
    case MEGB200_GRAD_ZERO:
      op.kind = MEGB200_OP_NONE;
      break;
    case MEGB200_GRAD_DENSE:
      op.kind = MEGB200_OP_DENSE;
      op.dtype = g->dtype;
      op.dense = g->dense;
      op.ld = g->ld;
      op.scale = -eta;
      break;
    case MEGB200_GRAD_CALLBACK:
      op.kind = MEGB200_OP_CALLBACK;
      op.apply = g->apply;
      op.apply_ctx = g->apply_ctx;
      op.scale = -eta;
      break;
    case MEGB200_GRAD_QUADMEAS:
      op.kind = MEGB200_OP_QUADMEAS;
      op.apply_ctx = g->apply_ctx;
      op.scale = -eta;
      break;
    case MEGB200_GRAD_FROBENIUS:
    case MEGB200_GRAD_STOCHASTIC:
      // -eta (X_g - M) = eta M - eta Vg diag(c) Vg^T - eta tail_g I
      op.kind = MEGB200_OP_DENSE;
      op.dtype = g->dtype;
      op.dense = g->dense;
      op.ld = g->ld;
      op.scale = eta;
      op.alpha += -eta * tail_g;
      merged = (g->gV == x->V && g->g_r == r && g->g_ldv == x->ldv);
      break;
    case MEGB200_GRAD_SAMPLED: {
      // -eta P_Omega(X_g - Mobs): values from the factors, once per step
      double* dcoef = s->small;
      s->h2d(dcoef, cg.data(), (int64_t)cg.size());
      csr_values(L, n, g->rowptr, g->col, g->obs, g->gV, g->g_ldv, (int)g->g_r, dcoef, tail_g, s->csr_g, nullptr,
                 0);
      op.kind = MEGB200_OP_CSR;
      op.rowptr = g->rowptr;
      op.col = g->col;
      op.val = s->csr_g;
      op.nnz = g->nnz;
      op.scale = -eta;
      break;
    }
  }
  // gather low-rank factors: [V_x | V_g (unless merged) | A]
  std::vector<double>& d = so.d;
  d = dx;
  if (merged)
    for (int64_t k = 0; k < r; ++k) d[k] += -eta * cg[k];
  const bool need_g = (g->kind == MEGB200_GRAD_FROBENIUS || g->kind == MEGB200_GRAD_STOCHASTIC) && !merged;
  const bool need_a = g->kind == MEGB200_GRAD_STOCHASTIC;
  const int64_t l = r + (need_g ? g->g_r : 0) + (need_a ? g->bsz : 0);
  if (l > s->max_lowrank) throw Error(MEGB200_ERR_PARAM, "low-rank width exceeds the solver's max_lowrank");
  if (!need_g && !need_a) {
    op.L = x->V;
    op.ldl = x->ldv;
  } else {
    copy_block(L, n, (int)r, x->V, x->ldv, s->L, s->max_lowrank);
    int64_t off = r;
    if (need_g) {
      copy_block(L, n, (int)g->g_r, g->gV, g->g_ldv, s->L + off, s->max_lowrank);
      for (int64_t k = 0; k < g->g_r; ++k) d.push_back(-eta * cg[k]);
      off += g->g_r;
    }
    if (need_a) {
      copy_block(L, n, (int)g->bsz, g->A, g->lda, s->L + off, s->max_lowrank);
      for (int64_t k = 0; k < g->bsz; ++k) d.push_back(-eta * g->sigma / (double)g->bsz);
      op.alpha += eta * g->sigma / (double)n;
    }
    op.L = s->L;
    op.ldl = s->max_lowrank;
  }
  op.l = (int)l;
  s->h2d(s->dvec, d.data(), l);
  op.d_dev = s->dvec;
  return so;
}

// Gram error max |V^T V - I| for an n x r block (LowRankIterate validation, meg.py:69-71)
double gram_error(megb200_solver* s, const double* V, int64_t ldv, int r) {
  Launch L = s->launch();
  coop_tn(L, s->n, V, ldv, r, V, ldv, r, s->G, r, nullptr, 1.0, s->red, s->sm_count);
  std::vector<double> g((size_t)r * r);
  s->d2h(g.data(), s->G, (int64_t)r * r);
  s->sync();
  double e = 0.0;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) e = std::max(e, fabs(g[(size_t)i * r + j] - (i == j ? 1.0 : 0.0)));
  return e;
}

}  // namespace

// ===========================================================================
// C ABI

namespace {
int guarded_impl(const std::function<void()>& body) {
  try {
    body();
    return MEGB200_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MEGB200_ERR_CUDA;
  } catch (...) {
    g_last_error = "unknown error";
    return MEGB200_ERR_CUDA;
  }
}
}  // namespace

extern "C" {

int megb200_abi_version(void) { return MEGB200_ABI_VERSION; }

const char* megb200_last_error(void) { return g_last_error.c_str(); }

int megb200_device_check(int* sm_count) {
  return guarded_impl([&] {
    int dev = 0, count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) throw Error(MEGB200_ERR_NO_DEVICE, "no CUDA device visible");
    MEG_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    MEG_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
      throw Error(MEGB200_ERR_NO_DEVICE, std::string("device is not sm_100 (Blackwell): ") + prop.name);
    if (sm_count) *sm_count = prop.multiProcessorCount;
  });
}

int megb200_solver_create(int64_t n, int32_t max_block, int32_t max_basis, int64_t max_lowrank, int64_t max_nnz,
                          megb200_solver** out) {
  return guarded_impl([&] {
    if (!out) throw Error(MEGB200_ERR_PARAM, "out is NULL");
    if (n < 2) throw Error(MEGB200_ERR_PARAM, "need n >= 2");
    if (max_block < 1 || max_block > kMaxBlock) throw Error(MEGB200_ERR_PARAM, "max_block must be in [1, 64]");
    if (max_basis < 2 || max_basis > kMaxBasis) throw Error(MEGB200_ERR_PARAM, "max_basis must be in [2, 112]");
    int sm = 148;
    int rc = megb200_device_check(&sm);
    if (rc != MEGB200_OK) throw Error(rc, g_last_error);
    auto* s = new megb200_solver();
    s->n = n;
    s->max_block = max_block;
    s->max_basis = max_basis;
    s->cap = max_basis + max_block;
    s->max_lowrank = std::max<int64_t>(1, max_lowrank);
    s->max_nnz = std::max<int64_t>(0, max_nnz);
    s->sm_count = sm;
    s->coop_sm = sm;
    s->ldq = s->cap;
    // apply partial slices: up to 16 (wave balancing of the persistent pass), <= 256 MiB
    s->part_slices = std::max<int64_t>(1, std::min<int64_t>(16, (256ll << 20) / (n * (int64_t)max_block * 8)));
    s->red_cap = (int64_t)sm * std::max<int64_t>((int64_t)s->cap * std::max<int>(s->cap, max_block),
                                                 s->max_lowrank * max_block);
    struct Item {
      double** p;
      int64_t count;
    };
    const int64_t nb = n * (int64_t)max_block;
    std::vector<Item> items = {
        {&s->Q, n * s->ldq},
        {&s->AQ, n * s->ldq},
        {&s->T, n * s->ldq},
        {&s->W, nb},
        {&s->part, s->part_slices * nb},
        {&s->red, s->red_cap},
        {&s->L, n * s->max_lowrank},
        {&s->E, s->max_lowrank * max_block},
        {&s->dvec, s->max_lowrank},
        {&s->dlam, 64},
        {&s->uT, 32 * n},  // 64 x n float32: [Uh | Ul]^T of the tcgen05 pass
        {&s->H, (int64_t)s->cap * s->cap},
        {&s->C, (int64_t)s->cap * max_block},
        {&s->C2, (int64_t)s->cap * max_block},
        {&s->G, (int64_t)s->cap * s->cap},
        {&s->R1, (int64_t)max_block * max_block},
        {&s->R2, (int64_t)max_block * max_block},
        {&s->Rinv, (int64_t)max_block * max_block},
        {&s->Rn, (int64_t)max_block * max_block},
        {&s->Rtmp, (int64_t)max_block * max_block},
        {&s->theta, s->cap},
        {&s->S, (int64_t)s->cap * s->cap},
        {&s->est, s->cap},
        {&s->info, 16},
        {&s->resid, s->cap},
        {&s->small, 4096},
        {&s->pack, s->cap + 64 + 136 + 64 * 64},
        {&s->csr_g, std::max<int64_t>(1, s->max_nnz)},
        {&s->rowsq, n},
    };
    int64_t total = 0;
    for (auto& it : items) total += align_up(it.count * (int64_t)sizeof(double), 256);
    total += align_up(kMaxBlock * sizeof(int), 256);
    cudaError_t e = cudaMalloc(&s->arena, total);
    if (e != cudaSuccess) {
      delete s;
      throw Error(MEGB200_ERR_CUDA, std::string("workspace allocation failed: ") + cudaGetErrorString(e));
    }
    s->arena_bytes = total;
    int64_t off = 0;
    for (auto& it : items) {
      *it.p = reinterpret_cast<double*>(s->arena + off);
      off += align_up(it.count * (int64_t)sizeof(double), 256);
    }
    s->mask = reinterpret_cast<int*>(s->arena + off);
    s->pack_resid = s->cap;
    s->pack_epi = s->cap + 64;
    s->pack_gram = s->cap + 64 + 136;
    s->pack_vgram = s->pack_gram + 32 * 32;  // after the fused kernel's Ritz-block Gram (<= 32 x 32)
    s->theta = s->pack;  // theta lives at the head of the pack
    s->resid = s->pack + s->pack_resid;
    // [pack copy | scratch | pipelined read-back slot 0 | slot 1]
    s->pack_len = (int64_t)s->cap + 64 + 136 + 64 * 64;
    s->h_buf_len = 5 * s->pack_len + 64;
    s->h_up_len = 8192;
    e = cudaMallocHost(&s->h_up, s->h_up_len * sizeof(double));
    if (e != cudaSuccess) {
      cudaFree(s->arena);
      delete s;
      throw Error(MEGB200_ERR_CUDA, "pinned upload ring allocation failed");
    }
    e = cudaMallocHost(&s->h_buf, s->h_buf_len * sizeof(double));
    if (e != cudaSuccess) {
      cudaFree(s->arena);
      delete s;
      throw Error(MEGB200_ERR_CUDA, "pinned staging allocation failed");
    }
    // device alias of the pinned staging buffer: the fused first-pass kernel writes its result pack there
    void* hd = nullptr;
    if (cudaHostGetDevicePointer(&hd, s->h_buf, 0) == cudaSuccess && getenv("MEGB200_NO_ZEROCOPY") == nullptr)
      s->h_buf_dev = static_cast<double*>(hd);
    cudaGetLastError();
    // words 0..127 tickets / flags of k_fused_first_pass, 128..255 its stamps (64 x u64),
    // 256..418 k_dense_step_mma (tile counters, tickets, flag), 420 the k_tile_gram ticket
    e = cudaMalloc(&s->fsync, 1024 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->fsync, 0, 1024 * sizeof(unsigned));
    if (e != cudaSuccess) {
      cudaFree(s->arena);
      cudaFreeHost(s->h_buf);
      delete s;
      throw Error(MEGB200_ERR_CUDA, "sync flag allocation failed");
    }
    if (cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      s->side = nullptr;  // no overlap: the wide Rayleigh-Ritz stays on the solver stream
    }
    *out = s;
    g_live_solvers.fetch_add(1);
  });
}

void megb200_solver_destroy(megb200_solver* s) {
  if (!s) return;
  g_live_solvers.fetch_sub(1);
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (s->side) {
    cudaStreamSynchronize(s->side);
    cudaStreamDestroy(s->side);
  }
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  cudaFree(s->arena);
  if (s->run_buf) cudaFree(s->run_buf);
  if (s->flush_buf) cudaFree(s->flush_buf);
  if (s->host_io) cudaFree(s->host_io);
  cudaFreeHost(s->h_buf);
  cudaFreeHost(s->h_up);
  if (s->fsync) cudaFree(s->fsync);
  if (s->qm_part) cudaFree(s->qm_part);
  if (s->csr_pp) cudaFree(s->csr_pp);
  delete s;
}

int megb200_solver_set_stream(megb200_solver* s, void* stream) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    s->stream = static_cast<cudaStream_t>(stream);
  });
}

int64_t megb200_solver_workspace_bytes(const megb200_solver* s) { return s ? s->arena_bytes : 0; }

int64_t megb200_kernel_launches(const megb200_solver* s) { return s ? s->launches : 0; }

int megb200_operator_apply(megb200_solver* s, const megb200_operator* op, const double* U, int64_t ldu, int32_t k,
                           double* W, int64_t ldw) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    if (!U || !W || k < 1) throw Error(MEGB200_ERR_PARAM, "invalid block");
    OpDev o = op_from_public(s, op);
    apply_op_wide(s, o, U, ldu, k, W, ldw);
  });
}

int megb200_logmap_apply(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g, double eta,
                         const double* U, int64_t ldu, int32_t k, double* W, int64_t ldw) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    check_iterate(s, x);
    check_gradient(s, g);
    if (!U || !W || k < 1) throw Error(MEGB200_ERR_PARAM, "invalid block");
    StepOperator so = build_step_operator(s, x, g, eta);
    apply_op_wide(s, so.op, U, ldu, k, W, ldw);
  });
}

int megb200_sym_eigh(megb200_solver* s, const double* A, int64_t lda, int32_t m, double* w, double* V) {
  return guarded_impl([&] {
    if (!s || !A || !w || !V) throw Error(MEGB200_ERR_PARAM, "null argument");
    if (m < 1 || m > kMaxBasis || lda < m) throw Error(MEGB200_ERR_PARAM, "sym_eigh needs 1 <= m <= 112, lda >= m");
    Launch L = s->launch();
    rr_wide(L, A, lda, m, w, V, s->info, 0);
  });
}

int megb200_gradient_apply(megb200_solver* s, const megb200_gradient* g, const double* U, int64_t ldu, int32_t k,
                           double* W, int64_t ldw) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    check_gradient(s, g);
    if (!U || !W || k < 1) throw Error(MEGB200_ERR_PARAM, "invalid block");
    Launch L = s->launch();
    const int64_t n = s->n;
    // grad u as a device operator: scale * Op u + L diag(d) L^T u + alpha u
    OpDev op;
    std::vector<double> d;
    std::vector<double> cg;
    double tail_g = 0.0;
    if (g->kind == MEGB200_GRAD_FROBENIUS || g->kind == MEGB200_GRAD_STOCHASTIC || g->kind == MEGB200_GRAD_SAMPLED)
      x_coeffs(n, g->g_r, g->g_lam, g->g_eps, cg, tail_g);
    switch (g->kind) {
      case MEGB200_GRAD_ZERO:
        op.kind = MEGB200_OP_NONE;
        break;
      case MEGB200_GRAD_DENSE:
        op.kind = MEGB200_OP_DENSE;
        op.dtype = g->dtype;
        op.dense = g->dense;
        op.ld = g->ld;
        op.scale = 1.0;
        break;
      case MEGB200_GRAD_CALLBACK:
        op.kind = MEGB200_OP_CALLBACK;
        op.apply = g->apply;
        op.apply_ctx = g->apply_ctx;
        op.scale = 1.0;
        break;
      case MEGB200_GRAD_QUADMEAS:
        op.kind = MEGB200_OP_QUADMEAS;
        op.apply_ctx = g->apply_ctx;
        op.scale = 1.0;
        break;
      case MEGB200_GRAD_FROBENIUS:
      case MEGB200_GRAD_STOCHASTIC: {
        // X_g - M (+ sigma ((1/b) A A^T - I/n)): -M streamed, the rest low-rank
        op.kind = MEGB200_OP_DENSE;
        op.dtype = g->dtype;
        op.dense = g->dense;
        op.ld = g->ld;
        op.scale = -1.0;
        op.alpha = tail_g;
        d = cg;
        const bool stoch = g->kind == MEGB200_GRAD_STOCHASTIC;
        const int64_t l = g->g_r + (stoch ? g->bsz : 0);
        if (l > s->max_lowrank) throw Error(MEGB200_ERR_PARAM, "low-rank width exceeds the solver's max_lowrank");
        copy_block(L, n, (int)g->g_r, g->gV, g->g_ldv, s->L, s->max_lowrank);
        if (stoch) {
          copy_block(L, n, (int)g->bsz, g->A, g->lda, s->L + g->g_r, s->max_lowrank);
          for (int64_t j = 0; j < g->bsz; ++j) d.push_back(g->sigma / (double)g->bsz);
          op.alpha -= g->sigma / (double)n;
        }
        op.L = s->L;
        op.ldl = s->max_lowrank;
        op.l = (int)l;
        break;
      }
      case MEGB200_GRAD_SAMPLED:
        s->h2d(s->small, cg.data(), (int64_t)cg.size());
        csr_values(L, n, g->rowptr, g->col, g->obs, g->gV, g->g_ldv, (int)g->g_r, s->small, tail_g, s->csr_g, nullptr,
                   0);
        op.kind = MEGB200_OP_CSR;
        op.rowptr = g->rowptr;
        op.col = g->col;
        op.val = s->csr_g;
        op.nnz = g->nnz;
        op.scale = 1.0;
        break;
    }
    if (op.l > 0) {
      s->h2d(s->dvec, d.data(), op.l);
      op.d_dev = s->dvec;
    }
    apply_op_wide(s, op, U, ldu, k, W, ldw);
  });
}

int megb200_top_r(megb200_solver* s, const megb200_operator* op, int32_t r, const megb200_eig_opts* opts,
                  megb200_eig_result* out) {
  return guarded_impl([&] {
    if (!s || !out) throw Error(MEGB200_ERR_PARAM, "solver/result is NULL");
    if (!(1 <= r && r < s->n))
      throw Error(MEGB200_ERR_PARAM, "need 1 <= r < n, got r=" + std::to_string(r) + ", n=" + std::to_string(s->n));
    OpDev o = op_from_public(s, op);
    EigParams P = params_from_opts(opts);
    int rc = 0;
    EigRun run = top_eigs(s, o, r, P, out->eigenvectors, out->ld_vec, out->ritz_block, out->ld_ritz, &rc);
    out->ritz_cols = out->ritz_block ? rc : 0;
    out->passes = run.passes;
    out->restarts = run.restarts;
    out->norm_est = run.norm_est;
    if (out->residual_norms)
      for (int j = 0; j < r; ++j) out->residual_norms[j] = run.resid[j];
    if (!run.converged) throw_lanczos(run, P.tol);
    if (out->eigenvalues)
      for (int j = 0; j < r; ++j) out->eigenvalues[j] = run.theta[j];
    s->sync();
  });
}

namespace {
void step_core(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g, double eta, double eps_next,
               const megb200_eig_opts* opts, megb200_step_result* out, double* v_host = nullptr,
               int64_t ld_host = 0, bool* v_host_done = nullptr);

// Step outputs from a converged solve's read-back: epilogue block
// [y (r+1) | lam (r) | lam_{r+1}, b_{r+1}, shift, lhs, holds, threshold, status]
// and the Gram of the gr-column Ritz block (V_next = its first r columns).
void fill_step_result(const double* hb, const double* gram, int gr, int r, const double* theta,
                      megb200_step_result* out) {
  const int nreq = r + 1;
  const double status = hb[2 * r + 1 + 6];
  if (status == 4.0) throw Error(MEGB200_ERR_KEPT_MASS, "kept mass vanished despite max-shift");
  if (status == 1.0) throw Error(MEGB200_ERR_PARAM, "certificate inputs invalid (partial trace <= 0 or lambda < 0)");
  for (int k = 0; k < nreq; ++k) out->y[k] = hb[k];
  for (int k = 0; k < r; ++k) out->lam_next[k] = hb[nreq + k];
  if (out->mu)
    for (int k = 0; k < nreq; ++k) out->mu[k] = theta[k];
  const double* t = hb + 2 * r + 1;
  out->lambda_r_plus_1 = t[0];
  out->b_r_plus_1 = t[1];
  out->shift = t[2];
  out->lhs_cheap = t[3];
  out->holds_cheap = t[4] != 0.0;
  out->threshold = t[5];
  double ge = 0.0, gall = 0.0;
  for (int i = 0; i < gr; ++i)
    for (int j = 0; j < gr; ++j) {
      const double e = fabs(gram[i * gr + j] - (i == j ? 1.0 : 0.0));
      gall = std::max(gall, e);
      if (i < r && j < r) ge = std::max(ge, e);
    }
  out->gram_err = ge;
  out->ritz_orth_err = gall;
}

// ---------------------------------------------------------------------------
// Pipelined warm steps.  A step whose start block is a verified-orthonormal
// Ritz block of exactly bw columns runs, in top_eigs, as: copy the block into
// Q, one pass, Rayleigh-Ritz + epilogue, read-back, and (when that converged)
// copies of the Ritz block and V_next.  fast_step_enqueue issues exactly that
// sequence without waiting for the read-back; fast_step_confirm then applies
// top_eigs' convergence rule to it.  When it holds, the enqueued work is the
// work step_core would have done (same kernels, same operands), so results are
// bit-identical; when it does not, the caller drains the stream and re-runs the
// step through step_core.
struct FastStep {
  int r = 0, nreq = 0, bw = 0, gr = 0;
  double tol = 0.0;
  double* dst = nullptr;  // pinned read-back slot
  cudaEvent_t done = nullptr;
  // completion by the kernel's marker in the mapped slot (no event between this step's fused kernel
  // and the next step's pass, whose programmatic launch it would serialise)
  const volatile double* marker = nullptr;
  double marker_value = 0.0;
};

void fast_step_enqueue(megb200_solver* s, const OpDev& op, int r, const EigShape& sh, double tol, const double* warm,
                       int64_t ld_warm, double eps_next, double* ritz_out, int64_t ld_ritz, double* V_next,
                       int64_t ld_next, double* dst, cudaEvent_t done, FastStep& fs) {
  Launch L = s->launch();
  const int64_t n = s->n;
  fs.r = r;
  fs.nreq = r + 1;
  fs.bw = sh.bw;
  fs.tol = tol;
  fs.dst = dst;
  fs.done = done;
  EpiSpec epi;
  epi.r = r;
  epi.eps_next = eps_next;
  fs.marker = nullptr;
  if (fused_ok(s, op, sh.bw, fs.nreq)) {
    // the fused first pass reads the warm block in place (no copy into the basis)
    fs.gr = fused_pass(s, op, warm, ld_warm, sh.bw, fs.nreq, &epi, ritz_out, ld_ritz, V_next, ld_next, r, dst);
    static const bool no_marker = getenv("MEGB200_NO_MARKER") != nullptr;  // diagnostics
    if (s->last_pack_host && !no_marker) {
      fs.marker = dst + s->last_pack_count;
      fs.marker_value = (double)s->last_fused_epoch;
      return;
    }
  } else {
    copy_block(L, n, sh.bw, warm, ld_warm, s->Q, s->ldq);
    block_pass(s, op, 0, sh.bw);
    fs.gr = rr_readback(s, sh.bw, fs.nreq, sh.bw, &epi, dst, ritz_out, ld_ritz, V_next, ld_next, r);
  }
  MEG_CUDA(cudaEventRecord(done, s->stream));
}

bool fast_step_confirm(megb200_solver* s, const FastStep& fs, megb200_step_result* out) {
  if (fs.marker) {
    // the kernel stores the marker after the whole pack (system-scope fence); a stuck marker falls
    // back to draining the stream, which surfaces any device error
    const auto t0 = std::chrono::steady_clock::now();
    while (*fs.marker != fs.marker_value) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) {
        s->sync();
        if (*fs.marker != fs.marker_value) throw Error(MEGB200_ERR_CUDA, "fused step did not complete");
        break;
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  } else {
    MEG_CUDA(cudaEventSynchronize(fs.done));
  }
  const double* pk = fs.dst;
  const RRDecision dec = rr_decide(s, pk, fs.bw, fs.nreq, fs.tol);
  if (!dec.ok) return false;
  out->passes = 1;
  out->restarts = 0;
  out->ritz_cols = std::min(fs.bw, std::max(fs.nreq, fs.bw));
  if (out->residual_norms)
    for (int j = 0; j < fs.nreq; ++j) out->residual_norms[j] = pk[s->pack_resid + j];
  fill_step_result(pk + s->pack_epi, pk + s->pack_gram, fs.gr, fs.r, pk, out);
  return true;
}


double eps_eval(const megb200_schedule& sc, int64_t t) {
  const double g2 = std::max(sc.G * sc.G, 1.0);
  double raw;
  switch (sc.eps_kind) {
    case MEGB200_EPS_EXPERIMENT: raw = 0.6 / std::pow((double)t + sc.c + 1.0, 2); break;
    case MEGB200_EPS_CUBIC_DET: raw = sc.eps0_tilde / (2.0 * g2) / std::pow((double)t + 1.0 + sc.c, 3); break;
    case MEGB200_EPS_CUBIC_DET_GENERAL:
      raw = 3.0 * sc.eps0_tilde / (2.0 * g2) / std::pow((double)t + sc.c + 1.0, 3);
      break;
    case MEGB200_EPS_QUADRATIC_STOCH: raw = (9.0 / 32.0) * sc.eps0_tilde / std::pow((double)t + sc.c + 1.0, 2); break;
    case MEGB200_EPS_CONSTANT: raw = sc.eps0_tilde; break;
    default: throw Error(MEGB200_ERR_PARAM, "unknown epsilon schedule");
  }
  return std::min(raw, 0.75);
}
double eta_eval(const megb200_schedule& sc, int64_t t) {
  if (sc.eta_kind == MEGB200_ETA_INV_SQRT) return sc.eta0 / std::sqrt((double)t + 1.0);
  if (sc.eta_kind == MEGB200_ETA_CONSTANT) return sc.eta0;
  throw Error(MEGB200_ERR_PARAM, "unknown step rule");
}
}  // namespace

namespace {
void dual_gap_core(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts, double m_trace,
                   double* gap, double* lambda_min, double* ritz_out, int64_t ld_ritz, int32_t* ritz_cols);
}

int megb200_meg_run(megb200_solver* s, const megb200_iterate* x0, const megb200_gradient* g,
                    const megb200_schedule* sch, int64_t t0, int64_t T, const megb200_eig_opts* opts,
                    uint64_t flush_bytes, double* V_out, int64_t ld_out, double* lam_out, double* eps_out,
                    megb200_run_record* rec) {
  return guarded_impl([&] {
    if (!s || !sch || !g) throw Error(MEGB200_ERR_PARAM, "null argument");
    if (T < 0) throw Error(MEGB200_ERR_PARAM, "T must be >= 0");
    check_iterate(s, x0);
    const int64_t n = s->n;
    const int r = (int)x0->r;
    if (r + 1 > 64 || r + 1 >= n) throw Error(MEGB200_ERR_PARAM, "run loop supports r + 1 <= 64, r + 1 < n");
    Launch L = s->launch();
    // three slots of (V, Ritz block): step i reads slot i % 3 and writes slot (i + 1) % 3, so a
    // speculatively enqueued step i + 1 never overwrites the inputs of a step i that must re-run
    // + two slots for the certificate's warm Ritz block (ping-pong)
    if (!s->run_buf) MEG_CUDA(cudaMalloc(&s->run_buf, (size_t)8 * n * 64 * sizeof(double)));
    const int cert_every = sch->cert_every;
    if (cert_every < 0) throw Error(MEGB200_ERR_PARAM, "cert_every must be >= 0");
    if (cert_every > 0 && g->kind != MEGB200_GRAD_FROBENIUS)
      throw Error(MEGB200_ERR_PARAM, "the dual-gap certificate cadence needs a Frobenius gradient");
    if (flush_bytes > s->flush_len) {
      if (s->flush_buf) MEG_CUDA(cudaFree(s->flush_buf));
      MEG_CUDA(cudaMalloc(&s->flush_buf, flush_bytes));
      s->flush_len = flush_bytes;
    }
    double* Vb[3];
    double* Wb[3];
    for (int k = 0; k < 3; ++k) {
      Vb[k] = s->run_buf + (int64_t)k * n * 64;
      Wb[k] = s->run_buf + (int64_t)(3 + k) * n * 64;
    }
    copy_block(L, n, r, x0->V, x0->ldv, Vb[0], r);
    std::vector<double> lam(x0->lam, x0->lam + r);
    double eps = x0->eps;
    megb200_eig_opts o{};
    if (opts) o = *opts;
    const EigParams P0 = params_from_opts(&o);
    const EigShape sh = eig_shape(s, r + 1, P0);
    // warm block of the current step: caller's block for step 0 (slot-free), then slot i % 3
    const double* warm = o.warm;
    int64_t warm_cols = o.warm ? o.warm_cols : 0, ld_warm = o.ld_warm;
    bool warm_orth = o.warm && o.warm_orthonormal;
    double last_orth = INFINITY;
    // pipelining: Frobenius steps (operator coefficients computable on the device), not under the tracer
    const char* nopipe = getenv("MEGB200_NO_PIPELINE");
    const bool pipe = g->kind == MEGB200_GRAD_FROBENIUS && !s->trace && !(nopipe && nopipe[0] == '1') &&
                      !sh.exhaust && sh.max_passes >= 1;
    std::vector<double> lam_next(r), y(r + 1), mu(r + 1), res(r + 1);
    // per-step device time: from the end of the previous step (or this step's
    // start) to this step's end, minus the flush; host turnaround gaps and
    // discarded speculative work count
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    std::vector<cudaEvent_t> evf;
    if (rec && rec->step_ms) {
      ev.resize((size_t)T);
      evf.resize((size_t)T);
      for (int64_t i = 0; i < T; ++i) {
        MEG_CUDA(cudaEventCreate(&ev[i].first));
        MEG_CUDA(cudaEventCreate(&ev[i].second));
        MEG_CUDA(cudaEventCreate(&evf[i]));
      }
    }
    cudaEvent_t done[2];
    for (auto& e : done) MEG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }
    } guard{done};
    double* hspec[2] = {s->h_buf + 2 * s->pack_len, s->h_buf + 3 * s->pack_len};

    // sub-range timing (rec->timed_count > 0): events bracket steps [tf, tl]
    const int64_t tf = (rec && rec->timed_count > 0) ? rec->timed_from : -1;
    const int64_t tl = tf >= 0 ? tf + rec->timed_count - 1 : -1;
    if (tf >= 0 && tl >= T) throw Error(MEGB200_ERR_PARAM, "timed steps outside [0, T)");
    cudaEvent_t tev[2] = {nullptr, nullptr};
    int64_t tlaunch0 = 0, tlaunch1 = 0;
    if (tf >= 0)
      for (auto& e : tev) MEG_CUDA(cudaEventCreate(&e));
    struct TevGuard {
      cudaEvent_t* e;
      ~TevGuard() {
        if (e[0]) cudaEventDestroy(e[0]);
        if (e[1]) cudaEventDestroy(e[1]);
      }
    } tguard{tev};
    auto begin_step = [&](int64_t i) {
      if (i == tf) {
        MEG_CUDA(cudaEventRecord(tev[0], s->stream));
        tlaunch0 = s->launches;
      }
      if (!ev.empty()) MEG_CUDA(cudaEventRecord(evf[i], s->stream));
      if (flush_bytes) MEG_CUDA(cudaMemsetAsync(s->flush_buf, (int)(i & 0xff), flush_bytes, s->stream));
      if (!ev.empty()) MEG_CUDA(cudaEventRecord(ev[i].first, s->stream));
    };
    auto end_step = [&](int64_t i) {
      if (!ev.empty()) MEG_CUDA(cudaEventRecord(ev[i].second, s->stream));
      if (i == tl) {  // re-recorded if step tl re-runs: the event marks its last completion
        MEG_CUDA(cudaEventRecord(tev[1], s->stream));
        tlaunch1 = s->launches;
      }
    };
    auto result_for = [&](int64_t i, megb200_step_result& out) {
      out = megb200_step_result{};
      out.V_next = Vb[(i + 1) % 3];
      out.ld_next = r;
      out.lam_next = lam_next.data();
      out.y = y.data();
      out.mu = mu.data();
      out.residual_norms = res.data();
      out.ritz_block = Wb[(i + 1) % 3];
      out.ld_ritz = 64;
    };
    // commit step i: records, then the iterate / warm block move to slot (i + 1) % 3
    auto commit = [&](int64_t i, const megb200_step_result& out, double eps_next) {
      if (rec) {
        if (rec->shift) rec->shift[i] = out.shift;
        if (rec->y) std::copy(y.begin(), y.end(), rec->y + i * (r + 1));
        if (rec->lam) std::copy(lam_next.begin(), lam_next.end(), rec->lam + i * r);
        if (rec->eps) rec->eps[i] = eps_next;
        if (rec->lhs) rec->lhs[i] = out.lhs_cheap;
        if (rec->holds) rec->holds[i] = out.holds_cheap;
        if (rec->passes) rec->passes[i] = out.passes;
      }
      lam = lam_next;
      eps = eps_next;
      warm = Wb[(i + 1) % 3];
      warm_cols = out.ritz_cols;
      ld_warm = 64;
      warm_orth = out.ritz_orth_err <= 1e-13;
      last_orth = out.ritz_orth_err;
    };
    // dual-gap certificate of X_{i+1} after step i when (t0 + i + 1) % cert_every == 0
    auto cert_due = [&](int64_t i) { return cert_every > 0 && (t0 + i + 1) % cert_every == 0; };
    double* gapW[2] = {s->run_buf + (int64_t)6 * n * 64, s->run_buf + (int64_t)7 * n * 64};
    int gap_slot = 0;
    int32_t gap_cols = 0;
    double m_trace = NAN;
    if (rec && (rec->gap || rec->lmin))
      for (int64_t k = 0; k < T; ++k) {
        if (rec->gap) rec->gap[k] = NAN;
        if (rec->lmin) rec->lmin[k] = NAN;
      }
    auto certify = [&](int64_t i) {  // after commit(i): (Vb[(i + 1) % 3], lam, eps) is X_{i+1}
      if (!cert_due(i)) return;
      if (isnan(m_trace)) {
        double a = 0.0;
        const int rc = megb200_dense_stats(s, g->dense, g->dtype, g->ld, &a, &m_trace);
        if (rc != MEGB200_OK) throw Error(rc, g_last_error);
      }
      megb200_gradient gg = *g;
      gg.gV = Vb[(i + 1) % 3];
      gg.g_r = r;
      gg.g_ldv = r;
      gg.g_lam = lam.data();
      gg.g_eps = eps;
      megb200_eig_opts go = o;
      go.seed = 0;
      go.warm = gap_cols > 0 ? gapW[gap_slot] : nullptr;
      go.warm_cols = gap_cols;
      go.ld_warm = 64;
      go.warm_orthonormal = 0;
      double gap = NAN, lmin = NAN;
      int32_t cols = 0;
      dual_gap_core(s, &gg, &go, m_trace, &gap, &lmin, gapW[gap_slot ^ 1], 64, &cols);
      gap_slot ^= 1;
      gap_cols = cols;
      if (rec && rec->gap) rec->gap[i] = gap;
      if (rec && rec->lmin) rec->lmin[i] = lmin;
    };
    auto gradient_for = [&](int64_t i, const double* V) {
      megb200_gradient gg = *g;
      if (gg.kind == MEGB200_GRAD_FROBENIUS || gg.kind == MEGB200_GRAD_STOCHASTIC || gg.kind == MEGB200_GRAD_SAMPLED) {
        gg.gV = V;
        gg.g_r = r;
        gg.g_ldv = r;
        gg.g_lam = lam.data();
        gg.g_eps = eps;
      }
      if (gg.kind == MEGB200_GRAD_STOCHASTIC) {
        if (!gg.A) throw Error(MEGB200_ERR_PARAM, "stochastic run needs a minibatch buffer g->A");
        fill_gaussian(L, n, (int)gg.bsz, stream_key(sch->minibatch_seed, 5), (uint64_t)(t0 + i) * n * gg.bsz,
                      1.0 / std::sqrt((double)n), sch->minibatch_round_f32 != 0, const_cast<double*>(gg.A), gg.lda);
      }
      return gg;
    };
    // full (synchronous) step through step_core
    auto full_step = [&](int64_t i) {
      const int64_t t = t0 + i;
      const double eta = eta_eval(*sch, t), eps_next = eps_eval(*sch, t + 1);
      const double* V = Vb[i % 3];
      megb200_gradient gg = gradient_for(i, V);
      megb200_iterate it{n, r, V, r, lam.data(), eps};
      megb200_eig_opts so = o;
      so.seed = (uint64_t)t;
      so.warm = warm;
      so.warm_cols = warm_cols;
      so.ld_warm = ld_warm;
      so.warm_orthonormal = warm_orth ? 1 : 0;
      megb200_step_result out;
      result_for(i, out);
      step_core(s, &it, &gg, eta, eps_next, &so, &out);
      end_step(i);
      commit(i, out, eps_next);
      certify(i);
    };
    auto fast_ok = [&]() { return pipe && warm && warm_cols == sh.bw && warm_orth; };
    FastStep fs[2];
    double host_enq = 0.0, host_wait = 0.0;  // diagnostics (MEGB200_HOST_TIMING)
    int64_t host_n = 0;
    int64_t i = 0;
    bool pending = false;  // step i is enqueued as a fast step (fs[i & 1]) and not yet confirmed
    while (i < T) {
      if (!pending) {
        begin_step(i);
        if (!fast_ok()) {
          full_step(i);
          ++i;
          continue;
        }
        // first fast step of a chain: coefficients from the host kept weights
        const int64_t t = t0 + i;
        const double* V = Vb[i % 3];
        megb200_gradient gg = gradient_for(i, V);
        megb200_iterate it{n, r, V, r, lam.data(), eps};
        check_gradient(s, &gg);
        StepOperator so = build_step_operator(s, &it, &gg, eta_eval(*sch, t));
        fast_step_enqueue(s, so.op, r, sh, P0.tol, warm, ld_warm, eps_eval(*sch, t + 1), Wb[(i + 1) % 3], 64,
                          Vb[(i + 1) % 3], r, hspec[i & 1], done[i & 1], fs[i & 1]);
        end_step(i);
        pending = true;
      }
      // speculate step i + 1 on step i's device outputs (V, Ritz block, kept weights in the pack)
      bool spec = false;
      // no speculation across a certificate: the certificate's solve reuses the solver workspace
      // (and the device pack the next step's coefficients come from)
      if (i + 1 < T && !cert_due(i)) {
        const int64_t t1 = t0 + i + 1;
        const double eps1 = eps_eval(*sch, t0 + i + 1);  // eps of iterate i + 1 = eps_next of step i
        const auto h0 = std::chrono::steady_clock::now();
        begin_step(i + 1);
        const double* V1 = Vb[(i + 1) % 3];
        OpDev op1 = frob_merged_op(g, V1, r, n, r, eps1, eta_eval(*sch, t1), s->pack + s->pack_epi + (r + 1));
        // L^T U = V_{t+1}^T W_{t+1} is block [0:r, 0:bw] of the Ritz-block Gram step t's
        // Rayleigh-Ritz launch just reduced (same rows, same order: bit-identical to reducing it again)
        op1.Eg = s->pack + s->pack_gram;
        op1.ldg = sh.bw;
        op1.Gu = s->pack + s->pack_gram;  // U^T U: the whole Ritz-block Gram
        op1.ldgu = sh.bw;
        fast_step_enqueue(s, op1, r, sh, P0.tol, Wb[(i + 1) % 3], 64, eps_eval(*sch, t1 + 1), Wb[(i + 2) % 3], 64,
                          Vb[(i + 2) % 3], r, hspec[(i + 1) & 1], done[(i + 1) & 1], fs[(i + 1) & 1]);
        end_step(i + 1);
        spec = true;
        host_enq += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
        ++host_n;
      }
      megb200_step_result out;
      result_for(i, out);
      const double eps_next = eps_eval(*sch, t0 + i + 1);
      const auto h1 = std::chrono::steady_clock::now();
      const bool conf = fast_step_confirm(s, fs[i & 1], &out);
      host_wait += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h1).count();
      if (conf) {
        commit(i, out, eps_next);
        certify(i);
        ++i;
        bool lam_pos = true;
        for (double v : lam) lam_pos = lam_pos && v > 0.0;
        // the speculation assumed an orthonormal bw-column warm block and valid kept weights
        pending = spec && fast_ok() && lam_pos;
        if (spec && !pending) s->sync();  // discard the speculative step; it re-runs from its inputs
        continue;
      }
      // step i did not converge in its first pass: drop the work enqueued after
      // it and run it through the full solver from its (intact) inputs
      s->sync();
      full_step(i);
      ++i;
      pending = false;
    }
    if (getenv("MEGB200_HOST_TIMING") && host_n > 0)
      fprintf(stderr, "meg_run host: enqueue %.1f us/step, confirm wait %.1f us/step (%lld speculative steps)\n",
              host_enq / host_n, host_wait / host_n, (long long)host_n);
    if (V_out) copy_block(L, n, r, Vb[T % 3], r, V_out, ld_out);
    if (rec && rec->ritz_block) {
      const int64_t wc = (T > 0) ? std::min<int64_t>(warm_cols, rec->ritz_cap) : 0;
      if (T > 0 && wc > 0) copy_block(L, n, (int)wc, warm, ld_warm, rec->ritz_block, rec->ld_ritz);
      rec->ritz_cols = wc;
      rec->ritz_orth_err = (T > 0 && wc == warm_cols) ? last_orth : INFINITY;
    }
    if (lam_out) std::copy(lam.begin(), lam.end(), lam_out);
    if (eps_out) *eps_out = eps;
    s->sync();
    if (tf >= 0) {
      float ms = 0.f;
      MEG_CUDA(cudaEventElapsedTime(&ms, tev[0], tev[1]));
      rec->timed_ms = ms;
      rec->timed_launches = tlaunch1 - tlaunch0;
    }
    for (int64_t k = 0; k < (int64_t)ev.size(); ++k) {
      float ms = 0.f, fl = 0.f;
      if (k == 0) {
        MEG_CUDA(cudaEventElapsedTime(&ms, ev[k].first, ev[k].second));
      } else {
        MEG_CUDA(cudaEventElapsedTime(&ms, ev[k - 1].second, ev[k].second));
        MEG_CUDA(cudaEventElapsedTime(&fl, evf[k], ev[k].first));
        ms -= fl;
      }
      rec->step_ms[k] = ms;
    }
    for (int64_t k = 0; k < (int64_t)ev.size(); ++k) {
      cudaEventDestroy(ev[k].first);
      cudaEventDestroy(ev[k].second);
      cudaEventDestroy(evf[k]);
    }
  });
}

int megb200_certificate_cheap(double lam_rp1, double b_rp1, double eps, int64_t n, int64_t r, double* lhs,
                              int32_t* holds, double* threshold) {
  return guarded_impl([&] {
    if (!(b_rp1 > 0.0)) throw Error(MEGB200_ERR_PARAM, "partial trace must be positive");
    if (lam_rp1 < 0.0) throw Error(MEGB200_ERR_PARAM, "lambda_(r+1) must be non-negative");
    const double v = lam_rp1 == 0.0 ? -INFINITY : log((double)(n - r) * lam_rp1 / (eps * b_rp1));
    if (lhs) *lhs = v;
    if (holds) *holds = v <= 2.0 * eps;
    if (threshold) *threshold = 2.0 * eps;
  });
}

}  // extern "C"

namespace {
// One low-rank MEG step (meg.py:327-364) -- shared by the single-step entry point
// and the native run loop.  Throws megb200::Error.
void step_core(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g, double eta, double eps_next,
               const megb200_eig_opts* opts, megb200_step_result* out, double* v_host, int64_t ld_host,
               bool* v_host_done) {
  if (!s || !out) throw Error(MEGB200_ERR_PARAM, "solver/result is NULL");
  if (!(eps_next > 0.0 && eps_next <= 0.75))
    throw Error(MEGB200_ERR_PARAM, "eps_next must lie in (0, 3/4], got " + std::to_string(eps_next));
  check_iterate(s, x);
  check_gradient(s, g);
  if (!out->V_next || !out->lam_next || !out->y) throw Error(MEGB200_ERR_PARAM, "step outputs missing");
  const int r = (int)x->r, nreq = r + 1;
  if (nreq >= s->n) throw Error(MEGB200_ERR_PARAM, "need r + 1 < n");
  Launch L = s->launch();
  StepOperator so = build_step_operator(s, x, g, eta);
  EigParams P = params_from_opts(opts);
  // warm start: caller's Ritz block if given, else the iterate's own factor V
  if (!P.warm) {
    P.warm = x->V;
    P.warm_cols = r;
    P.ld_warm = x->ldv;
  }
  int rc = 0;
  EpiSpec epi;
  epi.r = r;
  epi.eps_next = eps_next;
  // outputs are written before convergence is known unless they alias an operand of the solve
  // (an in-place V_next / Ritz block is then written after it)
  const int64_t n = s->n;
  auto overlaps = [n](const double* a, int64_t lda, int cols, const double* b, int64_t ldb, int bcols) {
    if (!a || !b) return false;
    const double* a1 = a + (n - 1) * lda + cols;
    const double* b1 = b + (n - 1) * ldb + bcols;
    return a < b1 && b < a1;
  };
  const bool v_alias = overlaps(out->V_next, out->ld_next, r, x->V, x->ldv, r) ||
                       overlaps(out->V_next, out->ld_next, r, g->gV, g->g_ldv, (int)g->g_r);
  const int ritz_cap = std::max(nreq, (int)s->max_block);
  // the warm block is an operand too: the fused first pass reads it in place (deferred warm) while
  // it writes the Ritz block, and a continued solve copies it into the basis afterwards
  const bool w_alias = overlaps(out->ritz_block, out->ld_ritz, ritz_cap, x->V, x->ldv, r) ||
                       overlaps(out->ritz_block, out->ld_ritz, ritz_cap, g->gV, g->g_ldv, (int)g->g_r) ||
                       overlaps(out->ritz_block, out->ld_ritz, ritz_cap, P.warm, P.ld_warm, (int)P.warm_cols);
  // V_next must not overwrite the warm block before the solve has read it either
  const bool v_warm_alias = overlaps(out->V_next, out->ld_next, r, P.warm, P.ld_warm, (int)P.warm_cols);
  if (!v_alias && !v_warm_alias) {
    epi.v_next = out->V_next;
    epi.ld_next = out->ld_next;
    epi.v_host = v_host;
    epi.ld_host = ld_host;
  }
  double* ritz_dst = w_alias ? s->W : out->ritz_block;
  const int64_t ld_ritz_dst = w_alias ? (int64_t)s->max_block : out->ld_ritz;
  EigRun run = top_eigs(s, so.op, nreq, P, nullptr, 0, out->ritz_block ? ritz_dst : nullptr, ld_ritz_dst, &rc, &epi);
  out->ritz_cols = out->ritz_block ? rc : 0;
  out->passes = run.passes;
  out->restarts = run.restarts;
  if (out->residual_norms)
    for (int j = 0; j < nreq; ++j) out->residual_norms[j] = run.resid[j];
  if (!run.converged) throw_lanczos(run, P.tol);
  // next iterate: V = top r Ritz vectors (written by top_eigs unless aliased); lam / certificate
  // came from the fused epilogue
  if (v_alias || v_warm_alias) copy_block(L, n, r, s->T, s->ldq, out->V_next, out->ld_next);
  if (v_host_done) *v_host_done = epi.v_host_done;
  if (w_alias && out->ritz_block) copy_block(L, n, out->ritz_cols, s->W, s->max_block, out->ritz_block, out->ld_ritz);
  fill_step_result(epi.host.data(), epi.host.data() + 2 * r + 8, epi.gr, r, run.theta.data(), out);
  s->mark("epilogue");
  s->trace_collect();
}
}  // namespace

extern "C" {

int megb200_lowrank_meg_step(megb200_solver* s, const megb200_iterate* x, const megb200_gradient* g, double eta,
                             double eps_next, const megb200_eig_opts* opts, megb200_step_result* out) {
  return guarded_impl([&] { step_core(s, x, g, eta, eps_next, opts, out); });
}

int megb200_lowrank_meg_step_host(megb200_solver* s, const megb200_iterate* x_host, const megb200_gradient* g,
                                  double eta, double eps_next, const megb200_eig_opts* opts, double* V_next_host,
                                  int64_t ld_next_host, megb200_step_result* out) {
  return guarded_impl([&] {
    if (!s || !x_host || !g || !out || !V_next_host) throw Error(MEGB200_ERR_PARAM, "null argument");
    const int64_t n = s->n, r = x_host->r;
    if (x_host->n != n) throw Error(MEGB200_ERR_PARAM, "iterate dimension does not match the solver");
    if (!(1 <= r && r < n) || r > 64) throw Error(MEGB200_ERR_PARAM, "need 1 <= r < n and r <= 64");
    if (!x_host->V || x_host->ldv < r || ld_next_host < r) throw Error(MEGB200_ERR_PARAM, "host factor missing");
    Launch L = s->launch();
    if (!s->host_io) MEG_CUDA(cudaMalloc(&s->host_io, (size_t)2 * n * 64 * sizeof(double)));
    double* Vd = s->host_io;
    double* Vn = s->host_io + n * 64;
    // a contiguous factor in mapped pinned memory is read by the kernels in place (the fused first
    // pass stages its rows once: no upload on the stream's critical path); otherwise it is
    // uploaded as one block (a pitched copy of 8r-byte rows is n tiny DMA rows)
    double* v_mapped = nullptr;
    // an output that overlaps the input factor in host memory disables zero-copy for both: the
    // factor is uploaded and validated from the device copy, never from memory the step writes
    const char* vh0 = reinterpret_cast<const char*>(x_host->V);
    const char* vh1 = reinterpret_cast<const char*>(x_host->V + (n - 1) * x_host->ldv + r);
    const char* oh0 = reinterpret_cast<const char*>(V_next_host);
    const char* oh1 = reinterpret_cast<const char*>(V_next_host + (n - 1) * ld_next_host + r);
    const bool io_overlap = vh0 < oh1 && oh0 < vh1;
    // (small factors only: a large one is not staged by the fused kernel and would be re-read
    // over the host link)
    // and only for the gradients whose warm steps take ONE pass (dense targets): the sampled and
    // stochastic gradients solve in 6-30 passes, each of which -- and the per-step sampled values --
    // would re-read the factor over the host link (cfg3: 10.4 -> 6.5 ms per host-buffer step)
    const bool one_pass_kind = g->kind == MEGB200_GRAD_ZERO || g->kind == MEGB200_GRAD_DENSE ||
                               g->kind == MEGB200_GRAD_FROBENIUS;
    if (!io_overlap && one_pass_kind && x_host->ldv == r && n * r * (int64_t)sizeof(double) <= (2 << 20) &&
        getenv("MEGB200_NO_ZEROCOPY") == nullptr &&
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&v_mapped), const_cast<double*>(x_host->V), 0) !=
            cudaSuccess) {
      cudaGetLastError();
      v_mapped = nullptr;
    }
    if (v_mapped)
      Vd = v_mapped;
    else if (x_host->ldv == r)
      MEG_CUDA(cudaMemcpyAsync(Vd, x_host->V, (size_t)n * r * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    else
      MEG_CUDA(cudaMemcpy2DAsync(Vd, r * sizeof(double), x_host->V, x_host->ldv * sizeof(double), r * sizeof(double),
                                 n, cudaMemcpyHostToDevice, s->stream));
    // LowRankIterate validation (meg.py:69-71): V^T V is reduced by the fused first pass (with
    // L^T U) and arrives in the result pack; a failed check discards the step and raises before
    // any result.  Steps that do not take the fused path form it separately after the solve.
    double* gram_dst = s->h_buf + 4 * s->pack_len;  // pinned slot (pack_len >= 64 x 64 doubles)
    s->want_vgram = (int)r;
    s->vgram_done = false;
    auto gram_fetch = [&]() {
      if (s->vgram_done) {
        std::copy(s->h_buf + s->pack_vgram, s->h_buf + s->pack_vgram + r * r, gram_dst);
      } else {
        coop_tn(L, n, Vd, r, (int)r, Vd, r, (int)r, s->G, (int)r, nullptr, 1.0, s->red, s->sm_count);
        s->d2h(gram_dst, s->G, r * r);
        s->sync();
      }
    };
    auto gram_check = [&]() {
      gram_fetch();
      double ge = 0.0;
      for (int i = 0; i < (int)r; ++i)
        for (int j = 0; j < (int)r; ++j) ge = std::max(ge, fabs(gram_dst[i * r + j] - (i == j ? 1.0 : 0.0)));
      if (!(ge <= 1e-10)) {
        char buf[96];
        snprintf(buf, sizeof buf, "V columns not orthonormal (error %.3e)", ge);
        throw Error(MEGB200_ERR_PARAM, buf);
      }
    };
    megb200_iterate it = *x_host;
    it.V = Vd;
    it.ldv = r;
    megb200_gradient gg = *g;
    if ((gg.kind == MEGB200_GRAD_FROBENIUS || gg.kind == MEGB200_GRAD_STOCHASTIC || gg.kind == MEGB200_GRAD_SAMPLED) &&
        !gg.gV) {
      gg.gV = Vd;
      gg.g_r = r;
      gg.g_ldv = r;
      gg.g_lam = x_host->lam;
      gg.g_eps = x_host->eps;
    }
    megb200_step_result o = *out;
    o.V_next = Vn;
    o.ld_next = r;
    bool v_done = false;
    // a mapped pinned destination takes V_next straight from the kernels (no read-back copy)
    double* vn_mapped = nullptr;
    // (one-pass gradients only: a multi-pass solve writes its Ritz vectors at every Rayleigh-Ritz)
    if (!io_overlap && one_pass_kind && ld_next_host == r && getenv("MEGB200_NO_ZEROCOPY") == nullptr &&
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&vn_mapped), V_next_host, 0) != cudaSuccess) {
      cudaGetLastError();
      vn_mapped = nullptr;
    }
    if (vn_mapped) o.V_next = vn_mapped;
    static const bool htime = getenv("MEGB200_HOST_TIMING") != nullptr;  // diagnostics
    static double acc[4] = {0, 0, 0, 0};
    static int64_t nacc = 0;
    const auto h0 = std::chrono::steady_clock::now();
    try {
      step_core(s, &it, &gg, eta, eps_next, opts, &o, (ld_next_host == r && !vn_mapped) ? V_next_host : nullptr, r,
                &v_done);
      if (vn_mapped) v_done = true;
      if (htime) {
        const auto h1 = std::chrono::steady_clock::now();
        acc[0] += std::chrono::duration<double, std::micro>(h1 - h0).count();
        if (++nacc % 200 == 0) {
          fprintf(stderr, "host step: step_core %.1f us avg over %lld calls\n", acc[0] / nacc, (long long)nacc);
        }
      }
    } catch (const Error&) {
      s->want_vgram = 0;
      s->sync();
      gram_check();  // an invalid factor takes precedence over what the step made of it
      throw;
    }
    s->want_vgram = 0;
    s->sync();
    gram_check();
    if (!v_done) {
      if (ld_next_host == r)
        MEG_CUDA(cudaMemcpyAsync(V_next_host, Vn, (size_t)n * r * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
      else
        MEG_CUDA(cudaMemcpy2DAsync(V_next_host, ld_next_host * sizeof(double), Vn, r * sizeof(double),
                                   r * sizeof(double), n, cudaMemcpyDeviceToHost, s->stream));
      s->sync();
    }
    double* keep_v = out->V_next;
    const int64_t keep_ld = out->ld_next;
    *out = o;
    out->V_next = keep_v;
    out->ld_next = keep_ld;
  });
}

int megb200_dense_stats(megb200_solver* s, const void* M, int32_t dtype, int64_t ld, double* norm2, double* trace) {
  return guarded_impl([&] {
    if (!s || !M) throw Error(MEGB200_ERR_PARAM, "solver/operand is NULL");
    Launch L = s->launch();
    const int slots = std::min<int>(s->sm_count * 2, 1024);
    dense_stats(L, M, dtype, ld, s->n, s->red, slots);
    reduce_sum(L, s->red, slots, 2, s->small);
    double h[2];
    s->d2h(h, s->small, 2);
    s->sync();
    if (norm2) *norm2 = h[0];
    if (trace) *trace = h[1];
  });
}

int megb200_objective_value(megb200_solver* s, const megb200_gradient* g, double m_norm2, double m_trace,
                            double* value) {
  return guarded_impl([&] {
    if (!s || !value) throw Error(MEGB200_ERR_PARAM, "solver/value is NULL");
    check_gradient(s, g);
    Launch L = s->launch();
    const int64_t n = s->n, r = g->g_r;
    std::vector<double> c;
    double tail = 0.0;
    x_coeffs(n, r, g->g_lam, g->g_eps, c, tail);
    if (g->kind == MEGB200_GRAD_SAMPLED) {
      s->h2d(s->small, c.data(), r);
      csr_values(L, n, g->rowptr, g->col, g->obs, g->gV, g->g_ldv, (int)r, s->small, tail, nullptr, s->rowsq, 0);
      // sum of per-row squares in fixed order: tn of a column vector with ones is avoided; reuse reduce over slots
      const int slots = (int)std::min<int64_t>(n, 1024);
      // rows -> slots partial sums via tn-like two-level reduction: treat rowsq as (n x 1) and use tn with a ones column
      std::vector<double> ones((size_t)n, 1.0);
      double* d_ones = s->T;  // n doubles of scratch (ld ldq) -> use contiguous column view of T
      s->h2d(d_ones, ones.data(), n);
      tn(L, n, s->rowsq, 1, 1, d_ones, 1, 1, s->small + 64, 1, nullptr, s->red, s->red_cap, s->sm_count);
      (void)slots;
      double h = 0.0;
      s->d2h(&h, s->small + 64, 1);
      s->sync();
      *value = 0.5 * h;
      return;
    }
    if (g->kind != MEGB200_GRAD_FROBENIUS && g->kind != MEGB200_GRAD_STOCHASTIC)
      throw Error(MEGB200_ERR_PARAM, "objective value needs a Frobenius or sampled gradient descriptor");
    if (isnan(m_norm2) || isnan(m_trace)) {
      if (s->m_cache_ptr != g->dense) {
        double a = 0, b = 0;
        int rc = megb200_dense_stats(s, g->dense, g->dtype, g->ld, &a, &b);
        if (rc != MEGB200_OK) throw Error(rc, g_last_error);
        s->m_norm2_cache = a;
        s->m_trace_cache = b;
        s->m_cache_ptr = g->dense;
      }
      if (isnan(m_norm2)) m_norm2 = s->m_norm2_cache;
      if (isnan(m_trace)) m_trace = s->m_trace_cache;
    }
    // M V -> T[:, 0:r]; diag(V^T M V)
    OpDev op;
    op.kind = MEGB200_OP_DENSE;
    op.dtype = g->dtype;
    op.dense = g->dense;
    op.ld = g->ld;
    op.scale = 1.0;
    apply_op_wide(s, op, g->gV, g->g_ldv, (int)r, s->T, s->ldq);
    tn(L, n, g->gV, g->g_ldv, (int)r, s->T, s->ldq, (int)r, s->G, r, nullptr, s->red, s->red_cap, s->sm_count);
    std::vector<double> vmv((size_t)r * r);
    s->d2h(vmv.data(), s->G, r * r);
    s->sync();
    double x2 = tail * tail * (double)(n - r), inner = tail * m_trace;
    for (int64_t k = 0; k < r; ++k) {
      const double kept = (1.0 - g->g_eps) * g->g_lam[k];
      x2 += kept * kept;
      inner += c[k] * vmv[(size_t)k * r + k];
    }
    *value = 0.5 * (x2 - 2.0 * inner + m_norm2);
  });
}

int megb200_objective_value_direct(megb200_solver* s, const megb200_gradient* g, double* value) {
  return guarded_impl([&] {
    if (!s || !value) throw Error(MEGB200_ERR_PARAM, "solver/value is NULL");
    check_gradient(s, g);
    if (g->kind == MEGB200_GRAD_SAMPLED) {  // the sampled value is already an entry-by-entry sum
      const int rc = megb200_objective_value(s, g, NAN, NAN, value);
      if (rc != MEGB200_OK) throw Error(rc, g_last_error);
      return;
    }
    if (g->kind != MEGB200_GRAD_FROBENIUS && g->kind != MEGB200_GRAD_STOCHASTIC)
      throw Error(MEGB200_ERR_PARAM, "objective value needs a Frobenius or sampled gradient descriptor");
    const int64_t n = s->n, r = g->g_r;
    if (r > 64) throw Error(MEGB200_ERR_PARAM, "direct objective value supports r <= 64");
    Launch L = s->launch();
    std::vector<double> c;
    double tail = 0.0;
    x_coeffs(n, r, g->g_lam, g->g_eps, c, tail);
    s->h2d(s->small, c.data(), r);
    const int slots = std::min<int>(s->sm_count * 4, 1024);
    frob_direct(L, g->dense, g->dtype, g->ld, n, g->gV, g->g_ldv, (int)r, s->small, tail, s->red, slots);
    reduce_sum(L, s->red, slots, 1, s->small + 64);
    double h = 0.0;
    s->d2h(&h, s->small + 64, 1);
    s->sync();
    *value = 0.5 * h;
  });
}

namespace {
void dual_gap_core(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts, double m_trace,
                   double* gap, double* lambda_min, double* ritz_out, int64_t ld_ritz, int32_t* ritz_cols);
}

int megb200_dual_gap(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts, double m_trace,
                     double* gap, double* lambda_min) {
  return guarded_impl([&] { dual_gap_core(s, g, opts, m_trace, gap, lambda_min, nullptr, 0, nullptr); });
}

int megb200_dual_gap_warm(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts,
                          double m_trace, double* gap, double* lambda_min, double* ritz_out, int64_t ld_ritz,
                          int32_t* ritz_cols) {
  return guarded_impl([&] {
    if (!ritz_out || !ritz_cols || ld_ritz < s->max_block) throw Error(MEGB200_ERR_PARAM, "Ritz block output missing");
    dual_gap_core(s, g, opts, m_trace, gap, lambda_min, ritz_out, ld_ritz, ritz_cols);
  });
}

namespace {
void dual_gap_core(megb200_solver* s, const megb200_gradient* g, const megb200_eig_opts* opts, double m_trace,
                   double* gap, double* lambda_min, double* ritz_out, int64_t ld_ritz, int32_t* ritz_cols) {
  {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    check_gradient(s, g);
    if (g->kind != MEGB200_GRAD_FROBENIUS && g->kind != MEGB200_GRAD_STOCHASTIC)
      throw Error(MEGB200_ERR_PARAM, "dual gap needs a Frobenius gradient descriptor");
    const int64_t n = s->n, r = g->g_r;
    std::vector<double> c;
    double tail = 0.0;
    x_coeffs(n, r, g->g_lam, g->g_eps, c, tail);
    // -grad = M - X = M - Vg diag(c) Vg^T - tail I; its top eigenvalue is -lambda_min(grad)
    OpDev op;
    op.kind = MEGB200_OP_DENSE;
    op.dtype = g->dtype;
    op.dense = g->dense;
    op.ld = g->ld;
    op.scale = 1.0;
    op.L = g->gV;
    op.ldl = g->g_ldv;
    op.l = (int)r;
    std::vector<double> d(r);
    for (int64_t k = 0; k < r; ++k) d[k] = -c[k];
    s->h2d(s->dvec, d.data(), r);
    op.d_dev = s->dvec;
    op.alpha = -tail;
    EigParams P = params_from_opts(opts);
    int rc_cols = 0;
    EigRun run = top_eigs(s, op, 1, P, nullptr, 0, ritz_out, ld_ritz, ritz_out ? &rc_cols : nullptr);
    if (!run.converged) throw_lanczos(run, P.tol);
    if (ritz_cols) *ritz_cols = rc_cols;
    const double lmin = -run.theta[0];
    // Tr(X grad) = ||X||^2 - <X, M>
    if (isnan(m_trace)) {
      double a = 0, b = 0;
      int rc = megb200_dense_stats(s, g->dense, g->dtype, g->ld, &a, &b);
      if (rc != MEGB200_OK) throw Error(rc, g_last_error);
      m_trace = b;
    }
    Launch L = s->launch();
    OpDev mop;
    mop.kind = MEGB200_OP_DENSE;
    mop.dtype = g->dtype;
    mop.dense = g->dense;
    mop.ld = g->ld;
    mop.scale = 1.0;
    apply_op_wide(s, mop, g->gV, g->g_ldv, (int)r, s->T, s->ldq);
    tn(L, n, g->gV, g->g_ldv, (int)r, s->T, s->ldq, (int)r, s->G, r, nullptr, s->red, s->red_cap, s->sm_count);
    std::vector<double> vmv((size_t)r * r);
    s->d2h(vmv.data(), s->G, r * r);
    s->sync();
    double x2 = tail * tail * (double)(n - r), inner = tail * m_trace;
    for (int64_t k = 0; k < r; ++k) {
      const double kept = (1.0 - g->g_eps) * g->g_lam[k];
      x2 += kept * kept;
      inner += c[k] * vmv[(size_t)k * r + k];
    }
    if (gap) *gap = (x2 - inner) - lmin;
    if (lambda_min) *lambda_min = lmin;
  }
}
}  // namespace

int megb200_qm_residuals(megb200_solver* s, const double* a, const double* b, const double* y, int64_t m,
                         const double* V, int64_t ldv, int32_t r, const double* lam_host, double eps, double tau,
                         double* res) {
  return guarded_impl([&] {
    if (!s || !a || !b || !y || !V || !lam_host || !res) throw Error(MEGB200_ERR_PARAM, "null argument");
    const int64_t n = s->n;
    if (m < 1) throw Error(MEGB200_ERR_PARAM, "need m >= 1");
    if (!(1 <= r && r < n) || r > 32 || ldv < r) throw Error(MEGB200_ERR_PARAM, "need 1 <= r < n, r <= 32");
    // eps = 0 evaluates the plain low-rank X = V diag(lam) V^T (any V: the spectral-init probe)
    if (!(eps >= 0.0 && eps <= 0.75)) throw Error(MEGB200_ERR_PARAM, "eps must lie in [0, 3/4]");
    QmCoef qc;
    qc.tau = tau;
    qc.eps = eps;
    qc.tail = eps / (double)(n - r);
    for (int k = 0; k < r; ++k) qc.lam[k] = lam_host[k];
    qm_residuals(s->launch(), a, b, y, m, n, V, ldv, r, qc, res);
  });
}

int megb200_qm_gradient(megb200_solver* s, const double* a, const double* b, const double* res, int64_t m,
                        double weight, double* G, int64_t ldg) {
  return guarded_impl([&] {
    if (!s || !a || !b || !res || !G) throw Error(MEGB200_ERR_PARAM, "null argument");
    const int64_t n = s->n;
    if (m < 1 || ldg < n) throw Error(MEGB200_ERR_PARAM, "need m >= 1 and ldg >= n");
    const int64_t need = qm_grad_part_doubles(m, n);
    if (need > s->qm_part_len) {
      s->sync();
      if (s->qm_part) MEG_CUDA(cudaFree(s->qm_part));
      s->qm_part = nullptr;
      MEG_CUDA(cudaMalloc(&s->qm_part, (size_t)need * sizeof(double)));
      s->qm_part_len = need;
    }
    qm_gradient(s->launch(), a, b, res, m, n, weight, G, ldg, s->qm_part);
  });
}

int megb200_qm_gradient_batch(megb200_solver* s, const double* a, const double* b, const double* res,
                              const int64_t* idx, int64_t L, double weight, double* G, int64_t ldg) {
  return guarded_impl([&] {
    if (!s || !a || !b || !res || !idx || !G) throw Error(MEGB200_ERR_PARAM, "null argument");
    const int64_t n = s->n;
    if (L < 1 || ldg < n) throw Error(MEGB200_ERR_PARAM, "need L >= 1 and ldg >= n");
    const int64_t need = qm_grad_part_doubles(L, n);
    if (need > s->qm_part_len) {
      s->sync();
      if (s->qm_part) MEG_CUDA(cudaFree(s->qm_part));
      s->qm_part = nullptr;
      MEG_CUDA(cudaMalloc(&s->qm_part, (size_t)need * sizeof(double)));
      s->qm_part_len = need;
    }
    qm_gradient(s->launch(), a, b, res, L, n, weight, G, ldg, s->qm_part, idx);
  });
}

int megb200_qm_value(megb200_solver* s, const double* res, int64_t m, double* value) {
  return guarded_impl([&] {
    if (!s || !res || !value || m < 1) throw Error(MEGB200_ERR_PARAM, "bad arguments");
    qm_sumsq(s->launch(), res, m, s->small);
    s->d2h(s->h_buf, s->small, 1);
    s->sync();
    *value = s->h_buf[0];
  });
}

int64_t megb200_qm_apply_scratch(megb200_solver* s, int64_t m, int32_t k) {
  if (!s || m < 1 || k < 1 || k > 32) return -1;
  return qm_apply_scratch_doubles(m, s->n, k, s->sm_count);
}

int megb200_qm_apply(megb200_solver* s, const megb200_qm_data* q, const double* U, int64_t ldu, int32_t k,
                     double* W, int64_t ldw) {
  return guarded_impl([&] {
    if (!s || !U || !W || k < 1 || ldu < k || ldw < k) throw Error(MEGB200_ERR_PARAM, "invalid block");
    check_qm_data(q);
    OpDev op;
    op.kind = MEGB200_OP_QUADMEAS;
    op.apply_ctx = const_cast<megb200_qm_data*>(q);
    op.scale = 1.0;
    apply_op_wide(s, op, U, ldu, k, W, ldw);
  });
}

int megb200_gen_sampled_pattern(megb200_solver* s, uint64_t seed, double p, int32_t* rowptr, int64_t* nnz) {
  return guarded_impl([&] {
    if (!s || !rowptr || !nnz) throw Error(MEGB200_ERR_PARAM, "null argument");
    if (!(p > 0.0 && p <= 1.0)) throw Error(MEGB200_ERR_PARAM, "sampling probability must lie in (0, 1]");
    const int64_t n = s->n;
    sampled_count(s->launch(), n, stream_key(seed, 3), p, rowptr + 1);
    std::vector<int32_t> c((size_t)n + 1, 0);
    MEG_CUDA(cudaMemcpyAsync(c.data() + 1, rowptr + 1, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    s->sync();
    int64_t acc = 0;
    for (int64_t i = 0; i <= n; ++i) {
      acc += c[(size_t)i];
      if (acc > INT32_MAX) throw Error(MEGB200_ERR_PARAM, "sampled pattern exceeds int32 indices");
      c[(size_t)i] = (int32_t)acc;
    }
    MEG_CUDA(cudaMemcpyAsync(rowptr, c.data(), ((size_t)n + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
    s->sync();
    *nnz = acc;
  });
}

int megb200_gen_sampled_values(megb200_solver* s, uint64_t seed, double p, const double* U, int64_t r,
                               const double* lam_host, double obs_noise, const int32_t* rowptr, int32_t* col,
                               double* val) {
  return guarded_impl([&] {
    if (!s || !U || !lam_host || !rowptr || !col || !val) throw Error(MEGB200_ERR_PARAM, "null argument");
    if (r < 0 || r > 64) throw Error(MEGB200_ERR_PARAM, "r must be in [0, 64]");
    s->h2d(s->small, lam_host, r);
    sampled_fill(s->launch(), s->n, stream_key(seed, 3), stream_key(seed, 4), p, U, (int)r, s->small, obs_noise, rowptr,
                 col, val);
    s->sync();
  });
}

int megb200_gen_dense_target(megb200_solver* s, const double* U, int64_t r, const double* lam_host, double sigma,
                             uint64_t seed, int32_t stream, void* M, int32_t dtype, int64_t ld) {
  return guarded_impl([&] {
    if (!s || !U || !M || !lam_host) throw Error(MEGB200_ERR_PARAM, "null argument");
    if (r < 0 || r > 64) throw Error(MEGB200_ERR_PARAM, "r must be in [0, 64]");
    s->h2d(s->small, lam_host, r);
    gen_dense_target(s->launch(), U, r, s->small, sigma, stream_key(seed, (uint64_t)stream), M, dtype, ld, s->n);
    s->sync();
  });
}

// Diagnostics (not part of the ABI header): phase timestamps of the last fused first pass
// (solver run with MEGB200_FUSED_STAMPS=1).
int megb200_debug_fused_ns(megb200_solver* s, unsigned long long* out, int32_t count) {
  return guarded_impl([&] {
    if (!s || !out || count < 1 || count > 64) throw Error(MEGB200_ERR_PARAM, "bad arguments");
    MEG_CUDA(cudaMemcpy(out, s->fsync + 128, count * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

int megb200_profile_enable(megb200_solver* s, int32_t enable) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    if (enable < 0) throw Error(MEGB200_ERR_PARAM, "profile stride must be >= 0");
    s->prof = enable;
    s->prof_seen = 0;
  });
}

int megb200_profile_read(megb200_solver* s, double* pass_ms, int64_t* passes, double* bytes) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    s->sync();
    double total = 0.0;
    for (auto& pr : s->ev_pending) {
      float ms = 0.f;
      MEG_CUDA(cudaEventElapsedTime(&ms, s->ev_pool[pr.first], s->ev_pool[pr.second]));
      total += ms;
    }
    if (pass_ms) *pass_ms = total;
    if (passes) *passes = s->prof_passes;
    if (bytes) *bytes = s->prof_bytes;
    s->ev_pending.clear();
    s->ev_next = 0;
    s->prof_bytes = 0.0;
    s->prof_passes = 0;
  });
}

int megb200_trace_enable(megb200_solver* s, int32_t enable) {
  return guarded_impl([&] {
    if (!s) throw Error(MEGB200_ERR_PARAM, "solver is NULL");
    s->trace = enable != 0;
    s->marks.clear();
    s->trace_next = 0;
    s->trace_acc.clear();
    s->trace_stat.clear();
  });
}

int megb200_trace_report(megb200_solver* s, char* buf, int64_t len) {
  return guarded_impl([&] {
    if (!s || !buf || len < 1) throw Error(MEGB200_ERR_PARAM, "null argument");
    std::string out;
    char line[160];
    for (auto& kv : s->trace_acc) {
      snprintf(line, sizeof line, "%-14s %10.2f us avg  x%lld\n", kv.first.c_str(),
               1e3 * kv.second.first / std::max<int64_t>(1, kv.second.second), (long long)kv.second.second);
      out += line;
    }
    for (auto& kv : s->trace_stat) {
      snprintf(line, sizeof line, "%-22s %8.2f avg  x%lld\n", kv.first.c_str(),
               kv.second.first / std::max<int64_t>(1, kv.second.second), (long long)kv.second.second);
      out += line;
    }
    snprintf(buf, (size_t)len, "%s", out.c_str());
  });
}

int megb200_gram_error(megb200_solver* s, const double* V, int64_t ldv, int32_t r, double* err) {
  return guarded_impl([&] {
    if (!s || !V || !err) throw Error(MEGB200_ERR_PARAM, "null argument");
    if (r < 1 || r > s->cap) throw Error(MEGB200_ERR_PARAM, "r out of range");
    *err = gram_error(s, V, ldv, r);
  });
}

int megb200_gen_gaussian(megb200_solver* s, uint64_t seed, int32_t stream, uint64_t base, int64_t n, int64_t k,
                         double scale, int32_t round_f32, double* out, int64_t ld) {
  return guarded_impl([&] {
    if (!s || !out) throw Error(MEGB200_ERR_PARAM, "null argument");
    fill_gaussian(s->launch(), n, (int)k, stream_key(seed, (uint64_t)stream), base, scale, round_f32 != 0, out, ld);
  });
}

}  // extern "C"
