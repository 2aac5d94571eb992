"""ctypes binding of the C ABI in include/megb200.h (libmegb200.so, built in-tree).

This is the binding a maintainer of the reference would add:
the reference is pure Python, so its FFI for this path is ctypes.  The
library is loaded lazily and any failure is loud: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmegb200.so")

OK, ERR_PARAM, ERR_LANCZOS, ERR_CUDA, ERR_KEPT_MASS, ERR_NO_DEVICE, ERR_CALLBACK = range(7)
F64, F32 = 0, 1
OP_NONE, OP_DENSE, OP_CSR, OP_CALLBACK, OP_QUADMEAS = 0, 1, 2, 3, 4
GRAD_ZERO, GRAD_DENSE, GRAD_FROBENIUS, GRAD_SAMPLED, GRAD_STOCHASTIC, GRAD_CALLBACK, GRAD_QUADMEAS = range(7)

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)


# int apply(void* ctx, const double* U, int64_t ldu, int32_t k, double* W, int64_t ldw, void* stream)
APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p)


class QmData(C.Structure):
    """megb200_qm_data: the matrix-free quadratic-measurement operator's device arrays."""

    _fields_ = [
        ("a", C.c_void_p), ("b", C.c_void_p), ("res", C.c_void_p), ("m", C.c_int64), ("idx", C.c_void_p), ("weight", C.c_double),
        ("scratch", C.c_void_p), ("scratch_len", C.c_int64),
    ]


class Operator(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("dtype", C.c_int32), ("n", C.c_int64),
        ("dense", C.c_void_p), ("ld", C.c_int64),
        ("rowptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p), ("nnz", C.c_int64),
        ("scale", C.c_double),
        ("L", C.c_void_p), ("l", C.c_int64), ("ldl", C.c_int64), ("d", c_double_p),
        ("alpha", C.c_double), ("apply", APPLY_FN), ("apply_ctx", C.c_void_p),
    ]


class Gradient(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("dtype", C.c_int32), ("n", C.c_int64),
        ("dense", C.c_void_p), ("ld", C.c_int64),
        ("rowptr", C.c_void_p), ("col", C.c_void_p), ("obs", C.c_void_p), ("nnz", C.c_int64),
        ("gV", C.c_void_p), ("g_r", C.c_int64), ("g_ldv", C.c_int64), ("g_lam", c_double_p), ("g_eps", C.c_double),
        ("A", C.c_void_p), ("bsz", C.c_int64), ("lda", C.c_int64), ("sigma", C.c_double),
        ("apply", APPLY_FN), ("apply_ctx", C.c_void_p),
    ]


class Iterate(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("r", C.c_int64), ("V", C.c_void_p), ("ldv", C.c_int64),
        ("lam", c_double_p), ("eps", C.c_double),
    ]


class EigOpts(C.Structure):
    _fields_ = [
        ("tol", C.c_double), ("max_passes", C.c_int32), ("restarts", C.c_int32),
        ("block", C.c_int32), ("basis", C.c_int32), ("keep", C.c_int32),
        ("seed", C.c_uint64), ("warm", C.c_void_p), ("warm_cols", C.c_int64), ("ld_warm", C.c_int64),
        ("warm_orthonormal", C.c_int32),
    ]


class EigResult(C.Structure):
    _fields_ = [
        ("eigenvalues", c_double_p), ("residual_norms", c_double_p),
        ("eigenvectors", C.c_void_p), ("ld_vec", C.c_int64),
        ("ritz_block", C.c_void_p), ("ld_ritz", C.c_int64),
        ("passes", C.c_int32), ("restarts", C.c_int32), ("norm_est", C.c_double), ("ritz_cols", C.c_int32),
    ]


class StepResult(C.Structure):
    _fields_ = [
        ("V_next", C.c_void_p), ("ld_next", C.c_int64),
        ("lam_next", c_double_p), ("y", c_double_p), ("mu", c_double_p), ("residual_norms", c_double_p),
        ("ritz_block", C.c_void_p), ("ld_ritz", C.c_int64),
        ("lambda_r_plus_1", C.c_double), ("b_r_plus_1", C.c_double), ("shift", C.c_double),
        ("lhs_cheap", C.c_double), ("holds_cheap", C.c_int32), ("threshold", C.c_double),
        ("gram_err", C.c_double), ("passes", C.c_int32), ("restarts", C.c_int32), ("ritz_cols", C.c_int32),
        ("ritz_orth_err", C.c_double),
        ("timed_from", C.c_int64), ("timed_count", C.c_int64), ("timed_ms", C.c_double),
        ("timed_launches", C.c_int64), ("gap", c_double_p), ("lmin", c_double_p),
    ]


class Schedule(C.Structure):
    _fields_ = [
        ("eps_kind", C.c_int32), ("eps0_tilde", C.c_double), ("G", C.c_double), ("c", C.c_double),
        ("eta_kind", C.c_int32), ("eta0", C.c_double),
        ("minibatch_seed", C.c_uint64), ("minibatch_round_f32", C.c_int32), ("cert_every", C.c_int32),
    ]


class RunRecord(C.Structure):
    _fields_ = [
        ("shift", c_double_p), ("y", c_double_p), ("lam", c_double_p), ("eps", c_double_p), ("lhs", c_double_p),
        ("holds", c_int32_p), ("passes", c_int32_p), ("step_ms", c_double_p),
        ("ritz_block", C.c_void_p), ("ld_ritz", C.c_int64), ("ritz_cap", C.c_int64), ("ritz_cols", C.c_int64),
        ("ritz_orth_err", C.c_double),
        ("timed_from", C.c_int64), ("timed_count", C.c_int64), ("timed_ms", C.c_double),
        ("timed_launches", C.c_int64), ("gap", c_double_p), ("lmin", c_double_p),
    ]


EPS_KINDS = {"experiment": 0, "cubic_det": 1, "cubic_det_general": 2, "quadratic_stoch": 3, "constant": 4}


# (name, restype, argtypes) for every symbol include/megb200.h declares
SIGNATURES = [
    ("megb200_abi_version", C.c_int, []),
    ("megb200_last_error", C.c_char_p, []),
    ("megb200_device_check", C.c_int, [C.POINTER(C.c_int)]),
    ("megb200_solver_create", C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]),
    ("megb200_solver_destroy", None, [C.c_void_p]),
    ("megb200_solver_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("megb200_solver_workspace_bytes", C.c_int64, [C.c_void_p]),
    ("megb200_operator_apply", C.c_int,
     [C.c_void_p, C.POINTER(Operator), C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64]),
    ("megb200_logmap_apply", C.c_int,
     [C.c_void_p, C.POINTER(Iterate), C.POINTER(Gradient), C.c_double, C.c_void_p, C.c_int64, C.c_int32,
      C.c_void_p, C.c_int64]),
    ("megb200_top_r", C.c_int, [C.c_void_p, C.POINTER(Operator), C.c_int32, C.POINTER(EigOpts), C.POINTER(EigResult)]),
    ("megb200_lowrank_meg_step", C.c_int,
     [C.c_void_p, C.POINTER(Iterate), C.POINTER(Gradient), C.c_double, C.c_double, C.POINTER(EigOpts),
      C.POINTER(StepResult)]),
    ("megb200_lowrank_meg_step_host", C.c_int,
     [C.c_void_p, C.POINTER(Iterate), C.POINTER(Gradient), C.c_double, C.c_double, C.POINTER(EigOpts),
      C.c_void_p, C.c_int64, C.POINTER(StepResult)]),
    ("megb200_meg_run", C.c_int,
     [C.c_void_p, C.POINTER(Iterate), C.POINTER(Gradient), C.POINTER(Schedule), C.c_int64, C.c_int64,
      C.POINTER(EigOpts), C.c_uint64, C.c_void_p, C.c_int64, c_double_p, c_double_p, C.POINTER(RunRecord)]),
    ("megb200_certificate_cheap", C.c_int,
     [C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, c_double_p, c_int32_p, c_double_p]),
    ("megb200_objective_value", C.c_int, [C.c_void_p, C.POINTER(Gradient), C.c_double, C.c_double, c_double_p]),
    ("megb200_objective_value_direct", C.c_int, [C.c_void_p, C.POINTER(Gradient), c_double_p]),
    ("megb200_sym_eigh", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    ("megb200_gradient_apply", C.c_int,
     [C.c_void_p, C.POINTER(Gradient), C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64]),
    ("megb200_dense_stats", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, c_double_p, c_double_p]),
    ("megb200_dual_gap", C.c_int,
     [C.c_void_p, C.POINTER(Gradient), C.POINTER(EigOpts), C.c_double, c_double_p, c_double_p]),
    ("megb200_dual_gap_warm", C.c_int,
     [C.c_void_p, C.POINTER(Gradient), C.POINTER(EigOpts), C.c_double, c_double_p, c_double_p, C.c_void_p, C.c_int64,
      c_int32_p]),
    ("megb200_qm_residuals", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, c_double_p,
      C.c_double, C.c_double, C.c_void_p]),
    ("megb200_qm_gradient", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64]),
    ("megb200_qm_value", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, c_double_p]),
    ("megb200_qm_apply_scratch", C.c_int64, [C.c_void_p, C.c_int64, C.c_int32]),
    ("megb200_qm_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64]),
    ("megb200_qm_gradient_batch", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64]),
    ("megb200_gen_dense_target", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, c_double_p, C.c_double, C.c_uint64, C.c_int32, C.c_void_p, C.c_int32,
      C.c_int64]),
    ("megb200_gen_sampled_pattern", C.c_int, [C.c_void_p, C.c_uint64, C.c_double, C.c_void_p, C.POINTER(C.c_int64)]),
    ("megb200_gen_sampled_values", C.c_int,
     [C.c_void_p, C.c_uint64, C.c_double, C.c_void_p, C.c_int64, c_double_p, C.c_double, C.c_void_p, C.c_void_p,
      C.c_void_p]),
    ("megb200_gen_gaussian", C.c_int,
     [C.c_void_p, C.c_uint64, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int32, C.c_void_p,
      C.c_int64]),
    ("megb200_gram_error", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, c_double_p]),
    ("megb200_profile_enable", C.c_int, [C.c_void_p, C.c_int32]),
    ("megb200_profile_read", C.c_int, [C.c_void_p, c_double_p, C.POINTER(C.c_int64), c_double_p]),
    ("megb200_trace_enable", C.c_int, [C.c_void_p, C.c_int32]),
    ("megb200_trace_report", C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    ("megb200_kernel_launches", C.c_int64, [C.c_void_p]),
]

_lib = None


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or failed to load (no fallback exists)."""


def load() -> C.CDLL:
    """Load libmegb200.so (once) and bind every declared symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 path)"
        )
    try:
        lib = C.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if lib.megb200_abi_version() != 1:
        raise NativeLibraryError("libmegb200.so ABI version mismatch")
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().megb200_last_error()
    return msg.decode() if msg else ""


def dptr(values) -> c_double_p:
    """Host float64 array -> double* (caller keeps the array alive)."""
    return values.ctypes.data_as(c_double_p)
