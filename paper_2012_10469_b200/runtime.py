"""Device plumbing: solver handles, stream binding, tensor conversion, error mapping.

torch supplies device memory and the current CUDA stream; every numeric
kernel is in libmegb200.so (csrc/).  There is no CPU fallback: on a machine
without a B200 the first call raises.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from .errors import LanczosError, ParameterError

_lock = threading.Lock()
_solvers: dict = {}

MAX_BLOCK = 64
MAX_BASIS = 112
MAX_LOWRANK = 160


class Solver:
    """Owns one native handle (device workspace arena) for dimension n."""

    def __init__(self, n: int, max_nnz: int = 0, max_lowrank: int = MAX_LOWRANK):
        lib = _lib.load()
        handle = C.c_void_p()
        check(lib.megb200_solver_create(int(n), MAX_BLOCK, MAX_BASIS, int(max_lowrank), int(max_nnz), C.byref(handle)))
        self.lib = lib
        self.handle = handle
        self.n = int(n)
        self.max_nnz = int(max_nnz)
        self.max_lowrank = int(max_lowrank)

    _bound_stream = None

    def bind_stream(self, dev_index: int | None = None) -> None:
        idx = torch.cuda.current_device() if dev_index is None else dev_index
        stream = torch._C._cuda_getCurrentRawStream(idx)
        if stream != self._bound_stream:
            check(self.lib.megb200_solver_set_stream(self.handle, C.c_void_p(stream)))
            self._bound_stream = stream

    @property
    def launches(self) -> int:
        return int(self.lib.megb200_kernel_launches(self.handle))

    @property
    def workspace_bytes(self) -> int:
        return int(self.lib.megb200_solver_workspace_bytes(self.handle))

    def __del__(self):
        try:
            if self.handle:
                self.lib.megb200_solver_destroy(self.handle)
        except Exception:
            pass


_fast = {}


def solver_for(n: int, max_nnz: int = 0, max_lowrank: int = MAX_LOWRANK) -> Solver:
    """Cached handle per dimension (grown when a larger nnz/low-rank width is needed)."""
    dev = torch.cuda.current_device()
    s = _fast.get((dev, n))
    if s is not None and s.max_nnz >= max_nnz and s.max_lowrank >= max_lowrank:
        s.bind_stream(dev)
        return s
    with _lock:
        s = _solvers.get((dev, n))
        if s is None or s.max_nnz < max_nnz or s.max_lowrank < max_lowrank:
            s = Solver(n, max(max_nnz, s.max_nnz if s else 0), max(max_lowrank, s.max_lowrank if s else 0))
            _solvers[(dev, n)] = s
        _fast[(dev, n)] = s
    s.bind_stream(dev)
    return s


def check(rc: int, residual_norms=None) -> None:
    """Map a native status to the reference's exception classes."""
    if rc == _lib.OK:
        return
    msg = _lib.last_error()
    if rc == _lib.ERR_PARAM:
        raise ParameterError(msg)
    if rc == _lib.ERR_LANCZOS:
        res = np.asarray(residual_norms if residual_norms is not None else [], dtype=float)
        raise LanczosError(msg, residual_norms=res)
    if rc == _lib.ERR_KEPT_MASS:
        raise AssertionError("kept mass vanished despite max-shift")
    if rc == _lib.ERR_NO_DEVICE:
        raise _lib.NativeLibraryError(msg)
    if rc == _lib.ERR_CALLBACK:
        from .callbacks import CallbackError

        raise CallbackError(msg)
    raise RuntimeError(f"megb200 CUDA error: {msg}")


_devices: dict = {}


def device() -> torch.device:
    if not _devices:
        if not torch.cuda.is_available():
            raise _lib.NativeLibraryError("no CUDA device: the B200 path has no CPU fallback")
    idx = torch.cuda.current_device()
    d = _devices.get(idx)
    if d is None:
        d = _devices[idx] = torch.device("cuda", idx)
    return d


def as_device_f64(a, shape=None) -> torch.Tensor:
    """numpy / torch -> contiguous float64 CUDA tensor (row-major)."""
    if (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.float64 and a.is_contiguous()
            and a.device.index == torch.cuda.current_device() and shape is None):
        return a
    if isinstance(a, torch.Tensor):
        t = a.to(device=device(), dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(device())
    t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ParameterError(f"expected shape {shape}, got {tuple(t.shape)}")
    return t


def as_device_operand(a, dtype: str) -> torch.Tensor:
    """Dense n x n operand in f64 or f32, contiguous on device."""
    tdt = torch.float64 if dtype == "f64" else torch.float32
    if isinstance(a, torch.Tensor):
        t = a.to(device=device(), dtype=tdt)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a))).to(device()).to(tdt)
    return t.contiguous()


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return _lib.F64
    if t.dtype == torch.float32:
        return _lib.F32
    raise ParameterError(f"unsupported operand dtype {t.dtype}")


def ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def host_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))
