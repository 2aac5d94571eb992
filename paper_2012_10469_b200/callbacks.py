"""Caller-supplied applications: the reference's Python callables on the device solver.

The reference passes plain callables -- `SymmetricOperator(dim, apply_fn)` (linalg.py:81-94)
and `lowrank_meg_step(x, grad_apply, ...)` (meg.py:327-335), e.g. `lambda u: g @ u`
(test_meg.py:153).  The B200 solver accepts them through the C ABI's callback operator
(MEGB200_OP_CALLBACK / MEGB200_GRAD_CALLBACK, include/megb200.h): once per block pass the
native solver calls back with device pointers to the n x k block U and the output W.

Two calling conventions:

* numpy (default, the reference's): the callable receives a numpy (n, k) block and returns
  one.  The block crosses the host link each pass; the solver itself stays on the device.
* device (`device_callable(fn)`): the callable receives a torch CUDA tensor view of U and
  returns a CUDA tensor; nothing leaves the device (the solver stream is drained before the
  call and the device synchronised after it).

Descriptor gradients (objectives.py) remain the fast path: they stream from HBM inside the
pass kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, runtime


class CallbackError(RuntimeError):
    """A callback failed without a Python exception to re-raise."""


def device_callable(fn):
    """Mark `fn` as taking and returning torch CUDA tensors (run on the solver stream)."""
    fn.__megb200_device__ = True
    return fn


class _DeviceBlock:
    """__cuda_array_interface__ view of an n x k float64 row-major block (ld elements)."""

    def __init__(self, ptr: int, n: int, k: int, ld: int):
        self.__cuda_array_interface__ = {
            "shape": (n, k), "strides": (ld * 8, 8), "typestr": "<f8", "data": (int(ptr), False), "version": 3,
        }


_H2D, _D2H = 1, 2
_cudart = None


def _cudart_sync(stream) -> None:
    _cudart_copy2d(None, 0, None, 0, 0, 0, 0, stream)


def _cudart_copy2d(dst, dpitch, src, spitch, width, height, kind, stream) -> None:
    """cudaMemcpy2DAsync (skipped for width 0) + cudaStreamSynchronize on `stream` (the solver's)."""
    global _cudart
    if _cudart is None:
        import ctypes
        import ctypes.util
        import glob
        import os

        cands = [ctypes.util.find_library("cudart")] + sorted(
            glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                   "libcudart.so*"))) + ["libcudart.so.12", "libcudart.so"]
        for c in cands:
            if not c:
                continue
            try:
                _cudart = ctypes.CDLL(c)
                break
            except OSError:
                continue
        if _cudart is None:
            raise CallbackError("libcudart not found for the host round trip of a numpy callable")
        _cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                              ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        _cudart.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]
    rc = _cudart.cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, stream) if width else 0
    if rc == 0:
        rc = _cudart.cudaStreamSynchronize(stream)
    if rc != 0:
        raise CallbackError(f"CUDA error {rc} in the callback's host round trip")


class ApplyCallback:
    """Wraps a Python apply function as a megb200_apply_fn (keep the object alive during calls)."""

    def __init__(self, fn, n: int, device: bool | None = None):
        if not callable(fn):
            raise TypeError("apply function must be callable")
        self.fn = fn
        self.n = int(n)
        self.device = bool(getattr(fn, "__megb200_device__", False)) if device is None else bool(device)
        self.error: BaseException | None = None
        self.calls = 0
        self.c_fn = _lib.APPLY_FN(self._call)

    def _call(self, ctx, U, ldu, k, W, ldw, stream):
        try:
            if self.device:
                # the block is ready once the solver stream drains; the user's torch work then runs on
                # torch's own stream and is waited for device-wide before the solver continues
                _cudart_sync(stream)
                dev = runtime.device()
                u = torch.as_tensor(_DeviceBlock(U, self.n, k, ldu), device=dev)
                w = torch.as_tensor(_DeviceBlock(W, self.n, k, ldw), device=dev)
                out = self.fn(u)
                out = torch.as_tensor(out, device=dev).to(torch.float64).reshape(self.n, k)
                w.copy_(out)
                torch.cuda.synchronize(dev)
            else:
                # host round trip by the CUDA runtime on the solver stream (pitched copies, synchronised)
                uh = np.empty((self.n, k), dtype=np.float64)
                _cudart_copy2d(uh.ctypes.data, k * 8, U, ldu * 8, k * 8, self.n, _D2H, stream)
                out = np.ascontiguousarray(np.asarray(self.fn(uh), dtype=np.float64).reshape(self.n, k))
                _cudart_copy2d(W, ldw * 8, out.ctypes.data, k * 8, k * 8, self.n, _H2D, stream)
            self.calls += 1
            return 0
        except BaseException as exc:  # re-raised by the caller of the native function
            self.error = exc
            return 1

    def raise_error(self):
        if self.error is not None:
            err, self.error = self.error, None
            raise err


def checked(rc: int, callbacks, residual_norms=None) -> None:
    """runtime.check, re-raising a callback's own exception when it caused the failure."""
    if rc == _lib.ERR_CALLBACK:
        for cb in callbacks:
            if cb is not None:
                cb.raise_error()
        raise CallbackError(_lib.last_error())
    runtime.check(rc, residual_norms=residual_norms)
