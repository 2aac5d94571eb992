"""Error types mirroring the reference (linalg.py:23-52), same bases and payloads."""

from __future__ import annotations

import numpy as np


class ParameterError(ValueError):
    """A structurally invalid argument (bad rank, bad shape) -- linalg.py:23-24."""


class EighError(RuntimeError):
    """Dense eigendecomposition failed to converge -- linalg.py:27-28."""


class RankDeficiencyError(ValueError):
    """Orthonormalization hit a numerically dependent column -- linalg.py:31-40."""

    def __init__(self, column: int, norm: float):
        self.column = column
        self.norm = norm
        super().__init__(f"column {column} is numerically dependent on the previous ones (residual norm {norm:.3e})")


class LanczosError(RuntimeError):
    """The eigensolver did not reach the residual tolerance -- linalg.py:43-52.

    Carries the best residual norms seen so the caller can decide whether to
    retry with a larger subspace.
    """

    def __init__(self, message: str, residual_norms: np.ndarray):
        self.residual_norms = residual_norms
        super().__init__(message)
