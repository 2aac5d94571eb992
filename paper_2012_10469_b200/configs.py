"""The five BASELINE.json configurations, pinned.

Mirrors oracle/inputs.CONFIGS (the oracle keeps its own copy so it never
imports the product); tests/test_host.py asserts the two tables agree.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    r: int
    spectrum: tuple
    noise: float
    iters: int
    dtype: str  # operand dtype: "f64" | "f32"
    block: int  # k
    kind: str  # "dense" | "sampled" | "stochastic"
    subspace: int | None = 64
    eta0: float = 1.0
    eta_decay: bool = False
    sample_p: float = 0.05
    obs_noise: float = 1e-3
    batch: int = 64
    sigma: float = 0.05
    cert_every: int = 0
    seed: int = 0

    def eta(self, t: int) -> float:
        return self.eta0 / math.sqrt(t + 1) if self.eta_decay else self.eta0

    def eps(self, t: int) -> float:
        """EpsilonSchedule.experiment(c=10) (meg.py:182-190)."""
        return min(0.6 / (t + 11.0) ** 2, 0.75)


def _geom(r, ratio):
    w = ratio ** np.arange(r)
    return tuple((w / w.sum()).tolist())


WORKLOADS = {
    "cfg1": Workload("cfg1", 500, 5, (0.4, 0.25, 0.15, 0.12, 0.08), 0.01, 200, "f64", 13, "dense", subspace=None),
    "cfg2": Workload("cfg2", 4096, 10, _geom(10, 0.7), 0.01, 300, "f64", 18, "dense"),
    "cfg3": Workload("cfg3", 8192, 10, _geom(10, 0.7), 0.0, 300, "f64", 14, "sampled", subspace=98),
    "cfg4": Workload("cfg4", 16384, 8, (0.3, 0.2, 0.15, 0.1, 0.1, 0.05, 0.05, 0.05), 0.0, 1000, "f32", 16,
                     "stochastic", eta_decay=True),
    "cfg5": Workload("cfg5", 32768, 20, _geom(20, 0.85), 1e-3, 100, "f32", 32, "dense", cert_every=10),
}
