"""Seeded synthetic inputs for the five BASELINE configs -- TEST INFRASTRUCTURE ONLY.

BASELINE.json names no public dataset; these generators stand in with the
shapes, sizes and value distributions the configs state.

Randomness comes from a counter-based generator (splitmix64 finaliser over
key + counter, Box-Muller in float64) so that the device generator in
`paper_2012_10469_b200/csrc/megb200_gen.cu` can produce the same arrays at
sizes the CPU cannot (n = 32768) without uploading them.  Stream ids:

    1  planted factor U (n x r Gaussian, then numpy QR)
    2  dense noise G (n x n, entry (i, j) at counter i*n + j; sym(G) used)
    3  sampling mask of config 3 (uniform at counter i*n + j, i <= j)
    4  observation noise of config 3 (Gaussian at counter i*n + j, i <= j)
    5  stochastic minibatch A_t of config 4 (counter (t*n + i)*b + j)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
TWO_PI = 6.283185307179586


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * GOLDEN + np.uint64(stream) * _M2
    return mix64(np.array([k], dtype=np.uint64))[0]


def _bits(key: np.uint64, ctr: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return mix64(key + (np.asarray(ctr, dtype=np.uint64) + np.uint64(1)) * GOLDEN)


def uniform(key: np.uint64, ctr) -> np.ndarray:
    """U[0,1) with 53 random bits at counter ctr."""
    return (_bits(key, ctr) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def gaussian(key: np.uint64, ctr) -> np.ndarray:
    """N(0,1) at counter ctr: Box-Muller on sub-counters 2c, 2c+1."""
    ctr = np.asarray(ctr, dtype=np.uint64)
    u1 = ((_bits(key, ctr * np.uint64(2)) >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)
    u2 = (_bits(key, ctr * np.uint64(2) + np.uint64(1)) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(TWO_PI * u2)


# ---------------------------------------------------------------------------
# config table (pinned here)


@dataclass(frozen=True)
class MegConfig:
    name: str
    n: int
    r: int
    spectrum: tuple
    noise: float  # sigma_M of the dense symmetric noise
    iters: int
    dtype: str  # "f64" | "f32" (dtype of the streamed operand)
    block: int  # k
    kind: str  # "dense" | "sampled" | "stochastic"
    subspace: int | None = 64  # reference svd_subspace
    eta0: float = 1.0
    eta_decay: bool = False  # eta_t = eta0 / sqrt(t + 1)
    sample_p: float = 0.05
    obs_noise: float = 1e-3
    batch: int = 64
    sigma: float = 0.05
    cert_every: int = 0  # dual-gap certificate cadence (config 5)
    seed: int = 0

    def eta(self, t: int) -> float:
        return self.eta0 / math.sqrt(t + 1) if self.eta_decay else self.eta0

    def eps(self, t: int) -> float:
        """experiment schedule (meg.py:182-190): 0.6/(t+11)^2."""
        return min(0.6 / (t + 11.0) ** 2, 0.75)

    def scaled(self, n: int, iters: int | None = None) -> "MegConfig":
        d = dict(self.__dict__)
        d["n"] = n
        d["name"] = f"{self.name}@n{n}"
        if iters is not None:
            d["iters"] = iters
        return MegConfig(**d)


def _geom(r, ratio):
    w = ratio ** np.arange(r)
    return tuple((w / w.sum()).tolist())


CONFIGS = {
    "cfg1": MegConfig("cfg1", 500, 5, (0.4, 0.25, 0.15, 0.12, 0.08), 0.01, 200, "f64", 13, "dense", subspace=None),
    "cfg2": MegConfig("cfg2", 4096, 10, _geom(10, 0.7), 0.01, 300, "f64", 18, "dense"),
    "cfg3": MegConfig("cfg3", 8192, 10, _geom(10, 0.7), 0.0, 300, "f64", 14, "sampled", subspace=98),
    "cfg4": MegConfig(
        "cfg4", 16384, 8, (0.3, 0.2, 0.15, 0.1, 0.1, 0.05, 0.05, 0.05), 0.0, 1000, "f32", 16, "stochastic",
        eta_decay=True,
    ),
    "cfg5": MegConfig("cfg5", 32768, 20, _geom(20, 0.85), 1e-3, 100, "f32", 32, "dense", cert_every=10),
}


def planted_factor(cfg: MegConfig) -> np.ndarray:
    """Random orthonormal n x r factor: QR of a stream-1 Gaussian block."""
    key = stream_key(cfg.seed, 1)
    g = gaussian(key, np.arange(cfg.n * cfg.r, dtype=np.uint64)).reshape(cfg.n, cfg.r)
    q, _ = np.linalg.qr(g)
    return np.ascontiguousarray(q)


def noise_rows(n: int, seed: int, i0: int, i1: int) -> np.ndarray:
    """Rows i0:i1 of sym(G) = (G + G^T)/2, G_ij ~ N(0, 1/n) at counter i*n + j (stream 2)."""
    key = stream_key(seed, 2)
    ii = np.arange(i0, i1, dtype=np.uint64)[:, None]
    jj = np.arange(n, dtype=np.uint64)[None, :]
    g = gaussian(key, ii * np.uint64(n) + jj)
    gt = gaussian(key, jj * np.uint64(n) + ii)
    return (0.5 / math.sqrt(n)) * (g + gt)


def dense_target(cfg: MegConfig, U: np.ndarray | None = None) -> np.ndarray:
    """M = U diag(Lambda) U^T + sigma sym(G); rounded to fp32 for f32 configs.

    Element formula (the device generator evaluates the same per entry):
    M_ij = sum_k U_ik Lambda_k U_jk + sigma * (g_ij + g_ji) / (2 sqrt(n)).
    """
    U = planted_factor(cfg) if U is None else U
    lam = np.asarray(cfg.spectrum)
    n = cfg.n
    m = (U * lam) @ U.T
    m = 0.5 * (m + m.T)  # exactly symmetric
    if cfg.noise:
        for i0 in range(0, n, 1024):
            i1 = min(n, i0 + 1024)
            m[i0:i1] += cfg.noise * noise_rows(n, cfg.seed, i0, i1)
    if cfg.dtype == "f32":
        m = m.astype(np.float32).astype(np.float64)
    return m


@dataclass
class SampledInstance:
    n: int
    rowptr: np.ndarray  # int32 (n+1)
    col: np.ndarray  # int32 (nnz), sorted within each row
    obs: np.ndarray  # float64 (nnz): M_ij + noise on the observed entries
    planted: np.ndarray  # n x n planted matrix (small n only; None when not kept)

    @property
    def nnz(self) -> int:
        return int(self.col.size)


def sampled_instance(cfg: MegConfig, U: np.ndarray | None = None, keep_planted: bool = True) -> SampledInstance:
    """Config 3: symmetric Bernoulli(p) mask over i <= j, mirrored; noisy observations.

    Observed value = (U Lambda U^T)_ij + obs_noise * N(0,1), noise drawn once
    per unordered pair (stream 4) so the observed matrix is symmetric.
    """
    n = cfg.n
    U = planted_factor(cfg) if U is None else U
    lam = np.asarray(cfg.spectrum)
    kmask, knoise = stream_key(cfg.seed, 3), stream_key(cfg.seed, 4)
    rows, cols, vals = [], [], []
    ul = U * lam
    for i0 in range(0, n, 512):
        i1 = min(n, i0 + 512)
        ii = np.arange(i0, i1, dtype=np.uint64)[:, None]
        jj = np.arange(n, dtype=np.uint64)[None, :]
        lo = np.minimum(ii, jj)
        hi = np.maximum(ii, jj)
        ctr = lo * np.uint64(n) + hi  # canonical (min, max) counter -> symmetric draws
        hit = uniform(kmask, ctr) < cfg.sample_p
        r_idx, c_idx = np.nonzero(hit)
        noise = gaussian(knoise, ctr[r_idx, c_idx])
        planted = (U[r_idx + i0] * U[c_idx]) @ lam  # U_ik U_jk commutes: exactly symmetric
        rows.append(r_idx + i0)
        cols.append(c_idx)
        vals.append(planted + cfg.obs_noise * noise)
    rows = np.concatenate(rows)
    col = np.concatenate(cols).astype(np.int32)
    obs = np.concatenate(vals)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int32)
    planted_m = (ul @ U.T) if keep_planted else None
    return SampledInstance(n=n, rowptr=rowptr, col=col, obs=obs, planted=planted_m)


def minibatch(cfg: MegConfig, t: int) -> np.ndarray:
    """Config 4: A_t ~ N(0, I/n)^{n x b}, stream 5, counter (t*n + i)*b + j."""
    n, b = cfg.n, cfg.batch
    key = stream_key(cfg.seed, 5)
    base = np.uint64(t) * np.uint64(n * b)
    a = gaussian(key, base + np.arange(n * b, dtype=np.uint64)).reshape(n, b) * (1.0 / math.sqrt(n))
    if cfg.dtype == "f32":
        a = a.astype(np.float32).astype(np.float64)
    return a
