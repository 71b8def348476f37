"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no mutation, weighting,
resampling, Philox or Kalman code).  It only builds, from fixed seeds:

* the model parameters of the five BASELINE.json configurations (C1..C5),
  rounded to fp32 because the C-ABI takes fp32 model values
  (SURVEY.md §8(b) "All values are fp32; the oracle uses the same fp32 values
  widened to fp64");
* observation sequences y_{0:T-1} simulated from the HMM of eq. `HMM`
   with numpy's PCG64 (reading R14);
* synthetic particle clouds xhat used as the common starting point of
  single-step parity tests.

The configurations follow BASELINE.json `configs`; the readings of the
under-specified parts (C2's orthogonal matrix, C4's coupling, initial laws)
are DESIGN.md readings R11-R13.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional

import numpy as np

PF_LG = 1
PF_SV = 2


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    kind: int           # PF_LG or PF_SV
    d: int              # state dimension
    dy: int             # observation dimension
    M: int              # particles per group
    m: int              # number of groups (2^S)
    T: int              # number of observations
    data_seed: int

    @property
    def N(self) -> int:
        return self.M * self.m

    @property
    def S(self) -> int:
        return int(round(math.log2(self.m)))

    def with_sizes(self, M: int, m: int, T: Optional[int] = None) -> "Config":
        return dataclasses.replace(self, M=M, m=m, T=self.T if T is None else T)


# BASELINE.json configs[0..4]; data_seed = 1000 + config number.
CONFIGS: Dict[str, Config] = {
    "C1": Config("C1", PF_LG, 1, 1, 64, 16, 50, 1001),
    "C2": Config("C2", PF_LG, 8, 8, 256, 4096, 100, 1002),
    "C3": Config("C3", PF_SV, 1, 1, 32, 1 << 19, 200, 1003),
    "C4": Config("C4", PF_LG, 4, 4, 64, 1 << 22, 50, 1004),
    "C5": Config("C5", PF_SV, 1, 1, 64, 1 << 20, 20, 1005),  # M swept in {2..8192}, N = 2^26
}
C5_SWEEP_M = (2, 8, 32, 128, 512, 2048, 8192)
C5_N = 1 << 26


def _orthogonal(rng: np.random.Generator, d: int) -> np.ndarray:
    """Haar orthogonal matrix: QR of a standard normal matrix, sign-fixed by diag(R)
    (reading R12)."""
    z = rng.standard_normal((d, d))
    q, r = np.linalg.qr(z)
    q = q * np.sign(np.diag(r))[None, :]
    return q


def model_params(cfg: Config) -> dict:
    """Model parameters as fp32 arrays (row-major, d x d etc.).

    LG keys: A, LQ (lower Cholesky of Q), H, Rinv, m0, L0 (lower Cholesky of P0),
    and Q, R, P0 (fp64, for the Kalman oracle).  SV keys: phi, sigma, beta, m0, s0.
    """
    f32 = np.float32
    if cfg.kind == PF_SV:
        phi, sigma, beta = 0.98, 0.16, 0.65
        s0 = math.sqrt(sigma * sigma / (1.0 - phi * phi))  # stationary sd (reading R11)
        return dict(kind=PF_SV, d=1, dy=1, phi=f32(phi), sigma=f32(sigma), beta=f32(beta),
                    m0=f32(0.0), s0=f32(s0))
    d = cfg.d
    if cfg.name == "C1":
        A = np.array([[0.9]])
        Q = np.array([[1.0]])
        R = np.array([[0.25]])
    elif cfg.name == "C2":
        rng = np.random.Generator(np.random.PCG64(cfg.data_seed))
        A = 0.95 * _orthogonal(rng, d)
        Q = 0.1 * np.eye(d)
        R = 0.25 * np.eye(d)
    elif cfg.name == "C4":
        A = 0.9 * np.eye(d)
        for i in range(d - 1):  # symmetric tridiagonal coupling (reading R13)
            A[i, i + 1] = 0.05
            A[i + 1, i] = 0.05
        Q = 0.2 * np.eye(d)
        R = 0.2 * np.eye(d)
    else:
        raise ValueError(cfg.name)
    H = np.eye(cfg.dy, d)
    P0 = np.eye(d)
    # Round to fp32 first; Kalman uses the rounded values too, so both filters
    # target the same model.
    A32 = A.astype(f32)
    Q32 = Q.astype(f32)
    R32 = R.astype(f32)
    H32 = H.astype(f32)
    LQ = np.linalg.cholesky(Q32.astype(np.float64)).astype(f32)
    Rinv = np.linalg.inv(R32.astype(np.float64)).astype(f32)
    L0 = np.linalg.cholesky(P0).astype(f32)
    return dict(kind=PF_LG, d=d, dy=cfg.dy, A=A32, LQ=LQ, H=H32, Rinv=Rinv,
                m0=np.zeros(d, f32), L0=L0,
                Q=LQ.astype(np.float64) @ LQ.astype(np.float64).T,
                R=np.linalg.inv(Rinv.astype(np.float64)),
                P0=L0.astype(np.float64) @ L0.astype(np.float64).T)


def simulate(cfg: Config, T: Optional[int] = None, data_seed: Optional[int] = None):
    """Simulate (x_{0:T-1}, y_{0:T-1}) from eq. HMM in fp64.

    Returns (x, y) with x fp64 (T x d) and y fp32 (T x dy).  Deterministic per seed.
    """
    T = cfg.T if T is None else T
    seed = cfg.data_seed if data_seed is None else data_seed
    p = model_params(cfg)
    rng = np.random.Generator(np.random.PCG64(seed))
    if cfg.kind == PF_SV:
        phi, sigma, beta = float(p["phi"]), float(p["sigma"]), float(p["beta"])
        x = np.empty((T, 1))
        y = np.empty((T, 1))
        xv = float(p["m0"]) + float(p["s0"]) * rng.standard_normal()
        for n in range(T):
            if n > 0:
                xv = phi * xv + sigma * rng.standard_normal()
            x[n, 0] = xv
            y[n, 0] = beta * math.exp(xv / 2.0) * rng.standard_normal()
        return x, y.astype(np.float32)
    A = p["A"].astype(np.float64)
    LQ = p["LQ"].astype(np.float64)
    H = p["H"].astype(np.float64)
    LR = np.linalg.cholesky(p["R"])
    d, dy = cfg.d, cfg.dy
    x = np.empty((T, d))
    y = np.empty((T, dy))
    xv = p["m0"].astype(np.float64) + p["L0"].astype(np.float64) @ rng.standard_normal(d)
    for n in range(T):
        if n > 0:
            xv = A @ xv + LQ @ rng.standard_normal(d)
        x[n] = xv
        y[n] = H @ xv + LR @ rng.standard_normal(dy)
    return x, y.astype(np.float32)


def particle_cloud(cfg: Config, N: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """A synthetic resampled particle cloud xhat (N x d, fp32) for single-step
    parity tests: iid N(0, scale^2 * P) with P the stationary (LG: prior) variance,
    plus a handful of exact duplicates, as resampled clouds have."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = model_params(cfg)
    d = 1 if cfg.kind == PF_SV else cfg.d
    sd = float(p["s0"]) * scale if cfg.kind == PF_SV else scale
    if N * d > (1 << 26):  # full-size clouds (C4: 2^30 values): drawn in fp32, scaled in place
        x = rng.standard_normal((N, d), dtype=np.float32)
        x *= np.float32(sd)
    else:
        x = (sd * rng.standard_normal((N, d))).astype(np.float32)
    if N >= 8:  # duplicates: copy a random 1/8 of the entries from random sources
        k = N // 8
        dst = rng.integers(0, N, size=k)
        src = rng.integers(0, N, size=k)
        x[dst] = x[src]
    return np.ascontiguousarray(x)


def observation_for_step(cfg: Config, seed: int, outlier_sigma: float = 0.0) -> np.ndarray:
    """One synthetic observation y (dy, fp32); outlier_sigma > 0 shifts it to
    stress weight degeneracy (SURVEY.md §8(d) "+6 sigma outlier")."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = rng.standard_normal(cfg.dy) * 0.7 + outlier_sigma
    return y.astype(np.float32)
