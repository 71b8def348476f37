"""Pins of the oracle's model layer (eq. HMM) and the Kalman oracle.

* log-potentials equal the closed-form Gaussian log-densities (scipy) up to the
  dropped constant (reading R9): differences between particles match;
* mutation / init moments match A xhat, Q and m0, P0 (closed form);
* Kalman: SPEC hand values (tests/golden/spec_kalman_hand.txt), dense == scalar,
  Riccati fixed point, zero observations -> zero means.
"""
import os

import numpy as np
import pytest
from scipy import stats

from oracle import kalman
from paper_1812_01502_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_lg_logweight_is_gaussian_logpdf(orc, name):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    rng = np.random.default_rng(1)
    x = rng.normal(size=(64, cfg.d))
    y = rng.normal(size=cfg.dy).astype(np.float32)
    lw = orc.logweight(p, y, x)
    H = p["H"].astype(np.float64)
    R = np.linalg.inv(p["Rinv"].astype(np.float64))
    ref = np.array([stats.multivariate_normal.logpdf(y.astype(np.float64), H @ xi, R) for xi in x])
    assert np.allclose(lw - lw[0], ref - ref[0], rtol=0, atol=1e-9)


def test_sv_logweight_is_gaussian_logpdf(orc):
    cfg = inputs.CONFIGS["C3"]
    p = inputs.model_params(cfg)
    x = np.linspace(-3, 3, 41)[:, None]
    y = np.array([0.7], np.float32)
    lw = orc.logweight(p, y, x)
    beta = float(p["beta"])
    ref = stats.norm.logpdf(float(y[0]), 0.0, beta * np.exp(x[:, 0] / 2.0))
    assert np.allclose(lw - lw[0], ref - ref[0], rtol=0, atol=1e-9)


def test_logweight_nonfinite_is_minus_inf(orc):
    p = inputs.model_params(inputs.CONFIGS["C1"])
    lw = orc.logweight(p, np.array([0.5], np.float32), np.array([[np.nan], [np.inf], [0.0]]))
    assert lw[0] == -np.inf and lw[1] == -np.inf and np.isfinite(lw[2])


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_mutation_moments(orc, name):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    N = 1 << 15
    c = np.linspace(-1, 1, cfg.d)
    xhat = np.tile(c, (N, 1))
    x = orc.mutate(p, 5, 7, xhat)
    mean = x.mean(axis=0)
    cov = np.cov(x.T)
    want_mean = p["A"].astype(np.float64) @ c
    assert np.all(np.abs(mean - want_mean) < 5 * np.sqrt(np.diag(p["Q"]) / N))
    assert np.allclose(cov, p["Q"], atol=6 * 0.2 * np.sqrt(2.0 / N) + 1e-3)


def test_sv_mutation_and_init(orc):
    cfg = inputs.CONFIGS["C3"]
    p = inputs.model_params(cfg)
    N = 1 << 15
    x = orc.mutate(p, 5, 7, np.full((N, 1), 0.5))
    assert abs(x.mean() - 0.98 * 0.5) < 5 * 0.16 / np.sqrt(N)
    assert abs(x.std() - 0.16) < 0.01
    x0 = orc.init(p, N, 3)
    assert abs(x0.mean()) < 5 * float(p["s0"]) / np.sqrt(N)
    assert abs(x0.std() / float(p["s0"]) - 1) < 0.02


def test_lg_init_moments(orc):
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N = 1 << 15
    x0 = orc.init(p, N, 3)
    assert np.all(np.abs(x0.mean(axis=0)) < 5 / np.sqrt(N))
    assert np.allclose(np.cov(x0.T), np.eye(4), atol=0.04)


def test_kalman_hand_values():
    rows = []
    with open(os.path.join(GOLDEN, "spec_kalman_hand.txt")) as f:
        for ln in f:
            if ln.strip() and not ln.startswith("#"):
                rows.append([float(v) for v in ln.split()])
    ys = np.array([[r[1]] for r in rows])
    means, covs = kalman.kalman_filter([[1.0]], [[1.0]], [[1.0]], [[0.25]], [0.0], [[1.0]], ys)
    for n, r in enumerate(rows):
        assert abs(means[n, 0] - r[2]) < 1e-9
        assert abs(covs[n, 0, 0] - r[3]) < 1e-9


def test_kalman_dense_equals_scalar_and_fixed_point():
    rng = np.random.default_rng(0)
    ys = rng.normal(size=(100, 1))
    m_d, P_d = kalman.kalman_filter([[0.9]], [[1.0]], [[1.0]], [[0.25]], [0.0], [[1.0]], ys)
    m_s, p_s = kalman.kalman_scalar(0.9, 1.0, 0.25, 0.0, 1.0, ys[:, 0])
    assert np.allclose(m_d[:, 0], m_s, atol=1e-12)
    assert np.allclose(P_d[:, 0, 0], p_s, atol=1e-12)
    # steady state of the random walk (a=1): v* = r (v*+q)/(v*+q+r)
    _, p_rw = kalman.kalman_scalar(1.0, 1.0, 0.25, 0.0, 1.0, ys[:, 0])
    v = p_rw[-1]
    assert abs(v - 0.25 * (v + 1.0) / (v + 1.25)) < 1e-10
    zero_means, _ = kalman.kalman_filter(np.eye(3) * 0.9, np.eye(3), np.eye(3), np.eye(3) * 0.2,
                                         np.zeros(3), np.eye(3), np.zeros((10, 3)))
    assert np.all(zero_means == 0.0)


def test_paper_raw_observation_mse_closed_form():
    """raw-observation MSE 2396 for the d=7 random walk (q=1, r=1/4,
    n_max=8000).  Closed form d*n_max*r^2/(P^- + r) with the steady-state Riccati
    solution; the paper's number must lie within 2 sd of it."""
    _, p = kalman.kalman_scalar(1.0, 1.0, 0.25, 0.0, 1.0, np.zeros(200))
    Pminus = p[-1] + 1.0
    per = 0.25 ** 2 / (Pminus + 0.25)
    expected = 7 * 8000 * per
    # (y - xbar) is Gaussian with variance per => sum of squares has sd per*sqrt(2*d*n_max)
    sd = per * np.sqrt(2 * 7 * 8000)
    assert abs(2396 - expected) < 2 * sd


def test_init_rows_is_init_restricted(orc):
    """orc_init_rows (full-size sampled parity) evaluates exactly orc_init's rows."""
    for name in ("C4", "C3", "C2"):
        p = inputs.model_params(inputs.CONFIGS[name])
        full = orc.init(p, 256, 17)
        rows = np.array([0, 1, 5, 128, 255])
        assert np.array_equal(orc.init_rows(p, 17, rows), full[rows])
