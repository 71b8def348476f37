"""Statistical pins of the whole oracle filter (Alg. 1 deploying Alg. 3).

* Filter means of the oracle BPF-with-augmented-resampling agree with the exact Kalman
  posterior means within 5 Monte Carlo standard errors, C1 model.
* Theorem 1: at fixed m the error decays as M^{-1/2}
  (log-log slope -0.5 +- 0.12), and at fixed M the RMSE scaled by sqrt(m / log2 m)
  stays bounded (the bound is an upper bound only).
"""
import numpy as np
import pytest

from oracle import kalman
from paper_1812_01502_b200 import inputs


def _c1(T=20):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=T)
    km, kc = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    return cfg, p, ys, km, kc


def test_filter_means_vs_kalman(orc):
    cfg, p, ys, km, kc = _c1(T=20)
    J = 24
    M, m = 64, 16
    runs = np.array([orc.run_filter(p, M, m, seed=100 + j, ys=ys)[:, 0] for j in range(J)])
    mean = runs.mean(axis=0)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    # 5 MC standard errors, floored at the fp32-state rounding level
    assert np.all(np.abs(mean - km[:, 0]) < 5 * se + 1e-6), (mean - km[:, 0]) / se


def _rmse_at_end(orc, p, ys, km, M, m, J, seed0):
    errs = []
    for j in range(J):
        est = orc.run_filter(p, M, m, seed=seed0 + j, ys=ys)
        errs.append(est[-1, 0] - km[-1, 0])
    return float(np.sqrt(np.mean(np.square(errs))))


@pytest.mark.slow
def test_theorem1_rate_fixed_m(orc):
    cfg, p, ys, km, _ = _c1(T=8)
    m = 16
    Ms = [8, 32, 128, 512]
    rmse = [_rmse_at_end(orc, p, ys, km, M, m, J=150, seed0=1000 * M) for M in Ms]
    slope = np.polyfit(np.log(Ms), np.log(rmse), 1)[0]
    assert -0.62 < slope < -0.38, (slope, rmse)


@pytest.mark.slow
def test_theorem1_fixed_M_bounded(orc):
    cfg, p, ys, km, _ = _c1(T=8)
    M = 16
    ms = [2, 8, 32, 128]
    scaled = []
    for m in ms:
        r = _rmse_at_end(orc, p, ys, km, M, m, J=120, seed0=7000 * m)
        scaled.append(r * np.sqrt(m / np.log2(m)))
    # RMSE <= C sqrt(S/N): the scaled error must not grow with m (within MC noise)
    assert max(scaled) < 1.5 * scaled[0] + 1e-9, scaled
    # and the raw RMSE decreases with m
    assert scaled[-1] / np.sqrt(ms[-1] / np.log2(ms[-1])) < scaled[0] / np.sqrt(ms[0] / np.log2(ms[0]))
