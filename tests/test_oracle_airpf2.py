"""Pins of the oracle's AIRPF with the fully adapted scheme, AIRPF2 (
orc_step_airpf_adaptive, reading R26):

* theta = 1 with unequal island weights runs every island stage and reproduces the plain
  AIRPF step (orc_step_airpf) bit for bit when nothing is carried;
* theta <= E_0 runs no island stage: the island map is the identity and x_hat is the
  within-island resample in place;
* the island ESS levels equal the paper's ESS formula on the exact
  rational island weights W_check_k = M^-1 sum g over island k (eq. out weight,
  PAPER.md:918-921) and their V_bar levels (oracle/exact.py with M = 1);
* the carried weight of island i is log V_bar_{S*} of its block minus log V_bar_S, the
  exact rational levels; the weighted islands after the stop are unbiased: sum_i
  V_bar_{S*}^i P(island i holds block j) = W_check_j exactly (island kernels K_s, M = 1);
* hand example: island weights (1, eps, 1, eps) -> E_0 = 1/2 + O(eps), one stage for
  theta = 0.9;
* the AIRPF2 filter tracks the exact Kalman means (C1, 5 MC sigma).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact, kalman
from paper_1812_01502_b200 import inputs


def _ess(v):
    n = len(v)
    s1 = sum(v, Fraction(0))
    s2 = sum((x * x for x in v), Fraction(0))
    return (s1 / n) ** 2 / (s2 / n)


def _cloud(cfg_name, N, seed):
    cfg = inputs.CONFIGS[cfg_name]
    return cfg, inputs.model_params(cfg), inputs.particle_cloud(cfg, N, seed)


def test_theta_one_is_plain_airpf(orc):
    cfg, p, x = _cloud("C4", 1 << 12, 3)
    N, M = 1 << 12, 16
    y = inputs.observation_for_step(cfg, 4, outlier_sigma=1.0)
    a = orc.step_airpf(p, N, M, 9, 2, y, x, modified=True)
    b = orc.step_airpf_adaptive(p, N, M, 9, 2, y, x, np.zeros(N), 1.0, modified=True)
    assert b["sstar"] == b["S"]
    for k in ("x", "lw", "a_w", "logW", "src", "logVbar", "Aisl", "xhat", "filter", "predict"):
        assert np.array_equal(a[k], b[k]), k
    assert np.allclose(b["lwc"], 0.0, atol=1e-12)  # V_bar_S over V_bar_S


def test_no_stage_when_ess_is_high(orc):
    cfg, p, x = _cloud("C1", 1024, 5)
    N, M = 1024, 64
    y = inputs.observation_for_step(cfg, 6)
    r = orc.step_airpf_adaptive(p, N, M, 2, 1, y, x, np.zeros(N), 1e-9)
    assert r["sstar"] == 0
    assert np.array_equal(r["Aisl"], np.arange(N // M))
    assert np.array_equal(r["xhat"], r["x"][r["a_w"]])
    lvS = r["logVbar"][-1]
    assert np.allclose(r["lwc"], np.repeat(r["logW"], M) - lvS, rtol=0, atol=1e-12)


@pytest.mark.parametrize("S,M,g", [(2, 2, (2, 1, 1, 4, 3, 1, 1, 2)), (3, 2, (9, 1, 1, 1, 2, 7, 1, 3, 1, 1, 1, 1, 5, 1, 2, 2)),
                                   (2, 4, tuple(range(1, 17)))])
def test_island_ess_and_carry_exact(orc, S, M, g, monkeypatch):
    """Drive the step's weights through the carried weight (x = 0, Rinv = 0: log g = 0), so
    lw = log g_i exactly; compare the island ESS levels and the carried weights with the
    exact rational island levels."""
    m, N = 2 ** S, M * 2 ** S
    cfg = inputs.CONFIGS["C4"]
    p = dict(inputs.model_params(cfg))
    p["Rinv"] = np.zeros_like(p["Rinv"])
    x = np.zeros((N, 4), np.float32)
    lwc = np.log(np.array(g, np.float64))
    W = [Fraction(sum(g[k * M:(k + 1) * M]), M) for k in range(m)]  # eq. out weight
    Vb = exact.V_levels(S, 1, W)
    want_ess = [float(_ess(Vb[s])) for s in range(S + 1)]
    for theta in sorted(set([0.0] + [min(1.0, e + 1e-9) for e in want_ess])):
        r = orc.step_airpf_adaptive(p, N, M, 11, 0, np.zeros(4, np.float32), x, lwc, theta)
        assert np.allclose(r["ess"], want_ess, rtol=1e-12, atol=0), (r["ess"], want_ess)
        ss = r["sstar"]
        assert ss == next((s for s in range(S) if want_ess[s] >= theta), S)
        lvS = math.log(Vb[S][0])
        for i in range(m):
            want = math.log(W[i] if ss == 0 else Vb[ss][i]) - lvS
            assert np.allclose(r["lwc"][i * M:(i + 1) * M], want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("S,W", [(2, (3, 1, 2, 5)), (3, (1, 2, 3, 4, 5, 6, 7, 8))])
def test_carried_islands_unbiased(S, W):
    """sum_i V_bar_s^i P(island i holds block j after s stages) = W_j for every s (the
    island form of the partial-product identity behind reading R18; Alg. 6 island law)."""
    Wf = [Fraction(w) for w in W]
    Ks = exact.K_matrices(S, 1, Wf)
    Vb = exact.V_levels(S, 1, Wf)
    P = None
    for s in range(1, S + 1):
        P = Ks[s - 1] if P is None else exact.matmul(Ks[s - 1], P)
        m = len(W)
        for j in range(m):
            assert sum(Vb[s][i] * P[i][j] for i in range(m)) == Wf[j]


def test_hand_stop_rule(orc):
    """Islands (1, eps, 1, eps): E_0 = (2 + 2 eps)^2 / (4 (2 + 2 eps^2)) ~ 1/2, level 1 pairs
    (1, eps) -> equal block weights -> E_1 = 1: theta = 0.9 stops after one stage."""
    M, S = 2, 2
    N = M * 2 ** S
    eps = 1e-3
    g = np.array([1, 1, eps, eps, 1, 1, eps, eps], np.float64)
    cfg = inputs.CONFIGS["C4"]
    p = dict(inputs.model_params(cfg))
    p["Rinv"] = np.zeros_like(p["Rinv"])
    r = orc.step_airpf_adaptive(p, N, M, 1, 0, np.zeros(4, np.float32), np.zeros((N, 4), np.float32),
                                np.log(g), 0.9)
    assert abs(r["ess"][0] - (2 + 2 * eps) ** 2 / (4 * (2 + 2 * eps ** 2))) < 1e-12
    assert abs(r["ess"][1] - 1.0) < 1e-12
    assert r["sstar"] == 1


def test_airpf2_filter_vs_kalman(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=12)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J = 24
    runs, stages = [], []
    for j in range(J):
        mu, st = orc.run_filter_airpf_adaptive(p, 64, 16, 900 + j, ys, theta=0.5)
        runs.append(mu[:, 0])
        stages.append(st)
    runs = np.array(runs)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)
    assert 0 < np.mean(stages) < 4  # the controller actually stops early on some steps
