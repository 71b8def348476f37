"""Pins of the oracle's fully adapted augmented resampling (AIRPF2,
PAPER.md:1279): the ESS of the stage weights, the stop rule, the carried weights.

* ESS levels (oracle/pf_oracle.c orc_ess_levels) against the ESS of the exact rational
  stage weights V_s = A_s V_{s-1} expanded to all N particles (oracle/exact.py), i.e. the
  paper's formula E = (N^-1 sum w)^2 / (N^-1 sum w^2) evaluated on V_s;
  closed forms (equal weights -> 1, one live particle -> 1/N, two-valued weights);
  E_S = 1 (Lemma facts_about_Vs (c)); E_s non-decreasing in s (V_s = A_s V_{s-1} is an
  average: sum V_s = sum V_{s-1}, sum V_s^2 <= sum V_{s-1}^2).
* Stop rule (strict, reading R17): hand-evaluated example m = 4, M = 1, weights
  (1, eps, 1, eps), theta = 0.9 -> exactly one stage; theta = 1 -> all S stages unless the
  weights are equal; equal weights -> no stage.
* Carried weights (reading R18): sum_i V_s^i P(xi_s^i = xi_0^j) = g_j exactly in rationals
  for every s (the weighted sample after an early stop is unbiased, the partial-product
  form of Prop. 1), and empirically on the oracle's partial resampling.
* Consistency: theta = 1 reproduces the plain step (same draws, zero carry); the adaptive
  filter tracks the exact Kalman means (C1).
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact, kalman
from paper_1812_01502_b200 import inputs


def _ess_exact(v):
    """(N^-1 sum v)^2 / (N^-1 sum v^2) in rationals."""
    n = len(v)
    s1 = sum(v, Fraction(0))
    s2 = sum((x * x for x in v), Fraction(0))
    return (s1 / n) ** 2 / (s2 / n)


CASES = [(1, 1, (3, 1)), (2, 1, (1, 3, 2, 5)), (2, 2, (2, 1, 1, 4, 3, 1, 1, 2)), (3, 1, (1, 2, 3, 4, 5, 6, 7, 8)),
         (3, 2, (9, 1, 1, 1, 2, 7, 1, 3, 1, 1, 1, 1, 5, 1, 2, 2)), (2, 4, tuple(range(1, 17)))]


@pytest.mark.parametrize("S,M,g", CASES)
def test_ess_levels_vs_exact(orc, S, M, g):
    gF = [Fraction(v) for v in g]
    V = exact.V_levels(S, M, gF)
    lw = np.log(np.array(g, np.float64))
    r = orc.augmented_resample(lw, M, 1, 1, tables=False)
    ess = orc.ess_levels(lw, M, r["logV"])
    want = np.array([float(_ess_exact(V[s])) for s in range(S + 1)])
    assert np.allclose(ess, want, rtol=1e-13, atol=0), (ess, want)
    assert ess[-1] == pytest.approx(1.0, abs=1e-14)


def test_ess_closed_forms(orc):
    M, m = 4, 8
    N = M * m
    S = 3
    # equal weights: every level 1
    lw = np.full(N, -2.5)
    r = orc.augmented_resample(lw, M, 1, 1, tables=False)
    assert np.allclose(orc.ess_levels(lw, M, r["logV"]), 1.0, atol=1e-15)
    # one live particle: E_0 = 1/N; level s: one live block of 2^s groups out of m/2^s
    lw = np.full(N, -np.inf)
    lw[5] = 0.0
    r = orc.augmented_resample(lw, M, 1, 1, tables=False)
    ess = orc.ess_levels(lw, M, r["logV"])
    assert ess[0] == pytest.approx(1.0 / N, rel=1e-14)
    for s in range(1, S + 1):
        assert ess[s] == pytest.approx(2.0 ** s / m, rel=1e-14)
    # two-valued weights (a on the first k particles, b elsewhere)
    a, b, k = 3.0, 0.5, 12
    w = np.where(np.arange(N) < k, a, b)
    r = orc.augmented_resample(np.log(w), M, 1, 1, tables=False)
    e0 = (k * a + (N - k) * b) ** 2 / (N * (k * a * a + (N - k) * b * b))
    assert orc.ess_levels(np.log(w), M, r["logV"])[0] == pytest.approx(e0, rel=1e-14)


def test_ess_monotone_in_stage(orc):
    rng = np.random.default_rng(7)
    for M, m in [(1, 64), (4, 32), (16, 16)]:
        for _ in range(5):
            lw = rng.normal(scale=2.0, size=M * m)
            r = orc.augmented_resample(lw, M, 1, 1, tables=False)
            ess = orc.ess_levels(lw, M, r["logV"])
            assert np.all(np.diff(ess) >= -1e-14), ess
            assert np.all((ess >= 1.0 / (M * m) - 1e-15) & (ess <= 1.0 + 1e-15))


def test_stop_rule_hand_example(orc):
    # m = 4, M = 1, weights (1, eps, 1, eps): stage 1 pairs (0,1), (2,3) -> V_1 constant
    eps = 1e-6
    lw = np.log(np.array([1.0, eps, 1.0, eps]))
    r = orc.augmented_resample(lw, 1, 1, 1, tables=False)
    ess = orc.ess_levels(lw, 1, r["logV"])
    assert ess[0] == pytest.approx((1 + eps) ** 2 / (2 * (1 + eps * eps)), rel=1e-12)  # ~ 1/2
    assert ess[1] == pytest.approx(1.0, abs=1e-15)
    assert orc.stages_to_run(ess, 0.9) == 1
    assert orc.stages_to_run(ess, 0.4) == 0
    # same weights paired the other way: stage 1 cannot mix, stage 2 does
    lw2 = np.log(np.array([1.0, 1.0, eps, eps]))
    r2 = orc.augmented_resample(lw2, 1, 1, 1, tables=False)
    assert orc.stages_to_run(orc.ess_levels(lw2, 1, r2["logV"]), 0.9) == 2


def test_stop_rule_boundaries(orc):
    rng = np.random.default_rng(3)
    lw = rng.normal(size=64)
    r = orc.augmented_resample(lw, 4, 1, 1, tables=False)
    ess = orc.ess_levels(lw, 4, r["logV"])
    assert orc.stages_to_run(ess, 1.0) == 4  # strict: E < 1 at every s < S
    assert orc.stages_to_run(ess, 1e-9) == 0
    flat = np.zeros(64)
    rf = orc.augmented_resample(flat, 4, 1, 1, tables=False)
    assert orc.stages_to_run(orc.ess_levels(flat, 4, rf["logV"]), 1.0) == 0


@pytest.mark.parametrize("S,M,g", CASES[:5])
def test_carried_weights_unbiased_exact(S, M, g):
    """sum_i V_s^i (K_s ... K_1)[i, j] = g_j for every s (rationals)."""
    gF = [Fraction(v) for v in g]
    V = exact.V_levels(S, M, gF)
    Ks = exact.K_matrices(S, M, gF)
    N = len(gF)
    P = None
    for s in range(1, S + 1):
        P = Ks[s - 1] if P is None else exact.matmul(Ks[s - 1], P)
        for j in range(N):
            assert sum((V[s][i] * P[i][j] for i in range(N)), Fraction(0)) == gF[j]


def test_carried_weights_unbiased_empirical(orc):
    """Weighted estimate after an early stop at s: E[sum_i V_s^i phi(xi_s^i)] / sum V_s =
    sum g phi / sum g (phi = indicator of source j), oracle draws."""
    g = np.array([5.0, 1.0, 1.0, 2.0, 3.0, 1.0, 4.0, 2.0, 1.0, 1.0, 6.0, 1.0, 2.0, 2.0, 1.0, 3.0])
    M, S = 2, 3
    lw = np.log(g)
    reps = 4000
    for s in (1, 2):
        acc = np.zeros(len(g))
        for rep in range(reps):
            r = orc.augmented_resample_partial(lw, M, 11, rep + 1, s)
            m = len(g) // M
            lvs = r["logV"][orc.level_offset(m, s): orc.level_offset(m, s) + (m >> s)]
            Vs = np.exp(lvs[(np.arange(len(g)) // M) >> s])
            np.add.at(acc, r["A"], Vs)
        est = acc / reps / g.sum()
        want = g / g.sum()
        se = np.sqrt(want * (1 - want) * 4 / reps)  # generous (weights <= 6 / mean)
        assert np.all(np.abs(est - want) < 5 * se + 1e-3), (s, est - want)


def test_theta_one_equals_plain_step(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    N, M = 256, 16
    x = inputs.particle_cloud(cfg, N, 9)
    y = np.array([0.7], np.float32)
    a = orc.step_adaptive(p, N, M, 5, 3, y, x, np.zeros(N), 1.0)
    b = orc.step(p, N, M, 5, 3, y, x)
    assert a["sstar"] == a["S"]
    assert np.array_equal(a["A"], b["A"]) and np.array_equal(a["xhat"], b["xhat"])
    assert np.all(a["lwc"] == 0.0)
    assert np.allclose(a["filter"], b["filter"], rtol=1e-14, atol=0)


def test_adaptive_filter_vs_kalman(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, M, m = 24, 64, 16
    runs, stages = [], []
    for j in range(J):
        mean, st = orc.run_filter_adaptive(p, M, m, seed=300 + j, ys=ys, theta=0.5)
        runs.append(mean[:, 0])
        stages.append(st)
    runs = np.array(runs)
    stages = np.array(stages)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)
    # the controller really adapts: some steps stop early, some run every stage
    assert stages.min() < 4 and stages.max() >= 1
