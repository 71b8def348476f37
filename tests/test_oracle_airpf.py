"""Pins of the oracle's AIRPF (Alg. 4): within-island resampling
(Alg. 5) and augmented island resampling (Alg. 6, PAPER.md:963-987;
modified form Alg. 7).

* Alg. 5: every draw stays in its island and follows g_j / sum_island g (chi-square
  against the exact categorical); W_out = the island mean of g (eq. out weight); the
  SPEC worked example m = 2, M = 2, potentials (3, 1, 1, 1).
* Alg. 6: the island levels equal V_bar_s = A_bar_s V_bar_{s-1} in rationals
  (oracle/exact.py with M = 1) and coincide with the particle-level V levels of Alg. 3
  (both are means of g over blocks of 2^s islands); per-stage side law
  V_bar_L / (V_bar_L + V_bar_R) and the composed island law (K_S..K_1 with M = 1) by
  chi-square; island unbiasedness sum_i P(A(i) = j) = m W_j / sum W exactly (the
  Proposition for Alg. 6); SPEC example m = 2, V_bar = (3, 1).
* Alg. 7: a pure exchange never survives, and the law of the multiset of blocks a pair
  holds is that of Alg. 6 (exact enumeration of the four joint outcomes).
* AIRPF filter means vs the exact Kalman means (C1), plain and modified.
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from oracle import exact, kalman
from paper_1812_01502_b200 import inputs


def _chi2_p(counts, probs):
    probs = np.asarray(probs, np.float64)
    keep = probs > 0
    assert counts[~keep].sum() == 0, "draw outside the support"
    if keep.sum() <= 1:
        return 1.0
    e = probs[keep] * counts.sum()
    return stats.chi2.sf(((counts[keep] - e) ** 2 / e).sum(), keep.sum() - 1)


def test_within_island_law(orc):
    g = np.array([3.0, 1.0, 1.0, 1.0, 0.5, 2.0, 4.0, 1.5, 1, 1, 1, 1, 9, 1, 1, 1])
    M = 4
    lw = np.log(g)
    reps = 3000
    counts = np.zeros((len(g), len(g)))
    for r in range(reps):
        out = orc.within_island(lw, M, 7, r + 1)
        np.add.at(counts, (np.arange(len(g)), out["a_w"]), 1)
    for i in range(len(g)):
        k = i // M
        probs = np.zeros(len(g))
        probs[k * M:(k + 1) * M] = g[k * M:(k + 1) * M] / g[k * M:(k + 1) * M].sum()
        assert _chi2_p(counts[i], probs) > 1e-4, i
    out = orc.within_island(lw, M, 7, 1)
    assert np.allclose(np.exp(out["logW"]), g.reshape(-1, M).mean(axis=1), rtol=1e-14)


def test_within_island_spec_example(orc):
    # m = 2, M = 2, potentials (3, 1, 1, 1): island 1 draws source 0 w.p. 3/4; W_out = (2, 2, 1, 1)
    lw = np.log(np.array([3.0, 1.0, 1.0, 1.0]))
    out = orc.within_island(lw, 2, 1, 1)
    assert np.allclose(np.exp(out["logW"]), [2.0, 1.0], rtol=1e-15)
    hits = sum(int(orc.within_island(lw, 2, 1, r)["a_w"][0] == 0) for r in range(1, 8001))
    assert abs(hits / 8000 - 0.75) < 4 * np.sqrt(0.75 * 0.25 / 8000)


@pytest.mark.parametrize("W", [(1, 3, 2, 5), (2, 1, 1, 4, 3, 1, 1, 2), (5, 1, 1, 1, 1, 1, 1, 9)])
def test_island_levels_exact_and_equal_to_alg3(orc, W):
    m = len(W)
    S = int(np.log2(m))
    logW = np.log(np.array(W, np.float64))
    out = orc.island_resample(logW, 3, 1, modified=False)
    V = exact.V_levels(S, 1, [Fraction(w) for w in W])
    for s in range(1, S + 1):
        lv = out["logVbar"][orc.level_offset(m, s): orc.level_offset(m, s) + (m >> s)]
        want = np.array([float(V[s][b << s]) for b in range(m >> s)])
        assert np.allclose(np.exp(lv), want, rtol=1e-13)
    # the same table as Alg. 3's V levels for particle weights whose island means are W
    M = 4
    g = np.repeat(np.array(W, np.float64), M) * np.tile([0.5, 1.5, 1.0, 1.0], m)
    r3 = orc.augmented_resample(np.log(g), M, 1, 1, tables=False)
    assert np.allclose(r3["logV"], out["logVbar"], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("W", [(3, 1), (1, 3, 2, 5), (2, 1, 1, 4, 3, 1, 1, 2)])
def test_island_stage_and_composed_law_plain(orc, W):
    m = len(W)
    S = int(np.log2(m))
    WF = [Fraction(w) for w in W]
    logW = np.log(np.array(W, np.float64))
    reps = 6000
    src = np.zeros((reps, S, m), np.int64)
    A = np.zeros((reps, m), np.int64)
    for r in range(reps):
        out = orc.island_resample(logW, 11, r + 1, modified=False)
        src[r] = out["src"]
        A[r] = out["Aisl"]
    Ks = exact.K_matrices(S, 1, WF)
    for s in range(S):
        for i in range(m):
            c = np.bincount(src[:, s, i], minlength=m)
            assert _chi2_p(c, [float(p) for p in Ks[s][i]]) > 1e-4, (s, i)
    P = exact.composed_marginal(S, 1, WF)
    for i in range(m):
        assert _chi2_p(np.bincount(A[:, i], minlength=m), [float(p) for p in P[i]]) > 1e-4, i
    # island unbiasedness, exactly: sum_i P(A(i) = j) = m W_j / sum W
    tot = sum(WF)
    for j in range(m):
        assert sum((P[i][j] for i in range(m)), Fraction(0)) == m * WF[j] / tot


def test_island_spec_example(orc):
    # m = 2, V_bar = (3, 1), plain: P(island 2 ends holding island 1's block) = 3/4
    logW = np.log(np.array([3.0, 1.0]))
    reps = 8000
    hits = sum(int(orc.island_resample(logW, 2, r, modified=False)["Aisl"][1] == 0) for r in range(1, reps + 1))
    assert abs(hits / reps - 0.75) < 4 * np.sqrt(0.75 * 0.25 / reps)


def test_modified_swap_avoidance(orc):
    """Alg. 7: no pure exchange survives; the multiset of blocks per pair keeps Alg. 6's law."""
    logW = np.log(np.array([1.0, 1.0]))  # p = 1/2: each joint outcome has probability 1/4
    reps = 12000
    plain = {"LR": 0, "LL": 0, "RR": 0, "swap": 0}
    mod = {"LR": 0, "LL": 0, "RR": 0, "swap": 0}
    for r in range(1, reps + 1):
        for tab, modified in ((plain, False), (mod, True)):
            a = orc.island_resample(logW, 5, r, modified=modified)["Aisl"]
            key = {(0, 1): "LR", (0, 0): "LL", (1, 1): "RR", (1, 0): "swap"}[(int(a[0]), int(a[1]))]
            tab[key] += 1
    assert mod["swap"] == 0
    # same draws: every plain swap became keep-keep, everything else is unchanged
    assert mod["LR"] == plain["LR"] + plain["swap"] and mod["LL"] == plain["LL"] and mod["RR"] == plain["RR"]
    # exact multiset law {L,R}: 1/2, {L,L}: 1/4, {R,R}: 1/4
    c = np.array([mod["LR"], mod["LL"], mod["RR"]])
    assert _chi2_p(c, [0.5, 0.25, 0.25]) > 1e-4


@pytest.mark.parametrize("modified", [False, True])
def test_airpf_filter_vs_kalman(orc, modified):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, M, m = 24, 64, 16
    runs = np.array([orc.run_filter_airpf(p, M, m, 900 + j, ys, modified=modified)[:, 0] for j in range(J)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)


def test_airpf_xhat_is_block_gather(orc):
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, M = 1024, 16
    x = inputs.particle_cloud(cfg, N, 4)
    r = orc.step_airpf(p, N, M, 3, 2, np.zeros(4, np.float32), x)
    src = (r["Aisl"][:, None] * M + np.arange(M)[None, :]).ravel()
    assert np.array_equal(r["xhat"], r["x"][r["a_w"][src]])
    # every block comes whole from one island and within-island ancestors stay in the island
    assert np.all(r["a_w"] // M == np.arange(N) // M)
