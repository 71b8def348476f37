"""Pins of stage rotation (start the next augmented resampling at the stage
after the last one executed), realised as a relabelling of the groups (R23).

* Law: running the standard stages 1..t on the layout g' = rotr_S(g, rho) is, in natural
  coordinates, the paper's rotated order sigma(1..t) = rho+1, ..., rho+t (mod S): the
  oracle's composed ancestors, mapped back to natural indices, follow the exact product
  K_sigma(t) ... K_sigma(1) built from A_sigma(u) and V_u = A_sigma(u) V_{u-1} in rationals
  (chi-square); the ESS levels equal the exact ESS of those V_u.
* theta = 1 (all S stages): the relabelling is the identity and the step is the plain one.
* The rotated fully adapted filter tracks the Kalman means (C1).
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from oracle import exact, kalman
from paper_1812_01502_b200 import inputs


def rotl(g, k, S):
    k %= S
    return ((g << k) | (g >> (S - k))) & ((1 << S) - 1) if k else g


def rotr(g, k, S):
    return rotl(g, (S - k % S) % S, S)


@pytest.mark.parametrize("S,M,rho,t,g", [(2, 2, 1, 1, (1, 3, 2, 1, 1, 1, 4, 2)),
                                         (3, 1, 1, 2, (1, 2, 3, 4, 5, 6, 7, 8)),
                                         (3, 1, 2, 2, (5, 1, 1, 2, 1, 3, 1, 1)),
                                         (3, 2, 2, 3, tuple(range(1, 17)))])
def test_relabelled_schedule_is_the_rotated_order(orc, S, M, rho, t, g):
    m, N = 1 << S, M << S
    gF = [Fraction(v) for v in g]
    # exact law of the rotated order in natural coordinates
    V = [gF]
    P = None
    for u in range(1, t + 1):
        s_nat = (rho + u - 1) % S + 1
        A = exact.A_matrix(S, M, s_nat)
        Vu = [sum((A[i][j] * V[-1][j] for j in range(N)), Fraction(0)) for i in range(N)]
        K = [[A[i][j] * V[-1][j] / Vu[i] for j in range(N)] for i in range(N)]
        P = K if P is None else exact.matmul(K, P)
        V.append(Vu)
    # natural index of the layout position p' = (g', j): (rotl(g', rho), j)
    nat = np.array([rotl(p // M, rho, S) * M + p % M for p in range(N)])
    lw_layout = np.log(np.array([float(gF[nat[p]]) for p in range(N)]))
    reps = 5000
    counts = np.zeros((N, N))
    for r in range(reps):
        out = orc.augmented_resample_partial(lw_layout, M, 3, r + 1, t)
        counts[nat, nat[out["A"]]] += 1
    for i in range(N):
        probs = np.array([float(p) for p in P[i]])
        keep = probs > 0
        assert counts[i][~keep].sum() == 0
        e = probs[keep] * reps
        if keep.sum() > 1:
            assert stats.chi2.sf(((counts[i][keep] - e) ** 2 / e).sum(), keep.sum() - 1) > 1e-4, i
    # ESS levels of the relabelled run = exact ESS of the rotated-order V_u
    out = orc.augmented_resample_partial(lw_layout, M, 3, 1, t)
    ess = orc.ess_levels(lw_layout, M, out["logV"])
    for u in range(t + 1):
        s1 = sum(V[u], Fraction(0)) / N
        s2 = sum((v * v for v in V[u]), Fraction(0)) / N
        assert ess[u] == pytest.approx(float(s1 * s1 / s2), rel=1e-12)


def test_rotation_with_all_stages_is_the_plain_step(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    N, M = 256, 16
    x = inputs.particle_cloud(cfg, N, 2)
    y = np.array([0.4], np.float32)
    a = orc.step_adaptive(p, N, M, 5, 2, y, x, np.zeros(N), 1.0, rotate=True)
    b = orc.step_adaptive(p, N, M, 5, 2, y, x, np.zeros(N), 1.0, rotate=False)
    assert a["sstar"] == a["S"]
    assert np.array_equal(a["xhat"], b["xhat"]) and np.array_equal(a["lwc"], b["lwc"])


def test_rotation_moves_blocks_by_the_stages_run(orc):
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, M = 1024, 16
    S = 6
    x = inputs.particle_cloud(cfg, N, 3)
    y = inputs.observation_for_step(cfg, 5, outlier_sigma=3.0)
    e = orc.step_adaptive(p, N, M, 9, 1, y, x, np.zeros(N), 1.0)["ess"]
    theta = 0.5 * (e[1] + e[2])  # S* = 2
    r0 = orc.step_adaptive(p, N, M, 9, 1, y, x, np.zeros(N), theta, rotate=False)
    r1 = orc.step_adaptive(p, N, M, 9, 1, y, x, np.zeros(N), theta, rotate=True)
    ss = r1["sstar"]
    assert ss == r0["sstar"] and 1 <= ss < S
    g = np.arange(N) // M
    j = np.arange(N) % M
    dst = np.array([rotr(int(gg), ss, S) for gg in g]) * M + j
    assert np.array_equal(r1["xhat"][dst], r0["xhat"]) and np.array_equal(r1["lwc"][dst], r0["lwc"])


def test_rotated_adaptive_filter_vs_kalman(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, M, m = 24, 64, 16
    runs = np.array([orc.run_filter_adaptive(p, M, m, 1500 + j, ys, 0.5, rotate=True)[0][:, 0] for j in range(J)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)
