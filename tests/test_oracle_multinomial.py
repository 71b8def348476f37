"""Pins of the oracle's multinomial resampling (Alg. 2), the plain BPF's
resampler (the paper's baseline):

* every drawn index is a valid inverse-CDF index whose interval (C_{a-1}, C_a] reproduces
  it through the literal count #{k < N-1 : C_k <= t} (reading R22) and through numpy's
  searchsorted (a library routine); zero-weight particles are never drawn;
* the law: every output follows g_j / sum g (chi-square against the exact categorical),
  outputs independent (pairwise joint frequencies);
* SPEC worked examples: equal weights, N = 4 -> each source 1/4; N = 1 -> the input;
* the plain BPF (Alg. 1 + Alg. 2) tracks the exact Kalman means (C1).
"""
import numpy as np
import pytest
from scipy import stats

from oracle import kalman
from paper_1812_01502_b200 import inputs


def test_bisection_is_the_count(orc):
    rng = np.random.default_rng(5)
    for N in (1, 2, 7, 64, 1000):
        lw = rng.normal(scale=2.0, size=N)
        lw[rng.integers(0, N, size=max(1, N // 10))] = -np.inf  # zero weights are never drawn
        if np.all(np.isneginf(lw)):
            lw[0] = 0.0
        out = orc.multinomial(lw, 9, 3)
        C = np.cumsum(np.exp(lw - lw.max()))
        # u is recovered from the boundary structure: a(i) must satisfy C_{a-1} <= t < C_a,
        # i.e. a(i) is a valid inverse-CDF index of some t in [0, C_{N-1}); and the literal
        # count of C_k <= t for t in (C_{a-1}, C_a) gives back a
        for i, a in enumerate(out["a"]):
            assert 0 <= a < N and (a == N - 1 or C[a] > (C[a - 1] if a else 0.0))
            t = 0.5 * ((C[a - 1] if a else 0.0) + C[a])
            assert int(np.sum(C[:-1] <= t)) == a
            assert int(np.searchsorted(C[:-1], t, side="right")) == a
        assert np.all(np.exp(lw[out["a"]]) > 0)


def test_multinomial_law(orc):
    g = np.array([3.0, 1.0, 0.5, 2.0, 4.0, 1.5, 1.0, 1.0])
    lw = np.log(g)
    reps = 6000
    A = np.array([orc.multinomial(lw, 4, r + 1)["a"] for r in range(reps)])
    p = g / g.sum()
    for i in range(len(g)):
        c = np.bincount(A[:, i], minlength=len(g))
        chi = ((c - reps * p) ** 2 / (reps * p)).sum()
        assert stats.chi2.sf(chi, len(g) - 1) > 1e-4, i
    # independence of two outputs: joint frequencies vs the product law
    joint = np.zeros((len(g), len(g)))
    np.add.at(joint, (A[:, 0], A[:, 5]), 1)
    e = reps * np.outer(p, p)
    chi = ((joint - e) ** 2 / e).sum()
    assert stats.chi2.sf(chi, (len(g) - 1) ** 2) > 1e-4


def test_multinomial_spec_examples(orc):
    reps = 20000
    counts = np.zeros(4)
    for r in range(1, reps // 4 + 1):
        np.add.at(counts, orc.multinomial(np.zeros(4), 2, r)["a"], 1)
    assert np.all(np.abs(counts / counts.sum() - 0.25) < 0.01)
    assert orc.multinomial(np.array([-3.0]), 2, 1)["a"][0] == 0


def test_plain_bpf_vs_kalman(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, N = 24, 1024
    runs = np.array([orc.run_filter_multinomial(p, N, 1100 + j, ys)[:, 0] for j in range(J)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)
