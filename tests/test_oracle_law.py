"""Pins of the oracle's augmented resampling (Alg. 3) against the
exact law, computed in rationals from the materialised A_s (oracle/exact.py):

* per-stage law of a_s(i) vs K_s = A_s V_{s-1} / V_s, chi-square;
* composed marginal P(A(i)=j) = (K_S..K_1)[i,j] and, for S <= 2, M <= 4, the full joint
  law by enumeration (BASELINE north_star: "brute-force enumeration ... S <= 2, M <= 4");
* V levels vs eq. V_defn_proofs; V_S = N^-1 sum g (Lemma facts_about_Vs (c));
* unbiasedness, Prop. 1 eq. aug_res_lack_of_bias (exactly, and empirically);
* SPEC worked example m=2, M=1; dissemination in log2 m rounds;
* stage-1 index = count of CDF values <= u*C (searchsorted, library routine).
"""
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from oracle import exact

SEED = 20240607


def _run_reps(orc, lw, M, reps, seed=SEED):
    N = lw.shape[0]
    S = int(round(np.log2(N // M)))
    a_all = np.zeros((reps, S, N), np.int64)
    A_all = np.zeros((reps, N), np.int64)
    for r in range(reps):
        out = orc.augmented_resample(lw, M, seed, n=r + 1)
        a_all[r] = out["a"]
        A_all[r] = out["A"]
    return a_all, A_all


def _chi2_ok(counts, probs, min_p=1e-4):
    probs = np.asarray([float(p) for p in probs])
    keep = probs > 0
    assert counts[~keep].sum() == 0, "draw outside the support of the exact law"
    exp_ = probs[keep] * counts.sum()
    if keep.sum() <= 1:
        return True
    chi = ((counts[keep] - exp_) ** 2 / exp_).sum()
    p = stats.chi2.sf(chi, keep.sum() - 1)
    return p > min_p


CASES = [(1, 1, (3, 1)), (1, 2, (1, 2, 3, 4)), (1, 4, (5, 1, 1, 2, 3, 1, 4, 2)),
         (2, 1, (1, 3, 2, 5)), (2, 2, (2, 1, 1, 4, 3, 1, 1, 2)), (2, 4, tuple(range(1, 17))),
         (3, 1, (1, 2, 3, 4, 5, 6, 7, 8))]


@pytest.mark.parametrize("S,M,g", CASES)
def test_stage_and_composed_law(orc, S, M, g):
    N = M * 2 ** S
    gF = [Fraction(v) for v in g]
    lw = np.log(np.array(g, np.float64))
    reps = 6000
    a_all, A_all = _run_reps(orc, lw, M, reps)
    Ks = exact.K_matrices(S, M, gF)
    for s in range(S):
        for i in range(N):
            counts = np.bincount(a_all[:, s, i], minlength=N)
            assert _chi2_ok(counts, Ks[s][i]), (s + 1, i)
    P = exact.composed_marginal(S, M, gF)
    for i in range(N):
        counts = np.bincount(A_all[:, i], minlength=N)
        assert _chi2_ok(counts, P[i]), i


@pytest.mark.parametrize("S,M,g", [(1, 1, (3, 1)), (1, 2, (1, 2, 3, 4)), (2, 1, (1, 3, 2, 5))])
def test_joint_law_enumeration(orc, S, M, g):
    gF = [Fraction(v) for v in g]
    law = exact.joint_law(S, M, gF)
    assert sum(law.values()) == 1
    lw = np.log(np.array(g, np.float64))
    reps = 20000
    _, A_all = _run_reps(orc, lw, M, reps, seed=SEED + 1)
    keys = list(law.keys())
    index = {k: t for t, k in enumerate(keys)}
    counts = np.zeros(len(keys), np.int64)
    for row in A_all:
        counts[index[tuple(int(v) for v in row)]] += 1  # KeyError = outcome outside the support
    assert _chi2_ok(counts, [law[k] for k in keys])


@pytest.mark.parametrize("S,M", [(1, 2), (2, 2), (3, 1), (3, 4)])
def test_V_levels_exact(orc, S, M):
    rng = np.random.default_rng(S * 10 + M)
    N = M * 2 ** S
    g = rng.integers(1, 9, size=N)
    V = exact.V_levels(S, M, [Fraction(int(v)) for v in g])
    out = orc.augmented_resample(np.log(g.astype(np.float64)), M, 1, 1)
    m = N // M
    for s in range(1, S + 1):
        lv = out["logV"][orc.level_offset(m, s): orc.level_offset(m, s) + (m >> s)]
        for i in range(N):
            blk = (i // M) >> s
            assert abs(np.exp(lv[blk]) / float(V[s][i]) - 1.0) < 1e-12
        for i in range(N):  # V_s <= ||g|| (Lemma facts_about_Vs (b))
            assert V[s][i] <= max(g)


@pytest.mark.parametrize("N,M", [(64, 2), (1024, 64), (4096, 8), (4096, 1024)])
def test_V_S_is_mean_g(orc, N, M):
    rng = np.random.default_rng(N + M)
    lw = rng.normal(-3.0, 2.0, size=N)
    out = orc.augmented_resample(lw, M, 5, 2, tables=False)
    m = N // M
    S = out["S"]
    root = out["logV"][orc.level_offset(m, S)]
    mean_g = np.exp(lw).mean()
    assert abs(np.exp(root) / mean_g - 1.0) < 1e-12


@pytest.mark.parametrize("S,M", [(1, 2), (2, 2), (3, 1), (2, 4)])
def test_unbiasedness_exact_and_empirical(orc, S, M):
    N = M * 2 ** S
    g = [Fraction(v) for v in range(1, N + 1)]
    P = exact.composed_marginal(S, M, g)
    tot = sum(g)
    for j in range(N):  # Prop. 1 with phi = indicator of particle j, exactly
        assert sum(P[i][j] for i in range(N)) / N == g[j] / tot
    lw = np.log(np.arange(1, N + 1, dtype=np.float64))
    reps = 20000
    _, A_all = _run_reps(orc, lw, M, reps, seed=SEED + 2)
    for j in range(N):
        frac = (A_all == j).mean(axis=1)  # N^-1 #{i : A(i) = j} per replicate
        want = float(g[j] / tot)
        se = frac.std(ddof=1) / np.sqrt(reps)
        assert abs(frac.mean() - want) < 4 * se + 1e-12


def test_spec_worked_example_m2_M1(orc):
    # each output independently = xi_0^1 w.p. w1/(w1+w2); V_1 = (w1+w2)/2
    w1, w2 = 3.0, 1.0
    out = orc.augmented_resample(np.log([w1, w2]), 1, 11, 1)
    assert abs(np.exp(out["logV"][0]) - (w1 + w2) / 2) < 1e-15
    a_all, _ = _run_reps(orc, np.log([w1, w2]), 1, 20000)
    frac = (a_all[:, 0, :] == 0).mean()
    assert abs(frac - 0.75) < 4 * np.sqrt(0.75 * 0.25 / 40000)


@pytest.mark.parametrize("S", [1, 2, 3, 4])
def test_dissemination_drill(orc, S):
    # one hot PE disseminates to all m PEs in log2(m) stages.
    M = 2
    m = 2 ** S
    lw = np.full(M * m, -70.0)
    lw[:M] = 0.0
    out = orc.augmented_resample(lw, M, 3, 4)
    a = out["a"]
    N = M * m
    for s in range(1, S + 1):
        # stage-0 ancestor of every stage-s particle in groups 0..2^s - 1 is hot
        for i in range(N):
            j = i
            for t in range(s, 0, -1):
                j = a[t - 1][j]
            if (i // M) < 2 ** s:
                assert j < M, (s, i)
    assert np.all(out["A"] < M)


@pytest.mark.parametrize("M", [1, 2, 4, 64])
def test_stage1_index_is_searchsorted(orc, M):
    rng = np.random.default_rng(M)
    N = 8 * M
    lw = rng.normal(0, 1.5, size=N)
    seed, n = 77, 9
    out = orc.augmented_resample(lw, M, seed, n)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for base in range(0, N, 2 * M):
        w = np.exp(lw[base: base + 2 * M] - lw[base: base + 2 * M].max())
        C = np.cumsum(w)  # library routine: sequential prefix sums
        for i in range(base, base + 2 * M):
            r = orc.philox([i >> 2, n, (3 << 24) | 1, 0], key)[i & 3]
            u = (int(r) >> 8) * 2.0 ** -24
            k = np.searchsorted(C[:-1], u * C[-1], side="right")
            assert out["a"][0][i] == base + k
            assert abs(out["delta"][0][i] - np.min(np.abs(u - C[:-1] / C[-1]))) <= 1e-7
