"""Pins of the relabelled exchange (oracle/pf_oracle.c orc_relabel_stage; SURVEY.md §8(f)3,
the surplus sketch of PAPER.md:826-850, reading R24) against exact laws.

* Every cross-stage exchange is a permutation of the stage's outputs (the multiset of
  sources is Alg. 3's), after it one of each matched pair of lists is empty (only the
  surplus reads across shards), and every matched output reads its own shard.
* Unbiasedness, Prop. 1 eq. aug_res_lack_of_bias, EXACTLY in rationals:
  the cross-stage tables are enumerated with their Alg. 3 probabilities (K_s rows,
  oracle/exact.py), the oracle's exchange is applied to each, and the local stages are
  folded in by the exact kernel product; then N^-1 sum_i P(A(i) = j) = g_j / sum g.
  Sizes S <= 3 with M <= 2 (S = 1 has no cross stage: a shard needs >= 2 groups).
* The count-imbalance law: the surplus of a shard pair is |c_r - c_r'| with
  c_r ~ Binomial(n, 1 - p), c_r' ~ Binomial(n, p) independent (n = N/G outputs per shard,
  p the pair's side probability): its exact expectation equals the enumerated one.
* Statistically: the relabelled filter tracks the Kalman means (5 MC sigma) and the
  resampled estimate is unbiased for the filter estimate (Prop. 1).
"""
import itertools
from fractions import Fraction
from math import comb

import numpy as np
import pytest

from oracle import exact, kalman
from paper_1812_01502_b200 import inputs


def _relabel_law(orc, S, M, G, g):
    """Exact P(A(i) = j) of Alg. 3 with the last log2 G stages relabelled."""
    N = M * 2 ** S
    L = G.bit_length() - 1
    Ks = exact.K_matrices(S, M, [Fraction(v) for v in g])
    # local stages 1..S-L: exact kernel product K_{S-L} ... K_1 (rows: stage S-L position)
    loc = Ks[S - L - 1]
    for K in reversed(Ks[: S - L - 1]):
        loc = exact.matmul(loc, K)
    cross = Ks[S - L:]
    supports = [[[j for j in range(N) if K[i][j] != 0] for i in range(N)] for K in cross]
    marg = [[Fraction(0)] * N for _ in range(N)]  # P(source at stage S-L of output i = k)
    surplus = Fraction(0)
    for combo in itertools.product(*[itertools.product(*rows) for rows in supports]):
        p = Fraction(1)
        for t, tab in enumerate(combo):
            for i, j in enumerate(tab):
                p *= cross[t][i][j]
        if p == 0:
            continue
        tabs = []
        for t, tab in enumerate(combo):
            rel, ex = orc.relabel_stage(np.array(tab), G, t + 1)
            assert sorted(rel.tolist()) == sorted(tab), "the exchange must permute the stage's outputs"
            nl = N // G
            half = 1 << t
            for r in range(G):
                rp = r ^ half
                assert min(ex[r], ex[rp]) == 0, "both lists of a pair keep a surplus"
                remote = sum(1 for i in range(r * nl, (r + 1) * nl) if rel[i] // nl == rp)
                assert remote == ex[r], "a matched output reads across the pair"
            surplus += p * int(ex.sum())
            tabs.append(rel)
        for i in range(N):
            k = i
            for t in range(L - 1, -1, -1):
                k = int(tabs[t][k])
            marg[i][k] += p
    P = exact.matmul(marg, loc)
    return P, surplus


CASES = [(2, 1, 2, (1, 3, 2, 5)), (2, 2, 2, (2, 1, 1, 4, 3, 1, 1, 2)), (3, 1, 2, (1, 2, 3, 4, 5, 6, 7, 8)),
         (3, 1, 4, (4, 1, 1, 2, 3, 1, 6, 2))]


@pytest.mark.parametrize("S,M,G,g", CASES)
def test_relabel_unbiased_exactly(orc, S, M, G, g):
    N = M * 2 ** S
    P, _ = _relabel_law(orc, S, M, G, g)
    tot = sum(g)
    for j in range(N):
        assert sum(P[i][j] for i in range(N)) / N == Fraction(g[j], tot), j
    for i in range(N):
        assert sum(P[i]) == 1


@pytest.mark.parametrize("S,M,G,g", [(2, 1, 2, (1, 3, 2, 5)), (2, 2, 2, (2, 1, 1, 4, 3, 1, 1, 2)),
                                     (3, 1, 2, (1, 2, 3, 4, 5, 6, 7, 8))])
def test_surplus_count_law(orc, S, M, G, g):
    """E[surplus] of the single cross stage = sum over pairs E|c_r - c_r'| with
    c_r ~ Bin(n, 1 - p), c_r' ~ Bin(n, p) (p = P(side = lower shard), exact V ratio)."""
    N = M * 2 ** S
    _, surplus = _relabel_law(orc, S, M, G, g)
    V = exact.V_levels(S, M, [Fraction(v) for v in g])[S - 1]  # V_{S-1}: constant per shard here
    nl = N // G

    def binom(n, q, k):
        return comb(n, k) * q ** k * (1 - q) ** (n - k)

    want = Fraction(0)
    for r in range(0, G, 2):
        p = V[r * nl] / (V[r * nl] + V[(r + 1) * nl])  # lower shard chosen
        for cr in range(nl + 1):
            for cp in range(nl + 1):
                want += binom(nl, 1 - p, cr) * binom(nl, p, cp) * abs(cr - cp)
    assert surplus == want


def test_relabel_no_cross_reads_when_balanced(orc):
    """Equal weights: p = 1/2 on every cross stage; the surplus is O(sqrt(N/G)), far below
    the N/G (1 - 1/G) of the plain exchange."""
    N, M, G = 1 << 16, 64, 8
    r = orc.augmented_resample_relabel(np.zeros(N), M, G, 5, 1)
    nl = N // G
    assert r["excess"].sum(axis=1).max() < 8 * np.sqrt(nl) * G
    ra = orc.augmented_resample(np.zeros(N), M, 5, 1)
    remote_plain = np.mean((ra["A"] // nl) != (np.arange(N) // nl))
    remote_rel = np.mean((r["A"] // nl) != (np.arange(N) // nl))
    assert remote_plain > 0.8 and remote_rel < 0.05


def test_relabel_local_stages_untouched(orc):
    """Stages 1..S-L are Alg. 3's tables, bit for bit."""
    rng = np.random.default_rng(3)
    N, M, G = 1 << 12, 16, 4
    lw = rng.normal(0, 1.5, N)
    a = orc.augmented_resample(lw, M, 9, 2)
    b = orc.augmented_resample_relabel(lw, M, G, 9, 2)
    S = a["a"].shape[0]
    assert np.array_equal(a["a"][: S - 2], b["a"][: S - 2])
    assert np.array_equal(a["logV"], b["logV"])
    for s in (S - 2, S - 1):
        assert sorted(a["a"][s].tolist()) == sorted(b["a"][s].tolist())


def test_relabel_resampled_unbiased_empirically(orc):
    N, M, G, d = 1024, 8, 4, 2
    rng = np.random.default_rng(11)
    x = rng.normal(size=(N, d))
    lw = rng.normal(0, 1.0, N)
    vals = []
    for seed in range(300):
        r = orc.augmented_resample_relabel(lw, M, G, seed, 1)
        vals.append(orc.estimates(d, lw, x, r["A"])["resampled"])
    vals = np.array(vals)
    f = orc.estimates(d, lw, x, None)["filter"]
    se = vals.std(axis=0, ddof=1) / np.sqrt(len(vals))
    assert np.all(np.abs(vals.mean(axis=0) - f) < 5 * se)


def test_relabel_filter_vs_kalman(orc):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=12)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J = 24
    runs = np.array([orc.run_filter_relabel(p, 64, 16, 4, 700 + j, ys)[:, 0] for j in range(J)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)
