"""Pins of the interaction structure (oracle/exact.py and the oracle's XOR pairing).

* Fig. 1 A_1, A_2 for m=4, M=3 (tests/golden/fig1_A_m4_M3.txt).
* Fig. 2 pairs for m=8 (tests/golden/fig2_pairs_m8.txt).
* Lemma `facts about A`: symmetric, idempotent, doubly stochastic,
  explicit nonzero pattern; Lemma `ones product` and the partial
  products of its proof.
* The XOR pairing the oracle and the CUDA path use (partner = g ^ 2^{s-1}) equals all
  of the above.
"""
import os
from fractions import Fraction

import pytest

from oracle import exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


def test_fig1_matrices():
    lines = _read_golden("fig1_A_m4_M3.txt")
    blocks = {}
    cur = None
    for ln in lines:
        if ln in ("A1", "A2"):
            cur = ln
            blocks[cur] = []
        else:
            blocks[cur].append([int(v) for v in ln.split()])
    for s, key in ((1, "A1"), (2, "A2")):
        A = exact.A_matrix(2, 3, s)
        for i in range(12):
            for j in range(12):
                want = Fraction(blocks[key][i // 3][j // 3], 2 * 3)  # (1/2) * 1_{1/3}
                assert A[i][j] == want, (s, i, j)


def test_fig2_pairs_and_pair_sequences():
    lines = _read_golden("fig2_pairs_m8.txt")[1:]
    for s, ln in enumerate(lines, start=1):
        want = [tuple(int(v) for v in p.strip("()").split(",")) for p in ln.split()]
        ls, rs = exact.pair_sequences(3, s)
        assert list(zip(ls, rs)) == want
        # XOR characterisation (0-based groups): partner(g) = g ^ 2^{s-1}
        for (l, r) in want:
            assert (l - 1) ^ (1 << (s - 1)) == r - 1


@pytest.mark.parametrize("S", [1, 2, 3, 4, 5, 6])
def test_lemma_pattern_is_xor(S):
    m = 2 ** S
    for s in range(1, S + 1):
        ls, rs = exact.pair_sequences(S, s)
        assert sorted(ls + rs) == list(range(1, m + 1))  # a partition of {1..m}
        for i in range(1, m + 1):
            cols = exact.lemma_nonzero_columns(S, s, i)
            assert cols == {i, ((i - 1) ^ (1 << (s - 1))) + 1}
        if S <= 4:
            Abar = exact.island_A_matrix(S, s)
            for i in range(m):
                nz = {j for j in range(m) if Abar[i][j] != 0}
                assert nz == {i, i ^ (1 << (s - 1))}
                assert Abar[i][i] == Fraction(1, 2)


@pytest.mark.parametrize("S,M", [(1, 1), (1, 2), (1, 3), (2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3), (4, 1), (4, 2)])
def test_A_properties_and_products(S, M):
    N = M * 2 ** S
    As = [exact.A_matrix(S, M, s) for s in range(1, S + 1)]
    for A in As:
        assert A == exact.transpose(A)                       # symmetric
        assert exact.matmul(A, A) == A                      # idempotent
        for i in range(N):                                  # doubly stochastic
            assert sum(A[i]) == 1
            assert sum(A[j][i] for j in range(N)) == 1
        assert {e for row in A for e in row} <= {Fraction(0), Fraction(1, 2 * M)}
    P = As[0]
    for k in range(2, S + 1):
        P = exact.matmul(As[k - 1], P)                      # prod_{s<=k} A_s = A_k ... A_1
        want = exact.kron(exact.kron(exact.identity(2 ** (S - k)), exact.ones_over(2 ** k)), exact.ones_over(M))
        assert P == want                                    # partial products
    assert P == exact.ones_over(N)                          # Lemma `ones product`
