"""Exact (rational) objects of augmented resampling, for pinning the oracle.

TEST INFRASTRUCTURE ONLY.  Pure Python with fractions.Fraction; small sizes only.

* A_s materialised from its Kronecker definition, eq. `A matrices`:
      A_s = I_{2^{S-s}} (x) 1_{1/2} (x) I_{2^{s-1}} (x) 1_{1/M},
  where 1_{1/k} is the k x k matrix with every entry 1/k.
* The explicit nonzero pattern of Lemma `facts about A` and the
  pair sequences (l_s^i, r_s^i) of PAPER.md:1044-1049.
* V recursion, eq. V_defn_proofs, and the one-stage kernels
      K_s[i, j] = A_s^{ij} V_{s-1}^j / V_s^i        (eq. P_in_terms_of_V_proofs)
* Composed marginal law of the stage-0 ancestor:  P(A(i) = j) = (K_S ... K_1)[i, j]
  (xi_S^i = xi_{S-1}^{a_S(i)}, each a_s drawn row-wise from K_s).
* Full joint law of (a_1, ..., a_S) by enumeration, for tiny sizes.
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from typing import List, Sequence

Matrix = List[List[Fraction]]


def identity(k: int) -> Matrix:
    return [[Fraction(int(i == j)) for j in range(k)] for i in range(k)]


def ones_over(k: int) -> Matrix:
    """1_{1/k}: k x k matrix of ones multiplied by 1/k."""
    return [[Fraction(1, k) for _ in range(k)] for _ in range(k)]


def kron(a: Matrix, b: Matrix) -> Matrix:
    ra, ca, rb, cb = len(a), len(a[0]), len(b), len(b[0])
    return [[a[i // rb][j // cb] * b[i % rb][j % cb] for j in range(ca * cb)] for i in range(ra * rb)]


def matmul(a: Matrix, b: Matrix) -> Matrix:
    n, k, p = len(a), len(b), len(b[0])
    return [[sum((a[i][t] * b[t][j] for t in range(k)), Fraction(0)) for j in range(p)] for i in range(n)]


def transpose(a: Matrix) -> Matrix:
    return [list(r) for r in zip(*a)]


def A_matrix(S: int, M: int, s: int) -> Matrix:
    """eq. A matrices: A_s = I_{2^{S-s}} (x) 1_{1/2} (x) I_{2^{s-1}} (x) 1_{1/M}."""
    assert 1 <= s <= S
    out = kron(identity(2 ** (S - s)), ones_over(2))
    out = kron(out, identity(2 ** (s - 1)))
    return kron(out, ones_over(M))


def island_A_matrix(S: int, s: int) -> Matrix:
    """The m x m factor I_{2^{S-s}} (x) 1_{1/2} (x) I_{2^{s-1}} (Lemma `facts about A`)."""
    return A_matrix(S, 1, s)


def lemma_nonzero_columns(S: int, s: int, i: int) -> set:
    """eq. explicit nonzero elements, 1-based i and result."""
    return {((i - 1) % 2 ** (s - 1)) + (q - 1) * 2 ** (s - 1) + 2 ** s * ((i - 1) // 2 ** s) + 1
            for q in (1, 2)}


def pair_sequences(S: int, s: int):
    """(l_s^1..l_s^{m/2}), (r_s^1..r_s^{m/2}) of PAPER.md:1044-1049 (1-based)."""
    ls, rs = [], []
    for i in range(1, 2 ** (S - s) + 1):
        for j in range(1, 2 ** (s - 1) + 1):
            ls.append(2 ** s * (i - 1) + (j - 1) + 1)
            rs.append(2 ** s * (i - 1) + (j - 1) + 1 + 2 ** (s - 1))
    return ls, rs


def V_levels(S: int, M: int, g: Sequence[Fraction]) -> List[List[Fraction]]:
    """V_0 = g, V_s = A_s V_{s-1} (eq. V_defn_proofs), per particle; returns [V_0..V_S]."""
    V = [list(map(Fraction, g))]
    for s in range(1, S + 1):
        A = A_matrix(S, M, s)
        prev = V[-1]
        V.append([sum((A[i][j] * prev[j] for j in range(len(prev))), Fraction(0)) for i in range(len(prev))])
    return V


def K_matrices(S: int, M: int, g: Sequence[Fraction]) -> List[Matrix]:
    """K_s[i][j] = A_s^{ij} V_{s-1}^j / V_s^i, s = 1..S."""
    V = V_levels(S, M, g)
    out = []
    for s in range(1, S + 1):
        A = A_matrix(S, M, s)
        N = len(A)
        out.append([[A[i][j] * V[s - 1][j] / V[s][i] for j in range(N)] for i in range(N)])
    return out


def composed_marginal(S: int, M: int, g: Sequence[Fraction]) -> Matrix:
    """P(A(i) = j) = (K_S K_{S-1} ... K_1)[i][j]."""
    Ks = K_matrices(S, M, g)
    P = Ks[-1]
    for K in reversed(Ks[:-1]):
        P = matmul(P, K)
    return P


def joint_law(S: int, M: int, g: Sequence[Fraction]):
    """Exact joint law of the composed map (A(0), ..., A(N-1)) by enumerating every
    stage's independent draws (one-step conditional independence).
    Returns dict: tuple(A) -> probability.  Only for (2M)^(N*S) small."""
    Ks = K_matrices(S, M, g)
    N = len(g)
    law = {}
    supports = [[[j for j in range(N) if K[i][j] != 0] for i in range(N)] for K in Ks]
    stage_choices = []
    for s in range(S):
        rows = supports[s]
        stage_choices.append(list(itertools.product(*rows)))
    for combo in itertools.product(*stage_choices):
        p = Fraction(1)
        for s, a in enumerate(combo):
            for i, j in enumerate(a):
                p *= Ks[s][i][j]
        if p == 0:
            continue
        A = []
        for i in range(N):
            j = i
            for s in range(S - 1, -1, -1):
                j = combo[s][j]
            A.append(j)
        A = tuple(A)
        law[A] = law.get(A, Fraction(0)) + p
    return law
