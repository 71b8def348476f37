"""Helpers for GPU <-> oracle parity (test infrastructure).

Tolerances:
  * x_n:       |x_gpu - x_orc| <= 1e-5 (1 + |x_orc|)      (fp32 mutation vs fp64)
  * log g:     |lw_gpu - lw_orc| <= 1e-5 (1 + |lw_orc|)
  * a_s(i):    bit-exact wherever the oracle's draw is >= 1e-6 from a decision boundary
               (BASELINE north_star); flagged draws are only counted
  * A(i):      bit-exact for outputs with no flagged draw on their ancestral path
  * log V_s:   |diff| <= 1e-5 (1 + |log V_orc|)  (fp32 log-weights carry relative error)
  * estimates: |diff| <= 1e-4 max(|ref|, posterior sd)   (reading R15)
"""
from __future__ import annotations

import numpy as np

BOUNDARY = 1e-6


def check_x(x_gpu, x_orc):
    x_gpu = np.asarray(x_gpu, np.float64).reshape(x_orc.shape)
    same_nonfinite = (~np.isfinite(x_orc)) & ((x_gpu == x_orc) | (np.isnan(x_gpu) & np.isnan(x_orc)))
    with np.errstate(invalid="ignore"):  # inf - inf where both sides agree (masked out)
        err = np.where(same_nonfinite, 0.0, np.abs(x_gpu - x_orc) / (1.0 + np.abs(x_orc)))
    assert np.all(err <= 1e-5), f"x mismatch: max rel err {err.max():.3g}"


def check_lw(lw_gpu, lw_orc):
    lw_gpu = np.asarray(lw_gpu, np.float64)
    both_inf = np.isneginf(lw_gpu) & np.isneginf(lw_orc)
    with np.errstate(invalid="ignore"):  # -inf - -inf where both sides agree (masked out)
        err = np.where(both_inf, 0.0, np.abs(lw_gpu - lw_orc) / (1.0 + np.abs(lw_orc)))
    assert np.all(err <= 1e-5), f"log-weight mismatch: max rel err {np.nanmax(err):.3g}"


def check_stage_tables(a_gpu, a_orc, delta):
    """a_gpu, a_orc: (S, N) ancestors; delta: (S, N) oracle boundary distances."""
    S = a_orc.shape[0]
    stats = []
    for s in range(S):
        ok = delta[s] >= BOUNDARY
        bad = np.nonzero(ok & (a_gpu[s] != a_orc[s]))[0]
        assert bad.size == 0, (f"stage {s + 1}: {bad.size} unflagged ancestor mismatches, first at i={bad[0]}: "
                               f"gpu {a_gpu[s][bad[0]]} orc {a_orc[s][bad[0]]} delta {delta[s][bad[0]]}")
        flagged = int((~ok).sum())
        stats.append((flagged, int((~ok & (a_gpu[s] != a_orc[s])).sum())))
    return stats


def path_flags(a_orc, delta):
    """True for outputs whose ancestral path contains a flagged draw (oracle tables)."""
    S, N = a_orc.shape
    flagged = np.zeros(N, bool)
    pos = np.arange(N)
    for s in range(S - 1, -1, -1):
        flagged |= delta[s][pos] < BOUNDARY
        pos = a_orc[s][pos]
    return flagged


def check_composed(A_gpu, A_orc, flagged):
    bad = np.nonzero(~flagged & (np.asarray(A_gpu) != np.asarray(A_orc)))[0]
    assert bad.size == 0, f"{bad.size} unflagged composed-ancestor mismatches (first i={bad[0]})"


def check_logV(lv_gpu, lv_orc):
    lv_gpu = np.asarray(lv_gpu, np.float64)
    both = np.isneginf(lv_gpu) & np.isneginf(lv_orc)
    err = np.where(both, 0.0, np.abs(lv_gpu - lv_orc) / (1.0 + np.abs(lv_orc)))
    assert np.all(err <= 1e-5), f"log V mismatch {np.nanmax(err):.3g}"


def check_estimate(gpu_mean, orc_mean, orc_second):
    sd = np.sqrt(np.maximum(orc_second - orc_mean ** 2, 0.0))
    tol = 1e-4 * np.maximum(np.abs(orc_mean), sd)
    err = np.abs(np.asarray(gpu_mean) - orc_mean)
    assert np.all(err <= tol + 1e-12), f"estimate mismatch {err} > {tol}"


def check_estimate_allow(gpu, ref, ref_second, allow, second=True):
    """check_estimate with an extra absolute allowance (outputs whose flagged path picked
    another ancestor).  second=False: a relative 1e-4 bound on a positive quantity."""
    gpu = np.asarray(gpu, np.float64)
    if second:
        sd = np.sqrt(np.maximum(ref_second - ref ** 2, 0.0))
        tol = 1e-4 * np.maximum(np.abs(ref), sd)
    else:
        tol = 1e-4 * np.abs(ref)
    err = np.abs(gpu - ref)
    assert np.all(err <= tol + allow + 1e-12), f"estimate mismatch {err} > {tol} + {allow}"
