"""Pins of the oracle's RNG (DESIGN.md §3 draw contract).

* Philox4x32-10: the oracle's independent implementation must equal cuRAND's
  library routine curand_Philox4x32_10 (host-compiled) on random and edge counters.
* Box-Muller normals: moments and a Kolmogorov-Smirnov test against scipy's normal CDF.
"""
import ctypes

import numpy as np
import pytest
from scipy import stats


def test_philox_matches_curand(orc, curand_host):
    rng = np.random.default_rng(7)
    n = 4096
    ctrs = rng.integers(0, 2 ** 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    keys = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    # edge cases: all-zero and all-ones counters/keys, and the draw-contract layout
    ctrs[0] = 0
    keys[0] = 0
    ctrs[1] = 0xFFFFFFFF
    keys[1] = 0xFFFFFFFF
    ctrs[2] = [12345, 17, (3 << 24) | 5, 0]
    keys[2] = [0xDEADBEEF, 1]
    ref = np.zeros((n, 4), np.uint32)
    curand_host.curand_philox_blocks(ctrs.ctypes.data_as(ctypes.c_void_p), keys.ctypes.data_as(ctypes.c_void_p),
                                     ref.ctypes.data_as(ctypes.c_void_p), n)
    for i in range(n):
        got = orc.philox(ctrs[i], keys[i])
        assert np.array_equal(got, ref[i]), (i, ctrs[i], keys[i], got, ref[i])


def test_box_muller_normals(orc):
    # 2^16 coordinates of the MUTATE field at n = 3
    z = np.array([orc.normal(99, orc.MUTATE, 3, c) for c in range(1 << 16)])
    assert abs(z.mean()) < 4.0 / np.sqrt(z.size)
    assert abs(z.var() - 1.0) < 4.0 * np.sqrt(2.0 / z.size)
    ks = stats.kstest(z, "norm")
    assert ks.pvalue > 1e-3
    # cos/sin pairs of one Box-Muller draw are uncorrelated
    assert abs(np.corrcoef(z[0::2], z[1::2])[0, 1]) < 4.0 / np.sqrt(z.size / 2)


def test_normal_fields_distinct(orc):
    """Different domains / steps / seeds give different draws (counter layout)."""
    a = orc.normal(1, orc.MUTATE, 1, 10)
    assert a != orc.normal(1, orc.INIT, 1, 10)
    assert a != orc.normal(1, orc.MUTATE, 2, 10)
    assert a != orc.normal(2, orc.MUTATE, 1, 10)
    assert a == orc.normal(1, orc.MUTATE, 1, 10)
