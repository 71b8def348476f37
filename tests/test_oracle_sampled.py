"""Pins of the oracle's full-size sampled step (oracle/pf_oracle.c orc_step_sampled) against
its full step (orc_step, pinned in test_oracle_*): on every output of small problems the
sampled paths give the same composed ancestors, boundary distances, resampled states and V
levels, and the one-pass estimates (running-max shift) equal the two-pass ones."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs


@pytest.mark.parametrize("name,N,M,n", [("C1", 1024, 64, 0), ("C4", 1 << 12, 16, 3), ("C3", 1 << 11, 2, 2),
                                        ("C2", 1 << 12, 256, 1)])
def test_sampled_equals_full_step(orc, name, N, M, n):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    x = inputs.particle_cloud(cfg, N, 7)
    y = inputs.observation_for_step(cfg, 5 + n, outlier_sigma=1.5)
    full = orc.step(p, N, M, 11, n, y, x)
    outs = np.arange(N)
    smp = orc.step_sampled(p, N, M, 11, n, y, x, outs)
    assert np.array_equal(smp["A"], full["A"])
    assert np.array_equal(smp["xhat"], full["xhat"])
    assert np.array_equal(smp["logV"], full["logV"])
    # pdelta[k, s-1] is the delta of the stage-s draw on output k's path
    pos = outs.copy()
    for s in range(full["S"], 0, -1):
        assert np.array_equal(smp["pdelta"][:, s - 1], full["delta"][s - 1][pos])
        pos = full["a"][s - 1][pos]
    assert np.allclose(smp["filter"], full["filter"], rtol=1e-12, atol=1e-300)
    assert np.allclose(smp["predict"], full["predict"], rtol=1e-12, atol=1e-300)
    # a subset of outputs, in any order, gives the same rows
    sub = np.array([N - 1, 0, N // 2, 3])
    s2 = orc.step_sampled(p, N, M, 11, n, y, x, sub)
    assert np.array_equal(s2["A"], full["A"][sub]) and np.array_equal(s2["xhat"], full["xhat"][sub])
