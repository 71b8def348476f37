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


@pytest.mark.parametrize("name,N,M,n,theta", [("C4", 1 << 12, 16, 3, 0.3), ("C1", 1024, 64, 1, 0.9),
                                              ("C3", 1 << 11, 2, 2, 0.05), ("C4", 1 << 12, 16, 3, 1e-9)])
def test_sampled_adaptive_equals_full_adaptive(orc, name, N, M, n, theta):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    x = inputs.particle_cloud(cfg, N, 8)
    y = inputs.observation_for_step(cfg, 6 + n, outlier_sigma=2.0)
    full = orc.step_adaptive(p, N, M, 13, n, y, x, np.zeros(N), theta)
    smp = orc.step_sampled(p, N, M, 13, n, y, x, np.arange(N), theta=theta)
    assert smp["sstar"] == full["sstar"]
    assert np.array_equal(smp["ess"], full["ess"])
    assert np.array_equal(smp["A"], full["A"])
    assert np.array_equal(smp["xhat"], full["xhat"])
    assert np.array_equal(smp["logV"], full["logV"])
    assert np.all(np.isinf(smp["pdelta"][:, smp["sstar"]:]))


@pytest.mark.parametrize("modified", [True, False])
@pytest.mark.parametrize("name,N,M,n", [("C4", 1 << 12, 16, 3), ("C1", 1024, 64, 1), ("C3", 1 << 11, 4, 2)])
def test_sampled_airpf_equals_full_airpf(orc, name, N, M, n, modified):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    x = inputs.particle_cloud(cfg, N, 9)
    y = inputs.observation_for_step(cfg, 7 + n, outlier_sigma=1.0)
    full = orc.step_airpf(p, N, M, 17, n, y, x, modified=modified)
    smp = orc.step_airpf_sampled(p, N, M, 17, n, y, x, np.arange(N), modified=modified)
    assert np.array_equal(smp["Aisl"], full["Aisl"])
    assert np.array_equal(smp["logW"], full["logW"])
    assert np.array_equal(smp["xhat"], full["xhat"])
    assert np.allclose(smp["filter"], full["filter"], rtol=1e-12, atol=1e-300)
    # sdelta = min over the within draw taken and both islands' draws at every stage
    m, S = N // M, full["S"]
    for i in range(0, N, max(1, N // 64)):
        c, dm = i // M, np.inf
        for s in range(S, 0, -1):
            dm = min(dm, full["idelta"][s - 1][c], full["idelta"][s - 1][c ^ (1 << (s - 1))])
            c = full["src"][s - 1][c]
        dm = min(dm, full["wdelta"][c * M + i % M])
        assert smp["sdelta"][i] == np.float32(dm)


@pytest.mark.parametrize("name,N,n", [("C4", 1 << 12, 3), ("C1", 1024, 0), ("C3", 1 << 11, 2)])
def test_sampled_multinomial_equals_full(orc, name, N, n):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    x = inputs.particle_cloud(cfg, N, 10)
    y = inputs.observation_for_step(cfg, 8 + n, outlier_sigma=1.0)
    full = orc.step_multinomial(p, N, 19, n, y, x)
    smp = orc.step_multinomial_sampled(p, N, 19, n, y, x, np.arange(N))
    assert np.array_equal(smp["a"], full["a"])
    assert np.array_equal(smp["sdelta"], full["delta"])
    assert np.array_equal(smp["xnb"][:, 2], full["xhat"])
    for o in (-2, -1, 1, 2):
        j = full["a"] + o
        ok = (j >= 0) & (j < N)
        assert np.array_equal(smp["xnb"][ok, 2 + o], full["x"][j[ok]])
        assert np.all(np.isnan(smp["xnb"][~ok, 2 + o]))
    assert np.allclose(smp["filter"], full["filter"], rtol=1e-12, atol=1e-300)
    # the eps window contains the draw and shrinks to it away from boundaries
    assert np.all((smp["klo"] <= smp["a"]) & (smp["a"] <= smp["khi"]))
    far = smp["sdelta"] > 1e-6
    assert np.array_equal(smp["klo"][far], smp["a"][far]) and np.array_equal(smp["khi"][far], smp["a"][far])
