"""GPU <-> oracle parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (non-debug handle, the plan of the full problem), on sampled outputs the oracle
evaluates one by one (oracle/pf_oracle.c orc_step_sampled):

* C4: N = 2^28, M = 64, S = 22, d = 4, one teacher-forced step with mutation (n = 1);
* C5 extremes: N = 2^26 with M = 2 (S = 25) and M = 8192 (S = 13).

Compared: every V level (the whole m - 1 table), the filter and predictive estimates
(tolerance of tests/parity_util.py), and for 4096 sampled outputs (random plus tile and
shard edges) the resampled state x_hat[i] = x_n[A(i)], except outputs whose ancestral path
holds a draw within 1e-6 of a decision boundary (reading R5; counted and bounded).
The fully adapted step (N1) and AIRPF (N2, Alg. 7 and 6) run the same check at C4's full
size (orc_step_sampled with theta, orc_step_airpf_sampled)."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import pf as pfb  # noqa: E402

from . import parity_util as pu  # noqa: E402


def _samples(N, k, seed):
    rng = np.random.default_rng(seed)
    edges = [0, 1, N - 1, N // 2 - 1, N // 2, 1023, 1024, 4095, 4096, N - 1024]
    return np.unique(np.concatenate([rng.integers(0, N, size=k - len(edges)), edges])).astype(np.int64)


@pytest.mark.parametrize("name,N,M,n", [("C4", 1 << 28, 64, 1), ("C5", 1 << 26, 2, 1), ("C5", 1 << 26, 8192, 1)])
def test_full_size_sampled_parity(orc, name, N, M, n):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    d = int(p["d"])
    xhat = inputs.particle_cloud(cfg, N, 29)
    y = inputs.observation_for_step(cfg, 31, outlier_sigma=1.0)
    outs = _samples(N, 4096, 3)
    o = orc.step_sampled(p, N, M, 41, n, y, xhat, outs)

    f = pfb.ParticleFilter(p, N, M, 41)
    f.set_state(xhat, n)
    del xhat
    f.step(y)
    pu.check_logV(f.debug_get(pfb.PF_DBG_LOGV), o["logV"])
    filt = f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER)
    pred = f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT)
    pu.check_estimate(filt, o["filter"][:d], o["filter"][d:])
    pu.check_estimate(pred, o["predict"][:d], o["predict"][d:])
    xg = f.debug_tensor(pfb.PF_DBG_XHAT).view(N, -1)[torch.from_numpy(outs).to("cuda"), :d].cpu().numpy()
    f.close()

    flagged = (o["pdelta"] < pu.BOUNDARY).any(axis=1)
    assert flagged.mean() < 0.05, f"{flagged.sum()} of {len(outs)} sampled paths flagged"  # M = 8192: ~3%
    pu.check_x(xg[~flagged], o["xhat"][~flagged])


def test_full_size_adaptive_sampled(orc):
    """Fully adapted step (N1) at C4's full size: ESS levels, S*, V table, estimates and
    sampled x_hat after S* stages."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, M, n, theta = cfg.N, cfg.M, 1, 0.5
    xhat = inputs.particle_cloud(cfg, N, 37)
    y = inputs.observation_for_step(cfg, 38, outlier_sigma=1.5)
    outs = _samples(N, 4096, 4)
    o = orc.step_sampled(p, N, M, 43, n, y, xhat, outs, theta=theta)
    if np.any(np.abs(o["ess"] - theta) < 1e-4 * theta):  # S* would be a rounding decision
        pytest.skip(f"theta within 1e-4 of an ESS level: {o['ess']}")
    f = pfb.ParticleFilter(p, N, M, 43, theta=theta)
    f.set_state(xhat, n)
    del xhat
    f.step(y)
    assert f.last_stages() == o["sstar"], (f.last_stages(), o["sstar"], o["ess"])
    assert np.allclose(f.debug_get(pfb.PF_DBG_ESS), o["ess"], rtol=2e-5, atol=0)
    pu.check_logV(f.debug_get(pfb.PF_DBG_LOGV), o["logV"])
    pu.check_estimate(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), o["filter"][:4], o["filter"][4:])
    pu.check_estimate(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT), o["predict"][:4], o["predict"][4:])
    xg = f.debug_tensor(pfb.PF_DBG_XHAT)[torch.from_numpy(outs).to("cuda")].cpu().numpy()
    f.close()
    flagged = (o["pdelta"] < pu.BOUNDARY).any(axis=1)
    assert flagged.mean() < 0.01
    pu.check_x(xg[~flagged], o["xhat"][~flagged])


@pytest.mark.parametrize("modified", [True, False])
def test_full_size_airpf_sampled(orc, modified):
    """AIRPF (N2) at C4's full size: island log-means, island map and x_hat on sampled
    outputs (path free of boundary draws), estimates."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, M, n = cfg.N, cfg.M, 1
    xhat = inputs.particle_cloud(cfg, N, 47)
    y = inputs.observation_for_step(cfg, 48, outlier_sigma=1.0)
    outs = _samples(N, 4096, 5)
    o = orc.step_airpf_sampled(p, N, M, 53, n, y, xhat, outs, modified=modified)
    f = pfb.ParticleFilter(p, N, M, 53, airpf=1 if modified else 2)
    f.set_state(xhat, n)
    del xhat
    f.step(y)
    pu.check_logV(f.debug_get(pfb.PF_DBG_ISLAND_LOGW), o["logW"])
    pu.check_estimate(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), o["filter"][:4], o["filter"][4:])
    pu.check_estimate(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT), o["predict"][:4], o["predict"][4:])
    A = f.debug_get(pfb.PF_DBG_ISLAND_A).astype(np.int64)
    xg = f.debug_tensor(pfb.PF_DBG_XHAT)[torch.from_numpy(outs).to("cuda")].cpu().numpy()
    f.close()
    ok = o["sdelta"] >= pu.BOUNDARY
    assert ok.mean() > 0.95
    blk = outs // M
    assert np.array_equal(A[blk[ok]], o["Aisl"][blk[ok]])
    pu.check_x(xg[ok], o["xhat"][ok])


def test_full_size_multinomial_sampled(orc):
    """The plain BPF with multinomial resampling (Alg. 2) at C4's full size.  With N = 2^28
    the CDF boundaries are ~1/N apart, closer than any fixed margin, so the check is: every
    sampled GPU ancestor lies in the oracle's window of draws for u -+ 1e-6 (the GPU's fp32
    tile CDFs, reading R22, round within it), most are exact, and x_hat is the ancestor's
    state.  The handle keeps the ancestors (PF_FLAG_DEBUG; same kernels and launches)."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, n = cfg.N, 1
    xhat = inputs.particle_cloud(cfg, N, 57)
    y = inputs.observation_for_step(cfg, 58, outlier_sigma=1.0)
    outs = _samples(N, 4096, 6)
    o = orc.step_multinomial_sampled(p, N, 59, n, y, xhat, outs, eps=1e-6)
    f = pfb.ParticleFilter(p, N, cfg.M, 59, multinomial=True, debug=True)
    f.set_state(xhat, n)
    del xhat
    f.step(y)
    pu.check_estimate(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), o["filter"][:4], o["filter"][4:])
    pu.check_estimate(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT), o["predict"][:4], o["predict"][4:])
    idx = torch.from_numpy(outs).to("cuda")
    ag = f.debug_tensor(pfb.PF_DBG_ANC_FINAL)[idx].cpu().numpy().astype(np.int64)
    xg = f.debug_tensor(pfb.PF_DBG_XHAT)[idx].cpu().numpy()
    f.close()
    inside = (o["klo"] <= ag) & (ag <= o["khi"])
    assert inside.all(), f"{(~inside).sum()} ancestors outside the 1e-6 window"
    exact = ag == o["a"]
    assert exact.mean() > 0.9, exact.mean()
    pu.check_x(xg[exact], o["xnb"][exact, 2])
