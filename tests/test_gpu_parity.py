"""GPU <-> oracle parity of one BPF step with augmented resampling, through the C-ABI.

Each case starts both sides from the same seeded synthetic particle cloud (inputs
module), the same (seed, n, y_n), and compares every intermediate element by
element: x_n, log g_n, each stage's ancestor table a_s, the composed ancestors A,
the V levels, the resampled particles and the estimates (tolerances in
tests/parity_util.py).  Sizes span several pass-1 tiles, several compose passes and
all BASELINE configurations' (d, M, S) shapes.
"""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import pf as pfb  # noqa: E402

from . import parity_util as pu  # noqa: E402


def _gpu_step(params, N, M, seed, n, xhat, y):
    f = pfb.ParticleFilter(params, N, M, seed, debug=True)
    f.set_state(xhat, n)
    f.step(y)
    S = f.S
    out = dict(
        x=f.debug_get(pfb.PF_DBG_X),
        lw=f.debug_get(pfb.PF_DBG_LOGW),
        a=np.stack([f.debug_get(pfb.PF_DBG_ANC_STAGE, s) for s in range(1, S + 1)]),
        A=f.debug_get(pfb.PF_DBG_ANC_FINAL),
        xhat=f.debug_get(pfb.PF_DBG_XHAT),
        logV=f.debug_get(pfb.PF_DBG_LOGV),
        filt=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER),
        filt2=f.estimate(pfb.PF_PHI_X2, pfb.PF_EST_FILTER),
        pred=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT),
        pred2=f.estimate(pfb.PF_PHI_X2, pfb.PF_EST_PREDICT),
        res=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_RESAMPLED),
        res2=f.estimate(pfb.PF_PHI_X2, pfb.PF_EST_RESAMPLED),
        launches=f.launches(),
    )
    f.close()
    return out


def _compare(orc, cfg_name, N, M, n, seed=1234, cloud_seed=99, outlier=0.0, xhat=None, params=None):
    cfg = inputs.CONFIGS[cfg_name]
    params = params or inputs.model_params(cfg)
    d = int(params["d"])
    if xhat is None:
        xhat = inputs.particle_cloud(cfg, N, cloud_seed)
    y = inputs.observation_for_step(cfg, cloud_seed + n, outlier_sigma=outlier)
    g = _gpu_step(params, N, M, seed, n, xhat, y)
    o = orc.step(params, N, M, seed, n, y, xhat)
    pu.check_x(g["x"], o["x"])
    pu.check_lw(g["lw"], o["lw"])
    stats = pu.check_stage_tables(g["a"], o["a"], o["delta"])
    flagged = pu.path_flags(o["a"], o["delta"])
    pu.check_composed(g["A"], o["A"], flagged)
    pu.check_logV(g["logV"], o["logV"])
    # resampled particles are exactly the gathered x_n of the GPU's own ancestors
    assert np.array_equal(g["xhat"].reshape(N, d), g["x"].reshape(N, d)[g["A"]], equal_nan=True)
    if not np.all(np.isfinite(o["x"])):
        return dict(stats=stats, flagged_paths=int(flagged.sum()), launches=g["launches"])
    pu.check_estimate(g["filt"], o["filter"][:d], o["filter"][d:])
    pu.check_estimate(g["pred"], o["predict"][:d], o["predict"][d:])
    assert np.all(np.abs(g["filt2"] - o["filter"][d:]) <= 1e-4 * np.abs(o["filter"][d:]) + 1e-12)
    assert np.all(np.abs(g["pred2"] - o["predict"][d:]) <= 1e-4 * np.abs(o["predict"][d:]) + 1e-12)
    # PF_EST_RESAMPLED: N^-1 sum phi(x_hat) against the oracle's resampled leg; outputs whose
    # (flagged) path picked another ancestor may move it by at most their share of the range
    nmis = int((g["A"] != o["A"]).sum())
    span = np.ptp(o["x"], axis=0) if N > 1 else np.zeros(d)
    allow = nmis / N * span
    pu.check_estimate_allow(g["res"], o["resampled"][:d], o["resampled"][d:], allow)
    pu.check_estimate_allow(g["res2"], o["resampled"][d:], None, nmis / N * np.ptp(o["x"] ** 2, axis=0),
                            second=False)
    return dict(stats=stats, flagged_paths=int(flagged.sum()), launches=g["launches"])


@pytest.mark.parametrize("n", [0, 1, 7])
def test_c1_full(orc, n):
    r = _compare(orc, "C1", 1024, 64, n)
    assert r["flagged_paths"] < 1024 * 0.05


@pytest.mark.parametrize("N,M,n", [(1 << 14, 64, 3), (1 << 16, 8, 2), (1 << 12, 2, 1), (1 << 15, 8192, 5),
                                   (1 << 14, 2048, 4), (1 << 16, 512, 1), (1 << 17, 32, 9), (4, 2, 1)])
def test_sv_shapes(orc, N, M, n):
    _compare(orc, "C3", N, M, n)


@pytest.mark.parametrize("N,M,n", [(1 << 16, 64, 2), (1 << 18, 64, 1), (1 << 14, 256, 3)])
def test_c4_model_shapes(orc, N, M, n):
    _compare(orc, "C4", N, M, n)


def test_c2_full(orc):
    _compare(orc, "C2", 1 << 20, 256, 4)


def test_c3_full_size_step(orc):
    _compare(orc, "C3", 1 << 24, 32, 11)


def test_outlier_degenerate_weights(orc):
    _compare(orc, "C4", 1 << 16, 64, 2, outlier=6.0)
    _compare(orc, "C1", 1024, 64, 2, outlier=8.0)


def test_equal_weights(orc):
    p = dict(inputs.model_params(inputs.CONFIGS["C4"]))
    p["Rinv"] = np.zeros_like(p["Rinv"])  # g_n == 1: uniform pools, p_s = 1/2
    _compare(orc, "C4", 1 << 14, 64, 3, params=p)


def test_nonfinite_particles(orc):
    cfg = inputs.CONFIGS["C4"]
    x = inputs.particle_cloud(cfg, 1 << 12, 5)
    x[3] = np.nan
    x[100:104] = np.inf
    _compare(orc, "C4", 1 << 12, 64, 0, xhat=x)


def test_minimum_topology(orc):
    _compare(orc, "C1", 4, 2, 1)
    _compare(orc, "C1", 8, 4, 0)
