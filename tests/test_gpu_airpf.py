"""GPU <-> oracle parity of one AIRPF step (Alg. 4 with Alg. 5 and Alg. 6/7; DESIGN.md
R19-R21) through the C-ABI (pf_set_airpf).

Both sides start from the same seeded cloud, seed, n and y.  Compared element by
element: x_n, the log-weights, the within-island ancestors (bit-exact away from a CDF
boundary), the island log-means and levels, every stage's island choices (bit-exact
where neither island of the pair drew within 1e-6 of its side threshold), the composed
island map, x_hat (the gathered blocks) and the estimates.  A two-step case checks that
the next step reads the island blocks; the GPU AIRPF filter must track the Kalman means.
"""
import numpy as np
import pytest

from oracle import kalman
from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import pf as pfb  # noqa: E402

from . import parity_util as pu  # noqa: E402


def _snap(f, d):
    S = f.S
    return dict(x=f.debug_get(pfb.PF_DBG_X), lw=f.debug_get(pfb.PF_DBG_LOGW), aw=f.debug_get(pfb.PF_DBG_ANC_STAGE, 1),
                logW=f.debug_get(pfb.PF_DBG_ISLAND_LOGW), logV=f.debug_get(pfb.PF_DBG_LOGV),
                choice=np.stack([f.debug_get(pfb.PF_DBG_ISLAND_CHOICE, s) for s in range(1, S + 1)]),
                A=f.debug_get(pfb.PF_DBG_ISLAND_A), xhat=f.debug_get(pfb.PF_DBG_XHAT),
                filt=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), pred=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT),
                res=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_RESAMPLED))


def _check(g, o, N, M, d):
    m, S = N // M, o["S"]
    pu.check_x(g["x"], o["x"])
    pu.check_lw(g["lw"], o["lw"])
    ok_w = o["wdelta"] >= pu.BOUNDARY
    bad = np.nonzero(ok_w & (g["aw"] != o["a_w"]))[0]
    assert bad.size == 0, f"{bad.size} within-island mismatches"
    pu.check_logV(g["logW"], o["logW"])
    pu.check_logV(g["logV"], o["logVbar"])
    isl = np.arange(m)
    flag_isl = np.zeros((S, m), bool)
    for s in range(1, S + 1):
        bits = (g["choice"][s - 1][isl >> 2] >> (isl & 3)) & 1
        src = isl ^ (bits.astype(np.int64) << (s - 1))
        fl = (o["idelta"][s - 1] < pu.BOUNDARY) | (o["idelta"][s - 1][isl ^ (1 << (s - 1))] < pu.BOUNDARY)
        flag_isl[s - 1] = fl
        bad = np.nonzero(~fl & (src != o["src"][s - 1]))[0]
        assert bad.size == 0, f"stage {s}: {bad.size} island choice mismatches"
    # composed island map, for islands with no flagged choice on their path
    path_fl = np.zeros(m, bool)
    pos = isl.copy()
    for s in range(S, 0, -1):
        path_fl |= flag_isl[s - 1][pos]
        pos = o["src"][s - 1][pos]
    bad = np.nonzero(~path_fl & (g["A"] != o["Aisl"]))[0]
    assert bad.size == 0, f"{bad.size} island map mismatches"
    # x_hat = the GPU's own within-resampled blocks, in the GPU's island order
    blocks = (g["A"].astype(np.int64)[:, None] * M + np.arange(M)[None, :]).ravel()
    assert np.array_equal(g["xhat"].reshape(N, d), g["x"].reshape(N, d)[g["aw"][blocks]], equal_nan=True)
    rows = np.repeat(~path_fl, M) & ok_w[blocks] if path_fl.any() else ok_w[blocks]
    pu.check_x(g["xhat"].reshape(N, d)[rows], o["xhat"][rows])
    pu.check_estimate(g["filt"], o["filter"][:d], o["filter"][d:])
    pu.check_estimate(g["pred"], o["predict"][:d], o["predict"][d:])
    # PF_EST_RESAMPLED through the island map = the mean of the materialised x_hat; against
    # the oracle's x_hat with an allowance for the flagged rows
    xh = g["xhat"].reshape(N, d).astype(np.float64)
    if np.all(np.isfinite(xh)):
        assert np.allclose(g["res"], xh.mean(axis=0), rtol=1e-5, atol=1e-6)
        nfl = N - int(rows.sum())
        pu.check_estimate_allow(g["res"], o["xhat"].mean(axis=0), (o["xhat"] ** 2).mean(axis=0),
                                nfl / N * np.ptp(o["x"], axis=0))
    return int(path_fl.sum()) + int((~ok_w).sum())


CASES = [("C1", 1024, 64, 1, 1), ("C1", 1024, 16, 2, 2), ("C4", 1 << 16, 64, 3, 1), ("C4", 1 << 14, 4, 5, 1),
         ("C3", 1 << 16, 32, 2, 1), ("C2", 1 << 16, 256, 1, 2), ("C4", 1 << 18, 64, 1, 1), ("C3", 1 << 15, 8192, 4, 1)]


@pytest.mark.parametrize("cfg_name,N,M,n,mode", CASES)
def test_airpf_step_parity(orc, cfg_name, N, M, n, mode):
    cfg = inputs.CONFIGS[cfg_name]
    params = inputs.model_params(cfg)
    d = int(params["d"])
    xhat = inputs.particle_cloud(cfg, N, 30 + n)
    y = inputs.observation_for_step(cfg, 60 + n, outlier_sigma=1.5)
    o = orc.step_airpf(params, N, M, 13, n, y, xhat, modified=(mode == 1))
    f = pfb.ParticleFilter(params, N, M, 13, debug=True, airpf=mode)
    f.set_state(xhat, n)
    f.step(y)
    g = _snap(f, d)
    f.close()
    _check(g, o, N, M, d)


def test_airpf_two_steps():
    """Step 2 must read the island blocks of step 1 (x_hat is never materialised)."""
    cfg = inputs.CONFIGS["C4"]
    params = inputs.model_params(cfg)
    N, M, d = 1 << 12, 16, 4
    from oracle import oracle as orc
    xhat = inputs.particle_cloud(cfg, N, 2)
    y1 = inputs.observation_for_step(cfg, 3)
    y2 = inputs.observation_for_step(cfg, 4)
    o1 = orc.step_airpf(params, N, M, 8, 1, y1, xhat)
    f = pfb.ParticleFilter(params, N, M, 8, debug=True, airpf=1)
    f.set_state(xhat, 1)
    f.step(y1)
    g1 = _snap(f, d)
    assert _check(g1, o1, N, M, d) == 0  # no flagged draw: both sides hold the same x_hat
    o2 = orc.step_airpf(params, N, M, 8, 2, y2, o1["xhat"].astype(np.float32))
    f.step(y2)
    g2 = _snap(f, d)
    f.close()
    _check(g2, o2, N, M, d)


def test_airpf_filter_vs_kalman():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, N, M = 32, 1024, 64
    runs = []
    for j in range(J):
        f = pfb.ParticleFilter(p, N, M, 700 + j, airpf=1)
        mean = []
        for y in ys:
            f.step(y)
            mean.append(f.estimate()[0])
        f.close()
        runs.append(mean)
    runs = np.array(runs)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)


def test_airpf_errors_and_switch_back():
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    f = pfb.ParticleFilter(p, 1 << 12, 16, 1)
    with pytest.raises(pfb.PFError):
        pfb.pf_set_airpf(f.h, 1)  # no PF_FLAG_AIRPF
    f.close()
    g = pfb.ParticleFilter(p, 1 << 12, 16, 1, airpf=1, debug=True)
    g.step(np.zeros(4, np.float32))
    xh = g.debug_get(pfb.PF_DBG_XHAT).copy()
    pfb.pf_set_airpf(g.h, 0)  # materialises x_hat, then plain augmented resampling
    assert np.array_equal(g.debug_get(pfb.PF_DBG_XHAT), xh)
    g.step(np.zeros(4, np.float32))
    assert g.last_stages() == g.S
    g.close()
