"""GPU parity of AIRPF2, AIRPF with the fully adapted scheme (DESIGN.md
reading R26; pf_set_airpf + pf_set_adaptive), against the oracle's orc_step_airpf_adaptive:
the island ESS levels (2e-5 relative), S* exactly (theta placed midway between two oracle
levels so S* is not a rounding decision), x_n, the log-weights with the carried island
weight, the within-island ancestors, the island log-means and levels, the island choices of
the stages that ran, the island map, x_hat and the estimates; two-step runs exercise the
carried weights (S* = 0 and 0 < S* < S); theta = 1 equals the plain AIRPF step bit for bit;
the AIRPF2 filter tracks the Kalman means."""
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
                A=f.debug_get(pfb.PF_DBG_ISLAND_A), xhat=f.debug_get(pfb.PF_DBG_XHAT), ess=f.debug_get(pfb.PF_DBG_ESS),
                ss=f.last_stages(), filt=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER),
                pred=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT))


def _check(g, o, N, M, d):
    m, ss = N // M, o["sstar"]
    assert np.allclose(g["ess"], o["ess"], rtol=2e-5, atol=0), (g["ess"], o["ess"])
    assert g["ss"] == ss
    pu.check_x(g["x"], o["x"])
    pu.check_lw(g["lw"], o["lw"])
    ok_w = o["wdelta"] >= pu.BOUNDARY
    assert not np.any(ok_w & (g["aw"] != o["a_w"])), "within-island mismatches"
    pu.check_logV(g["logW"], o["logW"])
    pu.check_logV(g["logV"], o["logVbar"])
    isl = np.arange(m)
    flag = np.zeros((max(ss, 1), m), bool)
    for s in range(1, ss + 1):
        bits = (g["choice"][s - 1][isl >> 2] >> (isl & 3)) & 1
        src = isl ^ (bits.astype(np.int64) << (s - 1))
        fl = (o["idelta"][s - 1] < pu.BOUNDARY) | (o["idelta"][s - 1][isl ^ (1 << (s - 1))] < pu.BOUNDARY)
        flag[s - 1] = fl
        assert not np.any(~fl & (src != o["src"][s - 1])), f"stage {s}: island choice mismatches"
    path_fl = np.zeros(m, bool)
    pos = isl.copy()
    for s in range(ss, 0, -1):
        path_fl |= flag[s - 1][pos]
        pos = o["src"][s - 1][pos]
    assert not np.any(~path_fl & (g["A"] != o["Aisl"])), "island map mismatches"
    blocks = (g["A"].astype(np.int64)[:, None] * M + np.arange(M)[None, :]).ravel()
    rows = np.repeat(~path_fl, M) & ok_w[blocks]
    pu.check_x(g["xhat"].reshape(N, d)[rows], o["xhat"][rows])
    pu.check_estimate(g["filt"], o["filter"][:d], o["filter"][d:])
    pu.check_estimate(g["pred"], o["predict"][:d], o["predict"][d:])
    return int(path_fl.sum()) + int((~ok_w).sum())


def _theta_between(ess, target):
    """theta midway between E_{target-1} and E_target (so S* = target unless the levels tie)."""
    e = np.asarray(ess)
    if target == 0:
        return max(1e-6, 0.5 * e[0])
    lo = max(e[:target])
    hi = e[target]
    return 0.5 * (lo + hi) if hi > lo else None


CASES = [("C4", 1 << 14, 16, 1), ("C1", 1024, 16, 2), ("C3", 1 << 14, 32, 1), ("C2", 1 << 14, 256, 1)]


@pytest.mark.parametrize("cfg_name,N,M,target", CASES)
def test_airpf2_step_parity(orc, cfg_name, N, M, target):
    cfg = inputs.CONFIGS[cfg_name]
    p = inputs.model_params(cfg)
    d = int(p["d"])
    x = inputs.particle_cloud(cfg, N, 12)
    y = inputs.observation_for_step(cfg, 13, outlier_sigma=2.0)
    probe = orc.step_airpf_adaptive(p, N, M, 5, 1, y, x, np.zeros(N), 1.0)
    theta = _theta_between(probe["ess"], target)
    if theta is None:
        pytest.skip("tied ESS levels")
    o = orc.step_airpf_adaptive(p, N, M, 5, 1, y, x, np.zeros(N), theta)
    f = pfb.ParticleFilter(p, N, M, 5, debug=True, airpf=1, theta=theta)
    f.set_state(x, 1)
    f.step(y)
    g = _snap(f, d)
    f.close()
    assert o["sstar"] == target
    _check(g, o, N, M, d)


@pytest.mark.parametrize("first_target", [0, 1, 2])
def test_airpf2_two_steps_carry(orc, first_target):
    """Step 2 reads the island blocks of step 1 and adds the carried island weight."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, M, d = 1 << 12, 16, 4
    x = inputs.particle_cloud(cfg, N, 21)
    y1 = inputs.observation_for_step(cfg, 22, outlier_sigma=1.5)
    y2 = inputs.observation_for_step(cfg, 23)
    probe = orc.step_airpf_adaptive(p, N, M, 3, 1, y1, x, np.zeros(N), 1.0)
    theta = _theta_between(probe["ess"], first_target)
    if theta is None:
        pytest.skip("tied ESS levels")
    o1 = orc.step_airpf_adaptive(p, N, M, 3, 1, y1, x, np.zeros(N), theta)
    f = pfb.ParticleFilter(p, N, M, 3, debug=True, airpf=1, theta=theta)
    f.set_state(x, 1)
    f.step(y1)
    g1 = _snap(f, d)
    if _check(g1, o1, N, M, d) != 0:
        f.close()
        pytest.skip("a boundary-flagged draw: the two sides may hold different samples")
    o2 = orc.step_airpf_adaptive(p, N, M, 3, 2, y2, o1["xhat"].astype(np.float32), o1["lwc"], theta)
    f.step(y2)
    g2 = _snap(f, d)
    f.close()
    _check(g2, o2, N, M, d)


def test_theta_one_is_plain_airpf_gpu():
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N, M = 1 << 14, 16
    x = inputs.particle_cloud(cfg, N, 4)
    _, ys = inputs.simulate(cfg, T=3)
    a = pfb.ParticleFilter(p, N, M, 9, airpf=1)
    b = pfb.ParticleFilter(p, N, M, 9, airpf=1, theta=1.0)
    for f in (a, b):
        f.set_state(x, 1)
    for n, y in enumerate(ys):
        a.step(y)
        b.step(y)
        assert np.array_equal(a.estimate(), b.estimate())
        assert np.array_equal(a.debug_get(pfb.PF_DBG_XHAT), b.debug_get(pfb.PF_DBG_XHAT))
    a.close()
    b.close()


def test_airpf2_filter_vs_kalman():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, N, M = 32, 1024, 64
    runs, stages = [], []
    for j in range(J):
        f = pfb.ParticleFilter(p, N, M, 300 + j, airpf=1, theta=0.5)
        mean = []
        for y in ys:
            f.step(y)
            mean.append(f.estimate()[0])
            stages.append(f.last_stages())
        f.close()
        runs.append(mean)
    runs = np.array(runs)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)
    assert np.mean(stages) < 4
