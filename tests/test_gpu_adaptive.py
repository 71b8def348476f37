"""GPU <-> oracle parity of the fully adapted step (R17/R18)
through the C-ABI (pf_set_adaptive).

Both sides start from the same seeded cloud, seed, n, y and theta.  Compared: the ESS
levels E_0..E_S, the number of stages run S*, x_n, the log-weights (carried weight +
log g), every executed stage's ancestor table, the composed ancestors, x_hat and the
estimates.  theta is placed midway between two oracle ESS levels so that S* is not a
rounding decision (the GPU sums the level-0 ESS in fp32 per tile: ~1e-6 relative).
Two-step cases check the carried weights of both kinds (S* = 0: particle carry;
0 < S* < S: block carry).  theta = 1 must reproduce the plain GPU step bit for bit, and
the adaptive GPU filter must track the exact Kalman means.
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
    ss = f.last_stages()
    out = dict(ss=ss, ess=f.debug_get(pfb.PF_DBG_ESS), x=f.debug_get(pfb.PF_DBG_X), lw=f.debug_get(pfb.PF_DBG_LOGW),
               a=np.stack([f.debug_get(pfb.PF_DBG_ANC_STAGE, s) for s in range(1, ss + 1)]) if ss else None,
               A=f.debug_get(pfb.PF_DBG_ANC_FINAL), xhat=f.debug_get(pfb.PF_DBG_XHAT),
               logV=f.debug_get(pfb.PF_DBG_LOGV),
               filt=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), pred=f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT))
    return out


def _rotr(g, k, S):
    k %= S
    return ((g >> k) | (g << (S - k))) & ((1 << S) - 1) if k else g


def _check(g, o, N, d, M=None, rotate=False):
    assert g["ss"] == o["sstar"], (g["ss"], o["sstar"], g["ess"], o["ess"])
    assert np.allclose(g["ess"], o["ess"], rtol=2e-5, atol=0), (g["ess"], o["ess"])
    pu.check_x(g["x"], o["x"])
    pu.check_lw(g["lw"], o["lw"])
    pu.check_logV(g["logV"], o["logV"])
    ss = o["sstar"]
    if ss:
        pu.check_stage_tables(g["a"], o["a"][:ss], o["delta"][:ss])
        flagged = pu.path_flags(o["a"][:ss], o["delta"][:ss])
        pu.check_composed(g["A"], o["A"], flagged)
    else:
        flagged = np.zeros(N, bool)
        assert np.array_equal(g["A"], np.arange(N))
    xh = g["xhat"].reshape(N, d)
    if rotate and 1 <= ss < o["S"]:  # x_hat is in the next layout: group g -> rotr_S(g, S*)
        pos = np.arange(N)
        dst = np.array([_rotr(int(p // M), ss, o["S"]) for p in pos]) * M + pos % M
        xh = xh[dst]
    assert np.array_equal(xh, g["x"].reshape(N, d)[g["A"]], equal_nan=True)
    pu.check_estimate(g["filt"], o["filter"][:d], o["filter"][d:])
    pu.check_estimate(g["pred"], o["predict"][:d], o["predict"][d:])
    return int(flagged.sum())


def _theta_for(orc, params, N, M, seed, n, xhat, y, lwc, target):
    """A theta midway between E_{target-1} and E_target of the oracle (so S* = target when
    the levels are separated), or None when they are too close to decide robustly."""
    o = orc.step_adaptive(params, N, M, seed, n, y, xhat, lwc, 1.0)
    e = o["ess"]
    if target == 0:
        th = 0.5 * e[0]
        return th if e[0] > 1e-3 else None
    lo, hi = e[target - 1], e[target]
    if hi - lo < 1e-3:
        return None
    return 0.5 * (lo + hi)


CASES = [("C1", 1024, 64, 1), ("C1", 1024, 16, 2), ("C4", 1 << 16, 64, 3), ("C4", 1 << 14, 16, 5),
         ("C3", 1 << 16, 32, 2), ("C2", 1 << 16, 256, 1), ("C3", 1 << 14, 2, 3), ("C3", 1 << 15, 8192, 2)]


@pytest.mark.parametrize("cfg_name,N,M,n", CASES)
def test_adaptive_step_parity(orc, cfg_name, N, M, n):
    cfg = inputs.CONFIGS[cfg_name]
    params = inputs.model_params(cfg)
    d = int(params["d"])
    S = int(np.log2(N // M))
    xhat = inputs.particle_cloud(cfg, N, 17 + n)
    y = inputs.observation_for_step(cfg, 40 + n, outlier_sigma=2.0)
    done = 0
    for target in sorted({0, 1, S // 2, S - 1, S}):
        th = _theta_for(orc, params, N, M, 77, n, xhat, y, np.zeros(N), target)
        if th is None:
            continue
        o = orc.step_adaptive(params, N, M, 77, n, y, xhat, np.zeros(N), th)
        assert o["sstar"] == target
        f = pfb.ParticleFilter(params, N, M, 77, debug=True, theta=th)
        f.set_state(xhat, n)
        f.step(y)
        g = _snap(f, d)
        f.close()
        _check(g, o, N, d)
        done += 1
    assert done >= 2


@pytest.mark.parametrize("first_target", [0, 2])
def test_adaptive_two_steps_carry(orc, first_target):
    """Step 1 stops at S* = first_target (0: particle carry, 2: block carry); step 2 starts
    from each side's own result and must agree (no flagged path in step 1)."""
    cfg = inputs.CONFIGS["C4"]
    params = inputs.model_params(cfg)
    d, N, M, n = 4, 1 << 12, 16, 3
    S = int(np.log2(N // M))
    xhat = inputs.particle_cloud(cfg, N, 5)
    y1 = inputs.observation_for_step(cfg, 8, outlier_sigma=3.0)
    y2 = inputs.observation_for_step(cfg, 9, outlier_sigma=1.0)
    th = _theta_for(orc, params, N, M, 3, n, xhat, y1, np.zeros(N), first_target)
    assert th is not None
    o1 = orc.step_adaptive(params, N, M, 3, n, y1, xhat, np.zeros(N), th)
    assert o1["sstar"] == first_target < S
    f = pfb.ParticleFilter(params, N, M, 3, debug=True, theta=th)
    f.set_state(xhat, n)
    f.step(y1)
    g1 = _snap(f, d)
    flagged = _check(g1, o1, N, d)
    assert flagged == 0
    o2 = orc.step_adaptive(params, N, M, 3, n + 1, y2, o1["xhat"].astype(np.float32), o1["lwc"], th)
    f.step(y2)
    g2 = _snap(f, d)
    f.close()
    _check(g2, o2, N, d)


def test_theta_one_equals_plain_gpu_step():
    cfg = inputs.CONFIGS["C4"]
    params = inputs.model_params(cfg)
    N, M = 1 << 16, 64
    _, ys = inputs.simulate(cfg, T=4)
    fa = pfb.ParticleFilter(params, N, M, 21, debug=True, theta=1.0)
    fp = pfb.ParticleFilter(params, N, M, 21, debug=True)
    for y in ys:
        fa.step(y)
        fp.step(y)
        assert fa.last_stages() == fa.S
        assert np.array_equal(fa.debug_get(pfb.PF_DBG_XHAT), fp.debug_get(pfb.PF_DBG_XHAT))
        assert np.array_equal(fa.estimate(), fp.estimate())
    fa.close()
    fp.close()


def test_adaptive_filter_vs_kalman():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, N, M = 32, 1024, 64
    runs, stages = [], []
    for j in range(J):
        f = pfb.ParticleFilter(p, N, M, 500 + j, theta=0.5)
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
    assert min(stages) < 4 and max(stages) >= 1


def test_adaptive_errors():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    f = pfb.ParticleFilter(p, 1024, 64, 1)
    with pytest.raises(pfb.PFError):
        pfb.pf_set_adaptive(f.h, 0.5)  # no PF_FLAG_ADAPTIVE
    f.close()
    g = pfb.ParticleFilter(p, 1024, 64, 1, theta=0.5)
    with pytest.raises(pfb.PFError):
        pfb.pf_set_adaptive(g.h, 1.5)
    pfb.pf_set_adaptive(g.h, 0.0)  # back to the plain step
    g.step(np.array([0.1], np.float32))
    assert g.last_stages() == g.S
    g.close()


@pytest.mark.parametrize("target,cfg_name,N,M", [(2, "C4", 1 << 14, 16), (7, "C4", 1 << 16, 64), (3, "C1", 1024, 16)])
def test_rotation_two_steps(orc, target, cfg_name, N, M):
    """Stage rotation (R23): step 1 stops at S* = target and writes the next
    layout (k_pass1 for S* <= k1, the last k_stages pass otherwise); step 2 runs in that
    layout with the rotated block carry and must agree with the oracle's rotated run."""
    cfg = inputs.CONFIGS[cfg_name]
    params = inputs.model_params(cfg)
    d = int(params["d"])
    S = int(np.log2(N // M))
    xhat = inputs.particle_cloud(cfg, N, 12)
    y1 = inputs.observation_for_step(cfg, 21, outlier_sigma=2.5)
    y2 = inputs.observation_for_step(cfg, 22, outlier_sigma=1.0)
    th = _theta_for(orc, params, N, M, 4, 2, xhat, y1, np.zeros(N), target)
    assert th is not None
    o1 = orc.step_adaptive(params, N, M, 4, 2, y1, xhat, np.zeros(N), th, rotate=True)
    assert o1["sstar"] == target < S
    f = pfb.ParticleFilter(params, N, M, 4, debug=True, theta=th, rotate=True)
    f.set_state(xhat, 2)
    f.step(y1)
    g1 = _snap(f, d)
    assert f.rotation_offset() == target % S
    flagged = _check(g1, o1, N, d, M, rotate=True)
    if flagged:
        pytest.skip("a boundary draw in step 1: the two sides hold different particles")
    pu.check_x(g1["xhat"], o1["xhat"])  # same particles, same (next) layout
    o2 = orc.step_adaptive(params, N, M, 4, 3, y2, o1["xhat"].astype(np.float32), o1["lwc"], th, rotate=True)
    f.step(y2)
    g2 = _snap(f, d)
    f.close()
    _check(g2, o2, N, d, M, rotate=True)
