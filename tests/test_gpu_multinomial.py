"""GPU <-> oracle parity of one plain BPF step (Alg. 1 with Alg. 2, multinomial
resampling over the whole population; reading R22) through the C-ABI
(pf_set_multinomial): x_n, the log-weights, the drawn ancestors (bit-exact wherever the
oracle's uniform is >= 1e-6 from a CDF boundary), x_hat = x[a] and the estimates; and the
GPU plain BPF against the Kalman means.
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


@pytest.mark.parametrize("cfg_name,N,M,n", [("C1", 1024, 64, 1), ("C4", 1 << 16, 64, 2), ("C3", 1 << 18, 32, 3),
                                            ("C2", 1 << 14, 256, 1), ("C1", 8, 4, 0), ("C4", 1 << 12, 16, 4)])
def test_multinomial_step_parity(orc, cfg_name, N, M, n):
    cfg = inputs.CONFIGS[cfg_name]
    params = inputs.model_params(cfg)
    d = int(params["d"])
    xhat = inputs.particle_cloud(cfg, N, 50 + n)
    y = inputs.observation_for_step(cfg, 70 + n, outlier_sigma=1.0)
    o = orc.step_multinomial(params, N, 21, n, y, xhat)
    f = pfb.ParticleFilter(params, N, M, 21, debug=True, multinomial=True)
    f.set_state(xhat, n)
    f.step(y)
    x = f.debug_get(pfb.PF_DBG_X)
    lw = f.debug_get(pfb.PF_DBG_LOGW)
    a = f.debug_get(pfb.PF_DBG_ANC_FINAL)
    xh = f.debug_get(pfb.PF_DBG_XHAT)
    filt, pred = f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT)
    f.close()
    pu.check_x(x, o["x"])
    pu.check_lw(lw, o["lw"])
    ok = o["delta"] >= pu.BOUNDARY
    bad = np.nonzero(ok & (a != o["a"]))[0]
    assert bad.size == 0, f"{bad.size} unflagged ancestor mismatches"
    assert np.array_equal(xh.reshape(N, d), x.reshape(N, d)[a])
    pu.check_estimate(filt, o["filter"][:d], o["filter"][d:])
    pu.check_estimate(pred, o["predict"][:d], o["predict"][d:])


def test_plain_bpf_gpu_vs_kalman():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J, N, M = 32, 1024, 64
    runs = []
    for j in range(J):
        f = pfb.ParticleFilter(p, N, M, 1300 + j, multinomial=True)
        mean = []
        for y in ys:
            f.step(y)
            mean.append(f.estimate()[0])
        f.close()
        runs.append(mean)
    runs = np.array(runs)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    assert np.all(np.abs(runs.mean(axis=0) - km[:, 0]) < 5 * se + 1e-6)


def test_one_scheme_at_a_time():
    p = inputs.model_params(inputs.CONFIGS["C1"])
    f = pfb.ParticleFilter(p, 1024, 64, 1, multinomial=True)
    with pytest.raises(pfb.PFError):
        pfb.pf_set_adaptive(f.h, 0.5)
    pfb.pf_set_multinomial(f.h, False)
    f.step(np.array([0.2], np.float32))
    assert f.last_stages() == f.S
    f.close()
