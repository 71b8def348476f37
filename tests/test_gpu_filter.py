"""Whole-filter behaviour of the CUDA path through the public C-ABI (multi-step runs):
statistical agreement with the exact Kalman posterior mean, determinism, pf_step vs
pf_step_dev equivalence, error codes."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from oracle import kalman  # noqa: E402
from paper_1812_01502_b200 import pf as pfb  # noqa: E402


def _run(params, N, M, seed, ys, dev=False):
    f = pfb.ParticleFilter(params, N, M, seed)
    d = int(params["d"])
    means = np.zeros((len(ys), d))
    yd = torch.tensor(np.asarray(ys, np.float32), device="cuda")
    for n, y in enumerate(ys):
        if dev:
            f.step_dev(yd[n])
        else:
            f.step(y)
        means[n] = f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER)
    xhat = f.debug_get(pfb.PF_DBG_XHAT)
    f.close()
    return means, xhat


def test_c1_vs_kalman():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J = 32
    runs = np.array([_run(p, cfg.N, cfg.M, 500 + j, ys)[0][:, 0] for j in range(J)])
    mean = runs.mean(axis=0)
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    z = (mean - km[:, 0]) / se
    assert np.all(np.abs(z) < 5.0), z


@pytest.mark.parametrize("name,N,M", [("C4", 1 << 18, 64), ("C2", 1 << 16, 256)])
def test_lg_large_vs_kalman(name, N, M):
    """16 independent runs: the per-step filter mean of the runs within 5 standard errors
    (their spread) of the exact Kalman mean, every coordinate (as test_c1_vs_kalman)."""
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=20)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    J = 16
    runs = np.array([_run(p, N, M, 40 + j, ys)[0] for j in range(J)])  # J x T x d
    se = runs.std(axis=0, ddof=1) / np.sqrt(J)
    z = (runs.mean(axis=0) - km) / np.maximum(se, 1e-12)
    assert np.all(np.abs(z) < 5.0), np.abs(z).max()


def test_determinism_and_step_dev():
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=5)
    m1, x1 = _run(p, 1 << 16, 64, 9, ys)
    m2, x2 = _run(p, 1 << 16, 64, 9, ys)
    m3, x3 = _run(p, 1 << 16, 64, 9, ys, dev=True)
    assert np.array_equal(m1, m2) and np.array_equal(x1, x2)
    assert np.array_equal(m1, m3) and np.array_equal(x1, x3)
    m4, _ = _run(p, 1 << 16, 64, 10, ys)
    assert not np.array_equal(m1, m4)


def test_error_codes():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    f = pfb.ParticleFilter(p, 1024, 64, 1)
    with pytest.raises(pfb.PFError) as e:
        f.estimate()
    assert e.value.code == pfb.PF_ESTATE
    with pytest.raises(pfb.PFError) as e:
        f.step(np.array([np.nan], np.float32))
    assert e.value.code == pfb.PF_EOBS
    with pytest.raises(pfb.PFError) as e:
        f.debug_get(pfb.PF_DBG_X)
    assert e.value.code == pfb.PF_ESTATE
    f.step(np.array([0.3], np.float32))
    with pytest.raises(pfb.PFError) as e:
        f.debug_get(pfb.PF_DBG_X)  # not a debug handle
    assert e.value.code == pfb.PF_ESTATE
    f.close()
    with pytest.raises(pfb.PFError) as e:
        pfb.ParticleFilter(p, 1024, 1024, 1)  # m = 1
    assert e.value.code == pfb.PF_EINVAL


def test_init_distribution():
    """x_0 ~ pi_0: the predictive mean/second moment at n = 0 match the prior."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    N = 1 << 20
    f = pfb.ParticleFilter(p, N, 64, 4)
    f.step(np.zeros(4, np.float32))
    m1 = f.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT)
    m2 = f.estimate(pfb.PF_PHI_X2, pfb.PF_EST_PREDICT)
    f.close()
    assert np.all(np.abs(m1) < 5 / np.sqrt(N))
    assert np.all(np.abs(m2 - 1.0) < 5 * np.sqrt(2.0 / N))


def _rmse_end(params, ys, km, N, M, J, seed0, **kw):
    errs = []
    for j in range(J):
        f = pfb.ParticleFilter(params, N, M, seed0 + j, **kw)
        for y in ys:
            f.step(y)
        errs.append(f.estimate()[0] - km[-1, 0])
        f.close()
    return float(np.sqrt(np.mean(np.square(errs))))


def test_theorem1_rate_on_gpu():
    """Theorem 1 on the CUDA path: at fixed m the error of the filter
    mean decays as M^-1/2 (log-log slope -0.5 +- 0.1 over M = 16 .. 4096)."""
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=8)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    m = 16
    Ms = [16, 64, 256, 1024, 4096]
    rmse = [_rmse_end(p, ys, km, m * M, M, J=160, seed0=20000 + 1000 * i) for i, M in enumerate(Ms)]
    slope = np.polyfit(np.log(Ms), np.log(rmse), 1)[0]
    assert -0.6 < slope < -0.4, (slope, rmse)


@pytest.mark.parametrize("kw", [dict(airpf=1), dict(theta=0.5), dict(theta=0.5, rotate=True), dict(multinomial=True)])
def test_variant_rates_on_gpu(kw):
    """The next-row variants converge at the Monte Carlo rate too (fixed m, M = 64 .. 4096)."""
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=8)
    km, _ = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    m = 16
    Ms = [64, 512, 4096]
    rmse = [_rmse_end(p, ys, km, m * M, M, J=120, seed0=40000 + 1000 * i, **kw) for i, M in enumerate(Ms)]
    slope = np.polyfit(np.log(Ms), np.log(rmse), 1)[0]
    assert -0.65 < slope < -0.35, (kw, slope, rmse)


def test_c4_full_size_filter_vs_kalman():
    """The bench's workload end to end: C4 at N = 2^28 over its T = 50 observations through
    pf_step_dev (as bench.py), two independent runs.  Their difference estimates the Monte
    Carlo error: with rho^2 = mean over steps and coordinates of (a - b)^2 / (2 sd^2) (sd the
    Kalman posterior sd; the relative error of a stable filter has a step-independent
    scale), the mean of the two runs must lie within 6 rho sd / sqrt(2) of the Kalman mean at
    every (step, coordinate) -- 200 tests at 6 sigma."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg)
    km, kc = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    yd = torch.tensor(np.asarray(ys, np.float32), device="cuda")
    runs = []
    for seed in (1, 2):
        f = pfb.ParticleFilter(p, cfg.N, cfg.M, seed)
        means = np.zeros((len(ys), cfg.d))
        for n in range(len(ys)):
            f.step_dev(yd[n])
            means[n] = f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER)
        f.close()
        runs.append(means)
    a, b = runs
    sd = np.sqrt(np.diagonal(kc, axis1=1, axis2=2))
    rho = np.sqrt(np.mean((a - b) ** 2 / (2 * sd ** 2)))
    err = np.abs(0.5 * (a + b) - km) / sd
    assert np.all(err < 6 * rho / np.sqrt(2) + 1e-6), (err.max(), rho)
    # and the Monte Carlo scale itself is that of N = 2^28 particles: rho <= a few sqrt(S/N)
    S = np.log2(cfg.N // cfg.M)
    assert rho < 10 * np.sqrt(S / cfg.N), rho


@pytest.mark.parametrize("kw", [{}, {"theta": 0.5}, {"airpf": 1}, {"multinomial": True}])
def test_run_dev_equals_steps(kw):
    """pf_run_dev (T steps in one call) gives bitwise the per-step results."""
    cfg = inputs.CONFIGS["C2"]
    p = inputs.model_params(cfg)
    N, M = 1 << 16, 256
    _, ys = inputs.simulate(cfg, T=6)
    yd = torch.tensor(np.asarray(ys, np.float32), device="cuda")
    a = pfb.ParticleFilter(p, N, M, 9, **kw)
    b = pfb.ParticleFilter(p, N, M, 9, **kw)
    est = a.run_dev(yd).cpu().numpy()
    for n in range(len(ys)):
        b.step_dev(yd[n])
        want = [b.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), b.estimate(pfb.PF_PHI_X2, pfb.PF_EST_FILTER),
                b.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT), b.estimate(pfb.PF_PHI_X2, pfb.PF_EST_PREDICT)]
        assert np.array_equal(est[n], np.stack(want)), n
    assert np.array_equal(a.debug_get(pfb.PF_DBG_XHAT), b.debug_get(pfb.PF_DBG_XHAT))
    assert a.run_dev(yd[:0], estimates=False) is None  # T = 0: nothing to do
    a.close()
    b.close()
