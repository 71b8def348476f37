"""Pins of the oracle's estimate legs (orc_estimates, oracle/pf_oracle.c), each against
something the mathematics fixes rather than a retyped formula:

* filter leg   pi_hat_n(phi) = sum_i g(x^i) phi(x^i) / sum_i g(x^i)
* predict leg  pi_n^N(phi)  = N^-1 sum_i phi(x^i)
* resampled    N^-1 sum_i phi(x_hat^i), x_hat^i = x^{A(i)}
for phi(x) = x and x^2.

Invariants: equal weights make the filter leg the predict leg; one live particle makes the
filter leg that particle (x and x^2); a common shift of the log-weights and a joint
permutation change nothing; the resampled leg with A = identity is the predict leg and
with A = const j is particle j.  Closed forms: the predict leg of a Gaussian sample is
within 5 standard errors of (mu, mu^2 + sigma^2).  Kalman: in the oracle filter the
predict leg targets the Kalman PRIOR (A m_{n-1}, A P A' + Q), the filter x^2 leg minus the
squared filter mean the Kalman POSTERIOR variance, and the resampled leg the posterior
mean (Prop. 1 unbiasedness) -- each within 5 Monte-Carlo standard errors over seeds."""
import numpy as np
import pytest

from oracle import kalman
from paper_1812_01502_b200 import inputs


def _cloud(N, d, seed):
    rng = np.random.default_rng(seed)
    return rng.normal(0.3, 1.7, size=(N, d)), rng.normal(0.0, 2.0, size=N)


def test_equal_weights_filter_is_predict(orc):
    x, _ = _cloud(4096, 4, 1)
    e = orc.estimates(4, np.full(4096, -3.25), x, None)
    assert np.allclose(e["filter"], e["predict"], rtol=1e-13, atol=0)


def test_single_live_particle(orc):
    x, lw = _cloud(257, 2, 2)
    lw[:] = -np.inf
    lw[131] = -40.0
    e = orc.estimates(2, lw, x, None)
    assert np.array_equal(e["filter"][:2], x[131])
    assert np.allclose(e["filter"][2:], x[131] ** 2, rtol=1e-15, atol=0)


def test_shift_and_permutation_invariance(orc):
    x, lw = _cloud(1000, 3, 3)
    e0 = orc.estimates(3, lw, x, None)
    e1 = orc.estimates(3, lw + 123.0, x, None)
    perm = np.random.default_rng(9).permutation(1000)
    e2 = orc.estimates(3, lw[perm], x[perm], None)
    for k in ("filter", "predict"):
        assert np.allclose(e0[k], e1[k], rtol=1e-12, atol=1e-14)
        assert np.allclose(e0[k], e2[k], rtol=1e-12, atol=1e-14)


def test_resampled_leg_special_maps(orc):
    x, lw = _cloud(512, 4, 4)
    e = orc.estimates(4, lw, x, np.arange(512))
    assert np.allclose(e["resampled"], e["predict"], rtol=1e-13, atol=0)
    e = orc.estimates(4, lw, x, np.full(512, 77))
    assert np.allclose(e["resampled"][:4], x[77], rtol=1e-12, atol=0)
    assert np.allclose(e["resampled"][4:], x[77] ** 2, rtol=1e-12, atol=0)


def test_predict_leg_gaussian_closed_form(orc):
    N, d = 1 << 16, 2
    rng = np.random.default_rng(5)
    mu, sig = np.array([1.5, -0.75]), np.array([0.5, 2.0])
    x = mu + sig * rng.standard_normal((N, d))
    e = orc.estimates(d, np.zeros(N), x, None)
    assert np.all(np.abs(e["predict"][:d] - mu) < 5 * sig / np.sqrt(N))
    m2 = mu ** 2 + sig ** 2
    sd2 = np.sqrt(4 * mu ** 2 * sig ** 2 + 2 * sig ** 4)  # sd of x^2 for a normal
    assert np.all(np.abs(e["predict"][d:] - m2) < 5 * sd2 / np.sqrt(N))


def _c1(T):
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=T)
    return cfg, p, ys


def test_legs_vs_kalman_prior_and_posterior(orc):
    """Oracle BPF (Alg. 1 + Alg. 3) on C1; per step n >= 1 and seed j collect all legs."""
    cfg, p, ys = _c1(T=8)
    A, Q = np.asarray(p["A"], np.float64), np.asarray(p["Q"], np.float64)
    km, kc = kalman.kalman_filter(p["A"], p["Q"], p["H"], p["R"], p["m0"], p["P0"], ys)
    M, m, J = 64, 16, 32
    N = M * m
    rec = {k: [] for k in ("f1", "f2", "p1", "p2", "r1")}
    for j in range(J):
        x = orc.init(p, N, 300 + j).astype(np.float32)
        rows = {k: [] for k in rec}
        for n, y in enumerate(ys):
            r = orc.step(p, N, M, 300 + j, n, y, x, tables=False)
            rows["f1"].append(r["filter"][0])
            rows["f2"].append(r["filter"][1])
            rows["p1"].append(r["predict"][0])
            rows["p2"].append(r["predict"][1])
            rows["r1"].append(r["resampled"][0])
            x = r["xhat"].astype(np.float32)
        for k in rec:
            rec[k].append(rows[k])
    R = {k: np.array(v) for k, v in rec.items()}  # J x T
    prior_m = np.concatenate([[float(np.asarray(p["m0"]).ravel()[0])], (A[0, 0] * km[:-1, 0])])
    prior_v = np.concatenate([[float(np.asarray(p["P0"]).ravel()[0])], A[0, 0] ** 2 * kc[:-1, 0, 0] + Q[0, 0]])

    def z(vals, target):
        se = vals.std(axis=0, ddof=1) / np.sqrt(J)
        return (vals.mean(axis=0) - target) / np.maximum(se, 1e-12)

    assert np.all(np.abs(z(R["p1"], prior_m)) < 5)               # predict x   -> prior mean
    assert np.all(np.abs(z(R["p2"] - R["p1"] ** 2, prior_v)) < 5)  # predict x^2 -> prior var (+ mean^2)
    assert np.all(np.abs(z(R["f2"] - R["f1"] ** 2, kc[:, 0, 0])) < 6)  # filter x^2 -> posterior var
    assert np.all(np.abs(z(R["r1"], km[:, 0])) < 5)              # resampled x -> posterior mean


@pytest.mark.parametrize("d", [1, 4])
def test_resampled_leg_unbiased(orc, d):
    """Prop. 1 (eq. aug_res_lack_of_bias): E[resampled | x, lw] = filter."""
    N, M = 256, 8
    x, lw = _cloud(N, d, 6)
    vals = []
    for seed in range(400):
        r = orc.augmented_resample(lw, M, seed, 0, tables=False)
        vals.append(orc.estimates(d, lw, x, r["A"])["resampled"])
    vals = np.array(vals)
    f = orc.estimates(d, lw, x, None)["filter"]
    se = vals.std(axis=0, ddof=1) / np.sqrt(len(vals))
    assert np.all(np.abs(vals.mean(axis=0) - f) < 5 * se)
