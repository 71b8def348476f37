"""GPU parity of the relabelled exchange (pf_relabel_begin / pf_relabel_end; DESIGN.md reading
R24) against the oracle's orc_step_relabel, through G shards on one GPU
(loopback transport: the partner's surplus buffer is handed over in place).

Compared: every local stage's table (bit-exact away from decision boundaries), every cross
stage's relabelled table and each shard's surplus count (exact for every shard pair whose
cross-stage draws are all >= 1e-6 from their boundaries: one flagged draw can shift the two
ordered lists of its pair), x_hat on outputs whose path crosses no flagged draw or
skipped pair, and the estimates.  The surplus that crosses shards is far below the plain
exchange's (1 - 1/G) of every shard."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import dist as pfd  # noqa: E402
from paper_1812_01502_b200 import pf as pfb  # noqa: E402

from . import parity_util as pu  # noqa: E402


def _run(orc, name, N, M, G, n, seed=41, outlier=0.0):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    d = int(p["d"])
    S = int(np.log2(N // M))
    L = G.bit_length() - 1
    xin = inputs.particle_cloud(cfg, N, 17 + n).reshape(N, d)
    y = inputs.observation_for_step(cfg, 50 + n, outlier_sigma=outlier)
    o = orc.step_relabel(p, N, M, G, seed, n, y, xin)
    nloc = N // G
    shards = [pfd.LibBackend(p, N, M, seed, r, G, debug=True) for r in range(G)]
    for r, b in enumerate(shards):
        b.set_state(xin[r * nloc:(r + 1) * nloc], n)
    pfd.loopback_step(shards, y, exchange="relabel")
    a = np.stack([np.concatenate([b.debug_get(pfb.PF_DBG_ANC_STAGE, s) for b in shards]) for s in range(1, S + 1)])
    xg = np.concatenate([b.debug_get(pfb.PF_DBG_XHAT) for b in shards]).reshape(N, d)
    surplus = np.stack([b.surplus for b in shards], axis=1)  # L x G states received
    est = [(b.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), b.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT)) for b in shards]
    for b in shards:
        b.close()
    # local stages: the plain Alg. 3 protocol
    pu.check_stage_tables(a[: S - L], o["a"][: S - L], o["delta"][: S - L])
    # cross stages: per shard pair, exact unless one of its draws is boundary-flagged
    bad = np.zeros((S, N), bool)  # (stage, position) whose table entry is not comparable
    skipped = 0
    for t in range(1, L + 1):
        s = S - L + t
        for r in range(G):
            if r & (1 << (t - 1)):
                continue
            rp = r | (1 << (t - 1))
            pos = np.r_[r * nloc:(r + 1) * nloc, rp * nloc:(rp + 1) * nloc]
            if (o["delta"][s - 1][pos] < pu.BOUNDARY).any():
                bad[s - 1][pos] = True
                skipped += 1
                continue
            assert np.array_equal(a[s - 1][pos], o["a"][s - 1][pos]), (t, r)
            assert surplus[t - 1][r] == o["excess"][t - 1][r] and surplus[t - 1][rp] == o["excess"][t - 1][rp], (t, r)
    # x_hat on outputs whose path holds no flagged draw and no skipped pair-stage
    flagged = pu.path_flags(o["a"], np.where(bad, 0.0, o["delta"]))
    pu.check_x(xg[~flagged], o["xhat"][~flagged])
    for f, pr in est:
        pu.check_estimate(f, o["filter"][:d], o["filter"][d:])
        pu.check_estimate(pr, o["predict"][:d], o["predict"][d:])
    return dict(surplus=surplus, skipped=skipped, flagged=int(flagged.sum()), nloc=nloc, L=L)


@pytest.mark.parametrize("name,N,M,G,n", [("C4", 1 << 15, 64, 2, 1), ("C4", 1 << 15, 64, 4, 2), ("C3", 1 << 14, 32, 8, 3),
                                          ("C2", 1 << 14, 256, 4, 1), ("C1", 1024, 16, 8, 0), ("C3", 1 << 12, 2, 4, 2)])
def test_relabel_matches_oracle(orc, name, N, M, G, n):
    r = _run(orc, name, N, M, G, n)
    assert r["skipped"] <= max(1, r["L"] * G // 4)


def test_relabel_outlier(orc):
    """Degenerate weights: one shard dominates, the surplus is large (the dissemination
    case of PAPER.md:568) and the exchange must still be exact."""
    _run(orc, "C4", 1 << 14, 64, 4, 2, outlier=6.0)


def test_relabel_moves_only_the_surplus(orc):
    """Balanced weights (equal-ish V): the states crossing a pair are O(sqrt(N/G)), the plain
    exchange moves ~ (1 - 1/G) N/G per shard."""
    cfg = inputs.CONFIGS["C4"]
    p = dict(inputs.model_params(cfg))
    p["Rinv"] = np.zeros_like(p["Rinv"])  # g = 1: p_s = 1/2 at every cross stage
    N, M, G = 1 << 18, 64, 8
    nloc = N // G
    shards = [pfd.LibBackend(p, N, M, 3, r, G) for r in range(G)]
    _, ys = inputs.simulate(cfg, T=2)
    for y in ys:
        pfd.loopback_step(shards, y, exchange="relabel")
    moved = np.stack([b.surplus for b in shards], axis=1).sum()  # states received over all stages
    for b in shards:
        b.close()
    assert moved / G < 8 * np.sqrt(nloc) * 3, moved
    assert moved < 0.05 * N
