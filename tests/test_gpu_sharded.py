"""Sharded step on one GPU through the loopback transport: G = 2, 4 shards must reproduce
the single-GPU run BITWISE (counter-based draws on global indices, shard-aligned V and
estimate trees) -- resampled particles, every stage's ancestor table and the estimates."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import dist as pfd  # noqa: E402
from paper_1812_01502_b200 import pf as pfb  # noqa: E402


@pytest.mark.parametrize("exchange", ["pairwise", "pull", "peer"])
@pytest.mark.parametrize("name,N,M,G", [("C4", 1 << 16, 64, 2), ("C4", 1 << 16, 64, 4), ("C3", 1 << 15, 32, 4),
                                        ("C2", 1 << 15, 256, 2), ("C3", 1 << 12, 2, 8), ("C1", 1024, 64, 8)])
def test_loopback_matches_single_gpu(name, N, M, G, exchange):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=3)
    S = int(np.log2(N // M))
    single = pfb.ParticleFilter(p, N, M, 21, debug=True)
    shards = [pfd.LibBackend(p, N, M, 21, r, G, debug=True) for r in range(G)]
    for n, y in enumerate(ys):
        single.step(y)
        pfd.loopback_step(shards, y, exchange=exchange)
        for phi in (pfb.PF_PHI_X, pfb.PF_PHI_X2):
            for kind in (pfb.PF_EST_FILTER, pfb.PF_EST_PREDICT):
                e1 = single.estimate(phi, kind)
                for b in shards:
                    assert np.array_equal(b.estimate(phi, kind), e1), (n, phi, kind)
        xs = single.debug_get(pfb.PF_DBG_XHAT)
        xg = np.concatenate([b.debug_get(pfb.PF_DBG_XHAT) for b in shards])
        assert np.array_equal(xs.reshape(xg.shape), xg), n
        for s in range(1, S + 1):
            a1 = single.debug_get(pfb.PF_DBG_ANC_STAGE, s)
            ag = np.concatenate([b.debug_get(pfb.PF_DBG_ANC_STAGE, s) for b in shards])
            assert np.array_equal(a1, ag), (n, s)
    single.close()
    for b in shards:
        b.close()


def test_peer_exchange_errors():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    N, M, G = 1024, 16, 2
    shards = [pfd.LibBackend(p, N, M, 3, r, G) for r in range(G)]
    _, ys = inputs.simulate(cfg, T=1)
    recs = [b.step_local(ys[0]) for b in shards]
    allr = torch.stack(recs)
    for b in shards:
        b.step_top(allr)
    with pytest.raises(pfb.PFError):  # no mapping yet
        shards[0].cross_peer()
    with pytest.raises(pfb.PFError):  # [rank] must be the own workspace
        shards[0].peer_set([shards[1].ws_ptr, shards[1].ws_ptr])
    with pytest.raises(pfb.PFError):  # NULL peer
        shards[0].peer_set([shards[0].ws_ptr, 0])
    pfd.loopback_peer(shards)  # now mapped: runs
    single = pfb.ParticleFilter(p, N, M, 3)
    with pytest.raises(pfb.PFError):  # not a sharded handle
        pfb._check(pfb.lib().pf_cross_peer(single.h), single.h)
    single.close()
    for b in shards:
        b.close()


@pytest.mark.parametrize("exchange", ["pairwise", "pull", "peer"])
@pytest.mark.parametrize("name,N,M,G,n", [("C4", 1 << 15, 64, 4, 1), ("C3", 1 << 14, 32, 8, 3),
                                          ("C2", 1 << 14, 256, 2, 2), ("C1", 1024, 16, 8, 0)])
def test_shards_match_oracle(orc, name, N, M, G, n, exchange):
    """Every shard against the fp64 oracle (not only against the one-GPU CUDA path): the
    shards start from slices of one seeded cloud; each stage's ancestor table (local
    stages from k_pass1 / k_stages, cross stages from k_cross / k_pull_compose /
    k_peer_gather) is bit-exact wherever the oracle's draw is >= 1e-6 from its boundary,
    x_hat matches on outputs whose path holds no flagged draw, estimates within R15."""
    from . import parity_util as pu
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    d = int(p["d"])
    S = int(np.log2(N // M))
    xin = inputs.particle_cloud(cfg, N, 31).reshape(N, d)
    y = inputs.observation_for_step(cfg, 40 + n)
    o = orc.step(p, N, M, 77, n, y, xin)
    nloc = N // G
    shards = [pfd.LibBackend(p, N, M, 77, r, G, debug=True) for r in range(G)]
    for r, b in enumerate(shards):
        b.set_state(xin[r * nloc:(r + 1) * nloc], n)
    pfd.loopback_step(shards, y, exchange=exchange)
    a = np.stack([np.concatenate([b.debug_get(pfb.PF_DBG_ANC_STAGE, s) for b in shards]) for s in range(1, S + 1)])
    pu.check_stage_tables(a, o["a"], o["delta"])
    flagged = pu.path_flags(o["a"], o["delta"])
    xg = np.concatenate([b.debug_get(pfb.PF_DBG_XHAT) for b in shards]).reshape(N, d)
    pu.check_x(xg[~flagged], o["xhat"][~flagged])
    for b in shards:
        pu.check_estimate(b.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER), o["filter"][:d], o["filter"][d:])
        pu.check_estimate(b.estimate(pfb.PF_PHI_X, pfb.PF_EST_PREDICT), o["predict"][:d], o["predict"][d:])
        b.close()
    assert flagged.mean() < 0.05
