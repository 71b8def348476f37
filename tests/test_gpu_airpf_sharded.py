"""Sharded AIRPF (reading R27; include/pf.h pf_island_map / pf_island_cross): G
shards on one GPU through the loopback transport (island maps exchanged per cross stage,
blocks read from their owners through peer pointers) must reproduce the one-GPU AIRPF step
BITWISE -- island maps (global block ids), the materialised x_hat, the estimates and every
stage's island choices -- over several steps (so the next step's block reads cross shards),
for Alg. 7 and Alg. 6.  The one-GPU AIRPF step is itself parity-tested against the oracle
(tests/test_gpu_airpf.py)."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import dist as pfd  # noqa: E402
from paper_1812_01502_b200 import pf as pfb  # noqa: E402


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name,N,M,G", [("C4", 1 << 16, 64, 2), ("C4", 1 << 15, 16, 4), ("C3", 1 << 15, 32, 8),
                                        ("C1", 1024, 16, 4)])
def test_sharded_airpf_is_bitwise_one_gpu(name, N, M, G, mode):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=4)
    m = N // M
    S = int(np.log2(m))
    single = pfb.ParticleFilter(p, N, M, 23, debug=True, airpf=mode)
    shards = [pfd.LibBackend(p, N, M, 23, r, G, debug=True, airpf=mode) for r in range(G)]
    mloc = m // G
    for n, y in enumerate(ys):
        single.step(y)
        pfd.loopback_step(shards, y, exchange="island")
        for kind in (pfb.PF_EST_FILTER, pfb.PF_EST_PREDICT):
            e1 = single.estimate(pfb.PF_PHI_X, kind)
            for b in shards:
                assert np.array_equal(b.estimate(pfb.PF_PHI_X, kind), e1), (n, kind)
        A1 = single.debug_get(pfb.PF_DBG_ISLAND_A)
        Ag = np.concatenate([b.island_map().cpu().numpy() for b in shards])
        assert np.array_equal(A1, Ag), n
        for s in range(1, S + 1):
            c1 = single.debug_get(pfb.PF_DBG_ISLAND_CHOICE, s)
            cg = np.concatenate([_choice(b, s, mloc) for b in shards])
            assert np.array_equal(c1, cg), (n, s)
        x1 = single.debug_get(pfb.PF_DBG_XHAT)
        xg = np.concatenate([_xhat(b) for b in shards])
        assert np.array_equal(x1.reshape(xg.shape), xg), n
    single.close()
    for b in shards:
        b.close()


def _choice(b, s, mloc):
    ptr = b.pf.pf_debug_ptr(b.h, pfb.PF_DBG_ISLAND_CHOICE, s)
    t = b._view(ptr, (mloc + 3) // 4, torch.uint8)
    b.stream.synchronize()
    return t.cpu().numpy()


def _xhat(b):
    ptr = b.pf.pf_debug_ptr(b.h, pfb.PF_DBG_XHAT, 0)
    nloc = b.N // b.world
    t = b._view(ptr, nloc * b.d * 4, torch.float32).view(nloc, b.d)
    b.stream.synchronize()
    return t.cpu().numpy()


def test_sharded_airpf_needs_peers_and_top():
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    shards = [pfd.LibBackend(p, 1 << 12, 16, 1, r, 2, airpf=1) for r in range(2)]
    _, ys = inputs.simulate(cfg, T=2)
    recs = [b.step_local(ys[0]) for b in shards]
    with pytest.raises(pfb.PFError):  # before pf_step_top
        shards[0].island_cross(1, shards[1].island_map())
    for b in shards:
        b.step_top(torch.stack(recs))
    maps = [b.island_map().clone() for b in shards]
    for r, b in enumerate(shards):
        b.island_cross(1, maps[1 - r])
    with pytest.raises(pfb.PFError):  # the next step reads remote blocks: no peer mapping yet
        shards[0].step_local(ys[1])
    for b in shards:
        b.close()
    with pytest.raises(pfb.PFError):  # m / world not a multiple of 4
        pfd.LibBackend(p, 1 << 8, 16, 1, 0, 8, airpf=1)
