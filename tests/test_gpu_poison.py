"""Memory-safety checks without compute-sanitizer (closed on this GPU pool): every step
variant runs on workspaces pre-filled with different bytes (0x00, 0xFF = NaN patterns,
0x7F) and must give BITWISE the same estimates and particles -- a read of a workspace byte
the step never wrote would make the result depend on the fill -- and must leave untouched
the 4 KiB gaps PF_FLAG_GUARD puts after every workspace region (pf_guard_check: no kernel
writes outside its buffer) and a 64 KiB band behind the workspace.  Sizes span several
tiles, the smallest and largest M of the configs, and d = 1, 4, 8."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import dist as pfd  # noqa: E402
from paper_1812_01502_b200 import pf as pfb  # noqa: E402

CASES = [("C1", 1024, 64), ("C2", 1 << 14, 256), ("C3", 1 << 13, 2), ("C4", 1 << 15, 64), ("C3", 1 << 15, 8192),
         ("C4", 1 << 22, 64)]
VARIANTS = ["plain", "debug", "adaptive", "rotate", "airpf1", "airpf2", "multinomial"]
FILLS = (0x00, 0xFF, 0x7F)


def _kw(variant):
    kw = dict(debug=variant == "debug")
    if variant in ("adaptive", "rotate"):
        kw.update(theta=0.5, rotate=variant == "rotate")
    if variant.startswith("airpf"):
        kw.update(airpf=int(variant[-1]))
    if variant == "multinomial":
        kw.update(multinomial=True)
    return kw


def _run(variant, name, N, M, fill):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=3)
    f = pfb.ParticleFilter(p, N, M, 8, poison=fill, **_kw(variant))
    out = []
    for y in ys:
        f.step(y)
        out.append(np.concatenate([f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER),
                                   f.estimate(pfb.PF_PHI_X2, pfb.PF_EST_PREDICT)]))
    if variant == "debug":
        out.append(f.debug_get(pfb.PF_DBG_XHAT).ravel())
        out.append(f.debug_get(pfb.PF_DBG_ANC_FINAL).astype(np.float64))
    ok = f.guard_intact()
    f.close()
    return out, ok


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name,N,M", CASES)
def test_fill_independent_and_guard(variant, name, N, M):
    if M < 4 and (variant == "rotate" or variant.startswith("airpf")):  # include/pf.h: needs M >= 4
        with pytest.raises(pfb.PFError):
            _run(variant, name, N, M, 0)
        return
    ref = None
    for fill in FILLS:
        out, ok = _run(variant, name, N, M, fill)
        assert ok, f"write past the workspace (fill {fill:#x})"
        if ref is None:
            ref = out
            assert all(np.all(np.isfinite(o)) for o in out[:3])
            continue
        for a, b in zip(ref, out):
            assert np.array_equal(a, b), f"result depends on the workspace fill ({fill:#x})"


@pytest.mark.parametrize("exchange", ["pairwise", "pull", "peer"])
@pytest.mark.parametrize("name,N,M", CASES[:4] + CASES[5:])
def test_sharded_fill_independent_and_guard(exchange, name, N, M):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=3)
    ref = None
    for fill in FILLS:
        shards = [pfd.LibBackend(p, N, M, 8, r, 2, poison=fill) for r in range(2)]
        out = []
        for y in ys:
            pfd.loopback_step(shards, y, exchange=exchange)
            out.append(shards[0].estimate())
        assert all(b.guard_intact() for b in shards), f"write past a shard workspace (fill {fill:#x})"
        for b in shards:
            b.close()
        if ref is None:
            ref = out
            continue
        for a, b in zip(ref, out):
            assert np.array_equal(a, b), f"sharded result depends on the workspace fill ({fill:#x})"


def test_guard_check_detects_a_stray_write():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    f = pfb.ParticleFilter(p, 1024, 64, 8, poison=0x5A)
    f.step(np.array([0.3], np.float32))
    assert f.guard_intact()
    xb = 1024 * 1 * 4  # X0 is the first region (N x d fp32); its gap follows it
    f.ws[f._off + xb + 17] = 0x00
    assert not f.guard_intact()
    bad = np.zeros(1, np.uint64)
    pfb._check(pfb.lib().pf_guard_check(f.h, 0x5A, bad.ctypes.data), f.h)
    assert int(bad[0]) == 1
    f.close()
    g = pfb.ParticleFilter(p, 1024, 64, 8)
    with pytest.raises(pfb.PFError):  # no PF_FLAG_GUARD
        pfb._check(pfb.lib().pf_guard_check(g.h, 0, bad.ctypes.data), g.h)
    g.close()
