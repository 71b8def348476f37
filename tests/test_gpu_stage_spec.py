"""The compile-time plan instances against the runtime-plan kernels they replace for the
benchmark plans: k_stages_wsc (the warp-specialised stage pass with K and b = log2 M fixed,
pf_stages.cuh) against k_stages_ws, and k_pass1c (the fused pass 1 with B, K1 and the quads
per thread fixed, pf_pass1c.cuh) against k_pass1.  The same draws and compositions must
give BITWISE the same resampled particles and estimates over several steps, the first one
without mutation (PF_STAGE_SPEC=0 / PF_PASS1_SPEC=0 force the runtime-plan kernels).
Both are also compared with the fp64 oracle at full size in tests/test_gpu_fullsize.py,
which runs the bench launch configuration (the specialised kernel for C4)."""
import os

import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import pf as pfb  # noqa: E402


def _run(name, N, M, spec, T=3, **kw):
    """spec: 0 runtime-plan kernels, 1 compile-time instances."""
    os.environ["PF_STAGE_SPEC"] = str(int(spec))
    os.environ["PF_PASS1_SPEC"] = "1" if spec else "0"
    try:
        cfg = inputs.CONFIGS[name]
        p = inputs.model_params(cfg)
        _, ys = inputs.simulate(cfg, T=T)
        f = pfb.ParticleFilter(p, N, M, 11, **kw)
        est = []
        for t in range(T):
            f.step(np.asarray(ys[t], np.float32))
            est.append(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER))
            est.append(f.estimate(pfb.PF_PHI_X2, pfb.PF_EST_PREDICT))
            est.append(f.estimate(pfb.PF_PHI_X, pfb.PF_EST_RESAMPLED))
        torch.cuda.synchronize()
        x = f.debug_get(pfb.PF_DBG_XHAT)
        f.close()
        return x, np.concatenate(est)
    finally:
        os.environ.pop("PF_STAGE_SPEC", None)
        os.environ.pop("PF_PASS1_SPEC", None)


# (config, N, M): plans with compile-time instances -- C4 (k_pass1c B = 6, K1 = 4; k_stages_wsc
# K = 6 or 5, b = 6; one CTA wave and several tiles per CTA), C2 (k_stages_wsc K = 3 and 2, b = 8,
# d = 8), C3 at full size (k_pass1c SV, B = 5, K1 = 6; k_stages_wsc K = 7 and 6, b = 5)
@pytest.mark.parametrize("spec", [1])
@pytest.mark.parametrize("name,N,M", [("C4", 1 << 16, 64), ("C4", 1 << 20, 64), ("C4", 1 << 22, 64),
                                      ("C2", 1 << 18, 256), ("C3", 1 << 24, 32)])
def test_spec_equals_generic(name, N, M, spec):
    xa, ea = _run(name, N, M, spec)
    xb, eb = _run(name, N, M, 0)
    assert np.isfinite(xa).all()
    assert np.array_equal(xa, xb)
    assert np.array_equal(ea, eb)


@pytest.mark.parametrize("spec", [1])
def test_spec_equals_generic_rotation(spec):
    """The fully adapted scheme with stage rotation (theta = 1: every stage, the last pass
    writes the next layout through out_rot)."""
    xa, ea = _run("C4", 1 << 16, 64, spec, theta=1.0, rotate=True)
    xb, eb = _run("C4", 1 << 16, 64, 0, theta=1.0, rotate=True)
    assert np.array_equal(xa, xb)
    assert np.array_equal(ea, eb)


@pytest.mark.parametrize("kw", [{"airpf": 1}, {"airpf": 2}, {"airpf": 1, "theta": 0.5}])
def test_spec_equals_generic_airpf(kw):
    """k_pass1c's AIRPF instance (Alg. 7 / Alg. 6, and AIRPF2 with carried island weights)
    against k_pass1's AIRPF mode: the within-resampled sample, the island map (through the
    resampled estimate) and every estimate, bitwise, over four steps."""
    xa, ea = _run("C4", 1 << 18, 64, 1, T=4, **kw)
    xb, eb = _run("C4", 1 << 18, 64, 0, T=4, **kw)
    assert np.isfinite(xa).all()
    assert np.array_equal(xa, xb)
    assert np.array_equal(ea, eb)


@pytest.mark.parametrize("kw", [{"theta": 0.5}, {"theta": 0.9}, {"theta": 0.5, "rotate": True}])
def test_spec_equals_generic_adaptive(kw):
    """k_pass1c's weigh and resample instances (the two halves of a fully adapted step, with
    early stops S* < K1 that draw fewer stages of the same tile, carried weights of both kinds
    and stage rotation) against k_pass1's modes, bitwise, over six steps."""
    xa, ea = _run("C4", 1 << 18, 64, 1, T=6, **kw)
    xb, eb = _run("C4", 1 << 18, 64, 0, T=6, **kw)
    assert np.isfinite(xa).all()
    assert np.array_equal(xa, xb)
    assert np.array_equal(ea, eb)
