"""pf_graph_capture / pf_graph_launch: T steps captured into one CUDA graph give bitwise the
eager steps' estimates and resampled particles (same kernels, same order); the handle
refuses to step while a captured graph is pending; the adaptive scheme is refused."""
import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import pf as pfb  # noqa: E402


@pytest.mark.parametrize("name,N,M,kw", [("C1", 1024, 64, {}), ("C3", 1 << 14, 32, {}), ("C4", 1 << 14, 16, {"airpf": 1}),
                                         ("C1", 1024, 64, {"multinomial": True})])
def test_graph_equals_eager(name, N, M, kw):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=12)
    yd = torch.tensor(np.asarray(ys, np.float32), device="cuda")
    st = torch.cuda.Stream()  # capture needs a non-default stream
    a = pfb.ParticleFilter(p, N, M, 5, **kw)
    est_a = a.run_dev(yd)
    b = pfb.ParticleFilter(p, N, M, 5, stream=st, **kw)
    est_b = b.graph_capture(yd, estimates=True)
    with pytest.raises(pfb.PFError):  # pending graph: no other step
        b.step(ys[0])
    b.graph_launch()
    torch.cuda.synchronize()
    c = pfb.ParticleFilter(p, N, M, 5, **kw)  # the legacy default stream cannot be captured
    with pytest.raises(pfb.PFError):
        c.graph_capture(yd)
    c.close()
    assert torch.equal(est_a, est_b)
    assert np.array_equal(a.debug_get(pfb.PF_DBG_XHAT), b.debug_get(pfb.PF_DBG_XHAT))
    b.step(ys[0])  # usable again
    a.close()
    b.close()


def test_graph_refuses_adaptive():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    f = pfb.ParticleFilter(p, 1024, 64, 1, theta=0.5, stream=torch.cuda.Stream())
    yd = torch.zeros((3, 1), dtype=torch.float32, device="cuda")
    with pytest.raises(pfb.PFError):
        f.graph_capture(yd)
    with pytest.raises(pfb.PFError):
        f.graph_launch()  # nothing captured
    f.close()
