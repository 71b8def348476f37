"""A0 parity: x_0 ~ pi_0 (Alg. 1 l.1-3) from k_init against the oracle's
orc_init, element by element (|x_gpu - x_orc| <= 1e-5 (1 + |x_orc|), tests/parity_util.py).

Both sides draw the INIT field of the draw contract (flat coordinate
c = i d + k is normal (c mod 4) of Philox block (c / 4, 0, INIT<<24)); the GPU's x_0 is read
back through PF_DBG_XHAT before any step.  Sharded handles (pos0 != 0) must produce the
slice [pos0, pos0 + N/G) of the one-GPU x_0."""
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


@pytest.mark.parametrize("name,N,M,seed", [("C1", 1024, 64, 7), ("C4", 1 << 16, 64, 11), ("C3", 1 << 14, 32, 5),
                                           ("C2", 1 << 14, 256, 3), ("C1", 4, 2, 1)])
def test_init_matches_oracle(orc, name, N, M, seed):
    p = inputs.model_params(inputs.CONFIGS[name])
    d = int(p["d"])
    f = pfb.ParticleFilter(p, N, M, seed)
    x0 = f.debug_get(pfb.PF_DBG_XHAT).reshape(N, d)
    f.close()
    pu.check_x(x0, orc.init(p, N, seed))


def test_init_full_size_c4_sampled(orc):
    """C4 at N = 2^28 (bench.py's handle): sampled rows, tile and end edges included."""
    cfg = inputs.CONFIGS["C4"]
    p = inputs.model_params(cfg)
    f = pfb.ParticleFilter(p, cfg.N, cfg.M, 1)
    x0 = f.debug_tensor(pfb.PF_DBG_XHAT)
    rng = np.random.default_rng(4)
    rows = np.unique(np.concatenate([rng.integers(0, cfg.N, 4096), [0, 1, 2, 3, 1023, 1024, cfg.N - 4, cfg.N - 1]]))
    got = x0[torch.as_tensor(rows, device=x0.device)].cpu().numpy()
    f.close()
    pu.check_x(got, orc.init_rows(p, 1, rows))


@pytest.mark.parametrize("name,N,M,G", [("C4", 1 << 14, 64, 2), ("C3", 1 << 12, 32, 4), ("C1", 1024, 64, 8)])
def test_init_sharded_slices(orc, name, N, M, G):
    p = inputs.model_params(inputs.CONFIGS[name])
    d = int(p["d"])
    xo = orc.init(p, N, 9)
    nloc = N // G
    for r in range(G):
        b = pfd.LibBackend(p, N, M, 9, r, G)
        x0 = b.debug_get(pfb.PF_DBG_XHAT).reshape(nloc, d)
        b.close()
        pu.check_x(x0, xo[r * nloc:(r + 1) * nloc])
