"""Small runs of every step variant for compute-sanitizer (SURVEY.md §4 tier T4):
python tools/sanitize_run.py <variant>, variant in plain, debug, adaptive, rotate, airpf1,
airpf2, multinomial, sharded-pairwise, sharded-pull, sharded-peer.  Each runs a few steps
at sizes that span several tiles and a ragged configuration mix (C1, C2, C3 with M = 2)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_01502_b200 import dist as pfd, inputs, pf  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "plain"
CASES = [("C1", 1024, 64), ("C2", 1 << 14, 256), ("C3", 1 << 13, 2), ("C4", 1 << 15, 64)]
for name, N, M in CASES:
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=3)
    if variant.startswith("sharded"):
        G = 2
        shards = [pfd.LibBackend(p, N, M, 5, r, G) for r in range(G)]
        for y in ys:
            pfd.loopback_step(shards, y, exchange=variant.split("-")[1])
        est = shards[0].estimate()
        for b in shards:
            b.close()
    else:
        kw = dict(debug=variant == "debug")
        if variant in ("adaptive", "rotate"):
            kw.update(theta=0.5, rotate=variant == "rotate")
        if variant.startswith("airpf"):
            kw.update(airpf=int(variant[-1]))
        if variant == "multinomial":
            kw.update(multinomial=True)
        f = pf.ParticleFilter(p, N, M, 5, **kw)
        for y in ys:
            f.step(y)
        est = f.estimate()
        f.close()
    torch.cuda.synchronize()
    print(variant, name, N, M, np.round(est, 4))
