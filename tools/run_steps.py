"""Run a few filter steps (for ncu / sanitizer captures): python tools/run_steps.py C4 N M steps"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_01502_b200 import inputs, pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = inputs.CONFIGS[name]
N = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.N
M = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.M
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
params = inputs.model_params(cfg)
_, ys = inputs.simulate(cfg, T=steps)
f = pf.ParticleFilter(params, N, M, 1)
for n in range(steps):
    f.step(ys[n])
print("mean", f.estimate())
f.close()
torch.cuda.synchronize()
