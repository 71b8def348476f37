"""Per-step host overhead on the small configurations: T steps through the binding one
call per step (pf_step_dev) vs one pf_run_dev call; device time per step (CUDA events).
python tools/run_dev_bench.py [T]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_01502_b200 import inputs, pf  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for name in ("C1", "C2", "C3"):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg)
    y = torch.tensor(np.asarray([ys[k % len(ys)] for k in range(T)], np.float32), device="cuda")
    res = {}
    for mode in ("step_dev", "run_dev"):
        f = pf.ParticleFilter(p, cfg.N, cfg.M, 1)
        f.run_dev(y[:5])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(f.stream)
        if mode == "step_dev":
            for k in range(T):
                f.step_dev(y[k])
        else:
            f.run_dev(y, estimates=True)
        e1.record(f.stream)
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / T
        f.close()
    print(f"{name} N={cfg.N} M={cfg.M}: ms/step step_dev {res['step_dev']:.4f}  run_dev {res['run_dev']:.4f}  "
          f"({cfg.N / res['run_dev'] / 1e6:.3g}e9 particle-steps/s with run_dev)")
