"""C5 (BASELINE.json): group-size sweep at fixed N = 2^26 of the 1-D stochastic-volatility
model, T = 20 -- throughput and the RMSE of the filter means against a 2^28-particle
reference (mean of 4 independent runs, M = 64; SURVEY.md reading A16).

    python tools/c5_sweep.py [J] > profiles/r1_c5_sweep.json
J independent seeds per M (default 4).  Plain augmented resampling and AIRPF (M >= 4)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_01502_b200 import inputs, pf  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = inputs.CONFIGS["C5"]
p = inputs.model_params(cfg)
_, ys = inputs.simulate(cfg)
T = len(ys)


def run(N, M, seed, **kw):
    f = pf.ParticleFilter(p, N, M, seed, **kw)
    means = np.zeros(T)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(f.stream)
    for n, y in enumerate(ys):
        f.step(y)
        means[n] = f.estimate()[0]  # synchronises: the timing includes the D2H of the estimate
    e1.record(f.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / T
    f.close()
    return means, ms


ref = np.mean([run(1 << 28, 64, 9000 + k)[0] for k in range(4)], axis=0)
out = {"config": "C5", "N": inputs.C5_N, "T": T, "J": J, "reference": "mean of 4 runs, N = 2^28, M = 64",
       "rows": []}
for M in inputs.C5_SWEEP_M:
    for alg, kw in (("augmented", {}), ("airpf", {"airpf": 1})):
        if alg == "airpf" and M < 4:
            continue
        errs, mss = [], []
        for j in range(J):
            means, ms = run(inputs.C5_N, M, 100 + 17 * j + M, **kw)
            errs.append(means - ref)
            mss.append(ms)
        errs = np.array(errs)
        out["rows"].append({"M": M, "m": inputs.C5_N // M, "algorithm": alg,
                            "rmse": float(np.sqrt(np.mean(errs ** 2))),
                            "ms_per_step": float(np.median(mss)),
                            "particle_steps_per_s": inputs.C5_N / (float(np.median(mss)) / 1e3)})
print(json.dumps(out, indent=1))
