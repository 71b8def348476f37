"""Projection of the sharded step on one GPU: G shards of a configuration run back to back
through the loopback transport (python tools/loopback_bench.py C4 8 [pull|pairwise|peer] [steps]).
Reports the device time per step summed over the shards, per kernel kind, and the bytes the
exchange would move between GPUs; a projection only (no NVLink, shards serialised).
Modes: pull, pairwise, peer, relabel (the relabelled exchange: only the surplus crosses; its
bytes are counted from the surplus every shard received)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_01502_b200 import dist as pfd, inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
mode = sys.argv[3] if len(sys.argv) > 3 else "pull"
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
cfg = inputs.CONFIGS[name]
p = inputs.model_params(cfg)
_, ys = inputs.simulate(cfg, T=steps + 2)
shards = [pfd.LibBackend(p, cfg.N, cfg.M, 3, r, G) for r in range(G)]
for n in range(2):
    pfd.loopback_step(shards, ys[n], exchange=mode)
torch.cuda.synchronize()
for b in shards:
    b.timing_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for n in range(2, 2 + steps):
    pfd.loopback_step(shards, ys[n], exchange=mode)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
kt = {}
for b in shards:
    for k, (t, c) in b.timing_read().items():
        a = kt.setdefault(k, [0.0, 0])
        a[0] += t / steps
        a[1] += c
state = 4 * cfg.d
moved = cfg.N * state * (1 - 1 / G) / G  # per rank, pull: states read from other shards
if mode == "relabel":
    sur = np.stack([b.surplus for b in shards], axis=1)  # L x G states received (last step)
    moved = float(sur.sum(axis=0).max()) * state           # the busiest rank
    print(f"relabel surplus per stage and rank (states): {sur.tolist()}; sqrt(N/G) = {np.sqrt(cfg.N / G):.0f}")
print(f"{name} G={G} {mode}: {ms:.3f} ms per step for all {G} shards on one GPU "
      f"({ms / G:.3f} ms per shard); per kernel kind (ms per step, all shards): "
      + ", ".join(f"{k} {v[0]:.3f}" for k, v in kt.items() if v[1]))
print(f"exchange per rank per step: pull ~{moved / 1e9:.3f} GB states + {cfg.N / G * (1 - 1 / G) * 4 / 1e9:.3f} GB requests; "
      f"pairwise {G.bit_length() - 1} x {cfg.N / G * state / 1e9:.3f} GB")
nvl = 770.0e9  # B200_PROFILING.md: measured peer copy per direction per GPU
local = ms / G
print(f"projection per rank: {local:.3f} ms of kernels + {moved / nvl * 1e3:.3f} ms NVLink ({moved / 1e9:.3f} GB at "
      f"770 GB/s) = {local + moved / nvl * 1e3:.3f} ms without overlap, {max(local, moved / nvl * 1e3):.3f} ms with "
      f"full overlap")
for b in shards:
    b.close()
