#!/usr/bin/env python
"""Benchmark of the BPF step with augmented resampling (arXiv 1812.01502) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One "step" = one pf_step: mutate + weight + S butterfly stages + composition over all
N particles.  Default workload: BASELINE.json configs[3]
(C4: 4-D linear-Gaussian HMM, N = 2^28, M = 64, S = 22), the configuration the
north_star's throughput/HBM target is quoted on; it fits one B200 (state 4 GiB).

Timing: W untimed warm-up steps, then K steps bracketed by a barrier +
torch.cuda.synchronize() and CUDA events on the filter's stream; max over ranks.
Inputs (x: 4 GiB, A: 1 GiB at C4) are far larger than the 126 MB L2, so no flush is
needed between steps.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec per BPF step (1/2/4/8 B200) and % of HBM roofline"
UNIT = "particle-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--N", type=int, default=0, help="override N (default: the config's)")
    ap.add_argument("--M", type=int, default=0, help="override M")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--theta", type=float, default=0.0,
                    help="ESS threshold of the fully adapted scheme (0: plain augmented resampling)")
    ap.add_argument("--airpf", type=int, default=0, choices=[0, 1, 2],
                    help="AIRPF (Alg. 4) with Alg. 7 (1) or Alg. 6 (2) instead of augmented resampling")
    ap.add_argument("--rotate", action="store_true",
                    help="with --theta: stage rotation (PAPER.md:1309)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "pull", "pairwise"],
                    help="N > 1: cross stages as one peer-memory gather over NVLink (default; the pull "
                         "exchange if a rank cannot map its peers), one all-to-all pull, or L pairwise rounds")
    ap.add_argument("--graph", type=int, default=-1, choices=[-1, 0, 1],
                    help="one GPU: the K timed steps as one CUDA graph (pf_graph_capture, untimed) launched "
                         "once (pf_graph_launch, timed); -1 (default): when N <= 2^22 and the scheme allows")
    ap.add_argument("--y-dev", action="store_true",
                    help="timed loop through pf_step_dev (observations read from device memory) instead of "
                         "the north_star pf_step(h, y_host) (observation in the launch parameters)")
    ap.add_argument("--multinomial", action="store_true",
                    help="the plain BPF (Alg. 2, multinomial resampling) instead of augmented resampling")
    return ap.parse_args()


def workload(args):
    from paper_1812_01502_b200 import inputs
    cfg = inputs.CONFIGS[args.config]
    if args.config == "C5" and not args.M:
        cfg = cfg.with_sizes(64, inputs.C5_N // 64)
    if args.M or args.N:
        M = args.M or cfg.M
        N = args.N or cfg.N
        cfg = cfg.with_sizes(M, N // M)
    return cfg


def config_dict(cfg, world, parallelism):
    return {"workload": cfg.name, "model": {1: "linear-Gaussian", 2: "stochastic-volatility"}[cfg.kind],
            "d": cfg.d, "N": cfg.N, "N_per_gpu": cfg.N // world, "M": cfg.M, "m": cfg.m, "S": cfg.S, "T": cfg.T,
            "parallelism": parallelism,
            "l2": "inputs larger than L2 (state + ancestor map >> 126 MB), no flush"}


# ----------------------------------------------------------------------------- oracle
def oracle_timed(cfg, n_sample, steps, warmup=0, threads=1):
    """Time the fp64 oracle (as it stands, never tuned) on a bounded sample of the
    workload: same model and M, N = n_sample particles per filter, `steps` mutating steps
    after `warmup` untimed ones.  threads > 1: that many independent filters (seeds 5..)
    run concurrently, one per host core (the oracle is a plain C library called through
    ctypes, which releases the GIL); throughput counts every thread's particle-steps.
    Returns the cpu_baseline dict plus the per-step wall times."""
    import threading

    from oracle import oracle as orc
    from paper_1812_01502_b200 import inputs
    params = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=warmup + steps + 1)
    xs = [inputs.particle_cloud(cfg, n_sample, 5 + t) for t in range(threads)]
    for t in range(threads):
        for n in range(1, warmup + 1):
            xs[t] = orc.step(params, n_sample, cfg.M, 1 + t, n, ys[n], xs[t], tables=False)["xhat"].astype("float32")
    step_wall = []
    for n in range(warmup + 1, warmup + steps + 1):
        def work(t, n=n):
            xs[t] = orc.step(params, n_sample, cfg.M, 1 + t, n, ys[n], xs[t], tables=False)["xhat"].astype("float32")
        th = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
        t0 = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        step_wall.append(time.perf_counter() - t0)
    dt = sum(step_wall)
    m = n_sample // cfg.M
    value = threads * n_sample * steps / dt
    return dict(value=value, unit=UNIT, cores=threads, kind="oracle",
                sample=f"{cfg.name} model, M={cfg.M}, N={n_sample} (m={m}, S={m.bit_length() - 1}) per filter, "
                       f"{threads} independent filter(s) on {threads} host thread(s), {steps} steps, fp64 C oracle, "
                       f"{dt:.1f} s"), step_wall


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def cpu_baseline(cfg):
    """The oracle on all host cores (one independent filter per core) next to one core."""
    n_sample = min(cfg.N, 1 << 20)
    one, _ = oracle_timed(cfg, n_sample, 2, threads=1)
    cores = host_cores()
    allc, _ = oracle_timed(cfg, n_sample, 2, threads=cores) if cores > 1 else (one, None)
    allc = dict(allc)
    allc["single_core_value"] = one["value"]
    allc["nproc"] = cores
    return allc


def run_reference(args):
    """The reference arm: the oracle as it stands, on all host cores, rank 0 only.  Each
    of the K timed steps is a bounded sample of the workload (same model and M; N shrunk so
    that the whole run takes ~1-3 min of wall time), run as one independent filter per
    core.  The config printed is the one timed (N, m, S of the sample)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = workload(args)
    from oracle import oracle as orc
    orc.build()
    steps = max(1, args.steps)
    cores = host_cores()
    n_sample = 1 << max(1, min(20, ((1 << 24) // steps).bit_length() - 1))
    n_sample = min(cfg.N, max(n_sample, 2 * cfg.M))
    cb, walls = oracle_timed(cfg, n_sample, steps, warmup=min(max(0, args.warmup), 1), threads=cores)
    timed = cfg.with_sizes(cfg.M, n_sample // cfg.M)
    conf = config_dict(timed, 1, f"fp64 CPU oracle, {cores} independent filters on {cores} host threads")
    conf.update({"sample_of": {"workload": cfg.name, "N": cfg.N, "m": cfg.m, "S": cfg.S},
                 "filters_per_step": cores})
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": conf, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "20"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for k, nm in enumerate(names):
                    if r[4 + k].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        loaded = [v for v in sm if mx and v > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- ours
NVLINK_PEER_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction per GPU (900 nominal)


def algorithmic_bytes(cfg, kernel: str, exchange: str = "pairwise") -> float:
    """Algorithmic HBM bytes per launch: the bytes the kernel must move
    once, with no sector amplification and no re-reads.  cfg: this rank's shard."""
    N, d = cfg.N, cfg.d
    if kernel in ("k_pass1", "k_stages"):
        return N * 8 * d   # read the tile's states once, write them once
    if kernel == "k_cross" and exchange == "peer":
        return N * 8 * d   # every output's state read once (mostly from peers) and written once
    if kernel == "k_cross":
        return N * 8 * d + N * 4 * d  # own read + write, partner half on average
    if kernel in ("k_cascade", "k_top"):
        return (cfg.m / 64) * 8 * 2
    return 0.0


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg, kernel, what=""):
    """Per-launch ncu figure recorded by tools/ncu_traffic.py: DRAM bytes (what = "") or
    issued warp instructions (what = ":warp_inst"); None when not captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            tr = json.load(f)
        return tr[f"{cfg.name}:N={cfg.N}:M={cfg.M}{what}"][kernel]
    except (OSError, KeyError, ValueError):
        return None


def issue_peak():
    """Warp instructions per second the SMs can issue: 148 SMs x 4 schedulers x SM clock
    (one warp instruction per scheduler per cycle; B200_PROFILING.md unit counts)."""
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except (OSError, ValueError):
        pass
    return 148 * 4 * mhz * 1e6


def run_ours(args):
    if (args.theta > 0 or args.airpf or args.multinomial) and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        raise SystemExit("--theta / --airpf / --multinomial run on one GPU only")
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1812_01502_b200 import inputs, pf

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    cfg = workload(args)
    params = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg)
    T = len(ys)
    ys32 = [np.ascontiguousarray(y, np.float32) for y in ys]
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        y_dev = torch.tensor(np.asarray(ys, np.float32), device=dev)
        if world == 1:
            f = pf.ParticleFilter(params, cfg.N, cfg.M, args.seed, stream=stream, theta=args.theta,
                                  airpf=args.airpf, multinomial=args.multinomial, rotate=args.rotate)

            def step(k):
                f.step_dev(y_dev[k % T])

            def step_host(k):  # the north_star call pf_step(h, y_host): y travels in the launch
                f.step(ys32[k % T])

            def estimate():
                return f.estimate(pf.PF_PHI_X, pf.PF_EST_FILTER)
        else:
            from paper_1812_01502_b200 import dist as pfd
            # strong scaling: the global N of the configuration is split over the ranks
            f = pfd.LibBackend(params, cfg.N, cfg.M, args.seed, rank, world, stream=stream)
            tr = pfd.TorchTransport()
            if args.exchange == "peer" and not pfd.peer_connect(f, tr):
                print(f"[bench] rank {rank}: peer mapping failed on some rank; pull exchange", file=sys.stderr)
                args.exchange = "pull"

            def step(k):
                pfd.sharded_step(f, tr, None, y_dev[k % T], exchange=args.exchange)

            def step_host(k):
                pfd.sharded_step(f, tr, ys32[k % T], exchange=args.exchange)

            def estimate():
                return f.estimate(pf.PF_PHI_X, pf.PF_EST_FILTER)
        for w in range(args.warmup):
            step(w)
        stream.synchronize()
        f.timing_enable(True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        stages = []
        use_graph = world == 1 and args.theta <= 0 and (args.graph == 1 or (args.graph == -1 and cfg.N <= (1 << 22)))
        if use_graph:  # K steps captured (untimed); the timed region is their one launch
            f.timing_enable(False)
            ks = (args.warmup + np.arange(args.steps)) % T
            f.graph_capture(y_dev[torch.as_tensor(ks, device=dev)].contiguous())
            stream.synchronize()
        e0.record(stream)
        if use_graph:
            f.graph_launch()
        else:
            timed_step = step if args.y_dev else step_host
            for k in range(args.steps):
                timed_step(args.warmup + k)
                if args.theta > 0:
                    stages.append(f.last_stages())  # the adaptive step has synchronised already
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
        ms = e0.elapsed_time(e1)
        if use_graph:  # per-kernel device times from K eager steps after the timed graph
            f.timing_enable(True)
            for k in range(args.steps):
                step(args.warmup + args.steps + k)
            stream.synchronize()
        kt = f.timing_read()
        f.timing_enable(False)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        kt = {k: v for k, v in kt.items() if v[1] > 0}
        launches = sum(n for _, n in kt.values())
        value = cfg.N * args.steps / (ms / 1e3)  # global particles (strong scaling)

        # roofline of the dominant kernel
        dom = max(kt, key=lambda k: kt[k][0])
        dom_ms, dom_n = kt[dom]
        cfg_loc = cfg.with_sizes(cfg.M, cfg.m // world)
        exch = args.exchange if world > 1 else ""
        alg = algorithmic_bytes(cfg_loc, dom, exch)
        achieved = alg / (dom_ms / dom_n / 1e3) / 1e9
        peak, peak_src = measured_peak()
        # the ncu figures are the plain one-GPU step's (per launch at the full N)
        plain = not (args.theta or args.airpf or args.multinomial) and world == 1
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": ncu_traffic(cfg, dom) if plain else None,
                    "algorithmic_bytes_per_launch": alg, "peak_source": peak_src,
                    "kernel_share_of_step": round(dom_ms / max(sum(v[0] for v in kt.values()), 1e-9), 3),
                    "step_alg_bytes_frac": round(value / world * 8 * cfg.d / 1e9 / peak, 4)}
        # peer exchange: bytes that must cross NVLink per launch = the states read from the
        # other ranks, (1 - 1/G) of the shard's outputs on average
        nvl_bytes = cfg_loc.N * 4 * cfg.d * (1 - 1 / world) if exch == "peer" else 0.0
        if dom == "k_cross" and nvl_bytes:
            nv = nvl_bytes / (dom_ms / dom_n / 1e3) / 1e9
            roofline.update({"bound": "nvlink", "achieved": round(nv, 1), "peak": NVLINK_PEER_GBS,
                             "frac": round(nv / NVLINK_PEER_GBS, 4), "traffic": None,
                             "algorithmic_bytes_per_launch": nvl_bytes,
                             "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)"})
        kernels = {k: {"ms_per_launch": round(v[0] / max(v[1], 1), 4), "launches": v[1]} for k, v in kt.items()}
        if nvl_bytes and "k_cross" in kernels and kernels["k_cross"]["ms_per_launch"] > 0:
            kernels["k_cross"]["nvlink_frac"] = round(
                nvl_bytes / (kernels["k_cross"]["ms_per_launch"] / 1e3) / 1e9 / NVLINK_PEER_GBS, 4)
        # per kernel: HBM fraction (algorithmic bytes) and issue fraction (ncu instruction count)
        for k, v in kernels.items():
            sec = v["ms_per_launch"] / 1e3
            if sec <= 0:
                continue
            ab = algorithmic_bytes(cfg_loc, k, exch)
            if ab:
                v["hbm_frac"] = round(ab / sec / 1e9 / peak, 4)
            wi = ncu_traffic(cfg, k, ":warp_inst")
            if wi is not None and plain:
                v["issue_frac"] = round(wi / sec / issue_peak(), 4)
        roofline["issue_frac_dominant"] = kernels.get(dom, {}).get("issue_frac")
        # which roofline bounds the dominant kernel: the larger of its HBM fraction (algorithmic
        # bytes) and its issue fraction (ncu warp instructions / the SMs' issue peak,
        # 148 SMs x 4 schedulers x clock) -- "alu" when the issue slots bind
        iss = roofline["issue_frac_dominant"]
        if roofline["bound"] == "hbm" and iss is not None and iss > roofline["frac"]:
            roofline.update({"bound": "alu", "hbm_frac": roofline["frac"], "achieved": round(iss * issue_peak(), 1),
                             "peak": issue_peak(), "unit": "warp-inst/s", "frac": iss,
                             "peak_source": "148 SMs x 4 schedulers x sm_max_mhz (MEASURED_PEAKS.json), one "
                                            "warp instruction per scheduler per cycle"})

        # end-to-end through the public API, the north_star calls: pf_step(h, y_host) -- the
        # observation (host memory) is copied into the launch parameters -- then
        # pf_estimate(h, PF_PHI_X, PF_EST_FILTER, out_host), which reads the estimate back
        # (device -> host) and synchronises.  Timed by the host clock, max over ranks.
        e2e = None
        if not args.no_e2e:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for k in range(args.steps):
                step_host(args.warmup + k)
                est = estimate()
            torch.cuda.synchronize()
            te = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([te], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                te = float(t.item())
            e2e = {"value": cfg.N * args.steps / te, "unit": UNIT, "h2d_bytes_per_step": 4 * cfg.dy,
                   "d2h_bytes_per_step": 8 * cfg.d, "api": "pf_step(h, y_host) + pf_estimate(h, PF_PHI_X, "
                   "PF_EST_FILTER, out_host)", "last_filter_mean": [float(v) for v in est]}
        f.close()

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(config_dict(cfg, world, "single" if world == 1 else f"groups sharded over {world} GPUs, {args.exchange} exchange"),
                               **({"theta": args.theta, "stage_rotation": bool(args.rotate),
                                   "stages_run_mean": float(np.mean(stages)),
                                   "stages_run_hist": np.bincount(stages, minlength=cfg.S + 1).tolist()}
                                  if args.theta > 0 else {}),
                               **({"algorithm": {1: "AIRPF (Alg. 4 + 5 + 7)", 2: "AIRPF (Alg. 4 + 5 + 6)"}[args.airpf]
                                   + (" with the fully adapted scheme: AIRPF2" if args.theta > 0 else "")}
                                  if args.airpf else {}),
                               **({"algorithm": "plain BPF (Alg. 1 + 2, multinomial)"} if args.multinomial else {})),
                "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
                "timed_as": ("one CUDA graph of the K steps (pf_graph_launch); kernels: K eager steps after it"
                             if use_graph else ("pf_step_dev (y in device memory)" if args.y_dev
                                                else "pf_step(h, y_host) (y in the launch parameters)")),
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
