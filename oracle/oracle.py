"""ctypes wrapper of the fp64 C oracle (oracle/pf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path
(paper_1812_01502_b200/).  It shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pf_oracle.c")
_LIB = os.path.join(_HERE, "libpforacle.so")

INIT, MUTATE, RESAMPLE, WITHIN, ISLAND, MULTI = 1, 2, 3, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-D_GNU_SOURCE", "-fPIC", "-shared", "-ffp-contract=off",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


class _Model(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("d", ctypes.c_int), ("dy", ctypes.c_int),
                ("A", ctypes.c_float * 64), ("LQ", ctypes.c_float * 64), ("H", ctypes.c_float * 64),
                ("Rinv", ctypes.c_float * 64), ("m0", ctypes.c_float * 8), ("L0", ctypes.c_float * 64),
                ("sv_phi", ctypes.c_float), ("sv_sigma", ctypes.c_float), ("sv_beta", ctypes.c_float),
                ("sv_m0", ctypes.c_float), ("sv_s0", ctypes.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        u64, u32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        _lib.orc_philox4x32_10.argtypes = [vp, vp, vp]
        _lib.orc_normal.argtypes = [u64, u32, u32, u64]
        _lib.orc_normal.restype = ctypes.c_double
        _lib.orc_init.argtypes = [vp, u64, u64, vp]
        _lib.orc_init_rows.argtypes = [vp, u64, u64, vp, vp]
        _lib.orc_mutate.argtypes = [vp, u64, u64, u32, vp, vp]
        _lib.orc_logweight.argtypes = [vp, u64, vp, vp, vp]
        _lib.orc_augmented_resample.argtypes = [u64, u64, u64, u32, vp, vp, vp, vp, vp]
        _lib.orc_augmented_resample_sampled.argtypes = [u64, u64, u64, u32, vp, u64, vp, vp, vp, vp, vp, vp]
        _lib.orc_estimates.argtypes = [ctypes.c_int, u64, vp, vp, vp, vp, vp, vp]
        _lib.orc_step.argtypes = [vp, u64, u64, u64, u32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_step_sampled.argtypes = [vp, u64, u64, u64, u32, vp, vp, ctypes.c_double, u64, vp, vp, vp, vp, vp,
                                          vp, vp, vp, vp]
        _lib.orc_step_multinomial_sampled.argtypes = [vp, u64, u64, u32, vp, vp, u64, vp, ctypes.c_double, vp, vp, vp,
                                                      vp, vp, vp, vp]
        _lib.orc_step_airpf_sampled.argtypes = [vp, u64, u64, u64, u32, vp, vp, ctypes.c_int, u64, vp, vp, vp, vp,
                                                vp, vp, vp]
        _lib.orc_augmented_resample_partial.argtypes = [u64, u64, u64, u32, vp, ctypes.c_int, vp, vp, vp, vp]
        _lib.orc_ess_levels.argtypes = [u64, u64, vp, vp, vp]
        _lib.orc_stages_to_run.argtypes = [ctypes.c_int, vp, ctypes.c_double]
        _lib.orc_stages_to_run.restype = ctypes.c_int
        _lib.orc_within_island.argtypes = [u64, u64, u64, u32, vp, vp, vp, vp]
        _lib.orc_island_resample.argtypes = [u64, u64, u32, vp, ctypes.c_int, vp, vp, vp, vp]
        _lib.orc_step_airpf.argtypes = [vp, u64, u64, u64, u32, vp, vp, ctypes.c_int, vp, vp, vp, vp, vp, vp,
                                        vp, vp, vp, vp, vp]
        _lib.orc_multinomial.argtypes = [u64, u64, u32, vp, vp, vp]
        _lib.orc_step_multinomial.argtypes = [vp, u64, u64, u32, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_step_adaptive.argtypes = [vp, u64, u64, u64, u32, vp, vp, vp, ctypes.c_double, vp, vp, vp, vp,
                                           vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_relabel_stage.argtypes = [u64, u64, ctypes.c_int, vp, vp]
        _lib.orc_augmented_resample_relabel.argtypes = [u64, u64, u64, u64, u32, vp, vp, vp, vp, vp, vp]
        _lib.orc_step_relabel.argtypes = [vp, u64, u64, u64, u64, u32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                          vp, vp]
        _lib.orc_island_resample_partial.argtypes = [u64, u64, u32, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]
        _lib.orc_step_airpf_adaptive.argtypes = [vp, u64, u64, u64, u32, vp, vp, vp, ctypes.c_double, ctypes.c_int,
                                                 vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_step_adaptive_rot.argtypes = [vp, u64, u64, u64, u32, vp, vp, vp, ctypes.c_double, ctypes.c_int,
                                               vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def make_model(params: dict) -> _Model:
    """Build the C model struct from inputs.model_params() (fp32 values)."""
    m = _Model()
    m.kind = int(params["kind"])
    m.d = int(params["d"])
    m.dy = int(params["dy"])
    if m.kind == 2:
        m.sv_phi = float(params["phi"])
        m.sv_sigma = float(params["sigma"])
        m.sv_beta = float(params["beta"])
        m.sv_m0 = float(params["m0"])
        m.sv_s0 = float(params["s0"])
    else:
        for name in ("A", "LQ", "H", "Rinv", "L0", "m0"):
            arr = np.ascontiguousarray(params[name], dtype=np.float32).ravel()
            getattr(m, name)[: arr.size] = arr.tolist()
    return m


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def normal(seed: int, domain: int, n: int, c: int) -> float:
    return lib().orc_normal(seed, domain, n, c)


def init(params: dict, N: int, seed: int) -> np.ndarray:
    mdl = make_model(params)
    x = np.zeros((N, mdl.d), np.float64)
    lib().orc_init(ctypes.byref(mdl), N, seed, _ptr(x))
    return x


def init_rows(params: dict, seed: int, rows: np.ndarray) -> np.ndarray:
    """x_0 of the particles rows[] (orc_init restricted to those indices)."""
    mdl = make_model(params)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    x = np.zeros((r.size, mdl.d), np.float64)
    lib().orc_init_rows(ctypes.byref(mdl), seed, r.size, _ptr(r), _ptr(x))
    return x


def mutate(params: dict, seed: int, n: int, xhat: np.ndarray) -> np.ndarray:
    mdl = make_model(params)
    xh = np.ascontiguousarray(xhat, dtype=np.float64)
    x = np.zeros_like(xh)
    lib().orc_mutate(ctypes.byref(mdl), xh.shape[0], seed, n, _ptr(xh), _ptr(x))
    return x


def logweight(params: dict, y: np.ndarray, x: np.ndarray) -> np.ndarray:
    mdl = make_model(params)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    lw = np.zeros(xx.shape[0], np.float64)
    lib().orc_logweight(ctypes.byref(mdl), xx.shape[0], _ptr(yy), _ptr(xx), _ptr(lw))
    return lw


def augmented_resample(lw: np.ndarray, M: int, seed: int, n: int, tables: bool = True) -> dict:
    """Alg. 3 on log-weights lw (N,). Returns dict(a[S,N], delta[S,N], logV[m-1], A[N])."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    m = N // M
    S = int(round(np.log2(m)))
    a = np.zeros((S, N), np.int32) if tables else None
    delta = np.zeros((S, N), np.float32) if tables else None
    logV = np.zeros(m - 1, np.float64)
    A = np.zeros(N, np.int64)
    rc = lib().orc_augmented_resample(N, M, seed, n, _ptr(lw), _ptr(a), _ptr(delta), _ptr(logV), _ptr(A))
    if rc != 0:
        raise ValueError(f"orc_augmented_resample rc={rc} (N={N}, M={M})")
    return dict(a=a, delta=delta, logV=logV, A=A, S=S, m=m)


def augmented_resample_sampled(lw: np.ndarray, M: int, seed: int, n: int, outputs: np.ndarray) -> dict:
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    m = N // M
    S = int(round(np.log2(m)))
    outs = np.ascontiguousarray(outputs, dtype=np.int64)
    k = outs.shape[0]
    path = np.zeros((k, S), np.int64)
    anc = np.zeros((k, S), np.int64)
    pdelta = np.zeros((k, S), np.float32)
    logV = np.zeros(m - 1, np.float64)
    A = np.zeros(k, np.int64)
    rc = lib().orc_augmented_resample_sampled(N, M, seed, n, _ptr(lw), k, _ptr(outs), _ptr(path),
                                              _ptr(anc), _ptr(pdelta), _ptr(logV), _ptr(A))
    if rc != 0:
        raise ValueError(f"orc_augmented_resample_sampled rc={rc}")
    return dict(path=path, anc=anc, delta=pdelta, logV=logV, A=A, S=S, m=m)


def level_offset(m: int, s: int) -> int:
    """Offset of level s (1..S) in the logV table: level s has m/2^s entries."""
    return m - (m >> (s - 1))


def estimates(d: int, lw: np.ndarray, x: np.ndarray, A: Optional[np.ndarray]) -> dict:
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    AA = None if A is None else np.ascontiguousarray(A, dtype=np.int64)
    f = np.zeros(2 * d)
    p = np.zeros(2 * d)
    r = np.zeros(2 * d)
    lib().orc_estimates(d, lw.shape[0], _ptr(lw), _ptr(xx), _ptr(AA), _ptr(f), _ptr(p), _ptr(r))
    return dict(filter=f, predict=p, resampled=r if A is not None else None)


def step(params: dict, N: int, M: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
         tables: bool = True) -> dict:
    """One time step from xin (fp32 xhat_{n-1}, or x_0 when n == 0).
    tables=False skips the per-stage ancestor / delta tables (same draws)."""
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    S = int(round(np.log2(m)))
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = dict(x=np.zeros((N, d)), lw=np.zeros(N), a=np.zeros((S, N), np.int32) if tables else None,
               delta=np.zeros((S, N), np.float32) if tables else None, logV=np.zeros(m - 1), A=np.zeros(N, np.int64),
               xhat=np.zeros((N, d)), filter=np.zeros(2 * d), predict=np.zeros(2 * d),
               resampled=np.zeros(2 * d))
    rc = lib().orc_step(ctypes.byref(mdl), N, M, seed, n, _ptr(yy), _ptr(xin), _ptr(out["x"]),
                        _ptr(out["lw"]), _ptr(out["a"]), _ptr(out["delta"]), _ptr(out["logV"]),
                        _ptr(out["A"]), _ptr(out["xhat"]), _ptr(out["filter"]), _ptr(out["predict"]),
                        _ptr(out["resampled"]))
    if rc != 0:
        raise ValueError(f"orc_step rc={rc}")
    out["S"], out["m"] = S, m
    return out


def step_sampled(params: dict, N: int, M: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
                 outputs: np.ndarray, theta: float = 0.0) -> dict:
    """One step at full size, evaluated on sampled outputs (orc_step_sampled): all V
    levels, the estimates, and for each sampled output its composed ancestor A, the
    boundary distances of the draws on its path (pdelta, samples x S, stage s at s-1)
    and its resampled state xhat.  theta > 0: the fully adapted step (ess, sstar)."""
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    S = int(round(np.log2(m)))
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    outs = np.ascontiguousarray(outputs, dtype=np.int64)
    k = len(outs)
    out = dict(logV=np.zeros(m - 1), ess=np.zeros(S + 1), A=np.zeros(k, np.int64),
               pdelta=np.zeros((k, S), np.float32), xhat=np.zeros((k, d)), filter=np.zeros(2 * d),
               predict=np.zeros(2 * d))
    ss = ctypes.c_int(0)
    rc = lib().orc_step_sampled(ctypes.byref(mdl), N, M, seed, n, _ptr(yy), _ptr(xin), float(theta), k, _ptr(outs),
                                _ptr(out["logV"]), _ptr(out["ess"]), ctypes.byref(ss), _ptr(out["A"]),
                                _ptr(out["pdelta"]), _ptr(out["xhat"]), _ptr(out["filter"]), _ptr(out["predict"]))
    if rc != 0:
        raise ValueError(f"orc_step_sampled rc={rc}")
    out["S"], out["m"], out["sstar"] = S, m, int(ss.value)
    return out


def step_airpf_sampled(params: dict, N: int, M: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
                       outputs: np.ndarray, modified: bool = True) -> dict:
    """One AIRPF step at full size on sampled outputs (orc_step_airpf_sampled): island
    log-means logW, island map Aisl, estimates, and per sampled output its resampled state
    xhat and the smallest boundary distance on its path (sdelta)."""
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    outs = np.ascontiguousarray(outputs, dtype=np.int64)
    k = len(outs)
    out = dict(logW=np.zeros(m), Aisl=np.zeros(m, np.int64), sdelta=np.zeros(k, np.float32), xhat=np.zeros((k, d)),
               filter=np.zeros(2 * d), predict=np.zeros(2 * d))
    rc = lib().orc_step_airpf_sampled(ctypes.byref(mdl), N, M, seed, n, _ptr(yy), _ptr(xin), 1 if modified else 0, k,
                                      _ptr(outs), _ptr(out["logW"]), _ptr(out["Aisl"]), _ptr(out["sdelta"]),
                                      _ptr(out["xhat"]), _ptr(out["filter"]), _ptr(out["predict"]))
    if rc != 0:
        raise ValueError(f"orc_step_airpf_sampled rc={rc}")
    return out


def run_filter(params: dict, M: int, m: int, seed: int, ys: np.ndarray, x0: Optional[np.ndarray] = None):
    """Alg. 1 with Alg. 3 for len(ys) steps; returns the per-step filter means (T x d).
    State is kept in fp32 between steps, as in the configurations (fp32 particles)."""
    N = M * m
    d = int(params["d"])
    x = (init(params, N, seed) if x0 is None else x0).astype(np.float32)
    means = np.zeros((len(ys), d))
    for n, y in enumerate(ys):
        r = step(params, N, M, seed, n, y, x, tables=False)
        means[n] = r["filter"][:d]
        x = r["xhat"].astype(np.float32)
    return means


# ----------------------------------------------------------------------------- fully adapted
def augmented_resample_partial(lw: np.ndarray, M: int, seed: int, n: int, S_exec: int) -> dict:
    """Alg. 3 with only stages 1..S_exec executed (all V levels computed)."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    m = N // M
    S = int(round(np.log2(m)))
    a = np.zeros((S, N), np.int32)
    delta = np.zeros((S, N), np.float32)
    logV = np.zeros(m - 1, np.float64)
    A = np.zeros(N, np.int64)
    rc = lib().orc_augmented_resample_partial(N, M, seed, n, _ptr(lw), int(S_exec), _ptr(a), _ptr(delta),
                                              _ptr(logV), _ptr(A))
    if rc != 0:
        raise ValueError(f"orc_augmented_resample_partial rc={rc}")
    return dict(a=a, delta=delta, logV=logV, A=A, S=S, m=m)


def ess_levels(lw: np.ndarray, M: int, logV: np.ndarray) -> np.ndarray:
    """ESS of the stage weights V_0 = w, V_1, ..., V_S."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    S = int(round(np.log2(N // M)))
    lv = np.ascontiguousarray(logV, dtype=np.float64)
    ess = np.zeros(S + 1)
    lib().orc_ess_levels(N, M, _ptr(lw), _ptr(lv), _ptr(ess))
    return ess


def stages_to_run(ess: np.ndarray, theta: float) -> int:
    e = np.ascontiguousarray(ess, dtype=np.float64)
    return int(lib().orc_stages_to_run(len(e) - 1, _ptr(e), float(theta)))


def step_adaptive(params: dict, N: int, M: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
                  lwc_in: np.ndarray, theta: float, rotate: bool = False) -> dict:
    """One step of the fully adapted filter (orc_step_adaptive_rot); rotate: stage rotation
    (reading R23) -- xhat and lwc come back in the next step's layout."""
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    S = int(round(np.log2(m)))
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    lwc = np.ascontiguousarray(lwc_in, dtype=np.float64).reshape(N)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = dict(x=np.zeros((N, d)), lw=np.zeros(N), a=np.zeros((S, N), np.int32), delta=np.zeros((S, N), np.float32),
               logV=np.zeros(m - 1), A=np.zeros(N, np.int64), xhat=np.zeros((N, d)), lwc=np.zeros(N),
               filter=np.zeros(2 * d), predict=np.zeros(2 * d), ess=np.zeros(S + 1))
    ss = ctypes.c_int(-1)
    rc = lib().orc_step_adaptive_rot(ctypes.byref(mdl), N, M, seed, n, _ptr(yy), _ptr(xin), _ptr(lwc),
                                     float(theta), int(bool(rotate)), _ptr(out["x"]), _ptr(out["lw"]), _ptr(out["a"]), _ptr(out["delta"]),
                                 _ptr(out["logV"]), _ptr(out["A"]), _ptr(out["xhat"]), _ptr(out["lwc"]),
                                 _ptr(out["filter"]), _ptr(out["predict"]), _ptr(out["ess"]), ctypes.byref(ss))
    if rc != 0:
        raise ValueError(f"orc_step_adaptive rc={rc}")
    out["S"], out["m"], out["sstar"] = S, m, int(ss.value)
    return out


def run_filter_adaptive(params: dict, M: int, m: int, seed: int, ys: np.ndarray, theta: float,
                        x0: Optional[np.ndarray] = None, rotate: bool = False):
    """The fully adapted filter for len(ys) steps: per-step filter means (T x d) and the
    number of stages run at each step."""
    N = M * m
    d = int(params["d"])
    x = (init(params, N, seed) if x0 is None else x0).astype(np.float32)
    lwc = np.zeros(N)
    means = np.zeros((len(ys), d))
    stages = np.zeros(len(ys), np.int32)
    for n, y in enumerate(ys):
        r = step_adaptive(params, N, M, seed, n, y, x, lwc, theta, rotate)
        means[n] = r["filter"][:d]
        stages[n] = r["sstar"]
        x = r["xhat"].astype(np.float32)
        lwc = r["lwc"]
    return means, stages


# ----------------------------------------------------------------------------- AIRPF
def within_island(lw: np.ndarray, M: int, seed: int, n: int) -> dict:
    """Alg. 5: within-island multinomial draws a_w (N), deltas, log island means (m)."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    a_w = np.zeros(N, np.int64)
    delta = np.zeros(N, np.float32)
    logW = np.zeros(N // M)
    rc = lib().orc_within_island(N, M, seed, n, _ptr(lw), _ptr(a_w), _ptr(delta), _ptr(logW))
    if rc != 0:
        raise ValueError(f"orc_within_island rc={rc}")
    return dict(a_w=a_w, delta=delta, logW=logW)


def island_resample(logW: np.ndarray, seed: int, n: int, modified: bool = True) -> dict:
    """Alg. 6 / Alg. 7 over m island log-weights: src (S, m), deltas, levels, Aisl (m)."""
    lw = np.ascontiguousarray(logW, dtype=np.float64)
    m = lw.shape[0]
    S = int(round(np.log2(m)))
    src = np.zeros((S, m), np.int32)
    delta = np.zeros((S, m), np.float32)
    lv = np.zeros(m - 1)
    A = np.zeros(m, np.int64)
    rc = lib().orc_island_resample(m, seed, n, _ptr(lw), int(bool(modified)), _ptr(src), _ptr(delta), _ptr(lv),
                                   _ptr(A))
    if rc != 0:
        raise ValueError(f"orc_island_resample rc={rc}")
    return dict(src=src, delta=delta, logVbar=lv, Aisl=A, S=S)


def step_airpf(params: dict, N: int, M: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
               modified: bool = True) -> dict:
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    S = int(round(np.log2(m)))
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = dict(x=np.zeros((N, d)), lw=np.zeros(N), a_w=np.zeros(N, np.int64), wdelta=np.zeros(N, np.float32),
               logW=np.zeros(m), src=np.zeros((S, m), np.int32), idelta=np.zeros((S, m), np.float32),
               logVbar=np.zeros(m - 1), Aisl=np.zeros(m, np.int64), xhat=np.zeros((N, d)),
               filter=np.zeros(2 * d), predict=np.zeros(2 * d))
    rc = lib().orc_step_airpf(ctypes.byref(mdl), N, M, seed, n, _ptr(yy), _ptr(xin), int(bool(modified)),
                              _ptr(out["x"]), _ptr(out["lw"]), _ptr(out["a_w"]), _ptr(out["wdelta"]),
                              _ptr(out["logW"]), _ptr(out["src"]), _ptr(out["idelta"]), _ptr(out["logVbar"]),
                              _ptr(out["Aisl"]), _ptr(out["xhat"]), _ptr(out["filter"]), _ptr(out["predict"]))
    if rc != 0:
        raise ValueError(f"orc_step_airpf rc={rc}")
    out["S"], out["m"] = S, m
    return out


def run_filter_airpf(params: dict, M: int, m: int, seed: int, ys: np.ndarray, modified: bool = True,
                     x0: Optional[np.ndarray] = None):
    N = M * m
    d = int(params["d"])
    x = (init(params, N, seed) if x0 is None else x0).astype(np.float32)
    means = np.zeros((len(ys), d))
    for n, y in enumerate(ys):
        r = step_airpf(params, N, M, seed, n, y, x, modified)
        means[n] = r["filter"][:d]
        x = r["xhat"].astype(np.float32)
    return means


def island_resample_partial(logW: np.ndarray, seed: int, n: int, S_exec: int, modified: bool = True) -> dict:
    """Alg. 6/7 with island stages 1..S_exec (all V_bar levels)."""
    lw = np.ascontiguousarray(logW, dtype=np.float64)
    m = lw.shape[0]
    S = int(round(np.log2(m)))
    out = dict(src=np.zeros((S, m), np.int32), delta=np.zeros((S, m), np.float32), logVbar=np.zeros(m - 1),
               Aisl=np.zeros(m, np.int64))
    rc = lib().orc_island_resample_partial(m, seed, n, _ptr(lw), int(bool(modified)), int(S_exec), _ptr(out["src"]),
                                           _ptr(out["delta"]), _ptr(out["logVbar"]), _ptr(out["Aisl"]))
    if rc != 0:
        raise ValueError(f"orc_island_resample_partial rc={rc}")
    return out


def step_airpf_adaptive(params: dict, N: int, M: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
                        lwc_in: np.ndarray, theta: float, modified: bool = True) -> dict:
    """One AIRPF2 step (orc_step_airpf_adaptive, reading R26): island stages 1..S* only;
    lwc = the weight every particle carries into the next step."""
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    S = int(round(np.log2(m)))
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    lwc = np.ascontiguousarray(lwc_in, dtype=np.float64).reshape(N)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = dict(x=np.zeros((N, d)), lw=np.zeros(N), a_w=np.zeros(N, np.int64), wdelta=np.zeros(N, np.float32),
               logW=np.zeros(m), src=np.zeros((S, m), np.int32), idelta=np.zeros((S, m), np.float32),
               logVbar=np.zeros(m - 1), Aisl=np.zeros(m, np.int64), xhat=np.zeros((N, d)), lwc=np.zeros(N),
               filter=np.zeros(2 * d), predict=np.zeros(2 * d), ess=np.zeros(S + 1))
    ss = ctypes.c_int(-1)
    rc = lib().orc_step_airpf_adaptive(ctypes.byref(mdl), N, M, seed, n, _ptr(yy), _ptr(xin), _ptr(lwc), float(theta),
                                       int(bool(modified)), _ptr(out["x"]), _ptr(out["lw"]), _ptr(out["a_w"]),
                                       _ptr(out["wdelta"]), _ptr(out["logW"]), _ptr(out["src"]), _ptr(out["idelta"]),
                                       _ptr(out["logVbar"]), _ptr(out["Aisl"]), _ptr(out["xhat"]), _ptr(out["lwc"]),
                                       _ptr(out["filter"]), _ptr(out["predict"]), _ptr(out["ess"]), ctypes.byref(ss))
    if rc != 0:
        raise ValueError(f"orc_step_airpf_adaptive rc={rc}")
    out["S"], out["m"], out["sstar"] = S, m, int(ss.value)
    return out


def run_filter_airpf_adaptive(params: dict, M: int, m: int, seed: int, ys: np.ndarray, theta: float,
                              modified: bool = True):
    """AIRPF2 for len(ys) steps: per-step filter means and the island stages run."""
    N = M * m
    d = int(params["d"])
    x = init(params, N, seed).astype(np.float32)
    lwc = np.zeros(N)
    means = np.zeros((len(ys), d))
    stages = np.zeros(len(ys), np.int32)
    for n, y in enumerate(ys):
        r = step_airpf_adaptive(params, N, M, seed, n, y, x, lwc, theta, modified)
        means[n] = r["filter"][:d]
        stages[n] = r["sstar"]
        x = r["xhat"].astype(np.float32)
        lwc = r["lwc"]
    return means, stages


# ----------------------------------------------------------------------------- Alg. 2
def multinomial(lw: np.ndarray, seed: int, n: int) -> dict:
    """Alg. 2 over the whole population: ancestors a (N) and boundary distances."""
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    a = np.zeros(N, np.int64)
    delta = np.zeros(N, np.float32)
    rc = lib().orc_multinomial(N, seed, n, _ptr(lw), _ptr(a), _ptr(delta))
    if rc != 0:
        raise ValueError(f"orc_multinomial rc={rc}")
    return dict(a=a, delta=delta)


def step_multinomial(params: dict, N: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray) -> dict:
    mdl = make_model(params)
    d = mdl.d
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = dict(x=np.zeros((N, d)), lw=np.zeros(N), a=np.zeros(N, np.int64), delta=np.zeros(N, np.float32),
               xhat=np.zeros((N, d)), filter=np.zeros(2 * d), predict=np.zeros(2 * d))
    rc = lib().orc_step_multinomial(ctypes.byref(mdl), N, seed, n, _ptr(yy), _ptr(xin), _ptr(out["x"]),
                                    _ptr(out["lw"]), _ptr(out["a"]), _ptr(out["delta"]), _ptr(out["xhat"]),
                                    _ptr(out["filter"]), _ptr(out["predict"]))
    if rc != 0:
        raise ValueError(f"orc_step_multinomial rc={rc}")
    return out


def step_multinomial_sampled(params: dict, N: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray,
                             outputs: np.ndarray, eps: float = 1e-6) -> dict:
    """Alg. 2 step at full size on sampled outputs (orc_step_multinomial_sampled): a, the
    boundary distance sdelta, the states of particles a + (-2..2) (xnb), the window
    [klo, khi] of the draws for u -+ eps, estimates."""
    mdl = make_model(params)
    d = mdl.d
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    outs = np.ascontiguousarray(outputs, dtype=np.int64)
    k = len(outs)
    out = dict(a=np.zeros(k, np.int64), klo=np.zeros(k, np.int64), khi=np.zeros(k, np.int64),
               sdelta=np.zeros(k, np.float32), xnb=np.zeros((k, 5, d)), filter=np.zeros(2 * d), predict=np.zeros(2 * d))
    rc = lib().orc_step_multinomial_sampled(ctypes.byref(mdl), N, seed, n, _ptr(yy), _ptr(xin), k, _ptr(outs),
                                            float(eps), _ptr(out["a"]), _ptr(out["klo"]), _ptr(out["khi"]),
                                            _ptr(out["sdelta"]), _ptr(out["xnb"]), _ptr(out["filter"]),
                                            _ptr(out["predict"]))
    if rc != 0:
        raise ValueError(f"orc_step_multinomial_sampled rc={rc}")
    return out


def run_filter_multinomial(params: dict, N: int, seed: int, ys: np.ndarray, x0: Optional[np.ndarray] = None):
    d = int(params["d"])
    x = (init(params, N, seed) if x0 is None else x0).astype(np.float32)
    means = np.zeros((len(ys), d))
    for n, y in enumerate(ys):
        r = step_multinomial(params, N, seed, n, y, x)
        means[n] = r["filter"][:d]
        x = r["xhat"].astype(np.float32)
    return means


# ----------------------------------------------------------------------------- relabelled exchange
def relabel_stage(table: np.ndarray, G: int, t: int):
    """orc_relabel_stage on one cross stage's table (output -> source), returning
    (relabelled table, excess[G])."""
    a = np.ascontiguousarray(table, dtype=np.int32).copy()
    ex = np.zeros(G, np.uint64)
    rc = lib().orc_relabel_stage(a.size, G, int(t), _ptr(a), _ptr(ex))
    if rc != 0:
        raise ValueError(f"orc_relabel_stage rc={rc}")
    return a, ex.astype(np.int64)


def augmented_resample_relabel(lw: np.ndarray, M: int, G: int, seed: int, n: int) -> dict:
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    N = lw.shape[0]
    m = N // M
    S, L = int(round(np.log2(m))), int(round(np.log2(G)))
    out = dict(a=np.zeros((S, N), np.int32), delta=np.zeros((S, N), np.float32), logV=np.zeros(m - 1),
               A=np.zeros(N, np.int64), excess=np.zeros((L, G), np.uint64))
    rc = lib().orc_augmented_resample_relabel(N, M, G, seed, n, _ptr(lw), _ptr(out["a"]), _ptr(out["delta"]),
                                              _ptr(out["logV"]), _ptr(out["A"]), _ptr(out["excess"]))
    if rc != 0:
        raise ValueError(f"orc_augmented_resample_relabel rc={rc}")
    out["excess"] = out["excess"].astype(np.int64)
    return out


def step_relabel(params: dict, N: int, M: int, G: int, seed: int, n: int, y: np.ndarray, xin: np.ndarray) -> dict:
    """One step with the relabelled exchange on G shards (orc_step_relabel)."""
    mdl = make_model(params)
    d = mdl.d
    m = N // M
    S, L = int(round(np.log2(m))), int(round(np.log2(G)))
    xin = np.ascontiguousarray(xin, dtype=np.float32).reshape(N, d)
    yy = np.ascontiguousarray(y, dtype=np.float32)
    out = dict(x=np.zeros((N, d)), lw=np.zeros(N), a=np.zeros((S, N), np.int32), delta=np.zeros((S, N), np.float32),
               logV=np.zeros(m - 1), A=np.zeros(N, np.int64), xhat=np.zeros((N, d)), filter=np.zeros(2 * d),
               predict=np.zeros(2 * d), resampled=np.zeros(2 * d), excess=np.zeros((L, G), np.uint64))
    rc = lib().orc_step_relabel(ctypes.byref(mdl), N, M, G, seed, n, _ptr(yy), _ptr(xin), _ptr(out["x"]),
                                _ptr(out["lw"]), _ptr(out["a"]), _ptr(out["delta"]), _ptr(out["logV"]), _ptr(out["A"]),
                                _ptr(out["xhat"]), _ptr(out["filter"]), _ptr(out["predict"]), _ptr(out["resampled"]),
                                _ptr(out["excess"]))
    if rc != 0:
        raise ValueError(f"orc_step_relabel rc={rc}")
    out["excess"] = out["excess"].astype(np.int64)
    out["S"], out["m"] = S, m
    return out


def run_filter_relabel(params: dict, M: int, m: int, G: int, seed: int, ys: np.ndarray):
    """Alg. 1 + Alg. 3 with the relabelled exchange on G shards; per-step filter means."""
    N = M * m
    d = int(params["d"])
    x = init(params, N, seed).astype(np.float32)
    means = np.zeros((len(ys), d))
    for n, y in enumerate(ys):
        r = step_relabel(params, N, M, G, seed, n, y, x)
        means[n] = r["filter"][:d]
        x = r["xhat"].astype(np.float32)
    return means
