"""Thin Python binding of the C-ABI in include/pf.h (argument marshalling only).

Every step of the filter runs in the CUDA kernels of libpf.so; there is no CPU or
PyTorch fallback: importing this module without the built library raises.
PyTorch is used only for device memory (the workspace tensor) and streams.

The functions carry the C names (pf_init, pf_step, pf_step_dev, pf_estimate,
pf_debug_get, pf_debug_set_state, ...); ParticleFilter wraps them for convenience.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpf.so")
if os.environ.get("PF_LIB"):  # an experiment build of the same sources (tools/build_variant.sh)
    LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ["PF_LIB"]))

PF_OK, PF_EINVAL, PF_EWORKSPACE, PF_ECUDA, PF_EOBS, PF_ESTATE = 0, -1, -2, -3, -4, -5
PF_LG, PF_SV = 1, 2
PF_FLAG_DEBUG = 1
PF_FLAG_ADAPTIVE = 2
PF_FLAG_AIRPF = 4
PF_FLAG_MULTINOMIAL = 8
PF_FLAG_GUARD = 16
PF_PHI_X, PF_PHI_X2 = 1, 2
PF_EST_FILTER, PF_EST_PREDICT, PF_EST_RESAMPLED = 1, 2, 3
PF_DBG_X, PF_DBG_LOGW, PF_DBG_ANC_STAGE, PF_DBG_ANC_FINAL, PF_DBG_XHAT, PF_DBG_LOGV, PF_DBG_THRESH = 1, 2, 3, 4, 5, 6, 7
PF_DBG_ESS = 8
PF_DBG_ISLAND_A, PF_DBG_ISLAND_CHOICE, PF_DBG_ISLAND_LOGW = 9, 10, 11


class PFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pf error {code}: {msg}")
        self.code = code


class pf_model(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("d", ctypes.c_int), ("dy", ctypes.c_int),
                ("A", ctypes.c_void_p), ("LQ", ctypes.c_void_p), ("H", ctypes.c_void_p),
                ("Rinv", ctypes.c_void_p), ("m0", ctypes.c_void_p), ("L0", ctypes.c_void_p),
                ("sv_phi", ctypes.c_float), ("sv_sigma", ctypes.c_float), ("sv_beta", ctypes.c_float),
                ("sv_m0", ctypes.c_float), ("sv_s0", ctypes.c_float)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libpf.so; raises if it has not been built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, u32, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t
        L.pf_workspace_bytes.argtypes = [vp, u64, u32, u32]
        L.pf_workspace_bytes.restype = sz
        L.pf_init.argtypes = [vp, u64, u32, u64, u32, vp, sz, vp, ctypes.POINTER(vp)]
        L.pf_step.argtypes = [vp, vp]
        L.pf_step_dev.argtypes = [vp, vp]
        L.pf_estimate.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
        L.pf_destroy.argtypes = [vp]
        L.pf_destroy.restype = None
        L.pf_last_error.argtypes = [vp]
        L.pf_last_error.restype = ctypes.c_char_p
        L.pf_debug_get.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, sz]
        L.pf_debug_ptr.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
        L.pf_debug_set_state.argtypes = [vp, vp, u32]
        L.pf_last_step_launches.argtypes = [vp]
        L.pf_timing_enable.argtypes = [vp, ctypes.c_int]
        L.pf_timing_read.argtypes = [vp, vp, vp]
        L.pf_workspace_bytes_sharded.argtypes = [vp, u64, u32, u32, ctypes.c_int]
        L.pf_workspace_bytes_sharded.restype = sz
        L.pf_init_sharded.argtypes = [vp, u64, u32, u64, u32, ctypes.c_int, ctypes.c_int, vp, sz, vp,
                                      ctypes.POINTER(vp)]
        L.pf_step_local.argtypes = [vp, vp, vp]
        L.pf_shard_record.argtypes = [vp, ctypes.POINTER(vp)]
        L.pf_step_top.argtypes = [vp, vp]
        L.pf_cross_buffer.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(sz)]
        L.pf_cross_stage.argtypes = [vp, ctypes.c_int, vp]
        L.pf_set_adaptive.argtypes = [vp, ctypes.c_double]
        L.pf_last_stages.argtypes = [vp]
        L.pf_set_airpf.argtypes = [vp, ctypes.c_int]
        L.pf_set_multinomial.argtypes = [vp, ctypes.c_int]
        L.pf_set_rotation.argtypes = [vp, ctypes.c_int]
        L.pf_cross_pull_plan.argtypes = [vp, vp]
        L.pf_cross_pull_pack.argtypes = [vp, vp, ctypes.POINTER(vp)]
        L.pf_cross_pull_serve.argtypes = [vp, vp, u64, ctypes.POINTER(vp)]
        L.pf_cross_pull_finish.argtypes = [vp, vp]
        L.pf_rotation_offset.argtypes = [vp]
        L.pf_peer_export.argtypes = [vp, vp, vp]
        L.pf_peer_open.argtypes = [vp, vp, vp]
        L.pf_peer_set.argtypes = [vp, vp]
        L.pf_cross_peer.argtypes = [vp]
        L.pf_guard_check.argtypes = [vp, ctypes.c_ubyte, vp]
        L.pf_run_dev.argtypes = [vp, vp, ctypes.c_uint32, vp]
        L.pf_graph_capture.argtypes = [vp, vp, ctypes.c_uint32, vp]
        L.pf_graph_launch.argtypes = [vp]
        L.pf_island_map.argtypes = [vp, ctypes.POINTER(vp)]
        L.pf_island_cross.argtypes = [vp, ctypes.c_int, vp]
        L.pf_step_local_begin.argtypes = [vp, vp, vp]
        L.pf_step_local_end.argtypes = [vp]
        L.pf_relabel_begin.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(vp), vp, vp]
        L.pf_relabel_end.argtypes = [vp, ctypes.c_int, vp]
        _lib = L
    return _lib


EXPORTED = ["pf_workspace_bytes", "pf_init", "pf_step", "pf_step_dev", "pf_estimate", "pf_destroy",
            "pf_last_error", "pf_debug_get", "pf_debug_ptr", "pf_debug_set_state", "pf_last_step_launches",
            "pf_timing_enable", "pf_timing_read", "pf_workspace_bytes_sharded", "pf_init_sharded",
            "pf_step_local", "pf_shard_record", "pf_step_top", "pf_cross_buffer", "pf_cross_stage",
            "pf_set_adaptive", "pf_last_stages", "pf_set_airpf", "pf_set_multinomial", "pf_set_rotation",
            "pf_rotation_offset", "pf_cross_pull_plan", "pf_cross_pull_pack", "pf_cross_pull_serve",
            "pf_cross_pull_finish", "pf_peer_export", "pf_peer_open", "pf_peer_set", "pf_cross_peer",
            "pf_guard_check", "pf_run_dev", "pf_relabel_begin", "pf_relabel_end",
            "pf_step_local_begin", "pf_step_local_end", "pf_island_map", "pf_island_cross",
            "pf_graph_capture", "pf_graph_launch"]
PF_IPC_HANDLE_BYTES = 64
GUARD_BYTES = 1 << 16  # guard band behind a poisoned workspace (ParticleFilter(poison=...))
PF_KERNEL_KINDS = 5
KERNEL_NAMES = ("k_pass1", "k_cascade", "k_stages", "k_top", "k_cross")


def _check(rc: int, h=None):
    if rc != PF_OK:
        msg = lib().pf_last_error(h)
        raise PFError(rc, msg.decode() if msg else "")


def make_model(params: dict):
    """pf_model from inputs.model_params(); returns (struct, keepalive arrays)."""
    keep = []
    m = pf_model()
    m.kind = int(params["kind"])
    m.d = int(params["d"])
    m.dy = int(params["dy"])
    if m.kind == PF_SV:
        m.sv_phi, m.sv_sigma, m.sv_beta = float(params["phi"]), float(params["sigma"]), float(params["beta"])
        m.sv_m0, m.sv_s0 = float(params["m0"]), float(params["s0"])
    else:
        for name in ("A", "LQ", "H", "Rinv", "m0", "L0"):
            arr = np.ascontiguousarray(params[name], dtype=np.float32)
            keep.append(arr)
            setattr(m, name, arr.ctypes.data)
    return m, keep


def pf_workspace_bytes(params: dict, N: int, M: int, flags: int = 0) -> int:
    m, keep = make_model(params)
    return int(lib().pf_workspace_bytes(ctypes.byref(m), N, M, flags))


def pf_init(params: dict, N: int, M: int, seed: int, flags: int, ws_ptr: int, ws_bytes: int, stream_ptr: int):
    m, keep = make_model(params)
    h = ctypes.c_void_p()
    _check(lib().pf_init(ctypes.byref(m), N, M, seed, flags, ws_ptr, ws_bytes, stream_ptr, ctypes.byref(h)))
    return h


def pf_step(h, y: np.ndarray):
    yy = np.ascontiguousarray(y, dtype=np.float32)
    _check(lib().pf_step(h, yy.ctypes.data), h)


def pf_step_dev(h, y_dev_ptr: int):
    _check(lib().pf_step_dev(h, y_dev_ptr), h)


def pf_estimate(h, d: int, phi: int = PF_PHI_X, kind: int = PF_EST_FILTER) -> np.ndarray:
    out = np.zeros(d, np.float64)
    _check(lib().pf_estimate(h, phi, kind, out.ctypes.data), h)
    return out


def pf_destroy(h):
    lib().pf_destroy(h)


def pf_debug_ptr(h, what: int, stage: int = 0) -> int:
    p = ctypes.c_void_p()
    _check(lib().pf_debug_ptr(h, what, stage, ctypes.byref(p)), h)
    return int(p.value)


def pf_set_adaptive(h, theta: float):
    _check(lib().pf_set_adaptive(h, float(theta)), h)


def pf_set_airpf(h, mode: int):
    _check(lib().pf_set_airpf(h, int(mode)), h)


def pf_set_multinomial(h, on: bool):
    _check(lib().pf_set_multinomial(h, 1 if on else 0), h)


def pf_set_rotation(h, on: bool):
    _check(lib().pf_set_rotation(h, 1 if on else 0), h)


def pf_last_stages(h) -> int:
    return int(lib().pf_last_stages(h))


def pf_debug_set_state(h, xhat: np.ndarray, n: int):
    x = np.ascontiguousarray(xhat, dtype=np.float32)
    _check(lib().pf_debug_set_state(h, x.ctypes.data, n), h)


class ParticleFilter:
    """One filter on one GPU: workspace in a torch uint8 tensor, work on a torch stream."""

    def __init__(self, params: dict, N: int, M: int, seed: int, debug: bool = False, device: str = "cuda",
                 stream=None, theta: float = 0.0, airpf: int = 0, multinomial: bool = False,
                 rotate: bool = False, poison: Optional[int] = None):
        """theta > 0: fully adapted augmented resampling with ESS threshold theta
        (pf_set_adaptive); airpf = 1 (Alg. 7) or 2 (Alg. 6): AIRPF (pf_set_airpf);
        multinomial: the plain BPF, Alg. 2 (pf_set_multinomial); rotate (with theta): stage
        rotation (pf_set_rotation).  The handle then reserves the buffers of that scheme.
        poison (a byte, checking aid): fill the workspace with it before pf_init, with a
        gap after every region (PF_FLAG_GUARD) and a band behind it (guard_intact()) --
        results must not depend on the byte."""
        import torch

        self.torch = torch
        self.params = params
        self.N, self.M, self.seed = int(N), int(M), int(seed)
        self.d = int(params["d"])
        self.dy = int(params["dy"])
        self.m = self.N // self.M
        self.S = int(round(np.log2(self.m)))
        self.flags = ((PF_FLAG_DEBUG if debug else 0) | (PF_FLAG_ADAPTIVE if theta > 0 else 0) |
                      (PF_FLAG_AIRPF if airpf else 0) | (PF_FLAG_MULTINOMIAL if multinomial else 0) |
                      (PF_FLAG_GUARD if poison is not None else 0))
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        nbytes = pf_workspace_bytes(params, self.N, self.M, self.flags)
        if nbytes == 0:
            raise PFError(PF_EINVAL, "invalid model/topology (pf_workspace_bytes returned 0)")
        self._guard = GUARD_BYTES if poison is not None else 0
        self.ws = torch.empty(nbytes + 256 + self._guard, dtype=torch.uint8, device=self.device)
        if poison is not None:
            self.ws.fill_(int(poison) & 0xFF)
            self._poison = int(poison) & 0xFF
        base = self.ws.data_ptr()
        self._off = (-base) % 256
        self.ws_ptr = base + self._off
        self.ws_bytes = nbytes
        self.h = pf_init(params, self.N, self.M, self.seed, self.flags, self.ws_ptr, nbytes, self.stream.cuda_stream)
        if theta > 0:
            pf_set_adaptive(self.h, theta)
            if rotate:
                pf_set_rotation(self.h, True)
        if airpf:
            pf_set_airpf(self.h, airpf)
        if multinomial:
            pf_set_multinomial(self.h, True)

    def guard_intact(self) -> bool:
        """With poison: the gaps between the workspace regions (PF_FLAG_GUARD, pf_guard_check)
        and the band behind the workspace still hold the poison byte."""
        if not self._guard:
            return True
        bad = np.zeros(1, np.uint64)
        _check(lib().pf_guard_check(self.h, self._poison, bad.ctypes.data), self.h)
        tail = self.ws[self._off + self.ws_bytes: self._off + self.ws_bytes + self._guard]
        return int(bad[0]) == 0 and bool((tail == self._poison).all().item())

    def rotation_offset(self) -> int:
        return int(lib().pf_rotation_offset(self.h))

    def last_stages(self) -> int:
        """S* of the last step (S for a plain step)."""
        return pf_last_stages(self.h)

    def close(self):
        if getattr(self, "h", None) is not None:
            pf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, y: np.ndarray):
        pf_step(self.h, y)

    def step_dev(self, y_dev):
        """y_dev: a CUDA tensor (float32, dy entries, contiguous)."""
        pf_step_dev(self.h, y_dev.data_ptr())

    def estimate(self, phi: int = PF_PHI_X, kind: int = PF_EST_FILTER) -> np.ndarray:
        return pf_estimate(self.h, self.d, phi, kind)

    def launches(self) -> int:
        return int(lib().pf_last_step_launches(self.h))

    def timing_enable(self, on: bool = True):
        _check(lib().pf_timing_enable(self.h, 1 if on else 0), self.h)

    def timing_read(self):
        """{kernel name: (summed ms, launches)} since the last enable/read."""
        ms = np.zeros(PF_KERNEL_KINDS, np.float64)
        n = np.zeros(PF_KERNEL_KINDS, np.int32)
        _check(lib().pf_timing_read(self.h, ms.ctypes.data, n.ctypes.data), self.h)
        return {KERNEL_NAMES[k]: (float(ms[k]), int(n[k])) for k in range(PF_KERNEL_KINDS)}

    def debug_tensor(self, what: int, stage: int = 0):
        """Device view (torch tensor into the workspace) of a debug table."""
        torch = self.torch
        ptr = pf_debug_ptr(self.h, what, stage)
        off = ptr - self.ws.data_ptr()
        if what in (PF_DBG_X, PF_DBG_XHAT):
            n, dt, shape = self.N * self.d * 4, torch.float32, (self.N, self.d)
        elif what == PF_DBG_LOGW:
            n, dt, shape = self.N * 4, torch.float32, (self.N,)
        elif what in (PF_DBG_ANC_STAGE, PF_DBG_ANC_FINAL):
            n, dt, shape = self.N * 4, torch.int32, (self.N,)
        elif what == PF_DBG_LOGV:
            n, dt, shape = (self.m - 1) * 8, torch.float64, (self.m - 1,)
        elif what == PF_DBG_THRESH:
            n, dt, shape = (self.m - 1) * 4, torch.int32, (self.m - 1,)
        elif what == PF_DBG_ESS:
            n, dt, shape = (self.S + 1) * 8, torch.float64, (self.S + 1,)
        elif what == PF_DBG_ISLAND_A:
            n, dt, shape = self.m * 4, torch.int32, (self.m,)
        elif what == PF_DBG_ISLAND_CHOICE:
            n, dt, shape = (self.m + 3) // 4, torch.uint8, ((self.m + 3) // 4,)
        elif what == PF_DBG_ISLAND_LOGW:
            n, dt, shape = self.m * 8, torch.float64, (self.m,)
        else:
            raise ValueError(what)
        return self.ws[off: off + n].view(dt).view(shape)

    def debug_get(self, what: int, stage: int = 0) -> np.ndarray:
        t = self.debug_tensor(what, stage)
        self.stream.synchronize()
        out = t.cpu().numpy()
        if what == PF_DBG_THRESH:
            out = out.view(np.uint32)
        return out

    def run_dev(self, y_dev, estimates: bool = True):
        """len(y_dev) consecutive steps (pf_run_dev); y_dev: device fp32 tensor (T, dy).
        Returns a device fp64 tensor (T, 4, d): filter x, filter x^2, predictive x,
        predictive x^2 after every step (or None with estimates=False)."""
        torch = self.torch
        y = y_dev.contiguous()
        T = int(y.shape[0])
        out = torch.empty((T, 4, self.d), dtype=torch.float64, device=self.device) if estimates else None
        _check(lib().pf_run_dev(self.h, y.data_ptr(), T, out.data_ptr() if out is not None else None), self.h)
        self._keep_y = y
        return out

    def graph_capture(self, y_dev, estimates: bool = False):
        """Capture len(y_dev) steps into one CUDA graph (pf_graph_capture); launch it with
        graph_launch().  Returns the device estimate rows tensor (or None)."""
        torch = self.torch
        y = y_dev.contiguous()
        T = int(y.shape[0])
        out = torch.empty((T, 4, self.d), dtype=torch.float64, device=self.device) if estimates else None
        _check(lib().pf_graph_capture(self.h, y.data_ptr(), T, out.data_ptr() if out is not None else None), self.h)
        self._keep_gy = (y, out)
        return out

    def graph_launch(self):
        _check(lib().pf_graph_launch(self.h), self.h)

    def set_state(self, xhat: np.ndarray, n: int):
        pf_debug_set_state(self.h, np.asarray(xhat, np.float32).reshape(self.N, self.d), n)
