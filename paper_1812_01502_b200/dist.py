"""Multi-GPU orchestration of the sharded BPF step.

G = 2^L ranks, one GPU each; rank r owns particles [r N/G, (r+1) N/G).  One time step:

    local      pf_step_local: mutate, weight, stages 1..S_loc (S_loc = S - L), all on-GPU
    allgather  the G shard records {log V_{S_loc}, estimate partial}      (8 (3+4d) B each)
    top        pf_step_top: V levels S_loc+1..S, cross thresholds, global estimate,
               identical on every rank (same fp64 operations as one GPU)
    cross      for t = 1..L: exchange the stage-(S_loc+t-1) state buffer with
               partner = rank ^ 2^(t-1) (the butterfly partner of PAPER.md:562-568,
               hypercube remark PAPER.md:1311), then pf_cross_stage(t)

The orchestration is written against a small Backend interface (the C-ABI library on a
GPU; tests substitute a CPU stand-in) and a Transport (torch.distributed over NCCL on
GPUs, gloo on CPU, or an in-process loopback that runs G shards on one GPU).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np


def partner(rank: int, t: int) -> int:
    """Partner rank at cross stage t (1-based): the ranks differ in bit t-1."""
    return rank ^ (1 << (t - 1))


def cross_stage_of(S: int, L: int, t: int) -> int:
    """Global stage number of cross stage t (1..L)."""
    return S - L + t


def exchange_schedule(world: int) -> List[List[tuple]]:
    """Per cross stage, the list of (rank, partner) pairs: a perfect matching of ranks."""
    L = world.bit_length() - 1
    if world < 1 or (1 << L) != world:
        raise ValueError("world must be a power of two")
    out = []
    for t in range(1, L + 1):
        pairs = sorted({(min(r, partner(r, t)), max(r, partner(r, t))) for r in range(world)})
        out.append(pairs)
    return out


# ----------------------------------------------------------------------------- transports
class TorchTransport:
    """torch.distributed transport: all_gather for the records, isend/irecv pairs for the
    state exchange (NCCL over NVLink on GPUs; gloo on CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

        self.nccl = dist.get_backend(group) == "nccl"
        self._recv = {}

    def allgather(self, rec):
        import torch
        if self.nccl:
            out = torch.empty((self.world,) + tuple(rec.shape), dtype=rec.dtype, device=rec.device)
            self.dist.all_gather_into_tensor(out, rec.contiguous(), group=self.group)
            return out
        outs = [torch.empty_like(rec) for _ in range(self.world)]
        self.dist.all_gather(outs, rec, group=self.group)
        return torch.stack(outs)

    def exchange(self, send, peer: int):
        import torch
        key = (send.numel(), send.dtype, str(send.device), peer)
        recv = self._recv.get(key)  # reused receive buffer: no per-step allocation
        if recv is None:
            recv = self._recv[key] = torch.empty_like(send)
        if self.nccl:
            ops = [self.dist.P2POp(self.dist.isend, send, peer, group=self.group),
                   self.dist.P2POp(self.dist.irecv, recv, peer, group=self.group)]
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        else:
            reqs = [self.dist.isend(send, peer, group=self.group), self.dist.irecv(recv, peer, group=self.group)]
            for r in reqs:
                r.wait()
        return recv


    def sendrecv(self, send, n_recv: int, peer: int):
        """Variable-size exchange with one peer: send the 1-D tensor `send` (may be empty),
        receive n_recv elements of its dtype (NCCL over NVLink on GPUs, gloo on CPU)."""
        import torch
        recv = torch.empty(int(n_recv), dtype=send.dtype, device=send.device)
        ops = []
        if self.nccl:
            if send.numel():
                ops.append(self.dist.P2POp(self.dist.isend, send.contiguous(), peer, group=self.group))
            if n_recv:
                ops.append(self.dist.P2POp(self.dist.irecv, recv, peer, group=self.group))
            if ops:
                for r in self.dist.batch_isend_irecv(ops):
                    r.wait()
        else:
            reqs = []
            if send.numel():
                reqs.append(self.dist.isend(send.contiguous(), peer, group=self.group))
            if n_recv:
                reqs.append(self.dist.irecv(recv, peer, group=self.group))
            for r in reqs:
                r.wait()
        return recv

    def allgather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def device_barrier(self, stream=None):
        """Every rank's work enqueued so far on `stream` is complete before anything enqueued
        after it runs: a 1-element NCCL all-reduce on the stream (no host synchronisation);
        with gloo a stream synchronisation and a host barrier."""
        import torch
        if self.nccl:
            if getattr(self, "_bar", None) is None:
                self._bar = torch.zeros(1, dtype=torch.float32, device="cuda")
            with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
                self.dist.all_reduce(self._bar, group=self.group)
        else:
            if stream is not None:
                stream.synchronize()
            self.dist.barrier(group=self.group)

    def all_to_all(self, send, send_splits, recv_splits):
        """One all-to-all of a 1-D tensor: send_splits[r] elements to rank r (in rank order),
        recv_splits[r] elements from rank r.  NCCL over NVLink on GPUs, gloo on CPU."""
        import torch
        out = torch.empty(int(sum(recv_splits)), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(out, send.contiguous(), output_split_sizes=[int(v) for v in recv_splits],
                                    input_split_sizes=[int(v) for v in send_splits], group=self.group)
        return out


# ----------------------------------------------------------------------------- backend
class LibBackend:
    """One shard on the current GPU through the C-ABI (libpf.so)."""

    def __init__(self, params: dict, N: int, M: int, seed: int, rank: int, world: int, debug: bool = False,
                 stream=None, poison: Optional[int] = None, airpf: int = 0):
        """poison (a byte, checking aid): as pf.ParticleFilter -- fill the workspace before
        pf_init_sharded and keep a guard band behind it (guard_intact())."""
        import torch

        from . import pf

        self.torch = torch
        self.pf = pf
        self.params = params
        self.N, self.M, self.rank, self.world = int(N), int(M), int(rank), int(world)
        self.d = int(params["d"])
        self.flags = ((pf.PF_FLAG_DEBUG if debug else 0) | (pf.PF_FLAG_GUARD if poison is not None else 0) |
                      (pf.PF_FLAG_AIRPF if airpf else 0))
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        L = pf.lib()
        m, keep = pf.make_model(params)
        nbytes = int(L.pf_workspace_bytes_sharded(ctypes.byref(m), self.N, self.M, self.flags, self.world))
        if nbytes == 0:
            raise pf.PFError(pf.PF_EINVAL, "invalid sharded topology")
        self._guard = pf.GUARD_BYTES if poison is not None else 0
        self.ws = torch.empty(nbytes + 256 + self._guard, dtype=torch.uint8, device="cuda")
        if poison is not None:
            self.ws.fill_(int(poison) & 0xFF)
            self._poison = int(poison) & 0xFF
        base = self.ws.data_ptr()
        self.ws_ptr = base + ((-base) % 256)
        self.ws_bytes = nbytes
        h = ctypes.c_void_p()
        pf._check(L.pf_init_sharded(ctypes.byref(m), self.N, self.M, seed, self.flags, self.rank, self.world,
                                    self.ws_ptr, nbytes, self.stream.cuda_stream, ctypes.byref(h)))
        self.h = h
        self.rec_len = 3 + 4 * self.d
        self.airpf = int(airpf)
        if airpf:
            pf.pf_set_airpf(h, int(airpf))

    def _view(self, ptr: int, nbytes: int, dtype):
        off = ptr - self.ws.data_ptr()
        return self.ws[off: off + nbytes].view(dtype)

    def step_local_begin(self, y, y_dev=None):
        """k_pass1 + k_cascade: returns this shard's record (final after these two)."""
        if y_dev is None:
            yy = np.ascontiguousarray(y, dtype=np.float32)
            self.pf._check(self.pf.lib().pf_step_local_begin(self.h, yy.ctypes.data, None), self.h)
        else:
            self.pf._check(self.pf.lib().pf_step_local_begin(self.h, None, y_dev.data_ptr()), self.h)
        p = ctypes.c_void_p()
        self.pf._check(self.pf.lib().pf_shard_record(self.h, ctypes.byref(p)), self.h)
        return self._view(int(p.value), 8 * self.rec_len, self.torch.float64)

    def step_local_end(self):
        """The local k_stages passes."""
        self.pf._check(self.pf.lib().pf_step_local_end(self.h), self.h)

    def step_local(self, y):
        yy = np.ascontiguousarray(y, dtype=np.float32)
        self.pf._check(self.pf.lib().pf_step_local(self.h, yy.ctypes.data, None), self.h)
        p = ctypes.c_void_p()
        self.pf._check(self.pf.lib().pf_shard_record(self.h, ctypes.byref(p)), self.h)
        return self._view(int(p.value), 8 * self.rec_len, self.torch.float64)

    def step_top(self, all_recs):
        all_recs = all_recs.contiguous()
        self._keep = all_recs
        self.pf._check(self.pf.lib().pf_step_top(self.h, all_recs.data_ptr()), self.h)

    def cross_buffer(self):
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        self.pf._check(self.pf.lib().pf_cross_buffer(self.h, ctypes.byref(p), ctypes.byref(n)), self.h)
        return self._view(int(p.value), int(n.value), self.torch.uint8)

    def cross_stage(self, t: int, partner_buf):
        self._keep_p = partner_buf
        self.pf._check(self.pf.lib().pf_cross_stage(self.h, t, partner_buf.data_ptr()), self.h)

    # pull exchange (include/pf.h pf_cross_pull_*)
    def pull_plan(self) -> np.ndarray:
        counts = np.zeros(self.world, np.uint64)
        self.pf._check(self.pf.lib().pf_cross_pull_plan(self.h, counts.ctypes.data), self.h)
        return counts.astype(np.int64)

    def pull_pack(self, offsets: np.ndarray):
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        p = ctypes.c_void_p()
        self.pf._check(self.pf.lib().pf_cross_pull_pack(self.h, off.ctypes.data, ctypes.byref(p)), self.h)
        nloc = self.N // self.world
        return self._view(int(p.value), 4 * nloc, self.torch.int32)

    def pull_serve(self, req_in):
        n = int(req_in.numel())
        p = ctypes.c_void_p()
        ptr = req_in.data_ptr() if n else None
        self.pf._check(self.pf.lib().pf_cross_pull_serve(self.h, ptr, n, ctypes.byref(p)), self.h)
        return self._view(int(p.value), 4 * self.d * n, self.torch.uint8)

    def pull_finish(self, states_in):
        self._keep_s = states_in
        self.pf._check(self.pf.lib().pf_cross_pull_finish(self.h, states_in.data_ptr()), self.h)

    # peer-memory exchange (include/pf.h pf_peer_* / pf_cross_peer)
    def peer_export(self):
        hd = np.zeros(self.pf.PF_IPC_HANDLE_BYTES, np.uint8)
        off = np.zeros(1, np.uint64)
        self.pf._check(self.pf.lib().pf_peer_export(self.h, hd.ctypes.data, off.ctypes.data), self.h)
        return hd.tobytes(), int(off[0])

    def peer_open(self, handles, offsets):
        hd = np.frombuffer(b"".join(handles), np.uint8).copy()
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.pf._check(self.pf.lib().pf_peer_open(self.h, hd.ctypes.data, off.ctypes.data), self.h)

    def peer_set(self, workspaces):
        ws = np.ascontiguousarray(workspaces, dtype=np.uint64)
        self.pf._check(self.pf.lib().pf_peer_set(self.h, ws.ctypes.data), self.h)

    def cross_peer(self):
        self.pf._check(self.pf.lib().pf_cross_peer(self.h), self.h)

    # sharded AIRPF (include/pf.h pf_island_map / pf_island_cross)
    def island_map(self):
        p = ctypes.c_void_p()
        self.pf._check(self.pf.lib().pf_island_map(self.h, ctypes.byref(p)), self.h)
        return self._view(int(p.value), 4 * (self.N // self.M // self.world), self.torch.int32)

    def island_cross(self, t: int, partner_map):
        self._keep_m = partner_map
        self.pf._check(self.pf.lib().pf_island_cross(self.h, int(t), partner_map.data_ptr()), self.h)

    def set_airpf(self, mode: int):
        self.pf.pf_set_airpf(self.h, mode)

    # relabelled exchange (include/pf.h pf_relabel_begin / pf_relabel_end)
    def relabel_begin(self, t: int):
        """Returns (send: uint8 view of the surplus states this rank sends, n_recv states)."""
        cnt = np.zeros(2, np.uint64)
        p = ctypes.c_void_p()
        ns, nr = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        self.pf._check(self.pf.lib().pf_relabel_begin(self.h, int(t), cnt.ctypes.data, ctypes.byref(p), ns.ctypes.data,
                                                      nr.ctypes.data), self.h)
        self.last_counts = cnt.astype(np.int64)
        n_send = int(ns[0])
        send = self._view(int(p.value), 4 * self.d * n_send, self.torch.uint8) if n_send else \
            self.torch.empty(0, dtype=self.torch.uint8, device="cuda")
        return send, int(nr[0])

    def relabel_end(self, t: int, recv):
        self._keep_r = recv
        ptr = recv.data_ptr() if recv is not None and recv.numel() else None
        self.pf._check(self.pf.lib().pf_relabel_end(self.h, int(t), ptr), self.h)

    def step_local_dev(self, y_dev):
        self.pf._check(self.pf.lib().pf_step_local(self.h, None, y_dev.data_ptr()), self.h)
        p = ctypes.c_void_p()
        self.pf._check(self.pf.lib().pf_shard_record(self.h, ctypes.byref(p)), self.h)
        return self._view(int(p.value), 8 * self.rec_len, self.torch.float64)

    def timing_enable(self, on: bool = True):
        self.pf._check(self.pf.lib().pf_timing_enable(self.h, 1 if on else 0), self.h)

    def timing_read(self):
        pf = self.pf
        ms = np.zeros(pf.PF_KERNEL_KINDS, np.float64)
        n = np.zeros(pf.PF_KERNEL_KINDS, np.int32)
        pf._check(pf.lib().pf_timing_read(self.h, ms.ctypes.data, n.ctypes.data), self.h)
        return {pf.KERNEL_NAMES[k]: (float(ms[k]), int(n[k])) for k in range(pf.PF_KERNEL_KINDS)}

    def estimate(self, phi=None, kind=None):
        pf = self.pf
        return pf.pf_estimate(self.h, self.d, phi or pf.PF_PHI_X, kind or pf.PF_EST_FILTER)

    def set_state(self, xhat_local: np.ndarray, n: int):
        """This shard's x_hat_{n-1} (N/G x d fp32, HOST): the next step is time step n."""
        nloc = self.N // self.world
        self.pf.pf_debug_set_state(self.h, np.asarray(xhat_local, np.float32).reshape(nloc, self.d), n)

    def debug_get(self, what: int, stage: int = 0) -> np.ndarray:
        pf = self.pf
        ptr = pf.pf_debug_ptr(self.h, what, stage)
        nloc = self.N // self.world
        if what in (pf.PF_DBG_X, pf.PF_DBG_XHAT):
            t = self._view(ptr, nloc * self.d * 4, self.torch.float32).view(nloc, self.d)
        elif what == pf.PF_DBG_LOGW:
            t = self._view(ptr, nloc * 4, self.torch.float32)
        elif what == pf.PF_DBG_ANC_STAGE:
            t = self._view(ptr, nloc * 4, self.torch.int32)
        else:
            raise ValueError(what)
        self.stream.synchronize()
        return t.cpu().numpy()

    def guard_intact(self) -> bool:
        if not self._guard:
            return True
        bad = np.zeros(1, np.uint64)
        self.pf._check(self.pf.lib().pf_guard_check(self.h, self._poison, bad.ctypes.data), self.h)
        off = self.ws_ptr - self.ws.data_ptr() + self.ws_bytes
        return int(bad[0]) == 0 and bool((self.ws[off: off + self._guard] == self._poison).all().item())

    def close(self):
        if getattr(self, "h", None) is not None:
            self.pf.lib().pf_destroy(self.h)
            self.h = None


# ----------------------------------------------------------------------------- steps
def sharded_step(backend, transport, y, y_dev=None, exchange: str = "pairwise") -> None:
    """One collective time step on this rank (every rank calls it with the same y; with
    y_dev the observation is read from device memory).  exchange: "pairwise" (L rounds of
    whole-buffer swaps with the butterfly partner) or "pull" (one all-to-all of exactly
    the states each rank's outputs read) or "peer" (one kernel reads them straight from
    the owners' memory over NVLink; peer_connect first)."""
    with _on_stream(backend):  # every transport call is ordered on the backend's stream
        if hasattr(backend, "step_local_begin") and getattr(transport, "nccl", False) and not getattr(
                backend, "airpf", 0):
            _local_overlapped(backend, transport, y, y_dev)
            if exchange == "peer":
                # the records were gathered BEFORE the stage passes: the owners' states are
                # final only once every rank has passed this barrier (the peer gather reads
                # them in place)
                transport.device_barrier(backend.stream)
        else:
            rec = backend.step_local(y) if y_dev is None else backend.step_local_dev(y_dev)
            backend.step_top(transport.allgather(rec))
        if exchange == "peer":
            peer_exchange(backend, transport)
            return
        if exchange == "pull":
            pull_exchange(backend, transport)
            return
        if exchange == "relabel":
            relabel_exchange(backend, transport)
            return
        if exchange == "island":
            island_exchange(backend, transport)
            return
        world = transport.world
        L = world.bit_length() - 1
        for t in range(1, L + 1):
            buf = backend.cross_buffer()
            recv = transport.exchange(buf, partner(transport.rank, t))
            backend.cross_stage(t, recv)


def _local_overlapped(backend, transport, y, y_dev=None) -> None:
    """The local phase with the records' all-gather off the critical path: after k_pass1 +
    k_cascade the record is final (every V_s is sigma(xi_0)-measurable, Lemma
    facts_about_Vs (a)), so the NCCL all-gather runs on a side stream while
    the k_stages passes run on the backend's; k_top waits for both (stream events)."""
    import torch
    main = backend.stream
    rec = backend.step_local_begin(y, y_dev)
    if not hasattr(backend, "_comm"):
        backend._comm = torch.cuda.Stream(device=rec.device)
        backend._ev = (torch.cuda.Event(), torch.cuda.Event())
    comm, (ev_rec, ev_gather) = backend._comm, backend._ev
    ev_rec.record(main)
    with torch.cuda.stream(comm):
        comm.wait_event(ev_rec)
        allr = transport.allgather(rec)
        ev_gather.record(comm)
    backend.step_local_end()            # the stage passes, concurrent with the all-gather
    main.wait_event(ev_gather)
    allr.record_stream(main)
    backend.step_top(allr)


def _on_stream(backend):
    """Context that makes the backend's CUDA stream torch's current stream, so NCCL
    collectives issued by the transport are stream-ordered after the library's kernels
    (a no-op for CPU stand-ins)."""
    import contextlib
    st = getattr(backend, "stream", None)
    if st is None or not hasattr(st, "cuda_stream"):
        return contextlib.nullcontext()
    import torch
    return torch.cuda.stream(st)


def relabel_exchange(backend, transport) -> None:
    """The L cross stages as relabelled pairwise rounds (include/pf.h pf_relabel_*; DESIGN.md
    reading R24): per stage each rank learns, without communication, which of its outputs
    and of its partner's cross the pair, swaps matched draws, and only the surplus states
    travel (a variable-size send/recv with the butterfly partner)."""
    L = transport.world.bit_length() - 1
    sb = 4 * backend.d
    for t in range(1, L + 1):
        send, n_recv = backend.relabel_begin(t)
        recv = transport.sendrecv(send, n_recv * sb, partner(transport.rank, t))
        backend.relabel_end(t, recv)


def island_exchange(backend, transport) -> None:
    """Sharded AIRPF (include/pf.h pf_island_*; reading R27): the L cross island
    stages exchange only the island maps (m / G int32 per rank and stage); the states move
    when the next step reads its blocks from their owners (peer mapping, peer_connect)."""
    L = transport.world.bit_length() - 1
    for t in range(1, L + 1):
        recv = transport.exchange(backend.island_map(), partner(transport.rank, t))
        backend.island_cross(t, recv)


def pull_exchange(backend, transport) -> None:
    """The L cross stages as one pull (include/pf.h pf_cross_pull_*): composed sources,
    requests to their owners (all-to-all), owners gather, states back (all-to-all)."""
    import torch
    counts = backend.pull_plan()                         # my outputs per owner rank
    cnt = torch.tensor(counts, dtype=torch.int64, device=transport_device(transport))
    asked = transport.all_to_all(cnt, [1] * transport.world, [1] * transport.world).cpu().numpy()
    offsets = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    req = backend.pull_pack(offsets)
    req_in = transport.all_to_all(req, counts, asked)    # positions others read from me
    served = backend.pull_serve(req_in)
    sb = 4 * backend.d                                   # state bytes
    states = transport.all_to_all(served, asked * sb, counts * sb)
    backend.pull_finish(states)


def peer_connect(backend, transport) -> bool:
    """Set-up of the peer-memory exchange: all-gather every rank's (ok, IPC handle, offset)
    ONCE and map the other ranks' workspaces (include/pf.h pf_peer_export / pf_peer_open).
    A rank whose export fails still takes part in the gather, so every rank sees the same
    verdict; the mapping results are agreed in a second gather.  Returns True when every
    rank mapped its peers (else the caller uses another exchange on every rank)."""
    try:
        hd, off = backend.peer_export()
        mine = (True, hd, off)
    except Exception:  # noqa: BLE001 -- any export failure means "no peer exchange here"
        mine = (False, b"", 0)
    got = transport.allgather_object(mine)
    if not all(g[0] for g in got):
        return False
    try:
        backend.peer_open([g[1] for g in got], [g[2] for g in got])
        ok = True
    except Exception:  # noqa: BLE001
        ok = False
    return all(transport.allgather_object(ok))


def peer_exchange(backend, transport) -> None:
    """The L cross stages as one peer-memory gather (pf_cross_peer).  Every rank's
    stage-S_loc states are complete before any rank reads them: the record all-gather
    that precedes pf_step_top completes only after every rank's local passes.  A device
    barrier after the gather keeps every rank's next step from overwriting them early."""
    backend.cross_peer()
    transport.device_barrier(getattr(backend, "stream", None))


def resampled_estimate(backend, transport, phi: int) -> np.ndarray:
    """PF_EST_RESAMPLED of the whole sharded sample: every rank's shard mean (equal shard
    sizes), all-gathered and averaged in rank order (the same value on every rank)."""
    import torch
    loc = backend.estimate(phi, backend.pf.PF_EST_RESAMPLED)
    t = torch.tensor(loc, dtype=torch.float64, device=transport_device(transport))
    allm = transport.allgather(t).cpu().numpy()
    return allm.sum(axis=0) / allm.shape[0]


def loopback_peer(backends: Sequence) -> None:
    """peer_exchange for G shards on one GPU: every shard maps the others' workspaces by
    address; the G gathers are independent stream-ordered kernels."""
    ws = [b.ws_ptr for b in backends]
    for b in backends:
        if getattr(b, "_peer_ws", None) != ws:
            b.peer_set(ws)
            b._peer_ws = ws
    for b in backends:
        b.cross_peer()


def transport_device(transport):
    return "cuda" if getattr(transport, "nccl", False) else "cpu"


def loopback_pull(backends: Sequence) -> None:
    """pull_exchange for G shards on one GPU (the all-to-alls are slices and copies)."""
    import torch
    G = len(backends)
    counts = [b.pull_plan() for b in backends]           # counts[q][r]: rank q's outputs read r
    reqs = []
    for q, b in enumerate(backends):
        off = np.concatenate([[0], np.cumsum(counts[q])[:-1]]).astype(np.int64)
        reqs.append((b.pull_pack(off), off))
    served = []
    for r, b in enumerate(backends):                     # requests to r, in requester order
        parts = [reqs[q][0][int(reqs[q][1][r]): int(reqs[q][1][r] + counts[q][r])] for q in range(G)]
        req_in = torch.cat(parts) if parts else torch.empty(0, dtype=torch.int32, device="cuda")
        served.append((b.pull_serve(req_in.contiguous()).clone(), [int(counts[q][r]) for q in range(G)]))
    sb = 4 * backends[0].d
    for q, b in enumerate(backends):                     # states back, grouped by owner
        parts = []
        for r in range(G):
            buf, per_q = served[r]
            start = sum(per_q[:q]) * sb
            parts.append(buf[start: start + per_q[q] * sb])
        b.pull_finish(torch.cat(parts).contiguous())


def loopback_relabel(backends: Sequence) -> List[np.ndarray]:
    """relabel_exchange for G shards on one GPU: every shard's begin (its lists and its
    surplus sends) runs before any shard's end; the partner's send buffer is the receive
    buffer.  Returns the per-stage surplus counts (L x G states received)."""
    G = len(backends)
    L = G.bit_length() - 1
    recvd = []
    for t in range(1, L + 1):
        sends = [b.relabel_begin(t) for b in backends]
        for r, b in enumerate(backends):
            send_p, _ = sends[partner(r, t)]
            n_recv = sends[r][1]
            assert send_p.numel() == n_recv * 4 * b.d, "surplus sizes disagree between partners"
            b.relabel_end(t, send_p.clone() if n_recv else None)
        recvd.append(np.array([s[1] for s in sends], np.int64))
    return recvd


def loopback_step(backends: Sequence, y, exchange: str = "pairwise") -> None:
    """The same collective sequence for G shards held by one process on one GPU (the
    exchange is a pointer hand-over; every kernel is stream-ordered, none waits on
    another shard's kernel)."""
    import torch
    recs = [b.step_local(y) for b in backends]
    allr = torch.stack([r for r in recs])
    for b in backends:
        b.step_top(allr)
    if exchange == "pull":
        loopback_pull(backends)
        return
    if exchange == "peer":
        loopback_peer(backends)
        return
    if exchange == "relabel":
        for b, r in zip(backends, zip(*loopback_relabel(backends))):
            b.surplus = np.array(r)
        return
    if exchange == "island":
        ws = [b.ws_ptr for b in backends]
        for b in backends:
            if getattr(b, "_peer_ws", None) != ws:
                b.peer_set(ws)
                b._peer_ws = ws
        G = len(backends)
        for t in range(1, G.bit_length()):
            maps = [b.island_map().clone() for b in backends]  # every map taken before any stage
            for r, b in enumerate(backends):
                b.island_cross(t, maps[partner(r, t)])
        return
    world = len(backends)
    L = world.bit_length() - 1
    for t in range(1, L + 1):
        bufs = [b.cross_buffer() for b in backends]  # all inputs taken before any stage runs
        for r, b in enumerate(backends):
            b.cross_stage(t, bufs[partner(r, t)])
