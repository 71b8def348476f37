"""The overlapped local phase of the sharded step (dist._local_overlapped; include/pf.h
pf_step_local_begin / pf_step_local_end): the shard records are gathered on a side stream
while the k_stages passes run, and k_top waits for both through stream events.  G ranks are
host threads on one GPU with a transport that gathers device records through a host
barrier (nothing on the GPU waits for another rank); the result must be bitwise the one-GPU
run, for the pairwise, pull and peer exchanges (the peer gather reads the owners' states in
place, so the overlapped path adds a device barrier after the local stage passes)."""
import threading

import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_1812_01502_b200 import dist as pfd  # noqa: E402
from paper_1812_01502_b200 import pf as pfb  # noqa: E402


class ThreadTransport:
    """NCCL-like (device tensors, stream-ordered) transport between host threads."""
    nccl = True

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    def _swap(self, key, val):
        self.sh["bar"].wait()
        self.sh.setdefault(key, {})[self.rank] = val
        self.sh["bar"].wait()
        out = dict(self.sh[key])
        self.sh["bar"].wait()
        if self.rank == 0:
            self.sh.pop(key, None)
        self.sh["bar"].wait()
        return out

    def allgather(self, rec):
        torch.cuda.current_stream().synchronize()  # the record is on this stream's timeline
        got = self._swap("ag", rec.clone())
        return torch.stack([got[r] for r in range(self.world)])

    def exchange(self, send, peer):
        torch.cuda.current_stream().synchronize()
        got = self._swap("ex", send.clone())
        return got[peer].clone()

    def all_to_all(self, send, send_splits, recv_splits):
        torch.cuda.current_stream().synchronize()
        got = self._swap("a2a", (send.clone(), [int(v) for v in send_splits]))
        parts = []
        for r in range(self.world):
            buf, splits = got[r]
            off = sum(splits[: self.rank])
            parts.append(buf[off: off + splits[self.rank]])
        return torch.cat(parts)

    def device_barrier(self, stream=None):
        (stream or torch.cuda.current_stream()).synchronize()
        self.sh["bar"].wait()


@pytest.mark.parametrize("exchange", ["pairwise", "pull", "peer"])
@pytest.mark.parametrize("name,N,M,G", [("C4", 1 << 16, 64, 2), ("C3", 1 << 15, 32, 4)])
def test_overlapped_local_phase_is_bitwise(name, N, M, G, exchange):
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=3)
    single = pfb.ParticleFilter(p, N, M, 13)
    ref = []
    for y in ys:
        single.step(y)
        ref.append((single.estimate(), single.debug_get(pfb.PF_DBG_XHAT).copy()))
    single.close()
    shared = {"bar": threading.Barrier(G)}
    out = [None] * G
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            b = pfd.LibBackend(p, N, M, 13, r, G, stream=st)
            tr = ThreadTransport(r, G, shared)
            if exchange == "peer":  # every rank's workspace is addressable on this GPU
                got = tr._swap("ws", b.ws_ptr)
                b.peer_set([got[q] for q in range(G)])
            res = []
            for y in ys:
                pfd.sharded_step(b, tr, y, exchange=exchange)
                st.synchronize()
                res.append((b.estimate(), b.debug_get(pfb.PF_DBG_XHAT).copy()))
            b.close()
            out[r] = res
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))
            shared["bar"].abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    nloc = N // G
    for n in range(len(ys)):
        for r in range(G):
            assert np.array_equal(out[r][n][0], ref[n][0]), (n, r)
            assert np.array_equal(out[r][n][1], ref[n][1][r * nloc:(r + 1) * nloc]), (n, r)


def test_begin_end_errors():
    cfg = inputs.CONFIGS["C1"]
    p = inputs.model_params(cfg)
    b = pfd.LibBackend(p, 1024, 16, 1, 0, 2)
    with pytest.raises(pfb.PFError):
        b.step_local_end()  # no begin
    b.step_local_begin(np.zeros(1, np.float32))
    with pytest.raises(pfb.PFError):
        b.step_local_begin(np.zeros(1, np.float32))  # end pending
    b.step_local_end()
    b.close()
    f = pfb.ParticleFilter(p, 1024, 16, 1)
    with pytest.raises(pfb.PFError):
        pfb._check(pfb.lib().pf_step_local_begin(f.h, np.zeros(1, np.float32).ctypes.data, None), f.h)
    f.close()
