"""The peer-memory exchange through real CUDA IPC mappings (include/pf.h pf_peer_export /
pf_peer_open / pf_cross_peer): two rank processes share this one GPU, map each other's
workspace, and run the sharded step with exchange="peer"; every rank's x_hat and the
estimates must equal the single-GPU run BITWISE.

The ranks' kernels never wait on one another (B200_PROFILING.md: no spinning kernels
across processes on one GPU): the ordering comes from host-side gloo collectives after a
stream synchronisation.  Across GPUs the same code path runs with NCCL device barriers."""
import os
import socket

import numpy as np
import pytest

from paper_1812_01502_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

CASES = [("C4", 1 << 16, 64, 2), ("C3", 1 << 14, 8, 2)]


def _worker(rank, world, port, q, name, N, M):
    try:
        from paper_1812_01502_b200 import dist as pfd
        from paper_1812_01502_b200 import pf as pfb

        class HostGatherTransport(pfd.TorchTransport):
            """gloo transport for device tensors: records all-gathered through host memory."""

            def allgather(self, rec):
                torch.cuda.current_stream().synchronize()
                out = super().allgather(rec.cpu())
                return out.to("cuda")

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = inputs.CONFIGS[name]
        p = inputs.model_params(cfg)
        _, ys = inputs.simulate(cfg, T=3)
        be = pfd.LibBackend(p, N, M, 33, rank, world, debug=True)
        tr = HostGatherTransport()
        assert pfd.peer_connect(be, tr)
        out = []
        for y in ys:
            pfd.sharded_step(be, tr, y, exchange="peer")
            out.append((be.debug_get(pfb.PF_DBG_XHAT), be.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER)))
        tr.device_barrier(be.stream)
        be.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("name,N,M,G", CASES)
def test_peer_exchange_ipc_two_processes(name, N, M, G):
    from paper_1812_01502_b200 import pf as pfb
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, q, name, N, M)) for r in range(G)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
    for r in range(G):
        assert not isinstance(res[r], str), res[r]
    cfg = inputs.CONFIGS[name]
    p = inputs.model_params(cfg)
    _, ys = inputs.simulate(cfg, T=3)
    single = pfb.ParticleFilter(p, N, M, 33, debug=True)
    for n, y in enumerate(ys):
        single.step(y)
        xs = single.debug_get(pfb.PF_DBG_XHAT).reshape(N, -1)
        xg = np.concatenate([res[r][n][0] for r in range(G)])
        assert np.array_equal(xs, xg), n
        e1 = single.estimate(pfb.PF_PHI_X, pfb.PF_EST_FILTER)
        for r in range(G):
            assert np.array_equal(res[r][n][1], e1), (n, r)
    single.close()
