"""The NCCL branch of the transport (dist.TorchTransport) on an NCCL process group of ONE
rank on this GPU: every collective the multi-GPU step issues (all_gather_into_tensor,
batch_isend_irecv -- here to the rank itself --, all_to_all_single, the 1-element all-reduce
device barrier) executes on NCCL on a non-default stream and returns what it must.

One rank is all one GPU allows (NCCL refuses two ranks on one device, and the library
refuses a sharded handle of world 1), so this covers the transport's NCCL calls and their
stream ordering, not the sharded step over NVLink: that step's kernels are compared with
the oracle through loopback shards, thread ranks and IPC processes (tests/test_gpu_sharded.py,
test_gpu_overlap.py, test_gpu_peer_ipc.py)."""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(port, q):
    try:
        import torch.distributed as dist
        from paper_1812_01502_b200 import dist as pfd
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        tr = pfd.TorchTransport()
        assert tr.nccl and tr.world == 1
        out = {}
        st = torch.cuda.Stream()  # every transport primitive once, on a non-default stream
        with torch.cuda.stream(st):
            rec = torch.arange(12, dtype=torch.float64, device="cuda").reshape(3, 4)
            out["allgather"] = tr.allgather(rec).cpu().numpy()
            send = torch.arange(1000, dtype=torch.uint8, device="cuda")
            out["exchange"] = tr.exchange(send, 0).cpu().numpy()
            out["sendrecv"] = tr.sendrecv(send[:77], 77, 0).cpu().numpy()
            out["sendrecv0"] = tr.sendrecv(send[:0], 0, 0).cpu().numpy()
            out["a2a"] = tr.all_to_all(send, [1000], [1000]).cpu().numpy()
            tr.device_barrier(st)
            tr.device_barrier(st)
            st.synchronize()
            out["bar"] = float(tr._bar.item())
        out["objs"] = tr.allgather_object(("x", 3))
        dist.destroy_process_group()
        q.put(out)
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(repr(e) + "\n" + traceback.format_exc())


def _run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_worker, args=(_free_port(), q))
    pr.start()
    res = q.get(timeout=600)
    pr.join(timeout=120)
    assert not isinstance(res, str), res
    return res


def test_transport_primitives_on_nccl():
    res = _run()
    assert np.array_equal(res["allgather"], np.arange(12, dtype=np.float64).reshape(1, 3, 4))
    ref = (np.arange(1000) % 256).astype(np.uint8)
    assert np.array_equal(res["exchange"], ref)
    assert np.array_equal(res["sendrecv"], ref[:77])
    assert res["sendrecv0"].size == 0
    assert np.array_equal(res["a2a"], ref)
    assert res["bar"] == 0.0
    assert res["objs"] == [("x", 3)]
