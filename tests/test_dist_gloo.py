"""Multi-rank orchestration of the sharded step (paper_1812_01502_b200/dist.py) with
world_size = 2 over gloo on CPU.  The per-shard compute is a CPU stand-in built from the
oracle (test infrastructure), so this checks the collective sequence itself: records
gathered in rank order, butterfly partners, every cross-stage source lies in the own or
the partner shard, the exchanged buffers, and the final shards = the oracle's x_hat; and
the pull exchange (composed sources, one all-to-all of requests, one of states); and the
peer exchange (handles all-gathered in rank order, every rank reads the owners' state
buffers in place -- stood in for by shared memory-mapped files -- and the barrier keeps
a fast rank from overwriting its buffer before the others have read it)."""
import os
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_01502_b200 import dist as pfd
from paper_1812_01502_b200 import inputs


def test_partners_and_schedule():
    for world in (2, 4, 8, 16):
        L = world.bit_length() - 1
        sched = pfd.exchange_schedule(world)
        assert len(sched) == L
        for t, pairs in enumerate(sched, start=1):
            seen = sorted(r for pr in pairs for r in pr)
            assert seen == list(range(world))  # a perfect matching
            for a, b in pairs:
                assert pfd.partner(a, t) == b and pfd.partner(b, t) == a
                assert a ^ b == 1 << (t - 1)
    assert pfd.cross_stage_of(22, 3, 1) == 20 and pfd.cross_stage_of(22, 3, 3) == 22
    with pytest.raises(ValueError):
        pfd.exchange_schedule(6)


class OracleShard:
    """CPU stand-in for LibBackend: one shard's view of the oracle's full step."""

    def __init__(self, params, N, M, seed, rank, world, peer_dir=None):
        from oracle import oracle as orc
        self.orc = orc
        self.params, self.N, self.M, self.seed = params, N, M, seed
        self.rank, self.world = rank, world
        self.d = int(params["d"])
        self.m = N // M
        self.S = int(np.log2(self.m))
        self.L = world.bit_length() - 1
        self.Sloc = self.S - self.L
        self.nloc = N // world
        self.pos0 = rank * self.nloc
        self.xhat = orc.init(params, N, seed).astype(np.float32)
        self.n = 0
        self.peer_dir = peer_dir
        if peer_dir:  # this shard's "workspace": the state buffer other ranks read in place
            self.mine = np.lib.format.open_memmap(os.path.join(peer_dir, f"ws{rank}.npy"), mode="w+",
                                                  dtype=np.float32, shape=(self.nloc, self.d))

    def _states_at(self, s):
        """Full-problem states at stage s positions: x[a_1(...a_s(i))]."""
        pos = np.arange(self.N)
        for st in range(s, 0, -1):
            pos = self.r["a"][st - 1][pos]
        return self.r["x"][pos].astype(np.float32)

    def step_local(self, y):
        if getattr(self, "relabel", False):  # the relabelled exchange's realisation (R24)
            self.r = self.orc.step_relabel(self.params, self.N, self.M, self.world, self.seed, self.n, y, self.xhat)
        else:
            self.r = self.orc.step(self.params, self.N, self.M, self.seed, self.n, y, self.xhat)
        self.stage = self.Sloc
        self.buf = self._states_at(self.Sloc)[self.pos0: self.pos0 + self.nloc].copy()
        if self.peer_dir:
            self.mine[:] = self.buf
            self.mine.flush()
        lv = self.r["logV"][self.orc.level_offset(self.m, self.Sloc) + self.rank]
        return torch.tensor([lv] + [0.0] * (2 + 4 * self.d), dtype=torch.float64)

    def step_top(self, all_recs):
        for q in range(self.world):
            want = self.r["logV"][self.orc.level_offset(self.m, self.Sloc) + q]
            assert float(all_recs[q][0]) == want, "records not gathered in rank order"

    def cross_buffer(self):
        return torch.from_numpy(self.buf.view(np.uint8).reshape(-1).copy())

    def cross_stage(self, t, recv):
        s = self.Sloc + t
        peer = pfd.partner(self.rank, t)
        pbuf = recv.numpy().view(np.float32).reshape(self.nloc, self.d)
        want = self._states_at(s - 1)[peer * self.nloc:(peer + 1) * self.nloc]
        assert np.array_equal(pbuf, want), "wrong partner buffer"
        a = self.r["a"][s - 1]
        out = np.empty_like(self.buf)
        for l in range(self.nloc):
            src = int(a[self.pos0 + l])
            owner = src // self.nloc
            assert owner in (self.rank, peer), "cross-stage source outside own/partner shard"
            out[l] = self.buf[src - self.pos0] if owner == self.rank else pbuf[src - peer * self.nloc]
        self.buf = out

    # relabelled exchange (dist.relabel_exchange): only the surplus travels
    def relabel_begin(self, t):
        s = self.Sloc + t
        peer = pfd.partner(self.rank, t)
        a = self.r["a"][s - 1]
        mine = np.arange(self.pos0, self.pos0 + self.nloc)
        theirs = np.arange(peer * self.nloc, (peer + 1) * self.nloc)
        # partner outputs (increasing position) that read this shard: their states, in order
        want = [int(a[i]) - self.pos0 for i in theirs if int(a[i]) // self.nloc == self.rank]
        self._remote = [l for l, i in enumerate(mine) if int(a[i]) // self.nloc == peer]
        # the stand-in checks the exchange's own invariants on the oracle's relabelled table
        assert min(len(want), len(self._remote)) == 0, "matched outputs still cross the pair"
        send = self.buf[np.array(want, np.int64)] if want else np.zeros((0, self.d), np.float32)
        self._t = t
        return torch.from_numpy(send.view(np.uint8).reshape(-1).copy()), len(self._remote)

    def relabel_end(self, t, recv):
        assert t == self._t
        s = self.Sloc + t
        a = self.r["a"][s - 1]
        rc = recv.numpy().view(np.float32).reshape(-1, self.d)
        assert rc.shape[0] == len(self._remote), "surplus size mismatch"
        out = np.empty_like(self.buf)
        k = 0
        for l in range(self.nloc):
            src = int(a[self.pos0 + l])
            if src // self.nloc == self.rank:
                out[l] = self.buf[src - self.pos0]
            else:
                out[l] = rc[k]
                k += 1
        self.buf = out

    # pull exchange (dist.pull_exchange)
    def pull_plan(self):
        pos = np.arange(self.pos0, self.pos0 + self.nloc)
        for s in range(self.S, self.Sloc, -1):
            pos = self.r["a"][s - 1][pos]
        self.src_owner = pos // self.nloc
        self.src_local = pos % self.nloc
        return np.bincount(self.src_owner, minlength=self.world).astype(np.int64)

    def pull_pack(self, offsets):
        order = np.argsort(self.src_owner, kind="stable")  # grouped by owner, output order within
        self.outpos = order
        starts = np.concatenate([[0], np.cumsum(np.bincount(self.src_owner, minlength=self.world))[:-1]])
        assert np.array_equal(starts, offsets)
        return torch.from_numpy(self.src_local[order].astype(np.int32))

    def pull_serve(self, req_in):
        idx = req_in.numpy().astype(np.int64)
        assert np.all((idx >= 0) & (idx < self.nloc))
        return torch.from_numpy(self.buf[idx].view(np.uint8).reshape(-1).copy())

    def pull_finish(self, states):
        st = states.numpy().view(np.float32).reshape(self.nloc, self.d)
        out = np.empty_like(self.buf)
        out[self.outpos] = st
        self.buf = out

    # peer exchange (dist.peer_connect / dist.peer_exchange)
    def peer_export(self):
        name = f"ws{self.rank}.npy".encode()
        return name.ljust(64, b"\0"), 0

    def peer_open(self, handles, offsets):
        assert len(handles) == self.world and all(o == 0 for o in offsets)
        names = [h.rstrip(b"\0").decode() for h in handles]
        assert names == [f"ws{q}.npy" for q in range(self.world)], "handles not gathered in rank order"
        self.peers = [np.load(os.path.join(self.peer_dir, nm), mmap_mode="r") for nm in names]

    def cross_peer(self):
        if self.rank:  # rank 0 runs ahead: without the barrier it overwrites its buffer early
            time.sleep(0.3)
        self.pull_plan()
        self.buf = np.stack([np.array(self.peers[o][l]) for o, l in zip(self.src_owner, self.src_local)])

    def finish(self):
        full = self.r["xhat"].astype(np.float32)
        assert np.array_equal(self.buf, full[self.pos0: self.pos0 + self.nloc])
        self.xhat = full
        self.n += 1


class OracleIslandShard:
    """CPU stand-in for a sharded AIRPF LibBackend (dist.island_exchange): the oracle's
    one-GPU AIRPF step (orc_step_airpf) gives every stage's island sources; this shard holds
    the island map of its islands after the local stages (global ids) and applies each cross
    stage from the oracle's table, taking the partner's map entry when the island took the
    partner's block.  The final maps must be the oracle's island map."""

    def __init__(self, params, N, M, seed, rank, world):
        from oracle import oracle as orc
        self.orc, self.params, self.N, self.M, self.seed = orc, params, N, M, seed
        self.rank, self.world = rank, world
        self.m = N // M
        self.S = int(np.log2(self.m))
        self.L = world.bit_length() - 1
        self.mloc = self.m // world
        self.i0 = rank * self.mloc
        self.xhat = orc.init(params, N, seed).astype(np.float32)
        self.n = 0

    def step_local(self, y):
        self.r = self.orc.step_airpf(self.params, self.N, self.M, self.seed, self.n, y, self.xhat, modified=True)
        src = self.r["src"]
        A = np.empty(self.mloc, np.int64)
        for i in range(self.mloc):  # compose the local stages 1..S - L
            c = self.i0 + i
            for s in range(self.S - self.L, 0, -1):
                c = int(src[s - 1][c])
            A[i] = c
        self.A = A
        lv = self.r["logVbar"][self.orc.level_offset(self.m, self.S - self.L) + self.rank]
        return torch.tensor([lv], dtype=torch.float64)

    def step_top(self, all_recs):
        for q in range(self.world):
            want = self.r["logVbar"][self.orc.level_offset(self.m, self.S - self.L) + q]
            assert float(all_recs[q][0]) == want, "records not gathered in rank order"

    def island_map(self):
        return torch.from_numpy(self.A.astype(np.int32).copy())

    def island_cross(self, t, partner_map):
        s = self.S - self.L + t
        peer = pfd.partner(self.rank, t)
        pm = partner_map.numpy().astype(np.int64)
        assert pm.shape == (self.mloc,)
        src = self.r["src"][s - 1]
        for i in range(self.mloc):
            g = self.i0 + i
            if int(src[g]) != g:  # took the partner's block (after Alg. 7's rule)
                assert int(src[g]) == g ^ (1 << (s - 1)) and int(src[g]) // self.mloc == peer
                self.A[i] = pm[i]

    def finish(self):
        want = self.r["Aisl"][self.i0: self.i0 + self.mloc]
        assert np.array_equal(self.A, want), "island map differs from the oracle's"
        self.xhat = self.r["xhat"].astype(np.float32)
        self.n += 1


def _worker(rank, world, port, q, exchange="pairwise", peer_dir=None):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = inputs.CONFIGS["C1"]
        params = inputs.model_params(cfg)
        N, M = 256, 16
        if exchange == "island":
            be = OracleIslandShard(params, N, M, 5, rank, world)
        else:
            be = OracleShard(params, N, M, 5, rank, world, peer_dir=peer_dir)
            be.relabel = exchange == "relabel"
        tr = pfd.TorchTransport()
        if exchange == "peer_fail":  # one rank cannot export: every rank agrees on "no peer"
            if rank == world - 1:
                def bad_export():
                    raise RuntimeError("no IPC on this rank")
                be.peer_export = bad_export
            assert pfd.peer_connect(be, tr) is False
            exchange = "pull"
        if exchange == "peer":
            dist.barrier()  # every rank's buffer file exists
            assert pfd.peer_connect(be, tr) is True
        _, ys = inputs.simulate(cfg, T=3)
        for y in ys:
            pfd.sharded_step(be, tr, y, exchange=exchange)
            be.finish()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,exchange", [(2, "pairwise"), (4, "pairwise"), (2, "pull"), (4, "pull"),
                                            (2, "peer"), (4, "peer"), (4, "peer_fail"), (2, "relabel"),
                                            (4, "relabel"), (2, "island"), (4, "island")])
def test_gloo_sharded_sequence(world, exchange, tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    peer_dir = str(tmp_path) if exchange == "peer" else None
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, exchange, peer_dir)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
