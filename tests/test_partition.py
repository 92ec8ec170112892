"""Vertex-range partitioning (C5 path): host-side partition/halo logic and the
multi-rank protocol, on CPU.  The 2-rank test runs the real DistExchange over
torch.distributed (gloo, 127.0.0.1) with a numpy stand-in for the per-part
GPU compute (test infrastructure, scipy's sequential csr_matvec = the
reference order), and checks the assembled trajectory bitwise against the
unpartitioned oracle."""

import os
import socket

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200 import generators as G
from paper_2605_05330_b200.partition import (DistExchange, LocalExchange, build_partitions, partition_ranges, vertex_cost,
                                             run_partition)


class NumpyBackend:
    """CPU stand-in for EngineBackend (tests only): same step, fp64."""

    def __init__(self, spec):
        import scipy.sparse as sp
        import torch

        self.torch, self.spec = torch, spec
        self.A = sp.csr_matrix((np.ones(len(spec.indices)), spec.indices, spec.indptr),
                               shape=(spec.n_own, spec.n_own + spec.n_ghost))
        self.v = np.sqrt(spec.w)

    def begin(self, x0_local, gammas):
        self.gam = gammas
        self.x = x0_local[: self.spec.n_own].copy()
        self.y = [self.v * x0_local, self.v * x0_local]
        self.si, self.fb, self.ms = [], [], []

    def step(self, k):
        yc = self.y[k & 1]
        s = self.A @ yc
        yi = self.v[: self.spec.n_own] * self.x
        d = yi + self.gam[k] * s
        ok = d > 1e-9
        o = np.where(ok, yi / np.where(ok, d, 1.0), 0.5)
        self.si.append(float(np.max(np.abs(o - self.x))) if len(o) else 0.0)
        self.fb.append(int(len(o) - np.count_nonzero(ok)))
        self.x = o
        self.y[(k & 1) ^ 1][: self.spec.n_own] = self.v[: self.spec.n_own] * o

    def step_boundary(self, k):  # the whole step: the split only matters for overlap
        self.step(k)

    def step_interior(self, k):
        pass

    def empty(self, count):
        return self.torch.empty(count, dtype=self.torch.float64)

    def pack(self, k, q):
        return self.torch.from_numpy(self.y[(k & 1) ^ 1][self.spec.send_idx[q]].copy())

    def unpack(self, k, q, buf):
        first = self.spec.n_own + int(self.spec.ghost_ptr[q])
        self.y[(k & 1) ^ 1][first:first + buf.numel()] = buf.numpy()

    def end(self, done):
        return np.clip(self.x, 0, 1), np.array(self.si), np.array(self.fb), np.zeros(done), -1


def _graph():
    return G.c5_rmat(11)


def test_partition_ranges_balance_and_cover():
    g = _graph().graph
    for parts in (1, 2, 3, 8):
        b = partition_ranges(g.indptr, parts)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
        cost = vertex_cost(g.indptr)
        loads = [cost[b[p]:b[p + 1]].sum() for p in range(parts)]
        assert max(loads) <= cost.sum() / parts + cost.max()


def test_local_views_reproduce_global_rows_and_halo_lists():
    g = _graph().graph
    specs = build_partitions(g, 3)
    for s in specs:
        glob = np.concatenate([np.arange(s.lo, s.hi), s.ghosts])
        for r in range(s.n_own):
            row = glob[s.indices[s.indptr[r]:s.indptr[r + 1]]]
            np.testing.assert_array_equal(row, g.neighbors(s.lo + r))  # same order
        for q, t in enumerate(specs):
            if q == s.p:
                continue
            owned_by_q = s.ghosts[s.ghost_ptr[q]:s.ghost_ptr[q + 1]]
            sent = t.send_idx.get(s.p, np.zeros(0, np.int32)) + t.lo
            np.testing.assert_array_equal(owned_by_q, sent)


def _send_lists_from_all_parts(g, parts):
    """The send lists as the peers see them: p sends to q the ids of q's
    ghosts that p owns (every part's rows are needed for this)."""
    specs = build_partitions(g, parts)
    out = {}
    for p, sp in enumerate(specs):
        for q, sq in enumerate(specs):
            need = sq.ghosts[sq.ghost_ptr[p]:sq.ghost_ptr[p + 1]]
            if q != p and len(need):
                out[(p, q)] = (need - sp.lo).astype(np.int32)
    return out


@pytest.mark.parametrize("parts", [2, 3, 5, 8])
def test_own_rows_send_lists_match_peer_ghost_lists(parts):
    """build_partition derives a part's send lists from its own rows only
    (the graph is symmetric); they equal the ghost lists of the peers."""
    from paper_2605_05330_b200 import generators as G

    for inst in (_graph(), G.c5_rmat(12), G.c3_ba(n=3000, m=4)):
        ref = _send_lists_from_all_parts(inst.graph, parts)
        got = {(p, q): v for p, sp in enumerate(build_partitions(inst.graph, parts)) for q, v in sp.send_idx.items()}
        assert ref.keys() == got.keys()
        for key in ref:
            np.testing.assert_array_equal(ref[key], got[key])


def test_local_exchange_protocol_is_bitwise_unpartitioned():
    inst = _graph()
    s = P.GammaSchedule.pursuit(iterations=200)
    specs = build_partitions(inst.graph, 4)
    backends = [NumpyBackend(sp) for sp in specs]
    ex = LocalExchange(backends)
    gam = s.table()
    for b, sp in zip(backends, specs):
        b.begin(sp.local_x0(inst.x0), gam)
    for k in range(len(gam)):
        for b in backends:
            b.step(k)
        ex.halo(k)
    x = np.concatenate([b.end(len(gam))[0] for b in backends])
    ref = O.run(inst.graph, inst.x0, gam, s.final_gamma)
    np.testing.assert_array_equal(x, ref.x)
    np.testing.assert_array_equal(np.max([b.si for b in backends], axis=0), ref.step_inf)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = _graph()
        s = P.GammaSchedule.pursuit(iterations=150)
        spec = build_partitions(inst.graph, world)[rank]
        be = NumpyBackend(spec)
        res = run_partition(be, DistExchange(be), spec.local_x0(inst.x0), s)
        out = [None] * world
        dist.all_gather_object(out, (spec.lo, res.x, res.step_inf, res.fallbacks))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_halo_exchange_is_bitwise_unpartitioned():
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    x = np.concatenate([o[1] for o in out])
    inst = _graph()
    s = P.GammaSchedule.pursuit(iterations=150)
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma)
    np.testing.assert_array_equal(x, ref.x)
    np.testing.assert_array_equal(np.max([o[2] for o in out], axis=0), ref.step_inf)
    np.testing.assert_array_equal(np.sum([o[3] for o in out], axis=0), ref.fallbacks)


# ---- the direct (peer-memory) halo protocol, two processes on CPU --------
# DistPeerExchange runs unchanged; the "device buffers" are POSIX shared
# memory blocks and the "CUDA IPC handles" their names, so the handle
# exchange, the slot arithmetic and the wait / push / signal ordering are
# exercised with two ranks that really run concurrently.

class _FakeLib:
    def __init__(self, be):
        self.be = be

    def gn_ipc_get_handle(self, ptr, h):
        import ctypes

        name = self.be.names[ptr].encode().ljust(64, b"\0")
        ctypes.memmove(h, name, 64)
        return 0

    def gn_ipc_open_handle(self, h, dev, pout):
        from multiprocessing import shared_memory

        name = bytes(h.raw).rstrip(b"\0").decode()
        shm = shared_memory.SharedMemory(name=name)
        pid = 10_000 + len(self.be.opened)
        self.be.opened[pid] = shm
        pout._obj.value = pid
        return 0

    def gn_ipc_close(self, ptr):
        shm = self.be.opened.pop(ptr, None)
        if shm is not None:
            shm.close()
        return 0


class _FakeE:
    def __init__(self, be):
        self._lib = _FakeLib(be)

    def lib(self):
        return self._lib

    @staticmethod
    def check(rc):
        assert rc == 0


class NumpyPeerBackend(NumpyBackend):
    """NumpyBackend whose halo is the peer protocol over shared memory."""

    def __init__(self, spec):
        super().__init__(spec)
        from types import SimpleNamespace

        self.E = _FakeE(self)
        self.device = SimpleNamespace(index=0)
        self.names, self.opened, self.own = {}, {}, []
        self._yblk = None
        self.epoch = 0

    def _block(self, key, shape, dtype):
        from multiprocessing import shared_memory

        shm = shared_memory.SharedMemory(create=True, size=max(int(np.prod(shape)) * np.dtype(dtype).itemsize, 8))
        self.own.append(shm)
        self.names[key] = shm.name
        a = np.ndarray(shape, dtype=dtype, buffer=shm.buf)
        a[...] = 0
        return a

    def _view(self, pid, dtype):
        shm = self.opened[pid]
        return np.ndarray((shm.size // np.dtype(dtype).itemsize,), dtype=dtype, buffer=shm.buf)

    def begin(self, x0_local, gammas):
        # as gn_part_begin: the buffers stay put across runs (the peers keep
        # their mappings), a new epoch, the flags are not reset
        super().begin(x0_local, gammas)
        nall = self.spec.n_own + self.spec.n_ghost
        if self._yblk is None:
            self._yblk = [self._block(1, (nall,), np.float64), self._block(2, (nall,), np.float64)]
        self.y = self._yblk
        self.y[0][:] = self.v * x0_local
        self.y[1][:] = self.v * x0_local
        self.epoch += 1

    def sync(self):
        pass

    def peer_init(self, parts, me, expect):
        self.me, self.expect, self.pushes = me, list(expect), []
        self.flags = self._block(3, (parts,), np.int64)
        self.inits = getattr(self, "inits", 0) + 1

    def peer_buffers(self):
        return 1, 2, 3

    def peer_add(self, rank, bufs, owned, slot0):
        self.pushes.append((rank, bufs, np.asarray(owned), int(slot0)))

    def peer_commit(self):
        pass

    def peer_wait(self, k):
        import time

        t0 = time.time()
        target = (self.epoch << 32) + k
        while k > 0 and any(self.flags[q] < target for q in self.expect):
            assert time.time() - t0 < 60, "peer flag did not arrive"
            time.sleep(0.0005)

    def step_boundary(self, k):
        self.step(k)
        nxt = self.y[(k & 1) ^ 1]
        for rank, bufs, owned, slot0 in self.pushes:  # straight into the peer's ghost slots
            self._view(bufs[(k + 1) & 1], np.float64)[slot0:slot0 + len(owned)] = nxt[owned]

    def peer_signal(self, k):
        for rank, bufs, owned, slot0 in self.pushes:
            self._view(bufs[2], np.int64)[self.me] = (self.epoch << 32) + k + 1

    def close(self):
        for shm in list(self.opened.values()) + self.own:
            shm.close()
        for shm in self.own:
            shm.unlink()


def _peer_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2605_05330_b200.partition import DistPeerExchange

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be = None
    try:
        inst = _graph()
        s = P.GammaSchedule.pursuit(iterations=120)
        spec = build_partitions(inst.graph, world)[rank]
        be = NumpyPeerBackend(spec)
        ex = DistPeerExchange(be)
        # two runs back to back on the same exchange: the second reuses the
        # first handshake, and the fence + epochs keep them apart
        res0 = run_partition(be, ex, spec.local_x0(inst.x0), s)
        res = run_partition(be, ex, spec.local_x0(inst.x0), s)
        assert be.inits == 1 and be.epoch == 2
        assert np.array_equal(res0.x, res.x)
        out = [None] * world
        dist.all_gather_object(out, (spec.lo, res.x, res.step_inf, res.fallbacks))
        if rank == 0:
            q.put(out)
        dist.barrier()
    finally:
        if be is not None:
            be.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_halo_protocol_multiprocess_is_bitwise_unpartitioned(world):
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    x = np.concatenate([o[1] for o in out])
    inst = _graph()
    s = P.GammaSchedule.pursuit(iterations=120)
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma)
    np.testing.assert_array_equal(x, ref.x)
    np.testing.assert_array_equal(np.max([o[2] for o in out], axis=0), ref.step_inf)
