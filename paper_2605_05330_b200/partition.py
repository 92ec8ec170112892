"""Vertex-range partitioning of one graph over several GPUs.

Each partition owns a contiguous range of vertices, chosen so every part
has about the same step cost (adjacency entries plus a per-row term; R-MAT
concentrates its hubs at low ids, so equal vertex counts would be badly
imbalanced).  A part's neighbours outside its range are its ghosts, grouped
by owning peer and, inside a peer's group, hubs first (global degree
descending, then global id) -- the gathers of hot ghosts then share lines as
the owned hubs' do.  Every iteration:

    step     each part updates its owned rows (csrc/gn_part.cu), reading the
             published values of owned vertices and ghosts
    halo     each part packs the published values its peers hold as ghosts
             and sends them; received buffers are unpacked into ghost slots.
             The boundary rows (those peers hold) are stepped first, so the
             exchange runs while the interior rows are stepped

Neighbour lists keep the global (reference) order, so a partitioned EXACT run
is bitwise the single-GPU EXACT run (and the reference).  Exchanges:
LocalExchange (all parts in one process, e.g. one GPU, for tests) and
DistExchange (one part per rank, torch.distributed send/recv: NCCL over
NVLink on GPUs, gloo on CPU tests) pack, send and unpack; LocalPeerExchange
and DistPeerExchange (CUDA IPC between the ranks of a node) fuse the halo
into the boundary kernel: each boundary value is stored straight into the
ghost slots of the peers that hold it, then a flag per peer (gn_part_peer_*).
The compute backend is pluggable; EngineBackend is the CUDA engine.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .dynamics import GammaSchedule, gamma_table


@dataclass
class PartSpec:
    """Local view of partition p."""

    p: int
    parts: int
    lo: int
    hi: int
    ghosts: np.ndarray        # global ids: grouped by owner, then global degree descending, then id
    ghost_ptr: np.ndarray     # [parts+1]: ghosts owned by peer q are ghosts[ghost_ptr[q]:ghost_ptr[q+1]]
    indptr: np.ndarray        # owned rows, local column ids
    indices: np.ndarray       # int32 in [0, n_own + n_ghost)
    w: np.ndarray             # n_own + n_ghost
    send_idx: dict = field(default_factory=dict)  # peer q -> local owned ids q holds as ghosts (q's order)

    @property
    def n_own(self) -> int:
        return self.hi - self.lo

    @property
    def n_ghost(self) -> int:
        return len(self.ghosts)

    def local_x0(self, x0_global: np.ndarray) -> np.ndarray:
        return np.concatenate([x0_global[self.lo:self.hi], x0_global[self.ghosts]]).astype(np.float64)


ROW_COST = 6  # adjacency entries one non-isolated row's update costs (state in, x' and y' out)


def vertex_cost(indptr: np.ndarray) -> np.ndarray:
    """Per-vertex step cost in adjacency-entry units: its entries, plus
    ROW_COST for a row with neighbours (the update's state traffic), plus 1.
    Fitted to one-GPU timings of the parts of C5 at scale 24 (2/4/8 parts,
    tools/probe_scaling.py): time ~ entries + ~4 per owned row, isolated rows
    being skipped after their third iteration."""
    deg = np.diff(np.asarray(indptr, dtype=np.int64))
    return deg + 1 + ROW_COST * (deg > 0)


def partition_ranges(indptr: np.ndarray, parts: int) -> np.ndarray:
    """Contiguous vertex ranges with about equal step cost (vertex_cost:
    adjacency entries plus a per-row term): [parts+1] boundaries."""
    n = len(indptr) - 1
    if parts < 1:
        raise ValueError("parts must be positive")
    cost = vertex_cost(indptr)
    cum = np.concatenate([[0], np.cumsum(cost)])
    targets = cum[-1] * np.arange(1, parts) / parts
    cuts = np.searchsorted(cum, targets, side="left")
    bounds = np.concatenate([[0], np.clip(cuts, 0, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def build_partition(g, parts: int, p: int, bounds: Optional[np.ndarray] = None) -> PartSpec:
    """Local view of partition p of g, from p's own rows only (host-side
    setup, once per rank): O(nnz of the part), whatever the part count.

    The graph is symmetric (graph.py:112-119), so the owned vertices peer q
    holds as ghosts are exactly the owned rows with a neighbour in q's range.
    q orders the ghosts p owns by (global degree descending, global id); p
    knows its own rows' degrees, so it orders its send list to q the same
    way, and no rank needs another's rows."""
    indptr = np.asarray(g.indptr)
    bounds = partition_ranges(indptr, parts) if bounds is None else np.asarray(bounds, dtype=np.int64)
    lo, hi = int(bounds[p]), int(bounds[p + 1])
    e0, e1 = int(indptr[lo]), int(indptr[hi])
    cols = np.asarray(g.indices[e0:e1]).astype(np.int64, copy=False)
    outside = (cols < lo) | (cols >= hi)
    uniq = np.unique(cols[outside])                      # ascending global id
    owner_u = np.searchsorted(bounds, uniq, side="right") - 1
    gdeg = (np.asarray(indptr[uniq + 1], dtype=np.int64) - np.asarray(indptr[uniq], dtype=np.int64))
    order = np.lexsort((uniq, -gdeg, owner_u))           # by owner, hubs first, then id
    ghosts = uniq[order]
    owner = owner_u[order]
    slot = np.empty(len(uniq), dtype=np.int64)
    slot[order] = np.arange(len(uniq), dtype=np.int64)
    ghost_ptr = np.searchsorted(owner, np.arange(parts + 1), side="left").astype(np.int64)
    local = cols - lo
    local[outside] = (hi - lo) + slot[np.searchsorted(uniq, cols[outside])]
    w = np.asarray(g.w, dtype=np.float64)
    row_ptr = (np.asarray(indptr[lo:hi + 1], dtype=np.int64) - e0)
    spec = PartSpec(p, parts, lo, hi, ghosts, ghost_ptr, row_ptr, local.astype(np.int32),
                    np.concatenate([w[lo:hi], w[ghosts]]))
    if len(ghosts):
        rows = np.repeat(np.arange(hi - lo, dtype=np.int64), np.diff(row_ptr))[outside]
        peer = np.searchsorted(bounds, cols[outside], side="right") - 1
        key = np.unique(peer * (hi - lo + 1) + rows)          # (peer, row), ascending row per peer
        kp, kr = key // (hi - lo + 1), key % (hi - lo + 1)
        rdeg = np.diff(row_ptr)
        for q in np.unique(kp).tolist():
            r_q = kr[kp == q]
            spec.send_idx[int(q)] = r_q[np.lexsort((r_q, -rdeg[r_q]))].astype(np.int32)  # q's ghost order
    return spec


def build_partitions(g, parts: int, bounds: Optional[np.ndarray] = None) -> list[PartSpec]:
    """Local views of every partition of g (all parts in one process: tests,
    one-GPU runs)."""
    bounds = partition_ranges(np.asarray(g.indptr), parts) if bounds is None else np.asarray(bounds, dtype=np.int64)
    return [build_partition(g, parts, p, bounds) for p in range(parts)]


# ---------------------------------------------------------------- backends

class EngineBackend:
    """One partition on the CUDA engine (gn_part_*)."""

    def __init__(self, spec: PartSpec, dtype="fp64", device: int = 0, exact: Optional[bool] = None):
        import torch

        from .dynamics import _opt

        from . import _engine as E
        from .graph import dtype_code

        self.E, self.torch, self.spec = E, torch, spec
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        E.check(E.lib().gn_part_create(spec.n_own, spec.n_ghost, E.ptr(np.ascontiguousarray(spec.indptr)),
                                       E.ptr(np.ascontiguousarray(spec.indices)), E.ptr(np.ascontiguousarray(spec.w)),
                                       dtype_code(dtype), device, ctypes.byref(h)))
        self.h = h
        # exact: every row summed sequentially (bitwise the single-GPU EXACT run);
        # otherwise rows longer than 512 are split over a warp
        self.flags = E.GN_EXACT if _opt("exact", exact) else 0
        self.elem = E.lib().gn_part_elem_bytes(h)
        self.tdtype = torch.float64 if self.elem == 8 else torch.float32
        self.send_idx = {q: torch.from_numpy(v).to(self.device) for q, v in spec.send_idx.items()}
        # rows peers hold as ghosts go first, so their exchange overlaps the interior rows
        bnd = (np.unique(np.concatenate(list(spec.send_idx.values()))).astype(np.int32) if spec.send_idx
               else np.zeros(0, np.int32))
        E.check(E.lib().gn_part_set_boundary(h, E.ptr(bnd), len(bnd)))

    def _stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def begin(self, x0_local: np.ndarray, gammas: np.ndarray) -> None:
        E = self.E
        self.gam = np.ascontiguousarray(gammas, dtype=np.float64)
        E.check(E.lib().gn_part_begin(self.h, E.ptr(np.ascontiguousarray(x0_local, dtype=np.float64)),
                                      E.ptr(self.gam), len(self.gam), self.flags))

    def step(self, k: int) -> None:
        self.E.check(self.E.lib().gn_part_step(self.h, k, self._stream()))

    def run(self, k0: int, k1: int) -> None:
        """Iterations [k0, k1) from the device-side schedule (gn_part_run: one
        CUDA-graph launch; with the direct halo the waits, pushes and flags
        are inside it)."""
        self.E.check(self.E.lib().gn_part_run(self.h, k0, k1, self._stream()))

    def sync(self) -> None:
        self.torch.cuda.synchronize(self.device)

    def step_boundary(self, k: int) -> None:
        self.E.check(self.E.lib().gn_part_step_range(self.h, k, 0, self._stream()))

    def step_interior(self, k: int) -> None:
        self.E.check(self.E.lib().gn_part_step_range(self.h, k, 1, self._stream()))

    def empty(self, count: int):
        return self.torch.empty(count, dtype=self.tdtype, device=self.device)

    def pack(self, k: int, q: int):
        idx = self.send_idx[q]
        buf = self.empty(len(idx))
        self.E.check(self.E.lib().gn_part_pack(self.h, k, ctypes.c_void_p(idx.data_ptr()), len(idx),
                                               ctypes.c_void_p(buf.data_ptr()), self._stream()))
        return buf

    def unpack(self, k: int, q: int, buf) -> None:
        first = int(self.spec.ghost_ptr[q])
        self.E.check(self.E.lib().gn_part_unpack(self.h, k, ctypes.c_void_p(buf.data_ptr()), first, buf.numel(),
                                                 self._stream()))

    # ---- direct halo over peer memory (gn_part_peer_*)
    def peer_init(self, parts: int, me: int, expect) -> None:
        ex = np.ascontiguousarray(expect, dtype=np.int32)
        self.E.check(self.E.lib().gn_part_peer_init(self.h, parts, me, self.E.ptr(ex), len(ex)))

    def peer_buffers(self) -> tuple[int, int, int]:
        a, b, f = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        self.E.check(self.E.lib().gn_part_peer_buffers(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(f)))
        return a.value, b.value, f.value

    def peer_add(self, rank: int, bufs, owned, slot0: int) -> None:
        own = np.ascontiguousarray(owned, dtype=np.int32)
        self.E.check(self.E.lib().gn_part_peer_add(self.h, rank, bufs[0], bufs[1], bufs[2], self.E.ptr(own),
                                                   len(own), int(slot0)))

    def peer_commit(self) -> None:
        self.E.check(self.E.lib().gn_part_peer_commit(self.h))

    def peer_wait(self, k: int) -> None:
        self.E.check(self.E.lib().gn_part_peer_wait(self.h, k, self._stream()))

    def peer_signal(self, k: int) -> None:
        self.E.check(self.E.lib().gn_part_peer_signal(self.h, k, self._stream()))

    def end(self, done: int):
        E = self.E
        x = np.empty(self.spec.n_own)
        si = np.zeros(max(done, 1))
        fb = np.zeros(max(done, 1), dtype=np.int64)
        ms = np.zeros(max(done, 1))
        bad = ctypes.c_int(-1)
        E.check(E.lib().gn_part_end(self.h, done, E.ptr(x), E.ptr(si), E.ptr(fb), E.ptr(ms), ctypes.byref(bad)))
        return x, si[:done], fb[:done], ms[:done], bad.value

    def gathers(self, done: int) -> np.ndarray:
        """Value gathers issued per iteration (GN_PART_COUNT=1 set before
        begin(); zeros otherwise): what the zero-row certificates left of the
        adjacency walk (measurement aid, gn_part_gathers)."""
        out = np.zeros(max(done, 1), dtype=np.int64)
        self.E.check(self.E.lib().gn_part_gathers(self.h, done, self.E.ptr(out)))
        return out[:done]

    def close(self) -> None:
        if getattr(self, "h", None) is not None:
            self.E.lib().gn_part_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- exchanges

class NoExchange:
    """A single part (one GPU): no halo; the iterations run from the
    device-side schedule."""

    device_schedule = True

    def __init__(self, backend=None):
        self.b = backend

    def fence(self) -> None:
        if self.b is not None and hasattr(self.b, "sync"):
            self.b.sync()

    def setup(self) -> None:
        pass

    def before(self, k: int) -> None:
        pass

    def after_boundary(self, k: int):
        return None

    def after_interior(self, k: int, pending) -> None:
        pass


def _sync_all(backends) -> None:
    for b in backends:
        if hasattr(b, "sync"):
            b.sync()


class _PackedHalo:
    """Halo protocol of the pack / send / unpack exchanges: the boundary
    values are packed and posted after the boundary rows, received and
    unpacked after the interior rows (host-driven: one Python step per
    iteration)."""

    device_schedule = False

    def setup(self) -> None:
        pass

    def before(self, k: int) -> None:
        pass

    def after_boundary(self, k: int):
        return self.start(k)

    def after_interior(self, k: int, pending) -> None:
        self.finish(k, pending)


class LocalExchange(_PackedHalo):
    """All partitions in this process: the halo is a buffer hand-over."""

    def __init__(self, backends: Sequence):
        self.backends = list(backends)

    def fence(self) -> None:
        _sync_all(self.backends)

    def start(self, k: int):
        return {(p, q): b.pack(k, q) for p, b in enumerate(self.backends) for q in b.spec.send_idx}

    def finish(self, k: int, outgoing) -> None:
        for (p, q), buf in outgoing.items():
            self.backends[q].unpack(k, p, buf)

    def halo(self, k: int) -> None:
        self.finish(k, self.start(k))


class DistExchange(_PackedHalo):
    """One partition per rank; grouped point-to-point sends/receives
    (torch.distributed: NCCL on GPUs, gloo on CPU)."""

    def __init__(self, backend, group=None):
        import torch.distributed as dist

        self.dist, self.b, self.group = dist, backend, group
        spec = backend.spec
        self.recv_from = [q for q in range(spec.parts) if q != spec.p and spec.ghost_ptr[q + 1] > spec.ghost_ptr[q]]

    def fence(self) -> None:
        _sync_all([self.b])
        self.dist.barrier(group=self.group)

    def start(self, k: int):
        """Pack the boundary values of step k and post the sends/receives (they
        run on the communicator's stream, after the packs)."""
        dist, b = self.dist, self.b
        spec = b.spec
        ops, recvs = [], []
        for q in self.recv_from:
            buf = b.empty(int(spec.ghost_ptr[q + 1] - spec.ghost_ptr[q]))
            recvs.append((q, buf))
            ops.append(dist.P2POp(dist.irecv, buf, q, self.group))
        for q in spec.send_idx:
            ops.append(dist.P2POp(dist.isend, b.pack(k, q), q, self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        return works, recvs

    def finish(self, k: int, pending) -> None:
        works, recvs = pending
        for r in works:
            r.wait()
        for q, buf in recvs:
            self.b.unpack(k, q, buf)

    def halo(self, k: int) -> None:
        self.finish(k, self.start(k))


def _expected_peers(spec: PartSpec) -> list[int]:
    """Peers whose vertices this part holds as ghosts: they push to it (and,
    the graph being symmetric, it pushes to them)."""
    return [q for q in range(spec.parts) if q != spec.p and spec.ghost_ptr[q + 1] > spec.ghost_ptr[q]]


class _PeerHalo:
    """Halo protocol of the direct (peer-memory) exchanges: no host work per
    iteration -- the interior launch pushes the boundary values, then
    per-peer flags; run_partition replays every iteration from one CUDA graph
    (gn_part_run).  The peers' buffers are mapped once and stay valid across
    runs while their addresses hold (gn_part_begin keeps them); flags carry
    the run epoch."""

    device_schedule = True

    def before(self, k: int) -> None:
        for b in self._mine():
            b.peer_wait(k)

    def after_boundary(self, k: int):
        return None

    def after_interior(self, k: int, pending) -> None:
        for b in self._mine():
            b.peer_signal(k)


class LocalPeerExchange(_PeerHalo):
    """All partitions in this process (e.g. on one GPU): the boundary step of
    each part stores its values straight into the other parts' ghost slots."""

    def __init__(self, backends: Sequence):
        self.backends = list(backends)
        self._mapped = None

    def _mine(self):
        return self.backends

    def fence(self) -> None:
        _sync_all(self.backends)

    def setup(self) -> None:
        bufs = [b.peer_buffers()[:2] if self._mapped is not None else None for b in self.backends]
        if self._mapped is not None and bufs == self._mapped:
            return  # same buffers as the last handshake: the pushes are still valid
        for b in self.backends:
            b.peer_init(b.spec.parts, b.spec.p, _expected_peers(b.spec))
        bufs = [b.peer_buffers() for b in self.backends]
        for p, b in enumerate(self.backends):
            for q, owned in b.spec.send_idx.items():
                peer = self.backends[q].spec
                b.peer_add(q, bufs[q], owned, peer.n_own + int(peer.ghost_ptr[p]))
            b.peer_commit()
        self._mapped = [tuple(x[:2]) for x in bufs]


class DistPeerExchange(_PeerHalo):
    """One partition per rank: the peers' buffers are mapped with CUDA IPC
    (handles exchanged once per run over torch.distributed), and the boundary
    kernel's stores travel over NVLink as the rows finish."""

    def __init__(self, backend, group=None):
        import torch.distributed as dist

        self.dist, self.b, self.group = dist, backend, group
        self._opened: list[int] = []
        self._mapped = None

    def _mine(self):
        return [self.b]

    def fence(self) -> None:
        """Every rank's previous run has finished on its device: no late push
        or flag can land in a buffer gn_part_begin is about to reset."""
        _sync_all([self.b])
        self.dist.barrier(group=self.group)

    def setup(self) -> None:
        E, b = self.b.E, self.b
        spec = b.spec
        if self._mapped is not None:
            same = [None] * spec.parts
            self.dist.all_gather_object(same, tuple(b.peer_buffers()[:2]) == self._mapped, group=self.group)
            if all(same):
                # buffers unchanged everywhere: the mappings and push lists
                # stand; every rank has finished gn_part_begin before any push
                self.dist.barrier(group=self.group)
                return
        for ptr in self._opened:
            E.lib().gn_ipc_close(ptr)
        self._opened = []
        b.peer_init(spec.parts, spec.p, _expected_peers(spec))
        handles = []
        for ptr in b.peer_buffers():
            h = ctypes.create_string_buffer(64)
            E.check(E.lib().gn_ipc_get_handle(ptr, h))
            handles.append(h.raw)
        allh = [None] * spec.parts
        self.dist.all_gather_object(allh, (spec.n_own, [int(x) for x in spec.ghost_ptr], handles), group=self.group)
        dev = b.device.index or 0
        for q, owned in spec.send_idx.items():
            n_own_q, ghost_ptr_q, hq = allh[q]
            ptrs = []
            for raw in hq:
                out = ctypes.c_void_p()
                E.check(E.lib().gn_ipc_open_handle(ctypes.create_string_buffer(raw, 64), dev, ctypes.byref(out)))
                ptrs.append(out.value)
                self._opened.append(out.value)
            b.peer_add(q, ptrs, owned, n_own_q + ghost_ptr_q[spec.p])
        b.peer_commit()
        self._mapped = tuple(b.peer_buffers()[:2])
        # every rank has reset its buffers (gn_part_begin) and mapped its peers
        self.dist.barrier(group=self.group)

    def close(self) -> None:
        """Unmap the peers' buffers (after the last run)."""
        for ptr in self._opened:
            self.b.E.lib().gn_ipc_close(ptr)
        self._opened = []


@dataclass
class PartResult:
    x: np.ndarray            # owned entries (clipped)
    step_inf: np.ndarray     # this part's per-iteration max|dx|
    fallbacks: np.ndarray
    mass: np.ndarray         # this part's w.x'
    bad: int


def partitioned_step(backend, exchange, k: int) -> None:
    """Step k of one partition with the halo overlapped: boundary rows, then
    their exchange in flight while the interior rows run, then the ghosts
    (pack/send/unpack exchanges), or the boundary rows' direct pushes and the
    peer flags (peer exchanges)."""
    exchange.before(k)
    backend.step_boundary(k)
    pending = exchange.after_boundary(k)
    backend.step_interior(k)
    exchange.after_interior(k, pending)


def run_partition(backend, exchange, x0_local: np.ndarray, schedule: GammaSchedule,
                  device_schedule: bool = True) -> PartResult:
    """The pursuit on one partition (all ranks call this together): fence
    the ranks, reset the run, then every iteration -- from the device-side
    schedule (one CUDA-graph launch) when the exchange allows it, else one
    host-driven step per iteration (dynamics.py:155-178)."""
    import time

    gam = gamma_table(schedule)
    t = [time.perf_counter()]
    exchange.fence()
    t.append(time.perf_counter())
    backend.begin(x0_local, gam)
    t.append(time.perf_counter())
    exchange.setup()
    t.append(time.perf_counter())
    if device_schedule and exchange.device_schedule and hasattr(backend, "run"):
        backend.run(0, len(gam))
    else:
        for k in range(len(gam)):
            partitioned_step(backend, exchange, k)
    t.append(time.perf_counter())
    x, si, fb, ms, bad = backend.end(len(gam))
    t.append(time.perf_counter())
    backend.last_times = dict(zip(("fence", "begin", "setup", "launch", "end (sync + out)"), np.diff(t)))
    return PartResult(x, si, fb, ms, bad)


def run_group(backends, k0: int, k1: int) -> None:
    """Iterations [k0, k1) of every part held by this process, interleaved in
    one captured schedule (gn_part_run_group: per k, per part: wait, boundary,
    interior + pushes, signal)."""
    b0 = backends[0]
    E = b0.E
    hs = (ctypes.c_void_p * len(backends))(*[b.h.value for b in backends])
    E.check(E.lib().gn_part_run_group(hs, len(backends), k0, k1, b0._stream()))


def run_local_partitions(g, x0: np.ndarray, schedule: GammaSchedule, parts: int, make_backend,
                         halo: str = "copy", device_schedule: bool = False, runs: int = 1) -> dict:
    """All parts of g in this process (e.g. on one GPU): returns the global x
    and the combined per-iteration trace (max / sum / sum over parts).
    halo: "copy" (pack / hand-over / unpack) or "peer" (direct pushes);
    device_schedule (peer halo): every iteration of every part from one
    captured CUDA graph; runs > 1 repeats the run on the same backends and
    exchange (the later runs reuse the first handshake; results of the last)."""
    specs = build_partitions(g, parts)
    backends = [make_backend(s) for s in specs]
    ex = LocalPeerExchange(backends) if halo == "peer" else LocalExchange(backends)
    gam = gamma_table(schedule)
    for _ in range(runs):
        outs = _local_run(backends, specs, ex, x0, gam, halo, device_schedule)
    x = np.concatenate([o[0] for o in outs])
    return {"x": x, "step_inf": np.max([o[1] for o in outs], axis=0), "fallbacks": np.sum([o[2] for o in outs], axis=0),
            "mass": np.sum([o[3] for o in outs], axis=0), "specs": specs, "backends": backends}


def _local_run(backends, specs, ex, x0, gam, halo, device_schedule):
    ex.fence()
    for b, s in zip(backends, specs):
        b.begin(s.local_x0(x0), gam)
    ex.setup()
    if halo == "peer" and device_schedule:
        run_group(backends, 0, len(gam))
        return [b.end(len(gam)) for b in backends]
    for k in range(len(gam)):
        if halo == "peer":
            for b in backends:  # each part: wait, boundary (pushes), interior, flags
                b.peer_wait(k)
                b.step_boundary(k)
                b.step_interior(k)
                b.peer_signal(k)
            continue
        for b in backends:
            b.step_boundary(k)
        pending = ex.start(k)
        for b in backends:
            b.step_interior(k)
        ex.finish(k, pending)
    return [b.end(len(gam)) for b in backends]
