"""GPU: the direct halo's CUDA IPC plumbing between processes, on one GPU.

DistPeerExchange (partition.py) maps the peers' ghost buffers and flag
arrays with CUDA IPC handles exchanged over torch.distributed, and the
interior step's push blocks store the boundary values straight into them.
Kernels of two ranks that spin on each other's flags must not share one GPU
(B200_PROFILING.md: context-switch timeouts), so this test runs two
processes on cuda:0 with every device-side wait replaced by a host
handshake: each iteration a rank runs its boundary and interior steps
(pushes included), synchronises its stream and meets the other rank at a
barrier before the next iteration.  What the test covers on real device
memory: handle export and import (gn_ipc_get_handle / gn_ipc_open_handle),
the per-peer slot arithmetic of the push list, the stores landing in the
other process's buffers, and stable mappings over repeated runs.  The
device-side wait/flag protocol itself is covered by the multi-part runs in
one process (test_partition_gpu.py) and by the CPU-process protocol tests
(test_partition.py).  Result: bitwise the oracle (EXACT) and the same run
with all parts in one process (fast mode).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ITERS = 120


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank: int, world: int, port: int, exact: bool, q) -> None:
    try:
        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2605_05330_b200 as P
        from paper_2605_05330_b200 import generators as G
        from paper_2605_05330_b200.partition import DistPeerExchange, EngineBackend, build_partition, run_partition

        class HostSyncPeerExchange(DistPeerExchange):
            """The IPC-mapped direct halo with the per-iteration device wait
            and flag replaced by stream sync + barrier (one GPU, two ranks)."""

            device_schedule = False

            def before(self, k):
                pass

            def after_interior(self, k, pending):
                torch.cuda.synchronize()
                self.dist.barrier()

        inst = G.c5_rmat(13)
        s = P.GammaSchedule.pursuit(iterations=ITERS)
        spec = build_partition(inst.graph, world, rank)
        be = EngineBackend(spec, dtype="fp64", exact=exact)
        ex = HostSyncPeerExchange(be)
        outs = []
        for _ in range(2):  # the second run reuses the mappings (stable buffers)
            r = run_partition(be, ex, spec.local_x0(inst.x0), s, device_schedule=False)
            outs.append((r.x.copy(), r.step_inf.copy(), r.fallbacks.copy()))
        ex.fence()
        ex.close()
        be.close()
        q.put((rank, spec.lo, spec.hi, outs, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, 0, 0, None, traceback.format_exc()))


def _run_two(exact: bool):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, exact, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[4] is None, f"rank {r[0]} failed:\n{r[4]}"
    return sorted(res)


@pytest.mark.parametrize("exact", [True, False])
def test_ipc_direct_halo_two_processes(exact):
    import gn_oracle as O
    import paper_2605_05330_b200 as P
    from paper_2605_05330_b200 import generators as G
    from paper_2605_05330_b200.partition import EngineBackend, run_local_partitions

    res = _run_two(exact)
    inst = G.c5_rmat(13)
    s = P.GammaSchedule.pursuit(iterations=ITERS)
    for run in range(2):
        x = np.empty(inst.graph.n)
        for rank, lo, hi, outs, _ in res:
            x[lo:hi] = outs[run][0]
        if exact:
            ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma)
            np.testing.assert_array_equal(x, ref.x)
        else:
            local = run_local_partitions(inst.graph, inst.x0, s, 2, lambda sp: EngineBackend(sp, dtype="fp64"),
                                         halo="peer")
            np.testing.assert_array_equal(x, local["x"])
