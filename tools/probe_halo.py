#!/usr/bin/env python3
"""The direct halo on one GPU: P parts of an R-MAT graph, every iteration of
every part from one captured schedule (gn_part_run_group), with the
boundary values pushed into the peers' ghost slots (LocalPeerExchange).

Prints ms per iteration (all parts), the pushed values per iteration, and
times the push blocks alone (gn_part_probe mode 7) inside an NVTX range
"push_probe" so that ncu can count their store sectors:

    ncu --nvtx --nvtx-include "push_probe/" --metrics \\
        l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum \\
        python tools/probe_halo.py --scale 22 --parts 3
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--parts", type=int, default=3)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--dtype", default="fp32")
    args = ap.parse_args()
    import torch

    import paper_2605_05330_b200 as P
    from paper_2605_05330_b200 import _engine as E
    from paper_2605_05330_b200 import generators as G
    from paper_2605_05330_b200.partition import (EngineBackend, LocalPeerExchange, build_partitions, run_group)

    E.load_library()
    inst = G.c5_rmat_gpu(args.scale) if args.scale >= 18 else G.c5_rmat(args.scale)
    g = inst.graph
    specs = build_partitions(g, args.parts)
    bes = [EngineBackend(s, dtype=args.dtype) for s in specs]
    ex = LocalPeerExchange(bes)
    tab = P.GammaSchedule.pursuit(iterations=args.iters).table()
    out = {"scale": args.scale, "parts": args.parts, "dtype": args.dtype, "n": g.n, "m": inst.m,
           "pushed_values_per_iteration": int(sum(len(v) for s in specs for v in s.send_idx.values())),
           "ghosts": [int(s.n_ghost) for s in specs], "owned": [int(s.n_own) for s in specs]}
    times = []
    for rep in range(3):
        ex.fence()
        for b, s in zip(bes, specs):
            b.begin(s.local_x0(inst.x0), tab)
        ex.setup()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_group(bes, 0, len(tab))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / len(tab))
    out["ms_per_iteration_all_parts"] = round(min(times), 4)
    res = [b.end(len(tab)) for b in bes]
    x = np.concatenate([r[0] for r in res])
    out["objective_last"] = float(np.sum([r[3][-1] for r in res]))
    torch.cuda.nvtx.range_push("push_probe")
    push_ms = []
    for b in bes:
        ms = ctypes.c_double()
        E.check(E.lib().gn_part_probe(b.h, 7, 3, ctypes.byref(ms)))
        push_ms.append(round(ms.value, 4))
    torch.cuda.nvtx.range_pop()
    out["push_only_ms_per_part"] = push_ms
    out["x_checksum"] = float(x.sum())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
