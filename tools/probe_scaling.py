#!/usr/bin/env python3
"""Strong-scaling projection of the partitioned C5 run from one GPU.

Only one B200 is available to this build, so the N-GPU strong-scaling curve
of `bench.py --gpus N` (C5, the vertex-range partition) cannot be measured
here.  This probe measures what each rank's GPU would compute: for every N
and every part p of the N-way partition it builds the part exactly as rank p
would (build_partition: its rows, its ghosts, its boundary-first numbering
and the long-row threshold of its size) and times its iterations from the
device-side schedule on cuda:0 without a halo (the ghosts keep their x0
values; the arithmetic per iteration is the same).  The projection of the
N-GPU step time is the slowest part's time; the halo's NVLink bytes per
iteration (the boundary values pushed to peers, before the delta halo drops
unchanged ones) are reported beside it.

    python tools/probe_scaling.py [--scale 24] [--iters 50] [--dtype fp64] [--gpus 1,2,4,8]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--dtype", default="fp64")
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--parts", default=None, help="only these part indices (e.g. for an ncu launch list)")
    args = ap.parse_args()
    import torch

    import paper_2605_05330_b200 as P
    from paper_2605_05330_b200 import _engine as E
    from paper_2605_05330_b200 import generators as G
    from paper_2605_05330_b200.partition import EngineBackend, build_partition

    E.load_library()
    inst = G.c5_rmat_gpu(args.scale) if args.scale >= 18 else G.c5_rmat(args.scale)
    g = inst.graph
    tab = P.GammaSchedule.pursuit(iterations=args.iters).table()
    elem = 8 if args.dtype == "fp64" else 4
    out = {"scale": args.scale, "n": g.n, "m": inst.m, "dtype": args.dtype, "iters": args.iters, "curve": []}
    t1 = None
    for n in [int(v) for v in args.gpus.split(",")]:
        parts = []
        for p in range(n):
            if args.parts is not None and p not in [int(v) for v in args.parts.split(",")]:
                continue
            t0 = time.perf_counter()
            spec = build_partition(g, n, p)
            be = EngineBackend(spec, dtype=args.dtype)
            setup = time.perf_counter() - t0
            x0 = spec.local_x0(inst.x0)
            best = None
            for _ in range(3):
                be.begin(x0, tab)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                be.run(0, len(tab))
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / len(tab)
                best = ms if best is None else min(best, ms)
            pushed = int(sum(len(v) for v in spec.send_idx.values()))
            parts.append({"p": p, "n_own": int(spec.n_own), "n_ghost": int(spec.n_ghost),
                          "nnz": int(len(spec.indices)), "ms_per_iter": round(best, 4),
                          "push_values": pushed, "push_mb": round(pushed * elem / 1e6, 2),
                          "setup_s": round(setup, 1)})
            be.close()
            del spec
        worst = max(q["ms_per_iter"] for q in parts)
        if n == 1:
            t1 = worst
        row = {"gpus": n, "projected_ms_per_iter": worst,
               "projected_gn_edge_updates_per_s": inst.m / (worst * 1e-3),
               "projected_efficiency": (t1 / (n * worst)) if t1 else None,
               "max_push_mb_per_iter": max(q["push_mb"] for q in parts), "parts": parts}
        out["curve"].append(row)
        print(json.dumps({k: v for k, v in row.items() if k != "parts"}), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
