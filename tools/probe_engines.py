#!/usr/bin/env python3
"""The same instance through the persistent loop kernel (run_engine, one
cooperative launch for all iterations) and through the partitioned engine
with one part (one step launch per iteration from a CUDA graph): ms per
iteration of each, fast mode, L2 flushed between runs.

    python tools/probe_engines.py [--config C3] [--dtype fp64] [--iters 1000]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--dtype", default="fp64")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2605_05330_b200 as P
    from paper_2605_05330_b200 import _engine as E
    from paper_2605_05330_b200 import generators as G
    from paper_2605_05330_b200.partition import EngineBackend, build_partition

    E.load_library()
    inst = {"C1": G.c1_er, "C2": G.c2_assignment, "C3": G.c3_ba}[args.config]()
    g = inst.graph
    s = P.GammaSchedule.pursuit(iterations=args.iters)
    tab = s.table()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"config": args.config, "dtype": args.dtype, "n": g.n, "m": inst.m, "iters": args.iters}

    def timed(fn, pre=None):
        best = None
        for _ in range(args.reps):
            flush.fill_(1)
            if pre is not None:
                pre()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.iters
            best = ms if best is None else min(best, ms)
        return round(best, 5)

    x0d = torch.from_numpy(inst.x0).cuda()
    P.run_engine(g, x0d, s, dtype=args.dtype, device_state=True)
    out["loop_ms_per_iter"] = timed(lambda: P.run_engine(g, x0d, s, dtype=args.dtype, device_state=True))
    spec = build_partition(g, 1, 0)
    be = EngineBackend(spec, dtype=args.dtype)
    x0l = spec.local_x0(inst.x0)

    def part():
        be.begin(x0l, tab)
        be.run(0, len(tab))

    part()
    out["part_ms_per_iter"] = timed(part)
    out["part_run_only_ms_per_iter"] = timed(lambda: be.run(0, len(tab)), pre=lambda: be.begin(x0l, tab))
    import time

    t0 = time.perf_counter()
    be.begin(x0l, tab)
    torch.cuda.synchronize()
    out["part_begin_ms"] = round(1e3 * (time.perf_counter() - t0), 3)
    be.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
