#!/usr/bin/env python3
"""What bounds the partitioned step on C5 (R-MAT scale 24, one part, fp32)?

Times (gn_part_probe, CUDA events, ms per launch) the step kernel and its two
halves (warp-split long rows, thread-per-row SELL slices), and the slices'
gather walk alone with real gathers, no gathers (the index stream), gathers
that all hit one 16 KB table (the walk's instruction/latency floor) and
random gathers (no locality).  GN_LIB selects an A/B build of the library.

    python tools/probe_c5.py [--scale 24] [--reps 10] [--dtype fp32]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

MODES = ["step", "step_long_rows_only", "step_slices_only", "walk_gathers", "walk_index_only", "walk_l1_hits",
         "walk_random"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dtype", default="fp32")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    import paper_2605_05330_b200 as P
    from paper_2605_05330_b200 import _engine as E
    from paper_2605_05330_b200 import generators as G
    from paper_2605_05330_b200.partition import EngineBackend, build_partition

    E.load_library()
    inst = G.c5_rmat_gpu(args.scale) if args.scale >= 18 else G.c5_rmat(args.scale)
    g = inst.graph
    spec = build_partition(g, 1, 0)
    be = EngineBackend(spec, dtype=args.dtype)
    tab = P.GammaSchedule.pursuit(iterations=args.iters).table()
    be.begin(spec.local_x0(inst.x0), tab)
    out = {"lib": os.environ.get("GN_LIB", "libgnb200.so"), "scale": args.scale, "dtype": args.dtype,
           "env": {k: v for k, v in os.environ.items() if k.startswith("GN_")},
           "n": g.n, "nnz": int(len(g.indices))}
    deg = np.diff(np.asarray(g.indptr))
    out["nnz_long_rows"] = int(deg[deg > 512].sum())
    out["long_rows"] = int((deg > 512).sum())
    for m, name in enumerate(MODES):
        ms = ctypes.c_double()
        E.check(E.lib().gn_part_probe(be.h, m, args.reps, ctypes.byref(ms)))
        out[name + "_ms"] = round(ms.value, 4)
    # the real schedule: every iteration from the CUDA graph
    import torch

    be.begin(spec.local_x0(inst.x0), tab)
    be.run(0, len(tab))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    be.begin(spec.local_x0(inst.x0), tab)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    be.run(0, len(tab))
    e1.record()
    torch.cuda.synchronize()
    out["run_ms_per_iter"] = round(e0.elapsed_time(e1) / len(tab), 4)
    res = be.end(len(tab))
    import hashlib

    out["x_sha1"] = hashlib.sha1(np.ascontiguousarray(res[0]).tobytes()).hexdigest()[:16]
    out["objective_last"] = float(res[3][-1])
    print(json.dumps(out), flush=True)
    be.close()


if __name__ == "__main__":
    main()
