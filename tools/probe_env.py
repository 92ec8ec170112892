"""Timing of one instance under several values of a run-time env knob (development aid).

    python tools/probe_env.py C5S24 GN_L1HOT 0,16384,32768 [iters] [reps]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402

name, var, vals = sys.argv[1], sys.argv[2], sys.argv[3].split(",")
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
inst = G.c5_rmat_gpu(int(name[3:])) if name.startswith("C5S") else G.CONFIGS[name]()
s = P.GammaSchedule.pursuit(iterations=iters)
P.run_engine(inst.graph, inst.x0, s, dtype=inst.dtype)
for v in vals:
    os.environ[var] = v
    best = min(P.run_engine(inst.graph, inst.x0, s, dtype=inst.dtype).stats["loop_ms"] for _ in range(reps))
    print(f"{name} {var}={v} us/iter {1e3 * best / iters:.3f}", flush=True)
