"""Break down the public-API (e2e) path of one C2 solve (development aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402

inst = G.c2_assignment()
g = inst.graph
s = P.GammaSchedule.pursuit()
for rep in range(4):
    t0 = time.perf_counter()
    r = P.run_engine(g, inst.x0, s, dtype="fp64")
    t1 = time.perf_counter()
    sol = P.round_to_mis(g, r.x)
    t2 = time.perf_counter()
    print(f"run_engine {1e3*(t1-t0):.2f} ms (loop {r.stats['loop_ms']:.2f}, call {r.stats['total_ms']:.2f}) "
          f"round_to_mis {1e3*(t2-t1):.2f} ms |MIS|={len(sol.members)}", flush=True)
