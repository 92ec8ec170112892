"""Rounding of the packed C4 shard (development aid): wall time of round_to_mis
and of the device call, for a launch list under ncu."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.dynamics import round_result  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
inst = G.c4_batch(graphs=1024).instance
g = inst.graph
r = P.run_engine(g, inst.x0, P.GammaSchedule.pursuit(), dtype="fp32")
P.round_to_mis(g, r.x)
a, b = [], []
for _ in range(reps):
    t0 = time.perf_counter()
    round_result(g, r.x)
    t1 = time.perf_counter()
    P.round_to_mis(g, r.x)
    t2 = time.perf_counter()
    a.append(t1 - t0)
    b.append(t2 - t1)
print("C4 device call %.3f ms, round_to_mis %.3f ms" % (min(a) * 1e3, min(b) * 1e3), flush=True)
