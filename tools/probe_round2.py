"""Rounding time split (development aid): device call vs the MisSolution build."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.dynamics import round_result  # noqa: E402

for name in sys.argv[1].split(","):
    inst = G.CONFIGS[name]()
    g = inst.graph
    r = P.run_engine(g, inst.x0, P.GammaSchedule.pursuit(), dtype=inst.dtype)
    P.round_to_mis(g, r.x)
    a, b = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        round_result(g, r.x)
        t1 = time.perf_counter()
        P.round_to_mis(g, r.x)
        t2 = time.perf_counter()
        a.append(t1 - t0)
        b.append(t2 - t1)
    print(name, "device call %.3f ms, round_to_mis %.3f ms" % (min(a) * 1e3, min(b) * 1e3), flush=True)
