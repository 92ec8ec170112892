"""Rounding timing probe (development aid): round_to_mis of a converged state."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402

for name in sys.argv[1].split(","):
    inst = G.c5_rmat_gpu(int(name[3:])) if name.startswith("C5S") else G.CONFIGS[name]()
    g = inst.graph
    r = P.run_engine(g, inst.x0, P.GammaSchedule.pursuit(iterations=300), dtype=inst.dtype)
    sol = P.round_to_mis(g, r.x)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        sol = P.round_to_mis(g, r.x)
        ts.append(time.perf_counter() - t)
    print(name, "n", g.n, "|MIS|", len(sol.members), "weight", repr(sol.weight), "round ms", round(min(ts) * 1e3, 3),
          flush=True)
