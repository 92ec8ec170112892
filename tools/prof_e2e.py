"""cProfile of the C2 e2e step's host side (development aid)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402

inst = G.c2_assignment()
g = inst.graph
s = P.GammaSchedule.pursuit()
for _ in range(3):
    r = P.run_engine(g, inst.x0, s, dtype="fp64")
    P.round_to_mis(g, r.x)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    r = P.run_engine(g, inst.x0, s, dtype="fp64")
    P.round_to_mis(g, r.x)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
