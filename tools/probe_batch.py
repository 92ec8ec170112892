"""Resident batch kernel timing (development aid)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.batch import GraphBatch  # noqa: E402

graphs = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dts = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fp32"]
b = G.c4_batch(graphs)
s = P.GammaSchedule.pursuit()
for dt in dts:
    bt = GraphBatch(b.instance.graph, b.offsets, dtype=dt)
    bt.run(b.instance.x0, s)
    r = bt.run(b.instance.x0, s)
    m = b.instance.m
    print(dt, "threads", r.stats["block_threads"], "graphs", graphs, "loop_ms", round(r.stats["loop_ms"], 3),
          "Geu/s", round(m * 1000 / (r.stats["loop_ms"] * 1e-3) / 1e9, 1), flush=True)
