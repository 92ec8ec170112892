"""Partitioned engine (gn_part_*) timing with one part (development aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.partition import EngineBackend, build_partitions  # noqa: E402

for name in sys.argv[1].split(","):
    inst = G.c5_rmat_gpu(int(name[3:])) if name.startswith("C5S") else G.CONFIGS[name]()
    for dt in sys.argv[2].split(","):
        spec = build_partitions(inst.graph, 1)[0]
        be = EngineBackend(spec, dtype=dt)
        gam = P.GammaSchedule.pursuit().table()
        x0 = spec.local_x0(inst.x0)
        best = 1e9
        for rep in range(3):
            be.begin(x0, gam)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for k in range(len(gam)):
                be.step(k)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(name, dt, "ms per 1000 iterations", round(best, 3), "Geu/s", round(inst.m * 1000 / best / 1e6, 2), flush=True)
        be.close()
