"""Multi-start engine timing (development aid): B starts per call, edge-updates/s over all starts."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="C2,C3")
ap.add_argument("--iters", type=int, default=1000)
ap.add_argument("--starts", default="16")
ap.add_argument("--dtypes", default="fp64,fp32")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
for name in args.which.split(","):
    t = time.time()
    inst = G.c5_rmat_gpu(int(name[3:])) if name.startswith("C5S") else G.CONFIGS[name]()
    print("gen", name, round(time.time() - t, 2), inst.graph, flush=True)
    s = P.GammaSchedule.pursuit(iterations=args.iters)
    for dt in args.dtypes.split(","):
        for B in [int(b) for b in args.starts.split(",")]:
            X = np.stack([P.init_random(inst.n, [7, b]) for b in range(B)])
            P.run_multi(inst.graph, X, s, dtype=dt)
            best = min((P.run_multi(inst.graph, X, s, dtype=dt).stats["loop_ms"] for _ in range(args.reps)))
            eus = inst.graph.num_edges * args.iters * B / (best * 1e-3)
            print(json.dumps({"inst": inst.name, "dtype": dt, "starts": B, "loop_ms": round(best, 3),
                              "us_per_iter": round(best * 1e3 / args.iters, 3),
                              "us_per_start_iter": round(best * 1e3 / args.iters / B, 3),
                              "Geu_s": round(eus / 1e9, 2)}), flush=True)
