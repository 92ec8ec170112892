"""Quick engine timing probe (development aid, not the bench contract)."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402


def probe(inst, iters=1000, grids=(0,), exact=False, reps=3, dtype=None):
    g = inst.graph
    dt = dtype or inst.dtype
    h = g.device_graph(dt)
    s = P.GammaSchedule.pursuit(iterations=iters)
    out = []
    for grid in grids:
        h.set_grid(grid)
        P.run_engine(g, inst.x0, s, dtype=dt, exact=exact)  # warm
        best = None
        for _ in range(reps):
            r = P.run_engine(g, inst.x0, s, dtype=dt, exact=exact)
            if best is None or r.stats["loop_ms"] < best["loop_ms"]:
                best = r.stats
        eus = g.num_edges * iters / (best["loop_ms"] * 1e-3)
        rec = {"inst": inst.name, "dtype": dt, "exact": exact, "grid": best["grid_blocks"],
               "loop_ms": round(best["loop_ms"], 3), "us_per_iter": round(best["loop_ms"] * 1e3 / iters, 3),
               "Geu_s": round(eus / 1e9, 2), "fallbacks": r.trace.total_fallbacks}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    h.set_grid(0)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="C1,C2,C3")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--grid", type=int, default=-1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dtypes", default="")
    args = ap.parse_args()
    which = args.which.split(",")
    if args.grid >= 0:
        for name in which:
            if name == "EDGELESS":
                inst = G.Instance("edgeless", P.from_csr(100000, np.zeros(100001, np.int64), np.zeros(0, np.int32),
                                                           np.ones(100000)), np.full(100000, 0.5), "fp64")
            elif name == "C4":
                inst = G.c4_batch(1024).instance
            elif name.startswith("C5S"):
                t = time.time()
                inst = G.c5_rmat_gpu(int(name[3:]))
                print("gen", name, time.time() - t, inst.graph, flush=True)
                t = time.time()
                inst.graph.device_graph(inst.dtype)
                print("graph create", time.time() - t, flush=True)
            else:
                inst = G.CONFIGS[name]()
            for dt in (args.dtypes.split(",") if args.dtypes else [None]):
                probe(inst, iters=args.iters, grids=(args.grid,), reps=args.reps, dtype=dt)
        raise SystemExit(0)
    if "C1" in which:
        probe(G.c1_er(), grids=(1, 2, 4, 0))
        probe(G.c1_er(), exact=True, grids=(0,))
    if "C2" in which:
        t = time.time(); inst = G.c2_assignment(); print("gen C2", time.time() - t, flush=True)
        probe(inst, grids=(148, 296, 444, 592, 0))
        probe(inst, exact=True, grids=(0,), reps=1)
        probe(inst, dtype="fp64", grids=(0,), reps=1)
    if "C3" in which:
        t = time.time(); inst = G.c3_ba(); print("gen C3", time.time() - t, flush=True)
        probe(inst, grids=(64, 148, 296, 592, 0))
        probe(inst, exact=True, grids=(0,), reps=1)
    if "C4" in which:
        t = time.time(); b = G.c4_batch(1024); print("gen C4", time.time() - t, flush=True)
        probe(b.instance, grids=(296, 592, 0))
