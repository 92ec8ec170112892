"""How much of the slice path is still active late in a pursuit (development
aid).  One-part partitioned engine on an R-MAT graph: per 100 iterations, the
mean share of rows that walk (GN_PART_COUNT=2) and of slices with at least one
walking row (GN_PART_COUNT=3), next to the gathers (GN_PART_COUNT=1)."""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.partition import EngineBackend, build_partition  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--iters", type=int, default=1000)
    args = ap.parse_args()
    inst = G.c5_rmat_gpu(args.scale) if args.scale >= 20 else G.c5_rmat(args.scale)
    g = inst.graph
    spec = build_partition(g, 1, 0)
    be = EngineBackend(spec, dtype="fp64")
    x0 = spec.local_x0(inst.x0)
    gam = P.GammaSchedule.pursuit(iterations=args.iters).table()
    iters = len(gam)
    deg = np.diff(np.asarray(g.indptr))
    rows = int((deg > 0).sum())
    out = {"scale": args.scale, "n": g.n, "rows_with_neighbours": rows, "slices": (rows + 31) // 32}
    for mode, name, denom in ((1, "gathers_frac", 2.0 * g.num_edges), (2, "rows_walked_frac", float(rows)),
                              (3, "slices_walked_frac", float((rows + 31) // 32))):
        os.environ["GN_PART_COUNT"] = str(mode)
        be.begin(x0, gam)
        be.run(0, iters)
        torch.cuda.synchronize()
        c = be.gathers(iters)
        be.end(iters)
        out[name + "_by_100"] = [round(float(c[k:k + 100].mean()) / denom, 4) for k in range(0, iters, 100)]
    print(json.dumps(out), flush=True)
    be.close()


if __name__ == "__main__":
    main()
