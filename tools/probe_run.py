"""One pursuit of the one-part partitioned engine on an R-MAT graph and
nothing else (the program ncu captures: `-k regex:k_part_step -s <iteration>
-c 1` picks one iteration's step launch).  Prints ms per iteration."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.partition import EngineBackend, build_partition  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--dtype", default="fp64")
    ap.add_argument("--runs", type=int, default=1)
    args = ap.parse_args()
    inst = G.c5_rmat_gpu(args.scale) if args.scale >= 20 else G.c5_rmat(args.scale)
    spec = build_partition(inst.graph, 1, 0)
    be = EngineBackend(spec, dtype=args.dtype)
    x0 = spec.local_x0(inst.x0)
    gam = P.GammaSchedule.pursuit(iterations=args.iters).table()
    for _ in range(args.runs):
        be.begin(x0, gam)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        be.run(0, len(gam))
        e1.record()
        torch.cuda.synchronize()
        be.end(len(gam))
        print(json.dumps({"scale": args.scale, "dtype": args.dtype, "ms_per_iter": e0.elapsed_time(e1) / len(gam)}),
              flush=True)
    be.close()


if __name__ == "__main__":
    main()
