"""Zero-row certificates A/B (development aid, not the bench contract).

One-part partitioned engine on an R-MAT graph (or C2/C3): the whole pursuit
with the certificates off (GN_PART_WITNESS=0) and on, timed with CUDA events
on the engine's stream; every output compared bit for bit between the two;
a counting run (GN_PART_COUNT=1) reports the value gathers issued per
iteration against the adjacency size.  One JSON line per mode + a summary.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.partition import EngineBackend, build_partition  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--inst", default="C5S24", help="C5S<scale>, C2 or C3")
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--dtype", default="fp64")
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    t = time.time()
    if args.inst.startswith("C5S"):
        sc = int(args.inst[3:])
        inst = G.c5_rmat_gpu(sc) if sc >= 20 else G.c5_rmat(sc)
    else:
        inst = G.CONFIGS[args.inst]()
    g = inst.graph
    print(f"gen {args.inst}: n={g.n} m={g.num_edges} {time.time() - t:.1f}s", file=sys.stderr, flush=True)
    spec = build_partition(g, 1, 0)
    be = EngineBackend(spec, dtype=args.dtype, exact=args.exact)
    x0 = spec.local_x0(inst.x0)
    gam = P.GammaSchedule.pursuit(iterations=args.iters).table()
    iters = len(gam)
    nnz = 2 * g.num_edges
    res = {}
    modes = {"0": ("0", "0"), "1": ("1", "0"), "2": ("1", "1")}  # certificates off / on / on + settled rows
    for mode in ("0", "1", "2"):
        os.environ["GN_PART_WITNESS"], os.environ["GN_PART_SETTLE"] = modes[mode]
        os.environ["GN_PART_COUNT"] = "0"
        best = None
        for _ in range(args.reps + 1):
            be.begin(x0, gam)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            be.run(0, iters)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out = be.end(iters)
        # per-100-iteration segments: host-issued steps (the GPU stays busy;
        # events between segments)
        be.begin(x0, gam)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(iters // 100 + 2)]
        ev[0].record()
        for k in range(iters):
            be.step(k)
            if (k + 1) % 100 == 0 or k + 1 == iters:
                ev[(k + 99) // 100].record()
        torch.cuda.synchronize()
        seg = [round(ev[j].elapsed_time(ev[j + 1]) / 100, 4) for j in range((iters + 99) // 100)]
        be.end(iters)
        os.environ["GN_PART_COUNT"] = "1"
        be.begin(x0, gam)
        be.run(0, iters)
        torch.cuda.synchronize()
        gat = be.gathers(iters)
        be.end(iters)
        res[mode] = (best, out, gat)
        rec = {"inst": args.inst, "dtype": args.dtype, "exact": args.exact, "mode": {"0": "off", "1": "certificates", "2": "certificates + settled rows"}[mode],
               "ms_per_iter": round(best / iters, 4), "Geu_s": round(g.num_edges * iters / best / 1e6, 2),
               "gathers_frac_of_nnz_total": round(float(gat.sum()) / (nnz * iters), 4),
               "gathers_frac_by_100": [round(float(gat[k:k + 100].mean()) / nnz, 3) for k in range(0, iters, 100)],
               "fallbacks": int(out[2].sum()), "ms_per_iter_by_100": seg}
        print(json.dumps(rec), flush=True)
    (b0, o0, _), (b1, o1, _), (b2, o2, _) = res["0"], res["1"], res["2"]
    same = {name: bool(np.array_equal(a, b) and np.array_equal(a, c)) for name, a, b, c in
            (("x", o0[0], o1[0], o2[0]), ("step_inf", o0[1], o1[1], o2[1]), ("fallbacks", o0[2], o1[2], o2[2]),
             ("mass", o0[3], o1[3], o2[3]))}
    print(json.dumps({"inst": args.inst, "speedup_certificates": round(b0 / b1, 3),
                      "speedup_settled": round(b0 / b2, 3), "bitwise_same": same}), flush=True)
    be.close()


if __name__ == "__main__":
    main()
