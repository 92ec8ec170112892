"""One-part partitioned engine timing on any config (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2605_05330_b200 as P  # noqa: E402
from paper_2605_05330_b200 import generators as G  # noqa: E402
from paper_2605_05330_b200.partition import EngineBackend, build_partitions  # noqa: E402

name = sys.argv[1]
dtype = sys.argv[2] if len(sys.argv) > 2 else None
inst = G.CONFIGS[name]()
spec = build_partitions(inst.graph, 1)[0]
be = EngineBackend(spec, dtype=dtype or inst.dtype)
gam = P.GammaSchedule.pursuit().table()
x0 = spec.local_x0(inst.x0)
for rep in range(3):
    be.begin(x0, gam)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(len(gam)):
        be.step(k)
    e1.record()
    torch.cuda.synchronize()
    print(name, dtype or inst.dtype, "us/iter %.3f" % (e0.elapsed_time(e1) * 1e3 / len(gam)), flush=True)
