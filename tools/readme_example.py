"""The README quick-start snippet (kept runnable: tools/readme_example.py)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2605_05330_b200 as gn
g = gn.erdos_renyi(1000, 0.01, seed=1)
x, trace = gn.run_wrgn(g, gn.init_random(g.n, 0), gn.GammaSchedule.pursuit())
sol = gn.round_to_mis(g, x)                  # MisSolution(members, weight, independent, maximal)
X0 = np.stack([gn.init_random(g.n, [0, b]) for b in range(16)])
res = gn.run_multi(g, X0, gn.GammaSchedule.pursuit())   # 16 starts in one engine call
print("ok", len(sol.members), sol.weight, res.x.shape)
