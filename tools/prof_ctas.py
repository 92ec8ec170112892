"""Per-CTA timeline of one loop-kernel iteration joined with the CTA's plan
(development aid): run with GN_PROF_ITER / GN_PLAN_DUMP=2 output files."""
import re
import sys

import numpy as np

prof, plan = sys.argv[1], sys.argv[2]
L = [l for l in open(prof) if not l.startswith("#")]
G = int(sys.argv[3]) if len(sys.argv) > 3 else 148
L = L[-G:]
cta = {}
for l in open(plan):
    m = re.match(r"\[cta (\d+)\] whole=(\d+) piece=(\d+) hub=(\d+) resident=(\d+) elems=(\d+) combs=(\d+)", l)
    if m:
        cta[int(m.group(1))] = tuple(int(x) for x in m.groups()[1:])
rows = []
for l in L:
    a, b = l.split("|")
    c = list(map(int, a.split()))
    w = list(map(int, b.split()))
    rows.append((c, w))
d = np.array([r[0][2] - r[0][1] for r in rows])
W = np.array([r[1] for r in rows])
print("pass us: min %.2f med %.2f p90 %.2f max %.2f" % (d.min() / 1e3, np.median(d) / 1e3, np.percentile(d, 90) / 1e3,
                                                       d.max() / 1e3))
print("warp items us: med %.2f max %.2f" % (np.median(W) / 1e3, W.max() / 1e3))
for i in np.argsort(-d)[:10]:
    print("CTA %3d pass %.2f warps max %.2f min %.2f plan(whole,piece,hub,res,elems,combs)=%s" % (
        i, d[i] / 1e3, W[i].max() / 1e3, W[i].min() / 1e3, cta.get(int(i))))
