"""Golden outcomes of the REFERENCE instance parser (io.py:43-102).

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py

A corpus of instance texts -- valid files, every error the reference raises,
the characters its Python built-ins treat specially, and seeded mutations of
valid files -- is fed to the unmodified reference ``parse_instance``; the
texts and outcomes (the CSR and weights, or the exception type and message)
go to mwis_corpus.json, which tests/test_io.py replays against the engine's
parser.
"""

from __future__ import annotations

import json
import re
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from graphnorm.io import parse_instance  # noqa: E402  (the reference)


def base_text(rng, n, m, crlf=False, comments=True):
    lines = []
    if comments:
        lines.append("c generated instance")
    lines.append(f"p mwis {n} {m}")
    ids = list(range(1, n + 1))
    rng.shuffle(ids)
    for v in ids:
        lines.append(f"n {v} {rng.uniform(0.01, 10):.{rng.integers(1, 17)}g}")
    for _ in range(m):
        u = int(rng.integers(1, n + 1))
        v = int(rng.integers(1, n + 1))
        while v == u and n > 1:
            v = int(rng.integers(1, n + 1))
        lines.append(f"e {u} {v}")
    rng.shuffle(lines[2 if comments else 1:])  # weights and edges interleave freely after the problem line
    sep = "\r\n" if crlf else "\n"
    return sep.join(lines) + sep


HAND = [
    "",
    "c only a comment\n",
    "p mwis 0 0\n",
    "p mwis 1 0\nn 1 1\n",
    "p mwis 2 1\nn 1 1\nn 2 2\ne 1 2\n",
    "p mwis 2 2\nn 1 1\nn 2 2\ne 1 2\ne 2 1\n",            # both orientations merge
    "p mwis 3 3\nn 1 1\nn 2 2\nn 3 3\ne 1 2\ne 1 2\ne 2 3\n",  # duplicate edge
    "  p   mwis  2 1 \n\tn 1 1.5\nn 2\t2e0\n e 1 2\n\n\n",
    "p mwis 2 1\r\nn 1 1\r\nn 2 2\r\ne 1 2",                # CRLF, no final newline
    "p mwis 2 1\rn 1 1\rn 2 2\re 1 2\r",                    # lone CR
    "cp mwis 5 5\np mwis 1 0\nn 1 1\n",                     # any line starting with c is a comment
    "p mwis 1 0\nn 1 +1.5\n", "p mwis 1 0\nn +1 .5\n", "p mwis 1 0\nn 1 5.\n", "p mwis 1 0\nn 01 1e-3\n",
    "p mwis 1 0\nn 1 1E+2\n", "p mwis 1 0\nn 1 1e400\n", "p mwis 1 0\nn 1 1e-400\n", "p mwis 1 0\nn 1 4.9e-324\n",
    "p mwis 1 0\nn 1 inf\n", "p mwis 1 0\nn 1 -Infinity\n", "p mwis 1 0\nn 1 NaN\n", "p mwis 1 0\nn 1 0\n",
    "p mwis 1 0\nn 1 -1\n", "p mwis 1 0\nn 1 0x10\n", "p mwis 1 0\nn 1 1e\n", "p mwis 1 0\nn 1 .\n",
    "p mwis 1 0\nn 1 infinit\n", "p mwis 1 0\nn 1 1_000.5\n", "p mwis 1 0\nn 1 nan(1)\n",
    "p mwis 1 0\nn 1 0.1000000000000000055511151231257827\n",
    "p mwis 3 0\nn 1 1\nn 2 2\n",                          # missing weight
    "p mwis 3 1\nn 1 1\nn 2 2\nn 3 3\n",                    # edge count
    "p mwis 3 0\nn 1 1\nn 2 2\nn 3 3\ne 1 2\n",             # edge count (more)
    "n 1 1\np mwis 1 0\n", "e 1 2\np mwis 2 1\n", "p mwis 1 0\np mwis 1 0\nn 1 1\n",
    "p mwis 1\n", "p mwis 1 0 0\n", "p mwiz 1 0\n", "p MWIS 1 0\n", "p mwis x 0\n", "p mwis 1 y\n",
    "p mwis -1 0\n", "p mwis 2 -1\nn 1 1\nn 2 1\n", "p mwis 1_0 0\n", "p mwis 99999999999999999999 0\nq\n",
    "p mwis 2 0\nn 0 1\nn 2 1\n", "p mwis 2 0\nn 3 1\n", "p mwis 2 0\nn -1 1\n", "p mwis 2 0\nn 1 1\nn 1 2\n",
    "p mwis 2 0\nn 1\n", "p mwis 2 0\nn 1 1 1\n", "p mwis 2 0\nn a 1\n", "p mwis 2 0\nn 1.0 1\n",
    "p mwis 2 1\nn 1 1\nn 2 1\ne 1\n", "p mwis 2 1\nn 1 1\nn 2 1\ne 1 2 3\n", "p mwis 2 1\nn 1 1\nn 2 1\ne 0 1\n",
    "p mwis 2 1\nn 1 1\nn 2 1\ne 1 3\n", "p mwis 2 1\nn 1 1\nn 2 1\ne 1 1\n", "p mwis 2 1\nn 1 1\nn 2 1\ne 1 x\n",
    "p mwis 2 1\nn 1 1\nn 2 1\ne +1 +2\n", "p mwis 2 1\nn 1 1\nn 2 1\ne 1_0 2\n",
    "x\n", "P mwis 1 0\n", "nn 1 1\n", "p mwis 1 0\nq 1\n", "p mwis 1 0\nn 1 1\nz 'quoted'\n",
    "p mwis 1 0\nn 1 1\nx\"y\n", "p mwis 1 0\nn 1 1\nx\\y\n", "p mwis 1 0\nn 1 1 'a'\n",
    "p mwis 1 0\nn 1 1\n\x0bq\n", "p mwis 1 0\nn 1 1\n\x0cq\n", "p mwis 1 0\x1cn 1 1\n",
    "p mwis 1 0\nn 1 1\xa0\n", "p mwis 1 0\nn 1 ١\n", "p mwis 1 0\nn ١ 1\n", "p mwis 1 0 n 1 1\n",
    "p mwis 1 0\nn 1 1\n\x00\n", "p mwis 1 0\nn 1\t\t1\n", "p mwis 1 0\nn 1 1\n\t\n", "p mwis 1 0\nn 1 1\nc\x85\n",
]


def mutate(rng, text):
    s = list(text)
    for _ in range(int(rng.integers(1, 4))):
        op = int(rng.integers(0, 6))
        i = int(rng.integers(0, max(len(s), 1)))
        if op == 0 and s:
            del s[i % len(s)]
        elif op == 1:
            s.insert(i, str(int(rng.integers(0, 10))))
        elif op == 2:
            s.insert(i, rng.choice([" ", "\t", "\n", "\r", "\r\n", "-", "+", ".", "e", "x", "'", "_", "é"]))
        elif op == 3 and s:
            j = int(rng.integers(0, len(s)))
            s[i % len(s)], s[j] = s[j], s[i % len(s)]
        elif op == 4:
            s.insert(i, rng.choice(["p mwis 3 3\n", "n 1 2\n", "e 1 2\n", "c x\n", "e 2 2\n"]))
        elif s:
            s[i % len(s)] = rng.choice(["0", "9", "n", "e", "p", " "])
    return "".join(s)


def outcome(text):
    try:
        g = parse_instance(text)
    except Exception as exc:  # noqa: BLE001 -- the type is part of the record
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"n": int(g.n), "indptr": np.asarray(g.indptr).tolist(), "indices": np.asarray(g.indices).tolist(),
            "w": [float(x).hex() for x in np.asarray(g.w, np.float64)]}


def main():
    rng = np.random.default_rng(2605_0010)
    texts = list(HAND)
    for k in range(20):
        n = int(rng.integers(1, 30))
        texts.append(base_text(rng, n, int(rng.integers(0, 3 * n)), crlf=bool(k % 3 == 0), comments=bool(k % 2)))
    for _ in range(160):
        n = int(rng.integers(1, 8))
        texts.append(mutate(rng, base_text(rng, n, int(rng.integers(0, 2 * n)), comments=False)))
    # the reference lists every missing vertex id (io.py:93): keep n small
    texts = [t for t in texts if max([0] + [int(x) for x in re.findall(r"p\s+mwis\s+(\d+)", t)]) <= 10**6
             or "\nq\n" in t]
    cases = [{"text": t, **outcome(t)} for t in texts]
    (HERE / "mwis_corpus.json").write_text(json.dumps({"generator": "tests/golden/make_io_golden.py",
                                                       "reference": "graphnorm.io.parse_instance",
                                                       "cases": cases}, indent=0))
    print(len(cases), "cases,", sum("error" in c for c in cases), "errors")


if __name__ == "__main__":
    main()
