#!/usr/bin/env python3
"""Model of the L1TEX cost of the partitioned step's gathers (C5, R-MAT).

The L1TEX unit processes one 128-byte line (a "wavefront") per cycle per SM
(B300_MICROARCH.md, "L1tex wavefront queue"): a warp gather whose 32 lanes
touch k distinct lines costs k cycles of that unit, hit or miss.  For the
thread-per-row SELL walk of gn_part.cu, the lanes of a slice gather
position p of 32 consecutive rows at once; for the warp-split long rows the
lanes gather 32 consecutive positions of one row.  This script counts the
distinct lines per warp gather for a vertex order, i.e. the wavefronts per
iteration, and what an order or a shared-memory hot set would save.

    python tools/wavefront_model.py --scale 20
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

LONG = 512


def relabel(indptr, indices, order):
    """CSR in the numbering new = position of the vertex in `order`."""
    n = len(indptr) - 1
    inv = np.empty(n, np.int64)
    inv[order] = np.arange(n)
    deg = np.diff(indptr)[order]
    nptr = np.concatenate([[0], np.cumsum(deg)])
    rows = np.repeat(order, deg)
    starts = indptr[order]
    off = np.arange(nptr[-1]) - np.repeat(nptr[:-1], deg)
    ncol = inv[indices[np.repeat(starts, deg) + off]]
    # fast mode: every row in ascending new id
    key = np.repeat(np.arange(n), deg) * np.int64(n) + ncol
    ncol = (np.sort(key) % n)
    return nptr, ncol


def wavefronts(nptr, ncol, elem=4, hot=0):
    """Distinct 128-byte lines per warp gather, summed (thread-per-row SELL
    slices of 32 rows for rows of degree <= 512; warp-split walks above),
    gathers of new ids < hot excluded (served from shared memory)."""
    per_line = 128 // elem
    deg = np.diff(nptr)
    n = len(deg)
    longr = np.flatnonzero(deg > LONG)
    total = 0
    gathers = 0
    # long rows: 32 consecutive positions per warp instruction
    for r in longr:
        c = ncol[nptr[r]:nptr[r + 1]]
        c = c[c >= hot]
        gathers += len(c)
        if len(c):
            grp = np.arange(len(c)) // 32
            total += len(np.unique(grp * (n // per_line + 1) + c // per_line))
    short = np.flatnonzero(deg <= LONG)
    # slices: 32 consecutive short rows; position p of each
    sl = np.arange(len(short)) // 32
    d = deg[short]
    rows = np.repeat(short, d)
    pos = np.arange(d.sum()) - np.repeat(np.concatenate([[0], np.cumsum(d)[:-1]]), d)
    slc = np.repeat(sl, d)
    c = ncol[np.repeat(nptr[short], d) + pos]
    keep = c >= hot
    gathers += int(keep.sum())
    key = (slc[keep].astype(np.int64) * (LONG + 1) + pos[keep]) * (n // per_line + 1) + c[keep] // per_line
    total += len(np.unique(key))
    return total, gathers


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    args = ap.parse_args()
    from paper_2605_05330_b200 import generators as G

    t = time.time()
    inst = G.c5_rmat(args.scale)
    g = inst.graph
    indptr, indices = np.asarray(g.indptr, np.int64), np.asarray(g.indices, np.int64)
    n = g.n
    deg = np.diff(indptr)
    print(f"scale {args.scale}: n={n} nnz={len(indices)} gen {time.time() - t:.1f}s", flush=True)
    # hot-set coverage in the global degree order
    srt = np.sort(deg)[::-1]
    cum = np.cumsum(srt) / srt.sum()
    for h in (1024, 4096, 16384, 49152, 65536):
        print(f"  top {h:6d} vertices by degree receive {100 * cum[min(h, n) - 1]:.1f}% of the gathers")
    orders = {}
    orders["caller"] = np.arange(n)
    orders["global degree"] = np.argsort(-deg, kind="stable")
    win = 1 << 18
    o = []
    for w0 in range(0, n, win):
        ids = np.arange(w0, min(n, w0 + win))
        o.append(ids[np.argsort(-deg[ids], kind="stable")])
    # engine: long rows first (global), then windows
    o = np.concatenate(o)
    lng = o[deg[o] > LONG]
    orders["engine (long first, degree in 2^18 windows)"] = np.concatenate([lng[np.argsort(-deg[lng], kind="stable")],
                                                                         o[deg[o] <= LONG]])
    for name, order in orders.items():
        nptr, ncol = relabel(indptr, indices, order)
        for hot in (0, 16384, 49152):
            wf, ga = wavefronts(nptr, ncol, hot=hot)
            print(f"{name:48s} hot={hot:6d}: {wf / 1e6:8.2f} M wavefronts, {ga / 1e6:8.2f} M L1 gathers, "
                  f"{wf / max(ga, 1) * 32:.2f} lines per 32 gathers", flush=True)


if __name__ == "__main__":
    main()
