"""Batches of independent graphs on one GPU (BASELINE config C4).

Each graph of the batch runs its own run_wrgn (dynamics.py:129-180) on one
CTA with the whole graph resident in shared memory (csrc/gn_batch.cu): the
same results, bit for bit, as calling run_wrgn graph by graph, without a grid
barrier or HBM traffic per iteration.  Multi-GPU sharding of a batch family is
in parallel.py (rank r takes its own slice of graphs, no collectives).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _engine as E
from .dynamics import GammaSchedule, NormalizationError, _opt, gamma_table
from .graph import WeightedGraph, csr_from_edges, dtype_code, from_csr


@dataclass
class BatchResult:
    x: np.ndarray                # packed final states (clipped), original vertex order
    step_inf: np.ndarray         # [B, iters] (entries past iters_run[b] are 0)
    fallbacks: np.ndarray        # [B, iters]
    objective: np.ndarray        # [B, iters]: w.x after each step
    iters_run: np.ndarray        # [B]
    status: np.ndarray           # [B]: 0, or the gn_run error code of that graph
    stats: dict

    def state(self, b: int, offsets: np.ndarray) -> np.ndarray:
        return self.x[offsets[b]:offsets[b + 1]]


class GraphBatch:
    """B independent graphs packed block-diagonally (graph b owns vertices
    offsets[b]..offsets[b+1]-1)."""

    def __init__(self, packed: WeightedGraph, offsets: Sequence[int], dtype=None, device: Optional[int] = None):
        self.graph = packed
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        if self.offsets[0] != 0 or self.offsets[-1] != packed.n:
            raise ValueError("offsets must run from 0 to the packed vertex count")
        self.B = len(self.offsets) - 1
        self.dtype = _opt("dtype", dtype)
        self.device = _opt("device", device)
        self._lib = E.lib()
        h = ctypes.c_void_p()
        ip = np.ascontiguousarray(packed.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(packed.indices, dtype=np.int32)
        w = np.ascontiguousarray(packed.w, dtype=np.float64)
        E.check(self._lib.gn_batch_create(self.B, E.ptr(self.offsets), packed.n, E.ptr(ip), E.ptr(ix), E.ptr(w),
                                          dtype_code(self.dtype), int(self.device), ctypes.byref(h)))
        self._h = h

    @classmethod
    def from_graphs(cls, graphs: Sequence[WeightedGraph], dtype=None, device=None) -> "GraphBatch":
        offs = np.zeros(len(graphs) + 1, dtype=np.int64)
        np.cumsum([g.n for g in graphs], out=offs[1:])
        rows, cols = [], []
        for g, o in zip(graphs, offs[:-1]):
            r = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.indptr))
            keep = np.asarray(g.indices) > r
            rows.append(r[keep] + o)
            cols.append(np.asarray(g.indices, dtype=np.int64)[keep] + o)
        n = int(offs[-1])
        indptr, indices = csr_from_edges(n, np.concatenate(rows) if rows else np.zeros(0, np.int64),
                                         np.concatenate(cols) if cols else np.zeros(0, np.int64))
        w = np.concatenate([np.asarray(g.w, dtype=np.float64) for g in graphs]) if graphs else np.zeros(0)
        return cls(from_csr(n, indptr, indices, w, validate=False), offs, dtype, device)

    def info(self) -> dict:
        B, n, db, sm = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        E.check(self._lib.gn_batch_info(self._h, ctypes.byref(B), ctypes.byref(n), ctypes.byref(db), ctypes.byref(sm)))
        return {"graphs": B.value, "n": n.value, "device_bytes": db.value, "smem_bytes_per_graph_cta": sm.value}

    def run(self, x0, schedule: GammaSchedule, early_exit: bool = False, *, raise_on_error: bool = False,
            device_x0=None, device_x_out=None, traces: bool = True) -> BatchResult:
        """run_wrgn on every graph.  x0 is the packed start (host numpy), or
        device_x0/device_x_out are fp64 CUDA pointers (inputs already in HBM)."""
        iters = schedule.iterations
        gam = gamma_table(schedule)
        B = self.B
        si = np.zeros((B, iters))
        fb = np.zeros((B, iters), dtype=np.int64)
        ob = np.zeros((B, iters))
        ran = np.zeros(B, dtype=np.int32)
        status = np.zeros(B, dtype=np.int32)
        fail = np.zeros(B, dtype=np.int32)
        st = E.RunStats()
        flags = E.GN_EARLY_EXIT if early_exit else 0
        if device_x0 is not None:
            flags |= E.GN_DEVICE_IO
            xin, xout, x = ctypes.c_void_p(device_x0), ctypes.c_void_p(device_x_out), None
        else:
            xh = np.ascontiguousarray(x0, dtype=np.float64)
            if xh.shape != (self.graph.n,):
                raise ValueError(f"x0 has shape {xh.shape}, expected ({self.graph.n},)")
            x = np.empty(self.graph.n)
            xin, xout = E.ptr(xh), E.ptr(x)
        tr = (E.ptr(si), E.ptr(fb), E.ptr(ob)) if traces else (None, None, None)
        rc = self._lib.gn_batch_run(self._h, xin, E.ptr(gam), iters, float(schedule.final_gamma), flags, xout,
                                    *tr, E.ptr(ran), E.ptr(status), E.ptr(fail), ctypes.byref(st))
        if rc not in (E.GN_OK, E.GN_ERR_NEGATIVE, E.GN_ERR_NOT_NORMALIZABLE, E.GN_ERR_NONFINITE):
            E.check(rc)
        if raise_on_error and rc != E.GN_OK:
            raise NormalizationError(E.last_error())
        stats = {f: getattr(st, f) for f, _ in E.RunStats._fields_}
        return BatchResult(x, si, fb, ob, ran, status, stats)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            self._lib.gn_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
