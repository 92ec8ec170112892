"""Several starts of run_wrgn on one graph, advanced together on the GPU
(the reference runs them one by one on a thread pool,
solver.py:100-153).

The engine keeps the B states start-minor (x[v][b]) so that one contiguous
read per neighbour serves every start (csrc/gn_multi.cu).  In EXACT mode each
start's trajectory is bitwise its own ``run_wrgn(..., exact=True)`` run: the
same per-row sequential sums, per-start checks, non-finite stop and early
exit.  The fast mode differs only in the rows it splits (hubs).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _engine as E
from .dynamics import GammaSchedule, SolveTrace, _opt, gamma_table
from .graph import device_graph

MAX_STARTS = 64

_STATUS_MESSAGES = {
    E.GN_ERR_NEGATIVE: "state entries must be nonnegative",
    E.GN_ERR_NOT_NORMALIZABLE: "initial state has a zero closed neighborhood sum",
}


@dataclass
class MultiResult:
    x: np.ndarray           # [B, n] final states (clipped)
    step_inf: np.ndarray    # [B, iters] (entries past iters_run[b] are 0)
    fallbacks: np.ndarray   # [B, iters]
    gammas: np.ndarray      # [iters]
    iters_run: np.ndarray   # [B]
    status: np.ndarray      # [B]: 0, or the gn_run error code of that start
    fail_iter: np.ndarray   # [B]: iteration of the non-finite state, else -1
    stats: dict

    def error(self, b: int) -> str | None:
        """The NormalizationError message run_wrgn would raise for start b."""
        st = int(self.status[b])
        if st == E.GN_OK:
            return None
        if st == E.GN_ERR_NONFINITE:
            return f"non-finite state at iteration {int(self.fail_iter[b])}"
        return _STATUS_MESSAGES.get(st, E.last_error())

    def trace(self, b: int) -> SolveTrace:
        k = int(self.iters_run[b])
        t = SolveTrace()
        t.gamma = self.gammas[:k].tolist()
        t.step_inf = self.step_inf[b, :k].tolist()
        t.fallbacks = self.fallbacks[b, :k].tolist()
        return t


def run_multi(g, x0s, schedule: GammaSchedule, early_exit: bool = False, *, dtype=None, exact=None,
              device=None, clip: bool = True) -> MultiResult:
    """run_wrgn(g, x0s[b], schedule) for every start b, in one engine call.

    ``x0s`` is [B, n] (1 <= B <= 64).  Starts that fail the initial checks or
    reach a non-finite state are reported in ``status`` (they do not stop the
    others); ``MultiResult.error(b)`` gives run_wrgn's message for them.
    With ``exact`` every start is bitwise its own ``run_wrgn(exact=True)``;
    otherwise rows longer than a warp's share of the work are summed in
    pieces (fixed piece order: deterministic, within the fp64 tolerance).
    """
    X = np.ascontiguousarray(np.asarray(x0s, dtype=np.float64))
    if X.ndim != 2 or X.shape[1] != g.n:
        raise ValueError(f"starts have shape {X.shape}, expected (B, {g.n})")
    B = X.shape[0]
    if not 1 <= B <= MAX_STARTS:
        raise ValueError(f"between 1 and {MAX_STARTS} starts per call")
    h = device_graph(g, _opt("dtype", dtype), _opt("device", device))
    gam = gamma_table(schedule)
    iters = len(gam)
    x = np.empty((B, g.n))
    si = np.zeros((B, iters))
    fb = np.zeros((B, iters), dtype=np.int64)
    ran = np.zeros(B, dtype=np.int32)
    status = np.zeros(B, dtype=np.int32)
    fail = np.full(B, -1, dtype=np.int32)
    st = E.RunStats()
    flags = (E.GN_EARLY_EXIT if early_exit else 0) | (0 if clip else E.GN_NO_CLIP)
    if _opt("exact", exact):
        flags |= E.GN_EXACT
    rc = E.lib().gn_multi_run(h.handle, B, E.ptr(X), E.ptr(gam), iters, float(schedule.final_gamma), flags,
                              E.ptr(x), E.ptr(si), E.ptr(fb), E.ptr(ran), E.ptr(status), E.ptr(fail),
                              ctypes.byref(st))
    if rc not in (E.GN_OK, E.GN_ERR_NEGATIVE, E.GN_ERR_NOT_NORMALIZABLE, E.GN_ERR_NONFINITE):
        E.check(rc)
    stats = {f: getattr(st, f) for f, _ in E.RunStats._fields_}
    return MultiResult(x, si, fb, gam, ran, status, fail, stats)
