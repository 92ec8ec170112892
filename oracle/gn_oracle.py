"""Python binding of the CPU oracle (oracle/libgn_oracle.so).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Imported by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg.  The product package must never import this module.

Each function restates a reference routine (see gn_oracle.c for the
file:line citations) and is pinned against the reference's own outputs in
tests/golden (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libgn_oracle.so"

OK = 0
ERR_NEGATIVE = 3
ERR_NOT_NORMALIZABLE = 4
ERR_NONFINITE = 5
TRACE = 1
EARLY_EXIT = 2

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.gno_max_threads.restype = ctypes.c_int
        L.gno_spmv.argtypes = [I64, P, P, P, P]
        L.gno_step.argtypes = [I64, P, P, P, P, ctypes.c_double, P, P, ctypes.c_int]
        L.gno_run.argtypes = [ctypes.c_int, I64, P, P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_uint,
                              ctypes.c_int, P, P, P, P, P, P, P, P, ctypes.c_int, P, P, P]
        L.gno_run.restype = ctypes.c_int
        L.gno_pairwise_sum.argtypes = [P, I64]
        L.gno_pairwise_sum.restype = ctypes.c_double
        L.gno_check.argtypes = [I64, P, P, P, P, P, P, P, P]
        L.gno_round.argtypes = [I64, P, P, P, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _csr(g):
    ip = np.ascontiguousarray(g.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(g.indices, dtype=np.int32)
    w = np.ascontiguousarray(g.w, dtype=np.float64)
    return ip, ix, w


def max_threads() -> int:
    return int(lib().gno_max_threads())


def spmv(g, y) -> np.ndarray:
    ip, ix, _ = _csr(g)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty(g.n, dtype=np.float64)
    lib().gno_spmv(g.n, _p(ip), _p(ix), _p(y), _p(out))
    return out


def step(g, x, gamma, threads: int = 1) -> tuple[np.ndarray, int]:
    ip, ix, w = _csr(g)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(g.n, dtype=np.float64)
    nfb = np.zeros(1, dtype=np.int64)
    lib().gno_step(g.n, _p(ip), _p(ix), _p(w), _p(x), float(gamma), _p(out), _p(nfb), threads)
    return out, int(nfb[0])


@dataclass
class OracleRun:
    status: int
    x: np.ndarray
    iters_run: int
    fail_iter: int
    step_inf: np.ndarray
    fallbacks: np.ndarray
    mass: np.ndarray
    energy: np.ndarray | None = None
    pre_energy: np.ndarray | None = None
    history: np.ndarray | None = None
    snaps: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def run(g, x0, gammas, final_gamma, *, dtype: str = "fp64", trace: bool = False, early_exit: bool = False,
        history: bool = False, threads: int = 1, snaps=None) -> OracleRun:
    """run_wrgn restated (dynamics.py:129-180); gammas = schedule table.
    snaps: ascending iteration indices whose (unclipped) states are returned
    in OracleRun.snaps (one row each)."""
    ip, ix, w = _csr(g)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    gam = np.ascontiguousarray(gammas, dtype=np.float64)
    iters = len(gam)
    x = np.empty(g.n, dtype=np.float64)
    si = np.zeros(iters)
    fb = np.zeros(iters, dtype=np.int64)
    mass = np.zeros(iters)
    en = np.zeros(iters) if trace else None
    pe = np.zeros(iters) if trace else None
    hist = np.zeros((iters, g.n)) if history else None
    sk = None if snaps is None else np.ascontiguousarray(snaps, dtype=np.int32)
    if sk is not None and (np.any(np.diff(sk) < 0) or (len(sk) and (sk[0] < 0 or sk[-1] >= iters))):
        raise ValueError("snaps must be ascending iteration indices below the iteration count")
    xs = None if sk is None else np.zeros((len(sk), g.n))
    ran = ctypes.c_int(0)
    fail = ctypes.c_int(-1)
    flags = (TRACE if trace else 0) | (EARLY_EXIT if early_exit else 0)
    code = {"fp64": 0, "fp32_pure": 1, "fp32": 2, "mixed": 2}[dtype]
    rc = lib().gno_run(code, g.n, _p(ip), _p(ix), _p(w), _p(x0), _p(gam), iters,
                       float(final_gamma), flags, threads, _p(x), _p(si), _p(fb), _p(mass), _p(en), _p(pe),
                       _p(hist), _p(sk), 0 if sk is None else len(sk), _p(xs), ctypes.byref(ran), ctypes.byref(fail))
    k = ran.value
    return OracleRun(rc, x, k, fail.value, si[:k], fb[:k], mass[:k],
                     en[:k] if trace else None, pe[:k] if trace else None,
                     hist[:k] if history else None, xs)


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().gno_pairwise_sum(_p(a), len(a)))


def check(g, mask) -> tuple[float, bool, bool, int]:
    ip, ix, w = _csr(g)
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    weight = ctypes.c_double()
    ind, mx = ctypes.c_int(), ctypes.c_int()
    cnt = ctypes.c_int64()
    lib().gno_check(g.n, _p(ip), _p(ix), _p(w), _p(m), ctypes.byref(weight), ctypes.byref(ind),
                    ctypes.byref(mx), ctypes.byref(cnt))
    return weight.value, bool(ind.value), bool(mx.value), cnt.value


def round_to_mis(g, x) -> tuple[np.ndarray, float, bool, bool]:
    """round_to_mis restated (dynamics.py:253-277): (mask, weight, independent, maximal)."""
    ip, ix, w = _csr(g)
    x = np.ascontiguousarray(x, dtype=np.float64)
    sel = np.zeros(max(g.n, 1), dtype=np.uint8)
    weight = ctypes.c_double()
    ind, mx = ctypes.c_int(), ctypes.c_int()
    cnt = ctypes.c_int64()
    lib().gno_round(g.n, _p(ip), _p(ix), _p(w), _p(x), _p(sel), ctypes.byref(weight), ctypes.byref(ind),
                    ctypes.byref(mx), ctypes.byref(cnt))
    return sel[: g.n].copy(), weight.value, bool(ind.value), bool(mx.value)


def schedule_table(gamma0, gamma1, iterations, mode="linear") -> np.ndarray:
    """GammaSchedule.gamma_at for every k (dynamics.py:65-69)."""
    if mode == "constant":
        return np.full(iterations, float(gamma0))
    out = np.empty(iterations)
    for k in range(iterations):
        p = float(k) / float(iterations - 1)
        out[k] = p * gamma1 + (1.0 - p) * gamma0
    return out


def default_threads() -> int:
    return int(os.environ.get("GN_ORACLE_THREADS", "0")) or (os.cpu_count() or 1)
