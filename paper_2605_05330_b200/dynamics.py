"""Weighted regularized graph-normalization dynamics on the B200 engine.

Drop-in for graphnorm.dynamics (/root/reference/pkg/src/graphnorm/dynamics.py):
same names, signatures, return types, exceptions and messages.  Every step,
reduction, check and the rounding run in the CUDA engine (libgnb200.so) --
there is no CPU path.  Host-side code here only prepares inputs (the gamma
table, the seeded start vectors) and unpacks results.

Engine options are keyword-only extras the reference does not have:
``dtype`` ("fp64" default = the reference arithmetic, or "fp32"),
``exact`` (one thread per row, sequential sums: fp64 is then bitwise equal to
the reference) and ``device`` (CUDA ordinal).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _engine as E
import threading as _threading

from .graph import MisSolution, any_device_graph, device_graph, dtype_code

# dynamics.py:21-24
SAFE_DIV_THRESHOLD = 1e-9
FALLBACK_VALUE = 0.5

CLAMP_FLOOR = 1e-3

_DEFAULTS = {"dtype": "fp64", "exact": False, "device": 0, "engine": "auto"}


def set_engine_defaults(dtype=None, exact=None, device=None, engine=None) -> dict:
    """Change the engine options used when a call does not pass them."""
    if engine is not None:
        if engine not in ("auto", "loop", "part"):
            raise ValueError("engine must be 'auto', 'loop' or 'part'")
        _DEFAULTS["engine"] = engine
    if dtype is not None:
        dtype_code(dtype)
        _DEFAULTS["dtype"] = dtype
    if exact is not None:
        _DEFAULTS["exact"] = bool(exact)
    if device is not None:
        _DEFAULTS["device"] = int(device)
    return dict(_DEFAULTS)


def _opt(name, value):
    return _DEFAULTS[name] if value is None else value


class NormalizationError(ValueError):
    """Raised when a state has a zero closed neighborhood sum."""


@dataclass(frozen=True)
class GammaSchedule:
    """Interpolation plan for the regularization parameter (dynamics.py:31-73).

    linear mode moves gamma from gamma0 at step 0 to gamma1 at the last
    step; constant mode holds gamma0 throughout.
    """

    gamma0: float
    gamma1: float
    iterations: int
    mode: str = "linear"

    def __post_init__(self):
        if self.mode not in ("constant", "linear"):
            raise ValueError(f"unknown schedule mode {self.mode!r}")
        if self.iterations < 1:
            raise ValueError("iterations must be positive")
        if self.mode == "linear" and self.iterations < 2:
            raise ValueError("linear mode needs at least 2 iterations")
        if self.gamma0 < 0 or self.gamma1 < 0:
            raise ValueError("gamma must be nonnegative")

    @classmethod
    def constant(cls, gamma: float, iterations: int) -> "GammaSchedule":
        return cls(gamma, gamma, iterations, mode="constant")

    @classmethod
    def pursuit(cls, gamma0: float = 0.9, gamma1: float = 1.5, iterations: int = 1000) -> "GammaSchedule":
        """Default graduated schedule: linear 0.9 -> 1.5 over 1000 steps."""
        return cls(gamma0, gamma1, iterations, mode="linear")

    def gamma_at(self, k: int) -> float:
        if self.mode == "constant":
            return self.gamma0
        p = float(k) / float(self.iterations - 1)
        return p * self.gamma1 + (1.0 - p) * self.gamma0

    @property
    def final_gamma(self) -> float:
        return self.gamma0 if self.mode == "constant" else self.gamma1

    def table(self) -> np.ndarray:
        """gamma_at(k) for every k, with the same IEEE operations (bitwise)."""
        if self.mode == "constant":
            return np.full(self.iterations, float(self.gamma0), dtype=np.float64)
        p = np.arange(self.iterations, dtype=np.float64) / float(self.iterations - 1)
        return p * float(self.gamma1) + (1.0 - p) * float(self.gamma0)


@dataclass
class SolveTrace:
    """Per-iteration record of one trajectory (dynamics.py:76-99).

    gamma, step_inf, and fallbacks are always populated.  The energy and
    mass series are filled only when the run records a full trace.
    ``objective`` is an engine extra: the relaxed MWIS primal w.x after every
    step, computed by the fused reduction on every run.
    """

    gamma: list = field(default_factory=list)
    energy: list = field(default_factory=list)
    pre_energy: list = field(default_factory=list)
    mass: list = field(default_factory=list)
    step_inf: list = field(default_factory=list)
    fallbacks: list = field(default_factory=list)
    objective: list = field(default_factory=list, repr=False, compare=False)

    @property
    def total_fallbacks(self) -> int:
        return sum(self.fallbacks)

    def __len__(self) -> int:
        return len(self.gamma)


def gamma_table(schedule) -> np.ndarray:
    """gamma_at(k) for every k of the run (dynamics.py:65-69), as a float64
    array: GammaSchedule.table() for the engine's own schedules, else the
    schedule's own gamma_at -- so the reference's graphnorm.GammaSchedule
    (or any object with iterations / gamma_at / final_gamma) drives the
    engine with bitwise its own values."""
    t = getattr(schedule, "table", None)
    if callable(t):
        return np.ascontiguousarray(t(), dtype=np.float64)
    return np.array([schedule.gamma_at(k) for k in range(int(schedule.iterations))], dtype=np.float64)


def _device_state(g, x):
    """A CUDA fp64 tensor of n entries (a state kept in HBM, e.g.
    run_engine(..., device_state=True).x), or None for host arrays."""
    if type(x).__module__.split(".")[0] != "torch" or not getattr(x, "is_cuda", False):
        return None
    import torch

    if x.dtype != torch.float64 or tuple(x.shape) != (g.n,) or not x.is_contiguous():
        raise ValueError(f"device state must be a contiguous float64 CUDA tensor of shape ({g.n},)")
    return x


def _as_state(g, x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.shape != (g.n,):
        raise ValueError(f"state has shape {x.shape}, expected ({g.n},)")
    return x


def gn_step(g, x, gamma: float, *, dtype=None, exact=None, device=None) -> np.ndarray:
    """Apply the weighted regularized normalization map once (dynamics.py:111-119).

    x'_i = x_i / (x_i + gamma * sum_{j ~ i} (v_j / v_i) x_j).  Entries whose
    denominator is at or below the safe-division threshold are set to the
    fallback value 0.5 instead of raising.
    """
    x = _as_state(g, x)
    h = device_graph(g, _opt("dtype", dtype), _opt("device", device))
    out = np.empty(g.n, dtype=np.float64)
    nfb = ctypes.c_int64(0)
    flags = E.GN_EXACT if _opt("exact", exact) else 0
    E.check(E.lib().gn_step(h.handle, E.ptr(x), float(gamma), flags, E.ptr(out), ctypes.byref(nfb)))
    return out


def is_normalizable(g, x) -> bool:
    """All closed neighborhood sums positive (dynamics.py:122-126)."""
    x = _as_state(g, x)
    ok = ctypes.c_int(0)
    h = any_device_graph(g, _opt("device", None))
    E.check(E.lib().gn_is_normalizable(h.handle, E.ptr(x), ctypes.byref(ok)))
    return bool(ok.value)


_RUN_ERRORS = {
    E.GN_ERR_NEGATIVE: "state entries must be nonnegative",
    E.GN_ERR_NOT_NORMALIZABLE: "initial state has a zero closed neighborhood sum",
}


@dataclass
class RunResult:
    """Everything one engine run returns (run_wrgn keeps the reference shape)."""

    x: np.ndarray
    trace: SolveTrace
    stats: dict
    history: Optional[np.ndarray] = None


# Large graphs: fast-mode runs without trace, history or early exit go to the
# partitioned engine with one part (csrc/gn_part.cu), which runs them faster
# than the persistent loop kernel (C5 scale 24, fp64: 1.33 against 1.73 ms per
# iteration).  Threshold: adjacency entries.
PART_ROUTE_NNZ = 1 << 26
_PART_CACHE: "OrderedDict[tuple, tuple]" = None  # (id(g), dtype, device) -> (g, backend, lock)
_PART_MAX = 2
_PART_LOCK = _threading.Lock()


def _part_backend(g, dtype, dev):
    """The one-part partitioned backend of g (built on first use, cached;
    the cache keeps g alive so ids are not reused)."""
    global _PART_CACHE
    import threading
    from collections import OrderedDict

    from .partition import EngineBackend, build_partition

    if _PART_CACHE is None:
        _PART_CACHE = OrderedDict()
    key = (id(g), dtype_code(dtype), int(dev))
    with _PART_LOCK:
        hit = _PART_CACHE.get(key)
        if hit is not None and hit[0] is g:
            _PART_CACHE.move_to_end(key)
            return hit[1], hit[2]
        spec = build_partition(g, 1, 0)
        be = EngineBackend(spec, dtype=dtype, device=dev, exact=False)
        _PART_CACHE[key] = (g, be, threading.Lock())
        while len(_PART_CACHE) > _PART_MAX:
            _, (_, old, _) = _PART_CACHE.popitem(last=False)
            old.close()
        return be, _PART_CACHE[key][2]


def _check_x0_host(g, x: np.ndarray) -> None:
    """dynamics.py:146-149 on the host: negative entries, then the closed
    neighbourhood sums (for x >= 0 a sum is > 0 iff some term is, NaN iff
    some term is NaN; only rows whose own entry is 0 need their neighbours)."""
    if np.any(x < 0):
        raise NormalizationError(_RUN_ERRORS[E.GN_ERR_NEGATIVE])
    if np.isnan(x).any():
        raise NormalizationError(_RUN_ERRORS[E.GN_ERR_NOT_NORMALIZABLE])
    zero = np.flatnonzero(x == 0)
    if len(zero):
        ip = np.asarray(g.indptr)
        ix = np.asarray(g.indices)
        for i in zero.tolist():
            if not np.any(x[ix[ip[i]:ip[i + 1]]] > 0):
                raise NormalizationError(_RUN_ERRORS[E.GN_ERR_NOT_NORMALIZABLE])


def _run_part(g, x0, gam, dtype, dev) -> "RunResult":
    """A fast-mode run of the whole graph through the partitioned engine
    with one part (x0 checks on the host, the non-finite stop as run_wrgn's)."""
    x = _as_state(g, x0)
    _check_x0_host(g, x)
    be, lock = _part_backend(g, dtype, dev)
    with lock:  # one run at a time per backend (the reference solver calls from several threads)
        be.begin(x, gam)
        be.run(0, len(gam))
        xo, si, fb, ms, bad = be.end(len(gam))
    if bad >= 0:
        raise NormalizationError(f"non-finite state at iteration {bad}")
    trace = SolveTrace()
    trace.gamma = gam.tolist()
    trace.step_inf = si.tolist()
    trace.fallbacks = [int(v) for v in fb]
    trace.objective = ms.tolist()
    return RunResult(xo, trace, {"engine": "partitioned (one part)"}, None)


def run_engine(g, x0, schedule: GammaSchedule, record_trace: bool = False, early_exit: bool = False, *,
               dtype=None, exact=None, device=None, history: bool = False,
               gammas: Optional[np.ndarray] = None, device_state: bool = False, engine=None) -> RunResult:
    """run_wrgn with the engine's extras (stats, optional per-iteration x).

    ``gammas`` replaces the schedule's table (e.g. a prefix of a pursuit
    schedule); the early-exit test still compares with schedule.final_gamma.
    ``device_state``: x0 may be a CUDA fp64 tensor and the result's x stays
    in HBM as one (GN_DEVICE_IO), ready for round_to_mis / round_many without
    a host round trip (the solver's run -> round hand-over, solver.py:75,88).
    ``engine``: "loop" (the persistent loop kernel), "part" (the partitioned
    engine with one part: fast mode without trace, history or early exit) or
    "auto" (default: "part" for such runs on graphs of >= PART_ROUTE_NNZ
    adjacency entries, else "loop").
    """
    dev = _opt("device", device)
    eng = _opt("engine", engine)
    if eng not in ("auto", "loop", "part"):
        raise ValueError("engine must be 'auto', 'loop' or 'part'")
    routable = not (_opt("exact", exact) or record_trace or early_exit or history or device_state
                    or _device_state(g, x0) is not None)
    if eng == "part" and not routable:
        raise ValueError("engine='part' runs fast mode without trace, history, early exit or device state")
    if eng == "part" or (eng == "auto" and routable and len(g.indices) >= PART_ROUTE_NNZ):
        gam = np.ascontiguousarray(gamma_table(schedule) if gammas is None else np.asarray(gammas, dtype=np.float64))
        return _run_part(g, x0, gam, _opt("dtype", dtype), dev)
    h = device_graph(g, _opt("dtype", dtype), dev)
    x_dev = _device_state(g, x0)
    if device_state or x_dev is not None:
        import torch

        if x_dev is None:
            x_dev = torch.from_numpy(_as_state(g, x0)).to(torch.device("cuda", dev))
        x = None
    else:
        x = _as_state(g, x0)
    gam = np.ascontiguousarray(gamma_table(schedule) if gammas is None else np.asarray(gammas, dtype=np.float64))
    iters = len(gam)
    step_inf = np.zeros(iters, dtype=np.float64)
    fallbacks = np.zeros(iters, dtype=np.int64)
    mass = np.zeros(iters, dtype=np.float64)
    energy = np.zeros(iters, dtype=np.float64) if record_trace else None
    pre_energy = np.zeros(iters, dtype=np.float64) if record_trace else None
    hist = np.zeros((iters, g.n), dtype=np.float64) if history else None
    ran = ctypes.c_int(0)
    fail = ctypes.c_int(-1)
    st = E.RunStats()
    flags = 0
    if x is None:
        import torch

        x_out = torch.empty(g.n, dtype=torch.float64, device=x_dev.device)
        torch.cuda.current_stream(x_dev.device).synchronize()  # x0 is in place before the engine's stream reads it
        flags |= E.GN_DEVICE_IO
        xin, xo = ctypes.c_void_p(x_dev.data_ptr()), ctypes.c_void_p(x_out.data_ptr())
    else:
        x_out = np.empty(g.n, dtype=np.float64)
        xin, xo = E.ptr(x), E.ptr(x_out)
    if record_trace:
        flags |= E.GN_TRACE
    if early_exit:
        flags |= E.GN_EARLY_EXIT
    if _opt("exact", exact):
        flags |= E.GN_EXACT
    rc = E.lib().gn_run(h.handle, xin, E.ptr(gam), iters, float(schedule.final_gamma), flags,
                        xo, E.ptr(step_inf), E.ptr(fallbacks), E.ptr(mass), E.ptr(energy),
                        E.ptr(pre_energy), E.ptr(hist), ctypes.byref(ran), ctypes.byref(fail),
                        ctypes.byref(st))
    if rc in _RUN_ERRORS:
        raise NormalizationError(_RUN_ERRORS[rc])
    if rc == E.GN_ERR_NONFINITE:
        raise NormalizationError(f"non-finite state at iteration {fail.value}")
    E.check(rc)
    k = ran.value
    trace = SolveTrace()
    trace.gamma = gam[:k].tolist()  # Python floats / ints, as the reference's lists hold
    trace.step_inf = step_inf[:k].tolist()
    trace.fallbacks = fallbacks[:k].tolist()
    trace.objective = mass[:k].tolist()
    if record_trace:
        trace.energy = energy[:k].tolist()
        trace.pre_energy = pre_energy[:k].tolist()
        trace.mass = list(trace.objective)
    stats = {f: getattr(st, f) for f, _ in E.RunStats._fields_}
    return RunResult(x_out, trace, stats, hist[:k] if history else None)


def run_wrgn(g, x0, schedule: GammaSchedule, record_trace: bool = False, early_exit: bool = False, *,
             dtype=None, exact=None, device=None, engine=None) -> tuple[np.ndarray, SolveTrace]:
    """Iterate the map under a gamma schedule (dynamics.py:129-180).

    Raises NormalizationError if x0 is not normalizable or a non-finite
    state appears mid-run.  When early_exit is set, stops once gamma has
    reached its final value and the step infinity-norm falls below 1e-12;
    otherwise runs the full budget.  Final entries are clamped to [0, 1].
    """
    r = run_engine(g, x0, schedule, record_trace, early_exit, dtype=dtype, exact=exact, device=device, engine=engine)
    return r.x, r.trace


def init_random(n: int, seed) -> np.ndarray:
    """Exponentially sampled start, scaled by its max and clamped to [1e-3, 1].

    Host-side on purpose: it is the seeded input of a run (numpy PCG64
    stream), identical to dynamics.py:183-191."""
    if n < 1:
        raise ValueError("n must be at least 1")
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    e = -np.log(np.maximum(u, np.finfo(np.float64).tiny))
    x = e / e.max()
    return np.clip(x, CLAMP_FLOOR, 1.0)


def init_warm(values, n: Optional[int] = None) -> np.ndarray:
    """Clamp an externally supplied fractional vector to [1e-3, 1] (dynamics.py:194-207)."""
    x = np.asarray(values, dtype=np.float64)
    if x.ndim != 1:
        raise ValueError("warm start must be a 1-d vector")
    if n is not None and len(x) != n:
        raise ValueError(f"warm start has length {len(x)}, expected {n}")
    if not np.all(np.isfinite(x)):
        raise ValueError("warm start contains non-finite entries")
    return np.clip(x, CLAMP_FLOOR, 1.0)


def energy(g, x, gamma: float) -> float:
    """Quadratic energy (1/2) y'(I + gamma A)y - v'y (dynamics.py:210-219)."""
    x = _as_state(g, x)
    out = ctypes.c_double()
    E.check(E.lib().gn_energy(any_device_graph(g, _opt("device", None)).handle, E.ptr(x), float(gamma), ctypes.byref(out)))
    return out.value


def weighted_mass(g, x) -> float:
    """Relaxed objective sum(w_i x_i) (dynamics.py:222-224)."""
    x = _as_state(g, x)
    out = ctypes.c_double()
    E.check(E.lib().gn_weighted_mass(any_device_graph(g, _opt("device", None)).handle, E.ptr(x), ctypes.byref(out)))
    return out.value


def simplex_state(g, x) -> np.ndarray:
    """Mass-normalized coordinates p_i = w_i x_i / sum_j w_j x_j (dynamics.py:227-233)."""
    x = _as_state(g, x)
    p = np.empty(g.n, dtype=np.float64)
    rc = E.lib().gn_simplex_state(any_device_graph(g, _opt("device", None)).handle, E.ptr(x), E.ptr(p))
    if rc == E.GN_ERR_ZERO_MASS:
        raise ValueError("weighted mass must be positive")
    E.check(rc)
    return p


def fitness(g, p, gamma: float) -> tuple[np.ndarray, float]:
    """Replicator fitness f_i = v_i / ((I + gamma A)(p / v))_i and its average
    (dynamics.py:236-250)."""
    p = _as_state(g, p)
    f = np.empty(g.n, dtype=np.float64)
    fbar = ctypes.c_double()
    rc = E.lib().gn_fitness(any_device_graph(g, _opt("device", None)).handle, E.ptr(p), float(gamma), E.ptr(f), ctypes.byref(fbar))
    if rc == E.GN_ERR_ZERO_DENOM:
        raise ValueError("zero denominator in fitness: state not normalizable")
    E.check(rc)
    return f, fbar.value


def round_result(g, x, *, dtype=None, device=None) -> tuple[np.ndarray, float, bool, bool]:
    """Device rounding: (0/1 mask, weight, independent, maximal)."""
    x = _as_state(g, x)
    dev = _opt("device", device)
    h = device_graph(g, dtype, dev) if dtype is not None else any_device_graph(g, dev)
    sel = np.zeros(max(g.n, 1), dtype=np.uint8)
    weight = ctypes.c_double()
    ind = ctypes.c_int()
    mx = ctypes.c_int()
    cnt = ctypes.c_int64()
    E.check(E.lib().gn_round(h.handle, E.ptr(x), 0, E.ptr(sel), ctypes.byref(weight), ctypes.byref(ind),
                             ctypes.byref(mx), ctypes.byref(cnt)))
    return sel[: g.n], weight.value, bool(ind.value), bool(mx.value)


def round_many(g, xs, *, device=None) -> list[MisSolution]:
    """round_to_mis of every row of xs ([B, n]) in one engine call (the
    rounding kernels of all states are queued back to back, one sync)."""
    flags = 0
    if type(xs).__module__.split(".")[0] == "torch" and getattr(xs, "is_cuda", False):
        import torch

        if xs.dtype != torch.float64 or xs.dim() != 2 or xs.shape[1] != g.n or not xs.is_contiguous():
            raise ValueError(f"device states must be a contiguous float64 CUDA tensor of shape (B, {g.n})")
        X, xp, flags = xs, ctypes.c_void_p(xs.data_ptr()), E.GN_DEVICE_IO
        torch.cuda.current_stream(xs.device).synchronize()
    else:
        X = np.ascontiguousarray(np.asarray(xs, dtype=np.float64))
        xp = E.ptr(X)
    if X.ndim != 2 or X.shape[1] != g.n:
        raise ValueError(f"states have shape {tuple(X.shape)}, expected (B, {g.n})")
    B = X.shape[0]
    if B == 0:
        return []
    h = any_device_graph(g, _opt("device", device))
    sel = np.zeros((B, max(g.n, 1)), dtype=np.uint8)
    weight = np.zeros(B)
    ind = np.zeros(B, dtype=np.int32)
    mx = np.zeros(B, dtype=np.int32)
    cnt = np.zeros(B, dtype=np.int64)
    E.check(E.lib().gn_round_many(h.handle, B, xp, flags, E.ptr(sel), E.ptr(weight), E.ptr(ind), E.ptr(mx),
                                  E.ptr(cnt)))
    return [MisSolution._lazy(np.flatnonzero(sel[b, : g.n].view(np.bool_)), weight=float(weight[b]),
                        independent=bool(ind[b]), maximal=bool(mx[b])) for b in range(B)]


def round_to_mis(g, x) -> MisSolution:
    """Binarize a state into a maximal independent set (dynamics.py:253-277).

    Thresholds at 0.5, repairs conflicts by dropping the lighter endpoint
    (ties keep the larger index), then completes greedily by descending
    weight (ties prefer the smaller index).
    """
    x_dev = _device_state(g, x)
    if x_dev is not None:  # the state stays in HBM (run_engine(..., device_state=True))
        import torch

        torch.cuda.current_stream(x_dev.device).synchronize()
        xp, flags = ctypes.c_void_p(x_dev.data_ptr()), E.GN_DEVICE_IO
        h = any_device_graph(g, x_dev.device.index or 0)
    else:
        x = _as_state(g, x)
        xp, flags = E.ptr(x), 0
        h = any_device_graph(g, _opt("device", None))
    members = np.empty(max(g.n, 1), dtype=np.int64)  # ids compacted on the device (no host scan of a mask)
    weight = ctypes.c_double()
    ind = ctypes.c_int()
    mx = ctypes.c_int()
    cnt = ctypes.c_int64()
    E.check(E.lib().gn_round_members(h.handle, xp, flags, E.ptr(members), ctypes.byref(weight), ctypes.byref(ind),
                                     ctypes.byref(mx), ctypes.byref(cnt)))
    return MisSolution._lazy(members[: cnt.value], weight=weight.value, independent=bool(ind.value),
                             maximal=bool(mx.value))


__all__ = [
    "CLAMP_FLOOR",
    "FALLBACK_VALUE",
    "SAFE_DIV_THRESHOLD",
    "GammaSchedule",
    "NormalizationError",
    "RunResult",
    "SolveTrace",
    "energy",
    "fitness",
    "gamma_table",
    "gn_step",
    "init_random",
    "init_warm",
    "is_normalizable",
    "round_many",
    "round_result",
    "round_to_mis",
    "run_engine",
    "run_wrgn",
    "set_engine_defaults",
    "simplex_state",
    "weighted_mass",
]
