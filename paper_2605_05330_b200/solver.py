"""Multi-start solve on the GPU (reference solver.py).

Same configuration, per-start RNG streams ([seed, i]), records and result
shape as graphnorm.solver.solve_instance (solver.py:100-153) and
graphnorm.io.make_result (io.py:260-280).  Where the reference fans the
starts out over a thread pool, the engine runs them together: graphs small
enough for the resident kernel (<= 4096 vertices) run all starts at once, one
CTA per start (the graph replicated B times in a batch, csrc/gn_batch.cu --
bitwise the per-start runs); larger graphs run all starts in one multi-start
engine call (the states stored start-minor, csrc/gn_multi.cu -- bitwise the
per-start EXACT runs).  Rounding and the MisSolution checks run on
the GPU per start.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .batch import GraphBatch
from .dynamics import GammaSchedule, NormalizationError, init_random, init_warm, round_many, round_to_mis, run_engine
from .graph import WeightedGraph, csr_from_edges, from_csr
from .multistart import MAX_STARTS, run_multi

FORMAT_VERSION = "0.1.0"  # the reference's result format version (io.py:32)


@dataclass
class RunConfig:
    """Knobs of a solve run; defaults follow the standard pursuit protocol (solver.py:29-54)."""

    gamma0: float = 0.9
    gamma1: float = 1.5
    iterations: int = 1000
    starts: int = 16
    seed: int = 0
    trace: bool = False
    jobs: Optional[int] = None  # accepted for compatibility; the GPU batches the starts instead

    def validate(self) -> None:
        if not self.gamma1 >= self.gamma0 > 0:
            raise ValueError("need gamma1 >= gamma0 > 0")
        mode = "constant" if self.gamma0 == self.gamma1 else "linear"
        if mode == "linear" and self.iterations < 2:
            raise ValueError("linear schedule needs at least 2 iterations")
        if self.iterations < 1:
            raise ValueError("iterations must be positive")
        if self.starts < 1:
            raise ValueError("starts must be at least 1")

    def schedule(self) -> GammaSchedule:
        mode = "constant" if self.gamma0 == self.gamma1 else "linear"
        return GammaSchedule(self.gamma0, self.gamma1, self.iterations, mode=mode)


@dataclass(frozen=True)
class StartRecord:
    """Outcome of a single trajectory (io.py:227-236)."""

    start: str
    objective: float
    valid: bool
    maximal: bool
    iterations: int
    wall_time_ms: float


@dataclass(frozen=True)
class SolveResult:
    """Aggregated outcome of a multi-start run on one instance (io.py:239-257)."""

    instance: str
    n: int
    edges: int
    starts: tuple
    best_objective: float
    schedule: dict
    reference_objective: Optional[float] = None
    gap_percent: Optional[float] = None
    version: str = FORMAT_VERSION

    @staticmethod
    def gap_of(reference: float, best: float) -> Optional[float]:
        if reference > 0:
            return (reference - best) / reference * 100.0
        return None


@dataclass
class RunStats:
    """Non-serialized run diagnostics (solver.py:57-63)."""

    fallback_events: int = 0
    aborted_starts: int = 0
    traces: dict = field(default_factory=dict)


def make_result(instance: str, g, starts: list, schedule: dict,
                reference_objective: Optional[float] = None) -> SolveResult:
    best = max((s.objective for s in starts), default=0.0)
    gap = SolveResult.gap_of(reference_objective, best) if reference_objective is not None else None
    return SolveResult(instance, g.n, len(g.indices) // 2, tuple(starts), best, schedule, reference_objective, gap)


def _replicate(g, copies: int) -> tuple[WeightedGraph, np.ndarray]:
    """The graph repeated `copies` times, block-diagonally."""
    n = g.n
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(np.asarray(g.indptr)))
    cols = np.asarray(g.indices, dtype=np.int64)
    keep = cols > rows
    r, c = rows[keep], cols[keep]
    offs = np.arange(copies + 1, dtype=np.int64) * n
    rr = (r[None, :] + offs[:-1, None]).ravel()
    cc = (c[None, :] + offs[:-1, None]).ravel()
    indptr, indices = csr_from_edges(n * copies, rr, cc)
    w = np.tile(np.asarray(g.w, dtype=np.float64), copies)
    return from_csr(n * copies, indptr, indices, w, validate=False), offs


def solve_instance(g, instance_name: str, config: RunConfig, warm_starts: Optional[list] = None,
                   reference_objective: Optional[float] = None, *, dtype=None,
                   device=None) -> tuple[SolveResult, RunStats]:
    """Run the configured starts and aggregate a SolveResult (solver.py:100-153)."""
    config.validate()
    schedule = config.schedule()
    tasks = []
    if warm_starts:
        for i, vec in enumerate(warm_starts):
            tasks.append((f"warm-{i}", init_warm(vec, g.n)))
    else:
        for i in range(config.starts):
            tasks.append((f"seed-{config.seed}.{i}", init_random(g.n, [config.seed, i])))
    stats = RunStats()
    records = []
    batched = 1 < len(tasks) and 0 < g.n <= 4096 and not config.trace
    if batched:
        packed, offs = _replicate(g, len(tasks))
        bt = GraphBatch(packed, offs, dtype=dtype, device=device)
        t0 = time.perf_counter()
        res = bt.run(np.concatenate([x for _, x in tasks]), schedule)
        elapsed = (time.perf_counter() - t0) * 1000.0
        for b, (start_id, _) in enumerate(tasks):
            if res.status[b] != 0:
                records.append(StartRecord(start_id, 0.0, False, False, 0, elapsed))
                stats.aborted_starts += 1
                continue
            sol = round_to_mis(g, res.state(b, offs))
            stats.fallback_events += int(res.fallbacks[b, : res.iters_run[b]].sum())
            records.append(StartRecord(start_id, sol.weight, sol.independent, sol.maximal, int(res.iters_run[b]),
                                       elapsed))
    elif len(tasks) > 1 and not config.trace:
        # all starts in one engine call (csrc/gn_multi.cu), up to 64 at a time
        for c0 in range(0, len(tasks), MAX_STARTS):
            chunk = tasks[c0:c0 + MAX_STARTS]
            t0 = time.perf_counter()
            res = run_multi(g, np.stack([x for _, x in chunk]), schedule, dtype=dtype, device=device)
            elapsed = (time.perf_counter() - t0) * 1000.0
            ok = [b for b in range(len(chunk)) if res.status[b] == 0]
            sols = dict(zip(ok, round_many(g, res.x[ok], device=device)))
            for b, (start_id, _) in enumerate(chunk):
                if res.status[b] != 0:
                    records.append(StartRecord(start_id, 0.0, False, False, 0, elapsed))
                    stats.aborted_starts += 1
                    continue
                sol = sols[b]
                stats.fallback_events += int(res.fallbacks[b, : res.iters_run[b]].sum())
                records.append(StartRecord(start_id, sol.weight, sol.independent, sol.maximal,
                                           int(res.iters_run[b]), elapsed))
    else:
        for start_id, x0 in tasks:
            t0 = time.perf_counter()
            try:
                r = run_engine(g, x0, schedule, record_trace=config.trace, dtype=dtype, device=device)
            except NormalizationError:
                records.append(StartRecord(start_id, 0.0, False, False, 0, (time.perf_counter() - t0) * 1000.0))
                stats.aborted_starts += 1
                continue
            elapsed = (time.perf_counter() - t0) * 1000.0
            sol = round_to_mis(g, r.x)
            stats.fallback_events += r.trace.total_fallbacks
            if config.trace:
                stats.traces[start_id] = r.trace
            records.append(StartRecord(start_id, sol.weight, sol.independent, sol.maximal, len(r.trace), elapsed))
    info = {"gamma0": schedule.gamma0, "gamma1": schedule.gamma1, "iterations": schedule.iterations,
            "mode": schedule.mode}
    return make_result(instance_name, g, records, info, reference_objective), stats
