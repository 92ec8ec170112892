"""GPU: the batched multi-start solver against per-start runs
and the reference solver's tests (test_solver_cli.py)."""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200 import generators as G
from paper_2605_05330_b200.solver import RunConfig, solve_instance

pytestmark = pytest.mark.gpu


def test_batched_starts_equal_oracle_per_start():
    inst = G.c1_er()
    cfg = RunConfig(starts=16, iterations=1000, seed=3)
    res, stats = solve_instance(inst.graph, "c1", cfg)
    s = cfg.schedule()
    for i, rec in enumerate(res.starts):
        x0 = P.init_random(inst.n, [3, i])
        ref = O.run(inst.graph, x0, s.table(), s.final_gamma)
        sel, w, ind, mx = O.round_to_mis(inst.graph, ref.x)
        assert rec.start == f"seed-3.{i}" and rec.objective == w and rec.valid and rec.maximal
        assert rec.iterations == 1000
    assert res.best_objective == max(r.objective for r in res.starts)
    assert stats.aborted_starts == 0


def test_reference_solver_cases(k2_heavy):
    res, stats = solve_instance(k2_heavy, "k2", RunConfig(starts=4, iterations=300))
    assert res.best_objective == 4.0 and all(s.valid and s.maximal for s in res.starts)
    assert stats.fallback_events == 0
    res, _ = solve_instance(k2_heavy, "k2", RunConfig(starts=2, iterations=300), reference_objective=4.0)
    assert res.gap_percent == pytest.approx(0.0)
    res, _ = solve_instance(k2_heavy, "k2", RunConfig(starts=16, iterations=300), warm_starts=[np.array([1.0, 0.0])])
    assert len(res.starts) == 1 and res.starts[0].start == "warm-0" and res.starts[0].objective == 4.0


def test_batched_and_sequential_paths_agree():
    g = P.build_graph(8, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (0, 7), (1, 6)],
                      [3, 1, 4, 1, 5, 9, 2, 6])
    a, _ = solve_instance(g, "ring", RunConfig(starts=6, iterations=150))
    b, st = solve_instance(g, "ring", RunConfig(starts=6, iterations=150, trace=True))  # sequential path
    assert [(s.start, s.objective, s.valid, s.maximal, s.iterations) for s in a.starts] == \
           [(s.start, s.objective, s.valid, s.maximal, s.iterations) for s in b.starts]
    assert set(st.traces) == {f"seed-0.{i}" for i in range(6)}
