"""GPU: several starts on one graph in one engine call (SURVEY 8f f1,
csrc/gn_multi.cu).  Every start must be bitwise its own single run in EXACT
mode (same per-row sequential sums), and the fp64 starts bitwise the oracle."""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200 import generators as G
from paper_2605_05330_b200.solver import RunConfig, solve_instance

pytestmark = pytest.mark.gpu


def _starts(n, B, seed=11):
    return np.stack([P.init_random(n, [seed, b]) for b in range(B)])


def _same_as_single(g, X, sched, dtype, early_exit=False):
    res = P.run_multi(g, X, sched, early_exit=early_exit, dtype=dtype, exact=True)
    for b in range(X.shape[0]):
        r = P.run_engine(g, X[b], sched, early_exit=early_exit, dtype=dtype, exact=True)
        k = len(r.trace)
        assert res.status[b] == 0 and res.iters_run[b] == k, (b, res.status[b], res.iters_run[b], k)
        assert np.array_equal(res.x[b], r.x), (dtype, b)
        assert np.array_equal(res.step_inf[b, :k], np.asarray(r.trace.step_inf)), (dtype, b)
        assert np.array_equal(res.fallbacks[b, :k], np.asarray(r.trace.fallbacks)), (dtype, b)
    return res


@pytest.mark.parametrize("B", [2, 5, 16])
def test_c1_fp64_bitwise_oracle(B):
    inst = G.c1_er()
    s = P.GammaSchedule.pursuit()
    X = _starts(inst.n, B)
    res = P.run_multi(inst.graph, X, s, dtype="fp64")
    for b in range(B):
        ref = O.run(inst.graph, X[b], s.table(), s.final_gamma)
        assert np.array_equal(res.x[b], ref.x)
        assert np.array_equal(res.step_inf[b], ref.step_inf)
        assert np.array_equal(res.fallbacks[b], ref.fallbacks)


@pytest.mark.parametrize("dtype,B", [("fp64", 3), ("fp64", 32), ("fp32", 4), ("fp32", 9), ("fp32_pure", 8),
                                     ("fp64", 64)])
def test_ba_hubs_equal_single_runs(dtype, B):
    # heavy-tailed degrees (hubs of degree ~1000 next to degree-5 rows)
    g = G.c3_ba(n=20_000).graph
    _same_as_single(g, _starts(g.n, B), P.GammaSchedule.pursuit(iterations=120), dtype)


def test_c2_full_size_fp64_equal_single_runs():
    inst = G.c2_assignment()
    _same_as_single(inst.graph, _starts(inst.n, 4), P.GammaSchedule.pursuit(iterations=60), "fp64")


def test_rmat_isolated_vertices_equal_single_runs():
    inst = G.c5_rmat(scale=14)
    _same_as_single(inst.graph, _starts(inst.n, 6), P.GammaSchedule.pursuit(iterations=80), "fp32")


def test_early_exit_per_start():
    # constant schedule: starts converge (and stop) at different iterations
    g = G.c1_er(n=600).graph
    s = P.GammaSchedule(1.2, 1.2, 3000, mode="constant")
    res = _same_as_single(g, _starts(g.n, 6, seed=5), s, "fp64", early_exit=True)
    assert res.iters_run.max() < 3000 and len(set(res.iters_run.tolist())) > 1


def test_failing_starts_do_not_stop_the_others():
    g = G.c1_er(n=500).graph
    s = P.GammaSchedule.pursuit(iterations=50)
    X = _starts(g.n, 4)
    X[1, 7] = -0.25              # negative entry
    X[2, :] = 0.0                # zero closed-neighbourhood sums
    res = P.run_multi(g, X, s, dtype="fp64", exact=True)
    assert res.error(1) == "state entries must be nonnegative"
    assert res.error(2) == "initial state has a zero closed neighborhood sum"
    assert res.iters_run[1] == 0 and res.iters_run[2] == 0
    for b in (0, 3):
        assert res.error(b) is None
        r = P.run_engine(g, X[b], s, dtype="fp64", exact=True)
        assert np.array_equal(res.x[b], r.x)


def test_edgeless_and_shape_errors():
    g = P.from_csr(50, np.zeros(51, np.int64), np.zeros(0, np.int32), np.linspace(0.5, 1.0, 50))
    s = P.GammaSchedule.pursuit(iterations=10)
    res = P.run_multi(g, np.full((3, 50), 0.25), s)
    assert np.array_equal(res.x, np.full((3, 50), 1.0))  # x / x = 1 for an isolated vertex
    with pytest.raises(ValueError):
        P.run_multi(g, np.zeros((3, 49)), s)
    with pytest.raises(ValueError):
        P.run_multi(g, np.zeros((65, 50)), s)


def test_solver_uses_multistart_for_large_graphs():
    inst = G.c3_ba(n=10_000)
    cfg = RunConfig(starts=5, iterations=200, seed=4)
    res, stats = solve_instance(inst.graph, "ba10k", cfg, dtype="fp64")
    s = cfg.schedule()
    for i, rec in enumerate(res.starts):
        ref = O.run(inst.graph, P.init_random(inst.n, [4, i]), s.table(), s.final_gamma)
        sel, w, ind, mx = O.round_to_mis(inst.graph, ref.x)
        assert rec.start == f"seed-4.{i}" and rec.objective == w and rec.valid and rec.maximal
        assert rec.iterations == 200
    assert stats.aborted_starts == 0


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_fast_mode_split_hubs_within_tolerance(dtype):
    # BA n=200k: the hubs exceed a warp's share and are summed in pieces
    inst = G.c3_ba()
    s = P.GammaSchedule.pursuit(iterations=200)
    X = _starts(inst.n, 4, seed=3)
    res = P.run_multi(inst.graph, X, s, dtype=dtype)
    ex = P.run_multi(inst.graph, X, s, dtype=dtype, exact=True)
    for b in range(4):
        ref = O.run(inst.graph, X[b], s.table(), s.final_gamma, threads=O.default_threads())
        tol = 1e-9 if dtype == "fp64" else 1e-3
        assert np.max(np.abs(res.x[b] - ref.x)) <= tol
        assert np.array_equal(res.fallbacks[b], ref.fallbacks)
        if dtype == "fp64":
            assert np.array_equal(ex.x[b], ref.x)  # EXACT stays bitwise
            assert np.allclose(res.step_inf[b], ref.step_inf, rtol=1e-6, atol=1e-12)
    again = P.run_multi(inst.graph, X, s, dtype=dtype)
    assert np.array_equal(again.x, res.x)  # deterministic piece order


def test_round_many_equals_round_to_mis():
    g = G.c3_ba(n=20_000).graph
    rng = np.random.default_rng(5)
    X = np.stack([rng.random(g.n) for _ in range(5)] + [np.full(g.n, 0.5), np.zeros(g.n)])
    many = P.round_many(g, X)
    for b in range(X.shape[0]):
        one = P.round_to_mis(g, X[b])
        sel, w, ind, mx = O.round_to_mis(g, X[b])
        assert many[b] == one
        assert list(many[b].members) == np.flatnonzero(sel).tolist() and many[b].weight == w
        assert many[b].independent and many[b].maximal
    assert P.round_many(g, np.zeros((0, g.n))) == []
