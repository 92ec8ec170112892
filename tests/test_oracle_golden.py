"""Pin the CPU oracle against the reference's own outputs (tests/golden).

The oracle (oracle/gn_oracle.c) is the checker for every GPU parity test, so
it must itself reproduce the reference: fp64 trajectories bitwise, fallback
counts and early-exit lengths exactly, rounding members and MIS weight
bitwise, trace energies to 1e-12.  CPU only.
"""

import numpy as np
import pytest

import gn_oracle as O
from conftest import golden_graph, golden_schedule, load_golden

RUN_CASES = [
    "c1_er1000_pursuit",
    "c1_er1000_f32inputs_trace",
    "c3like_ba3000",
    "trace_er24_pursuit300",
    "trace_er24_const",
    "early_exit_er20",
    "fallback_isolated",
    "k2_fractional",
]


@pytest.mark.parametrize("name", RUN_CASES)
def test_oracle_run_matches_reference_bitwise(name):
    d = load_golden(name)
    g = golden_graph(d)
    s = golden_schedule(d)
    trace = "energy" in d
    r = O.run(g, d["x0"], s.table(), s.final_gamma, trace=trace, early_exit=bool(d["early_exit"]),
              history="snap_k" in d, threads=2)
    assert r.status == O.OK
    assert r.iters_run == int(d["iters_run"])
    np.testing.assert_array_equal(r.x, d["x_final"])
    np.testing.assert_array_equal(r.step_inf, d["step_inf"])
    np.testing.assert_array_equal(r.fallbacks, d["fallbacks"])
    if "snap_k" in d:
        np.testing.assert_array_equal(r.history[d["snap_k"]], d["snap_x"])
    if trace:
        # the reference uses BLAS dots; ours are sequential: same value to ~1 ulp of the terms
        for key, got in (("energy", r.energy), ("pre_energy", r.pre_energy), ("mass", r.mass)):
            ref = d[key]
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.max(np.abs(ref)))


def test_oracle_gamma_table_matches_schedule():
    from paper_2605_05330_b200 import GammaSchedule

    for s in (GammaSchedule.pursuit(), GammaSchedule.pursuit(0.3, 2.1, 777), GammaSchedule.constant(1.2, 9)):
        ref = [s.gamma_at(k) for k in range(s.iterations)]
        np.testing.assert_array_equal(s.table(), ref)
        np.testing.assert_array_equal(O.schedule_table(s.gamma0, s.gamma1, s.iterations, s.mode), ref)


def test_oracle_rounding_corpus():
    d = load_golden("rounding_corpus")
    for c in range(int(d["count"])):
        g = golden_graph(d, f"{c}_")
        sel, weight, ind, mx = O.round_to_mis(g, d[f"{c}_x"])
        np.testing.assert_array_equal(np.flatnonzero(sel), d[f"{c}_members"])
        assert weight == d[f"{c}_weight"]  # bitwise: numpy pairwise restated
        assert (ind, mx) == tuple(bool(v) for v in d[f"{c}_flags"])
        out, _ = O.step(g, d[f"{c}_x"], float(d[f"{c}_gamma"]))
        np.testing.assert_array_equal(out, d[f"{c}_step"])


@pytest.mark.parametrize("name", ["c1_er1000_pursuit", "c3like_ba3000", "fallback_isolated"])
def test_oracle_final_rounding(name):
    d = load_golden(name)
    g = golden_graph(d)
    sel, weight, ind, mx = O.round_to_mis(g, d["x_final"])
    np.testing.assert_array_equal(np.flatnonzero(sel), d["members"])
    assert weight == d["mis_weight"]
    assert ind == bool(d["independent"]) and mx == bool(d["maximal"])


def test_pairwise_sum_restatement_is_numpy_bitwise():
    rng = np.random.default_rng(5)
    for n in list(range(0, 300)) + [1000, 4097, 100_000]:
        a = rng.random(n) * 10.0 ** rng.uniform(-6, 6, n)
        assert O.pairwise_sum(a) == float(a.sum())


def test_oracle_errors_match_reference_order():
    from paper_2605_05330_b200 import build_graph

    p3 = build_graph(3, [(0, 1), (1, 2)], [1.0, 1.0, 1.0])
    gam = np.full(5, 1.0)
    assert O.run(p3, np.zeros(3), gam, 1.0).status == O.ERR_NOT_NORMALIZABLE
    assert O.run(p3, np.array([0.5, -0.1, 0.5]), gam, 1.0).status == O.ERR_NEGATIVE
    r = O.run(p3, np.array([np.inf, 0.5, 0.5]), gam, 1.0)
    assert r.status == O.ERR_NONFINITE and r.fail_iter == 0


def test_oracle_threads_do_not_change_bits():
    d = load_golden("c3like_ba3000")
    g = golden_graph(d)
    s = golden_schedule(d)
    a = O.run(g, d["x0"], s.table(), s.final_gamma, threads=1)
    b = O.run(g, d["x0"], s.table(), s.final_gamma, threads=4)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.step_inf, b.step_inf)
