"""GPU parity: the CUDA engine (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle.

Gates (BASELINE.md section 4 / SURVEY.md 8c):
  fp64 EXACT   bitwise equal to the reference (every iteration's x,
               step_inf, fallbacks, final x, MIS)
  fp64 fast    per-iteration x within 1e-9 relative (warp-tree sums), same
               fallbacks, identical final indicator and MIS weight
  fp32         against the fp64 reference on fp32-representable inputs:
               per-iteration objective <= 1e-4 relative, per-iteration
               max|dx| <= 1e-4 absolute (excursions listed), identical final
               indicator and MIS weight; against the fp32 oracle: EXACT
               bitwise, fast within 1e-4 absolute.
"""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from conftest import golden_graph, golden_schedule, load_golden

pytestmark = pytest.mark.gpu

FP64_CASES = [
    "c1_er1000_pursuit",
    "c3like_ba3000",
    "trace_er24_pursuit300",
    "trace_er24_const",
    "early_exit_er20",
    "fallback_isolated",
    "k2_fractional",
]


def _run(d, **kw):
    g = golden_graph(d)
    s = golden_schedule(d)
    trace = "energy" in d
    return g, P.run_engine(g, d["x0"], s, record_trace=trace, early_exit=bool(d["early_exit"]),
                           history="snap_k" in d, **kw)


@pytest.mark.parametrize("name", FP64_CASES)
def test_fp64_exact_is_bitwise_reference(name):
    d = load_golden(name)
    g, r = _run(d, dtype="fp64", exact=True)
    assert len(r.trace) == int(d["iters_run"])
    np.testing.assert_array_equal(r.x, d["x_final"])
    np.testing.assert_array_equal(r.trace.step_inf, d["step_inf"])
    np.testing.assert_array_equal(r.trace.fallbacks, d["fallbacks"])
    np.testing.assert_array_equal(r.trace.gamma, d["gamma"])
    if "snap_k" in d:
        np.testing.assert_array_equal(r.history[d["snap_k"]], d["snap_x"])
    if "energy" in d:
        for key in ("energy", "pre_energy", "mass"):
            ref = d[key]
            np.testing.assert_allclose(getattr(r.trace, key), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("name", FP64_CASES)
def test_fp64_fast_within_1e9(name):
    d = load_golden(name)
    g, r = _run(d, dtype="fp64", exact=False)
    assert len(r.trace) == int(d["iters_run"]) or bool(d["early_exit"])
    np.testing.assert_array_equal(r.trace.fallbacks, d["fallbacks"][: len(r.trace)])
    if "snap_k" in d:
        ref = d["snap_x"]
        got = r.history[d["snap_k"]]
        np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-300)
    np.testing.assert_allclose(r.x, d["x_final"], rtol=1e-9, atol=1e-12)
    sol = P.round_to_mis(g, r.x)
    assert list(sol.members) == d["members"].tolist()
    assert sol.weight == d["mis_weight"]


def test_fp64_fast_full_history_c1():
    d = load_golden("c1_er1000_pursuit")
    g = golden_graph(d)
    s = golden_schedule(d)
    ref = O.run(g, d["x0"], s.table(), s.final_gamma, history=True, threads=4)
    r = P.run_engine(g, d["x0"], s, history=True)
    rel = np.abs(r.history - ref.history) / np.maximum(np.abs(ref.history), 1e-300)
    assert rel.max() <= 1e-9, f"max per-iteration relative deviation {rel.max():.3e}"


def test_fp32_against_fp64_reference_gates():
    d = load_golden("c1_er1000_f32inputs_trace")
    g = golden_graph(d)
    s = golden_schedule(d)
    ref = O.run(g, d["x0"], s.table(), s.final_gamma, history=True, trace=True)
    r = P.run_engine(g, d["x0"], s, record_trace=True, dtype="fp32", history=True)
    mass_rel = np.abs(np.array(r.trace.mass) - d["mass"]) / np.abs(d["mass"])
    assert mass_rel.max() <= 1e-4, mass_rel.max()
    dx = np.abs(r.history - ref.history).max(axis=1)
    excursions = [(int(k), float(dx[k])) for k in np.flatnonzero(dx > 1e-4)]
    assert not excursions, f"per-iteration |dx| > 1e-4 at {excursions[:10]}"
    np.testing.assert_array_equal(r.trace.fallbacks, d["fallbacks"])
    sol = P.round_to_mis(g, r.x)
    assert list(sol.members) == d["members"].tolist()
    assert sol.weight == d["mis_weight"]


@pytest.mark.parametrize("dtype", ["fp32", "fp32_pure"])
def test_fp32_exact_is_bitwise_same_precision_oracle(dtype):
    """EXACT mode walks every row sequentially, so the engine must equal the
    oracle carried out in the same precision bit for bit."""
    d = load_golden("c1_er1000_f32inputs_trace")
    g = golden_graph(d)
    s = golden_schedule(d)
    ref = O.run(g, d["x0"], s.table(), s.final_gamma, dtype=dtype, history=True)
    r = P.run_engine(g, d["x0"], s, dtype=dtype, exact=True, history=True)
    np.testing.assert_array_equal(r.history, ref.history)
    np.testing.assert_array_equal(r.trace.step_inf, ref.step_inf)
    np.testing.assert_array_equal(r.x, ref.x)


def test_rounding_corpus_matches_reference():
    d = load_golden("rounding_corpus")
    for c in range(int(d["count"])):
        g = golden_graph(d, f"{c}_")
        x = d[f"{c}_x"]
        sol = P.round_to_mis(g, x)
        assert list(sol.members) == d[f"{c}_members"].tolist(), f"case {c}"
        assert sol.weight == d[f"{c}_weight"], f"case {c}"
        assert (sol.independent, sol.maximal) == tuple(bool(v) for v in d[f"{c}_flags"])
        gam = float(d[f"{c}_gamma"])
        np.testing.assert_array_equal(P.gn_step(g, x, gam, exact=True), d[f"{c}_step"])
        np.testing.assert_allclose(P.gn_step(g, x, gam), d[f"{c}_step"], rtol=1e-12)
        assert P.energy(g, x, gam) == pytest.approx(float(d[f"{c}_energy"]), rel=1e-12, abs=1e-12)
        assert P.weighted_mass(g, x) == pytest.approx(float(d[f"{c}_mass"]), rel=1e-12)
        assert P.is_normalizable(g, x) == bool(d[f"{c}_normalizable"])


def test_final_rounding_of_golden_runs():
    for name in ("c1_er1000_pursuit", "c3like_ba3000", "fallback_isolated", "early_exit_er20"):
        d = load_golden(name)
        g = golden_graph(d)
        sol = P.round_to_mis(g, d["x_final"])
        assert list(sol.members) == d["members"].tolist()
        assert sol.weight == d["mis_weight"]
        assert sol.independent == bool(d["independent"]) and sol.maximal == bool(d["maximal"])


def test_errors_match_reference(p3_uniform):
    with pytest.raises(P.NormalizationError, match="zero closed neighborhood"):
        P.run_wrgn(p3_uniform, np.zeros(3), P.GammaSchedule.constant(1.0, 5))
    with pytest.raises(P.NormalizationError, match="nonnegative"):
        P.run_wrgn(p3_uniform, np.array([0.5, -0.1, 0.5]), P.GammaSchedule.constant(1.0, 5))
    with pytest.raises(P.NormalizationError, match="non-finite state at iteration 0"):
        P.run_wrgn(p3_uniform, np.array([np.inf, 0.5, 0.5]), P.GammaSchedule.constant(1.0, 5))


def test_trace_determinism_and_constant_gamma_reuse():
    d = load_golden("trace_er24_const")
    g = golden_graph(d)
    s = golden_schedule(d)
    a = P.run_engine(g, d["x0"], s, record_trace=True)
    b = P.run_engine(g, d["x0"], s, record_trace=True)
    assert a.trace.energy == b.trace.energy and a.trace.mass == b.trace.mass
    # at unchanged gamma the pre-step energy IS the previous post-step energy (dynamics.py:158-161)
    assert a.trace.pre_energy[1:] == a.trace.energy[:-1]


def test_empty_and_edgeless_graphs():
    g0 = P.build_graph(0, [], [])
    x, tr = P.run_wrgn(g0, np.zeros(0), P.GammaSchedule.pursuit(iterations=10))
    assert x.shape == (0,) and tr.step_inf == [0.0] * 10
    sol = P.round_to_mis(g0, np.zeros(0))
    assert sol.members == () and sol.weight == 0.0 and sol.independent and sol.maximal
    g = P.build_graph(3, [], [1, 2, 3])
    x, tr = P.run_wrgn(g, np.array([0.2, 0.5, 1.0]), P.GammaSchedule.pursuit(iterations=10))
    np.testing.assert_array_equal(x, [1.0, 1.0, 1.0])
    assert P.round_to_mis(g, np.array([0.2, 0.1, 0.3])).members == (0, 1, 2)
