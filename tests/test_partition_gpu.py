"""GPU: the partitioned engine (gn_part_*) with all parts on one device
(LocalExchange) equals the unpartitioned oracle bit for bit."""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200 import generators as G
from paper_2605_05330_b200.partition import EngineBackend, run_local_partitions

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,parts", [("fp64", 3), ("fp32", 4), ("fp32_pure", 2)])
def test_partitioned_engine_bitwise(dtype, parts):
    inst = G.c5_rmat(13)
    s = P.GammaSchedule.pursuit(iterations=300)
    out = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype=dtype, exact=True))
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma, dtype=dtype)
    np.testing.assert_array_equal(out["x"], ref.x)
    np.testing.assert_array_equal(out["step_inf"], ref.step_inf)
    np.testing.assert_array_equal(out["fallbacks"], ref.fallbacks)
    np.testing.assert_allclose(out["mass"], ref.mass, rtol=1e-12)


@pytest.mark.parametrize("parts", [1, 3])
def test_partitioned_fast_mode_within_tolerance(parts):
    # R-MAT hubs (degree > 512) are split over warps: fixed fold order
    inst = G.c5_rmat(14)
    assert np.diff(inst.graph.indptr).max() > 512
    s = P.GammaSchedule.pursuit(iterations=300)
    out = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64"))
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma)
    assert np.max(np.abs(out["x"] - ref.x)) <= 1e-9
    np.testing.assert_array_equal(out["fallbacks"], ref.fallbacks)
    np.testing.assert_allclose(out["step_inf"], ref.step_inf, rtol=1e-6, atol=1e-12)
    again = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64"))
    np.testing.assert_array_equal(again["x"], out["x"])


@pytest.mark.parametrize("dtype,parts", [("fp64", 3), ("fp32", 4)])
def test_peer_halo_bitwise(dtype, parts):
    # the boundary kernel stores straight into the peers' ghost slots (gn_part_peer_*)
    inst = G.c5_rmat(13)
    s = P.GammaSchedule.pursuit(iterations=200)
    out = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype=dtype, exact=True),
                               halo="peer")
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma, dtype=dtype)
    np.testing.assert_array_equal(out["x"], ref.x)
    np.testing.assert_array_equal(out["step_inf"], ref.step_inf)
    np.testing.assert_array_equal(out["fallbacks"], ref.fallbacks)


def test_peer_halo_fast_mode_equals_copy_halo():
    inst = G.c5_rmat(14)
    s = P.GammaSchedule.pursuit(iterations=150)
    a = run_local_partitions(inst.graph, inst.x0, s, 3, lambda sp: EngineBackend(sp, dtype="fp32"), halo="peer")
    b = run_local_partitions(inst.graph, inst.x0, s, 3, lambda sp: EngineBackend(sp, dtype="fp32"), halo="copy")
    np.testing.assert_array_equal(a["x"], b["x"])
    np.testing.assert_array_equal(a["step_inf"], b["step_inf"])


@pytest.mark.parametrize("dtype,parts", [("fp64", 3), ("fp32", 2)])
def test_peer_halo_device_schedule_bitwise_over_repeated_runs(dtype, parts):
    """Every iteration of every part from one captured CUDA graph
    (gn_part_run_group), three runs on the same backends: the later runs
    reuse the first handshake (stable buffers, epoch-tagged flags) and stay
    bitwise the oracle."""
    inst = G.c5_rmat(13)
    s = P.GammaSchedule.pursuit(iterations=200)
    out = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype=dtype, exact=True),
                               halo="peer", device_schedule=True, runs=3)
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma, dtype=dtype)
    np.testing.assert_array_equal(out["x"], ref.x)
    np.testing.assert_array_equal(out["step_inf"], ref.step_inf)
    np.testing.assert_array_equal(out["fallbacks"], ref.fallbacks)


def test_one_part_device_schedule_equals_host_loop():
    """run_partition with one part (NoExchange) replays every iteration from
    one CUDA graph (gn_part_run); equal to the host-driven loop, and a second
    run reuses the captured graph."""
    from paper_2605_05330_b200 import _engine as E
    from paper_2605_05330_b200.partition import NoExchange, build_partition, run_partition

    inst = G.c5_rmat(14)
    s = P.GammaSchedule.pursuit(iterations=250)
    spec = build_partition(inst.graph, 1, 0)
    be = EngineBackend(spec, dtype="fp32")
    ex = NoExchange(be)
    a = run_partition(be, ex, spec.local_x0(inst.x0), s, device_schedule=False)
    l0 = E.launch_count()
    b = run_partition(be, ex, spec.local_x0(inst.x0), s)
    l1 = E.launch_count()
    c = run_partition(be, ex, spec.local_x0(inst.x0), s)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(b.x, c.x)
    np.testing.assert_array_equal(a.step_inf, c.step_inf)
    assert l1 - l0 >= 250  # one step launch per iteration, counted at replay
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma, dtype="fp32")
    assert np.max(np.abs(c.x - ref.x)) <= 1e-4
    be.close()


@pytest.mark.parametrize("env", [{"GN_PART_LONG": "64", "GN_PART_CHUNK": "0"}, {"GN_PART_LONG": "64"},
                                 {"GN_PART_LONG": "256", "GN_PART_CHUNK": "96"},
                                 {"GN_PART_LONG": "64", "GN_PART_DELTA": "0"}, {"GN_PART_LEX": "0"},
                                 {"GN_PART_LEX": "3"}])
@pytest.mark.parametrize("parts", [1, 3])
def test_partition_layout_options(env, parts, monkeypatch):
    """The numbering and long-row layouts (the degree threshold of the long
    rows, their chunks or warp pieces, the equal-degree ordering): fast mode
    within 1e-9 of the oracle with identical fallbacks and deterministic;
    EXACT bitwise (layouts never change its reference-order sums)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inst = G.c5_rmat(14)
    s = P.GammaSchedule.pursuit(iterations=200)
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma)
    out = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64"), halo="peer")
    np.testing.assert_allclose(out["x"], ref.x, rtol=1e-9, atol=1e-250)
    np.testing.assert_array_equal(out["fallbacks"], ref.fallbacks)
    again = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64"), halo="peer")
    np.testing.assert_array_equal(again["x"], out["x"])
    ex = run_local_partitions(inst.graph, inst.x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64", exact=True))
    np.testing.assert_array_equal(ex["x"], ref.x)


def test_run_wrgn_partitioned_route():
    """run_engine(engine="part") -- the route run_wrgn takes for large graphs
    in fast mode -- within the fp64 contract of the oracle and of the loop
    kernel, the reference's x0 errors raised in the same order with the same
    messages, the non-finite stop at the same iteration, and the options it
    cannot serve refused."""
    inst = G.c5_rmat(14)
    g, s = inst.graph, P.GammaSchedule.pursuit(iterations=150)
    ref = O.run(g, inst.x0, s.table(), s.final_gamma)
    r = P.run_engine(g, inst.x0, s, engine="part")
    np.testing.assert_allclose(r.x, ref.x, rtol=1e-9, atol=1e-250)
    np.testing.assert_array_equal(r.trace.fallbacks, ref.fallbacks)
    np.testing.assert_allclose(r.trace.step_inf, ref.step_inf, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(r.trace.objective, ref.mass, rtol=1e-12)
    again = P.run_engine(g, inst.x0, s, engine="part")  # the cached backend
    np.testing.assert_array_equal(again.x, r.x)
    bad = inst.x0.copy()
    bad[5] = -0.1
    with pytest.raises(P.NormalizationError, match="nonnegative"):
        P.run_engine(g, bad, s, engine="part")
    bad[5] = np.nan
    with pytest.raises(P.NormalizationError, match="zero closed neighborhood"):
        P.run_engine(g, bad, s, engine="part")
    iso = int(np.flatnonzero(np.diff(np.asarray(g.indptr)) == 0)[0])
    bad = inst.x0.copy()
    bad[iso] = 0.0
    with pytest.raises(P.NormalizationError, match="zero closed neighborhood"):
        P.run_engine(g, bad, s, engine="part")
    bad = inst.x0.copy()
    bad[3] = np.inf
    with pytest.raises(P.NormalizationError, match="non-finite state at iteration 0"):
        P.run_engine(g, bad, s, engine="part")
    with pytest.raises(ValueError):
        P.run_engine(g, inst.x0, s, engine="part", record_trace=True)
