"""GPU: the resident CTA-per-graph kernel (batches, and small single graphs
routed through gn_run) against per-graph runs and the oracle."""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200 import generators as G
from paper_2605_05330_b200.batch import GraphBatch

pytestmark = pytest.mark.gpu


def _corpus(count=24, seed=77):
    rng = np.random.default_rng(seed)
    return [P.erdos_renyi(int(rng.integers(2, 300)), float(rng.uniform(0.01, 0.3)), [seed, k])
            for k in range(count)]


@pytest.mark.parametrize("dtype", ["fp64", "fp32", "fp32_pure"])
def test_batch_equals_per_graph_oracle_bitwise(dtype):
    graphs = _corpus()
    s = P.GammaSchedule.pursuit(iterations=300)
    x0s = [P.init_random(g.n, [5, k]) for k, g in enumerate(graphs)]
    bt = GraphBatch.from_graphs(graphs, dtype=dtype)
    res = bt.run(np.concatenate(x0s), s)
    assert (res.status == 0).all()
    for b, (g, x0) in enumerate(zip(graphs, x0s)):
        ref = O.run(g, x0, s.table(), s.final_gamma, dtype=dtype)
        np.testing.assert_array_equal(res.state(b, bt.offsets), ref.x)
        np.testing.assert_array_equal(res.step_inf[b], ref.step_inf)
        np.testing.assert_array_equal(res.fallbacks[b], ref.fallbacks)
        np.testing.assert_allclose(res.objective[b], ref.mass, rtol=1e-12)


def test_batch_per_graph_early_exit_and_errors():
    graphs = _corpus(6, seed=9)
    s = P.GammaSchedule.constant(1.5, 20000)
    x0s = [P.init_random(g.n, [1, k]) for k, g in enumerate(graphs)]
    x0s[2] = np.zeros(graphs[2].n)            # not normalizable
    x0s[4] = x0s[4].copy()
    x0s[4][0] = -0.1                          # negative
    bt = GraphBatch.from_graphs(graphs)
    res = bt.run(np.concatenate(x0s), s, early_exit=True)
    assert res.status[2] == 4 and res.status[4] == 3
    for b in (0, 1, 3, 5):
        ref = O.run(graphs[b], x0s[b], s.table(), s.final_gamma, early_exit=True)
        assert res.status[b] == 0 and res.iters_run[b] == ref.iters_run
        np.testing.assert_array_equal(res.state(b, bt.offsets), ref.x)


def test_single_small_graph_routes_to_resident_kernel():
    inst = G.c1_er()
    s = P.GammaSchedule.pursuit()
    r = P.run_engine(inst.graph, inst.x0, s, record_trace=True, history=True)
    ref = O.run(inst.graph, inst.x0, s.table(), s.final_gamma, trace=True, history=True)
    assert r.stats["grid_blocks"] == 1  # one CTA: the resident kernel
    np.testing.assert_array_equal(r.history, ref.history)
    np.testing.assert_allclose(r.trace.energy, ref.energy, rtol=1e-12)
    np.testing.assert_allclose(r.trace.pre_energy, ref.pre_energy, rtol=1e-12)


def test_c4_shard_batch_vs_packed_streaming():
    b = G.c4_batch(graphs=32)
    inst = b.instance
    s = P.GammaSchedule.pursuit()
    bt = GraphBatch(inst.graph, b.offsets, dtype="fp32")
    res = bt.run(inst.x0, s)
    packed = P.run_engine(inst.graph, inst.x0, s, dtype="fp32", exact=True)
    # the packed streaming run (EXACT: sequential sums) is the same computation
    np.testing.assert_array_equal(res.x, packed.x)
    np.testing.assert_array_equal(res.step_inf.max(axis=0), np.array(packed.trace.step_inf))
    np.testing.assert_array_equal(res.fallbacks.sum(axis=0), np.array(packed.trace.fallbacks))


def test_batch_x0_checks_match_the_reference_predicate():
    """Per-graph x0 checks (early exit at the first positive entry, NaN per
    vertex) against all(x + A @ x > 0) on sparse-zero, NaN and all-zero starts."""
    import scipy.sparse as sp

    graphs = _corpus(40, seed=31)
    rng = np.random.default_rng(5)
    x0s = []
    for k, g in enumerate(graphs):
        x = np.zeros(g.n)
        kind = k % 4
        if kind == 0:
            x = P.init_random(g.n, [3, k])
        elif kind == 1:  # mostly zero: some rows have no positive closed entry
            pick = rng.random(g.n) < 0.15
            x[pick] = rng.random(int(pick.sum())) + 0.01
        elif kind == 2:
            x = P.init_random(g.n, [3, k])
            x[int(rng.integers(g.n))] = np.nan
        x0s.append(x)
    bt = GraphBatch.from_graphs(graphs)
    res = bt.run(np.concatenate(x0s), P.GammaSchedule.pursuit(iterations=5))
    for b, (g, x) in enumerate(zip(graphs, x0s)):
        A = sp.csr_matrix((np.ones(len(g.indices)), g.indices, g.indptr), shape=(g.n, g.n))
        with np.errstate(invalid="ignore"):
            ok = bool(np.all(x + A @ x > 0))
        assert res.status[b] == (0 if ok else 4), (b, k % 4)
