"""GPU: seeded random graphs of every layout class through every engine path
against the oracle -- the single-start loop (uint16 and int32 ids, skewed and
flat degrees, hubs, isolated vertices), the multi-start engine and the
partitioned engine: EXACT bitwise, fast mode within the fp64 contract."""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200.graph import csr_from_edges
from paper_2605_05330_b200.partition import EngineBackend, run_local_partitions

pytestmark = pytest.mark.gpu


def _graph(kind: str, n: int, seed: int):
    rng = np.random.default_rng(seed)
    if kind == "er":
        m = 6 * n
        u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    elif kind == "powerlaw":  # Zipf-like endpoints: hubs of every size, many isolated vertices
        m = 5 * n
        u = np.minimum((rng.pareto(1.1, m) * 3).astype(np.int64), n - 1)
        v = rng.integers(0, n, m)
        perm = rng.permutation(n)
        u = perm[u]
    elif kind == "stars":  # a few giant hubs on a sparse background
        k = 4
        u = np.concatenate([rng.integers(0, k, 3 * n), rng.integers(0, n, n)])
        v = np.concatenate([rng.integers(k, n, 3 * n), rng.integers(0, n, n)])
    else:
        raise ValueError(kind)
    keep = u != v
    indptr, indices = csr_from_edges(n, u[keep], v[keep])
    w = 1.0 - rng.random(n)
    return P.from_csr(n, indptr, indices, w), P.init_random(n, seed + 1)


CASES = [("er", 3000, 1), ("powerlaw", 5000, 2), ("stars", 4000, 3),
         ("er", 90000, 4), ("powerlaw", 120000, 5), ("stars", 70000, 6)]


@pytest.mark.parametrize("kind,n,seed", CASES)
def test_loop_engine_exact_and_fast(kind, n, seed):
    g, x0 = _graph(kind, n, seed)
    s = P.GammaSchedule.pursuit(iterations=120)
    ref = O.run(g, x0, s.table(), s.final_gamma, threads=O.default_threads())
    re = P.run_engine(g, x0, s, exact=True)
    np.testing.assert_array_equal(re.x, ref.x)
    np.testing.assert_array_equal(re.trace.step_inf, ref.step_inf)
    rf = P.run_engine(g, x0, s)
    np.testing.assert_allclose(rf.x, ref.x, rtol=1e-9, atol=1e-300)
    np.testing.assert_array_equal(rf.trace.fallbacks, ref.fallbacks)


@pytest.mark.parametrize("kind,n,seed", CASES[3:])
def test_multistart_and_partitioned_exact(kind, n, seed):
    g, x0 = _graph(kind, n, seed)
    s = P.GammaSchedule.pursuit(iterations=80)
    X = np.stack([P.init_random(n, [seed, b]) for b in range(3)])
    rm = P.run_multi(g, X, s, exact=True)
    for b in range(3):
        ref = O.run(g, X[b], s.table(), s.final_gamma, threads=O.default_threads())
        np.testing.assert_array_equal(rm.x[b], ref.x)
    ref = O.run(g, x0, s.table(), s.final_gamma, threads=O.default_threads())
    for halo in ("copy", "peer"):
        out = run_local_partitions(g, x0, s, 3, lambda sp: EngineBackend(sp, dtype="fp64", exact=True), halo=halo)
        np.testing.assert_array_equal(out["x"], ref.x)


@pytest.mark.parametrize("kind,n,seed", CASES)
@pytest.mark.parametrize("long_degree", ["1024", "48"])
def test_partitioned_fast_mode(kind, n, seed, long_degree, monkeypatch):
    """The partitioned engine's fast mode (rows above the long threshold as
    128-entry chunks, 16-bit delta slices where the gaps fit, equal-degree
    rows ordered by their hottest neighbours, hubs-first ghosts) on every
    graph class, 1 and 3 parts: within the fp64 contract, identical
    fallbacks, deterministic."""
    monkeypatch.setenv("GN_PART_LONG", long_degree)
    g, x0 = _graph(kind, n, seed)
    s = P.GammaSchedule.pursuit(iterations=80)
    ref = O.run(g, x0, s.table(), s.final_gamma, threads=O.default_threads())
    for parts in (1, 3):
        out = run_local_partitions(g, x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64"), halo="peer")
        np.testing.assert_allclose(out["x"], ref.x, rtol=1e-9, atol=1e-300)
        np.testing.assert_array_equal(out["fallbacks"], ref.fallbacks)
        again = run_local_partitions(g, x0, s, parts, lambda sp: EngineBackend(sp, dtype="fp64"), halo="peer")
        np.testing.assert_array_equal(again["x"], out["x"])
