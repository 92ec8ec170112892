"""GPU: canonical CSR from edge lists on the device (SURVEY 8f f2,
gn_csr_from_edges) against the host builder and build_graph's errors."""

import numpy as np
import pytest

import paper_2605_05330_b200 as P
from paper_2605_05330_b200.graph import GPU_INGEST_MIN_EDGES, GraphError, csr_from_edges, csr_from_edges_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m", [(1, 0), (2, 1), (1000, 5000), (70000, 300000)])
def test_same_csr_as_host(n, m):
    rng = np.random.default_rng(n + m)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    keep = u != v
    u, v = u[keep], v[keep]
    # duplicates and both orientations of the same edge
    u2 = np.concatenate([u, v[: len(v) // 3], u[: len(u) // 5]])
    v2 = np.concatenate([v, u[: len(u) // 3], v[: len(v) // 5]])
    ip_h, ix_h = csr_from_edges(n, u2, v2)
    ip_d, ix_d = csr_from_edges_gpu(n, u2, v2)
    assert np.array_equal(ip_h, ip_d) and np.array_equal(ix_h, ix_d)


def test_errors_name_the_first_offending_edge():
    u = np.array([0, 1, 2, 3, 7])
    v = np.array([1, 2, 2, 9, 7])
    with pytest.raises(GraphError, match=r"self-loop at vertex 2"):
        csr_from_edges_gpu(8, u, v)
    with pytest.raises(GraphError, match=r"edge \(3,9\) has an endpoint outside \[0,8\)"):
        csr_from_edges_gpu(8, u[3:], v[3:])
    with pytest.raises(GraphError):
        csr_from_edges_gpu(0, np.array([0]), np.array([1]))
    ip, ix = csr_from_edges_gpu(0, np.zeros(0, np.int64), np.zeros(0, np.int64))
    assert ip.tolist() == [0] and len(ix) == 0


def test_build_graph_large_edge_array_uses_the_device_builder():
    rng = np.random.default_rng(3)
    n, m = 200_000, GPU_INGEST_MIN_EDGES + 1000
    e = rng.integers(0, n, (m, 2))
    e = e[e[:, 0] != e[:, 1]]
    e = np.concatenate([e, e[:5000, ::-1]])  # reversed duplicates
    w = rng.random(n) + 0.5
    g = P.build_graph(n, e, w)
    ip, ix = csr_from_edges(n, e[:, 0], e[:, 1])
    assert np.array_equal(np.asarray(g.indptr), ip) and np.array_equal(np.asarray(g.indices), ix)
    bad = e.copy()
    bad[len(bad) // 2] = (11, 11)
    with pytest.raises(GraphError, match="self-loop at vertex 11"):
        P.build_graph(n, bad, w)
