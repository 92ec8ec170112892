"""Synthetic-config generators (host) -- shapes the bench and parity tests rely on."""

import numpy as np
import pytest

from paper_2605_05330_b200 import generators as G


def _canonical_ok(g):
    ip, ix = np.asarray(g.indptr), np.asarray(g.indices, dtype=np.int64)
    rows = np.repeat(np.arange(g.n), np.diff(ip))
    assert np.all(ix != rows)
    key = rows * g.n + ix
    assert np.all(np.diff(key) > 0)  # sorted rows, no duplicates
    rev = np.sort(ix * g.n + rows)
    np.testing.assert_array_equal(rev, key)  # symmetric


def test_c2_structure():
    inst = G.c2_assignment(16)
    g = inst.graph
    assert g.n == 256 and np.all(np.diff(g.indptr) == 30)
    _canonical_ok(g)
    i, j = divmod(37, 16)
    nb = set(g.neighbors(37).tolist())
    assert nb == {16 * i + t for t in range(16) if t != j} | {16 * t + j for t in range(16) if t != i}
    assert np.all(inst.graph.w > 0) and np.all(inst.graph.w <= 1)
    np.testing.assert_array_equal(inst.graph.w, np.asarray(inst.graph.w, np.float32).astype(np.float64))


def test_c1_c3_c4_c5_canonical():
    for inst in (G.c1_er(), G.c3_ba(3000), G.c4_batch(4).instance, G.c5_rmat(11)):
        _canonical_ok(inst.graph)
        assert inst.x0.shape == (inst.graph.n,)
        assert np.all(inst.x0 >= 1e-3) and np.all(inst.x0 <= 1)


def test_c3_edge_count_matches_networkx_algorithm():
    inst = G.c3_ba(2000, 5)
    assert inst.m == 5 + (2000 - 5 - 1) * 5


def test_c4_shards_compose():
    full = G.c4_batch(6)
    a, b = G.c4_batch(3, first=0), G.c4_batch(3, first=3)
    np.testing.assert_array_equal(full.instance.x0, np.concatenate([a.instance.x0, b.instance.x0]))
    np.testing.assert_array_equal(full.instance.graph.w, np.concatenate([a.instance.graph.w, b.instance.graph.w]))


@pytest.mark.gpu
def test_gpu_rmat_is_bitwise_cpu_rmat():
    for scale in (8, 12):
        cpu = G.c5_rmat(scale).graph
        ip, ix = G.rmat_csr_gpu(scale)
        np.testing.assert_array_equal(ip, cpu.indptr)
        np.testing.assert_array_equal(ix, cpu.indices)
