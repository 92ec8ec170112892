"""GPU: the x0 checks of run_wrgn (dynamics.py:146-149) on rows of every
length class of the check kernel: lane rows (<= 1024), warp rows and giant
rows (> 32768 neighbours, one CTA each)."""

import numpy as np
import pytest

import gn_oracle as O

import paper_2605_05330_b200 as P
from paper_2605_05330_b200.graph import csr_from_edges

pytestmark = pytest.mark.gpu


def _star_with_partners(leaves: int):
    """Centre 0 joined to `leaves` leaves; each leaf also joined to its own
    partner.  With x = 0 on the centre and the leaves and > 0 on the partners,
    only the centre's closed neighbourhood sums to zero."""
    c = 0
    leaf = np.arange(1, leaves + 1)
    partner = leaf + leaves
    us = np.concatenate([np.full(leaves, c), leaf])
    vs = np.concatenate([leaf, partner])
    n = 2 * leaves + 1
    indptr, indices = csr_from_edges(n, us, vs)
    g = P.from_csr(n, indptr, indices, np.ones(n))
    x0 = np.zeros(n)
    x0[partner] = 0.5
    return g, x0


@pytest.mark.parametrize("leaves", [600, 5000, 40000])
def test_zero_closed_neighbourhood_found_in_any_row_class(leaves):
    g, x0 = _star_with_partners(leaves)
    s = P.GammaSchedule.pursuit(iterations=5)
    with pytest.raises(P.NormalizationError, match="zero closed neighborhood sum"):
        P.run_wrgn(g, x0, s)
    x1 = x0.copy()
    x1[leaves] = 1e-300  # one positive leaf: the centre passes, and so does every row
    x, tr = P.run_wrgn(g, x1, s)
    assert len(tr) == 5 and np.all(np.isfinite(x))
    ref = O.run(g, x1, s.table(), s.final_gamma)  # hub rows of every class, int32 layouts from 40000 leaves
    np.testing.assert_allclose(x, ref.x, rtol=1e-9, atol=0)
    xe, _ = P.run_wrgn(g, x1, s, exact=True)
    np.testing.assert_array_equal(xe, ref.x)


@pytest.mark.parametrize("leaves", [5000, 40000])
def test_nan_and_negative_entries_in_long_rows(leaves):
    g, x0 = _star_with_partners(leaves)
    x0[1 : leaves + 1] = 0.25
    s = P.GammaSchedule.pursuit(iterations=3)
    x = x0.copy()
    x[0] = -1.0  # negativity is reported before normalisability (dynamics.py:146-149)
    with pytest.raises(P.NormalizationError, match="nonnegative"):
        P.run_wrgn(g, x, s)
    x = x0.copy()
    x[leaves // 2] = np.nan
    with pytest.raises(P.NormalizationError):
        P.run_wrgn(g, x, s)


@pytest.mark.parametrize("n,p", [(0, 0.0), (1, 0.0), (300, 0.05), (20000, 0.0005)])
def test_round_members_match_the_mask(n, p):
    """round_to_mis's device-compacted member ids (gn_round_members) equal the
    mask of gn_round, and the flags and weight agree."""
    from paper_2605_05330_b200.dynamics import round_result

    rng = np.random.default_rng([7, n])
    iu, ju = np.triu_indices(n, 1) if n < 1000 else (rng.integers(0, n, 10 * n), rng.integers(0, n, 10 * n))
    keep = (rng.random(len(iu)) < p) & (iu != ju) if n < 1000 else iu != ju
    indptr, indices = csr_from_edges(n, iu[keep], ju[keep])
    g = P.from_csr(n, indptr, indices, 1.0 - rng.random(n))
    x = rng.random(n)
    sol = P.round_to_mis(g, x)
    sel, weight, ind, mx = round_result(g, x)
    assert sol.members == tuple(int(i) for i in np.flatnonzero(sel))
    assert (sol.weight, sol.independent, sol.maximal) == (weight, ind, mx)
    assert sol.independent and sol.maximal


@pytest.mark.parametrize("leaves", [600, 5000, 40000])
@pytest.mark.parametrize("pattern", ["sparse_pos", "centre_only", "one_leaf", "nan_leaf", "nan_partner", "all_zero_leaves"])
def test_x0_check_early_exit_matches_the_reference_predicate(leaves, pattern):
    """The run's x0 check stops a row at its first positive entry and tests
    NaN per vertex; on rows of every length class it must agree with the
    reference predicate all(x + A @ x > 0) (dynamics.py:122-126,148-149)."""
    import scipy.sparse as sp

    g, _ = _star_with_partners(leaves)
    n = g.n
    rng = np.random.default_rng([leaves, len(pattern)])
    x = np.zeros(n)
    if pattern == "sparse_pos":
        x[rng.choice(n, n // 3, replace=False)] = rng.random(n // 3) + 0.1
    elif pattern == "centre_only":
        x[0] = 1.0
    elif pattern == "one_leaf":
        x[leaves] = 1e-300
        x[leaves + 1 :] = 0.5
    elif pattern == "nan_leaf":
        x[:] = 0.5
        x[leaves // 2 + 1] = np.nan
    elif pattern == "nan_partner":
        x[:] = 0.5
        x[-1] = np.nan
    else:
        x[leaves + 1 :] = 0.5
    A = sp.csr_matrix((np.ones(len(g.indices)), g.indices, g.indptr), shape=(n, n))
    with np.errstate(invalid="ignore"):
        expect = bool(np.all(x + A @ x > 0))
    s = P.GammaSchedule.pursuit(iterations=2)
    if expect:
        P.run_wrgn(g, x, s)
    else:
        with pytest.raises(P.NormalizationError, match="zero closed neighborhood sum"):
            P.run_wrgn(g, x, s)
