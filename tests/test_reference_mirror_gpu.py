"""The reference's own test strategy, re-run against the
drop-in on the GPU: known answers and properties of /root/reference/pkg/tests/
test_dynamics.py, and acceptance criteria 1, 2, 3, 6, 7 of test_acceptance.py
(SPEC.md:623-633).  Written against the public API only."""

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2605_05330_b200 as P
from paper_2605_05330_b200.dynamics import FALLBACK_VALUE

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- known answers (test_dynamics.py:30-45)

def test_known_steps(k2_uniform, p3_uniform, k2_heavy):
    np.testing.assert_allclose(P.gn_step(k2_uniform, [1, 1], 1.0), [0.5, 0.5])
    np.testing.assert_array_equal(P.gn_step(p3_uniform, [1, 0, 1], 1.0), [1.0, 0.0, 1.0])
    np.testing.assert_allclose(P.gn_step(k2_heavy, [1, 1], 1.0), [2 / 3, 1 / 3])
    lone = P.build_graph(1, [], [1.0])
    assert P.gn_step(lone, [1e-12], 1.0)[0] == FALLBACK_VALUE


@st.composite
def small_graph_state(draw, n_max=9, zero_ok=True):
    n = draw(st.integers(1, n_max))
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    keep = draw(st.lists(st.booleans(), min_size=len(pairs), max_size=len(pairs)))
    w = draw(st.lists(st.floats(0.1, 10.0, allow_nan=False), min_size=n, max_size=n))
    g = P.build_graph(n, [p for p, k in zip(pairs, keep) if k], w)
    lo = 0.0 if zero_ok else 0.01
    x = np.array(draw(st.lists(st.floats(lo, 1.0, allow_nan=False), min_size=n, max_size=n)))
    return g, x


@settings(max_examples=40, deadline=None)
@given(small_graph_state(), st.floats(0.0, 3.0))
def test_step_stays_in_unit_box(gx, gamma):
    g, x = gx
    out = P.gn_step(g, x, gamma)
    assert np.all(out >= 0.0) and np.all(out <= 1.0)


@settings(max_examples=40, deadline=None)
@given(small_graph_state(), st.floats(0.01, 3.0))
def test_zero_pattern_preserved(gx, gamma):
    g, x = gx
    x = np.where(x < 0.5, 0.0, x)
    if not P.is_normalizable(g, x):
        return
    np.testing.assert_array_equal(P.gn_step(g, x, gamma) > 0, x > 0)


@settings(max_examples=40, deadline=None)
@given(small_graph_state(zero_ok=False), st.floats(0.01, 3.0), st.floats(0.001, 1000.0))
def test_scale_invariance(gx, gamma, alpha):
    g, x = gx
    np.testing.assert_allclose(P.gn_step(g, x, gamma), P.gn_step(g, alpha * x, gamma), rtol=1e-12, atol=1e-12)


def test_components_evolve_independently_bitwise():
    g = P.build_graph(5, [(0, 1), (1, 2), (3, 4)], [2.0, 1.0, 3.0, 5.0, 0.5])
    ga = P.build_graph(3, [(0, 1), (1, 2)], [2.0, 1.0, 3.0])
    gb = P.build_graph(2, [(0, 1)], [5.0, 0.5])
    x = np.array([0.9, 0.4, 0.7, 0.2, 0.8])
    xa, xb = x[:3].copy(), x[3:].copy()
    for k in range(50):
        gam = 0.9 + k * 0.01
        x, xa, xb = P.gn_step(g, x, gam), P.gn_step(ga, xa, gam), P.gn_step(gb, xb, gam)
        assert np.array_equal(x, np.concatenate([xa, xb]))


def test_maximal_independent_set_is_fixed_point():
    g = P.erdos_renyi(12, 0.4, [3, 0])
    x = np.zeros(12)
    for i in range(12):
        if not any(x[j] > 0 for j in g.neighbors(i)):
            x[i] = 1.0
    for gam in (0.5, 1.0, 1.7):
        np.testing.assert_array_equal(P.gn_step(g, x, gam), x)


# ---------------------------------------------------------------- runs (test_dynamics.py:144-202)

def test_k2_runs():
    k2 = P.build_graph(2, [(0, 1)], [1.0, 1.0])
    x, _ = P.run_wrgn(k2, np.array([0.6, 0.4]), P.GammaSchedule.constant(1.5, 300))
    np.testing.assert_allclose(x, [1.0, 0.0], atol=1e-6)
    g = P.build_graph(2, [(0, 1)], [2.0, 1.0])
    x, _ = P.run_wrgn(g, np.array([0.1, 0.9]), P.GammaSchedule.constant(1.0, 2000))
    np.testing.assert_allclose(x, [1.0, 0.0], atol=1e-6)
    gam = 0.25
    x, _ = P.run_wrgn(g, np.array([0.5, 0.5]), P.GammaSchedule.constant(gam, 5000))
    apex = (1 - gam * math.sqrt(2)) / (3 - 2 * gam * math.sqrt(2))
    assert P.simplex_state(g, x)[1] == pytest.approx(apex, abs=1e-9)


def test_early_exit_stops_short():
    g = P.erdos_renyi(20, 0.3, [11, 0])
    x, tr = P.run_wrgn(g, P.init_random(20, 42), P.GammaSchedule.constant(1.5, 100_000), early_exit=True)
    assert len(tr) < 100_000 and tr.step_inf[-1] < 1e-12


def test_descent_per_step_moving_gamma_and_monotone_constant_gamma():
    g = P.erdos_renyi(24, 0.3, [14, 0])
    _, tr = P.run_wrgn(g, P.init_random(24, 5), P.GammaSchedule.pursuit(iterations=300), record_trace=True)
    assert np.all(np.array(tr.energy) - np.array(tr.pre_energy) <= 1e-10)
    g = P.erdos_renyi(24, 0.3, [13, 0])
    _, tr = P.run_wrgn(g, P.init_random(24, 7), P.GammaSchedule.constant(1.2, 400), record_trace=True)
    e, m = np.array(tr.energy), np.array(tr.mass)
    assert np.all(np.diff(e) <= 1e-10) and np.all(np.diff(m) >= -1e-10)
    moving = np.array(tr.step_inf)[1:] > 1e-4
    assert np.all(np.diff(e)[moving] < 0) and np.all(np.diff(m)[moving] > 0)
    assert tr.total_fallbacks == 0


# ---------------------------------------------------------------- energy / fitness literals (test_dynamics.py:237-283)

def test_energy_mass_simplex_fitness_literals(k2_uniform, k2_heavy):
    assert P.energy(k2_uniform, [0, 0], 1.7) == 0.0
    assert P.energy(k2_uniform, [1, 0], 0.3) == pytest.approx(-0.5)
    assert P.weighted_mass(k2_heavy, [0.5, 0.5]) == pytest.approx(2.5)
    np.testing.assert_allclose(P.simplex_state(k2_heavy, [1, 1]), [0.8, 0.2])
    with pytest.raises(ValueError):
        P.simplex_state(k2_heavy, [0.0, 0.0])
    f, fbar = P.fitness(k2_uniform, np.array([0.75, 0.25]), 1.0)
    np.testing.assert_allclose(f, [1.0, 1.0])
    p3 = P.build_graph(3, [(0, 1), (1, 2)], [1, 1, 1])
    with pytest.raises(ValueError):
        P.fitness(p3, np.array([1.0, 0.0, 0.0]), 0.0)


@settings(max_examples=30, deadline=None)
@given(small_graph_state(zero_ok=False), st.floats(0.1, 2.5))
def test_gradient_and_replicator_identities(gx, gamma):
    g, x = gx
    y = g.v * x
    xn = P.gn_step(g, x, gamma)
    yn = g.v * xn
    grad = y + gamma * (g.adjacency() @ y) - g.v
    scale = max(np.abs(y).max(), np.abs(yn).max(), 1e-30)
    assert np.abs((yn - y) + (yn / g.v) * grad).max() / scale < 1e-10
    if gamma > 1.05:
        _, fbar = P.fitness(g, P.simplex_state(g, x), gamma)
        assert abs(P.weighted_mass(g, xn) - fbar) / abs(fbar) < 1e-12


# ---------------------------------------------------------------- rounding (test_dynamics.py:317-341)

def test_rounding_rules(k2_uniform, k2_heavy):
    assert P.round_to_mis(k2_uniform, np.array([0.99, 0.01])).members == (0,)
    assert P.round_to_mis(k2_uniform, np.array([0.6, 0.7])).members == (1,)
    assert P.round_to_mis(k2_heavy, np.array([0.9, 0.9])).members == (0,)
    assert P.round_to_mis(P.build_graph(3, [], [1, 1, 1]), np.array([0.2, 0.1, 0.3])).members == (0, 1, 2)


@settings(max_examples=40, deadline=None)
@given(small_graph_state())
def test_rounding_valid_and_maximal(gx):
    g, x = gx
    sol = P.round_to_mis(g, x)
    assert sol.independent and sol.maximal


# ---------------------------------------------------------------- acceptance (test_acceptance.py)

@pytest.fixture(scope="module")
def corpus():
    rng = np.random.default_rng(20_240_001)
    return [P.erdos_renyi(int(rng.integers(4, 65)), 0.3, [20_240_001, k]) for k in range(200)]


def test_criterion_1_lyapunov(corpus):
    bad_e = bad_m = 0
    for i, g in enumerate(corpus):
        for gam in (1.2, 1.5):
            _, tr = P.run_wrgn(g, P.init_random(g.n, [1001, i]), P.GammaSchedule.constant(gam, 500),
                               record_trace=True)
            bad_e += int(np.sum(np.array(tr.energy) - np.array(tr.pre_energy) > 1e-10))
            bad_m += int(np.sum(np.diff(tr.mass) < -1e-10))
            assert tr.total_fallbacks == 0
    assert bad_e == 0 and bad_m == 0


def test_criterion_3_binarization(corpus):
    valid = near = 0
    for i, g in enumerate(corpus):
        x, _ = P.run_wrgn(g, P.init_random(g.n, [3001, i]), P.GammaSchedule.pursuit())
        sol = P.round_to_mis(g, x)
        valid += int(sol.independent and sol.maximal)
        near += int(np.max(np.minimum(x, 1.0 - x)) <= 1e-3)
    assert valid == 200 and near >= 198


def _exhaustive_mwis(g):
    """Best-weight independent set by bitmask enumeration (n <= 16), ties by
    the lexicographically smallest member tuple -- test infrastructure."""
    n = g.n
    nbr = [0] * n
    for i in range(n):
        for j in g.neighbors(i):
            nbr[i] |= 1 << int(j)
    best, best_set = -1.0, ()
    for mask in range(1 << n):
        ok = True
        m = mask
        while m:
            i = (m & -m).bit_length() - 1
            if nbr[i] & mask:
                ok = False
                break
            m &= m - 1
        if not ok:
            continue
        members = tuple(i for i in range(n) if mask >> i & 1)
        wsum = float(np.sum(g.w[list(members)])) if members else 0.0
        if wsum > best + 1e-12 or (abs(wsum - best) <= 1e-12 and members < best_set):
            best, best_set = wsum, members
    return best_set


def test_criterion_6_attractor():
    rng = np.random.default_rng(6001)
    trials = recovered = 0
    for k in range(60):
        n = int(rng.integers(2, 13))
        g = P.erdos_renyi(n, 0.3, [6001, k])
        opt = _exhaustive_mwis(g)
        ind = np.zeros(n)
        ind[list(opt)] = 1.0
        for t in range(2):
            x0 = np.clip(ind + np.random.default_rng([6001, k, t]).uniform(-1e-3, 1e-3, n), 0.0, None)
            x, _ = P.run_wrgn(g, x0, P.GammaSchedule.constant(1.5, 400))
            trials += 1
            recovered += int(P.round_to_mis(g, x).members == opt)
    assert recovered == trials


def test_criterion_7_k2_transitions():
    for w0 in (2.0, 4.0):
        g = P.build_graph(2, [(0, 1)], [w0, 1.0])
        gb, gd = 1 / math.sqrt(w0), math.sqrt(w0)

        def limit(p, gam):
            x = np.asarray(p, float) / g.w
            x, _ = P.run_wrgn(g, x / x.max(), P.GammaSchedule.constant(gam, 200_000), early_exit=True)
            return x

        grid = np.round(np.arange(0.01, gd + 0.30, 0.05), 2)
        first_bin = None
        for gam in grid:
            x = limit([0.5, 0.5], float(gam))
            if np.max(np.minimum(x, 1 - x)) < 1e-3:
                first_bin = first_bin or float(gam)
            else:
                p1 = P.simplex_state(g, x)[1]
                apex = (1 - gam * math.sqrt(w0)) / (1 + w0 - 2 * gam * math.sqrt(w0))
                assert abs(p1 - apex) <= 1e-4 and gam <= gb + 1e-9
        assert first_bin is not None and abs(first_bin - gb) <= 0.05 + 1e-9
        for gam in grid:
            reached_light = P.round_to_mis(g, limit([0.01, 0.99], float(gam))).members == (1,)
            if gam > gd + 0.01 + 1e-9:
                assert reached_light
            if gam < gd - 1e-9:
                assert not reached_light


# ---------------------------------------------------------------- solver-style concurrency (test_solver_cli.py:54-64)

def test_concurrent_callers_are_deterministic():
    g = P.build_graph(8, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (0, 7), (1, 6)],
                      [3, 1, 4, 1, 5, 9, 2, 6])
    s = P.GammaSchedule.pursuit(iterations=150)
    x0s = [P.init_random(8, [0, i]) for i in range(6)]

    def one(x0):
        x, tr = P.run_wrgn(g, x0, s, record_trace=True)
        sol = P.round_to_mis(g, x)
        return x.tobytes(), tuple(tr.energy), sol.members, sol.weight

    serial = [one(x0) for x0 in x0s]
    with ThreadPoolExecutor(6) as pool:
        parallel = list(pool.map(one, x0s))
    assert serial == parallel


@pytest.mark.parametrize("n", [6000, 120000])
def test_concurrent_callers_on_the_loop_kernel_are_deterministic(n):
    """Threads sharing one graph large enough for the cooperative loop kernel
    (and the cooperative greedy of the rounding) -- a few CTAs, and a grid
    that fills the GPU: each call owns its stream and workspace, so results
    equal the serial ones bit for bit."""
    from paper_2605_05330_b200.graph import csr_from_edges

    rng = np.random.default_rng(11)
    us, vs = rng.integers(0, n, 8 * n), rng.integers(0, n, 8 * n)
    keep = us != vs
    indptr, indices = csr_from_edges(n, us[keep], vs[keep])
    g = P.from_csr(n, indptr, indices, 1.0 - rng.random(n))
    s = P.GammaSchedule.pursuit(iterations=200)
    x0s = [P.init_random(n, [1, i]) for i in range(8)]
    assert P.run_engine(g, x0s[0], s).stats["grid_blocks"] > (1 if n < 10000 else 100)

    def one(x0):
        x, tr = P.run_wrgn(g, x0, s)
        sol = P.round_to_mis(g, x)
        return x.tobytes(), tuple(tr.step_inf), sol.members, sol.weight

    serial = [one(x0) for x0 in x0s]
    with ThreadPoolExecutor(8) as pool:
        parallel = list(pool.map(one, x0s))
    assert serial == parallel
