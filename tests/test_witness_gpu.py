"""GPU: the partitioned engine's zero-row certificates and settled rows
(gn_part.cu, `gn_part::witness`, `gn_part::frz`) never change a bit of any
output.

A row whose state is exactly 0 keeps y_i = 0 and x_i' = 0/d = 0 for any
d = y_i + gamma*s > 1e-9 (reference `_step`, dynamics.py:102-108); one
neighbour j with gamma*y_j > 1e-9 proves d > 1e-9 without the row's walk.
These tests run every mode with the certificates on (default) and off
(GN_PART_WITNESS=0) on inputs that have many exact zeros, compare every
output bit for bit, check EXACT runs against the oracle, and use the gather
counter (GN_PART_COUNT=1, gn_part_gathers) to show the certificates fired.

Settled rows (on with the certificates; GN_PART_SETTLE=0: off): a row with
state exactly 1 whose neighbours are all owned rows with state exactly 0 is a
fixed point together with them (it computes s = 0, x' = v/v = 1; each
neighbour's d >= gamma*v > 1e-9 for the smallest gamma still to come), so
these rows are skipped altogether.  Every test below runs three ways: both
off, certificates only, certificates + settled rows."""

import numpy as np
import pytest

import gn_oracle as O
import paper_2605_05330_b200 as P
from paper_2605_05330_b200 import generators as G
from paper_2605_05330_b200.partition import EngineBackend, NoExchange, build_partition, run_local_partitions, run_partition

pytestmark = pytest.mark.gpu


def _zeroed_x0(inst, frac, seed):
    """x0 with exact zeros on about `frac` of the vertices that keep a
    positive neighbour (every closed neighbourhood stays positive)."""
    g = inst.graph
    rng = np.random.default_rng(seed)
    x0 = np.array(inst.x0, dtype=np.float64)
    indptr, indices = np.asarray(g.indptr), np.asarray(g.indices)
    cand = rng.permutation(g.n)[: int(frac * g.n)]
    keep = np.ones(g.n, dtype=bool)  # vertices that stay positive
    for i in cand:
        nb = indices[indptr[i]:indptr[i + 1]]
        if len(nb) and keep[nb].any():
            # zero i only if no already-zeroed neighbour relies on i alone
            ok = True
            for j in nb[~keep[nb]]:
                nj = indices[indptr[j]:indptr[j + 1]]
                if keep[nj].sum() <= 1:
                    ok = False
                    break
            if ok:
                keep[i] = False
    x0[~keep] = 0.0
    assert (~keep).sum() > 0.2 * frac * g.n
    return x0


def _run(inst, x0, s, parts, monkeypatch, witness, settle=True, **kw):
    monkeypatch.setenv("GN_PART_WITNESS", "1" if witness else "0")
    monkeypatch.setenv("GN_PART_SETTLE", "1" if settle else "0")
    halo = kw.pop("halo", "copy")
    return run_local_partitions(inst.graph, x0, s, parts, lambda sp: EngineBackend(sp, **kw), halo=halo)


def _same(a, b):
    for key in ("x", "step_inf", "fallbacks"):
        np.testing.assert_array_equal(a[key], b[key], err_msg=key)
    # the objective's terms are the same, bit for bit; the walking rows of
    # partly settled slices are regrouped, which reorders the threads' sums
    np.testing.assert_allclose(a["mass"], b["mass"], rtol=1e-13, err_msg="mass")


@pytest.mark.parametrize("dtype,exact,parts,halo", [
    ("fp64", False, 1, "copy"), ("fp64", False, 3, "peer"), ("fp64", True, 2, "copy"),
    ("fp32", False, 1, "copy"), ("fp32", False, 3, "peer"), ("fp32", True, 2, "peer"),
    ("fp32_pure", True, 1, "copy")])
def test_certificates_change_no_bit(dtype, exact, parts, halo, monkeypatch):
    inst = G.c5_rmat(14)
    x0 = _zeroed_x0(inst, 0.5, seed=11)
    s = P.GammaSchedule.pursuit(iterations=200)
    on = _run(inst, x0, s, parts, monkeypatch, True, dtype=dtype, exact=exact, halo=halo)
    off = _run(inst, x0, s, parts, monkeypatch, False, dtype=dtype, exact=exact, halo=halo)
    cert = _run(inst, x0, s, parts, monkeypatch, True, settle=False, dtype=dtype, exact=exact, halo=halo)
    _same(on, off)
    _same(cert, off)
    if exact:
        ref = O.run(inst.graph, x0, s.table(), s.final_gamma, dtype=dtype)
        np.testing.assert_array_equal(on["x"], ref.x)
        np.testing.assert_array_equal(on["step_inf"], ref.step_inf)
        np.testing.assert_array_equal(on["fallbacks"], ref.fallbacks)
    else:
        ref = O.run(inst.graph, x0, s.table(), s.final_gamma)
        np.testing.assert_array_equal(on["fallbacks"], ref.fallbacks)
        if dtype == "fp64":
            np.testing.assert_allclose(on["x"], ref.x, rtol=1e-9, atol=1e-250)


@pytest.mark.parametrize("env", [{"GN_PART_LONG": "64"}, {"GN_PART_LONG": "64", "GN_PART_CHUNK": "0"},
                                 {"GN_PART_LONG": "64", "GN_PART_DELTA": "0"}])
def test_certificates_on_long_rows(env, monkeypatch):
    """Zero rows among the chunked / warp-piece long rows (threshold forced
    down so a scale-14 graph has hundreds of them): certified chunks are
    neither walked nor read by the combine."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inst = G.c5_rmat(14)
    x0 = _zeroed_x0(inst, 0.6, seed=5)
    deg = np.diff(np.asarray(inst.graph.indptr))
    assert ((deg > 64) & (x0 == 0)).sum() > 20
    s = P.GammaSchedule.pursuit(iterations=150)
    for dtype in ("fp64", "fp32"):
        on = _run(inst, x0, s, 2, monkeypatch, True, dtype=dtype, halo="peer")
        off = _run(inst, x0, s, 2, monkeypatch, False, dtype=dtype, halo="peer")
        cert = _run(inst, x0, s, 2, monkeypatch, True, settle=False, dtype=dtype, halo="peer")
        _same(on, off)
        _same(cert, off)


def test_certificates_with_fallback_rows(monkeypatch):
    """Zero rows whose neighbourhood sum is too small take the 0.5 fallback
    (d fails the 1e-9 test): no certificate may stand for them, and a row
    whose witness decays below the threshold goes back to walking."""
    inst = G.c5_rmat(13)
    g = inst.graph
    indptr, indices = np.asarray(g.indptr), np.asarray(g.indices)
    x0 = np.array(inst.x0, dtype=np.float64)
    deg = np.diff(indptr)
    # the reference rejects a zero closed neighbourhood at x0, so the
    # neighbourhoods of 200 zeroed low-degree vertices are made tiny instead:
    # with neighbours at 1e-300, gamma*s stays below 1e-9 -> 0.5 fallbacks
    rng = np.random.default_rng(3)
    centers = rng.choice(np.flatnonzero((deg >= 1) & (deg <= 4)), size=200, replace=False)
    for c in centers:
        x0[c] = 0.0
        x0[indices[indptr[c]:indptr[c + 1]]] = 1e-300
    s = P.GammaSchedule.pursuit(iterations=120)
    ref = O.run(g, x0, s.table(), s.final_gamma)
    assert ref.fallbacks.sum() > 0
    on = _run(inst, x0, s, 2, monkeypatch, True, dtype="fp64", exact=True)
    off = _run(inst, x0, s, 2, monkeypatch, False, dtype="fp64", exact=True)
    cert = _run(inst, x0, s, 2, monkeypatch, True, settle=False, dtype="fp64", exact=True)
    _same(on, off)
    _same(cert, off)
    np.testing.assert_array_equal(on["x"], ref.x)
    np.testing.assert_array_equal(on["fallbacks"], ref.fallbacks)
    fast = _run(inst, x0, s, 1, monkeypatch, True, dtype="fp64")
    np.testing.assert_array_equal(fast["fallbacks"], ref.fallbacks)
    np.testing.assert_allclose(fast["x"], ref.x, rtol=1e-9, atol=1e-250)


def test_certificates_skip_gathers_and_repeat(monkeypatch):
    """The counter shows the certificates at work (fewer value gathers than
    adjacency entries once zero rows hold a witness; fewer again with settled
    rows), and repeated runs on one backend (witnesses and flags reset at
    begin) are bitwise equal."""
    inst = G.c5_rmat(14)
    g = inst.graph
    nnz = int(np.asarray(g.indptr)[-1])
    x0 = _zeroed_x0(inst, 0.5, seed=2)
    s = P.GammaSchedule.pursuit(iterations=100)
    spec = build_partition(g, 1, 0)
    monkeypatch.setenv("GN_PART_COUNT", "1")
    outs = {}
    for mode, (wit, settle) in {"settle": ("1", "1"), "cert": ("1", "0"), "off": ("0", "0")}.items():
        monkeypatch.setenv("GN_PART_WITNESS", wit)
        monkeypatch.setenv("GN_PART_SETTLE", settle)
        be = EngineBackend(spec, dtype="fp64")
        a = run_partition(be, NoExchange(be), spec.local_x0(x0), s)
        ga = be.gathers(100)
        b = run_partition(be, NoExchange(be), spec.local_x0(x0), s)
        gb = be.gathers(100)
        np.testing.assert_array_equal(a.x, b.x)
        np.testing.assert_array_equal(ga, gb)
        outs[mode] = (a, ga)
        be.close()
    for mode in ("settle", "cert"):
        np.testing.assert_array_equal(outs[mode][0].x, outs["off"][0].x)
        np.testing.assert_array_equal(outs[mode][0].step_inf, outs["off"][0].step_inf)
        np.testing.assert_allclose(outs[mode][0].mass, outs["off"][0].mass, rtol=1e-13)
    g_on, g_cert = outs["settle"][1], outs["cert"][1]
    # iteration 0 has no witnesses yet: every row walks (the counter runs with
    # the certificates only; zero rows add their certificate test)
    assert g_cert[0] >= nnz and g_on[0] >= nnz
    assert g_cert[5:].max() < 0.8 * g_cert[0]
    # settled rows: the members whose neighbours were all zeroed stop walking,
    # settled zero rows stop looking at their witness
    assert (g_on <= g_cert).all() and g_on[10:].sum() < g_cert[10:].sum()
