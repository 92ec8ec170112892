"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records, for seeded inputs, what the reference's run_wrgn / gn_step /
round_to_mis / energy / weighted_mass return.  The fixtures (small .npz files)
are committed; the GPU box never needs /root/reference.  Graph inputs are
stored in the fixtures as CSR so tests do not depend on any generator.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import graphnorm as R  # noqa: E402  (the reference)
from graphnorm.dynamics import _step  # noqa: E402

SNAP = (0, 1, 2, 3, 5, 10, 25, 50, 100, 150, 200, 250, 300, 400, 500, 700, 999)


def csr_of(g):
    return dict(n=np.int64(g.n), indptr=np.asarray(g.indptr, np.int64),
                indices=np.asarray(g.indices, np.int32), w=np.asarray(g.w, np.float64))


def ref_graph(n, us, vs, w):
    return R.build_graph(n, list(zip(np.asarray(us).tolist(), np.asarray(vs).tolist())), list(w))


def trajectory(g, x0, sched, snaps):
    """x after step k for k in snaps, by replaying run_wrgn's own _step."""
    x = np.asarray(x0, np.float64).copy()
    out = {}
    fbs = []
    for k in range(sched.iterations):
        x, nfb = _step(g, x, sched.gamma_at(k))
        fbs.append(nfb)
        if k in snaps:
            out[k] = x.copy()
    ks = np.array(sorted(out), dtype=np.int64)
    return ks, np.stack([out[k] for k in ks]), np.array(fbs, np.int64)


def run_case(name, g, x0, sched, extra=None, snaps=SNAP, trace=False, early_exit=False):
    xf, tr = R.run_wrgn(g, x0, sched, record_trace=trace, early_exit=early_exit)
    sol = R.round_to_mis(g, xf)
    d = csr_of(g)
    d.update(
        x0=np.asarray(x0, np.float64),
        gamma=np.asarray(tr.gamma, np.float64),
        x_final=xf,
        step_inf=np.asarray(tr.step_inf, np.float64),
        fallbacks=np.asarray(tr.fallbacks, np.int64),
        iters_run=np.int64(len(tr)),
        members=np.asarray(sol.members, np.int64),
        mis_weight=np.float64(sol.weight),
        independent=np.bool_(sol.independent),
        maximal=np.bool_(sol.maximal),
        sched=np.array([sched.gamma0, sched.gamma1, sched.iterations, 1 if sched.mode == "linear" else 0],
                       np.float64),
        early_exit=np.bool_(early_exit),
    )
    if trace:
        d.update(energy=np.asarray(tr.energy), pre_energy=np.asarray(tr.pre_energy), mass=np.asarray(tr.mass))
    if snaps and not early_exit:
        ks, xs, fbs = trajectory(g, x0, sched, set(s for s in snaps if s < sched.iterations))
        assert np.array_equal(fbs, d["fallbacks"])
        d.update(snap_k=ks, snap_x=xs)
    if extra:
        d.update(extra)
    np.savez_compressed(HERE / f"{name}.npz", **d)
    print(f"{name}: n={g.n} m={g.num_edges} iters={len(tr)} fallbacks={sum(tr.fallbacks)} "
          f"|MIS|={len(sol.members)} w={sol.weight!r}")


def ba_pairs(n, m, rng):
    """Small Barabasi-Albert (networkx algorithm), for the C3-like case."""
    src, dst = [0] * m, list(range(1, m + 1))
    repeated = [0] * m + list(range(1, m + 1))
    for s in range(m + 1, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(repeated[int(rng.random() * len(repeated))])
        tg = sorted(chosen)
        src += [s] * m
        dst += tg
        repeated += tg + [s] * m
    return np.array(src), np.array(dst)


def main():
    # C1: ER n=1000, d=10, w = 1 - U, x0 = init_random  (BASELINE configs[0])
    rng = np.random.default_rng(2605_0001)
    n = 1000
    iu, ju = np.triu_indices(n, k=1)
    pick = rng.random(len(iu)) < 10 / (n - 1)
    w = 1.0 - rng.random(n)
    g = ref_graph(n, iu[pick], ju[pick], w)
    x0 = R.init_random(n, [2605_0001, 1])
    run_case("c1_er1000_pursuit", g, x0, R.GammaSchedule.pursuit())

    # C1 in binary32-representable inputs: the fp64 reference against which the
    # fp32 engine is gated (mass / |dx| / final indicator)
    w32 = np.asarray(w, np.float32).astype(np.float64)
    g32 = ref_graph(n, iu[pick], ju[pick], w32)
    x032 = np.asarray(x0, np.float32).astype(np.float64)
    run_case("c1_er1000_f32inputs_trace", g32, x032, R.GammaSchedule.pursuit(), trace=True)

    # C3-like: BA n=3000 m=5, integer weights (ties), pursuit
    rng = np.random.default_rng(2605_0003)
    s, d = ba_pairs(3000, 5, rng)
    wi = rng.integers(1, 201, size=3000).astype(np.float64)
    g = ref_graph(3000, s, d, wi)
    run_case("c3like_ba3000", g, R.init_random(3000, [2605_0003, 1]), R.GammaSchedule.pursuit())

    # trace under a moving schedule (test_dynamics.py:180-187 instance)
    g = R.erdos_renyi(24, 0.3, [14, 0])
    run_case("trace_er24_pursuit300", g, R.init_random(24, 5), R.GammaSchedule.pursuit(iterations=300),
             trace=True)
    # trace at constant gamma: pre_energy reuses energy bit for bit (dynamics.py:158-161)
    g = R.erdos_renyi(24, 0.3, [13, 0])
    run_case("trace_er24_const", g, R.init_random(24, 7), R.GammaSchedule.constant(1.2, 400), trace=True)

    # early exit at constant gamma (test_dynamics.py:172-177)
    g = R.erdos_renyi(20, 0.3, [11, 0])
    run_case("early_exit_er20", g, R.init_random(20, 42), R.GammaSchedule.constant(1.5, 100_000),
             early_exit=True, snaps=())

    # fallback inside run_wrgn: an isolated vertex starting at 1e-12 (d <= 1e-9)
    g = R.build_graph(4, [(0, 1), (1, 2)], [1.0, 2.0, 3.0, 0.5])
    run_case("fallback_isolated", g, np.array([0.5, 0.7, 0.2, 1e-12]), R.GammaSchedule.pursuit(iterations=50))

    # K2 fractional regime (test_dynamics.py:155-162), long constant run
    g = R.build_graph(2, [(0, 1)], [2.0, 1.0])
    run_case("k2_fractional", g, np.array([0.5, 0.5]), R.GammaSchedule.constant(0.25, 5000), snaps=(0, 1, 4999))

    # rounding corpus: raw (non-converged) states with conflicts, ties and completion
    xs, gs, res = [], [], []
    rng = np.random.default_rng(2605_0007)
    cases = {}
    for c in range(60):
        nn = int(rng.integers(2, 120))
        pp = float(rng.uniform(0.02, 0.4))
        tie = c % 3 == 0
        gg = R.erdos_renyi(nn, pp, [2605_0007, c], 1.0, 10.0)
        if tie:  # integer weights -> many equal-weight comparisons
            iu2, ju2 = np.triu_indices(nn, k=1)
            pk = np.random.default_rng([2605_0008, c]).random(len(iu2)) < pp
            wt = np.random.default_rng([2605_0009, c]).integers(1, 4, nn).astype(float)
            gg = ref_graph(nn, iu2[pk], ju2[pk], wt)
        xx = np.random.default_rng([2605_0010, c]).random(nn)
        sol = R.round_to_mis(gg, xx)
        for key, val in csr_of(gg).items():
            cases[f"{c}_{key}"] = val
        cases[f"{c}_x"] = xx
        cases[f"{c}_members"] = np.asarray(sol.members, np.int64)
        cases[f"{c}_weight"] = np.float64(sol.weight)
        cases[f"{c}_flags"] = np.array([sol.independent, sol.maximal])
        # energy / mass / fitness literals at this state
        gam = float(rng.uniform(0.2, 2.0))
        cases[f"{c}_gamma"] = np.float64(gam)
        cases[f"{c}_energy"] = np.float64(R.energy(gg, xx, gam))
        cases[f"{c}_mass"] = np.float64(R.weighted_mass(gg, xx))
        cases[f"{c}_step"] = R.gn_step(gg, xx, gam)
        cases[f"{c}_normalizable"] = np.bool_(R.is_normalizable(gg, xx))
    cases["count"] = np.int64(60)
    np.savez_compressed(HERE / "rounding_corpus.npz", **cases)
    print("rounding_corpus: 60 cases")


if __name__ == "__main__":
    main()
