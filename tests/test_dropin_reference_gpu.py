"""GPU: the engine dropped into the UNMODIFIED reference.

INTEGRATION.md section 1 rebinds `graphnorm.solver.run_wrgn` and
`round_to_mis` onto the engine; the reference's own solver
(`solve_instance`, solver.py:100-153, which calls them at :75 and :88), its
CLI (`cmd_solve` with --trace, cli.py:109-125; `cmd_bench` over an instance
directory, cli.py:191-247) and its thread pool then run unchanged on the
GPU.  The outputs are compared with what the reference itself produced on
the same instances (tests/golden/make_solver_golden.py): result JSON with
the wall-clock fields blanked (the reference's determinism view,
test_solver_cli.py:46-64) equal as text, exit codes equal, bench tables
equal up to the timing column, and the per-iteration --trace payload equal
(energies, masses within 1e-12 relative).

The reference package comes from baseline/_ref (pip install --target, see
DESIGN.md) or, in the build container, /root/reference/pkg/src.
"""

from __future__ import annotations

import contextlib
import io
import json
import re
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "solver_cli.json").read_text())

pytestmark = pytest.mark.gpu


def _reference():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "graphnorm" / "cli.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import graphnorm  # noqa: F401

            return p
    pytest.fail("the reference package is not importable: install it into baseline/_ref "
                "(python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of "
                "/root/reference/pkg>)")


@pytest.fixture
def rebound(monkeypatch):
    """graphnorm.solver on the engine, exactly as INTEGRATION.md section 1."""
    _reference()
    import graphnorm.solver as S

    import paper_2605_05330_b200 as gn

    monkeypatch.setattr(S, "run_wrgn", gn.run_wrgn)
    monkeypatch.setattr(S, "round_to_mis", gn.round_to_mis)
    return S


def _stable_view(result_text: str) -> str:
    obj = json.loads(result_text)
    for start in obj["starts"]:
        start["wall_time_ms"] = None
    return json.dumps(obj, indent=2)


def _cli(argv):
    from graphnorm.cli import main

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = main(argv)
    return code, buf.getvalue()


def _calls(monkeypatch):
    """Count the engine calls the reference makes through the rebinding."""
    import graphnorm.solver as S

    n = {"run": 0, "round": 0}
    run, rnd = S.run_wrgn, S.round_to_mis

    def r(*a, **k):
        n["run"] += 1
        return run(*a, **k)

    def m(*a, **k):
        n["round"] += 1
        return rnd(*a, **k)

    monkeypatch.setattr(S, "run_wrgn", r)
    monkeypatch.setattr(S, "round_to_mis", m)
    return n


@pytest.mark.parametrize("name", sorted(GOLD["solve"]))
def test_reference_cli_solve_with_trace_on_the_engine(rebound, monkeypatch, tmp_path, name):
    gold = GOLD["solve"][name]
    calls = _calls(monkeypatch)
    f = tmp_path / f"{name}.mwis"
    f.write_text(GOLD["instances"][name])
    out = tmp_path / f"{name}.json"
    code, _ = _cli(["solve", str(f)] + gold["argv_tail"][:-1] + ["--output", str(out), "--trace"])
    assert code == gold["code"]
    assert _stable_view(out.read_text()) == gold["result"]
    assert calls["run"] == 4 and calls["round"] == 4  # every start went through the engine
    trace = json.loads(Path(str(out) + ".trace.json").read_text())
    assert trace.keys() == gold["trace"].keys()
    for sid, tr in trace.items():
        g = gold["trace"][sid]
        assert tr["gamma"] == g["gamma"] and tr["fallbacks"] == g["fallbacks"]
        for key in ("energy", "pre_energy", "mass"):
            np.testing.assert_allclose(tr[key], g[key], rtol=1e-12, atol=1e-13, err_msg=f"{sid} {key}")
        np.testing.assert_allclose(tr["step_inf"], g["step_inf"], rtol=1e-9, atol=1e-12)


def test_reference_cli_bench_on_the_engine(rebound, monkeypatch, tmp_path):
    calls = _calls(monkeypatch)
    d = tmp_path / "bench"
    d.mkdir()
    for name in ("k2", "ring", "er60"):
        (d / f"{name}.mwis").write_text(GOLD["instances"][name])
    refs = tmp_path / "refs.csv"
    refs.write_text("k2,4\nring,21\n")
    code, out = _cli(["bench", str(d), "--starts", "3", "--iterations", "200", "--reference", str(refs)])
    assert code == GOLD["bench"]["code"]
    assert re.sub(r"\s+[0-9.]+ms", " <ms>", out) == GOLD["bench"]["table"]
    assert calls["run"] == 9 and calls["round"] == 9


@pytest.mark.parametrize("name", sorted(GOLD["solve_instance"]))
def test_reference_solve_instance_thread_pool_on_the_engine(rebound, name):
    """solve_instance's ThreadPoolExecutor (solver.py:124-134) calls the
    engine from 3 threads at once on one shared graph."""
    from graphnorm.io import parse_instance, write_result

    gold = GOLD["solve_instance"][name]
    g = parse_instance(GOLD["instances"][name])
    res, stats = rebound.solve_instance(g, name, rebound.RunConfig(starts=5, iterations=250, seed=gold["seed"],
                                                                   jobs=3))
    assert _stable_view(write_result(res)) == gold["result"]
    assert stats.fallback_events == gold["fallback_events"] and stats.aborted_starts == gold["aborted_starts"]


@pytest.mark.parametrize("name", sorted(GOLD["solve_instance"]))
def test_engine_solver_mirror_writes_the_reference_result(name):
    """The engine's own solve_instance (all starts in one engine call)
    rendered by the reference's write_result equals the reference run."""
    _reference()
    from graphnorm.io import parse_instance, write_result

    from paper_2605_05330_b200 import solver as GS

    gold = GOLD["solve_instance"][name]
    g = parse_instance(GOLD["instances"][name])
    res, stats = GS.solve_instance(g, name, GS.RunConfig(starts=5, iterations=250, seed=gold["seed"]))
    assert res.version == "0.1.0"
    assert _stable_view(write_result(res)) == gold["result"]
    assert stats.fallback_events == gold["fallback_events"]
