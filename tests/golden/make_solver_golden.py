"""Record what the REFERENCE's own solver and CLI produce.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_solver_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
runs its `graphnorm.cli.main(["solve", ...])` (cli.py:109-125, with --trace),
`main(["bench", ...])` (cli.py:191-247) and `solver.solve_instance`
(solver.py:100-153) on small seeded instances, recording:

* the instance texts (io.write_instance), so the GPU test needs no generator;
* each result JSON with the wall-clock fields blanked, exactly as the
  reference's determinism test does (tests/test_solver_cli.py:46-64,
  `_stable_view`);
* the --trace payload (cli.py:87-99) and the exit codes;
* the bench table with its timing column blanked.

tests/test_dropin_reference_gpu.py rebinds `graphnorm.solver.run_wrgn` /
`round_to_mis` onto the engine and replays the
same commands against these fixtures.
"""

from __future__ import annotations

import contextlib
import io
import json
import re
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import graphnorm as R  # noqa: E402  (the reference)
from graphnorm.cli import main  # noqa: E402
from graphnorm.io import write_instance, write_result  # noqa: E402
from graphnorm.solver import RunConfig, solve_instance  # noqa: E402


def stable_view(result_text: str) -> str:
    """tests/test_solver_cli.py:46-51: the result JSON, wall-clock blanked."""
    obj = json.loads(result_text)
    for start in obj["starts"]:
        start["wall_time_ms"] = None
    return json.dumps(obj, indent=2)


def stable_bench(text: str) -> str:
    """cmd_bench's table with the mean wall time per start blanked."""
    return re.sub(r"\s+[0-9.]+ms", " <ms>", text)


def instances() -> dict[str, str]:
    rng = np.random.default_rng([2605, 77])
    out = {"k2": "p mwis 2 1\nn 1 4\nn 2 1\ne 1 2\n"}
    g = R.build_graph(8, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (0, 7), (1, 6)],
                      [3, 1, 4, 1, 5, 9, 2, 6])
    out["ring"] = write_instance(g)
    # an ER graph and a star-heavy graph (one row longer than a warp's share)
    n = 60
    us, vs = np.triu_indices(n, 1)
    keep = rng.random(len(us)) < 0.12
    w = (1.0 - rng.random(n)).round(6) + 0.001
    out["er60"] = write_instance(R.build_graph(n, list(zip(us[keep].tolist(), vs[keep].tolist())), w.tolist()))
    n = 700
    edges = [(0, j) for j in range(1, n)] + [(j, j + 1) for j in range(1, n - 1, 3)]
    w = rng.integers(1, 200, n).astype(float)
    out["star700"] = write_instance(R.build_graph(n, edges, w.tolist()))
    return out


def run_cli(argv) -> tuple[int, str]:
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = main(argv)
    return code, buf.getvalue()


def main_() -> None:
    texts = instances()
    rec: dict = {"instances": texts, "solve": {}, "solve_instance": {}}
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        for name, text in texts.items():
            f = d / f"{name}.mwis"
            f.write_text(text)
            out = d / f"{name}.json"
            argv = ["solve", str(f), "--starts", "4", "--iterations", "300", "--output", str(out), "--trace"]
            code, _ = run_cli(argv)
            trace = json.loads(Path(str(out) + ".trace.json").read_text())
            rec["solve"][name] = {"argv_tail": argv[2:6] + ["--trace"], "code": code,
                                  "result": stable_view(out.read_text()), "trace": trace}
        refs = d / "refs.csv"
        refs.write_text("k2,4\nring,21\n")
        bdir = d / "bench"
        bdir.mkdir()
        for name in ("k2", "ring", "er60"):
            (bdir / f"{name}.mwis").write_text(texts[name])
        code, out = run_cli(["bench", str(bdir), "--starts", "3", "--iterations", "200", "--reference", str(refs)])
        rec["bench"] = {"code": code, "table": stable_bench(out)}
    for name, seed in (("ring", 5), ("star700", 9)):
        g = R.io.parse_instance(texts[name])
        res, stats = solve_instance(g, name, RunConfig(starts=5, iterations=250, seed=seed, jobs=3))
        rec["solve_instance"][name] = {"seed": seed, "result": stable_view(write_result(res)),
                                       "fallback_events": stats.fallback_events,
                                       "aborted_starts": stats.aborted_starts}
    (HERE / "solver_cli.json").write_text(json.dumps(rec, indent=1) + "\n")
    print("wrote", HERE / "solver_cli.json")


if __name__ == "__main__":
    main_()
