"""CPU: the pieces of the drop-in that need no device.

The reference's own schedule objects drive the engine (gamma_table reads
their gamma_at, bitwise), and the engine's result records render through the
reference's write_result exactly as the reference's own do (same
FORMAT_VERSION)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _reference():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "graphnorm" / "dynamics.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return p
    pytest.skip("reference package not present (neither baseline/_ref nor /root/reference)")


@pytest.mark.parametrize("args", [(0.9, 1.5, 1000, "linear"), (0.3, 0.3, 17, "constant"), (0.5, 2.0, 2, "linear"),
                                  (1.1, 1.7, 333, "linear")])
def test_reference_schedule_drives_the_engine_table(args):
    _reference()
    from graphnorm.dynamics import GammaSchedule as RS

    import paper_2605_05330_b200 as P

    ref = RS(*args[:3], mode=args[3])
    ours = P.GammaSchedule(*args[:3], mode=args[3])
    want = np.array([ref.gamma_at(k) for k in range(ref.iterations)])
    np.testing.assert_array_equal(P.gamma_table(ref), want)
    np.testing.assert_array_equal(P.gamma_table(ours), want)
    assert ours.final_gamma == ref.final_gamma


def test_engine_records_render_as_the_reference_result():
    _reference()
    from graphnorm.io import SolveResult as RR
    from graphnorm.io import StartRecord as RSt
    from graphnorm.io import write_result

    from paper_2605_05330_b200 import solver as GS

    sched = {"gamma0": 0.9, "gamma1": 1.5, "iterations": 1000, "mode": "linear"}
    recs = [("seed-0.0", 4.0, True, True, 1000, 1.25), ("seed-0.1", 3.5, True, False, 1000, 2.5)]
    ours = GS.SolveResult("k2", 2, 1, tuple(GS.StartRecord(*r) for r in recs), 4.0, sched, 4.0, 0.0)
    ref = RR("k2", 2, 1, tuple(RSt(*r) for r in recs), 4.0, sched, 4.0, 0.0)
    assert ours.version == ref.version == "0.1.0"
    assert write_result(ours) == write_result(ref)
