"""The C-ABI library loads and exports every symbol include/gn_b200.h
declares; without a device every entry point fails loudly (no CPU path)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, gpu_available

HEADER = ROOT / "include" / "gn_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(gn_\w+)\s*\(", text, re.M)))


def test_header_declares_the_bound_symbols():
    from paper_2605_05330_b200 import _engine as E

    assert declared_symbols() == sorted(E.EXPORTED)


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2605_05330_b200 import _engine as E

    lib = ctypes.CDLL(str(E.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.gn_abi_version() == 1


def test_no_cpu_fallback_without_device():
    if gpu_available():
        pytest.skip("device present: covered by the gpu tests")
    import paper_2605_05330_b200 as P

    g = P.build_graph(3, [(0, 1), (1, 2)], [1.0, 3.0, 1.0])
    with pytest.raises(P.EngineUnavailable, match="no CPU fallback"):
        P.run_wrgn(g, np.array([0.5, 0.5, 0.5]), P.GammaSchedule.pursuit(iterations=10))
    with pytest.raises(P.EngineUnavailable):
        P.round_to_mis(g, np.array([1.0, 0.0, 1.0]))
    with pytest.raises(P.EngineUnavailable):
        P.gn_step(g, [1, 1, 1], 1.0)


def test_mis_solution_value_semantics():
    import copy
    import pickle

    from paper_2605_05330_b200.graph import MisSolution

    a = MisSolution(members=(1, 5, 7), weight=2.5, independent=True, maximal=False)
    b = MisSolution._lazy(np.array([1, 5, 7]), 2.5, True, False)  # as engine results are built
    assert a == b and hash(a) == hash(b) and repr(a) == repr(b)
    assert pickle.loads(pickle.dumps(b)) == a and copy.deepcopy(b) == a
    assert b.members == (1, 5, 7) and all(type(m) is int for m in b.members)
    with pytest.raises(Exception):
        b.weight = 3.0


def test_null_handles_are_argument_errors_with_messages():
    """The C ABI validates its handles before touching a device: a NULL
    graph / batch / partition is GN_ERR_ARG with a message (runs on CPU)."""
    from paper_2605_05330_b200 import _engine as E

    L = E.load_library()
    z = None
    cases = {
        "gn_run": (L.gn_run, (z,) * 16, "null graph"),
        "gn_round": (L.gn_round, (z, z, 0, z, z, z, z, z), "null graph"),
        "gn_round_members": (L.gn_round_members, (z, z, 0, z, z, z, z, z), "null graph"),
        "gn_round_many": (L.gn_round_many, (z, 1, z, 0, z, z, z, z, z), "null graph"),
        "gn_check_members": (L.gn_check_members, (z, z, z, z, z, z), "null graph"),
        "gn_spmv": (L.gn_spmv, (z, z, z), "null graph"),
        "gn_is_normalizable": (L.gn_is_normalizable, (z, z, z), "null graph"),
        "gn_weighted_mass": (L.gn_weighted_mass, (z, z, z), "null graph"),
        "gn_simplex_state": (L.gn_simplex_state, (z, z, z), "null graph"),
        "gn_graph_info": (L.gn_graph_info, (z,) * 7, "null graph"),
        "gn_batch_info": (L.gn_batch_info, (z,) * 5, "null batch"),
        "gn_part_info": (L.gn_part_info, (z,) * 4, "null partition"),
    }
    for name, (fn, args, msg) in cases.items():
        nargs = len(fn.argtypes)
        call_args = list(args[:nargs]) + [None] * (nargs - len(args))
        for k, t in enumerate(fn.argtypes):  # scalars: zero of their type
            if t in (ctypes.c_int, ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64, ctypes.c_double) and call_args[k] is None:
                call_args[k] = 0
        assert fn(*call_args) == E.GN_ERR_ARG, name
        assert msg in E.last_error(), name
