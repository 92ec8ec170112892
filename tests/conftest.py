import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"

try:
    import hypothesis

    hypothesis.settings.register_profile("default", deadline=None, max_examples=60, print_blob=True)
    hypothesis.settings.register_profile("fast", deadline=None, max_examples=15)
    hypothesis.settings.load_profile(os.environ.get("HYPOTHESIS_PROFILE", "default"))
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")


def gpu_available() -> bool:
    try:
        from paper_2605_05330_b200 import _engine as E

        E.load_library()
        return E.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # GPU tests must fail loudly on a GPU box when the engine is broken; they
    # are only skipped when the run explicitly has no device.
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_graph(d: dict, prefix: str = ""):
    from paper_2605_05330_b200 import from_csr

    return from_csr(int(d[prefix + "n"]), d[prefix + "indptr"], d[prefix + "indices"], d[prefix + "w"])


def golden_schedule(d: dict):
    from paper_2605_05330_b200 import GammaSchedule

    g0, g1, it, lin = d["sched"]
    return GammaSchedule(float(g0), float(g1), int(it), "linear" if lin else "constant")


@pytest.fixture
def k2_uniform():
    from paper_2605_05330_b200 import build_graph

    return build_graph(2, [(0, 1)], [1.0, 1.0])


@pytest.fixture
def k2_heavy():
    from paper_2605_05330_b200 import build_graph

    return build_graph(2, [(0, 1)], [4.0, 1.0])


@pytest.fixture
def p3_uniform():
    from paper_2605_05330_b200 import build_graph

    return build_graph(3, [(0, 1), (1, 2)], [1.0, 1.0, 1.0])


@pytest.fixture
def p3_weighted():
    from paper_2605_05330_b200 import build_graph

    return build_graph(3, [(0, 1), (1, 2)], [1.0, 3.0, 1.0])
