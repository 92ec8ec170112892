"""CPU: the instance parser (io.py mirror: native scanner csrc/gn_io.cpp +
build_graph) against the reference parser's outcomes on a committed corpus
(tests/golden/make_io_golden.py): the same CSR and weights bit for bit, or
the same exception type and message."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2605_05330_b200 import io as gio

CASES = json.loads((Path(__file__).parent / "golden" / "mwis_corpus.json").read_text())["cases"]


@pytest.mark.parametrize("k", range(len(CASES)))
def test_parse_instance_matches_reference(k):
    case = CASES[k]
    if "error" in case:
        with pytest.raises(Exception) as info:
            gio.parse_instance(case["text"])
        assert type(info.value).__name__ == case["error"]
        assert str(info.value) == case["message"]
        return
    g = gio.parse_instance(case["text"])
    assert g.n == case["n"]
    assert np.asarray(g.indptr).tolist() == case["indptr"]
    assert np.asarray(g.indices).tolist() == case["indices"]
    assert [float(x).hex() for x in np.asarray(g.w)] == case["w"]


def test_native_scanner_takes_plain_ascii():
    plain = [c["text"] for c in CASES if c["text"].isascii() and "_" not in c["text"]
             and all(ch >= " " or ch in "\t\n\r" for ch in c["text"]) and "error" not in c]
    assert len(plain) > 20
    for t in plain:
        assert gio._scan_native(t) is not None


def test_registry_and_unknown_format():
    assert gio.INSTANCE_PARSERS["mwis"] is gio.parse_instance
    g = gio.parse_instance_as("p mwis 1 0\nn 1 2.5\n")
    assert g.n == 1 and float(g.w[0]) == 2.5
    with pytest.raises(gio.FormatError, match="no parser registered for format 'dimacs'"):
        gio.parse_instance_as("", "dimacs")


def test_large_instance():
    rng = np.random.default_rng(5)
    n, m = 20000, 100000
    u = rng.integers(1, n + 1, m)
    v = (u + rng.integers(1, n, m) - 1) % n + 1
    w = rng.uniform(0.1, 5.0, n)
    text = "p mwis %d %d\n" % (n, m) + "".join(f"n {i + 1} {float(w[i])!r}\n" for i in range(n)) + \
        "".join(f"e {a} {b}\n" for a, b in zip(u, v))
    assert gio._scan_native(text) is not None
    g = gio.parse_instance(text)
    assert g.n == n and np.array_equal(np.asarray(g.w), w)
    assert np.asarray(g.indptr)[-1] == len(g.indices) and len(g.indices) % 2 == 0
