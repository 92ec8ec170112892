"""MWIS instance text -> WeightedGraph (reference io.py:43-121).

``parse_instance`` reads the DIMACS-flavoured instance format::

    c optional comments
    p mwis <n> <m>
    n <vertex-id> <weight>     (one line per vertex, ids 1-based)
    e <u> <v>                  (one line per edge, ids 1-based)

with the reference's checks, in its order, and its FormatError messages.
The text is scanned by the native parser (csrc/gn_io.cpp, ``gn_mwis_parse``)
and the graph is built by ``build_graph`` (large edge lists on the device).
Texts outside the native ASCII grammar -- characters Python's str methods,
int() or float() read beyond it (non-ASCII, control characters, '_' digit
separators, integers beyond 18 digits) -- are read by ``_scan_python``, a
line-for-line restatement of the reference's rules.
"""

from __future__ import annotations

import ctypes
from typing import Callable

import numpy as np

from . import _engine as E
from .graph import GraphError, WeightedGraph, build_graph


class FormatError(ValueError):
    """Raised on malformed instance text (io.py:38-39)."""


def _scan_native(text: str):
    """(n, weights[n], edges[m, 2] 0-based) or None when the text needs the
    Python scanner.  Raises FormatError like the reference."""
    raw = text.encode("utf-8", "surrogatepass")
    out = ctypes.c_void_p()
    err = ctypes.create_string_buffer(512)
    lib = E.lib()
    rc = lib.gn_mwis_parse(raw, len(raw), ctypes.byref(out), err, len(err))
    if rc == E.GN_PARSE_FALLBACK:
        return None
    if rc == E.GN_ERR_FORMAT:
        raise FormatError(err.value.decode())
    E.check(rc)
    try:
        n, m = ctypes.c_int64(), ctypes.c_int64()
        E.check(lib.gn_mwis_info(out, ctypes.byref(n), ctypes.byref(m)))
        w = np.empty(max(n.value, 0), dtype=np.float64)
        edges = np.empty((m.value, 2), dtype=np.int64)
        E.check(lib.gn_mwis_copy(out, E.ptr(w), E.ptr(edges)))
    finally:
        lib.gn_mwis_free(out)
    return n.value, w, edges


def _scan_python(text: str):
    """The reference's line rules (io.py:49-96) for any text."""
    n = m = None
    weights: dict[int, float] = {}
    edges: list[tuple[int, int]] = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("c"):
            continue
        parts = line.split()
        kind = parts[0]
        where = f"line {lineno}: "
        try:
            if kind == "p":
                if len(parts) != 4 or parts[1] != "mwis":
                    raise FormatError(f"{where}malformed problem line {line!r}")
                if n is not None:
                    raise FormatError(f"{where}duplicate problem line")
                n, m = int(parts[2]), int(parts[3])
            elif kind in ("n", "e"):
                if n is None:
                    what = "weight" if kind == "n" else "edge"
                    raise FormatError(f"{where}{what} line before problem line")
                if len(parts) != 3:
                    what = "weight" if kind == "n" else "edge"
                    raise FormatError(f"{where}malformed {what} line {line!r}")
                if kind == "n":
                    vid = int(parts[1])
                    if not 1 <= vid <= n:
                        raise FormatError(f"{where}vertex id {vid} outside 1..{n}")
                    if vid in weights:
                        raise FormatError(f"{where}duplicate weight for vertex {vid}")
                    weights[vid] = float(parts[2])
                else:
                    u, v = int(parts[1]), int(parts[2])
                    if not (1 <= u <= n and 1 <= v <= n):
                        raise FormatError(f"{where}edge ({u},{v}) outside 1..{n}")
                    edges.append((u - 1, v - 1))
            else:
                raise FormatError(f"{where}unknown line type {kind!r}")
        except FormatError:
            raise
        except ValueError as exc:
            raise FormatError(f"{where}cannot parse number in {line!r}") from exc
    if n is None:
        raise FormatError("missing problem line")
    if len(edges) != m:
        raise FormatError(f"problem line declares {m} edges, file has {len(edges)}")
    for vid in range(1, n + 1):
        if vid not in weights:
            raise FormatError(f"missing weight for vertex {vid}")
    w = np.array([weights[vid] for vid in range(1, n + 1)], dtype=np.float64)
    e = np.array(edges, dtype=np.int64).reshape(-1, 2)
    return n, w, e


def parse_instance(text: str) -> WeightedGraph:
    """Parse a DIMACS-flavoured MWIS instance into a validated graph
    (io.py:43-102).  Vertex ids are 1-based in the file, 0-based here."""
    got = _scan_native(text)
    n, w, edges = got if got is not None else _scan_python(text)
    try:
        return build_graph(n, edges, w)
    except GraphError as exc:
        raise FormatError(str(exc)) from exc


# io.py:109-121: the format registry, with the native parser under "mwis"
INSTANCE_PARSERS: dict[str, Callable[[str], WeightedGraph]] = {"mwis": parse_instance}


def parse_instance_as(text: str, fmt: str = "mwis") -> WeightedGraph:
    """Parse an instance in a registered format (see INSTANCE_PARSERS)."""
    try:
        parser = INSTANCE_PARSERS[fmt]
    except KeyError:
        raise FormatError(f"no parser registered for format {fmt!r}; known: {sorted(INSTANCE_PARSERS)}") from None
    return parser(text)


__all__ = ["FormatError", "INSTANCE_PARSERS", "parse_instance", "parse_instance_as"]
