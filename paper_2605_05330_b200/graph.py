"""Weighted-graph container and MIS predicates (drop-in for graphnorm.graph).

Same names, fields, argument meaning and exceptions as the reference
(/root/reference/pkg/src/graphnorm/graph.py).  The CSR arrays live on the host
for callers that inspect them, and are uploaded once per dtype to the GPU
engine, which does all the arithmetic: the independence / maximality / weight
predicates run on the device (gn_check_members).  ``build_graph`` is
vectorised numpy instead of the reference's per-edge Python loops
(graph.py:98-123) and produces the identical canonical CSR.
"""

from __future__ import annotations

import ctypes

import threading
from collections import OrderedDict
import dataclasses
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _engine as E


class GraphError(ValueError):
    """Raised for invalid graph construction or out-of-range vertex indices."""


_DTYPES = {"fp64": E.GN_F64, "float64": E.GN_F64, "f64": E.GN_F64,
           "fp32": E.GN_F32, "float32": E.GN_F32, "f32": E.GN_F32, "mixed": E.GN_F32,
           "fp32_pure": E.GN_F32_PURE, "f32_pure": E.GN_F32_PURE}


def dtype_code(dtype) -> int:
    if dtype is None:
        return E.GN_F64
    if isinstance(dtype, int):
        return dtype
    if dtype is np.float64:
        return E.GN_F64
    if dtype is np.float32:
        return E.GN_F32
    try:
        return _DTYPES[str(dtype).lower()]
    except KeyError:
        raise ValueError(f"unsupported engine dtype {dtype!r}") from None


class WeightedGraph:
    """Undirected simple graph with positive vertex weights (graph.py:22-75).

    Attributes:
        n: vertex count.
        indptr, indices: CSR neighbor lists, each list sorted ascending.
        w: float64 weight per vertex, strictly positive and finite.
        v: cached sqrt(w).

    Immutable after construction (arrays are write-protected) and safe for
    unrestricted concurrent reads; device copies are created lazily, once per
    engine dtype, and shared by every caller.
    """

    __slots__ = ("n", "indptr", "indices", "w", "v", "_handles", "_lock", "__weakref__")

    def __init__(self, n: int, indptr: np.ndarray, indices: np.ndarray, w: np.ndarray):
        self.n = int(n)
        self.indptr = indptr
        self.indices = indices
        self.w = w
        self.v = np.sqrt(w)
        for a in (self.indptr, self.indices, self.w, self.v):
            a.setflags(write=False)
        self._handles: dict = {}
        self._lock = threading.Lock()

    @property
    def num_edges(self) -> int:
        return len(self.indices) // 2

    def neighbors(self, i: int) -> np.ndarray:
        return self.indices[self.indptr[i] : self.indptr[i + 1]]

    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def adjacency(self) -> "DeviceAdjacency":
        """0/1 adjacency operator; ``A @ y`` runs on the GPU (fp64, scipy order)."""
        return DeviceAdjacency(self)

    def edges(self) -> Iterable[tuple[int, int]]:
        """Edges as (u, v) with u < v, in ascending order."""
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.indptr))
        keep = self.indices > rows
        for u, v in zip(rows[keep].tolist(), np.asarray(self.indices)[keep].tolist()):
            yield u, v

    def has_edge(self, u: int, v: int) -> bool:
        nb = self.neighbors(u)
        j = np.searchsorted(nb, v)
        return bool(j < len(nb) and nb[j] == v)

    def device_graph(self, dtype=None, device: int = 0) -> E.GraphHandle:
        """The engine handle for this graph (uploaded on first use)."""
        key = (dtype_code(dtype), int(device))
        h = self._handles.get(key)
        if h is None:
            with self._lock:
                h = self._handles.get(key)
                if h is None:
                    h = E.GraphHandle(self.n, self.indptr, self.indices, self.w, key[0], key[1])
                    self._handles[key] = h
        return h

    def release_device(self) -> None:
        with self._lock:
            for h in self._handles.values():
                h.close()
            self._handles.clear()

    def __repr__(self) -> str:
        return f"WeightedGraph(n={self.n}, m={self.num_edges})"


# Foreign graphs (e.g. the reference's own graphnorm.WeightedGraph, which has
# no __weakref__ slot) get their device copy from a bounded cache that keeps
# the graph object alive while its handle is cached, so ids cannot be reused.
_FOREIGN_CACHE: "OrderedDict[tuple, tuple[object, E.GraphHandle]]" = OrderedDict()
_FOREIGN_LOCK = threading.Lock()
_FOREIGN_MAX = 16


def device_graph(g, dtype=None, device: int = 0) -> E.GraphHandle:
    if isinstance(g, WeightedGraph):
        return g.device_graph(dtype, device)
    key = (id(g), dtype_code(dtype), int(device))
    with _FOREIGN_LOCK:
        hit = _FOREIGN_CACHE.get(key)
        if hit is not None and hit[0] is g:
            _FOREIGN_CACHE.move_to_end(key)
            return hit[1]
        h = E.GraphHandle(g.n, g.indptr, g.indices, g.w, key[1], key[2])
        _FOREIGN_CACHE[key] = (g, h)
        while len(_FOREIGN_CACHE) > _FOREIGN_MAX:
            _FOREIGN_CACHE.popitem(last=False)
        return h


def any_device_graph(g, device: int = 0) -> E.GraphHandle:
    """An existing handle of g on `device` whatever its dtype (the rounding,
    checks and fp64 helpers only use the dtype-independent original CSR and
    fp64 weights), else a new fp64 one."""
    if isinstance(g, WeightedGraph):
        for (dt, dev), h in list(g._handles.items()):
            if dev == device:
                return h
        return g.device_graph(None, device)
    with _FOREIGN_LOCK:
        for (gid, dt, dev), (obj, h) in list(_FOREIGN_CACHE.items()):
            if obj is g and dev == device:
                return h
    return device_graph(g, None, device)


class DeviceAdjacency:
    """Stand-in for the reference's scipy adjacency (graph.py:55-57): only the
    mat-vec the dynamics and tests use, executed by the engine."""

    def __init__(self, g):
        self._g = g
        self.shape = (g.n, g.n)
        self.nnz = len(g.indices)

    def __matmul__(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        if y.shape != (self._g.n,):
            raise ValueError(f"dimension mismatch: {y.shape} vs {self.shape}")
        out = np.empty(self._g.n, dtype=np.float64)
        h = any_device_graph(self._g)
        E.check(E.lib().gn_spmv(h.handle, E.ptr(y), E.ptr(out)))
        return out

    def dot(self, y):
        return self @ y


# edge lists at least this long are turned into CSR on the GPU (gn_csr_from_edges)
GPU_INGEST_MIN_EDGES = 1 << 20


def _have_device() -> bool:
    try:
        return E.device_count() > 0
    except E.EngineUnavailable:
        return False


def csr_from_edges_gpu(n: int, us, vs, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Canonical CSR built on the device (csrc/gn_gen.cu): sort, deduplicate,
    symmetrise, sort -- identical to csr_from_edges.  Raises GraphError for
    the first edge (input order) outside [0, n) or a self-loop."""
    us = np.ascontiguousarray(us, dtype=np.int64)
    vs = np.ascontiguousarray(vs, dtype=np.int64)
    bad = ctypes.c_int64(-1)
    nnz = ctypes.c_int64()
    pp, pc = ctypes.c_void_p(), ctypes.c_void_p()
    rc = E.lib().gn_csr_from_edges(n, len(us), E.ptr(us), E.ptr(vs), device, ctypes.byref(bad), ctypes.byref(nnz),
                                   ctypes.byref(pp), ctypes.byref(pc))
    if rc == E.GN_ERR_ARG and bad.value >= 0:
        u, v = int(us[bad.value]), int(vs[bad.value])
        if not (0 <= u < n and 0 <= v < n):
            raise GraphError(f"edge ({u},{v}) has an endpoint outside [0,{n})")
        raise GraphError(f"self-loop at vertex {u}")
    E.check(rc)
    try:
        indptr = np.ctypeslib.as_array(ctypes.cast(pp, ctypes.POINTER(ctypes.c_int64)), shape=(n + 1,)).copy()
        indices = (np.ctypeslib.as_array(ctypes.cast(pc, ctypes.POINTER(ctypes.c_int32)), shape=(nnz.value,))
                   .astype(np.int64) if nnz.value else np.zeros(0, np.int64))
    finally:
        E.lib().gn_free_host(pp)
        E.lib().gn_free_host(pc)
    return indptr, indices


def csr_from_edges(n: int, us: np.ndarray, vs: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Canonical symmetric CSR (sorted rows, no duplicates) from edge endpoints.

    Endpoints must already be validated (in range, no self-loops)."""
    us = np.asarray(us, dtype=np.int64)
    vs = np.asarray(vs, dtype=np.int64)
    lo = np.minimum(us, vs)
    hi = np.maximum(us, vs)
    key = np.unique(lo * np.int64(max(n, 1)) + hi)
    lo = key // max(n, 1)
    hi = key % max(n, 1)
    rows = np.concatenate([lo, hi])
    cols = np.concatenate([hi, lo])
    order = np.lexsort((cols, rows))
    rows = rows[order]
    cols = cols[order]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    return indptr, np.ascontiguousarray(cols, dtype=np.int64)


def build_graph(
    n: int,
    edges: Sequence[tuple[int, int]],
    weights: Sequence[float],
) -> WeightedGraph:
    """Validate and build a WeightedGraph (graph.py:78-124).

    Duplicate edges and both orientations of the same edge are merged.
    Raises GraphError on self-loops, out-of-range indices, or weights
    that are missing, non-positive, or non-finite.
    """
    if n < 0:
        raise GraphError(f"vertex count must be nonnegative, got {n}")
    w = np.asarray(weights, dtype=np.float64)
    if w.shape != (n,):
        raise GraphError(f"expected {n} weights, got {w.shape}")
    if not np.all(np.isfinite(w)) or np.any(w <= 0.0):
        bad = int(np.argmin(np.where(np.isfinite(w), w, -np.inf)))
        raise GraphError(f"weight of vertex {bad} must be positive and finite, got {w[bad]}")
    if isinstance(edges, np.ndarray):
        e = edges.astype(np.int64).reshape(-1, 2)
        if len(e) >= GPU_INGEST_MIN_EDGES and _have_device():
            # large edge lists: validation, dedup, symmetrisation and CSR on the device
            indptr, indices = csr_from_edges_gpu(n, e[:, 0], e[:, 1])
            return WeightedGraph(n, indptr, indices, w)
    else:
        lst = [(int(u), int(v)) for u, v in edges]
        e = np.array(lst, dtype=np.int64).reshape(-1, 2) if lst else np.zeros((0, 2), np.int64)
    us, vs = e[:, 0], e[:, 1]
    out = ~((us >= 0) & (us < n) & (vs >= 0) & (vs < n))
    loop = us == vs
    badmask = out | loop
    if badmask.any():
        k = int(np.argmax(badmask))
        u, v = int(us[k]), int(vs[k])
        if out[k]:
            raise GraphError(f"edge ({u},{v}) has an endpoint outside [0,{n})")
        raise GraphError(f"self-loop at vertex {u}")
    indptr, indices = csr_from_edges(n, us, vs)
    return WeightedGraph(n, indptr, indices, w)


def from_csr(n: int, indptr, indices, w, validate: bool = True) -> WeightedGraph:
    """Wrap an existing canonical CSR (sorted, symmetric, deduplicated rows)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    if validate:
        if indptr.shape != (n + 1,) or indptr[0] != 0 or indptr[-1] != len(indices):
            raise GraphError("malformed indptr")
        if w.shape != (n,) or not np.all(np.isfinite(w)) or np.any(w <= 0.0):
            raise GraphError("weights must be positive and finite")
        if len(indices) and (indices.min() < 0 or indices.max() >= n):
            raise GraphError("column index outside [0,n)")
    return WeightedGraph(n, indptr, indices, w)


def _check_members(g, members: Iterable[int]) -> np.ndarray:
    idx = np.fromiter((int(i) for i in members), dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= g.n):
        raise GraphError(f"vertex index outside [0,{g.n})")
    return np.unique(idx)


def _member_report(g, idx: np.ndarray) -> tuple[float, bool, bool]:
    mask = np.zeros(max(g.n, 1), dtype=np.uint8)
    mask[idx] = 1
    weight = E.ctypes.c_double()
    ind = E.ctypes.c_int()
    mx = E.ctypes.c_int()
    cnt = E.ctypes.c_int64()
    h = any_device_graph(g)
    E.check(E.lib().gn_check_members(h.handle, E.ptr(mask), E.ctypes.byref(weight), E.ctypes.byref(ind),
                                     E.ctypes.byref(mx), E.ctypes.byref(cnt)))
    return weight.value, bool(ind.value), bool(mx.value)


def is_independent(g, members: Iterable[int]) -> bool:
    """True iff no edge joins two members (graph.py:134-142)."""
    return _member_report(g, _check_members(g, members))[1]


def is_maximal_independent(g, members: Iterable[int]) -> bool:
    """True iff members form an independent set dominating every outside
    vertex (graph.py:145-156)."""
    return _member_report(g, _check_members(g, members))[2]


def set_weight(g, members: Iterable[int]) -> float:
    """Total weight of a vertex subset; the empty set weighs 0 (graph.py:159-162)."""
    return _member_report(g, _check_members(g, members))[0]


class MisSolution:
    """A vertex subset claimed independent, with validity flags (graph.py:165-186).

    members is sorted ascending; weight is the recomputable sum of
    vertex weights over members.

    Same fields, construction, equality, hashing, repr and immutability as
    the reference's frozen dataclass.  A solution made by the engine keeps
    its members as an index array and builds the ``members`` tuple of
    Python ints on first access (a 14M-member R-MAT MIS costs ~0.4 s of
    tuple building otherwise, paid only by callers that read it).
    """

    __slots__ = ("_members", "_idx", "weight", "independent", "maximal")

    def __init__(self, members: Iterable[int] = (), weight: float = 0.0, independent: bool = False,
                 maximal: bool = False):
        object.__setattr__(self, "_members", tuple(members))
        object.__setattr__(self, "_idx", None)
        object.__setattr__(self, "weight", weight)
        object.__setattr__(self, "independent", independent)
        object.__setattr__(self, "maximal", maximal)

    @classmethod
    def _lazy(cls, idx: np.ndarray, weight: float, independent: bool, maximal: bool) -> "MisSolution":
        """From a sorted index array (engine results): members built on first access."""
        sol = cls.__new__(cls)
        object.__setattr__(sol, "_members", None)
        object.__setattr__(sol, "_idx", np.asarray(idx, dtype=np.int64))
        object.__setattr__(sol, "weight", weight)
        object.__setattr__(sol, "independent", independent)
        object.__setattr__(sol, "maximal", maximal)
        return sol

    @property
    def members(self) -> tuple[int, ...]:
        if self._members is None:
            object.__setattr__(self, "_members", tuple(self._idx.tolist()))
            object.__setattr__(self, "_idx", None)
        return self._members

    def __setattr__(self, name, value):
        raise dataclasses.FrozenInstanceError(f"cannot assign to field {name!r}")

    def __delattr__(self, name):
        raise dataclasses.FrozenInstanceError(f"cannot delete field {name!r}")

    def _key(self):
        return (self.members, self.weight, self.independent, self.maximal)

    def __eq__(self, other):
        if other.__class__ is not self.__class__:
            return NotImplemented
        return self._key() == other._key()

    def __hash__(self):
        return hash(self._key())

    def __reduce__(self):  # pickle / copy: the reference dataclass's fields
        return (MisSolution, (self.members, self.weight, self.independent, self.maximal))

    def __repr__(self):
        return (f"MisSolution(members={self.members!r}, weight={self.weight!r}, "
                f"independent={self.independent!r}, maximal={self.maximal!r})")

    @classmethod
    def from_members(cls, g, members: Iterable[int]) -> "MisSolution":
        idx = _check_members(g, members)
        weight, ind, mx = _member_report(g, idx)
        return cls(members=tuple(np.asarray(idx, dtype=np.int64).tolist()), weight=weight, independent=ind, maximal=mx)


def erdos_renyi(
    n: int,
    p: float,
    seed,
    weight_low: float = 0.1,
    weight_high: float = 10.0,
) -> WeightedGraph:
    """G(n, p) with i.i.d. uniform vertex weights; deterministic per seed.

    Same random stream as graph.py:189-202, so the same seed gives the same
    graph as the reference."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    pick = rng.random(len(iu)) < p
    weights = rng.uniform(weight_low, weight_high, size=n)
    indptr, indices = csr_from_edges(n, iu[pick], ju[pick])
    return WeightedGraph(n, indptr, indices, np.asarray(weights, dtype=np.float64))
