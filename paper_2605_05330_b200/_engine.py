"""ctypes binding of libgnb200.so (the C ABI in include/gn_b200.h).

This is the only place the package touches native code.  There is no CPU
fallback: if the library or a CUDA device is missing, every engine call
raises ``EngineUnavailable`` with the loader's or the driver's reason.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libgnb200.so"

GN_F64 = 0
GN_F32 = 1
GN_F32_PURE = 2

GN_OK = 0
GN_ERR_ARG = 1
GN_ERR_CUDA = 2
GN_ERR_NEGATIVE = 3
GN_ERR_NOT_NORMALIZABLE = 4
GN_ERR_NONFINITE = 5
GN_ERR_NOMEM = 6
GN_ERR_NODEV = 7
GN_ERR_ZERO_DENOM = 8
GN_ERR_ZERO_MASS = 9
GN_ERR_FORMAT = 10
GN_PARSE_FALLBACK = 11

GN_TRACE = 0x1
GN_EARLY_EXIT = 0x2
GN_EXACT = 0x4
GN_DEVICE_IO = 0x8
GN_NO_CHECK = 0x10
GN_NO_CLIP = 0x20
GN_NONFINITE_OK = 0x40

# every symbol include/gn_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "gn_abi_version",
    "gn_last_error",
    "gn_device_count",
    "gn_launch_count",
    "gn_graph_create",
    "gn_graph_destroy",
    "gn_graph_info",
    "gn_graph_set_grid",
    "gn_run",
    "gn_step",
    "gn_is_normalizable",
    "gn_spmv",
    "gn_energy",
    "gn_weighted_mass",
    "gn_simplex_state",
    "gn_fitness",
    "gn_round",
    "gn_round_members",
    "gn_round_many",
    "gn_check_members",
    "gn_multi_run",
    "gn_batch_create",
    "gn_batch_destroy",
    "gn_batch_info",
    "gn_batch_run",
    "gn_part_create",
    "gn_part_destroy",
    "gn_part_info",
    "gn_part_elem_bytes",
    "gn_part_begin",
    "gn_part_step",
    "gn_part_set_boundary",
    "gn_part_step_range",
    "gn_part_pack",
    "gn_part_unpack",
    "gn_part_end",
    "gn_gen_rmat",
    "gn_csr_from_edges",
    "gn_free_host",
    "gn_part_peer_init",
    "gn_part_peer_buffers",
    "gn_part_peer_add",
    "gn_part_peer_commit",
    "gn_part_peer_wait",
    "gn_part_peer_signal",
    "gn_part_run",
    "gn_part_run_group",
    "gn_part_probe",
    "gn_part_gathers",
    "gn_ipc_get_handle",
    "gn_ipc_open_handle",
    "gn_ipc_close",
    "gn_mwis_parse",
    "gn_mwis_info",
    "gn_mwis_copy",
    "gn_mwis_free",
)


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library or device missing)."""


class EngineError(RuntimeError):
    """A CUDA or argument error reported by the engine."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[gn status {code}] {message}")
        self.code = code
        self.message = message


class RunStats(ctypes.Structure):
    _fields_ = [
        ("loop_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("launches", ctypes.c_int64),
        ("grid_blocks", ctypes.c_int64),
        ("block_threads", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_U32 = ctypes.c_uint32
_D = ctypes.c_double
_PD = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PI = ctypes.POINTER(ctypes.c_int)

_SIGNATURES = {
    "gn_abi_version": (_I32, []),
    "gn_last_error": (ctypes.c_char_p, []),
    "gn_device_count": (_I32, [_PI]),
    "gn_launch_count": (_I64, []),
    "gn_graph_create": (_I32, [_I64, _P, _P, _P, _I32, _I32, ctypes.POINTER(_P)]),
    "gn_graph_destroy": (_I32, [_P]),
    "gn_graph_info": (_I32, [_P, _PI64, _PI64, _PI, _PI, _PI64, _PI]),
    "gn_graph_set_grid": (_I32, [_P, _I32]),
    "gn_run": (
        _I32,
        [_P, _P, _P, _I32, _D, _U32, _P, _P, _P, _P, _P, _P, _P, _PI, _PI, ctypes.POINTER(RunStats)],
    ),
    "gn_step": (_I32, [_P, _P, _D, _U32, _P, _PI64]),
    "gn_is_normalizable": (_I32, [_P, _P, _PI]),
    "gn_spmv": (_I32, [_P, _P, _P]),
    "gn_energy": (_I32, [_P, _P, _D, _PD]),
    "gn_weighted_mass": (_I32, [_P, _P, _PD]),
    "gn_simplex_state": (_I32, [_P, _P, _P]),
    "gn_fitness": (_I32, [_P, _P, _D, _P, _PD]),
    "gn_round": (_I32, [_P, _P, _U32, _P, _PD, _PI, _PI, _PI64]),
    "gn_round_members": (_I32, [_P, _P, _U32, _P, _PD, _PI, _PI, _PI64]),
    "gn_round_many": (_I32, [_P, _I32, _P, _U32, _P, _P, _P, _P, _P]),
    "gn_check_members": (_I32, [_P, _P, _PD, _PI, _PI, _PI64]),
    "gn_multi_run": (
        _I32,
        [_P, _I32, _P, _P, _I32, _D, _U32, _P, _P, _P, _P, _P, _P, ctypes.POINTER(RunStats)],
    ),
    "gn_batch_create": (_I32, [_I64, _P, _I64, _P, _P, _P, _I32, _I32, ctypes.POINTER(_P)]),
    "gn_batch_destroy": (_I32, [_P]),
    "gn_batch_info": (_I32, [_P, _PI64, _PI64, _PI64, _PI64]),
    "gn_batch_run": (
        _I32,
        [_P, _P, _P, _I32, _D, _U32, _P, _P, _P, _P, _P, _P, _P, ctypes.POINTER(RunStats)],
    ),
    "gn_part_create": (_I32, [_I64, _I64, _P, _P, _P, _I32, _I32, ctypes.POINTER(_P)]),
    "gn_part_destroy": (_I32, [_P]),
    "gn_part_info": (_I32, [_P, _PI64, _PI64, _PI64]),
    "gn_part_elem_bytes": (_I32, [_P]),
    "gn_part_begin": (_I32, [_P, _P, _P, _I32, _U32]),
    "gn_part_step": (_I32, [_P, _I32, ctypes.c_size_t]),
    "gn_part_set_boundary": (_I32, [_P, _P, _I64]),
    "gn_part_step_range": (_I32, [_P, _I32, _I32, ctypes.c_size_t]),
    "gn_part_pack": (_I32, [_P, _I32, _P, _I64, _P, ctypes.c_size_t]),
    "gn_part_unpack": (_I32, [_P, _I32, _P, _I64, _I64, ctypes.c_size_t]),
    "gn_part_end": (_I32, [_P, _I32, _P, _P, _P, _P, _PI]),
    "gn_gen_rmat": (_I32, [_I32, _I32, _D, _D, _D, ctypes.c_uint64, _I32, _PI64, ctypes.POINTER(_P),
                           ctypes.POINTER(_P)]),
    "gn_csr_from_edges": (_I32, [_I64, _I64, _P, _P, _I32, _PI64, _PI64, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "gn_part_peer_init": (_I32, [_P, _I32, _I32, _P, _I32]),
    "gn_part_peer_buffers": (_I32, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "gn_part_peer_add": (_I32, [_P, _I32, _P, _P, _P, _P, _I64, _I64]),
    "gn_part_peer_commit": (_I32, [_P]),
    "gn_part_peer_wait": (_I32, [_P, _I32, ctypes.c_uint64]),
    "gn_part_peer_signal": (_I32, [_P, _I32, ctypes.c_uint64]),
    "gn_part_run": (_I32, [_P, _I32, _I32, ctypes.c_uint64]),
    "gn_part_run_group": (_I32, [_P, _I32, _I32, _I32, ctypes.c_uint64]),
    "gn_part_probe": (_I32, [_P, _I32, _I32, ctypes.POINTER(ctypes.c_double)]),
    "gn_part_gathers": (_I32, [_P, _I32, _P]),
    "gn_ipc_get_handle": (_I32, [_P, _P]),
    "gn_ipc_open_handle": (_I32, [_P, _I32, ctypes.POINTER(_P)]),
    "gn_ipc_close": (_I32, [_P]),
    "gn_mwis_parse": (_I32, [ctypes.c_char_p, _I64, ctypes.POINTER(_P), ctypes.c_char_p, _I64]),
    "gn_mwis_info": (_I32, [_P, _PI64, _PI64]),
    "gn_mwis_copy": (_I32, [_P, _P, _P]),
    "gn_mwis_free": (None, [_P]),
    "gn_free_host": (None, [_P]),
}

_lib = None
_lib_lock = threading.Lock()
_load_error: str | None = None


def load_library(path: os.PathLike | str | None = None) -> ctypes.CDLL:
    """Load libgnb200.so (built in-tree by ``make`` / ``__graft_entry__.build``)."""
    global _lib, _load_error
    with _lib_lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("GN_LIB") or LIB_PATH)
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:
            _load_error = f"cannot load {p}: {exc} (run `make -C paper_2605_05330_b200`)"
            raise EngineUnavailable(_load_error) from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load_library()


def last_error() -> str:
    return lib().gn_last_error().decode(errors="replace")


def check(code: int) -> None:
    if code == GN_OK:
        return
    msg = last_error()
    if code == GN_ERR_NODEV:
        raise EngineUnavailable(msg)
    raise EngineError(code, msg)


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = lib().gn_device_count(ctypes.byref(c))
    return c.value if rc == GN_OK else 0


def launch_count() -> int:
    return int(lib().gn_launch_count())


def ptr(a: np.ndarray | None):
    """Raw data pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "engine arrays must be C-contiguous"
    return ctypes.c_void_p(a.ctypes.data)


class GraphHandle:
    """Owns one device-resident gn_graph.  Immutable, shareable across threads."""

    def __init__(self, n: int, indptr: np.ndarray, indices: np.ndarray, w: np.ndarray,
                 dtype: int = GN_F64, device: int = 0):
        self._lib = lib()
        self.n = int(n)
        self.dtype = dtype
        self.device = device
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        ww = np.ascontiguousarray(w, dtype=np.float64)
        h = ctypes.c_void_p()
        check(self._lib.gn_graph_create(self.n, ptr(ip), ptr(ix), ptr(ww), dtype, device,
                                        ctypes.byref(h)))
        self._h = h

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise EngineError(GN_ERR_ARG, "graph handle already destroyed")
        return self._h

    def info(self) -> dict:
        n, nnz, dev_bytes = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        dt, dev, nb = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(self._lib.gn_graph_info(self.handle, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(dt),
                                      ctypes.byref(dev), ctypes.byref(dev_bytes), ctypes.byref(nb)))
        return {"n": n.value, "nnz": nnz.value, "dtype": dt.value, "device": dev.value,
                "device_bytes": dev_bytes.value, "num_bins": nb.value}

    def set_grid(self, blocks: int) -> None:
        check(self._lib.gn_graph_set_grid(self.handle, int(blocks)))

    def close(self) -> None:
        if self._h is not None:
            self._lib.gn_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
