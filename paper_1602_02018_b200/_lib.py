"""ctypes binding of ``libcsc_b200.so`` (the C ABI declared in ``include/csc_b200.h``).

This is the only module that talks to native code.  The library is built
in-tree (``make -C paper_1602_02018_b200/csrc``, or ``__graft_entry__.build()``)
and there is deliberately no fallback: if it is missing, or no CUDA device is
present, every hot-path call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
from pathlib import Path

import numpy as np

from ._errors import GraphError

LIB_PATH = Path(__file__).resolve().parent / "libcsc_b200.so"

CSC_OK, CSC_ERR_INVALID, CSC_ERR_GRAPH, CSC_ERR_CUDA, CSC_ERR_NOMEM = 0, 1, 2, 3, 4
CSC_F64, CSC_F32 = 0, 1
CSC_SELF_LOOPS_ERROR, CSC_SELF_LOOPS_DROP = 0, 1

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_f64 = C.c_double

# name -> argtypes (restype is always int status, except csc_last_error / csc_abi_version)
SIGNATURES: dict[str, list] = {
    "csc_abi_version": [],
    "csc_last_error": [],
    "csc_launch_count": [_p],
    "csc_set_option": [C.c_char_p, _i64],
    "csc_get_option": [C.c_char_p, _p],
    "csc_profile_read": [_p, _p, _p],
    "csc_profile_reset": [],
    "csc_graph_create": [_i64, _i64, _p, _p, _p, _i32, _i32, _p, _p],
    "csc_graph_build_coo": [_i64, _i64, _p, _p, _p, _i32, _i32, _i32, _p, _p],
    "csc_graph_destroy": [_p],
    "csc_graph_info": [_p, _p, _p, _p, _p],
    "csc_graph_export": [_p, _p, _p, _p, _p, _p, _p],
    "csc_edgelist_read": [C.c_char_p, _i32, _p],
    "csc_edgelist_info": [_p, _p, _p, _p, _p],
    "csc_edgelist_rows": [_p, _p, _p, _p, _p],
    "csc_edgelist_complex": [_p, _p, _p, _p, _p],
    "csc_edgelist_destroy": [_p],
    "csc_edgelist_write": [C.c_char_p, _i64, _p, _p, _p, _i32],
    "csc_float_repr": [_f64, _p, _i32, _p],
    "csc_laplacian_apply": [_p, _p, _i64, _p, _i64, _i32, _i32, _p],
    "csc_cheb_filter": [_p, _p, _i32, _p, _i64, _p, _i64, _i32, _i32, _p],
    "csc_eigencount": [_p, _p, _i32, _p, _i64, _i32, _i32, _p, _p],
    "csc_build_features": [_p, _p, _i32, _p, _i64, _i32, _i32, _p, _i64, _p, _p, _p],
    "csc_filter_rowsq": [_p, _p, _i32, _p, _i64, _i32, _i32, _p, _i64, _p, _p],
    "csc_normalize_rows": [_p, _i64, _i64, _i32, _i32, _p, _p, _i64, _p, _p, _i32, _p],
    "csc_system_apply": [_p, _p, _i32, _f64, _f64, _p, _p, _i64, _p, _i64, _i32, _i32, _p],
    "csc_gather_rows": [_p, _i64, _i64, _i32, _i32, _p, _i64, _p, _i64, _i32, _p],
    "csc_block_cg": [_p, _p, _i32, _f64, _f64, _p, _i64, _p, _i32, _f64, _i64, _p, _i64, _i32,
                     _p, _p, _p, _p, _p],
    "csc_assign": [_p, _i64, _i64, _i32, _i32, _p, _p, _p, _i32, _p],
    "csc_kmeans_lloyd": [_p, _i64, _i32, _p, _i32, _i64, _f64, _p, _p, _p, _p, _i32, _p],
    "csc_kmeans_replicates": [_p, _i64, _i32, _i32, _i32, _p, _p, _p, _i64, _f64, _p, _p, _p, _p, _p, _i32, _p],
    "csc_set_normal_tables": [_p, _p, _p],
    "csc_numpy_normals": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _i64, _f64, _p, _p, _i32, _p],
    "csc_set_exponential_tables": [_p, _p, _p],
    "csc_sbm_edges": [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _i64, _p, _p, _p, _p, _p, _p, _p, _i64, _p, _p,
                      _p, _p, _i32, _p],
    "csc_dcsbm_edges": [_i64, _i32, _p, _p, _f64, _f64, C.c_uint64, _i32, _i64, _p, _p, _p],
    "csc_panel_row_bytes": [_i64, _i32, _i32, _i32, _i64, _p],
    "csc_peers_create": [_i32, _i32, _i32, C.c_size_t, _p],
    "csc_peers_handle": [_p, _p],
    "csc_peers_attach": [_p, _i32, _p],
    "csc_peers_set_host_barrier": [_p, _p, _p],
    "csc_peers_destroy": [_p],
    "csc_cheb_filter_rows_peers": [_p, _p, _p, _i32, _p, _i64, _p, _i64, _i32, _i32, _i32, _p, _p],
    "csc_comm_unique_id": [_p],
    "csc_comm_create": [_p, _i32, _i32, _i32, _p],
    "csc_comm_destroy": [_p],
    "csc_graph_create_row_shard": [_i64, _i32, _i32, _p, _i64, _p, _p, _p, _i32, _i32, _p, _p],
    "csc_cheb_filter_rows_group": [_p, _i32, _p, _i32, _p, _p, _p, _p, _i32, _i32, _i32, _p, _p],
    "csc_cheb_filter_rows": [_p, _p, _p, _i32, _p, _i64, _p, _i64, _i32, _i32, _i32, _p, _p],
    "csc_assign_partial": [_p, _i64, _i64, _i32, _i32, _i64, _p, _p, _p, _p, _i32, _p],
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load the native library once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {LIB_PATH.parent / 'csrc'}` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(str(LIB_PATH))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = C.c_int
        lib.csc_last_error.restype = C.c_char_p
        if lib.csc_abi_version() != 1:
            raise ImportError("libcsc_b200.so ABI version mismatch")
        _lib = lib
        return lib


def check(status: int) -> None:
    """Map a C status to the reference's exception types."""
    if status == CSC_OK:
        return
    msg = (load().csc_last_error() or b"").decode("utf-8", "replace")
    if status == CSC_ERR_INVALID:
        raise ValueError(msg)
    if status == CSC_ERR_GRAPH:
        raise GraphError(msg)
    if status == CSC_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA failure in libcsc_b200: {msg}")


def call(name: str, *args) -> None:
    status = getattr(load(), name)(*args)
    if status == CSC_ERR_NOMEM and "torch" in sys.modules:
        # the library already handed its own pool's cached blocks back; torch's caching
        # allocator may hold the rest.  Entry points are pure (outputs fully rewritten), so
        # one retry after emptying torch's cache is safe.
        import torch

        if torch.cuda.is_available():
            torch.cuda.empty_cache()
            status = getattr(load(), name)(*args)
    check(status)


def ptr(a) -> int | None:
    """Raw data pointer of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def dtype_code(dt) -> int:
    s = str(dt)
    if s in ("float64", "torch.float64", "f64", "double"):
        return CSC_F64
    if s in ("float32", "torch.float32", "f32", "float"):
        return CSC_F32
    raise ValueError(f"unsupported dtype {dt!r}: use float64 or float32")


def launch_count() -> int:
    v = C.c_int64(0)
    call("csc_launch_count", C.byref(v))
    return int(v.value)


def set_option(key: str, value: int) -> None:
    call("csc_set_option", key.encode(), int(value))


def get_option(key: str) -> int:
    v = C.c_int64(0)
    call("csc_get_option", key.encode(), C.byref(v))
    return int(v.value)


def profile_read() -> tuple[float, int, float]:
    ms, n, b = C.c_double(0), C.c_int64(0), C.c_double(0)
    call("csc_profile_read", C.byref(ms), C.byref(n), C.byref(b))
    return float(ms.value), int(n.value), float(b.value)


def profile_reset() -> None:
    call("csc_profile_reset")


def default_device() -> int:
    """Device for new operators: CSC_DEVICE, else LOCAL_RANK, else 0."""
    for key in ("CSC_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


def current_stream(device: int) -> int | None:
    """torch's current stream on ``device`` when torch is already in use, else the default stream."""
    import sys

    torch = sys.modules.get("torch")
    if torch is None or not torch.cuda.is_available() or not torch.cuda.is_initialized():
        return None
    return torch.cuda.current_stream(device).cuda_stream or None
