"""Graphs in canonical CSR and the device-resident normalized Laplacian.

Drop-in for ``cscluster.graph`` (reference ``graph.py``).  The data model is the
reference's: a symmetric CSR with sorted, de-duplicated columns, no loops,
fp64 weights and fp64 row-sum degrees (graph.py:23-55), and the operator
``L = I - D^-1/2 W D^-1/2`` with ``d^-1/2 = 0`` on isolated nodes
(graph.py:128-169).  What changes is where the work happens:

- ``build_graph`` validates on the host with the reference's messages
  (graph.py:87-120) and canonicalises on the device (K1, ``csc_graph_build_coo``);
- ``laplacian_op`` uploads the CSR once and keeps ``Wn = D^-1/2 W D^-1/2`` on the
  GPU in fp64 or fp32 (K1, ``csc_graph_create``);
- ``LaplacianOp.apply`` runs the SpMM kernel (``csc_laplacian_apply``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._errors import GraphError

__all__ = [
    "Graph",
    "GraphError",
    "LaplacianOp",
    "apply_laplacian",
    "build_graph",
    "laplacian_op",
    "read_edge_list",
    "write_edge_list",
]


class DeviceGraph:
    """Owner of one native ``csc_graph`` handle (freed with the object)."""

    def __init__(self, handle: int, num_nodes: int, nnz: int, dtype: int, device: int):
        self.handle = handle
        self.num_nodes = num_nodes
        self.nnz = nnz
        self.dtype = dtype
        self.device = device

    @classmethod
    def from_csr(cls, indptr, indices, weights, num_nodes: int, dtype: int, device: int) -> "DeviceGraph":
        indptr = np.ascontiguousarray(indptr, dtype=np.int32)
        indices = np.ascontiguousarray(indices, dtype=np.int32)
        weights = np.ascontiguousarray(weights, dtype=np.float64)
        out = C.c_void_p()
        _lib.call(
            "csc_graph_create", int(num_nodes), int(indices.size), _lib.ptr(indptr), _lib.ptr(indices),
            _lib.ptr(weights), dtype, device, _lib.current_stream(device), C.byref(out),
        )
        return cls(out.value, int(num_nodes), int(indices.size), dtype, device)

    @classmethod
    def from_edges(cls, src, dst, weights, num_nodes: int, self_loops: str, dtype: int, device: int) -> "DeviceGraph":
        if isinstance(src, np.ndarray) or not hasattr(src, "data_ptr"):
            src = np.ascontiguousarray(src, dtype=np.int64)
            dst = np.ascontiguousarray(dst, dtype=np.int64)
        else:  # CUDA int64 tensors on `device` (edges generated on the GPU)
            src, dst = src.contiguous(), dst.contiguous()
            if src.dtype != dst.dtype or str(src.dtype) != "torch.int64" or src.numel() != dst.numel():
                raise ValueError("device edge arrays must be int64 tensors of equal length")
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        mode = _lib.CSC_SELF_LOOPS_DROP if self_loops == "drop" else _lib.CSC_SELF_LOOPS_ERROR
        out = C.c_void_p()
        _lib.call(
            "csc_graph_build_coo", int(num_nodes), int(src.shape[0]), _lib.ptr(src), _lib.ptr(dst), _lib.ptr(w),
            mode, dtype, device, _lib.current_stream(device), C.byref(out),
        )
        nnz = C.c_int64(0)
        _lib.call("csc_graph_info", out.value, None, C.byref(nnz), None, None)
        return cls(out.value, int(num_nodes), int(nnz.value), dtype, device)

    def export(self):
        n, nnz = self.num_nodes, self.nnz
        indptr = np.empty(n + 1, dtype=np.int32)
        indices = np.empty(nnz, dtype=np.int32)
        weights = np.empty(nnz, dtype=np.float64)
        degrees = np.empty(n, dtype=np.float64)
        dis = np.empty(n, dtype=np.float64)
        _lib.call(
            "csc_graph_export", self.handle, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(weights),
            _lib.ptr(degrees), _lib.ptr(dis), _lib.current_stream(self.device),
        )
        return indptr, indices, weights, degrees, dis

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h and _lib._lib is not None:
            _lib._lib.csc_graph_destroy(h)


@dataclass
class Graph:
    """Symmetric graph stored as canonical CSR (sorted, deduplicated, no loops).

    Same fields and invariants as the reference (graph.py:23-55).  Device
    operators built from it are cached per (dtype, device).
    """

    num_nodes: int
    indptr: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    degrees: np.ndarray
    _csr: object | None = field(default=None, repr=False, compare=False)
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def num_edges(self) -> int:
        """Number of undirected edges (stored entry pairs / 2)."""
        return int(self.indices.size) // 2

    @property
    def isolated_nodes(self) -> np.ndarray:
        return np.flatnonzero(self.degrees == 0.0)

    def adjacency(self):
        """scipy CSR view sharing the buffers (container only; not on the hot path)."""
        if self._csr is None:
            import scipy.sparse as sp

            self._csr = sp.csr_matrix((self.weights, self.indices, self.indptr), shape=(self.num_nodes, self.num_nodes))
        return self._csr

    def device_graph(self, dtype: int = _lib.CSC_F64, device: int | None = None) -> DeviceGraph:
        dev = _lib.default_device() if device is None else int(device)
        key = (dtype, dev)
        dg = self._device.get(key)
        if dg is None:
            dg = DeviceGraph.from_csr(self.indptr, self.indices, self.weights, self.num_nodes, dtype, dev)
            self._device[key] = dg
        return dg

    @classmethod
    def _from_device(cls, dg: DeviceGraph) -> tuple["Graph", np.ndarray]:
        indptr, indices, weights, degrees, dis = dg.export()
        g = cls(num_nodes=dg.num_nodes, indptr=indptr, indices=indices, weights=weights, degrees=degrees)
        g._device[(dg.dtype, dg.device)] = dg
        return g, dis


def _edge_array(edges) -> np.ndarray:
    if isinstance(edges, np.ndarray):
        arr = np.asarray(edges, dtype=np.float64)
    else:
        arr = np.asarray(list(edges), dtype=np.float64)
    arr = np.atleast_2d(arr)
    if arr.size == 0:
        return arr.reshape(0, 3)
    if arr.shape[1] == 2:
        return np.column_stack([arr, np.ones(arr.shape[0])])
    if arr.shape[1] != 3:
        raise GraphError(f"edges must be (i, j) or (i, j, w) rows, got shape {arr.shape}")
    return arr


def build_graph(
    edges: Iterable[Sequence[float]] | np.ndarray,
    num_nodes: int | None = None,
    *,
    self_loops: str = "error",
    device: int | None = None,
) -> Graph:
    """Canonical symmetric graph from (i, j[, weight]) triples (reference graph.py:73-125).

    Validation and its messages follow the reference (graph.py:87-120); the
    canonicalisation (per-direction duplicate sum, max-symmetrisation, sort,
    zero elimination, degrees) runs on the device.
    """
    if self_loops not in ("error", "drop"):
        raise ValueError(f"self_loops must be 'error' or 'drop', got {self_loops!r}")
    arr = _edge_array(edges)
    src_f, dst_f, w = arr[:, 0], arr[:, 1], arr[:, 2]
    if not (np.array_equal(src_f, np.floor(src_f)) and np.array_equal(dst_f, np.floor(dst_f))):
        raise GraphError("node indices must be integers")
    src = src_f.astype(np.int64)
    dst = dst_f.astype(np.int64)
    neg = np.flatnonzero(w < 0)
    if neg.size:
        b = int(neg[0])
        raise GraphError(f"negative weight {w[b]} on edge ({src[b]}, {dst[b]})")
    if (src < 0).any() or (dst < 0).any():
        raise GraphError("negative node index")
    top = int(max(src.max(), dst.max())) if src.size else -1
    if num_nodes is None:
        num_nodes = top + 1
    elif top >= num_nodes:
        raise GraphError(f"node index {top} out of range for num_nodes={num_nodes}")
    loops = np.flatnonzero(src == dst)
    if loops.size and self_loops == "error":
        raise GraphError(f"self-loop on node {int(src[loops[0]])}")
    dev = _lib.default_device() if device is None else int(device)
    dg = DeviceGraph.from_edges(src, dst, w, int(num_nodes), self_loops, _lib.CSC_F64, dev)
    graph, _ = Graph._from_device(dg)
    return graph


@dataclass
class LaplacianOp:
    """Normalized Laplacian ``L = I - D^-1/2 W D^-1/2`` resident on a GPU.

    Same surface as the reference operator (graph.py:128-161): ``graph``,
    ``d_inv_sqrt``, ``num_nodes``, ``shape``, ``apply``, ``dense``.  ``dtype`` is
    the compute precision of the device operator ("float64" or "float32").
    """

    graph: Graph
    d_inv_sqrt: np.ndarray
    dtype: str = "float64"
    device: int = 0

    @property
    def num_nodes(self) -> int:
        return self.graph.num_nodes

    @property
    def shape(self) -> tuple[int, int]:
        return (self.graph.num_nodes, self.graph.num_nodes)

    @property
    def handle(self) -> int:
        return self.graph.device_graph(_lib.dtype_code(self.dtype), self.device).handle

    @property
    def compute_code(self) -> int:
        return _lib.dtype_code(self.dtype)

    def apply(self, x):
        """Return L x for a vector or an N-row block (numpy or CUDA torch tensor)."""
        from ._blocks import as_block, from_block

        blk = as_block(x, self.num_nodes, "signal")
        out = blk.empty_like()
        _lib.call(
            "csc_laplacian_apply", self.handle, blk.ptr, blk.ld, out.ptr, out.ld, blk.ncols, blk.code,
            _lib.current_stream(self.device),
        )
        return from_block(out, x)

    def dense(self) -> np.ndarray:
        """Dense N x N Laplacian (test/oracle use; O(N^2) memory, host)."""
        W = self.graph.adjacency().toarray()
        S = self.d_inv_sqrt
        return np.eye(self.num_nodes) - S[:, None] * W * S[None, :]


def laplacian_op(graph: Graph, dtype: str = "float64", device: int | None = None) -> LaplacianOp:
    """Build (and upload) the normalized Laplacian operator (reference graph.py:164-169)."""
    dev = _lib.default_device() if device is None else int(device)
    graph.device_graph(_lib.dtype_code(dtype), dev)  # upload + normalise now (K1), cached on the graph
    d = graph.degrees
    with np.errstate(divide="ignore"):
        dis = np.where(d > 0, 1.0 / np.sqrt(np.where(d > 0, d, 1.0)), 0.0)
    return LaplacianOp(graph=graph, d_inv_sqrt=dis, dtype=str(np.dtype(dtype)), device=dev)


def apply_laplacian(op: LaplacianOp, x):
    """Functional alias for ``op.apply(x)``."""
    return op.apply(x)


def parse_edge_list(path: str | Path) -> tuple[np.ndarray, int | None]:
    """The parse of read_edge_list (graph.py:188-212): rows (E x 3 float64, file order) and
    the ``# nodes N`` header value (None when absent).

    The line loop runs in the library (``csc_edgelist_read``, multi-threaded); lines whose
    tokens it does not convert itself (non-ASCII, underscores, inf/nan, wrong token counts,
    ...) come back as "complex" and are parsed here with the reference's own rules, in file
    order, so values, row order and the first error raised match the reference."""
    path = Path(path)
    h = C.c_void_p()
    _lib.call("csc_edgelist_read", str(path).encode(), 0, C.byref(h))
    try:
        nr, ncx, hn, hl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.call("csc_edgelist_info", h, C.byref(nr), C.byref(ncx), C.byref(hn), C.byref(hl))
        src, dst, w = np.empty(nr.value), np.empty(nr.value), np.empty(nr.value)
        cx = np.empty(nr.value, dtype=np.uint8)
        _lib.call("csc_edgelist_rows", h, _lib.ptr(src), _lib.ptr(dst), _lib.ptr(w), _lib.ptr(cx))
        lines, slots, offs, lens = (np.empty(ncx.value, dtype=np.int64) for _ in range(4))
        _lib.call("csc_edgelist_complex", h, _lib.ptr(lines), _lib.ptr(slots), _lib.ptr(offs), _lib.ptr(lens))
    finally:
        _lib.call("csc_edgelist_destroy", h)
    header_nodes = int(hn.value) if hl.value > 0 else None
    header_line = int(hl.value)
    keep = np.ones(nr.value, dtype=bool)
    if ncx.value:
        with path.open("rb") as fh:
            for lineno, slot, off, ln in zip(lines.tolist(), slots.tolist(), offs.tolist(), lens.tolist()):
                fh.seek(off)
                stripped = fh.read(ln).decode("utf-8").strip()
                if not stripped or stripped.startswith("#"):
                    if slot >= 0:
                        keep[slot] = False
                    parts = stripped[1:].split() if stripped else []
                    if len(parts) == 2 and parts[0] == "nodes":
                        try:
                            value = int(parts[1])
                        except ValueError:
                            pass
                        else:
                            if lineno > header_line:
                                header_nodes, header_line = value, lineno
                    continue
                parts = stripped.split()
                if len(parts) not in (2, 3):
                    raise GraphError(f"{path}:{lineno}: expected 'src dst [weight]', got {stripped!r}")
                try:
                    i, j = int(parts[0]), int(parts[1])
                    wt = float(parts[2]) if len(parts) == 3 else 1.0
                except ValueError as exc:
                    raise GraphError(f"{path}:{lineno}: {exc}") from None
                src[slot], dst[slot], w[slot] = float(i), float(j), wt
    rows = np.column_stack([src[keep], dst[keep], w[keep]])
    return rows, header_nodes


def read_edge_list(path: str | Path, num_nodes: int | None = None) -> Graph:
    """Parse ``src dst [weight]`` lines (``#`` comments, ``# nodes N`` header), as graph.py:177-214."""
    rows, header_nodes = parse_edge_list(path)
    if num_nodes is None:
        num_nodes = header_nodes
    return build_graph(rows, num_nodes=num_nodes, self_loops="error")


def write_edge_list(graph: Graph, path: str | Path) -> None:
    """One ``src dst weight`` line per undirected edge (i < j) in CSR order, after a ``# nodes N``
    header (graph.py:215-225); written by ``csc_edgelist_write`` (Python's repr() of each weight)."""
    indptr = np.ascontiguousarray(graph.indptr, dtype=np.int32)
    indices = np.ascontiguousarray(graph.indices, dtype=np.int32)
    weights = np.ascontiguousarray(graph.weights, dtype=np.float64)
    _lib.call("csc_edgelist_write", str(Path(path)).encode(), int(graph.num_nodes), _lib.ptr(indptr),
              _lib.ptr(indices), _lib.ptr(weights), 0)
