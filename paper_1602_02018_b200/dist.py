"""Column-sharded execution over ranks (one process per GPU, torch.distributed).

Every hot-path stage is column-separable (filters.py:140 acts columnwise,
spectrum.py:86 sums over columns, sampling.py:133-135 is per-column CG), so the
graph is replicated and ranks own contiguous slices of the signal / indicator
columns.  The only exchanges are small:

  eigencount   per-rank partial counts (1 fp64), all-gathered, summed in rank order
  features     per-rank row sums of squares (N fp64), all-gathered and summed in
               rank order, then each rank normalises its own columns
  gather       the n sampled rows of each rank's columns (n x d_r), all-gathered
  CG           none per iteration; per-column diagnostics all-gathered at the end
  assign       per-row (best normalised value, global column, nonzero) triples,
               all-gathered and merged with the reference's lowest-index tie rule

Sums are taken in rank order on every rank, so results do not depend on the
collective's internal reduction order.  Random draws stay the reference's: every
rank draws the full probe / signal block from the same named numpy substream and
keeps its column slice, so the sharded run sees exactly the single-GPU inputs.

Per-rank compute goes through a backend (``DeviceBackend`` = the C ABI on the
rank's GPU).  Tests plug in a CPU backend built on the oracle to exercise the
exchange logic with the gloo backend.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._rng import substream
from ._signals import normal_block
from .filters import PolyFilter, coeff_array, design_lowpass, matched_highpass
from .kmeans import kmeans, labels_to_indicators
from .result import ClusterResult
from .sampling import CgInfo, InterpolationConfig, SamplingSet, draw_sampling
from .spectrum import default_num_signals, round_half_up


def column_slice(ncols: int, world: int, rank: int) -> slice:
    """Contiguous balanced split of ``ncols`` columns: the first ncols % world ranks get one extra."""
    base, extra = divmod(ncols, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))


@dataclass
class Group:
    """A torch.distributed process group plus this rank's position and comm device."""

    rank: int
    world: int
    group: object = None
    device: object = "cpu"

    @classmethod
    def current(cls, group=None) -> "Group":
        import torch
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized():
            return cls(0, 1, None, "cpu")
        dev = "cpu"
        if dist.get_backend(group) == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
        return cls(dist.get_rank(group), dist.get_world_size(group), group, dev)

    def _t(self, a):
        import torch

        if isinstance(a, torch.Tensor):
            return a.contiguous().to(self.device)
        return torch.as_tensor(np.ascontiguousarray(a)).to(self.device)

    def all_gather(self, a):
        """All ranks' copies of an equally-shaped array (numpy in -> numpy out,
        tensor in -> tensors on the communication device), in rank order."""
        if self.world == 1:
            return [a if not isinstance(a, np.ndarray) else np.asarray(a)]
        import torch
        import torch.distributed as dist

        t = self._t(a)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        if isinstance(a, torch.Tensor):
            return [p.to(a.device) for p in parts]
        return [p.cpu().numpy() for p in parts]

    def all_gather_var(self, a: np.ndarray) -> list[np.ndarray]:
        """All-gather arrays whose first-axis lengths differ per rank."""
        if self.world == 1:
            return [np.asarray(a)]
        a = np.asarray(a)
        lens = [int(x[0]) for x in self.all_gather(np.array([a.shape[0]], dtype=np.int64))]
        top = max(lens)
        pad = np.zeros((top,) + a.shape[1:], dtype=a.dtype)
        pad[: a.shape[0]] = a
        return [p[:n] for p, n in zip(self.all_gather(pad), lens)]

    def sum_in_order(self, a: np.ndarray) -> np.ndarray:
        """Sum over ranks, accumulated in rank order (deterministic)."""
        parts = self.all_gather(a)
        total = parts[0].clone() if hasattr(parts[0], "clone") else parts[0].copy()
        for p in parts[1:]:
            total = total + p
        return total


class DeviceBackend:
    """Per-rank compute on the rank's GPU through the C ABI (host numpy in/out, device-resident blocks)."""

    def __init__(self, op):
        self.num_edges = op.graph.num_edges
        import torch

        self.op = op
        self.dev = torch.device("cuda", op.device)
        self.stream = lambda: _lib.current_stream(op.device)

    def _dev(self, a):
        import torch

        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.contiguous()
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(self.dev)

    def normal_columns(self, rng, n: int, w: int, cols: slice):
        """This rank's columns of the next n x w block of numpy's stream (every rank draws the
        whole block, so the ranks see the reference's single stream), drawn on the GPU."""
        from ._signals import device_normal_block, device_rng_available, normal_block

        if not device_rng_available():
            return np.ascontiguousarray(normal_block(rng, n, w)[:, cols])
        return device_normal_block(rng, n, w, self.dev.index)[:, cols].contiguous()

    def count(self, filt: PolyFilter, R: np.ndarray) -> float:
        if R.shape[1] == 0:
            return 0.0
        c = coeff_array(filt)
        Rd = self._dev(R)
        out = C.c_double(0.0)
        _lib.call("csc_eigencount", self.op.handle, _lib.ptr(c), int(c.size), Rd.data_ptr(), int(Rd.shape[1]),
                  int(Rd.shape[1]), _lib.dtype_code(Rd.dtype), C.byref(out), self.stream())
        return float(out.value)

    def filter_rowsq(self, filt: PolyFilter, R: np.ndarray):
        import torch

        c = coeff_array(filt)
        Rd = self._dev(R)
        Y = torch.empty_like(Rd)
        rowsq = torch.zeros(R.shape[0], dtype=torch.float64, device=self.dev)
        if R.shape[1]:
            _lib.call("csc_filter_rowsq", self.op.handle, _lib.ptr(c), int(c.size), Rd.data_ptr(), int(Rd.shape[1]),
                      int(Rd.shape[1]), _lib.dtype_code(Rd.dtype), Y.data_ptr(), int(Y.shape[1]), rowsq.data_ptr(),
                      self.stream())
        return Y, rowsq  # stays on the device; the group sums it over NCCL

    def normalize(self, Y, rowsq):
        import torch

        F = torch.empty_like(Y)
        flags = torch.zeros(Y.shape[0], dtype=torch.uint8, device=self.dev)
        nz = C.c_int64(0)
        rq = self._dev(rowsq)
        if Y.shape[1]:
            _lib.call("csc_normalize_rows", Y.data_ptr(), int(Y.shape[1]), int(Y.shape[0]), int(Y.shape[1]),
                      _lib.dtype_code(Y.dtype), rq.data_ptr(), F.data_ptr(), int(F.shape[1]), flags.data_ptr(),
                      C.byref(nz), self.op.device, self.stream())
            zero = flags.nonzero().flatten().cpu().numpy() if nz.value else np.empty(0, dtype=np.int64)
        else:
            zero = np.flatnonzero(rq.cpu().numpy() <= 0.0)
        return F, zero.astype(np.int64)

    def gather(self, F, idx: np.ndarray) -> np.ndarray:
        from .pipeline import _gather_rows

        if F.shape[1] == 0:
            return np.zeros((idx.size, 0))
        return _gather_rows(F, idx, self.op.device)

    def block_cg(self, cfg: InterpolationConfig, sampling: SamplingSet, reduced: np.ndarray):
        import torch

        from .sampling import block_cg_into

        X = torch.empty((self.op.num_nodes, reduced.shape[1]), dtype=torch.float64, device=self.dev)
        if reduced.shape[1] == 0:
            return X, CgInfo(np.zeros(0, np.int64), np.zeros(0), np.zeros(0, bool))
        return X, block_cg_into(self.op, cfg, sampling, reduced, X)

    def kmeans(self, points: np.ndarray, cfg):
        return kmeans(points, cfg, device=self.op.device)

    def row_best(self, soft, col0: int):
        N, k = int(soft.shape[0]), int(soft.shape[1])
        val = np.full(N, -np.inf)
        col = np.zeros(N, dtype=np.int64)
        nz = np.zeros(N, dtype=np.uint8)
        any_norm = C.c_int(0)
        if k:
            _lib.call("csc_assign_partial", soft.data_ptr(), int(soft.stride(0)), N, k, _lib.CSC_F64, int(col0),
                      _lib.ptr(val), _lib.ptr(col), _lib.ptr(nz), C.byref(any_norm), self.op.device, self.stream())
        return val, col, nz.astype(bool), bool(any_norm.value)


def merge_argmax(values: list[np.ndarray], columns: list[np.ndarray]) -> np.ndarray:
    """Per-row winner over rank candidates: larger value, ties -> lower column (sampling.py:210-213)."""
    best_v = values[0].copy()
    best_c = columns[0].copy()
    for v, c in zip(values[1:], columns[1:]):
        take = (v > best_v) | ((v == best_v) & (c < best_c))
        best_v = np.where(take, v, best_v)
        best_c = np.where(take, c, best_c)
    return best_c


def sharded_count(backend, filt: PolyFilter, R_local: np.ndarray, grp: Group) -> float:
    """Eigencount over all ranks' probe columns (spectrum.py:86)."""
    return float(grp.sum_in_order(np.array([backend.count(filt, R_local)]))[0])


def sharded_features(backend, filt: PolyFilter, R_local, grp: Group):
    """This rank's feature columns, normalised by the global row norms (features.py:79-87)."""
    Y, rowsq = backend.filter_rowsq(filt, R_local)
    return backend.normalize(Y, grp.sum_in_order(rowsq))


def sharded_assign(backend, soft_local, col0: int, grp: Group):
    """Global argmax labels from column-sharded soft indicators (sampling.py:197-220)."""
    val, col, nz, any_norm = backend.row_best(soft_local, col0)
    if not any(bool(x[0]) for x in grp.all_gather(np.array([any_norm]))):
        raise ValueError("all indicator vectors are zero")
    labels = merge_argmax(grp.all_gather(val), grp.all_gather(col))
    nonzero = np.zeros(val.size, dtype=bool)
    for part in grp.all_gather(nz):
        nonzero |= part.astype(bool)
    fallback = np.flatnonzero(~nonzero)
    labels[fallback] = 0  # raw argmax of an all-zero row
    return labels.astype(np.int64), fallback


def _normal_columns(backend, rng, n: int, w: int, cols: slice):
    """This rank's columns of the next n x w normal block; every rank draws the whole block
    (identical stream), on the device when the backend can."""
    if hasattr(backend, "normal_columns"):
        return backend.normal_columns(rng, n, w, cols)
    return np.ascontiguousarray(normal_block(rng, n, w)[:, cols])


def estimate_lambda_k_sharded(backend, N: int, k: int, order: int, ds: int | None, rng, grp: Group,
                              max_steps: int = 20, refine: bool = False):
    """Dichotomy of spectrum.py:90-140 with the probe columns sharded over ranks."""
    if not 1 <= k < N:
        raise ValueError(f"k={k} out of range for N={N}")
    ds = ds if ds is not None else default_num_signals(N)
    cols = column_slice(ds, grp.world, grp.rank)
    lo, hi = 0.0, 2.0
    trace: list[tuple[float, float]] = []

    def probe(lam):
        filt = design_lowpass(min(lam, 2.0 - 1e-12), order, damping="jackson")
        cnt = sharded_count(backend, filt, _normal_columns(backend, rng, N, ds, cols), grp)
        trace.append((float(lam), cnt))
        return cnt

    for _ in range(max_steps):
        mid = 0.5 * (lo + hi)
        r = round_half_up(probe(mid))
        if r == k:
            lam = mid
            if refine and (hi - lo) > 0.01 and round_half_up(probe(0.5 * (lo + mid))) == k:
                lam = 0.5 * (lo + mid)
            return lam, trace, False
        if r > k:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi), trace, True


def run_csc_sharded(backend, num_nodes: int, params, grp: Group) -> ClusterResult:
    """run_csc (pipeline.py:113-225) with signal and indicator columns sharded over ranks."""
    N = num_nodes
    prm = params.resolve(N)
    t_run = time.perf_counter()
    timings: dict[str, float] = {}
    warnings: list[str] = []
    t0 = time.perf_counter()
    if prm.lambda_k is not None:
        lam, trace, warn, source = float(prm.lambda_k), [], False, "override"
    else:
        lam, trace, warn = estimate_lambda_k_sharded(backend, N, prm.k, prm.p, prm.probe_signals,
                                                     substream(prm.seed, "probe"), grp, prm.probe_max_steps,
                                                     prm.probe_refine)
        source = "estimated"
        if warn:
            warnings.append("lambda_k bracket fallback")
    timings["probe"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    low = design_lowpass(lam, prm.p, damping=prm.damping)
    high = matched_highpass(low)
    timings["design"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dcols = column_slice(prm.d, grp.world, grp.rank)
    R = _normal_columns(backend, substream(prm.seed, "signals"), N, prm.d, dcols)
    timings["signals"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    F, zero_rows = sharded_features(backend, low, R, grp)
    del R
    if zero_rows.size:
        warnings.append(f"{zero_rows.size} zero-norm feature rows")
    timings["filter"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sampling = draw_sampling(N, prm.n, substream(prm.seed, "sampling"), exclude=zero_rows)
    timings["sampling"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    # ranks own different numbers of feature columns when d % world != 0: exchange the
    # sampled rows column-major so the variable extent is the leading axis
    part = np.ascontiguousarray(np.asarray(backend.gather(F, sampling.indices)).T)
    rows = np.ascontiguousarray(np.concatenate(grp.all_gather_var(part), axis=0).T)
    labeling = backend.kmeans(rows, prm.kmeans)
    timings["kmeans"] = time.perf_counter() - t0
    counts = np.bincount(labeling.labels, minlength=prm.k)
    if np.any(counts == 0):
        from .pipeline import DegenerateClusteringError

        raise DegenerateClusteringError(f"empty cluster(s) {np.flatnonzero(counts == 0).tolist()} in the reduced k-means")
    reduced = labels_to_indicators(labeling.labels, prm.k, prm.n)
    icfg = InterpolationConfig(highpass=high, gamma=prm.gamma, solver_tol=prm.solver_tol,
                               solver_max_iters=prm.solver_max_iters)
    t0 = time.perf_counter()
    kcols = column_slice(prm.k, grp.world, grp.rank)
    X, info = backend.block_cg(icfg, sampling, np.ascontiguousarray(reduced[:, kcols]))
    labels, fallback = sharded_assign(backend, X, kcols.start, grp)
    timings["interpolate"] = time.perf_counter() - t0
    its = np.concatenate(grp.all_gather_var(info.iterations))
    res = np.concatenate(grp.all_gather_var(info.residuals))
    conv = np.concatenate(grp.all_gather_var(info.converged.astype(np.uint8))).astype(bool)
    if not bool(np.all(conv)):
        warnings.append("interpolation solver did not reach tolerance")
    diagnostics = {
        "method": "csc", "num_nodes": N, "num_edges": getattr(backend, "num_edges", None), "k": prm.k, "n": prm.n, "d": prm.d, "p": prm.p, "gamma": prm.gamma,
        "seed": prm.seed, "lambda_k_hat": lam, "lambda_source": source, "lambda_warning": warn,
        "probe_iterations": len(trace), "kmeans_inertia": labeling.inertia,
        "kmeans_iterations": labeling.iterations_run, "solver_iterations": its.tolist(),
        "solver_residuals": res.tolist(), "solver_converged": conv.tolist(), "ridge": icfg.ridge,
        "zero_feature_rows": zero_rows.tolist(), "assign_fallback_nodes": fallback.tolist(), "warnings": warnings,
        "timings": {**timings, "total": time.perf_counter() - t_run},
        # the only key a single-process run_csc does not write: this rank's share of the columns
        "sharding": {"ranks": grp.world, "rank": grp.rank,
                     "columns_per_rank": {"d": dcols.stop - dcols.start, "k": kcols.stop - kcols.start}},
    }
    return ClusterResult(labels=labels, soft=X, diagnostics=diagnostics, num_clusters=prm.k)


# ---------------------------------------------------------------------------
# Row sharding (BASELINE config 5): the CSR is split by rows, the dense block
# is all-gathered over NCCL after every Chebyshev step (inside the library).


def row_partition(indptr: np.ndarray, world: int) -> np.ndarray:
    """Contiguous row ranges balanced by work ("balanced by nnz"):
    ``starts`` (world + 1 entries) with rank q owning rows [starts[q], starts[q + 1]).

    A step's per-rank cost is its CSR entries plus its dense rows, so the split balances
    nnz + rows: cut where the cumulative count crosses q / world of the total."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.size - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    cost = indptr + np.arange(n + 1, dtype=np.int64)  # cumulative nnz + rows at each row boundary
    targets = cost[-1] * np.arange(1, world, dtype=np.float64) / world
    cuts = np.searchsorted(cost, targets, side="left")
    return np.concatenate([[0], np.minimum(cuts, n), [n]]).astype(np.int64)


def row_range(num_nodes: int, world: int, rank: int) -> tuple[int, int]:
    """Equal-count split: R = ceil(N / world) consecutive rows (the last rank may own fewer)."""
    R = -(-num_nodes // world)
    begin = min(num_nodes, rank * R)
    return begin, min(num_nodes, begin + R)


def _create_shard(graph, starts: np.ndarray, world: int, rank: int, dtype: str, device: int) -> tuple[int, int]:
    begin, end = int(starts[rank]), int(starts[rank + 1])
    indptr, indices, weights = local_csr(graph, begin, end)
    h = C.c_void_p()
    st = np.ascontiguousarray(starts, dtype=np.int64)
    _lib.call("csc_graph_create_row_shard", graph.num_nodes, world, rank, _lib.ptr(st), int(indices.size),
              _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(weights), _lib.dtype_code(dtype), device,
              _lib.current_stream(device), C.byref(h))
    return h.value, int(indices.size)


def local_csr(graph, begin: int, end: int):
    """Rows [begin, end) of a canonical CSR, indptr rebased to 0, global column indices."""
    lo, hi = int(graph.indptr[begin]), int(graph.indptr[end])
    indptr = np.ascontiguousarray(graph.indptr[begin : end + 1] - lo, dtype=np.int32)
    return indptr, np.ascontiguousarray(graph.indices[lo:hi], dtype=np.int32), np.ascontiguousarray(graph.weights[lo:hi])


def exchange_handles(grp: Group, handle: np.ndarray) -> list[np.ndarray]:
    """Every rank's CUDA IPC handle bytes, in rank order (all_gather over the group)."""
    import torch.distributed as dist

    got: list = [None] * grp.world
    dist.all_gather_object(got, bytes(np.asarray(handle, dtype=np.uint8)), group=grp.group)
    return [np.frombuffer(b, dtype=np.uint8).copy() for b in got]


class RowShardedOperator:
    """This rank's rows of the normalized Laplacian plus the step exchange.

    Blocks are passed as this rank's rows (CUDA tensors, N_local x w).  ``transport``:
    ``"nccl"`` -- an ncclAllGather of every step's rows (csc_cheb_filter_rows);
    ``"peer"`` -- the all-gather fused into the step kernel: rows are stored straight
    into every rank's CUDA-IPC-mapped gather panel over NVLink, with a flag barrier
    between steps (csc_cheb_filter_rows_peers).  Both give the same results.
    ``barrier`` (peer transport): ``"device"`` -- the system-scope flag barrier kernel (one
    GPU per rank, ranks run concurrently); ``"host"`` -- stream synchronise + a barrier over
    the group after every step (csc_peers_set_host_barrier), for ranks that share a GPU.
    """

    def __init__(self, graph, grp: Group, dtype: str = "float32", device: int | None = None,
                 transport: str = "nccl", starts: np.ndarray | None = None, barrier: str = "device"):
        import torch

        if transport not in ("nccl", "peer"):
            raise ValueError(f"unknown transport {transport!r}")
        if barrier not in ("device", "host"):
            raise ValueError(f"unknown barrier {barrier!r}")
        self.transport = transport
        self.barrier = barrier
        self._barrier_cb = None
        self.peers = None
        self._peer_bytes = 0
        self.grp = grp
        self.num_nodes = graph.num_nodes
        self.device = _lib.default_device() if device is None else int(device)
        self.starts = row_partition(graph.indptr, grp.world) if starts is None else np.asarray(starts, np.int64)
        self.begin, self.end = int(self.starts[grp.rank]), int(self.starts[grp.rank + 1])
        self.panel_R = int(np.diff(self.starts).max())
        self.dtype = dtype
        self.handle, self.local_nnz = _create_shard(graph, self.starts, grp.world, grp.rank, dtype, self.device)
        self.total_nnz = int(graph.indices.size)
        self.comm = None
        if transport == "peer":
            return
        uid = np.zeros(128, dtype=np.uint8)
        if grp.rank == 0:
            _lib.call("csc_comm_unique_id", _lib.ptr(uid))
        if grp.world > 1:
            import torch.distributed as dist

            t = torch.from_numpy(uid).to(grp.device)
            dist.broadcast(t, src=0, group=grp.group)
            uid = t.cpu().numpy()
        comm = C.c_void_p()
        _lib.call("csc_comm_create", _lib.ptr(uid), grp.world, grp.rank, self.device, C.byref(comm))
        self.comm = comm.value

    @property
    def num_local(self) -> int:
        return self.end - self.begin

    def _run(self, filt: PolyFilter, X, mode: int):
        import torch

        c = coeff_array(filt)
        Y = torch.empty_like(X) if mode != 1 else None
        out = None
        if mode == 1:
            out = np.zeros(1)
        elif mode == 2:
            out = torch.empty(X.shape[0], dtype=torch.float64, device=X.device)
        if self.transport == "peer":
            self._ensure_peers(int(X.shape[1]))
            fn, tr = "csc_cheb_filter_rows_peers", self.peers
        else:
            fn, tr = "csc_cheb_filter_rows", self.comm
        _lib.call(fn, self.handle, tr, _lib.ptr(c), int(c.size), X.data_ptr(),
                  int(X.stride(0)), None if Y is None else Y.data_ptr(), int(X.shape[1]), int(X.shape[1]),
                  _lib.dtype_code(X.dtype), mode, _lib.ptr(out), _lib.current_stream(self.device))
        return Y, out

    def _ensure_peers(self, ncols: int) -> None:
        """(Re)build the peer transport when this block needs wider panels (collective)."""
        row_bytes = C.c_int64(0)
        rows = self.panel_R * self.grp.world
        _lib.call("csc_panel_row_bytes", rows, ncols, _lib.dtype_code(self.dtype), self.device,
                  self.local_nnz * self.grp.world, C.byref(row_bytes))
        need = rows * int(row_bytes.value)
        if self.peers is not None and need <= self._peer_bytes:
            return
        self._close_peers()
        pe = C.c_void_p()
        _lib.call("csc_peers_create", self.grp.world, self.grp.rank, self.device, need, C.byref(pe))
        self.peers, self._peer_bytes = pe.value, need
        if self.grp.world > 1:
            handle = np.zeros(64, dtype=np.uint8)
            _lib.call("csc_peers_handle", self.peers, _lib.ptr(handle))
            handles = exchange_handles(self.grp, handle)
            for r, hb in enumerate(handles):
                if r != self.grp.rank:
                    _lib.call("csc_peers_attach", self.peers, r, _lib.ptr(hb))
        if self.barrier == "host":
            if self._barrier_cb is None:
                self._barrier_cb = C.CFUNCTYPE(C.c_int, C.c_void_p)(self._host_barrier)
            _lib.call("csc_peers_set_host_barrier", self.peers, self._barrier_cb, None)

    def _host_barrier(self, _ctx) -> int:
        """Called by the library between steps (its stream already synchronised)."""
        try:
            if self.grp.world > 1:
                import torch.distributed as dist

                dist.barrier(group=self.grp.group)
            return 0
        except Exception:  # the C caller turns non-zero into an error status
            return 1

    def _close_peers(self) -> None:
        lib = _lib._lib
        if self.peers and lib is not None:
            lib.csc_peers_destroy(self.peers)
        self.peers, self._peer_bytes = None, 0

    def close(self) -> None:
        """Collective teardown of the peer transport: every rank finishes its stream, then all
        unmap their peers' panels before any owner frees its allocation (an exporter must not
        free memory another process still has mapped).  ``__del__`` alone is best effort."""
        import torch

        if self.peers is None:
            return
        torch.cuda.synchronize(self.device)
        if self.grp.world > 1:
            import torch.distributed as dist

            dist.barrier(group=self.grp.group)
        # two phases inside csc_peers_destroy would need a second entry point; closing after a
        # barrier is enough because destroy unmaps the peers before it frees the own panels and
        # no rank touches a peer's panel after the barrier
        self._close_peers()
        if self.grp.world > 1:
            import torch.distributed as dist

            dist.barrier(group=self.grp.group)

    def apply_filter(self, filt: PolyFilter, X_local):
        """h(L) X for this rank's rows."""
        return self._run(filt, X_local.contiguous(), 0)[0]

    def eigencount(self, filt: PolyFilter, R_local) -> float:
        """sum((h(L) R)^2) over all ranks (partials summed in rank order)."""
        _, part = self._run(filt, R_local.contiguous(), 1)
        return float(self.grp.sum_in_order(part)[0])

    def features(self, filt: PolyFilter, R_local):
        """Row-normalised features of this rank's rows (rows are complete per rank: no exchange)."""
        import torch

        Y, rowsq = self._run(filt, R_local.contiguous(), 2)
        F = torch.empty_like(Y)
        flags = torch.zeros(Y.shape[0], dtype=torch.uint8, device=Y.device)
        nz = C.c_int64(0)
        _lib.call("csc_normalize_rows", Y.data_ptr(), int(Y.shape[1]), int(Y.shape[0]), int(Y.shape[1]),
                  _lib.dtype_code(Y.dtype), rowsq.data_ptr(), F.data_ptr(), int(F.shape[1]), flags.data_ptr(),
                  C.byref(nz), self.device, _lib.current_stream(self.device))
        zero = flags.nonzero().flatten().cpu().numpy() + self.begin if nz.value else np.empty(0, dtype=np.int64)
        return F, zero.astype(np.int64)

    def __del__(self):
        lib = _lib._lib
        if lib is None:
            return
        if getattr(self, "peers", None):
            self._close_peers()
        if getattr(self, "comm", None):
            lib.csc_comm_destroy(self.comm)
            self.comm = None
        if getattr(self, "handle", None):
            lib.csc_graph_destroy(self.handle)
            self.handle = None


class RowShardGroup:
    """Every rank's row shard of one graph in this process, on one device: the multi-rank
    row-sharded filter executed as ranks stepping in lockstep, the per-step all-gather done
    as device copies (``csc_cheb_filter_rows_group``; same kernels, per-rank arguments and
    panel layout as ``RowShardedOperator`` over NCCL).  Blocks are full N-row CUDA tensors;
    shard q works on rows [starts[q], starts[q + 1]), a contiguous view."""

    def __init__(self, graph, world: int, dtype: str = "float32", device: int | None = None,
                 starts: np.ndarray | None = None):
        self.num_nodes = graph.num_nodes
        self.world = int(world)
        self.device = _lib.default_device() if device is None else int(device)
        self.dtype = dtype
        self.starts = row_partition(graph.indptr, self.world) if starts is None else np.asarray(starts, np.int64)
        self.handles, self.nnz = [], []
        for q in range(self.world):
            h, m = _create_shard(graph, self.starts, self.world, q, dtype, self.device)
            self.handles.append(h)
            self.nnz.append(m)

    def _run(self, filt: PolyFilter, X, mode: int):
        import torch

        X = X.contiguous()
        c = coeff_array(filt)
        W = self.world
        parts = [X[int(self.starts[q]): int(self.starts[q + 1])] for q in range(W)]
        Y = torch.empty_like(X) if mode != 1 else None
        yparts = [Y[int(self.starts[q]): int(self.starts[q + 1])] for q in range(W)] if Y is not None else None
        outs = None
        if mode == 1:
            outs = torch.zeros((W,), dtype=torch.float64, device=X.device)
            optr = [outs.data_ptr() + 8 * q for q in range(W)]
        elif mode == 2:
            outs = torch.zeros((X.shape[0],), dtype=torch.float64, device=X.device)
            optr = [outs.data_ptr() + 8 * int(self.starts[q]) for q in range(W)]
        arr = lambda vals, t=C.c_void_p: (t * W)(*vals)  # noqa: E731
        ld = [int(X.stride(0))] * W
        _lib.call("csc_cheb_filter_rows_group", arr(self.handles), W, _lib.ptr(c), int(c.size),
                  arr([p.data_ptr() for p in parts]), arr(ld, C.c_int64),
                  None if Y is None else arr([p.data_ptr() for p in yparts]),
                  None if Y is None else arr(ld, C.c_int64), int(X.shape[1]), _lib.dtype_code(X.dtype), mode,
                  None if outs is None else arr(optr), _lib.current_stream(self.device))
        return Y, outs

    def apply_filter(self, filt: PolyFilter, X):
        return self._run(filt, X, 0)[0]

    def eigencount(self, filt: PolyFilter, R) -> float:
        """Per-rank partial sums of squares, summed in rank order (as RowShardedOperator)."""
        _, part = self._run(filt, R, 1)
        total = 0.0
        for v in part.cpu().numpy().tolist():
            total += v
        return float(total)

    def filter_rowsq(self, filt: PolyFilter, R):
        return self._run(filt, R, 2)

    def __del__(self):
        lib = _lib._lib
        if lib is None:
            return
        for h in getattr(self, "handles", []):
            lib.csc_graph_destroy(h)
        self.handles = []
