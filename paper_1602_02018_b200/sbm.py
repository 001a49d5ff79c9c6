"""Synthetic stochastic-block-model inputs and the clustering quality metric.

Inputs, not hot path: this module only produces the
graphs the benchmarks and parity tests run on.  ``sbm_generate`` reproduces the
reference generator draw for draw (sbm.py:83-155: geometric gap skipping per
community pair in row-major pair order, strict-upper-triangle unpacking for
intra-community blocks), so for the same ``SbmConfig`` it yields the same
graph as the reference; the COO -> canonical CSR step then runs on the device
(K1).  ``dcsbm_generate`` is the degree-corrected variant BASELINE config 4
asks for, which the reference does not have.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .graph import DeviceGraph, Graph
from . import _lib

__all__ = [
    "SbmConfig",
    "adjusted_rand_index",
    "critical_epsilon",
    "dcsbm_generate",
    "sbm_edges",
    "sbm_edges_device",
    "sbm_generate",
]


@dataclass
class SbmConfig:
    num_nodes: int
    k: int
    avg_degree: float
    epsilon: float
    sizes: list[int] | None = None
    seed: int = 0

    def __post_init__(self) -> None:
        if not 0.0 <= self.epsilon <= 1.0:
            raise ValueError(f"epsilon must lie in [0, 1], got {self.epsilon}")
        if self.sizes is None:
            base, extra = divmod(self.num_nodes, self.k)
            self.sizes = [base + (1 if i < extra else 0) for i in range(self.k)]
        if len(self.sizes) != self.k:
            raise ValueError(f"{len(self.sizes)} sizes for k={self.k} communities")
        if any(s <= 0 for s in self.sizes):
            raise ValueError("community sizes must be positive")
        if sum(self.sizes) != self.num_nodes:
            raise ValueError(f"sizes sum to {sum(self.sizes)}, expected {self.num_nodes}")
        if not 0.0 < self.q1 <= 1.0:
            raise ValueError(f"derived q1={self.q1:.4g} outside (0, 1]; lower avg_degree or raise N")

    @property
    def q1(self) -> float:
        """Intra-community edge probability s k / (N (1 + eps (k - 1)))."""
        return self.avg_degree * self.k / (self.num_nodes * (1.0 + self.epsilon * (self.k - 1)))

    @property
    def q2(self) -> float:
        return self.epsilon * self.q1


def critical_epsilon(avg_degree: float, k: int) -> float:
    """Detectability threshold (s - sqrt s) / (s + sqrt s (k - 1))."""
    if avg_degree <= 1:
        raise ValueError("average degree must exceed 1")
    r = math.sqrt(avg_degree)
    return (avg_degree - r) / (avg_degree + r * (k - 1))


def _success_positions(cells: int, q: float, rng: np.random.Generator) -> np.ndarray:
    """Indices of the successes among ``cells`` Bernoulli(q) trials via geometric gaps.

    Batch sizing and the draw sequence match the reference (sbm.py:83-100) so the
    generator state advances identically.
    """
    if cells <= 0 or q <= 0.0:
        return np.empty(0, dtype=np.int64)
    if q >= 1.0:
        return np.arange(cells, dtype=np.int64)
    mean = q * cells
    batch = max(64, int(mean + 10.0 * math.sqrt(mean) + 10.0))
    chunks = []
    last = -1
    while last < cells:
        pos = last + np.cumsum(rng.geometric(q, size=batch))
        chunks.append(pos)
        last = int(pos[-1])
    pos = np.concatenate(chunks)
    return pos[pos < cells]


def _unpack_lower(t: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """t = i(i-1)/2 + j with 0 <= j < i  ->  (i, j), exact for int64 t."""
    i = ((1.0 + np.sqrt(1.0 + 8.0 * t.astype(np.float64))) / 2.0).astype(np.int64)
    i = np.where(i * (i - 1) // 2 > t, i - 1, i)
    i = np.where(i * (i - 1) // 2 + i <= t, i + 1, i)
    return i, t - i * (i - 1) // 2


def sbm_edges(cfg: SbmConfig) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Undirected edge list (each pair once) and ground-truth labels."""
    rng = np.random.default_rng(cfg.seed)
    sizes = np.asarray(cfg.sizes, dtype=np.int64)
    first = np.concatenate([[0], np.cumsum(sizes)])
    src: list[np.ndarray] = []
    dst: list[np.ndarray] = []
    for a in range(cfg.k):
        for b in range(a, cfg.k):
            if a == b:
                pos = _success_positions(int(sizes[a]) * (int(sizes[a]) - 1) // 2, cfg.q1, rng)
                if pos.size:
                    i, j = _unpack_lower(pos)
                    src.append(first[a] + i)
                    dst.append(first[a] + j)
            else:
                pos = _success_positions(int(sizes[a]) * int(sizes[b]), cfg.q2, rng)
                if pos.size:
                    src.append(first[a] + pos // sizes[b])
                    dst.append(first[b] + pos % sizes[b])
    labels = np.repeat(np.arange(cfg.k), sizes)
    if not src:
        return np.empty(0, np.int64), np.empty(0, np.int64), labels
    return np.concatenate(src), np.concatenate(dst), labels


def _device_build(src, dst, num_nodes: int, device: int | None) -> Graph:
    dev = _lib.default_device() if device is None else int(device)
    dg = DeviceGraph.from_edges(src, dst, None, num_nodes, "error", _lib.CSC_F64, dev)
    graph, _ = Graph._from_device(dg)
    return graph


def _sbm_pairs(cfg: SbmConfig):
    """Per community pair (a <= b, the reference's loop order, sbm.py:133-145) the
    quantities of _success_positions: cells, q and the batch size, for the pairs that
    contribute (cells > 0, q > 0); ``search`` is set when one of them has q >= 1/3."""
    sizes = np.asarray(cfg.sizes, dtype=np.int64)
    first = np.concatenate([[0], np.cumsum(sizes)])
    a, b = np.triu_indices(cfg.k)
    diag = a == b
    cells = np.where(diag, sizes[a] * (sizes[a] - 1) // 2, sizes[a] * sizes[b])
    q = np.where(diag, cfg.q1, cfg.q2)
    live = (cells > 0) & (q > 0.0)  # pairs that contribute edges (q >= 1: all cells, no draws)
    search = bool(np.any(live & (q >= 1.0 / 3.0)))
    a, b, diag, cells, q = a[live], b[live], diag[live], cells[live], q[live]
    mean = q * cells.astype(np.float64)
    batch = np.maximum(64, (mean + 10.0 * np.sqrt(mean) + 10.0).astype(np.int64))
    return a, b, diag, cells, q, batch, first, sizes, search


def sbm_edges_device(cfg: SbmConfig, device: int | None = None):
    """``sbm_edges`` on the device (csc_sbm_edges): the same edges in the same order as
    int64 CUDA tensors, plus the labels; ``None`` when a pair probability is >= 1/3
    (numpy's search branch, left to the host) or numpy's tables are unavailable."""
    import torch

    from ._npzig import exponential_tables, pcg_state

    dev = _lib.default_device() if device is None else int(device)
    a, b, diag, cells, q, batch, first, sizes, search = _sbm_pairs(cfg)
    labels = np.repeat(np.arange(cfg.k), sizes)
    if search:
        return None
    try:
        ke, we, fe = exponential_tables()
    except RuntimeError:
        return None
    _lib.call("csc_set_exponential_tables", _lib.ptr(ke), _lib.ptr(we), _lib.ptr(fe))
    st, inc = pcg_state(np.random.default_rng(cfg.seed))
    l1mq = np.array([math.log1p(-float(x)) for x in (cfg.q1, cfg.q2)])[np.where(diag, 0, 1)]
    cap = int(batch.sum())
    tdev = torch.device("cuda", dev)
    src = torch.empty(max(cap, 1), dtype=torch.int64, device=tdev)
    dst = torch.empty(max(cap, 1), dtype=torch.int64, device=tdev)
    n_e, raws = C.c_int64(0), C.c_int64(0)
    m = _MASK64
    pairs = [np.ascontiguousarray(x) for x in (cells.astype(np.int64), l1mq, batch.astype(np.int64),
                                               diag.astype(np.int32), first[a].astype(np.int64),
                                               first[b].astype(np.int64), sizes[b].astype(np.int64))]
    _lib.call("csc_sbm_edges", st >> 64, st & m, inc >> 64, inc & m, int(a.size), *[_lib.ptr(x) for x in pairs],
              cap, src.data_ptr(), dst.data_ptr(), C.byref(n_e), C.byref(raws), dev, _lib.current_stream(dev))
    return src[: n_e.value], dst[: n_e.value], labels


_MASK64 = (1 << 64) - 1


def sbm_generate(cfg: SbmConfig, *, device: int | None = None) -> tuple[Graph, np.ndarray]:
    """SBM graph (unit weights, nodes ordered by community) and its labels (reference sbm.py:118-155).

    The edges are drawn on the device when every pair probability is below 1/3
    (``sbm_edges_device``; bit-identical to the host restatement ``sbm_edges``)."""
    out = sbm_edges_device(cfg, device)
    if out is None:
        src, dst, labels = sbm_edges(cfg)
    else:
        src, dst, labels = out
    return _device_build(src, dst, cfg.num_nodes, device), labels


def dcsbm_edges(cfg: SbmConfig, pareto_alpha: float = 2.5) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """Degree-corrected SBM edges (BASELINE config 4; not in the reference).

    SURVEY.md section 8(d)'s spec: propensities theta_i = 1 + Pareto(alpha) (classical
    Pareto, x_m = 1, ``rng.pareto`` of ``default_rng(cfg.seed)``), normalised to mean 1
    within each community; independent Bernoulli edges with
    P(i~j) = min(1, theta_i theta_j q_{c_i c_j}), q = cfg.q1 inside a community and
    cfg.q2 across (the SbmConfig formulas, sbm.py:60-61), so E[deg_i] ~= theta_i *
    avg_degree.  The edges are drawn natively (``csc_dcsbm_edges``: rejection over
    geometric skipping, expected O(N + #E)) from a seed taken from the same generator.
    Returns (src, dst) sorted with src < dst, the community labels and theta.
    """
    rng = np.random.default_rng(cfg.seed)
    sizes = np.asarray(cfg.sizes, dtype=np.int64)
    first = np.concatenate([[0], np.cumsum(sizes)])
    comm = np.repeat(np.arange(cfg.k), sizes)
    theta = 1.0 + rng.pareto(pareto_alpha, size=cfg.num_nodes)
    sums = np.add.reduceat(theta, first[:-1])
    theta = np.ascontiguousarray(theta / (sums / sizes)[comm])
    seed = int(rng.integers(0, 2**63 - 1))
    n_e = C.c_int64(0)
    cap = int(cfg.num_nodes * cfg.avg_degree / 2 * 1.1) + 1024
    for _ in range(2):
        src = np.empty(cap, dtype=np.int64)
        dst = np.empty(cap, dtype=np.int64)
        _lib.call("csc_dcsbm_edges", int(cfg.num_nodes), int(cfg.k), _lib.ptr(sizes), _lib.ptr(theta),
                  C.c_double(cfg.q1), C.c_double(cfg.q2), C.c_uint64(seed), 0, C.c_int64(cap), _lib.ptr(src), _lib.ptr(dst), C.byref(n_e))
        if n_e.value <= cap:
            break
        cap = int(n_e.value)
    m = int(n_e.value)
    order = np.lexsort((dst[:m], src[:m]))
    return src[:m][order], dst[:m][order], comm, theta


def c4_config(seed: int = 0) -> SbmConfig:
    """BASELINE config 4: N=334,863, k=250, mean degree 5.5, eps = eps_c(5.5, 250)/4."""
    return SbmConfig(num_nodes=334_863, k=250, avg_degree=5.5, epsilon=critical_epsilon(5.5, 250) / 4.0, seed=seed)


def dcsbm_generate(cfg: SbmConfig, pareto_alpha: float = 2.5, *, device: int | None = None):
    """Degree-corrected SBM graph, labels and propensities (see ``dcsbm_edges``)."""
    src, dst, labels, theta = dcsbm_edges(cfg, pareto_alpha)
    return _device_build(src, dst, cfg.num_nodes, device), labels, theta


def adjusted_rand_index(labels_a: Sequence[int], labels_b: Sequence[int]) -> float:
    """Hubert-Arabie ARI from the contingency table (reference sbm.py:158-185)."""
    a = np.asarray(labels_a)
    b = np.asarray(labels_b)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError("label vectors must be 1-d and of equal length")
    n = a.size
    if n < 2:
        return 1.0
    _, ai = np.unique(a, return_inverse=True)
    _, bi = np.unique(b, return_inverse=True)
    nb = int(bi.max()) + 1
    joint = np.bincount(ai * nb + bi, minlength=(int(ai.max()) + 1) * nb).astype(np.float64)
    pairs = lambda x: float(np.sum(x * (x - 1.0))) / 2.0  # noqa: E731
    s_ij = pairs(joint)
    s_a = pairs(np.bincount(ai).astype(np.float64))
    s_b = pairs(np.bincount(bi).astype(np.float64))
    expected = s_a * s_b / pairs(float(n))
    top = 0.5 * (s_a + s_b)
    if top == expected:
        return 1.0
    return (s_ij - expected) / (top - expected)
