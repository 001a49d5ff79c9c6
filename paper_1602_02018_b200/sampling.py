"""Uniform sampling, device block-CG interpolation and device argmax assignment.

Drop-in for ``cscluster.sampling``.  Sampling stays a host numpy draw so the
indices are bit-exact (sampling.py:64-88).  The regularised interpolation
(sampling.py:119-180) runs entirely on the GPU (``csc_block_cg``): the system
operator ``M^T M + gamma (g(L) + ridge I)`` is one high-pass filter pass whose
last step fuses the mask/ridge/gamma terms and the CG dot products.  ``assign``
(sampling.py:197-220) is a device argmax (``csc_assign``).
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._blocks import as_block, from_block
from .filters import PolyFilter, coeff_array, psd_ridge
from .result import ClusterResult

logger = logging.getLogger(__name__)

__all__ = [
    "SamplingSet",
    "InterpolationConfig",
    "CgInfo",
    "ClusterResult",
    "draw_sampling",
    "interpolate",
    "interpolate_all",
    "assign",
]


@dataclass
class SamplingSet:
    """Ordered distinct node indices: (M x)_i = x[indices[i]] (sampling.py:40-61)."""

    indices: np.ndarray
    num_nodes: int

    @property
    def size(self) -> int:
        return int(self.indices.size)

    def restrict(self, x):
        return x[self.indices]

    def adjoint(self, y) -> np.ndarray:
        out = np.zeros((self.num_nodes,) + np.shape(y)[1:], dtype=np.float64)
        out[self.indices] = y
        return out


def draw_sampling(num_nodes: int, n: int, seed, *, exclude: np.ndarray | None = None) -> SamplingSet:
    """n distinct nodes uniformly without replacement, optionally excluding some (sampling.py:64-88)."""
    rng = np.random.default_rng(seed)
    eligible = None
    if exclude is not None and len(exclude):
        eligible = np.setdiff1d(np.arange(num_nodes), np.asarray(exclude, dtype=np.int64))
    pool = num_nodes if eligible is None else eligible.size
    if not 1 <= n <= pool:
        raise ValueError(f"cannot draw n={n} from {pool} eligible nodes")
    if eligible is None:
        picked = rng.choice(num_nodes, size=n, replace=False)
    else:
        picked = eligible[rng.choice(pool, size=n, replace=False)]
    return SamplingSet(indices=picked.astype(np.int64), num_nodes=num_nodes)


@dataclass
class InterpolationConfig:
    highpass: PolyFilter
    gamma: float = 1e-3
    solver_tol: float = 1e-6
    solver_max_iters: int = 1000
    ridge: float | None = None

    def __post_init__(self) -> None:
        if self.gamma <= 0:
            raise ValueError("gamma must be positive")
        if self.ridge is None:
            self.ridge = psd_ridge(self.highpass)


@dataclass
class CgInfo:
    iterations: np.ndarray
    residuals: np.ndarray
    converged: np.ndarray

    @property
    def max_iterations(self) -> int:
        return int(self.iterations.max(initial=0))


def _system_apply(op, cfg: InterpolationConfig, mask, X):
    """``mask * X + gamma * (g(L) X + ridge * X)`` on the GPU (sampling.py:119-121).

    ``mask`` is the 0/1 sampling mask (nonzero entries count as sampled).
    """
    blk = as_block(X, op.num_nodes, "signal")
    m = np.ascontiguousarray(np.asarray(mask) != 0, dtype=np.uint8)
    c = coeff_array(cfg.highpass)
    out = blk.empty_like()
    _lib.call(
        "csc_system_apply", op.handle, _lib.ptr(c), int(c.size), float(cfg.gamma), float(cfg.ridge), _lib.ptr(m),
        blk.ptr, blk.ld, out.ptr, out.ld, blk.ncols, blk.code, _lib.current_stream(op.device),
    )
    return from_block(out)


def block_cg_into(op, cfg: InterpolationConfig, sampling: SamplingSet, reduced: np.ndarray, out) -> CgInfo:
    """Run the device block CG writing X into ``out`` (numpy fp64 or CUDA tensor, N x k)."""
    reduced = np.ascontiguousarray(reduced, dtype=np.float64)
    n, k = reduced.shape
    idx = np.ascontiguousarray(sampling.indices, dtype=np.int64)
    c = coeff_array(cfg.highpass)
    its = np.zeros(k, dtype=np.int64)
    res = np.zeros(k, dtype=np.float64)
    conv = np.zeros(k, dtype=np.uint8)
    run = C.c_int64(0)
    if hasattr(out, "data_ptr"):
        optr, ld, code = out.data_ptr(), int(out.stride(0)), _lib.dtype_code(out.dtype)
    else:
        optr, ld, code = _lib.ptr(out), int(out.strides[0] // 8), _lib.CSC_F64
    _lib.call(
        "csc_block_cg", op.handle, _lib.ptr(c), int(c.size), float(cfg.gamma), float(cfg.ridge), _lib.ptr(idx),
        int(n), _lib.ptr(reduced), int(k), float(cfg.solver_tol), int(cfg.solver_max_iters), optr, ld, code,
        _lib.ptr(its), _lib.ptr(res), _lib.ptr(conv), C.byref(run), _lib.current_stream(op.device),
    )
    active = conv == 0
    if active.any():
        logger.warning(
            "interpolation CG did not converge for %d of %d classes within %d iterations",
            int(active.sum()), k, cfg.solver_max_iters,
        )
    return CgInfo(iterations=its, residuals=res, converged=conv.astype(bool))


def interpolate_all(op, cfg: InterpolationConfig, sampling: SamplingSet, reduced: np.ndarray):
    """Solve the k interpolation problems as one blocked CG run (reference sampling.py:124-180)."""
    reduced = np.asarray(reduced, dtype=np.float64)
    n, k = reduced.shape
    if n != sampling.size:
        raise ValueError(f"reduced indicators have {n} rows, sampling has {sampling.size}")
    X = np.empty((op.num_nodes, k), dtype=np.float64)
    info = block_cg_into(op, cfg, sampling, reduced, X)
    return X, info


def interpolate(op, cfg: InterpolationConfig, sampling: SamplingSet, reduced: np.ndarray):
    reduced = np.asarray(reduced, dtype=np.float64)
    if reduced.ndim != 1:
        raise ValueError("interpolate expects a single reduced vector; use interpolate_all for blocks")
    X, info = interpolate_all(op, cfg, sampling, reduced[:, None])
    return X[:, 0], info


def assign(soft, *, return_info: bool = False, device: int | None = None):
    """Hard labels = argmax_j soft_ij / ||soft_:j|| on the GPU (reference sampling.py:197-220)."""
    is_dev = hasattr(soft, "is_cuda") and soft.is_cuda
    if is_dev:
        if soft.dim() != 2:
            raise ValueError("soft indicators must be (N, k)")
        s = soft if soft.stride(1) == 1 else soft.contiguous()
        N, k = int(s.shape[0]), int(s.shape[1])
        sptr, ld, code, dev = s.data_ptr(), int(max(s.stride(0), 1)), _lib.dtype_code(s.dtype), s.device.index
    else:
        s = np.asarray(soft, dtype=np.float64)
        if s.ndim != 2:
            raise ValueError("soft indicators must be (N, k)")
        s = np.ascontiguousarray(s)
        N, k = s.shape
        sptr, ld, code = _lib.ptr(s), int(max(k, 1)), _lib.CSC_F64
        dev = _lib.default_device() if device is None else int(device)
    if N == 0 or k == 0:
        raise ValueError("all indicator vectors are zero")
    labels = np.empty(N, dtype=np.int64)
    fb = np.zeros(N, dtype=np.uint8)
    nfb = C.c_int64(0)
    _lib.call("csc_assign", sptr, ld, N, k, code, _lib.ptr(labels), _lib.ptr(fb), C.byref(nfb), dev,
              _lib.current_stream(dev))
    fallback = np.flatnonzero(fb) if nfb.value else np.empty(0, dtype=np.int64)
    if fallback.size:
        logger.warning("%d node(s) with all-zero indicators assigned by raw argmax: %s ...", fallback.size,
                       fallback[:10].tolist())
    if return_info:
        return labels, {"fallback_nodes": fallback}
    return labels
