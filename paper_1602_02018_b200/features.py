"""Random-signal node features: filtered signals, row-normalised on the GPU.

Drop-in for ``cscluster.features``.  ``generate_signals`` is the reference's
numpy draw (features.py:50-67).  ``build_features`` (features.py:70-93) runs the
low-pass filter and the row normalisation in one device call (K2 with the ROWSQ
epilogue + a normalising pass, ``csc_build_features``); zero rows
(norm <= 1e-300) are flagged and left zero as in the reference.
"""

from __future__ import annotations

import ctypes as C
import json
import logging
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any

import numpy as np

from . import _lib
from ._blocks import as_block
from ._signals import bernoulli_block, normal_block
from .filters import PolyFilter, coeff_array

logger = logging.getLogger(__name__)

ZERO_ROW_TOL = 1e-300  # features.py:23

__all__ = [
    "FeatureMatrix",
    "RandomSignals",
    "build_features",
    "generate_signals",
    "load_features",
    "pairwise_distance",
    "save_features",
]


@dataclass
class RandomSignals:
    matrix: np.ndarray
    distribution: str
    seed: Any

    @property
    def num_signals(self) -> int:
        return int(self.matrix.shape[1])


@dataclass
class FeatureMatrix:
    rows: Any  # numpy (N, d) fp64, or a CUDA tensor when built device-resident
    normalized: bool
    zero_rows: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    provenance: dict[str, Any] = field(default_factory=dict)


def generate_signals(num_nodes: int, num_signals: int, distribution: str = "gaussian", seed=0,
                     out: np.ndarray | None = None) -> RandomSignals:
    """N x d i.i.d. N(0, 1/d) or +-1/sqrt(d) signals from ``default_rng(seed)``.

    ``out`` (optional, gaussian only) receives the draw in place, e.g. a pinned buffer.
    """
    if num_signals < 1:
        raise ValueError("num_signals must be >= 1")
    if distribution not in ("gaussian", "bernoulli"):
        raise ValueError(f"unknown distribution {distribution!r}")
    rng = np.random.default_rng(seed)
    if distribution == "gaussian":
        matrix = normal_block(rng, num_nodes, num_signals, out)
    else:
        matrix = bernoulli_block(rng, num_nodes, num_signals)
    return RandomSignals(matrix=matrix, distribution=distribution, seed=seed if isinstance(seed, int) else None)


def _provenance(filt: PolyFilter, signals: RandomSignals) -> dict:
    return {
        "filter": {"cutoff": filt.cutoff, "order": filt.order, "damping": filt.damping, "kind": filt.kind},
        "distribution": signals.distribution,
        "seed": signals.seed,
    }


def features_into(op, filt: PolyFilter, matrix, out, *, zero_rows: bool = True) -> np.ndarray | None:
    """Filter + row-normalise ``matrix`` into ``out``; returns the zero-row indices.

    ``matrix``/``out`` are both host arrays (fp64) or both CUDA tensors of the
    same dtype.  Zero-row flags stay on the device for device outputs.  With
    ``zero_rows=False`` and device buffers the call does not synchronise with the
    host (the zero rows are still left zero) and returns None.
    """
    blk = as_block(matrix, op.num_nodes, "signals")
    ob = as_block(out, op.num_nodes, "features")
    if ob.data is not out and not (hasattr(out, "data_ptr") and ob.data.data_ptr() == out.data_ptr()):
        raise ValueError("features output must be a C-contiguous fp64 array or a CUDA tensor")
    if blk.code != ob.code:
        raise ValueError("signals and features must share a dtype")
    c = coeff_array(filt)
    if not zero_rows and ob.on_device:
        _lib.call(
            "csc_build_features", op.handle, _lib.ptr(c), int(c.size), blk.ptr, blk.ld, blk.ncols, blk.code, ob.ptr,
            ob.ld, None, None, _lib.current_stream(op.device),
        )
        return None
    if ob.on_device:
        import torch

        flags = torch.zeros(op.num_nodes, dtype=torch.uint8, device=out.device)
    else:
        flags = np.zeros(op.num_nodes, dtype=np.uint8)
    nz = C.c_int64(0)
    _lib.call(
        "csc_build_features", op.handle, _lib.ptr(c), int(c.size), blk.ptr, blk.ld, blk.ncols, blk.code, ob.ptr,
        ob.ld, _lib.ptr(flags), C.byref(nz), _lib.current_stream(op.device),
    )
    if not nz.value:
        return np.empty(0, dtype=np.int64)
    if ob.on_device:
        return flags.nonzero().flatten().cpu().numpy().astype(np.int64)
    return np.flatnonzero(flags)


def build_features(op, filt: PolyFilter, signals: RandomSignals, *, out: np.ndarray | None = None) -> FeatureMatrix:
    """Filter the signals and normalise each node's row (reference features.py:70-93).

    ``out`` optionally receives the rows (an N x d C-contiguous fp64 array, e.g. pinned memory).
    """
    if signals.num_signals == 1:
        logger.warning("single random signal: rank-1 embedding, distances are degenerate")
    rows = np.empty((op.num_nodes, signals.num_signals), dtype=np.float64) if out is None else out
    zero_rows = features_into(op, filt, signals.matrix, rows)
    if zero_rows.size:
        logger.warning("%d feature row(s) with zero norm (nodes %s ...)", zero_rows.size, zero_rows[:10].tolist())
    return FeatureMatrix(rows=rows, normalized=True, zero_rows=zero_rows, provenance=_provenance(filt, signals))


def pairwise_distance(features: FeatureMatrix, i: int, j: int) -> float:
    rows = features.rows
    return float(np.linalg.norm(np.asarray(rows[i]) - np.asarray(rows[j])))


def save_features(features: FeatureMatrix, path) -> None:
    """JSON header line + row-major fp64 payload (reference features.py:101-116)."""
    rows = np.ascontiguousarray(np.asarray(features.rows), dtype=np.float64)
    header = {
        "normalized": features.normalized,
        "num_nodes": int(rows.shape[0]),
        "num_signals": int(rows.shape[1]),
        "provenance": features.provenance,
        "zero_rows": np.asarray(features.zero_rows).tolist(),
    }
    with Path(path).open("wb") as fh:
        fh.write((json.dumps(header, sort_keys=True) + "\n").encode("utf-8"))
        fh.write(rows.tobytes())


def load_features(path) -> FeatureMatrix:
    with Path(path).open("rb") as fh:
        header = json.loads(fh.readline().decode("utf-8"))
        payload = np.frombuffer(fh.read(), dtype=np.float64)
    return FeatureMatrix(
        rows=payload.reshape(header["num_nodes"], header["num_signals"]).copy(),
        normalized=bool(header["normalized"]),
        zero_rows=np.asarray(header["zero_rows"], dtype=np.int64),
        provenance=header.get("provenance", {}),
    )
