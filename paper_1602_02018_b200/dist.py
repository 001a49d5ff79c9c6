"""Column-sharded execution over ranks (one process per GPU, torch.distributed).

Every hot-path stage is column-separable (filters.py:140 acts columnwise,
spectrum.py:86 sums over columns, sampling.py:133-135 is per-column CG), so the
graph is replicated and ranks own contiguous slices of the signal / indicator
columns.  The only exchanges are small:

  eigencount   per-rank partial counts, all-gathered and summed in rank order
  features     per-rank row sums of squares (N fp64), all-gathered and summed
               in rank order, then each rank normalises its own columns
  gather       the n sampled rows of each rank's columns, all-gathered
  assign       per-row (best value, global column) pairs, all-gathered and
               merged with the reference's lowest-index tie rule

Sums are taken in rank order on every rank, so results do not depend on the
collective's internal reduction order.  The per-rank compute goes through a
backend object (``DeviceBackend`` = the C ABI on this rank's GPU); tests swap in
a CPU backend to exercise the exchange logic with the gloo backend.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .filters import PolyFilter, coeff_array


def column_slice(ncols: int, world: int, rank: int) -> slice:
    """Contiguous balanced split of ``ncols`` columns: the first ncols % world ranks get one extra."""
    base, extra = divmod(ncols, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))


class DeviceBackend:
    """Per-rank compute on the rank's GPU through the C ABI (inputs/outputs are CUDA tensors)."""

    def __init__(self, op):
        self.op = op

    def filter_rowsq(self, filt: PolyFilter, R):
        import torch

        c = coeff_array(filt)
        Y = torch.empty_like(R)
        rowsq = torch.empty(R.shape[0], dtype=torch.float64, device=R.device)
        _lib.call("csc_filter_rowsq", self.op.handle, _lib.ptr(c), int(c.size), R.data_ptr(), int(R.stride(0)),
                  int(R.shape[1]), _lib.dtype_code(R.dtype), Y.data_ptr(), int(Y.stride(0)), rowsq.data_ptr(),
                  _lib.current_stream(self.op.device))
        return Y, rowsq

    def normalize(self, Y, rowsq):
        import torch

        F = torch.empty_like(Y)
        flags = torch.zeros(Y.shape[0], dtype=torch.uint8, device=Y.device)
        nz = C.c_int64(0)
        _lib.call("csc_normalize_rows", Y.data_ptr(), int(Y.stride(0)), int(Y.shape[0]), int(Y.shape[1]),
                  _lib.dtype_code(Y.dtype), rowsq.data_ptr(), F.data_ptr(), int(F.stride(0)), flags.data_ptr(),
                  C.byref(nz), self.op.device, _lib.current_stream(self.op.device))
        zero = torch.nonzero(flags).flatten().cpu().numpy() if nz.value else np.empty(0, dtype=np.int64)
        return F, zero

    def count(self, filt: PolyFilter, R) -> float:
        c = coeff_array(filt)
        out = C.c_double(0.0)
        _lib.call("csc_eigencount", self.op.handle, _lib.ptr(c), int(c.size), R.data_ptr(), int(R.stride(0)),
                  int(R.shape[1]), _lib.dtype_code(R.dtype), C.byref(out), _lib.current_stream(self.op.device))
        return float(out.value)

    def zeros(self, n, dtype="float64"):
        import torch

        return torch.zeros(n, dtype=getattr(torch, dtype), device=f"cuda:{self.op.device}")


@dataclass
class Group:
    """The torch.distributed group plus this rank's position."""

    rank: int
    world: int
    group: object = None

    @classmethod
    def current(cls, group=None) -> "Group":
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized():
            return cls(0, 1, None)
        return cls(dist.get_rank(group), dist.get_world_size(group), group)

    def gather_sum(self, x):
        """Sum of ``x`` (tensor) over ranks, accumulated in rank order (deterministic)."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return x
        parts = [torch.empty_like(x) for _ in range(self.world)]
        dist.all_gather(parts, x.contiguous(), group=self.group)
        total = parts[0].clone()
        for p in parts[1:]:
            total += p
        return total

    def all_gather(self, x):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return [x]
        parts = [torch.empty_like(x) for _ in range(self.world)]
        dist.all_gather(parts, x.contiguous(), group=self.group)
        return parts


def sharded_features(backend, filt: PolyFilter, R_local, grp: Group):
    """Features for this rank's signal columns, normalised by the global row norms."""
    Y, rowsq = backend.filter_rowsq(filt, R_local)
    total = grp.gather_sum(rowsq)
    return backend.normalize(Y, total)


def sharded_count(backend, filt: PolyFilter, R_local, grp: Group) -> float:
    """Eigencount over all ranks' probe columns (spectrum.py:86)."""
    import torch

    local = backend.count(filt, R_local)
    t = torch.tensor([local], dtype=torch.float64, device=getattr(R_local, "device", "cpu"))
    return float(grp.gather_sum(t).item())


def merge_argmax(values: np.ndarray, columns: np.ndarray) -> np.ndarray:
    """Per-row winner over rank candidates (ranks x N): larger value, ties -> lower column."""
    best_v = values[0].copy()
    best_c = columns[0].copy()
    for v, c in zip(values[1:], columns[1:]):
        take = (v > best_v) | ((v == best_v) & (c < best_c))
        best_v = np.where(take, v, best_v)
        best_c = np.where(take, c, best_c)
    return best_c
