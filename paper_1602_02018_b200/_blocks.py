"""N x w signal blocks at the C-ABI boundary.

The reference takes and returns fp64 numpy arrays (``np.asarray(x, float64)``,
graph.py:149, filters.py:143).  Here a block is either such a numpy array (host:
the library stages it) or a CUDA torch tensor (device: used in place), viewed as
row-major with a leading dimension.  Host inputs come back as fp64 numpy arrays;
device inputs come back as tensors of their own dtype on their own device.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def _is_torch(x) -> bool:
    return type(x).__module__.split(".")[0] == "torch"


class Block:
    def __init__(self, data, ncols: int, ld: int, code: int, on_device: bool, vector: bool):
        self.data = data
        self.ncols = ncols
        self.ld = ld
        self.code = code
        self.on_device = on_device
        self.vector = vector

    @property
    def ptr(self):
        return _lib.ptr(self.data)

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    def empty_like(self, ncols: int | None = None) -> "Block":
        w = self.ncols if ncols is None else ncols
        if self.on_device:
            import torch

            out = torch.empty((self.rows, w), dtype=self.data.dtype, device=self.data.device)
        else:
            out = np.empty((self.rows, w), dtype=np.float64)
        return Block(out, w, w, self.code, self.on_device, self.vector)


def as_block(x, num_nodes: int, what: str = "signal") -> Block:
    if _is_torch(x):
        import torch

        if not x.is_cuda:
            x = x.numpy()
        else:
            if x.dtype not in (torch.float64, torch.float32):
                x = x.to(torch.float64)
            vector = x.dim() == 1
            t = x.reshape(-1, 1) if vector else x
            if t.dim() != 2:
                raise ValueError(f"{what} must be a vector or an N-row matrix")
            if t.shape[0] != num_nodes:
                raise ValueError(f"{what} has {t.shape[0]} rows, graph has {num_nodes} nodes")
            if t.stride(1) != 1 or t.stride(0) < max(t.shape[1], 1):
                t = t.contiguous()
            return Block(t, int(t.shape[1]), int(max(t.stride(0), 1)), _lib.dtype_code(t.dtype), True, vector)
    a = np.asarray(x, dtype=np.float64)
    vector = a.ndim == 1
    m = a.reshape(-1, 1) if vector else a
    if m.ndim != 2:
        raise ValueError(f"{what} must be a vector or an N-row matrix")
    if m.shape[0] != num_nodes:
        raise ValueError(f"{what} has {m.shape[0]} rows, graph has {num_nodes} nodes")
    if m.strides[1] != 8 or m.strides[0] < 8 * max(m.shape[1], 1) or m.strides[0] % 8:
        m = np.ascontiguousarray(m)
    ld = max(m.strides[0] // 8, m.shape[1], 1)
    return Block(m, int(m.shape[1]), int(ld), _lib.CSC_F64, False, vector)


def from_block(out: Block, like=None):
    data = out.data
    if out.vector:
        return data.reshape(-1)
    return data
