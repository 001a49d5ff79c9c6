"""Host-side random signal blocks, drawn by numpy exactly as the reference draws them.

Parity requires the reference's seeded numpy streams, so
signals are generated on the host.  Two things make that cheaper without
changing a single value:

- blocks are written into page-locked (pinned) buffers with
  ``rng.standard_normal(out=...)`` and scaled in place, so the device copy runs
  at full PCIe/C2C rate and no temporary is allocated;
- ``ProbeStream`` draws the next eigencount probe block on a worker thread while
  the GPU filters the current one.  The probe stream is lambda-independent
  (spectrum.py:84), so the i-th block is the same whatever the dichotomy does.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """numpy array in page-locked memory when a CUDA torch is available, else plain."""
    try:
        import torch

        if torch.cuda.is_available():
            t = torch.empty(tuple(int(s) for s in shape), dtype=torch.float64 if np.dtype(dtype) == np.float64
                            else torch.float32, pin_memory=True)
            return t.numpy()  # the array's base keeps the pinned tensor alive
    except Exception:
        pass
    return np.empty(shape, dtype=dtype)


def normal_block(rng: np.random.Generator, n: int, w: int, out: np.ndarray | None = None) -> np.ndarray:
    """``rng.standard_normal((n, w)) / sqrt(w)`` (spectrum.py:84, features.py:63), in place."""
    if out is None:
        out = np.empty((n, w), dtype=np.float64)
    rng.standard_normal(out=out)
    out /= np.sqrt(w)
    return out


def bernoulli_block(rng: np.random.Generator, n: int, w: int) -> np.ndarray:
    """``(2 * rng.integers(0, 2, (n, w)) - 1) / sqrt(w)`` (features.py:65)."""
    return (2.0 * rng.integers(0, 2, size=(n, w)) - 1.0) / np.sqrt(w)


class ProbeStream:
    """Sequential N x ds probe blocks from one generator, one block drawn ahead.

    Only for generators private to the caller (run_csc's "probe" substream):
    drawing ahead advances the generator by one extra block.
    """

    def __init__(self, rng: np.random.Generator, n: int, ds: int, pinned_buffers: bool = True):
        self.rng, self.n, self.ds = rng, n, ds
        mk = pinned_empty if pinned_buffers else (lambda s: np.empty(s))
        self._bufs = [mk((n, ds)), mk((n, ds))]
        self._i = 0
        self._pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="csc-probe-rng")
        self._next = self._pool.submit(normal_block, rng, n, ds, self._bufs[0])

    def take(self) -> np.ndarray:
        block = self._next.result()
        self._i += 1
        self._next = self._pool.submit(normal_block, self.rng, self.n, self.ds, self._bufs[self._i % 2])
        return block

    def close(self) -> None:
        try:
            self._next.result()
        finally:
            self._pool.shutdown(wait=True)


# ---------------------------------------------------------------------------
# device parity RNG (numpy's PCG64 + ziggurat reproduced bit for bit, csc_numpy_normals)

_tables_loaded = False


def device_rng_available() -> bool:
    """True when numpy's ziggurat tables could be read and verified (see _npzig)."""
    global _tables_loaded
    if _tables_loaded:
        return True
    try:
        from . import _lib
        from ._npzig import ziggurat_tables

        ki, wi, fi = ziggurat_tables()
        _lib.call("csc_set_normal_tables", _lib.ptr(ki), _lib.ptr(wi), _lib.ptr(fi))
        _tables_loaded = True
    except Exception:
        _tables_loaded = False
    return _tables_loaded


def device_normal_block(rng: np.random.Generator, n: int, w: int, device: int = 0, out=None, stream=None):
    """``rng.standard_normal((n, w)) / sqrt(w)`` drawn on the GPU into a CUDA fp64 tensor,
    bit-identical to numpy; ``rng`` is advanced exactly as the host draw would advance it.
    ``stream``: a torch.cuda.Stream to run on (default: the current stream)."""
    import ctypes as C

    import torch

    from . import _lib
    from ._npzig import pcg_state

    if not device_rng_available():
        raise RuntimeError("device parity RNG unavailable (numpy ziggurat tables not found)")
    state, inc = pcg_state(rng)
    if out is None:
        out = torch.empty((n, w), dtype=torch.float64, device=f"cuda:{device}")
    consumed = C.c_int64(0)
    divisor = float(np.sqrt(w))
    _lib.call("csc_numpy_normals", C.c_uint64(state >> 64), C.c_uint64(state & ((1 << 64) - 1)),
              C.c_uint64(inc >> 64), C.c_uint64(inc & ((1 << 64) - 1)), int(n) * int(w), divisor, out.data_ptr(),
              C.byref(consumed), int(device), stream.cuda_stream if stream is not None else _lib.current_stream(device))
    # advance() also clears PCG64's buffered 32-bit half; the host standard_normal draw
    # leaves it alone, so carry it over
    buffered = rng.bit_generator.state
    rng.bit_generator.advance(int(consumed.value))
    if buffered["has_uint32"]:
        st = rng.bit_generator.state
        st["has_uint32"], st["uinteger"] = buffered["has_uint32"], buffered["uinteger"]
        rng.bit_generator.state = st
    return out


class DeviceProbeStream:
    """Sequential probe blocks drawn on the GPU (same values as ProbeStream), ``depth``
    blocks ahead: a worker thread draws blocks t + 1 .. t + depth in order on its own
    CUDA stream (kernels + the host walk of the rare slow paths) while the caller
    filters block t.  A draw takes about as long as a probe's filter, so one block of
    lookahead stalls whenever a draw runs late; the generator is private to the caller
    (run_csc's "probe" substream), so drawing blocks that end up unused changes nothing."""

    def __init__(self, rng: np.random.Generator, n: int, ds: int, device: int, depth: int = 2):
        import torch

        self.rng, self.n, self.ds, self.device = rng, n, ds, device
        self.depth = max(1, int(depth))
        self.side = torch.cuda.Stream(device=device)
        self.bufs = [torch.empty((n, ds), dtype=torch.float64, device=f"cuda:{device}")
                     for _ in range(self.depth + 1)]
        self.i = 0
        self.pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="csc-probe-devrng")
        self.pending = [self.pool.submit(self._draw, k) for k in range(self.depth)]

    def _draw(self, slot: int):
        return device_normal_block(self.rng, self.n, self.ds, self.device, self.bufs[slot], self.side)

    def take(self):
        block = self.pending.pop(0).result()  # drawn and synchronised on the side stream
        # the slot of block i - 1 is free again: the caller's use of it has finished
        # (eigencount returns after a sync)
        self.pending.append(self.pool.submit(self._draw, (self.i + self.depth) % (self.depth + 1)))
        self.i += 1
        return block

    def close(self) -> None:
        try:
            for f in self.pending:
                f.result()
        finally:
            self.pool.shutdown(wait=True)
