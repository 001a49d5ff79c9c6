"""Named per-stage random streams from one master seed (reference _rng.py).

The (seed, stage) -> SeedSequence mapping must be the reference's so every
random draw on the hot path (probe, signals, sampling, kmeans) is bit-identical:
entropy = (seed,) + the first 16 bytes of sha256(stage) as 4 little-endian u32.
"""

from __future__ import annotations

import hashlib

import numpy as np


def _stage_words(stage: str) -> tuple[int, ...]:
    d = hashlib.sha256(stage.encode("utf-8")).digest()[:16]
    return tuple(int.from_bytes(d[o : o + 4], "little") for o in (0, 4, 8, 12))


def _seed_sequence(seed: int, stage: str) -> np.random.SeedSequence:
    return np.random.SeedSequence((int(seed),) + _stage_words(stage))


def substream(seed: int, stage: str) -> np.random.Generator:
    return np.random.default_rng(_seed_sequence(seed, stage))


def substream_seed(seed: int, stage: str) -> int:
    """Integer seed derived from the same sequence (state[0] ^ (state[1] >> 1))."""
    lo, hi = _seed_sequence(seed, stage).generate_state(2, dtype=np.uint64)
    return int(lo ^ (hi >> np.uint64(1)))
