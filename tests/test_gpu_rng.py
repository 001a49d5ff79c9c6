"""Device parity RNG: numpy's Generator(PCG64).standard_normal reproduced bit for bit on the GPU."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1602_02018_b200._rng import substream
from paper_1602_02018_b200._signals import device_normal_block, device_rng_available

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,w", [(1, 1), (3, 5), (1000, 7), (100_000, 28), (1_000_000, 28)])
def test_device_normals_bit_exact(n, w):
    assert device_rng_available()
    for seed in (0, 1, 20160219):
        a, b = np.random.default_rng(seed), np.random.default_rng(seed)
        ref = b.standard_normal((n, w)) / np.sqrt(w)
        got = device_normal_block(a, n, w).cpu().numpy()
        assert np.array_equal(got, ref)
        assert a.bit_generator.state == b.bit_generator.state  # same stream position afterwards
        assert a.standard_normal() == b.standard_normal()


def test_device_normals_keep_buffered_uint32():
    """A generator holding a pending 32-bit half (after a 32-bit integers draw) keeps it."""
    a, b = np.random.default_rng(5), np.random.default_rng(5)
    a.integers(0, 1000, dtype=np.uint32)
    b.integers(0, 1000, dtype=np.uint32)
    assert a.bit_generator.state["has_uint32"] == 1
    got = device_normal_block(a, 1000, 3).cpu().numpy()
    assert np.array_equal(got, b.standard_normal((1000, 3)) / np.sqrt(3))
    assert a.bit_generator.state == b.bit_generator.state
    assert a.integers(0, 1000, 5, dtype=np.uint32).tolist() == b.integers(0, 1000, 5, dtype=np.uint32).tolist()


def test_device_normals_continue_the_stream():
    """Consecutive blocks (the dichotomy's probes) match consecutive numpy draws."""
    a, b = substream(0, "probe"), substream(0, "probe")
    for _ in range(3):
        got = device_normal_block(a, 20_000, 14).cpu().numpy()
        assert np.array_equal(got, b.standard_normal((20_000, 14)) / np.sqrt(14))


def test_run_csc_same_with_host_and_device_rng(c1_golden):
    from conftest import D_C1
    from gpu_util import c1_op
    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import pipeline

    results = []
    for flag in (True, False):
        pipeline.USE_DEVICE_RNG = flag
        try:
            results.append(P.run_csc(c1_op(), P.CscParams(k=20, d=D_C1, seed=0)))
        finally:
            pipeline.USE_DEVICE_RNG = True
    assert results[0].to_json() == results[1].to_json()
    assert np.array_equal(results[0].labels, c1_golden["labels"])
