"""BASELINE config 5 (SBM N = 16e6, k = 500, s = 16; 2.56e8 stored entries) on one GPU:
size-independent properties at full size (the oracle cannot run at this size)."""

from __future__ import annotations

import functools

import numpy as np
import pytest

import paper_1602_02018_b200 as P
from paper_1602_02018_b200 import dist as D

pytestmark = pytest.mark.gpu

N5, K5 = 16_000_000, 500


@functools.lru_cache(maxsize=1)
def c5_graph():
    cfg = P.SbmConfig(num_nodes=N5, k=K5, avg_degree=16, epsilon=P.critical_epsilon(16, K5) / 4, seed=0)
    return P.sbm_generate(cfg)


def _rel(a, b):
    import torch

    return float(torch.linalg.norm((a - b).double()) / torch.linalg.norm(b.double()))


def test_c5_graph_invariants():
    g, labels = c5_graph()
    assert g.num_nodes == N5 and labels.size == N5
    assert g.indices.size == 2 * g.num_edges
    assert abs(g.indices.size / N5 - 16.0) < 0.05  # mean degree s = 16
    assert float(g.degrees.sum()) == float(g.indices.size)  # unit weights
    # canonical CSR: strictly increasing columns inside a row, no self loops (spot check)
    for r in (0, 1, 7_999_999, N5 - 1):
        cols = g.indices[g.indptr[r]: g.indptr[r + 1]]
        assert np.all(np.diff(cols) > 0) and r not in cols


def test_c5_complementarity_linearity_symmetry_fp64():
    import torch

    g, _ = c5_graph()
    op = P.laplacian_op(g)
    gen = torch.Generator(device="cuda").manual_seed(5)
    X = torch.randn(N5, 4, dtype=torch.float64, device="cuda", generator=gen)
    Z = torch.randn(N5, 4, dtype=torch.float64, device="cuda", generator=gen)
    low = P.design_lowpass(0.2, 50)
    high = P.matched_highpass(low)
    lx = P.apply_filter(low, op, X)
    assert float((lx + P.apply_filter(high, op, X) - X).abs().max()) < 1e-11
    lz = P.apply_filter(low, op, Z)
    assert _rel(P.apply_filter(low, op, 2 * X - 3 * Z), 2 * lx - 3 * lz) < 1e-12
    assert abs(float((lx * Z).sum() - (X * lz).sum())) < 1e-9 * float(lx.norm() * Z.norm())


def test_c5_fp32_vs_fp64_and_row_sharded_transports():
    """fp32 mode within 1e-4 of fp64 at full size; the row-sharded operator (one rank, NCCL
    and fused peer transports) reproduces the replicated fp32 path."""
    import torch

    g, _ = c5_graph()
    gen = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn(N5, 6, dtype=torch.float64, device="cuda", generator=gen)
    filt = P.design_lowpass(0.2, 50)
    y64 = P.apply_filter(filt, P.laplacian_op(g), X)
    X32 = X.float()
    y32 = P.apply_filter(filt, P.laplacian_op(g, dtype="float32"), X32)
    assert _rel(y32, y64) < 1e-4
    for transport in ("nccl", "peer"):
        rop = D.RowShardedOperator(g, D.Group(0, 1), dtype="float32", transport=transport)
        yr = rop.apply_filter(filt, X32)
        assert _rel(yr, y32) < 1e-6, transport
        del rop
