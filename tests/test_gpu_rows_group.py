"""Row-sharded filter at world > 1 on one GPU (BASELINE config 5).

``RowShardGroup`` runs every rank's shard of ``csc_cheb_filter_rows_group`` in lockstep with
the per-step all-gather done as device copies: the same kernels, per-rank arguments,
nnz-balanced partition and padded panel layout as the NCCL transport, without ranks that
wait on one another (B200_PROFILING.md).  Sharding must not change a single bit: world
2..8 equals world 1, and world 1 equals the replicated operator to rounding.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import relerr
from gpu_util import c1_op, oracle_csr
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P
from paper_1602_02018_b200 import dist as D

pytestmark = pytest.mark.gpu


def _dcsbm_graph():
    cfg = P.SbmConfig(num_nodes=30_000, k=30, avg_degree=5.5, epsilon=P.critical_epsilon(5.5, 30) / 4.0, seed=3)
    return P.dcsbm_generate(cfg)[0]


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("which", ["c1", "dcsbm"])
def test_group_world_n_bit_equal_to_world_1(dtype, which):
    import torch

    g = c1_op().graph if which == "c1" else _dcsbm_graph()
    tdt = torch.float64 if dtype == "float64" else torch.float32
    X = torch.tensor(np.random.default_rng(4).standard_normal((g.num_nodes, 21)), dtype=tdt, device="cuda")
    filt = P.design_lowpass(0.45, 50)
    one = D.RowShardGroup(g, 1, dtype=dtype)
    y1 = one.apply_filter(filt, X)
    c1 = one.eigencount(filt, X)
    r1 = one.filter_rowsq(filt, X)[1]
    for world in (2, 3, 8):
        grp = D.RowShardGroup(g, world, dtype=dtype)
        assert torch.equal(grp.apply_filter(filt, X), y1), world
        _, rq = grp.filter_rowsq(filt, X)
        assert torch.equal(rq, r1), world
        # the eigencount partials are summed in rank order: equal to rounding
        assert abs(grp.eigencount(filt, X) - c1) <= 1e-13 * c1
    # world 1 is the replicated operator
    op = P.laplacian_op(g, dtype=dtype)
    ref = P.apply_filter(filt, op, X.double().cpu().numpy())
    assert relerr(y1.double().cpu().numpy(), ref) <= (1e-12 if dtype == "float64" else 1e-5)


def test_group_matches_oracle_and_heavy_partition():
    """fp64 vs the CPU oracle on the DC-SBM graph with 8 nnz-balanced shards (heavy rows put
    far fewer rows on some ranks: the panel slots are padded to the largest shard)."""
    import torch

    g = _dcsbm_graph()
    grp = D.RowShardGroup(g, 8, dtype="float64")
    sizes = np.diff(grp.starts)
    assert sizes.min() < sizes.max()  # unequal row counts exercise the padded slots
    X = np.random.default_rng(6).standard_normal((g.num_nodes, 9))
    filt = P.design_lowpass(0.3, 50)
    y = grp.apply_filter(filt, torch.tensor(X, device="cuda")).cpu().numpy()
    ref = O.apply_filter(filt.coeffs, oracle_csr(g), X)
    assert relerr(y, ref) <= 1e-9


@pytest.mark.parametrize("order", [0, 1, 2, 3])
def test_group_low_orders_and_wide_blocks(order):
    """Every recurrence branch (orders 0-3) and a multi-panel block (w = 100)."""
    import torch

    g = c1_op().graph
    X = torch.tensor(np.random.default_rng(order).standard_normal((1000, 100)), device="cuda")
    filt = P.design_lowpass(0.6, order) if order else P.PolyFilter(np.array([0.7]), 0.6, 0, "none", "lowpass")
    y1 = D.RowShardGroup(g, 1, dtype="float64").apply_filter(filt, X)
    y4 = D.RowShardGroup(g, 4, dtype="float64").apply_filter(filt, X)
    assert torch.equal(y1, y4)
    ref = P.apply_filter(filt, c1_op(), X.cpu().numpy())
    assert relerr(y4.cpu().numpy(), ref) <= 1e-12


def test_group_more_ranks_than_rows():
    """Empty shards (world > N) still step and exchange."""
    import torch

    g = P.build_graph([(0, 1, 1.0), (1, 2, 2.0), (2, 3, 1.0), (3, 0, 0.5), (4, 5, 1.0)], num_nodes=7)
    X = torch.tensor(np.random.default_rng(1).standard_normal((7, 3)), device="cuda")
    filt = P.design_lowpass(0.8, 5)
    y = D.RowShardGroup(g, 9, dtype="float64").apply_filter(filt, X)
    ref = P.apply_filter(filt, P.laplacian_op(g), X.cpu().numpy())
    assert relerr(y.cpu().numpy(), ref) <= 1e-12
