"""Relational properties the reference's own tests check (restated against the device paths):
relabelling equivariance, degenerate k-means, determinism of the full pipeline."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import relerr
from gpu_util import c1_graph, c1_op
import paper_1602_02018_b200 as P

pytestmark = pytest.mark.gpu


def test_filter_relabelling_equivariance():
    """h(L_perm) (X permuted) == (h(L) X) permuted: the operator does not depend on node order."""
    g, _ = c1_graph()
    rng = np.random.default_rng(11)
    perm = rng.permutation(g.num_nodes)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    rows = np.repeat(np.arange(g.num_nodes), np.diff(g.indptr))
    edges = np.column_stack([inv[rows], inv[g.indices], g.weights])
    edges = edges[edges[:, 0] < edges[:, 1]]
    gp = P.build_graph(edges, num_nodes=g.num_nodes)
    X = rng.standard_normal((g.num_nodes, 7))
    filt = P.design_lowpass(0.45, 50)
    y = P.apply_filter(filt, c1_op(), X)
    yp = P.apply_filter(filt, P.laplacian_op(gp), X[perm])
    assert relerr(yp, y[perm]) <= 1e-12


def test_kmeans_k_equals_n_and_duplicates():
    pts = np.random.default_rng(4).standard_normal((12, 3))
    lab = P.kmeans(pts, P.KmeansConfig(k=12, seed=2, replicates=3))
    # distances are |p|^2 + |c|^2 - 2 p.c clipped at 0 (kmeans.py:39-43): zero up to rounding
    assert lab.inertia <= 1e-12 and np.array_equal(np.sort(lab.labels), np.arange(12))
    dup = np.repeat(pts[:3], 4, axis=0)  # three distinct points, k = 3: zero inertia
    lab = P.kmeans(dup, P.KmeansConfig(k=3, seed=5, replicates=4))
    assert lab.inertia <= 1e-12 and np.unique(lab.labels).size == 3


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_run_csc_bitwise_deterministic(dtype):
    """Fixed-order reductions everywhere: two runs give bit-identical soft interpolants."""
    op = c1_op(dtype)
    prm = P.CscParams(k=20, d=28, seed=3)
    a = P.run_csc(op, prm)
    b = P.run_csc(op, prm)
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(np.asarray(a.soft), np.asarray(b.soft))
    for key in ("lambda_k_hat", "solver_iterations", "solver_residuals", "kmeans_inertia"):
        assert a.diagnostics[key] == b.diagnostics[key], key
