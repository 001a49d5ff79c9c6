"""K1 (device CSR build + normalisation) and the Laplacian SpMM against the reference."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import c1_config, relerr
from gpu_util import oracle_csr
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P

pytestmark = pytest.mark.gpu


def test_build_graph_messy_edges_bit_exact(graphs_golden):
    g = P.build_graph(graphs_golden["messy_edges"], num_nodes=75)
    assert np.array_equal(g.indptr, graphs_golden["messy_indptr"])
    assert np.array_equal(g.indices, graphs_golden["messy_indices"])
    assert np.array_equal(g.weights, graphs_golden["messy_weights"])
    assert np.array_equal(g.degrees, graphs_golden["messy_degrees"])


def test_sbm_graph_bit_exact(graphs_golden):
    g, truth = P.sbm_generate(c1_config())
    assert np.array_equal(g.indptr, graphs_golden["c1_indptr"])
    assert np.array_equal(g.indices, graphs_golden["c1_indices"])
    assert np.array_equal(g.weights, graphs_golden["c1_weights"])
    assert np.array_equal(g.degrees, graphs_golden["c1_degrees"])
    assert np.array_equal(truth, graphs_golden["c1_truth"])


def test_build_semantics():
    k3 = P.build_graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    assert np.allclose(k3.degrees, [2, 2, 2]) and k3.num_edges == 3
    g = P.build_graph([(0, 1, 2.5)], num_nodes=3)
    assert np.allclose(g.degrees, [2.5, 2.5, 0.0]) and g.isolated_nodes.tolist() == [2]
    g = P.build_graph([(0, 1, 1.0), (1, 0, 1.0)])
    assert g.num_edges == 1
    g = P.build_graph([(0, 1, 1.0), (0, 1, 2.0), (1, 0, 5.0)])
    W = g.adjacency().toarray()
    assert W[0, 1] == 5.0 and W[1, 0] == 5.0
    g = P.build_graph([(1, 1, 1.0), (0, 1, 1.0)], self_loops="drop")
    assert g.num_edges == 1 and g.adjacency().diagonal().sum() == 0.0
    g = P.build_graph([(0, 1)])  # missing weight = 1
    assert g.weights.tolist() == [1.0, 1.0]
    e = P.build_graph(np.empty((0, 3)), num_nodes=4)
    assert e.num_nodes == 4 and e.indices.size == 0


def test_build_errors():
    with pytest.raises(P.GraphError, match="negative weight"):
        P.build_graph([(0, 1, -0.5)])
    with pytest.raises(P.GraphError, match="out of range"):
        P.build_graph([(0, 7, 1.0)], num_nodes=3)
    with pytest.raises(P.GraphError, match="self-loop"):
        P.build_graph([(1, 1, 1.0), (0, 1, 1.0)])
    with pytest.raises(ValueError):
        P.build_graph([(0, 1)], self_loops="keep")


def test_symmetrization_idempotent_and_sorted():
    rng = np.random.default_rng(3)
    e = [(i, j, rng.uniform(0.2, 2)) for i in range(40) for j in range(i + 1, 40) if rng.random() < 0.15]
    g = P.build_graph(e, num_nodes=40)
    W = g.adjacency().tocoo()
    h = P.build_graph(np.column_stack([W.row, W.col, W.data]), num_nodes=40)
    assert np.array_equal(h.indptr, g.indptr) and np.array_equal(h.indices, g.indices)
    assert np.array_equal(h.weights, g.weights)
    for i in range(40):
        assert np.all(np.diff(g.indices[g.indptr[i]:g.indptr[i + 1]]) > 0)


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 2e-6)])
def test_laplacian_weighted_vs_golden(graphs_golden, dtype, tol):
    e = graphs_golden["w60_edges"]
    g = P.build_graph(e, num_nodes=60)
    op = P.laplacian_op(g, dtype=dtype)
    X = graphs_golden["w60_X"]
    assert relerr(op.apply(X), graphs_golden["w60_LX"]) <= tol
    L = O.dense_laplacian(oracle_csr(g))
    assert relerr(op.apply(X), L @ X) <= tol


def test_laplacian_properties():
    k3 = P.build_graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    op = P.laplacian_op(k3)
    assert np.linalg.norm(P.apply_laplacian(op, np.sqrt(k3.degrees))) < 1e-14
    two = P.build_graph([(0, 1, 1.0), (2, 3, 1.0)])
    op2 = P.laplacian_op(two)
    assert np.linalg.norm(op2.apply(np.sqrt(two.degrees) * np.array([1.0, 1, 0, 0]))) < 1e-14
    iso = P.laplacian_op(P.build_graph([(0, 1, 1.0)], num_nodes=3))
    assert np.allclose(iso.apply(np.array([0.0, 0.0, 5.0])), [0, 0, 5])
    with pytest.raises(ValueError, match="rows"):
        op.apply(np.ones(5))
    rng = np.random.default_rng(13)
    e = [(i, j, rng.uniform(0.2, 2)) for i in range(40) for j in range(i + 1, 40) if rng.random() < 0.2]
    op = P.laplacian_op(P.build_graph(e, num_nodes=40))
    x, y = rng.standard_normal(40), rng.standard_normal(40)
    assert abs(op.apply(x) @ y - x @ op.apply(y)) < 1e-12
    q = x @ op.apply(x)
    assert -1e-10 <= q <= 2 * (x @ x) + 1e-10


def test_graph_from_arrays_uses_create_path(graphs_golden):
    g = P.Graph(num_nodes=1000, indptr=graphs_golden["c1_indptr"], indices=graphs_golden["c1_indices"],
                weights=graphs_golden["c1_weights"], degrees=graphs_golden["c1_degrees"])
    op = P.laplacian_op(g)
    X = np.random.default_rng(0).standard_normal((1000, 3))
    ref = O.laplacian_apply(oracle_csr(g), X)
    assert relerr(op.apply(X), ref) <= 1e-13
    assert np.array_equal(op.d_inv_sqrt, O.Csr(1000, g.indptr, g.indices, g.weights, g.degrees).dis)


def test_create_rejects_bad_csr():
    bad = P.Graph(num_nodes=3, indptr=np.array([0, 2, 1, 2], np.int32), indices=np.array([1, 2], np.int32),
                  weights=np.ones(2), degrees=np.ones(3))
    with pytest.raises(P.GraphError):
        P.laplacian_op(bad)
    bad2 = P.Graph(num_nodes=3, indptr=np.array([0, 1, 1, 1], np.int32), indices=np.array([9], np.int32),
                   weights=np.ones(1), degrees=np.ones(3))
    with pytest.raises(P.GraphError):
        P.laplacian_op(bad2)


def test_edge_list_round_trip(tmp_path):
    rng = np.random.default_rng(5)
    e = [(i, j, rng.uniform(0.2, 2)) for i in range(35) for j in range(i + 1, 35) if rng.random() < 0.2]
    g = P.build_graph(e, num_nodes=36)
    P.write_edge_list(g, tmp_path / "g.edges")
    h = P.read_edge_list(tmp_path / "g.edges")
    assert h.num_nodes == 36
    assert np.array_equal(h.indptr, g.indptr) and np.array_equal(h.weights, g.weights)
    (tmp_path / "bad.edges").write_text("0 1\nnonsense line here oops\n")
    with pytest.raises(P.GraphError, match=":2"):
        P.read_edge_list(tmp_path / "bad.edges")


def test_read_edge_list_matches_reference(tmp_path):
    """read_edge_list on the messy golden file: the reference's CSR, node count from the last
    '# nodes' header; a self loop raises as in the reference (build_graph, self_loops='error')."""
    import json

    from conftest import golden

    eg = golden("edgelists")
    p = tmp_path / "messy.edges"
    p.write_bytes(bytes(eg["messy_text"]))
    g = P.read_edge_list(p)
    assert g.num_nodes == int(eg["messy_n"])
    assert np.array_equal(g.indptr, eg["messy_indptr"]) and np.array_equal(g.indices, eg["messy_indices"])
    assert np.array_equal(g.weights, eg["messy_weights"])
    msgs = json.loads(bytes(eg["error_msgs"]).decode())
    q = tmp_path / "loop.edges"
    q.write_text(json.loads(bytes(eg["error_texts"]).decode())["self_loop"])
    with pytest.raises(P.GraphError, match=msgs["self_loop"][1]):
        P.read_edge_list(q)


def test_edge_list_round_trip_bit_identical(tmp_path):
    """write_edge_list -> read_edge_list reproduces the CSR bit for bit (test_graph.py:146-162),
    including trailing isolated nodes, and the file is the oracle's bytes."""
    rng = np.random.default_rng(5)
    n, m = 300, 2000
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = src != dst
    w = 10.0 ** rng.uniform(-6, 8, m)
    g = P.build_graph(np.column_stack([src[keep], dst[keep], w[keep]]), num_nodes=n + 4)
    path = tmp_path / "rt.edges"
    P.write_edge_list(g, path)
    assert path.read_bytes() == O.format_edge_list(g.num_nodes, g.indptr, g.indices, g.weights)
    g2 = P.read_edge_list(path)
    assert g2.num_nodes == n + 4
    assert np.array_equal(g2.indptr, g.indptr) and np.array_equal(g2.indices, g.indices)
    assert np.array_equal(g2.weights, g.weights)
