"""The CPU oracle is pinned to the real reference: bit-exact on its golden fixtures."""

from __future__ import annotations

import numpy as np

from conftest import D_C1, c1_config
from oracle import cpu_ref as O
from paper_1602_02018_b200.sbm import sbm_edges


def c1_csr():
    src, dst, _ = sbm_edges(c1_config())
    return O.sbm_csr(src, dst, 1000)


def test_sbm_generator_matches_reference_graph(graphs_golden):
    g = c1_csr()
    assert np.array_equal(g.indptr, graphs_golden["c1_indptr"])
    assert np.array_equal(g.indices, graphs_golden["c1_indices"])
    assert np.array_equal(g.weights, graphs_golden["c1_weights"])
    assert np.array_equal(g.degrees, graphs_golden["c1_degrees"])
    _, _, truth = sbm_edges(c1_config())
    assert np.array_equal(truth, graphs_golden["c1_truth"])


def test_oracle_build_graph_messy(graphs_golden):
    e = graphs_golden["messy_edges"]
    g = O.build_csr(e[:, 0].astype(np.int64), e[:, 1].astype(np.int64), e[:, 2], 75)
    assert np.array_equal(g.indptr, graphs_golden["messy_indptr"])
    assert np.array_equal(g.indices, graphs_golden["messy_indices"])
    assert np.array_equal(g.weights, graphs_golden["messy_weights"])
    assert np.array_equal(g.degrees, graphs_golden["messy_degrees"])


def test_oracle_weighted_laplacian_and_filter(graphs_golden):
    e = graphs_golden["w60_edges"]
    g = O.build_csr(e[:, 0].astype(np.int64), e[:, 1].astype(np.int64), e[:, 2], 60)
    X = graphs_golden["w60_X"]
    assert np.array_equal(O.laplacian_apply(g, X), graphs_golden["w60_LX"])
    assert np.array_equal(O.apply_filter(O.lowpass_coeffs(0.9, 30), g, X), graphs_golden["w60_low"])
    L = O.dense_laplacian(g)
    assert np.linalg.norm(L @ X - graphs_golden["w60_LX"]) <= 1e-12 * np.linalg.norm(L @ X)


def test_oracle_filter_c1(filter_golden):
    g = c1_csr()
    X = filter_golden["X"]
    low = O.lowpass_coeffs(0.37, 50)
    assert np.array_equal(low, filter_golden["low_coeffs"])
    assert np.array_equal(O.highpass_coeffs(low), filter_golden["high_coeffs"])
    assert np.array_equal(O.apply_filter(low, g, X), filter_golden["Y_low"])
    assert np.array_equal(O.apply_filter(O.highpass_coeffs(low), g, X), filter_golden["Y_high"])
    assert np.array_equal(O.laplacian_apply(g, X[:, :4]), filter_golden["LX"])
    assert O.psd_ridge(O.highpass_coeffs(low)) == float(filter_golden["ridge"])
    assert np.array_equal(O.apply_filter(O.lowpass_coeffs(1.3, 2), g, X[:, :5]), filter_golden["Y_order2"])
    assert np.array_equal(O.apply_filter(O.lowpass_coeffs(0.8, 1, "none"), g, X[:, :3]), filter_golden["Y_order1"])


def test_oracle_pipeline_c1(c1_golden):
    g = c1_csr()
    r = O.run_csc(g, 20, d=D_C1, seed=0)
    assert np.array_equal(np.asarray(r["trace"]), c1_golden["trace"])
    assert r["lambda_k_hat"] == float(c1_golden["lambda_k_hat"])
    assert np.array_equal(r["indices"], c1_golden["indices"])
    assert np.array_equal(r["zero_rows"], c1_golden["zero_rows"])
    assert np.array_equal(r["features"], c1_golden["features"])
    assert np.array_equal(r["kmeans_labels"], c1_golden["kmeans_labels"])
    assert r["ridge"] == float(c1_golden["ridge"])
    assert np.array_equal(r["soft"], c1_golden["soft"])
    assert np.array_equal(r["solver_iterations"], c1_golden["solver_iterations"])
    assert np.array_equal(r["labels"], c1_golden["labels"])
