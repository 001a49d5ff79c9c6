"""Randomised parity (hypothesis): device graph build and filters against the oracle on messy
edge lists -- duplicates in both directions, self loops (dropped), zero weights, isolated nodes."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from conftest import relerr
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P

pytestmark = pytest.mark.gpu

WEIGHTS = st.one_of(st.sampled_from([0.0, 0.5, 1.0, 2.25, 3.0]),
                    st.floats(min_value=1e-3, max_value=10.0, allow_nan=False, allow_infinity=False))


@st.composite
def edge_lists(draw):
    n = draw(st.integers(min_value=2, max_value=60))
    m = draw(st.integers(min_value=1, max_value=4 * n))
    src = draw(st.lists(st.integers(0, n - 1), min_size=m, max_size=m))
    dst = draw(st.lists(st.integers(0, n - 1), min_size=m, max_size=m))
    w = draw(st.lists(WEIGHTS, min_size=m, max_size=m))
    return n, np.array(src), np.array(dst), np.array(w, dtype=np.float64)


def _oracle_csr(n, src, dst, w):
    keep = src != dst  # self_loops="drop"
    return O.build_csr(src[keep], dst[keep], w[keep], n)


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(edge_lists())
def test_graph_build_matches_oracle(case):
    n, src, dst, w = case
    ref = _oracle_csr(n, src, dst, w)
    g = P.build_graph(np.column_stack([src, dst, w]), num_nodes=n, self_loops="drop")
    assert np.array_equal(g.indptr, ref.indptr) and np.array_equal(g.indices, ref.indices)
    assert np.array_equal(g.weights, ref.weights) and np.array_equal(g.degrees, ref.degrees)


@settings(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(edge_lists(), st.sampled_from([1, 2, 5, 30]), st.integers(1, 9), st.integers(0, 1))
def test_filter_matches_oracle(case, order, width, rec):
    n, src, dst, w = case
    ref = _oracle_csr(n, src, dst, w)
    g = P.build_graph(np.column_stack([src, dst, w]), num_nodes=n, self_loops="drop")
    X = np.random.default_rng(order * 31 + width).standard_normal((n, width))
    filt = P.design_lowpass(0.7, order)
    want = O.apply_filter(filt.coeffs, ref, X)
    P._lib.set_option("recurrence", rec)
    try:
        got64 = P.apply_filter(filt, P.laplacian_op(g), X)
        got32 = P.apply_filter(filt, P.laplacian_op(g, dtype="float32"), X)
    finally:
        P._lib.set_option("recurrence", 0)
    assert relerr(got64, want) <= 1e-12
    assert relerr(got32, want) <= 1e-4


@pytest.mark.parametrize("dtype,pw,tol", [("float64", 64, 1e-12), ("float32", 128, 1e-4), ("float64", 8, 1e-12)])
@pytest.mark.parametrize("rec", [0, 1])
def test_wide_panels_heavy_weighted_rows(dtype, pw, rec, tol):
    """32-lane panel rows (512 B: 8-slot neighbour chunks, only lanes < 8 hold indices) on a
    weighted graph with heavy-tailed degrees (up to ~70), so rows span many 8-slot chunks and the
    warp-uniform chunk loop ends mid-chunk; every width up to two panels."""
    rng = np.random.default_rng(11)
    n = 700
    deg = np.minimum(rng.pareto(1.5, n) * 6 + 1, 60).astype(int)
    deg[rng.choice(n, 25, replace=False)] = 0  # rows with incoming edges only
    src = np.repeat(np.arange(n), deg)
    dst = rng.integers(0, n, src.size)
    w = rng.choice([0.5, 1.0, 2.25, 3.0], src.size)
    ref = _oracle_csr(n, src, dst, w)
    assert np.diff(ref.indptr).max() > 48
    g = P.build_graph(np.column_stack([src, dst, w]), num_nodes=n, self_loops="drop")
    op = P.laplacian_op(g, dtype=dtype)
    filt = P.design_lowpass(0.6, 20)
    old_pw, old_rec = P._lib.get_option("panel_width"), P._lib.get_option("recurrence")
    P._lib.set_option("panel_width", pw)
    P._lib.set_option("recurrence", rec)
    try:
        for width in (1, pw // 2 + 3, pw, pw + 5):
            X = rng.standard_normal((n, width))
            assert relerr(P.apply_filter(filt, op, X), O.apply_filter(filt.coeffs, ref, X)) <= tol, width
    finally:
        P._lib.set_option("panel_width", old_pw)
        P._lib.set_option("recurrence", old_rec)


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_lean_kernel_unit_weights_isolated_and_heavy_rows(dtype, weighted):
    """Unit-weight graph (the lean mid-step kernel's case) with isolated nodes and degrees from
    0 to ~90: every panel width that routes to k_cheb_mid (16- to 512-B rows) and the 32-B rows
    that do not, bit-identical to the general kernel and within tolerance of the oracle."""
    rng = np.random.default_rng(23)
    n = 900
    deg = np.minimum(rng.pareto(1.3, n) * 5 + 1, 80).astype(int)
    deg[rng.choice(n, 40, replace=False)] = 0
    src = np.repeat(np.arange(n), deg)
    dst = rng.integers(0, n - 30, src.size)  # the last 30 nodes only get edges from their own rows
    keep = src != dst
    src, dst = src[keep], dst[keep]
    w = rng.choice([0.5, 1.0, 2.25, 3.0], src.size) if weighted else np.ones(src.size)
    ref = O.build_csr(src, dst, w, n)
    g = P.build_graph(np.column_stack([src, dst, w]), num_nodes=n)
    assert (np.diff(ref.indptr) == 0).any() and np.diff(ref.indptr).max() > 64
    op = P.laplacian_op(g, dtype=dtype)
    filt = P.design_lowpass(0.55, 25)
    tol = 1e-12 if dtype == "float64" else 1e-4
    vec = 2 if dtype == "float64" else 4
    old = {k: P._lib.get_option(k) for k in ("panel_width", "lean_mid")}
    try:
        for pw in (vec, 2 * vec, 4 * vec, 8 * vec, 16 * vec, 32 * vec):
            X = rng.standard_normal((n, pw - 1 if pw > 1 else 1))
            want = O.apply_filter(filt.coeffs, ref, X)
            P._lib.set_option("panel_width", pw)
            P._lib.set_option("lean_mid", 0)
            general = P.apply_filter(filt, op, X)
            P._lib.set_option("lean_mid", 1)
            lean = P.apply_filter(filt, op, X)
            assert np.array_equal(general, lean), pw
            assert relerr(lean, want) <= tol, pw
    finally:
        for k, v in old.items():
            P._lib.set_option(k, v)
