"""Device backend of the column-sharded path, and full-size (BASELINE config 3) properties."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import D_C1, relerr, sbm_config
from gpu_util import c1_op, options
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P
from paper_1602_02018_b200 import dist as D

pytestmark = pytest.mark.gpu


def test_device_backend_single_rank_matches_reference(c1_golden):
    grp = D.Group(0, 1)
    res = D.run_csc_sharded(D.DeviceBackend(c1_op()), 1000, P.CscParams(k=20, d=D_C1, seed=0), grp)
    assert res.diagnostics["lambda_k_hat"] == float(c1_golden["lambda_k_hat"])
    assert res.diagnostics["solver_iterations"] == c1_golden["solver_iterations"].tolist()
    assert np.array_equal(res.labels, c1_golden["labels"])


def test_device_backend_partial_assign_matches_oracle():
    import torch

    rng = np.random.default_rng(7)
    soft = rng.standard_normal((3000, 23))
    soft[5] = 0.0
    be = D.DeviceBackend(c1_op())
    val, col, nz, any_norm = be.row_best(torch.tensor(soft[:, 10:], device="cuda"), 10)
    q = soft[:, 10:] / np.linalg.norm(soft[:, 10:], axis=0)
    assert np.array_equal(col, 10 + q.argmax(axis=1))
    assert np.allclose(val, q.max(axis=1), rtol=1e-14, atol=0)
    assert not nz[5] and nz.sum() == 2999 and any_norm


_big: dict = {}


def c3_graph():
    if "g" not in _big:
        _big["g"] = P.sbm_generate(sbm_config(1_000_000, 100))
    return _big["g"]


def test_c3_graph_build_matches_scipy_path():
    g, _ = c3_graph()
    src, dst, _ = P.sbm.sbm_edges(sbm_config(1_000_000, 100))
    ref = O.sbm_csr(src, dst, 1_000_000)
    assert O.csr_digest(O.Csr(g.num_nodes, g.indptr, g.indices, g.weights, g.degrees)) == O.csr_digest(ref)


def test_c3_fp32_vs_fp64_and_low_order_oracle():
    """Full size: fp32 mode within 1e-4 of fp64; fp64 within 1e-12 of the oracle on a short filter."""
    g, _ = c3_graph()
    d = int(math.ceil(4 * math.log(1e6)))
    X = np.random.default_rng(3).standard_normal((1_000_000, d)) / np.sqrt(d)
    filt = P.design_lowpass(0.43, 50)
    y64 = P.apply_filter(filt, P.laplacian_op(g), X)
    y32 = P.apply_filter(filt, P.laplacian_op(g, dtype="float32"), X)
    assert relerr(y32, y64) <= 1e-4
    short = P.design_lowpass(0.43, 3)
    csr = O.Csr(g.num_nodes, g.indptr, g.indices, g.weights, g.degrees)
    assert relerr(P.apply_filter(short, P.laplacian_op(g), X[:, :4]), O.apply_filter(short.coeffs, csr, X[:, :4])) <= 1e-12


def test_c3_size_independent_properties():
    """Complementarity (low + high = I), linearity and symmetry at N = 1e6, both recurrences."""
    g, _ = c3_graph()
    op = P.laplacian_op(g)
    rng = np.random.default_rng(5)
    X = rng.standard_normal((1_000_000, 6))
    Z = rng.standard_normal((1_000_000, 6))
    low = P.design_lowpass(0.43, 50)
    high = P.matched_highpass(low)
    for rec in (0, 1):
        with options(recurrence=rec):
            lx = P.apply_filter(low, op, X)
            assert np.abs(lx + P.apply_filter(high, op, X) - X).max() < 1e-11
            lz = P.apply_filter(low, op, Z)
            assert relerr(P.apply_filter(low, op, 2 * X - 3 * Z), 2 * lx - 3 * lz) < 1e-12
            assert abs(np.sum(lx * Z) - np.sum(X * lz)) < 1e-9 * np.sqrt(np.sum(lx**2) * np.sum(Z**2))


def test_c3_eigencount_full_spectrum():
    g, _ = c3_graph()
    est = P.eigencount(P.laplacian_op(g, dtype="float32"), 2.0, rng=np.random.default_rng(0))
    assert abs(est.count - 1_000_000) <= 0.02 * 1_000_000


def test_dcsbm_heavy_rows_parity():
    """Degree-corrected SBM (BASELINE config 4 shape, smaller N): heavy-tailed rows vs the oracle."""
    cfg = P.SbmConfig(num_nodes=40_000, k=40, avg_degree=5.5, epsilon=P.critical_epsilon(5.5, 40) / 4.0, seed=0)
    g, truth, _ = P.dcsbm_generate(cfg)
    deg = np.diff(g.indptr)
    assert deg.max() > 15 * deg.mean()
    csr = O.Csr(g.num_nodes, g.indptr, g.indices, g.weights, g.degrees)
    src, dst, _, _ = P.sbm.dcsbm_edges(cfg)
    assert O.csr_digest(csr) == O.csr_digest(O.sbm_csr(src, dst, cfg.num_nodes))
    X = np.random.default_rng(1).standard_normal((cfg.num_nodes, 19))
    filt = P.design_lowpass(0.3, 50)
    ref = O.apply_filter(filt.coeffs, csr, X)
    assert relerr(P.apply_filter(filt, P.laplacian_op(g), X), ref) <= 1e-12
    assert relerr(P.apply_filter(filt, P.laplacian_op(g, dtype="float32"), X), ref) <= 1e-4
    iso = g.isolated_nodes
    y = P.apply_filter(filt, P.laplacian_op(g), X)
    if iso.size:  # isolated nodes: h(1) X
        assert np.allclose(y[iso], filt.evaluate(1.0) * X[iso], rtol=1e-12, atol=1e-14)


def test_dcsbm_run_csc_vs_oracle():
    cfg = P.SbmConfig(num_nodes=20_000, k=20, avg_degree=5.5, epsilon=P.critical_epsilon(5.5, 20) / 4.0, seed=0)
    g, truth, _ = P.dcsbm_generate(cfg)
    csr = O.Csr(g.num_nodes, g.indptr, g.indices, g.weights, g.degrees)
    d = int(math.ceil(4 * math.log(cfg.num_nodes)))
    r = P.run_csc(P.laplacian_op(g), P.CscParams(k=20, d=d, seed=0))
    o = O.run_csc(csr, 20, d=d, seed=0)
    assert r.diagnostics["lambda_k_hat"] == o["lambda_k_hat"]
    assert r.diagnostics["zero_feature_rows"] == o["zero_rows"].tolist()
    assert P.adjusted_rand_index(r.labels, o["labels"]) >= 0.99


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_row_sharded_single_rank_matches_replicated(transport):
    """Row-sharded operator (NCCL all-gather after every step, or peer stores fused into the
    step kernel) with one rank == the replicated path."""
    import torch

    g = c1_op().graph
    for dtype, tol in (("float64", 1e-12), ("float32", 1e-5)):
        rop = D.RowShardedOperator(g, D.Group(0, 1), dtype=dtype, transport=transport)
        op = P.laplacian_op(g, dtype=dtype)
        X = np.random.default_rng(2).standard_normal((1000, 21))
        filt = P.design_lowpass(0.45, 50)
        tdt = torch.float64 if dtype == "float64" else torch.float32
        Xt = torch.tensor(X, dtype=tdt, device="cuda")
        y = rop.apply_filter(filt, Xt).double().cpu().numpy()
        assert relerr(y, P.apply_filter(filt, op, X)) <= tol
        cnt = rop.eigencount(filt, Xt)
        ref = float(np.sum(P.apply_filter(filt, op, X) ** 2))
        assert abs(cnt - ref) <= tol * ref
        F, zero = rop.features(filt, Xt)
        fref = P.build_features(op, filt, P.features.RandomSignals(X, "gaussian", None))
        assert relerr(F.double().cpu().numpy(), fref.rows) <= tol
        assert np.array_equal(zero, fref.zero_rows)


def test_row_sharded_peer_transport_bit_equal_to_nccl():
    """The fused peer-store transport moves the same values as the NCCL all-gather: results are
    bit-identical for every recurrence branch (orders 0-3 and 50), several panels per block and
    repeated calls (epochs advance; the transport grows for wider blocks)."""
    import torch

    g = c1_op().graph
    for dtype in ("float64", "float32"):
        tdt = torch.float64 if dtype == "float64" else torch.float32
        a = D.RowShardedOperator(g, D.Group(0, 1), dtype=dtype, transport="nccl")
        b = D.RowShardedOperator(g, D.Group(0, 1), dtype=dtype, transport="peer")
        for w in (5, 100, 7):
            X = torch.tensor(np.random.default_rng(w).standard_normal((1000, w)), dtype=tdt, device="cuda")
            for order in (0, 1, 2, 3, 50):
                filt = P.design_lowpass(0.6, order) if order else P.PolyFilter(np.array([0.7]), 0.6, 0, "none", "lowpass")
                ya, yb = a.apply_filter(filt, X), b.apply_filter(filt, X)
                assert torch.equal(ya, yb), (dtype, w, order)
            assert a.eigencount(filt, X) == b.eigencount(filt, X)
            fa, za = a.features(filt, X)
            fb, zb = b.features(filt, X)
            assert torch.equal(fa, fb) and np.array_equal(za, zb)
