"""K2: the fused Chebyshev filter against the reference (golden) and the oracle."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import relerr
from gpu_util import c1_graph, c1_op, options, oracle_csr
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-9  # north_star: 1e-9 relative in fp64
FP32_TOL = 1e-4  # north_star: 1e-4 relative in fp32 mode

VARIANTS = [dict(recurrence=r, panel_width=pw) for r in (0, 1) for pw in (0, 4, 8, 16)]


@pytest.mark.parametrize("opt", VARIANTS, ids=lambda o: f"rec{o['recurrence']}-pw{o['panel_width']}")
def test_filter_c1_fp64_golden(filter_golden, opt):
    op = c1_op()
    X = filter_golden["X"]
    low = P.design_lowpass(0.37, 50)
    with options(**opt):
        assert relerr(P.apply_filter(low, op, X), filter_golden["Y_low"]) <= FP64_TOL
        assert relerr(P.apply_filter(P.matched_highpass(low), op, X), filter_golden["Y_high"]) <= FP64_TOL
        assert relerr(P.apply_filter(P.design_lowpass(1.3, 2), op, X[:, :5]), filter_golden["Y_order2"]) <= FP64_TOL
        y1 = P.apply_filter(P.design_lowpass(0.8, 1, damping="none"), op, X[:, :3])
        assert relerr(y1, filter_golden["Y_order1"]) <= FP64_TOL
        assert relerr(op.apply(X[:, :4]), filter_golden["LX"]) <= 1e-13


@pytest.mark.parametrize("rec", [0, 1])
def test_filter_c1_fp32(filter_golden, rec):
    op = c1_op("float32")
    X = filter_golden["X"]
    with options(recurrence=rec):
        y = P.apply_filter(P.design_lowpass(0.37, 50), op, X)
    assert y.dtype == np.float64
    assert relerr(y, filter_golden["Y_low"]) <= FP32_TOL


def test_fp64_is_tight(filter_golden):
    """fp64 should be far inside the 1e-9 bar (rounding only)."""
    y = P.apply_filter(P.design_lowpass(0.37, 50), c1_op(), filter_golden["X"])
    assert relerr(y, filter_golden["Y_low"]) <= 1e-12


def test_identity_filter_is_exact():
    g = P.build_graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
    op = P.laplacian_op(g)
    ident = P.PolyFilter(coeffs=np.array([1.0]), cutoff=1.0, order=0, damping="none", kind="lowpass")
    X = np.random.default_rng(0).standard_normal((3, 4))
    assert np.array_equal(P.apply_filter(ident, op, X), X)


def test_vector_and_device_tensor_inputs(filter_golden):
    import torch

    op = c1_op()
    low = P.design_lowpass(0.37, 50)
    x = filter_golden["X"][:, 0].copy()
    y = P.apply_filter(low, op, x)
    assert y.shape == (1000,)
    assert relerr(y, filter_golden["Y_low"][:, 0]) <= FP64_TOL
    Xt = torch.tensor(filter_golden["X"], device="cuda")
    Yt = P.apply_filter(low, op, Xt)
    assert Yt.is_cuda and Yt.dtype == torch.float64
    assert relerr(Yt.cpu().numpy(), filter_golden["Y_low"]) <= FP64_TOL
    Xs = Xt[:, ::2]  # strided view -> made contiguous at the boundary
    assert relerr(P.apply_filter(low, op, Xs).cpu().numpy(), filter_golden["Y_low"][:, ::2]) <= FP64_TOL
    Y32 = P.apply_filter(low, c1_op("float32"), Xt.float())
    assert Y32.dtype == torch.float32
    assert relerr(Y32.cpu().numpy(), filter_golden["Y_low"]) <= FP32_TOL


def test_matches_spectral_oracle():
    rng = np.random.default_rng(8)
    e = [(i, j, rng.uniform(0.2, 2)) for i in range(80) for j in range(i + 1, 80) if rng.random() < 0.1]
    g = P.build_graph(e, num_nodes=80)
    op = P.laplacian_op(g)
    L = O.dense_laplacian(oracle_csr(g))
    w, U = np.linalg.eigh(L)
    filt = P.design_lowpass(0.9, 30)
    X = rng.standard_normal((80, 5))
    ref = U @ (filt.evaluate(w)[:, None] * (U.T @ X))
    assert np.linalg.norm(P.apply_filter(filt, op, X) - ref) <= 1e-10 * np.linalg.norm(ref)


def test_linearity_symmetry_complementarity():
    op = c1_op()
    rng = np.random.default_rng(1)
    f = P.design_lowpass(0.6, 20)
    X, Y = rng.standard_normal((1000, 3)), rng.standard_normal((1000, 3))
    lhs = P.apply_filter(f, op, 2.0 * X - 3.0 * Y)
    rhs = 2.0 * P.apply_filter(f, op, X) - 3.0 * P.apply_filter(f, op, Y)
    assert np.linalg.norm(lhs - rhs) < 1e-10 * np.linalg.norm(rhs)
    x, y = rng.standard_normal(1000), rng.standard_normal(1000)
    assert abs(P.apply_filter(f, op, x) @ y - x @ P.apply_filter(f, op, y)) < 1e-9
    low = P.design_lowpass(1.1, 35)
    rec = P.apply_filter(low, op, X) + P.apply_filter(P.matched_highpass(low), op, X)
    assert np.abs(rec - X).max() < 1e-12


def test_oracle_agreement_many_widths():
    """Widths that exercise every panel shape (1..70 columns) against the oracle."""
    g, _ = c1_graph()
    op = c1_op()
    csr = oracle_csr(g)
    f = P.design_lowpass(0.5, 12)
    rng = np.random.default_rng(4)
    for w in (1, 2, 3, 5, 7, 9, 16, 17, 33, 47, 64, 70):
        X = rng.standard_normal((1000, w))
        assert relerr(P.apply_filter(f, op, X), O.apply_filter(f.coeffs, csr, X)) <= 1e-12, w


def test_dimension_mismatch():
    op = c1_op()
    with pytest.raises(ValueError):
        P.apply_filter(P.design_lowpass(1.0, 5), op, np.ones((5, 2)))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_lean_mid_step_kernel_matches_general_kernel(filter_golden, dtype):
    """The 32-register mid-step kernel (k_cheb_mid, default for 128/256-B unit-weight rows)
    gives the general step kernel's results bit for bit, for both recurrences and the panel
    widths that route to it; and both match the reference."""
    op = c1_op(dtype)
    X = filter_golden["X"]
    low = P.design_lowpass(0.37, 50)
    for pw in (0, 4, 8, 16, 32, 64):
        for rec in (0, 1):
            with options(panel_width=pw, recurrence=rec, lean_mid=0):
                general = P.apply_filter(low, op, X)
            with options(panel_width=pw, recurrence=rec, lean_mid=1):
                lean = P.apply_filter(low, op, X)
            assert np.array_equal(general, lean), (pw, rec)
            assert relerr(lean, filter_golden["Y_low"]) <= (FP64_TOL if dtype == "float64" else FP32_TOL)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_programmatic_dependent_launch_is_bit_identical(filter_golden, dtype):
    """Step kernels launched with programmatic stream serialization (option pdl: the next step's
    CSR prologue overlaps the previous step's drain, its panels are touched after
    griddepcontrol.wait) give the plainly serialised launches' results bit for bit -- lean and
    general kernels, both recurrences, single- and multi-panel blocks, back-to-back filters."""
    op = c1_op(dtype)
    X = filter_golden["X"]
    low, high = P.design_lowpass(0.37, 50), P.matched_highpass(P.design_lowpass(0.37, 50))
    for pw in (0, 8, 32):
        for rec in (0, 1):
            for lean in (0, 1):
                with options(panel_width=pw, recurrence=rec, lean_mid=lean, pdl=0):
                    ref = [P.apply_filter(f, op, X) for f in (low, high, low)]
                with options(panel_width=pw, recurrence=rec, lean_mid=lean, pdl=1):
                    got = [P.apply_filter(f, op, X) for f in (low, high, low)]
                for a, b in zip(ref, got):
                    assert np.array_equal(a, b), (pw, rec, lean)


def test_profile_modes_count_launches_and_bytes(filter_golden):
    """profile 1 (per launch) and 2 (per filter span) count the same launches and bytes; the span
    covers at least the sum of the launches' own times."""
    from paper_1602_02018_b200 import _lib

    op = c1_op("float32")
    X = filter_golden["X"]
    low = P.design_lowpass(0.37, 50)
    got = {}
    for mode in (1, 2):
        _lib.profile_reset()
        with options(profile=mode):
            P.apply_filter(low, op, X)
            got[mode] = _lib.profile_read()
        _lib.profile_reset()
    (ms1, n1, b1), (ms2, n2, b2) = got[1], got[2]
    assert n1 == n2 == 50 and b1 == b2 > 0 and ms1 > 0 and ms2 > 0
