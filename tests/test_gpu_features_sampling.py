"""Features (filter + row normalisation), block CG and assignment against the reference."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import D_C1, relerr
from gpu_util import c1_graph, c1_op, options, oracle_csr
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P
from paper_1602_02018_b200._rng import substream

pytestmark = pytest.mark.gpu


def c1_features(op, golden):
    low = P.design_lowpass(float(golden["lambda_k_hat"]), 50)
    sig = P.generate_signals(1000, D_C1, "gaussian", substream(0, "signals"))
    return P.build_features(op, low, sig)


@pytest.mark.parametrize("rec", [0, 1])
@pytest.mark.parametrize("pw", [0, 8])
def test_features_c1_golden(c1_golden, rec, pw):
    with options(recurrence=rec, panel_width=pw):
        f = c1_features(c1_op(), c1_golden)
    assert relerr(f.rows, c1_golden["features"]) <= 1e-9
    assert np.abs(f.rows - c1_golden["features"]).max() <= 1e-9
    assert np.array_equal(f.zero_rows, c1_golden["zero_rows"])
    assert f.normalized and f.provenance["filter"]["order"] == 50


def test_features_c1_fp32(c1_golden):
    f = c1_features(c1_op("float32"), c1_golden)
    assert relerr(f.rows, c1_golden["features"]) <= 1e-4


def test_zero_rows_and_cliques():
    k3 = P.laplacian_op(P.build_graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)]))
    ident = P.PolyFilter(coeffs=np.array([1.0]), cutoff=1.0, order=0, damping="none", kind="lowpass")
    sig = P.generate_signals(3, 4, "gaussian", 0)
    sig.matrix[1] = 0.0
    f = P.build_features(k3, ident, sig)
    assert f.zero_rows.tolist() == [1] and np.all(f.rows[1] == 0.0)
    assert np.allclose(np.linalg.norm(f.rows[[0, 2]], axis=1), 1.0)
    edges = [(c * 10 + i, c * 10 + j, 1.0) for c in range(3) for i in range(10) for j in range(i + 1, 10)]
    op = P.laplacian_op(P.build_graph(edges, num_nodes=30))
    f = P.build_features(op, P.design_lowpass(0.5, 200), P.generate_signals(30, 8, "gaussian", 0))
    truth = np.repeat(np.arange(3), 10)
    for c in range(3):
        rows = f.rows[truth == c]
        assert np.abs(rows - rows[0]).max() < 1e-4
    assert P.pairwise_distance(f, 0, 10) > 0.5


def reduced_c1(golden):
    n = golden["indices"].size
    red = np.zeros((n, 20))
    red[np.arange(n), golden["kmeans_labels"]] = 1.0
    return red


@pytest.mark.parametrize("rec", [0, 1])
def test_block_cg_c1_golden(c1_golden, rec):
    hp = P.matched_highpass(P.design_lowpass(float(c1_golden["lambda_k_hat"]), 50))
    cfg = P.InterpolationConfig(highpass=hp)
    assert cfg.ridge == float(c1_golden["ridge"])
    samp = P.SamplingSet(indices=c1_golden["indices"], num_nodes=1000)
    with options(recurrence=rec):
        X, info = P.interpolate_all(c1_op(), cfg, samp, reduced_c1(c1_golden))
    assert relerr(X, c1_golden["soft"]) <= 1e-9
    assert np.array_equal(info.iterations, c1_golden["solver_iterations"])
    assert np.allclose(info.residuals, c1_golden["solver_residuals"], rtol=1e-6, atol=0)
    assert bool(np.all(info.converged))


def test_block_cg_c1_fp32(c1_golden):
    hp = P.matched_highpass(P.design_lowpass(float(c1_golden["lambda_k_hat"]), 50))
    cfg = P.InterpolationConfig(highpass=hp)
    samp = P.SamplingSet(indices=c1_golden["indices"], num_nodes=1000)
    X, info = P.interpolate_all(c1_op("float32"), cfg, samp, reduced_c1(c1_golden))
    assert relerr(X, c1_golden["soft"]) <= 1e-4
    lab = P.assign(X)
    assert P.adjusted_rand_index(lab, c1_golden["labels"]) >= 0.99


def test_system_apply_vs_oracle():
    g, _ = c1_graph()
    hp = P.design_highpass(0.5, 30)
    cfg = P.InterpolationConfig(highpass=hp)
    mask = np.zeros(1000)
    mask[np.random.default_rng(2).choice(1000, 40, replace=False)] = 1.0
    X = np.random.default_rng(3).standard_normal((1000, 6))
    ref = O.system_apply(oracle_csr(g), hp.coeffs, cfg.gamma, cfg.ridge, mask, X)
    assert relerr(P.sampling._system_apply(c1_op(), cfg, mask, X), ref) <= 1e-12
    q = float(X[:, 0] @ P.sampling._system_apply(c1_op(), cfg, mask, X[:, :1]).ravel())
    assert q >= -1e-10


def test_cg_dense_direct_and_contracts():
    g, _ = c1_graph()
    op = c1_op()
    L = O.dense_laplacian(oracle_csr(g))
    w, U = np.linalg.eigh(L)
    cfg = P.InterpolationConfig(highpass=P.design_highpass(0.45, 40), solver_tol=1e-10)
    samp = P.draw_sampling(1000, 60, 8)
    c_r = np.random.default_rng(0).standard_normal(60)
    x, info = P.interpolate(op, cfg, samp, c_r)
    assert bool(np.all(info.converged))
    mask = np.zeros(1000)
    mask[samp.indices] = 1.0
    A = np.diag(mask) + cfg.gamma * (U @ ((cfg.highpass.evaluate(w) + cfg.ridge)[:, None] * U.T))
    ref = np.linalg.solve(A, samp.adjoint(c_r))
    assert np.linalg.norm(x - ref) <= 1e-6 * np.linalg.norm(ref)
    # zero data -> zero solution, no iterations
    z, zi = P.interpolate(op, cfg, samp, np.zeros(60))
    assert np.all(z == 0.0) and zi.max_iterations == 0 and bool(np.all(zi.converged))
    # non-convergence is flagged, not raised
    bad = P.InterpolationConfig(highpass=P.design_highpass(0.45, 40), solver_tol=1e-12, solver_max_iters=2)
    _, bi = P.interpolate(op, bad, samp, c_r)
    assert not bool(np.all(bi.converged)) and bi.iterations[0] == 2 and bi.residuals[0] > 0
    with pytest.raises(ValueError):
        P.interpolate_all(op, cfg, samp, np.zeros((59, 2)))


def test_assign_semantics():
    assert P.assign(np.eye(4)).tolist() == [0, 1, 2, 3]
    rng = np.random.default_rng(0)
    soft = np.abs(rng.standard_normal((30, 4)))
    base = P.assign(soft)
    assert np.array_equal(P.assign(soft * np.array([3.0, 0.1, 7.5, 1.0])), base)
    soft = np.eye(3)
    soft[1] = 0.0
    lab, info = P.assign(soft, return_info=True)
    assert lab[1] == 0 and info["fallback_nodes"].tolist() == [1]
    with pytest.raises(ValueError):
        P.assign(np.zeros((4, 2)))
    assert P.assign(np.array([[0.5, 0.5], [0.2, 0.8]])).tolist() == [0, 1]
    z = np.array([[0.0, 1.0, 0.0], [0.0, 2.0, 0.0], [0.0, 0.5, 0.0]])  # zero-norm columns never win
    assert P.assign(-z).tolist() == [1, 1, 1]
    for seed in range(3):
        soft = np.random.default_rng(seed).standard_normal((5000, 37))
        assert np.array_equal(P.assign(soft), O.assign(soft)[0])


def test_gather_rows(c1_golden):
    import torch

    from paper_1602_02018_b200.pipeline import _gather_rows

    F = torch.tensor(c1_golden["features"], device="cuda")
    rows = _gather_rows(F, c1_golden["indices"], 0)
    assert np.array_equal(rows, c1_golden["features"][c1_golden["indices"]])


def test_kmeans_matches_golden(c1_golden):
    from paper_1602_02018_b200._rng import substream_seed

    rows = c1_golden["features"][c1_golden["indices"]]
    lab = P.kmeans(rows, P.KmeansConfig(k=20, seed=substream_seed(0, "kmeans")))
    assert np.array_equal(lab.labels, c1_golden["kmeans_labels"])
    assert abs(lab.inertia - float(c1_golden["kmeans_inertia"])) <= 1e-12 * float(c1_golden["kmeans_inertia"])


def test_kmeans_matches_oracle_random():
    rng = np.random.default_rng(3)
    for k, seed in ((6, 11), (9, 5)):
        pts = np.concatenate([rng.normal(c, 0.35, (40, 5)) for c in range(6)])
        a = P.kmeans(pts, P.KmeansConfig(k=k, seed=seed, replicates=5))
        b = O.kmeans(pts, k, seed, replicates=5)
        assert np.array_equal(a.labels, b[0]) and a.iterations_run == b[2]
        assert abs(a.inertia - b[1]) <= 1e-12 * b[1]
    # empty-cluster repair path: more clusters than distinct points
    pts = np.repeat(np.eye(3), 4, axis=0)
    a = P.kmeans(pts, P.KmeansConfig(k=5, seed=1, replicates=2))
    b = O.kmeans(pts, 5, 1, replicates=2)
    assert np.array_equal(a.labels, b[0]) and a.iterations_run == b[2]


def _device_seeds(pts, k, children, max_iters=0):
    from paper_1602_02018_b200 import _lib
    from paper_1602_02018_b200.kmeans import _MASK64

    n, d = pts.shape
    R = len(children)
    first = np.empty(R, dtype=np.int64)
    pcg = np.empty((R, 4), dtype=np.uint64)
    for r, ch in enumerate(children):
        rng = np.random.default_rng(ch)
        first[r] = rng.integers(n)
        st = rng.bit_generator.state["state"]
        pcg[r] = (st["state"] >> 64, st["state"] & _MASK64, st["inc"] >> 64, st["inc"] & _MASK64)
    labels = np.empty((R, n), dtype=np.int64)
    cent = np.empty((R, k, d))
    inertia, iters = np.empty(R), np.empty(R, dtype=np.int64)
    status = np.empty(R, dtype=np.int32)
    _lib.call("csc_kmeans_replicates", _lib.ptr(pts), n, d, k, R, _lib.ptr(first), _lib.ptr(pcg), None, max_iters,
              1e-6, _lib.ptr(labels), _lib.ptr(cent), _lib.ptr(inertia), _lib.ptr(iters), _lib.ptr(status), 0, None)
    return cent, status, labels, inertia, iters


@pytest.mark.parametrize("n,d,k", [(7, 3, 4), (922, 56, 100), (1000, 9, 30), (300, 130, 12)])
def test_kmeanspp_seeding_bit_exact(n, d, k):
    """Device D^2 sampling == the reference's numpy seeding (kmeans.py:52-61), bit for bit."""
    rng = np.random.default_rng(n + d)
    pts = rng.standard_normal((n, d)) * np.exp(rng.standard_normal((n, 1)))
    children = np.random.SeedSequence(17).spawn(6)
    cent, status, *_ = _device_seeds(pts, k, children)
    assert np.all(status == 0)
    for r, ch in enumerate(children):
        ref = O._seed_kmeanspp(pts, k, np.random.default_rng(ch))
        assert np.array_equal(cent[r], ref), r


def test_kmeans_seeding_zero_total_flagged():
    pts = np.repeat(np.eye(3), 4, axis=0)
    _, status, *_ = _device_seeds(pts, 5, np.random.SeedSequence(1).spawn(3))
    assert np.all(status == 1)


def test_kmeans_replicates_large_k_global_centroids():
    """k x d centroids beyond shared memory (global-memory path), many replicates."""
    rng = np.random.default_rng(8)
    k, d = 260, 100
    centers = rng.normal(0, 10, (k, d))
    pts = centers[rng.integers(k, size=1200)] + rng.normal(0, 0.5, (1200, d))
    a = P.kmeans(pts, P.KmeansConfig(k=k, seed=4, replicates=3))
    b = O.kmeans(pts, k, 4, replicates=3)
    assert np.array_equal(a.labels, b[0]) and a.iterations_run == b[2]
    assert abs(a.inertia - b[1]) <= 1e-9 * b[1]


def test_kmeans_random_seeding_matches_host_replicates():
    from paper_1602_02018_b200.kmeans import _initial_centers, _lloyd_device

    rng = np.random.default_rng(12)
    pts = np.concatenate([rng.normal(c, 0.4, (30, 4)) for c in range(5)])
    cfg = P.KmeansConfig(k=5, seed=9, replicates=4, seeding="random")
    a = P.kmeans(pts, cfg)
    best = None
    for ch in np.random.SeedSequence(9).spawn(4):
        lab, inert, it = _lloyd_device(pts, _initial_centers(pts, 5, np.random.default_rng(ch), "random"), 100, 1e-6, 0)
        if best is None or inert < best[1]:
            best = (lab, inert, it)
    assert np.array_equal(a.labels, best[0]) and a.inertia == best[1] and a.iterations_run == best[2]


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 1e-5)])
def test_block_cg_column_compaction_is_exact(c1_golden, dtype, tol):
    """Moving still-active columns into narrower panels (cg_compact) keeps every column's CG:
    same iteration counts and convergence flags, X equal up to reduction-order rounding."""
    hp = P.matched_highpass(P.design_lowpass(float(c1_golden["lambda_k_hat"]), 50))
    cfg = P.InterpolationConfig(highpass=hp)
    samp = P.SamplingSet(indices=c1_golden["indices"], num_nodes=1000)
    red = reduced_c1(c1_golden)
    with options(cg_compact=0):
        Xa, ia = P.interpolate_all(c1_op(dtype), cfg, samp, red)
    with options(cg_compact=1):
        Xb, ib = P.interpolate_all(c1_op(dtype), cfg, samp, red)
    assert np.array_equal(ia.iterations, ib.iterations) and np.array_equal(ia.converged, ib.converged)
    assert relerr(Xb, Xa) <= tol
    assert len(set(ia.iterations.tolist())) > 1  # staggered convergence: compaction actually happened


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_fast_single_panel_normalisation_bit_identical(c1_golden, dtype):
    """The vectorised single-/equal-width-panel normaliser (default) and the general one give the same bytes,
    zero rows and flags included (isolated nodes whose signal rows are zero), for host fp64 and
    device outputs of the compute dtype, at widths that fill a panel exactly and partially."""
    import torch

    g, _ = c1_graph()
    src, dst = np.repeat(np.arange(g.num_nodes), np.diff(g.indptr)), g.indices
    gi = P.build_graph(np.column_stack([src, dst, g.weights]), num_nodes=g.num_nodes + 5)  # 5 isolated nodes
    op = P.laplacian_op(gi, dtype=dtype)
    low = P.design_lowpass(0.4, 30)
    rng = np.random.default_rng(9)
    # panel_width forced narrow: multi-panel blocks (equal-width panels take the vectorised
    # normaliser too, e.g. w = 31 as 4 x 8 fp32 columns; w = 28 ends in a narrower panel)
    narrow = 8 if dtype == "float32" else 4
    for w, pwopt in [(3, 0), (16, 0), (28, 0), (31, 0), (64 if dtype == "float32" else 32, 0), (28, narrow),
                     (31, narrow), (2 * narrow, narrow)]:
        X = rng.standard_normal((gi.num_nodes, w))
        X[-5:-2] = 0.0
        out = {}
        for fast in (0, 1):
            with options(fast_normalize=fast, panel_width=pwopt):
                F = np.empty_like(X)
                z = P.features.features_into(op, low, X, F)
                Xd = torch.tensor(X, device="cuda", dtype=torch.float32 if dtype == "float32" else torch.float64)
                Fd = torch.empty_like(Xd)
                zd = P.features.features_into(op, low, Xd, Fd)
                out[fast] = (F, z, Fd.cpu().numpy(), zd)
        assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][2], out[1][2]), w
        assert out[0][1].tolist() == out[1][1].tolist() == out[0][3].tolist() == out[1][3].tolist() == [
            gi.num_nodes - 5, gi.num_nodes - 4, gi.num_nodes - 3], w
        rows, zero = O.build_features(low.coeffs, O.Csr(gi.num_nodes, gi.indptr, gi.indices, gi.weights, gi.degrees), X)
        assert relerr(out[1][0], rows) <= (1e-9 if dtype == "float64" else 1e-4), w


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_block_cg_remainder_panel_overlap_is_exact(c1_golden, dtype):
    """k = 20 in 8-wide panels (8 + 8 + 4): the 4-wide remainder panel's CG runs on the side
    stream / worker thread (cg_overlap=1) or in line (0) with bit-identical X, iteration counts
    and residuals, both matching the reference."""
    hp = P.matched_highpass(P.design_lowpass(float(c1_golden["lambda_k_hat"]), 50))
    cfg = P.InterpolationConfig(highpass=hp)
    samp = P.SamplingSet(indices=c1_golden["indices"], num_nodes=1000)
    res = {}
    for ov in (0, 1, 2):  # in line, remainder beside the main panels, panels alternating streams
        with options(panel_width=8, cg_overlap=ov):
            res[ov] = P.interpolate_all(c1_op(dtype), cfg, samp, reduced_c1(c1_golden))
    (X0, i0), (X1, i1) = res[0], res[1]
    for X, i in (res[1], res[2]):
        assert np.array_equal(X0, X)
        assert np.array_equal(i0.iterations, i.iterations) and np.array_equal(i0.residuals, i.residuals)
    assert relerr(X1, c1_golden["soft"]) <= (1e-9 if dtype == "float64" else 1e-4)
    if dtype == "float64":
        assert np.array_equal(i1.iterations, c1_golden["solver_iterations"])


def test_block_cg_two_wide_panels_split_streams_exact(c1_golden):
    """fp32, k = 200 on C1: two 128-wide panels of 512-B rows with a small gather source, the
    case the CG scheduler runs on two streams without the full-width token; results must be
    bit-identical to the in-line run and within the fp32 bar of the oracle."""
    hp = P.matched_highpass(P.design_lowpass(float(c1_golden["lambda_k_hat"]), 50))
    cfg = P.InterpolationConfig(highpass=hp)
    samp = P.SamplingSet(indices=c1_golden["indices"], num_nodes=1000)
    n, k = c1_golden["indices"].size, 200
    reduced = np.zeros((n, k))
    reduced[np.arange(n), np.random.default_rng(4).integers(0, k, n)] = 1.0
    res = {}
    for ov in (0, 1):
        with options(cg_overlap=ov):
            res[ov] = P.interpolate_all(c1_op("float32"), cfg, samp, reduced)
    (X0, i0), (X1, i1) = res[0], res[1]
    assert np.array_equal(X0, X1) and np.array_equal(i0.iterations, i1.iterations)
    g, _ = c1_graph()
    X, its, _, _ = O.interpolate_all(oracle_csr(g), hp.coeffs, cfg.gamma, cfg.ridge, samp.indices, reduced,
                                     cfg.solver_tol, cfg.solver_max_iters)
    assert relerr(X1, X) <= 1e-4


def test_features_async_device_call_matches(c1_golden):
    """features_into(..., zero_rows=False) on device buffers (no host synchronisation) writes the
    same features as the synchronous call."""
    import torch

    op = c1_op("float32")
    X = torch.tensor(np.random.default_rng(2).standard_normal((1000, 28)), device="cuda", dtype=torch.float32)
    low = P.design_lowpass(0.4, 30)
    F0, F1 = torch.empty_like(X), torch.empty_like(X)
    z = P.features.features_into(op, low, X, F0)
    assert P.features.features_into(op, low, X, F1, zero_rows=False) is None
    torch.cuda.synchronize()
    assert z.size == 0 and torch.equal(F0, F1)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_overlapped_host_upload_bit_identical(c1_golden, dtype):
    """Multi-panel blocks in pinned host memory are uploaded panel by panel on a copy stream,
    narrowest panel first, each packed when its filter starts (option h2d_overlap): features,
    filter output and eigencount are the same bytes as the one-copy path."""
    import torch

    from paper_1602_02018_b200.spectrum import eigencount

    g, _ = c1_graph()
    op = P.laplacian_op(g, dtype=dtype)
    low = P.design_lowpass(0.4, 50)
    narrow = 8 if dtype == "float32" else 4
    X = torch.empty((g.num_nodes, 31), dtype=torch.float64).pin_memory().numpy()
    X[:] = np.random.default_rng(17).standard_normal(X.shape)
    out = {}
    for ov in (0, 1):
        with options(h2d_overlap=ov, panel_width=narrow):
            F = torch.empty(X.shape, dtype=torch.float64).pin_memory().numpy()
            z = P.features.features_into(op, low, X, F)
            Y = P.apply_filter(low, op, X)
            cnt = eigencount(op, 0.4, rng=np.random.default_rng(3), num_signals=31, _signals=X)
            out[ov] = (F.copy(), z, Y, cnt.count)
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1].tolist() == out[1][1].tolist()
    assert np.array_equal(out[0][2], out[1][2])
    assert out[0][3] == out[1][3]
