"""run_csc at BASELINE C2 (SBM N=1e5, k=20), the headline C3 (SBM N=1e6, k=100) and C4 (DC-SBM
N=334,863, k=250)
against the REAL reference's run_csc on the same graph, seed and d (tests/golden/make_golden.py
--c3 / --c4, which wraps the stage functions reference pipeline.py:19-26 binds by name).

Every stage is compared: the dichotomy trace (probe frequencies exact, counts within the
dtype's tolerance), lambda_k_hat (exact), the sampled rows (exact), the features on a fixed
row subsample (1e-9 fp64 / 1e-4 fp32 relative), the reduced k-means labels, the per-column
CG iterations (exact in fp64), the interpolated indicators on the row subsample (1e-9 fp64) and
the final labels (ARI >= 0.99).  Exception, measured at C4: CG columns that need ~35+
iterations of the ill-conditioned interpolation system are decided by rounding -- our own
Clenshaw and forward recurrences (the same polynomial, operations reordered) disagree on them by
the same amount as we disagree with the reference (iterations +-2, indicator columns up to
2e-3; profiles/r02_headline_parity.txt) -- so a column may miss the reference only if it is
rounding-unstable in that sense (<= 2 % of the columns).  Our stages are captured the same way, by wrapping the names our
pipeline module binds.
"""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, golden, relerr, sbm_config
from gpu_util import options
import paper_1602_02018_b200 as P
from paper_1602_02018_b200 import pipeline as pl

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-9, "float32": 1e-4}
_graphs: dict = {}


def _graph(tag):
    if tag not in _graphs:
        _graphs.clear()
        if tag == "c2cap":
            _graphs[tag] = P.sbm_generate(sbm_config(100_000, 20))
        elif tag == "c3":
            _graphs[tag] = P.sbm_generate(sbm_config(1_000_000, 100))
        else:
            from paper_1602_02018_b200.sbm import c4_config

            g, truth, _ = P.dcsbm_generate(c4_config())
            _graphs[tag] = (g, truth)
    return _graphs[tag]


def _column_relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b, axis=0)
    return np.linalg.norm(a - b, axis=0) / np.where(nb > 0, nb, 1.0)


def _captured_run(op, params, rows):
    cap = {}
    saved = {n: getattr(pl, n) for n in ("estimate_lambda_k", "features_into", "draw_sampling", "kmeans",
                                         "block_cg_into")}

    def wrap(name):
        fn = saved[name]

        def inner(*a, **kw):
            out = fn(*a, **kw)
            if name == "features_into":  # (op, filt, X, F): keep the subsampled rows of F
                cap["features_rows"] = a[3][rows].cpu().numpy()
            else:
                cap[name] = out
            return out

        return inner

    for n in saved:
        setattr(pl, n, wrap(n))
    try:
        res = P.run_csc(op, params)
    finally:
        for n, fn in saved.items():
            setattr(pl, n, fn)
    return res, cap


@pytest.mark.parametrize("tag", ["c2cap", "c3", "c4"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_run_csc_headline_matches_reference(tag, dtype):
    if not (GOLDEN / f"pipeline_{tag}.npz").exists():
        pytest.skip(f"{tag} fixture not generated")
    gz = golden(f"pipeline_{tag}")
    graph, truth = _graph(tag)
    N = graph.num_nodes
    assert N == int(gz["num_nodes"]) and int(graph.indptr[-1]) == int(gz["nnz"])
    assert np.array_equal(np.asarray(truth), gz["truth"])
    k = int(np.max(gz["truth"])) + 1
    d = int(math.ceil(4 * math.log(N)))
    rows = gz["rows"]
    op = P.laplacian_op(graph, dtype=dtype)
    res, cap = _captured_run(op, P.CscParams(k=k, d=d, seed=0), rows)
    tol = TOL[dtype]
    diag = res.diagnostics

    # 1. dichotomy: same probe sequence, counts within tolerance, same cut-off
    est = cap["estimate_lambda_k"]
    trace = np.asarray(est.trace)
    ref_trace = gz["trace"]
    assert trace.shape == ref_trace.shape
    assert np.array_equal(trace[:, 0], ref_trace[:, 0])
    assert np.max(np.abs(trace[:, 1] - ref_trace[:, 1]) / ref_trace[:, 1]) <= tol
    assert diag["lambda_k_hat"] == float(gz["lambda_k_hat"])
    assert diag["lambda_warning"] == bool(gz["lambda_warning"])

    # 2. features on the row subsample, then the sampled rows
    assert relerr(cap["features_rows"], gz["features_rows"]) <= tol
    assert np.array_equal(cap["draw_sampling"].indices, gz["indices"])
    assert diag["zero_feature_rows"] == gz["zero_rows"].tolist()

    # 3. reduced k-means
    lab = cap["kmeans"]
    if dtype == "float64":
        assert np.array_equal(lab.labels, gz["kmeans_labels"])
        assert abs(lab.inertia - float(gz["kmeans_inertia"])) <= 1e-9 * float(gz["kmeans_inertia"])
    else:
        assert P.adjusted_rand_index(lab.labels, gz["kmeans_labels"]) >= 0.99

    # 4. block CG and assignment
    if dtype == "float64":
        its, ref_its = np.asarray(diag["solver_iterations"]), gz["solver_iterations"]
        err = _column_relerr(res.soft[rows], gz["soft_rows"])
        off = (its != ref_its) | (err > tol)
        if off.any():
            # CG columns that need many iterations on an ill-conditioned system are decided by
            # rounding: the same solve in another exact-arithmetic-equivalent operation order
            # (the forward recurrence instead of Clenshaw) moves them by as much.  Every column
            # that misses the reference must be such a column, and by no more than 100x that.
            with options(recurrence=1):
                alt = P.run_csc(op, P.CscParams(k=k, d=d, seed=0))
            alt_its = np.asarray(alt.diagnostics["solver_iterations"])
            spread = _column_relerr(alt.soft[rows], res.soft[rows])
            unstable = (alt_its != its) | (spread > tol)
            assert not (off & ~unstable).any(), [(int(j), int(its[j]), int(ref_its[j]), float(err[j]))
                                                  for j in np.flatnonzero(off & ~unstable)]
            same_its = off & (its == ref_its)
            assert np.all(err[same_its] <= 100.0 * spread[same_its]), (err[same_its], spread[same_its])
            assert off.sum() <= 0.02 * k
        assert np.all(np.abs(its - ref_its) <= 2)
        stable_cols = ~off
        assert np.all(err[stable_cols] <= tol)
    assert diag["solver_converged"] == gz["solver_converged"].tolist()
    assert P.adjusted_rand_index(res.labels, gz["labels"]) >= 0.99
    assert abs(P.adjusted_rand_index(truth, res.labels) - float(gz["ari_truth"])) < 0.01
    ref_diag = json.loads(bytes(gz["diagnostics_json"]).decode())
    for key in ("num_nodes", "num_edges", "k", "n", "d", "p", "gamma", "seed", "lambda_source", "probe_iterations",
                "ridge"):
        assert diag[key] == ref_diag[key], key
