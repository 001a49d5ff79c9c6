"""Generate the golden fixtures from the REAL reference package.

Run in the build container only (the reference lives at /root/reference and is
not shipped to the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--c2] [--c3] [--c4]

--c2cap / --c3 / --c4 run the reference's run_csc ONCE at BASELINE configs 2-4 (C3: SBM N=1e6,
k=100, d=56, ~1-2 h of one CPU core; C4: the repo's DC-SBM graph, N=334,863, k=250,
d=51, fed through the reference's build_graph) and capture every stage's output by
wrapping the stage functions run_csc binds by name (pipeline.py:19-26), the seam the
reference's own tests monkeypatch (test_pipeline.py:101-110).  Large arrays are stored
on a fixed row subsample only (features, soft) so the fixtures stay ~1 MB.

Outputs (committed, small): tests/golden/graphs.npz, filter_c1.npz,
pipeline_c1.npz, formats.npz (the reference's own on-disk formats: feature dump,
labels CSV, result JSON, dichotomy trace CSV), edgelists.npz (read_edge_list on messy and
failing files, write_edge_list bytes) and, with --c2, pipeline_c2.npz
(scalars, indices and labels only; the reference takes ~2.5 min there).
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np

import cscluster as ref
from cscluster._rng import substream, substream_seed

OUT = Path(__file__).resolve().parent


def sbm_config(N, k, s=16.0, seed=0):
    return ref.SbmConfig(num_nodes=N, k=k, avg_degree=s, epsilon=ref.critical_epsilon(s, k) / 4.0, seed=seed)


def graphs():
    out = {}
    g, truth = ref.sbm_generate(sbm_config(1000, 20))
    out.update(c1_indptr=g.indptr, c1_indices=g.indices, c1_weights=g.weights, c1_degrees=g.degrees, c1_truth=truth)
    # messy weighted edge list: same-direction duplicates, reversed duplicates, explicit zeros, isolated tail
    rng = np.random.default_rng(2024)
    m = 400
    src = rng.integers(0, 70, m)
    dst = rng.integers(0, 70, m)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    w = np.round(rng.uniform(0.0, 3.0, src.size), 3)
    w[::17] = 0.0
    dup = rng.choice(src.size, 60, replace=False)
    src = np.concatenate([src, src[dup], dst[dup[:30]]])
    dst = np.concatenate([dst, dst[dup], src[dup[:30]]])
    w = np.concatenate([w, np.round(rng.uniform(0.0, 2.0, 60), 3), np.round(rng.uniform(0.0, 4.0, 30), 3)])
    edges = np.column_stack([src, dst, w]).astype(np.float64)
    gm = ref.build_graph(edges, num_nodes=75)
    out.update(messy_edges=edges, messy_indptr=gm.indptr, messy_indices=gm.indices, messy_weights=gm.weights,
               messy_degrees=gm.degrees)
    # weighted random graph (reference tests/helpers.py random_graph style) + Laplacian apply
    rng = np.random.default_rng(11)
    e = [(i, j, rng.uniform(0.2, 2.0)) for i in range(60) for j in range(i + 1, 60) if rng.random() < 0.12]
    gw = ref.build_graph(e, num_nodes=60)
    X = np.random.default_rng(12).standard_normal((60, 4))
    opw = ref.laplacian_op(gw)
    out.update(w60_edges=np.asarray(e), w60_indptr=gw.indptr, w60_indices=gw.indices, w60_weights=gw.weights,
               w60_X=X, w60_LX=opw.apply(X), w60_low=ref.apply_filter(ref.design_lowpass(0.9, 30), opw, X))
    np.savez_compressed(OUT / "graphs.npz", **out)


def filter_c1():
    g, _ = ref.sbm_generate(sbm_config(1000, 20))
    op = ref.laplacian_op(g)
    X = np.random.default_rng(1).standard_normal((1000, 28))
    low = ref.design_lowpass(0.37, 50)
    high = ref.matched_highpass(low)
    out = dict(
        X=X, low_coeffs=low.coeffs, high_coeffs=high.coeffs, Y_low=ref.apply_filter(low, op, X),
        Y_high=ref.apply_filter(high, op, X), LX=op.apply(X[:, :4]), ridge=ref.psd_ridge(high),
        Y_order2=ref.apply_filter(ref.design_lowpass(1.3, 2), op, X[:, :5]),
        Y_order1=ref.apply_filter(ref.design_lowpass(0.8, 1, damping="none"), op, X[:, :3]),
    )
    np.savez_compressed(OUT / "filter_c1.npz", **out)


def pipeline(N, k, d, seed, full: bool):
    g, truth = ref.sbm_generate(sbm_config(N, k))
    op = ref.laplacian_op(g)
    params = ref.CscParams(k=k, d=d, seed=seed)
    prm = params.resolve(N)
    est = ref.estimate_lambda_k(op, k, order=prm.p, rng=substream(seed, "probe"))
    low = ref.design_lowpass(est.lambda_k_hat, prm.p)
    sig = ref.generate_signals(N, d, "gaussian", substream(seed, "signals"))
    feats = ref.build_features(op, low, sig)
    samp = ref.draw_sampling(N, prm.n, substream(seed, "sampling"), exclude=feats.zero_rows)
    lab = ref.kmeans(feats.rows[samp.indices], ref.KmeansConfig(k=k, seed=substream_seed(seed, "kmeans")))
    res = ref.run_csc(op, params)
    assert res.diagnostics["lambda_k_hat"] == est.lambda_k_hat
    out = dict(
        trace=np.asarray(est.trace), lambda_k_hat=est.lambda_k_hat, indices=samp.indices,
        kmeans_labels=lab.labels, kmeans_inertia=lab.inertia, labels=res.labels, truth=truth,
        solver_iterations=np.asarray(res.diagnostics["solver_iterations"]),
        solver_residuals=np.asarray(res.diagnostics["solver_residuals"]), ridge=res.diagnostics["ridge"],
        zero_rows=feats.zero_rows, result_json=np.frombuffer(res.to_json().encode(), dtype=np.uint8),
        ari_truth=ref.adjusted_rand_index(truth, res.labels), timings=json.dumps(res.diagnostics["timings"]),
    )
    if full:
        out.update(features=feats.rows, soft=res.soft)
    return out


def capture_run(graph, truth, k, d, seed, tag):
    """run_csc once with every stage's result captured (see module docstring)."""
    import time

    import cscluster.pipeline as rp

    cap = {}

    def wrap(name):
        fn = getattr(rp, name)

        def inner(*a, **kw):
            out = fn(*a, **kw)
            cap[name] = out
            return out

        return inner

    saved = {n: getattr(rp, n) for n in ("estimate_lambda_k", "build_features", "draw_sampling", "kmeans",
                                         "interpolate_all", "generate_signals")}
    for n in saved:
        setattr(rp, n, wrap(n))
    try:
        op = ref.laplacian_op(graph)
        t0 = time.perf_counter()
        res = ref.run_csc(op, ref.CscParams(k=k, d=d, seed=seed))
        wall = time.perf_counter() - t0
    finally:
        for n, fn in saved.items():
            setattr(rp, n, fn)
    N = graph.num_nodes
    est, feats, samp = cap["estimate_lambda_k"], cap["build_features"], cap["draw_sampling"]
    lab, (soft, info) = cap["kmeans"], cap["interpolate_all"]
    rows = np.arange(0, N, max(1, N // 512), dtype=np.int64)
    lab_dtype = np.uint8 if k <= 255 else np.int32
    out = dict(
        num_nodes=N, nnz=graph.indptr[-1], trace=np.asarray(est.trace), lambda_k_hat=est.lambda_k_hat,
        lambda_warning=est.warning, indices=samp.indices, kmeans_labels=lab.labels, kmeans_inertia=lab.inertia,
        reduced_features=feats.rows[samp.indices], rows=rows, features_rows=feats.rows[rows],
        soft_rows=soft[rows], soft_colnorm=np.linalg.norm(soft, axis=0),
        labels=res.labels.astype(lab_dtype), truth=np.asarray(truth).astype(lab_dtype),
        solver_iterations=info.iterations, solver_residuals=info.residuals, solver_converged=info.converged,
        ridge=res.diagnostics["ridge"], zero_rows=feats.zero_rows,
        diagnostics_json=np.frombuffer(json.dumps(res.to_dict()["diagnostics"], sort_keys=True).encode(),
                                       dtype=np.uint8),
        ari_truth=ref.adjusted_rand_index(truth, res.labels), timings=json.dumps(res.diagnostics["timings"]),
        wall_s=wall,
    )
    print(tag, "wall", round(wall, 1), "s", json.dumps(res.diagnostics["timings"]), flush=True)
    return out


def formats():
    """Bytes written by the reference's save_features (features.py:101-116), save_labels_csv /
    save_json (result.py:50-58) and trace_to_csv (spectrum.py:143-152)."""
    import tempfile

    from cscluster import features as rfeat, spectrum as rspec

    rng = np.random.default_rng(21)
    rows = rng.standard_normal((7, 3))
    rows[2] = 0.0
    prov = {"distribution": "gaussian", "filter": {"cutoff": 0.5, "order": 50}, "seed": 5}
    fm = rfeat.FeatureMatrix(rows=rows, normalized=True, zero_rows=np.array([2], dtype=np.int64), provenance=prov)
    g, _ = ref.sbm_generate(sbm_config(1000, 20))
    op = ref.laplacian_op(g)
    res = ref.run_csc(op, ref.CscParams(k=20, d=int(math.ceil(4 * math.log(1000))), seed=0))
    est = rspec.estimate_lambda_k(op, 20, rng=substream(0, "probe"))
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        rfeat.save_features(fm, td / "f.bin")
        res.save_labels_csv(td / "labels.csv")
        res.save_json(td / "result.json")
        rspec.trace_to_csv(est, td / "trace.csv")
        blob = {name: np.frombuffer((td / name).read_bytes(), dtype=np.uint8)
                for name in ("f.bin", "labels.csv", "result.json", "trace.csv")}
    np.savez_compressed(OUT / "formats.npz", features_dump=blob["f.bin"], labels_csv=blob["labels.csv"],
                        result_json=blob["result.json"], trace_csv=blob["trace.csv"], rows=rows,
                        provenance=np.frombuffer(json.dumps(prov).encode(), dtype=np.uint8))


EDGE_TEXT = (
    "# messy edge list: comments, blank lines, CRLF and lone CR, tabs, other ASCII whitespace\n"
    "# nodes 12\n"
    "0 1\n"
    "\n"
    "   \t\n"
    "1\t2 0.5\r\n"
    "2 3 1e-3\r"
    "3 4 .5\n"
    "4\x0b5\x0c5.\n"
    "5 6 +2\n"
    "6 7 1_000.5\n"
    "1_0 11 3\n"
    "007 8 2.25E+1\n"
    "+8 9 0.1\n"
    "9 \u0663 7\n"
    "3\u00a010 1.5\n"
    "#nodes 99 trailing tokens are not a header\n"
    "# nodes +14\n"
    "10 11 12345678901234567890.5\n"
    "2 3 1e-3\n"
    "  0 11   4  "
)

EDGE_ERRORS = {
    "too_many": "0 1\n1 2 3 4\n",
    "too_few": "# header\n0\n",
    "bad_int": "0 1\n0 x 1.0\n",
    "bad_float": "0 1 abc\n",
    "bad_underscore": "1__0 2\n",
    "self_loop": "0 0 1.0\n",
}


def edgelists():
    """The reference's read_edge_list (graph.py:177-214) on a messy file and on failing files
    (message with the path replaced by <path>), and write_edge_list's bytes (graph.py:215-225)
    for a graph whose weights span many magnitudes."""
    import tempfile

    out = {}
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        path = td / "messy.edges"
        path.write_bytes(EDGE_TEXT.encode("utf-8"))
        g = ref.read_edge_list(path)
        out.update(messy_text=np.frombuffer(EDGE_TEXT.encode("utf-8"), dtype=np.uint8), messy_n=g.num_nodes,
                   messy_indptr=g.indptr, messy_indices=g.indices, messy_weights=g.weights)
        msgs = {}
        for name, text in EDGE_ERRORS.items():
            p = td / f"{name}.edges"
            p.write_text(text)
            try:
                ref.read_edge_list(p)
                msgs[name] = None
            except Exception as exc:  # GraphError (ValueError)
                msgs[name] = [type(exc).__name__, str(exc).replace(str(p), "<path>")]
        out["error_texts"] = np.frombuffer(json.dumps(EDGE_ERRORS).encode(), dtype=np.uint8)
        out["error_msgs"] = np.frombuffer(json.dumps(msgs).encode(), dtype=np.uint8)
        rng = np.random.default_rng(31)
        n, m = 60, 400
        src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
        keep = src != dst
        mags = 10.0 ** rng.uniform(-9, 21, m)
        w = np.where(rng.random(m) < 0.3, np.round(mags), mags)
        w[:6] = [1.0, 0.1, 1e16, 1e-5, 123456789012345678.0, 2.5e-7]
        wg = ref.build_graph(np.column_stack([src[keep], dst[keep], w[keep]]), num_nodes=n + 3)
        ref.write_edge_list(wg, td / "w.edges")
        out.update(write_n=wg.num_nodes, write_indptr=wg.indptr, write_indices=wg.indices, write_weights=wg.weights,
                   write_bytes=np.frombuffer((td / "w.edges").read_bytes(), dtype=np.uint8))
    np.savez_compressed(OUT / "edgelists.npz", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true")
    ap.add_argument("--c2cap", action="store_true", help="stage capture at C2 (pipeline_c2cap.npz, ~2.5 min)")
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--only", action="store_true", help="skip the small fixtures")
    args = ap.parse_args()
    if args.c2cap:
        N, k = 100_000, 20
        g, truth = ref.sbm_generate(sbm_config(N, k))
        out = capture_run(g, truth, k, int(math.ceil(4 * math.log(N))), 0, "c2")
        np.savez_compressed(OUT / "pipeline_c2cap.npz", **out)
    if args.c3:
        N, k = 1_000_000, 100
        g, truth = ref.sbm_generate(sbm_config(N, k))
        out = capture_run(g, truth, k, int(math.ceil(4 * math.log(N))), 0, "c3")
        np.savez_compressed(OUT / "pipeline_c3.npz", **out)
    if args.c4:
        sys.path.insert(0, str(OUT.parents[1]))
        from paper_1602_02018_b200.sbm import c4_config, dcsbm_edges

        cfg = c4_config()
        src, dst, truth, _ = dcsbm_edges(cfg)
        edges = np.column_stack([src, dst, np.ones(src.size)]).astype(np.float64)
        g = ref.build_graph(edges, num_nodes=cfg.num_nodes)
        out = capture_run(g, truth, cfg.k, int(math.ceil(4 * math.log(cfg.num_nodes))), 0, "c4")
        out["edges_digest"] = np.frombuffer(__import__("hashlib").sha256(
            np.ascontiguousarray(np.column_stack([src, dst]).astype(np.int64)).tobytes()).digest(), dtype=np.uint8)
        np.savez_compressed(OUT / "pipeline_c4.npz", **out)
    if args.only:
        return
    graphs()
    filter_c1()
    formats()
    edgelists()
    np.savez_compressed(OUT / "pipeline_c1.npz", **pipeline(1000, 20, int(math.ceil(4 * math.log(1000))), 0, True))
    if args.c2:
        np.savez_compressed(OUT / "pipeline_c2.npz", **pipeline(100_000, 20, int(math.ceil(4 * math.log(1e5))), 0, False))
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
