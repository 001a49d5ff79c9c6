"""Host-side logic of the drop-in (no GPU): designs, RNG streams, k-means, sampling, params, generators."""

from __future__ import annotations

import re

import numpy as np
import pytest

from conftest import D_C1, ROOT, c1_config, has_gpu
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P
from paper_1602_02018_b200 import _lib
from paper_1602_02018_b200._rng import substream, substream_seed
from paper_1602_02018_b200.features import generate_signals
from paper_1602_02018_b200.sbm import dcsbm_edges


# ---- C ABI surface ----------------------------------------------------------


def header_functions() -> list[str]:
    text = (ROOT / "include" / "csc_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(csc_\w+)\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES)
    assert lib.csc_abi_version() == 1


def test_options_roundtrip_and_validation():
    old = _lib.get_option("panel_width")
    _lib.set_option("panel_width", 16)
    assert _lib.get_option("panel_width") == 16
    _lib.set_option("panel_width", old)
    with pytest.raises(ValueError):
        _lib.set_option("recurrence", 7)
    with pytest.raises(ValueError):
        _lib.set_option("no_such_knob", 1)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_hot_path_fails_loudly_without_gpu():
    with pytest.raises(RuntimeError, match="CUDA"):
        P.build_graph([(0, 1, 1.0)])


# ---- filter design (bit-identical coefficients) ------------------------------


@pytest.mark.parametrize("cut,order,damp", [(0.37, 50, "jackson"), (1.3, 2, "jackson"), (0.8, 1, "none"),
                                            (1.999999999999, 50, "jackson")])
def test_design_matches_oracle(cut, order, damp):
    low = P.design_lowpass(cut, order, damp)
    assert np.array_equal(low.coeffs, O.lowpass_coeffs(cut, order, damp))
    hi = P.matched_highpass(low)
    assert np.array_equal(hi.coeffs, O.highpass_coeffs(O.lowpass_coeffs(cut, order, damp)))
    assert P.psd_ridge(hi) == O.psd_ridge(hi.coeffs)
    grid = np.linspace(0, 2, 301)
    assert np.array_equal(low.evaluate(grid), O.evaluate(low.coeffs, grid))


def test_design_golden(filter_golden):
    low = P.design_lowpass(0.37, 50)
    assert np.array_equal(low.coeffs, filter_golden["low_coeffs"])
    assert P.psd_ridge(P.matched_highpass(low)) == float(filter_golden["ridge"])


def test_design_validation_and_json(tmp_path):
    for bad in (0.0, 2.0):
        with pytest.raises(ValueError):
            P.design_lowpass(bad, 10)
    with pytest.raises(ValueError):
        P.design_lowpass(1.0, 0)
    with pytest.raises(ValueError):
        P.matched_highpass(P.design_highpass(0.5, 10))
    f = P.design_lowpass(0.7321, 33)
    f.save(tmp_path / "f.json")
    g = P.PolyFilter.load(tmp_path / "f.json")
    assert np.array_equal(g.coeffs, f.coeffs) and g.cutoff == f.cutoff and g.kind == f.kind


# ---- random streams, sampling, k-means ----------------------------------------


def test_substreams_match_oracle():
    for stage in ("probe", "signals", "sampling", "kmeans"):
        a = substream(7, stage).standard_normal(5)
        b = O.substream(7, stage).standard_normal(5)
        assert np.array_equal(a, b)
        assert substream_seed(7, stage) == O.substream_seed(7, stage)


def test_signals_and_sampling_match_golden(c1_golden):
    sig = generate_signals(1000, D_C1, "gaussian", substream(0, "signals"))
    ref = O.gaussian_signals(1000, D_C1, O.substream(0, "signals"))
    assert np.array_equal(sig.matrix, ref)
    s = P.draw_sampling(1000, 120, substream(0, "sampling"), exclude=c1_golden["zero_rows"])
    assert np.array_equal(s.indices, c1_golden["indices"])
    with pytest.raises(ValueError):
        P.draw_sampling(5, 6, 0)
    with pytest.raises(ValueError):
        P.draw_sampling(5, 4, 0, exclude=np.arange(3))


def test_kmeanspp_seeding_consumes_rng_like_reference():
    from paper_1602_02018_b200.kmeans import _initial_centers

    rng_pts = np.random.default_rng(3)
    pts = np.concatenate([rng_pts.normal(c, 0.3, (40, 5)) for c in range(6)])
    for child in np.random.SeedSequence(11).spawn(3):
        a = _initial_centers(pts, 6, np.random.default_rng(child), "kmeanspp")
        b = O._seed_kmeanspp(pts, 6, np.random.default_rng(child))
        assert np.array_equal(a, b)


def test_labels_to_indicators():
    ind = P.labels_to_indicators(np.array([0, 2, 1, 2]), 3, 4)
    assert ind.tolist() == [[1, 0, 0], [0, 0, 1], [0, 1, 0], [0, 0, 1]]
    with pytest.raises(ValueError):
        P.labels_to_indicators(np.array([0, 3]), 3, 2)


# ---- parameters --------------------------------------------------------------


def test_params_resolve_and_dict():
    prm = P.CscParams(k=20).resolve(1000)
    assert (prm.n, prm.d) == (120, 20)
    assert P.default_num_samples(3) == 7 and P.default_num_signals(7) == 8
    with pytest.raises(ValueError, match="n="):
        P.CscParams(k=5, n=3).resolve(100)
    with pytest.raises(ValueError, match="k must"):
        P.CscParams(k=1).resolve(100)
    with pytest.raises(ValueError, match="exceeds"):
        P.CscParams(k=3, n=50).resolve(20)
    with pytest.raises(ValueError, match="gamma"):
        P.CscParams(k=3, gamma=0.0).resolve(100)
    p = P.CscParams(k=7, p=80, gamma=2e-3, seed=5)
    assert P.CscParams.from_dict(p.to_dict()) == p
    with pytest.raises(ValueError, match="unknown"):
        P.CscParams.from_dict({"k": 3, "shrink": True})


# ---- generators and metric -----------------------------------------------------


def test_sbm_config_and_threshold():
    cfg = c1_config()
    assert cfg.sizes == [50] * 20
    assert abs(P.critical_epsilon(16.0, 20) - 12.0 / 92.0) < 1e-15
    with pytest.raises(ValueError):
        P.SbmConfig(num_nodes=10, k=2, avg_degree=4.0, epsilon=1.5)


def test_dcsbm_degrees_heavy_tailed():
    cfg = P.SbmConfig(num_nodes=20000, k=20, avg_degree=5.5, epsilon=P.critical_epsilon(5.5, 20) / 4.0, seed=0)
    src, dst, labels, theta = dcsbm_edges(cfg)
    assert np.all(src < dst)
    key = src * cfg.num_nodes + dst
    assert np.unique(key).size == key.size
    deg = np.bincount(np.concatenate([src, dst]), minlength=cfg.num_nodes)
    assert 4.8 < deg.mean() < 6.0
    assert deg.max() > 8 * deg.mean()  # heavy tail (Pareto 2.5 propensities)
    for a in range(cfg.k):
        assert abs(theta[labels == a].mean() - 1.0) < 1e-12
    intra = (labels[src] == labels[dst]).mean()
    expect = 1.0 / (1.0 + cfg.epsilon * (cfg.k - 1))
    assert abs(intra - expect) < 0.03


def test_ari():
    a = np.array([0, 0, 1, 1, 2, 2])
    assert P.adjusted_rand_index(a, a) == 1.0
    assert P.adjusted_rand_index(a, np.array([5, 5, 3, 3, 1, 1])) == 1.0
    assert abs(P.adjusted_rand_index(a, np.array([0, 1, 0, 1, 0, 1]))) < 0.5


def test_numpy_ziggurat_restatement():
    """Tables read from numpy's binary + the restated PCG64/ziggurat reproduce numpy (incl. slow paths)."""
    from paper_1602_02018_b200 import _npzig as Z

    ki, wi, fi = Z.ziggurat_tables()  # verifies internally on 2 x 20000 draws
    rng = np.random.default_rng(99)
    s, inc = Z.pcg_state(rng)
    ns = Z.NormalStream(s, inc, (ki, wi, fi))
    got = np.array([ns.normal() for _ in range(50_000)])
    assert np.array_equal(got, rng.standard_normal(50_000))
    assert (ns.s, ns.inc) == Z.pcg_state(rng)
    assert ns.raw_count > 50_000  # slow paths consumed extra raws


def test_numpy_geometric_restatement():
    """numpy's geometric (exponential ziggurat / inversion, and the search branch) restated draw for draw."""
    from paper_1602_02018_b200 import _npzig as Z

    tabs = Z.ziggurat_tables(), Z.exponential_tables()
    for p in (2e-5, 1e-3, 0.3, 0.5):
        rng = np.random.default_rng(7)
        ns = Z.NormalStream(*Z.pcg_state(rng), *tabs)
        got = [ns.geometric(p) for _ in range(4000)]
        assert np.array_equal(got, rng.geometric(p, size=4000)), p
        assert (ns.s, ns.inc) == Z.pcg_state(rng)


def test_sbm_pair_table_matches_reference_loop():
    """The per-pair table handed to csc_sbm_edges follows _success_positions' batch rule and pair order."""
    import math

    from paper_1602_02018_b200.sbm import SbmConfig, _sbm_pairs

    cfg = SbmConfig(num_nodes=2003, k=7, avg_degree=9, epsilon=0.05, seed=1)
    a, b, diag, cells, q, batch, first, sizes, search = _sbm_pairs(cfg)
    assert not search
    exp = []
    for i in range(cfg.k):
        for j in range(i, cfg.k):
            c = cfg.sizes[i] * (cfg.sizes[i] - 1) // 2 if i == j else cfg.sizes[i] * cfg.sizes[j]
            qq = cfg.q1 if i == j else cfg.q2
            if c > 0 and qq > 0:
                mean = qq * c
                exp.append((i, j, c, max(64, int(mean + 10.0 * math.sqrt(mean) + 10.0))))
    assert [(int(x), int(y), int(c), int(bb)) for x, y, c, bb in zip(a, b, cells, batch)] == exp


def test_new_abi_argument_validation():
    """csc_kmeans_replicates / csc_sbm_edges reject bad arguments before touching a device."""
    pts = np.zeros((3, 2))
    lab = np.empty((1, 3), dtype=np.int64)
    inert, its = np.empty(1), np.empty(1, dtype=np.int64)
    with pytest.raises(ValueError, match="at least k"):
        _lib.call("csc_kmeans_replicates", _lib.ptr(pts), 3, 2, 5, 1, None, None, _lib.ptr(np.zeros((1, 5, 2))), 10,
                  1e-6, _lib.ptr(lab), None, _lib.ptr(inert), _lib.ptr(its), None, 0, None)
    with pytest.raises(ValueError, match="seeding states or initial centroids"):
        _lib.call("csc_kmeans_replicates", _lib.ptr(pts), 3, 2, 2, 1, None, None, None, 10, 1e-6, _lib.ptr(lab),
                  None, _lib.ptr(inert), _lib.ptr(its), None, 0, None)
    one = lambda v, dt: np.array([v], dtype=dt)  # noqa: E731
    n_e = np.zeros(1, dtype=np.int64)
    args = [one(100, np.int64), one(np.log1p(-0.5), np.float64), one(64, np.int64), one(1, np.int32),
            one(0, np.int64), one(0, np.int64), one(15, np.int64)]
    with pytest.raises(ValueError, match="1/3"):
        _lib.call("csc_sbm_edges", 1, 2, 3, 5, 1, *[_lib.ptr(x) for x in args], 0, None, None, _lib.ptr(n_e), None,
                  0, None)


def test_feature_dump_format_matches_reference():
    """save_features writes the reference's bytes (features.py:101-116); load_features reads its dump."""
    import json
    from pathlib import Path

    from conftest import ROOT
    from paper_1602_02018_b200.features import FeatureMatrix, load_features, save_features

    gold = np.load(Path(ROOT) / "tests" / "golden" / "formats.npz")
    prov = json.loads(bytes(gold["provenance"]).decode())
    fm = FeatureMatrix(rows=gold["rows"], normalized=True, zero_rows=np.array([2], dtype=np.int64), provenance=prov)
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "f.bin"
        save_features(fm, p)
        assert p.read_bytes() == bytes(gold["features_dump"])
        q = Path(td) / "ref.bin"
        q.write_bytes(bytes(gold["features_dump"]))
        back = load_features(q)
    assert np.array_equal(back.rows, gold["rows"]) and back.zero_rows.tolist() == [2]
    assert back.normalized is True and back.provenance == prov


def test_bench_reference_arm_contract_on_cpu():
    """bench.py --impl reference (the reference algorithm on the host cores) prints one JSON line
    with the contract's keys; C1 keeps it to a second."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "dtype", "config", "e2e", "cpu_baseline"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] in ("port", "reference")
    assert line["scaling"] == "strong" and line["n_gpus"] == 1


def test_bench_self_launches_ranks_for_gpus_n():
    """bench.py --gpus 2 without WORLD_SIZE re-launches itself under torch.distributed.run: two
    ranks start, rank 0 alone prints the line (reference arm: CPU-only, so it runs here)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=300, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert "2 rank(s)" in line["config"]["parallelism"]
