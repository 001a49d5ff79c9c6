"""Time the device k-means (all replicates) on C3-shaped reduced features (n=922, d=56, k=100),
or on a headline capture's real reduced features: python tools/kmeans_timing.py [c4|c3]."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1602_02018_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
if len(sys.argv) > 1:
    gz = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"pipeline_{sys.argv[1]}.npz")
    pts = np.ascontiguousarray(gz["reduced_features"])
    n, d = pts.shape
    k = int(gz["truth"].max()) + 1
else:
    k, n, d = 100, 922, 56
    centers = rng.standard_normal((k, d))
    pts = centers[rng.integers(k, size=n)] + 0.3 * rng.standard_normal((n, d))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
cfg = P.KmeansConfig(k=k, seed=3)
P.kmeans(pts, cfg)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lab = P.kmeans(pts, cfg)
    print(f"kmeans 20 replicates: {(time.perf_counter() - t0) * 1e3:.2f} ms, iterations {lab.iterations_run}", flush=True)

# split: seeding only (max_iters = 0) vs full, 1 vs 20 replicates (direct ABI calls)
from paper_1602_02018_b200 import _lib  # noqa: E402
from paper_1602_02018_b200.kmeans import _MASK64  # noqa: E402


def run(R, max_iters):
    children = np.random.SeedSequence(3).spawn(R)
    first = np.empty(R, dtype=np.int64)
    pcg = np.empty((R, 4), dtype=np.uint64)
    for r, ch in enumerate(children):
        g = np.random.default_rng(ch)
        first[r] = g.integers(n)
        st = g.bit_generator.state["state"]
        pcg[r] = (st["state"] >> 64, st["state"] & _MASK64, st["inc"] >> 64, st["inc"] & _MASK64)
    lab = np.empty((R, n), dtype=np.int64)
    inert, its = np.empty(R), np.empty(R, dtype=np.int64)
    stat = np.empty(R, dtype=np.int32)
    t0 = time.perf_counter()
    _lib.call("csc_kmeans_replicates", _lib.ptr(pts), n, d, k, R, _lib.ptr(first), _lib.ptr(pcg), None, max_iters,
              1e-6, _lib.ptr(lab), None, _lib.ptr(inert), _lib.ptr(its), _lib.ptr(stat), 0, None)
    return (time.perf_counter() - t0) * 1e3, its.max()


for R in (1, 20):
    for mi in (0, 300):
        run(R, mi)
        t, it = run(R, mi)
        print(f"replicates {R:2d} max_iters {mi:3d}: {t:7.2f} ms (max iterations {it})", flush=True)
