"""Time edge-list text I/O at a BASELINE size on the host: the library's multi-threaded
reader/writer (csc_edgelist_read / csc_edgelist_write) against the reference algorithm
(oracle restatement of graph.py:188-225, a Python line loop).  No GPU needed.

python tools/edgelist_timing.py [--nodes 1000000] [--degree 16] [--oracle-lines 2000000]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle import cpu_ref as O  # noqa: E402
from paper_1602_02018_b200 import _lib, graph as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=1_000_000)
    ap.add_argument("--degree", type=float, default=16.0)
    ap.add_argument("--oracle-lines", type=int, default=2_000_000, help="oracle sample (lines), scaled up")
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    n = args.nodes
    m = int(n * args.degree / 2)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    keep = src != dst
    src, dst = np.minimum(src, dst)[keep], np.maximum(src, dst)[keep]
    w = np.where(rng.random(src.size) < 0.5, 1.0, rng.uniform(0.01, 10.0, src.size))
    # a CSR with entries in both directions (what write_edge_list walks)
    order = np.lexsort((np.concatenate([dst, src]), np.concatenate([src, dst])))
    rows = np.concatenate([src, dst])[order]
    cols = np.concatenate([dst, src])[order]
    ww = np.concatenate([w, w])[order]
    indptr = np.zeros(n + 1, dtype=np.int32)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr).astype(np.int32)
    indices = cols.astype(np.int32)
    td = Path(tempfile.mkdtemp())
    path = td / "g.edges"
    t0 = time.perf_counter()
    _lib.call("csc_edgelist_write", str(path).encode(), n, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(ww), 0)
    t_write = time.perf_counter() - t0
    size = path.stat().st_size
    t0 = time.perf_counter()
    rows_native, hdr = G.parse_edge_list(path)
    t_read = time.perf_counter() - t0
    lines = rows_native.shape[0]
    # reference algorithm on a sample of the same file, scaled to the whole file
    text = path.read_bytes().decode("utf-8")
    cut = text.find("\n", int(len(text) * min(1.0, args.oracle_lines / max(lines, 1)))) + 1 or len(text)
    sample = text[:cut]
    t0 = time.perf_counter()
    orows, _ = O.parse_edge_text(sample)
    t_oread = (time.perf_counter() - t0) * lines / max(orows.shape[0], 1)
    assert np.array_equal(rows_native[: orows.shape[0]], orows)
    k = max(1, int(n * min(1.0, args.oracle_lines / max(lines, 1))))
    t0 = time.perf_counter()
    O.format_edge_list(k, indptr[: k + 1], indices, ww)
    t_owrite = (time.perf_counter() - t0) * n / k
    print(json.dumps({
        "nodes": n, "lines": int(lines), "file_mb": round(size / 1e6, 1), "threads": os.cpu_count(),
        "native_read_s": round(t_read, 3), "native_write_s": round(t_write, 3),
        "reference_read_s_extrapolated": round(t_oread, 1), "reference_write_s_extrapolated": round(t_owrite, 1),
        "reference_sample_lines": int(orows.shape[0]),
    }))


if __name__ == "__main__":
    main()
