"""Does within-warp row-length imbalance cost K2 time?  (hypothesis test, B200)

A warp of k_cheb_mid handles 32/LPR rows at once and loops to the longest one (in chunks of
max(LPR, 4) slots), so a row group of Poisson(16) rows issues ~23 slots per row where 16 carry a
gather.  This times the order-50 filter on relabelings of the C3 graph that change only which
rows share a warp:

  natural      the SBM's community order
  wsort<W>     rows sorted by degree inside windows of W consecutive rows (locality kept at W)
  regular16    every row cut / padded to exactly 16 neighbours (same community mix): upper bound

python tools/microbench/degree_balance.py [--widths 32,56] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def relabel(indptr, indices, order):
    """Graph with new node r = old node order[r]; each row keeps its neighbour order."""
    n = indptr.size - 1
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    deg = np.diff(indptr)[order]
    ip = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=ip[1:])
    starts = indptr[order]
    idx = np.repeat(starts - ip[:-1], deg) + np.arange(ip[-1])
    return ip.astype(np.int32), inv[indices[idx]].astype(np.int32)


def window_order(indptr, W):
    n = indptr.size - 1
    deg = np.diff(indptr)
    win = np.arange(n) // W
    return np.lexsort((np.arange(n), deg, win))  # by window, then degree, stable


def regular16(indptr, indices, k, rng):
    n = indptr.size - 1
    csize = n // k
    out = np.empty((n, 16), dtype=np.int32)
    for i in range(n):
        nb = indices[indptr[i]:indptr[i + 1]][:16]
        if nb.size < 16:
            c = i // csize
            extra = rng.integers(c * csize, min(n, (c + 1) * csize), 16 - nb.size)
            nb = np.concatenate([nb, extra])
        out[i] = np.sort(nb)
    return (np.arange(n + 1, dtype=np.int64) * 16).astype(np.int32), out.ravel()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--widths", default="32,56")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--windows", default="16,64,256,4096")
    args = ap.parse_args()
    import torch

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200.features import features_into
    from paper_1602_02018_b200.graph import Graph
    from bench import CONFIGS, make_graph

    cfg = CONFIGS["c3"]
    g0, _ = make_graph(P, cfg)
    ip0, ix0 = g0.indptr.astype(np.int64), g0.indices.astype(np.int64)
    variants = {"natural": (g0.indptr, g0.indices)}
    for W in map(int, args.windows.split(",")):
        variants[f"wsort{W}"] = relabel(ip0, ix0, window_order(ip0, W))
    variants["regular16"] = regular16(g0.indptr, g0.indices, cfg["k"], np.random.default_rng(0))
    filt = P.design_lowpass(0.43, 50)
    res = {}
    for name, (ip, ix) in variants.items():
        deg = np.diff(ip).astype(np.float64)
        g = Graph(num_nodes=g0.num_nodes, indptr=np.ascontiguousarray(ip, np.int32),
                  indices=np.ascontiguousarray(ix, np.int32), weights=np.ones(ix.size), degrees=deg)
        op = P.laplacian_op(g, dtype="float32")
        # slot efficiency of 4-row groups, chunks of 8 (the 128-B-row schedule)
        dg = np.diff(ip)[: (g0.num_nodes // 4) * 4].reshape(-1, 4)
        eff = dg.sum() / (4 * 8 * np.ceil(dg.max(1) / 8)).sum()
        row = {"nnz": int(ix.size), "slot_eff_4x8": round(float(eff), 3)}
        for w in map(int, args.widths.split(",")):
            X = torch.randn(g0.num_nodes, w, dtype=torch.float64, device="cuda").div_(math.sqrt(w)).float()
            F = torch.empty_like(X)
            for _ in range(3):
                features_into(op, filt, X, F, zero_rows=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                features_into(op, filt, X, F, zero_rows=False)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            row[f"w{w}_ms"] = round(ms, 3)
            row[f"w{w}_ns_per_edge_step"] = round(ms * 1e6 / (50 * ix.size), 4)
        res[name] = row
        print(name, json.dumps(row), flush=True)
        del op, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
