"""Column-sharded exchange logic (dist.py) with world_size 2 over gloo on CPU.

The per-rank compute is an oracle-based CPU backend (test-only); what is under
test is the sharding, the collectives and the merge rules, against the
single-process oracle."""

from __future__ import annotations

import os
import socket

import json

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import D_C1, c1_config
from oracle import cpu_ref as O
from paper_1602_02018_b200 import dist as D
from paper_1602_02018_b200.filters import design_lowpass
from paper_1602_02018_b200.pipeline import CscParams
from paper_1602_02018_b200.sampling import CgInfo
from paper_1602_02018_b200.sbm import sbm_edges

pytestmark = pytest.mark.timeout(900)  # a lost rank must fail the run, not hang it


class OracleBackend:
    """CPU per-rank compute for the tests (the product uses dist.DeviceBackend)."""

    def __init__(self, csr):
        self.csr = csr
        rows = np.repeat(np.arange(csr.num_nodes), np.diff(csr.indptr))
        self.num_edges = int(np.count_nonzero(np.asarray(csr.indices) > rows))  # Graph.num_edges: i < j entries

    def count(self, filt, R):
        if R.shape[1] == 0:
            return 0.0
        Y = O.apply_filter(filt.coeffs, self.csr, R)
        return float(np.sum(Y * Y))

    def filter_rowsq(self, filt, R):
        Y = O.apply_filter(filt.coeffs, self.csr, R) if R.shape[1] else np.zeros_like(R)
        return Y, np.sum(Y * Y, axis=1)

    def normalize(self, Y, rowsq):
        nrm = np.sqrt(rowsq)
        zero = np.flatnonzero(nrm <= 1e-300)
        safe = nrm.copy()
        safe[zero] = 1.0
        F = Y / safe[:, None]
        F[zero] = 0.0
        return F, zero

    def gather(self, F, idx):
        return F[idx]

    def block_cg(self, cfg, sampling, reduced):
        if reduced.shape[1] == 0:
            return np.zeros((self.csr.num_nodes, 0)), CgInfo(np.zeros(0, np.int64), np.zeros(0), np.zeros(0, bool))
        X, its, res, conv = O.interpolate_all(self.csr, cfg.highpass.coeffs, cfg.gamma, cfg.ridge, sampling.indices,
                                              reduced, cfg.solver_tol, cfg.solver_max_iters)
        return X, CgInfo(its, res, conv)

    def kmeans(self, points, cfg):
        from paper_1602_02018_b200.kmeans import Labeling

        lab, inert, its = O.kmeans(points, cfg.k, cfg.seed, cfg.replicates, cfg.max_iters, cfg.tol)
        return Labeling(lab, inert, its)

    def row_best(self, soft, col0):
        norms = np.linalg.norm(soft, axis=0)
        q = np.where(norms > 0, soft / np.where(norms > 0, norms, 1.0), -np.inf) if soft.shape[1] else np.full(
            (soft.shape[0], 1), -np.inf)
        idx = q.argmax(axis=1)
        return q[np.arange(q.shape[0]), idx], col0 + idx, np.any(soft != 0, axis=1), bool(np.any(norms > 0))


def c1_csr():
    src, dst, _ = sbm_edges(c1_config())
    return O.sbm_csr(src, dst, 1000)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = fn(D.Group.current())
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), fn, out), nprocs=world, join=True)
    return [out[r] for r in range(world)]


def test_column_slice_partitions():
    for ncols in (1, 2, 7, 28, 56, 100):
        for world in (1, 2, 3, 4, 8):
            parts = [D.column_slice(ncols, world, r) for r in range(world)]
            cover = np.concatenate([np.arange(p.start, p.stop) for p in parts])
            assert np.array_equal(cover, np.arange(ncols))
            sizes = [p.stop - p.start for p in parts]
            assert max(sizes) - min(sizes) <= 1


def test_merge_argmax_tie_rule():
    v = [np.array([0.5, 0.2, 0.7]), np.array([0.5, 0.9, 0.1])]
    c = [np.array([3, 1, 0]), np.array([7, 6, 5])]
    assert D.merge_argmax(v, c).tolist() == [3, 6, 0]


def _features_and_count(grp):
    csr = c1_csr()
    be = OracleBackend(csr)
    R = O.gaussian_signals(1000, D_C1, O.substream(0, "signals"))
    cols = D.column_slice(D_C1, grp.world, grp.rank)
    filt = design_lowpass(0.45, 30)
    F, zero = D.sharded_features(be, filt, np.ascontiguousarray(R[:, cols]), grp)
    cnt = D.sharded_count(be, filt, np.ascontiguousarray(R[:, cols]), grp)
    return cols.start, cols.stop, F, zero, cnt


def test_sharded_features_and_count_match_single_process():
    parts = run_world(_features_and_count)
    csr = c1_csr()
    R = O.gaussian_signals(1000, D_C1, O.substream(0, "signals"))
    filt = design_lowpass(0.45, 30)
    rows, zero = O.build_features(filt.coeffs, csr, R)
    F = np.zeros_like(rows)
    for c0, c1, Fl, z, cnt in parts:
        F[:, c0:c1] = Fl
        assert np.array_equal(z, zero)
        ref = float(np.sum(O.apply_filter(filt.coeffs, csr, R) ** 2))
        assert abs(cnt - ref) <= 1e-12 * ref
    assert np.abs(F - rows).max() <= 1e-13


def _run_sharded(grp):
    be = OracleBackend(c1_csr())
    res = D.run_csc_sharded(be, 1000, CscParams(k=20, d=D_C1, seed=0), grp)
    return res.labels, res.diagnostics["lambda_k_hat"], res.diagnostics["solver_iterations"], res.num_clusters, \
        res.diagnostics


@pytest.mark.parametrize("world", [2, 3])
def test_run_csc_sharded_matches_reference(c1_golden, world):
    # world 3: uneven column slices (d = 28, k = 20, ds = 14 do not divide by 3)
    ref = json.loads(bytes(c1_golden["result_json"]).decode())["diagnostics"]
    parts = run_world(_run_sharded, world=world)
    for labels, lam, its, k, diag in parts:
        assert lam == float(c1_golden["lambda_k_hat"])
        assert its == c1_golden["solver_iterations"].tolist()
        assert np.array_equal(labels, c1_golden["labels"])
        assert k == 20
        # same diagnostics schema as the reference (to_json drops timings), plus one nested key
        assert set(diag) - {"timings", "sharding"} == set(ref)
        assert set(diag["timings"]) == {"probe", "design", "signals", "filter", "sampling", "kmeans", "interpolate",
                                        "total"}
        assert diag["num_edges"] == ref["num_edges"]
        assert diag["sharding"]["ranks"] == world


# ---- row sharding (BASELINE config 5) -----------------------------------------


def test_row_range_partitions():
    for N in (1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            ranges = [D.row_range(N, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == N
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            assert max(b - a for a, b in ranges) == -(-N // world)


def test_row_partition_balances_nnz():
    """row_partition cuts contiguous ranges whose nnz + rows cost is within one row of the
    ideal share, also on heavy-tailed DC-SBM rows."""
    from paper_1602_02018_b200.sbm import SbmConfig, critical_epsilon, dcsbm_edges

    cfg = SbmConfig(num_nodes=20000, k=20, avg_degree=5.5, epsilon=critical_epsilon(5.5, 20) / 4.0, seed=0)
    src, dst, _, _ = dcsbm_edges(cfg)
    deg = np.bincount(np.concatenate([src, dst]), minlength=cfg.num_nodes)
    indptr = np.concatenate([[0], np.cumsum(deg)])
    row_cost = deg + 1
    for world in (1, 2, 3, 8, 64):
        st = D.row_partition(indptr, world)
        assert st[0] == 0 and st[-1] == cfg.num_nodes and np.all(np.diff(st) >= 0) and st.size == world + 1
        costs = [int(row_cost[st[q]:st[q + 1]].sum()) for q in range(world)]
        assert max(costs) <= row_cost.sum() / world + row_cost.max()
    # equal-cost rows reduce to the equal-count split
    flat = np.arange(0, 16 * 1001, 16)
    assert D.row_partition(flat, 4).tolist() == [0, 250, 500, 750, 1000]


def _row_sharded_filter(grp):
    """The row-sharded recurrence of rows.cu, restated with numpy: local rows x full block,
    nnz-balanced row ranges (row_partition), block all-gathered after every step in equal
    R = max-rows slots (padded), read back through the slot layout."""
    import scipy.sparse as sp

    csr = c1_csr()
    N = csr.num_nodes
    starts = D.row_partition(csr.indptr, grp.world)
    b, e = int(starts[grp.rank]), int(starts[grp.rank + 1])
    R = int(np.diff(starts).max())
    indptr, indices, weights = D.local_csr(csr, b, e)
    Wl = sp.csr_matrix((weights, indices, indptr), shape=(e - b, N))
    dis = csr.dis
    X = O.gaussian_signals(N, 9, O.substream(0, "signals"))
    c = design_lowpass(0.4, 30).coeffs

    def gather(local):
        pad = np.zeros((R, local.shape[1]))
        pad[: local.shape[0]] = local
        slots = grp.all_gather(pad)
        return np.concatenate([slots[q][: starts[q + 1] - starts[q]] for q in range(grp.world)], axis=0)

    def A(full, rows):  # (L - I) restricted to this rank's rows: -D^-1/2 W D^-1/2
        return -(dis[b:e, None] * (Wl @ (dis[:, None] * full)))

    Xl = X[b:e]
    out = c[0] * Xl
    t_prev, t_cur = Xl, A(X, Xl)
    out = out + c[1] * t_cur
    for l in range(2, c.size):
        t_prev, t_cur = t_cur, 2.0 * A(gather(t_cur), t_cur) - t_prev
        out = out + c[l] * t_cur
    return b, e, out


def test_row_sharded_recurrence_matches_oracle():
    parts = run_world(_row_sharded_filter)
    csr = c1_csr()
    X = O.gaussian_signals(1000, 9, O.substream(0, "signals"))
    ref = O.apply_filter(design_lowpass(0.4, 30).coeffs, csr, X)
    got = np.zeros_like(ref)
    for b, e, out in parts:
        got[b:e] = out
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def _exchange(grp):
    handle = np.full(64, 10 + grp.rank, dtype=np.uint8)
    return [h.tolist() for h in D.exchange_handles(grp, handle)]


def test_peer_handle_exchange_rank_order():
    """The peer transport's IPC handle exchange returns every rank's handle in rank order."""
    got = run_world(_exchange)
    for per_rank in got:
        assert per_rank == [[10] * 64, [11] * 64]
