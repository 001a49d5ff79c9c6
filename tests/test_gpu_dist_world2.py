"""The column-sharded pipeline with several ranks, each running the real device backend.

World sizes 2 and 3 share cuda:0 and exchange over gloo (host-side collectives), so
no rank's kernel ever waits on another rank's kernel: this exercises the multi-rank
device code path (column slices of the probe / signal / indicator blocks drawn by
the device parity RNG, row-norm and count exchanges, the sampled-row gather, the
per-rank block CG and the argmax merge) against the reference's single-process
outputs.  The NCCL transport itself needs one GPU per rank and is not run here.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import D_C1
from test_dist_gloo import run_world

# a lost rank must fail the run, not hang it (pytest-timeout; the spawn helper also tears the world down)
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _device_run(grp):
    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import dist as D
    from gpu_util import c1_op

    res = D.run_csc_sharded(D.DeviceBackend(c1_op()), 1000, P.CscParams(k=20, d=D_C1, seed=0), grp)
    d = res.diagnostics
    return res.labels, d["lambda_k_hat"], d["solver_iterations"], d["probe_iterations"], res.num_clusters


@pytest.mark.parametrize("world", [2, 3])
def test_device_backend_multi_rank_matches_reference(c1_golden, world):
    parts = run_world(_device_run, world=world)
    assert len(parts) == world
    for labels, lam, its, probes, k in parts:
        assert lam == float(c1_golden["lambda_k_hat"])
        assert its == c1_golden["solver_iterations"].tolist()
        assert np.array_equal(labels, c1_golden["labels"])
        assert k == 20
    assert len({p[3] for p in parts}) == 1  # every rank walked the same dichotomy


def _device_features(grp):
    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import dist as D
    from gpu_util import c1_op
    from oracle import cpu_ref as O

    be = D.DeviceBackend(c1_op())
    R = O.gaussian_signals(1000, D_C1, O.substream(0, "signals"))
    cols = D.column_slice(D_C1, grp.world, grp.rank)
    filt = P.design_lowpass(0.45, 30)
    F, zero = D.sharded_features(be, filt, np.ascontiguousarray(R[:, cols]), grp)
    F = F.cpu().numpy() if hasattr(F, "cpu") else np.asarray(F)
    cnt = D.sharded_count(be, filt, np.ascontiguousarray(R[:, cols]), grp)
    return cols.start, cols.stop, F, np.asarray(zero), cnt


def test_device_sharded_features_match_oracle():
    from oracle import cpu_ref as O
    from paper_1602_02018_b200.filters import design_lowpass
    from test_dist_gloo import c1_csr

    parts = run_world(_device_features, world=2)
    csr = c1_csr()
    R = O.gaussian_signals(1000, D_C1, O.substream(0, "signals"))
    filt = design_lowpass(0.45, 30)
    rows, zero = O.build_features(filt.coeffs, csr, R)
    ref_cnt = float(np.sum(O.apply_filter(filt.coeffs, csr, R) ** 2))
    F = np.zeros_like(rows)
    for c0, c1, Fl, z, cnt in parts:
        F[:, c0:c1] = Fl
        assert np.array_equal(z, zero)
        assert abs(cnt - ref_cnt) <= 1e-12 * ref_cnt
    assert np.abs(F - rows).max() <= 1e-12


def _peer_rows(grp, dtype="float64", widths=(5, 40, 7), orders=(0, 1, 2, 3, 50)):
    """One rank of the row-sharded peer transport; ranks are separate processes on cuda:0.

    The step boundary goes through the host (stream synchronise + gloo barrier), so no kernel
    ever waits on another rank's kernel; everything else is the multi-GPU path: panels exported
    and mapped by CUDA IPC across processes, rows stored into the other process's panels by the
    step kernel's epilogue, ping-pong panel reuse across steps and calls.
    """
    import torch
    import torch.distributed as dist

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import dist as D
    from gpu_util import c1_op

    g = c1_op().graph
    tdt = torch.float64 if dtype == "float64" else torch.float32
    rop = D.RowShardedOperator(g, grp, dtype=dtype, device=0, transport="peer", barrier="host")
    out = {"range": (rop.begin, rop.end)}
    for w in widths:
        X = np.random.default_rng(w).standard_normal((1000, w))
        Xl = torch.tensor(X[rop.begin:rop.end], dtype=tdt, device="cuda:0")
        filt = None
        for order in orders:
            filt = P.design_lowpass(0.6, order) if order else P.PolyFilter(np.array([0.7]), 0.6, 0, "none", "lowpass")
            out[("y", w, order)] = rop.apply_filter(filt, Xl).cpu().numpy()
        out[("count", w)] = rop.eigencount(filt, Xl)
        F, zero = rop.features(filt, Xl)
        out[("F", w)] = F.cpu().numpy()
        out[("zero", w)] = zero
    rop.close()  # collective: nobody unmaps or frees a panel a peer may still be storing into
    return out


def _peer_rows32(grp):
    return _peer_rows(grp, dtype="float32", widths=(21,), orders=(1, 50))


@pytest.mark.parametrize("world,fn,dtype", [(2, _peer_rows, "float64"), (3, _peer_rows, "float64"),
                                           (2, _peer_rows32, "float32")])
def test_row_sharded_peer_transport_across_processes(world, fn, dtype):
    """World 2 and 3 as processes sharing cuda:0 == the replicated path, bit for bit."""
    import torch

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import dist as D
    from gpu_util import c1_op

    parts = run_world(fn, world=world)
    g = c1_op().graph
    tdt = torch.float64 if dtype == "float64" else torch.float32
    one = D.RowShardedOperator(g, D.Group(0, 1), dtype=dtype, transport="peer")
    ranges = [p["range"] for p in parts]
    assert ranges[0][0] == 0 and ranges[-1][1] == 1000 and all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    keys = [k for k in parts[0] if k != "range"]
    for key in keys:
        if key[0] == "y":
            _, w, order = key
            X = torch.tensor(np.random.default_rng(w).standard_normal((1000, w)), dtype=tdt, device="cuda")
            filt = P.design_lowpass(0.6, order) if order else P.PolyFilter(np.array([0.7]), 0.6, 0, "none", "lowpass")
            ref = one.apply_filter(filt, X).cpu().numpy()
            got = np.concatenate([p[key] for p in parts])
            assert np.array_equal(got, ref), key
    order = max(k[2] for k in keys if k[0] == "y")
    filt = P.design_lowpass(0.6, order)
    for w in sorted({k[1] for k in keys if k[0] == "F"}):
        X = torch.tensor(np.random.default_rng(w).standard_normal((1000, w)), dtype=tdt, device="cuda")
        Fref, zref = one.features(filt, X)
        assert np.array_equal(np.concatenate([p[("F", w)] for p in parts]), Fref.cpu().numpy())
        assert np.array_equal(np.concatenate([p[("zero", w)] for p in parts]), zref)
        cref = one.eigencount(filt, X)
        for p in parts:  # every rank holds the rank-ordered sum of the partials
            assert p[("count", w)] == parts[0][("count", w)]
            assert abs(p[("count", w)] - cref) <= (1e-12 if dtype == "float64" else 1e-5) * cref


def test_host_barrier_single_rank_and_failure():
    """One rank: the host-barrier transport equals the device-barrier one bit for bit, and a
    failing barrier callback fails the call (CSC_ERR_INVALID -> ValueError) instead of hanging."""
    import torch

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import dist as D
    from gpu_util import c1_op

    g = c1_op().graph
    X = torch.tensor(np.random.default_rng(0).standard_normal((1000, 9)), dtype=torch.float64, device="cuda")
    filt = P.design_lowpass(0.6, 20)
    dev = D.RowShardedOperator(g, D.Group(0, 1), dtype="float64", transport="peer")
    host = D.RowShardedOperator(g, D.Group(0, 1), dtype="float64", transport="peer", barrier="host")
    assert torch.equal(dev.apply_filter(filt, X), host.apply_filter(filt, X))

    host._host_barrier = lambda _ctx: 1  # a barrier that reports a lost peer
    host._barrier_cb = None
    host._close_peers()
    with pytest.raises(ValueError, match="host barrier"):
        host.apply_filter(filt, X)
    host.close()
    dev.close()
