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

pytestmark = pytest.mark.gpu


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
