"""Device SBM generator (csc_sbm_edges) == the reference generator's draws, edge for edge.

The host restatement ``sbm_edges`` is pinned to the reference's golden graphs
(test_oracle_golden / test_gpu_graph); the device path must reproduce it exactly,
in the same order."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1602_02018_b200 as P
from paper_1602_02018_b200.sbm import SbmConfig, sbm_edges, sbm_edges_device

pytestmark = pytest.mark.gpu


def _cfg(N, k, s, div=4.0, seed=0, sizes=None, eps=None):
    e = P.critical_epsilon(s, k) / div if eps is None else eps
    return SbmConfig(num_nodes=N, k=k, avg_degree=s, epsilon=e, seed=seed, sizes=sizes)


@pytest.mark.parametrize("cfg", [
    _cfg(1000, 20, 16),                      # C1
    _cfg(100_000, 20, 16),                   # C2
    _cfg(20_011, 150, 8, seed=3),            # uneven sizes, 11325 pairs
    _cfg(5000, 7, 12, eps=0.0),              # no inter-community draws (q2 = 0)
    _cfg(3000, 3, 30, sizes=[1, 1499, 1500]),  # a single-node community (no diagonal cells)
], ids=["c1", "c2", "uneven", "eps0", "singleton"])
def test_device_sbm_edges_match_host(cfg):
    src_h, dst_h, lab_h = sbm_edges(cfg)
    out = sbm_edges_device(cfg, 0)
    assert out is not None
    src_d, dst_d, lab_d = out
    assert np.array_equal(src_d.cpu().numpy(), src_h)
    assert np.array_equal(dst_d.cpu().numpy(), dst_h)
    assert np.array_equal(lab_d, lab_h)


def test_device_sbm_c3_graph_matches_host():
    cfg = _cfg(1_000_000, 100, 16)
    src_h, dst_h, _ = sbm_edges(cfg)
    src_d, dst_d, _ = sbm_edges_device(cfg, 0)
    assert src_d.numel() == src_h.size == 7_999_925
    assert np.array_equal(src_d.cpu().numpy(), src_h) and np.array_equal(dst_d.cpu().numpy(), dst_h)
    g, _ = P.sbm_generate(cfg)
    assert g.num_edges == src_h.size


def test_dense_pairs_fall_back_to_host():
    cfg = _cfg(60, 2, 20)  # q1 > 1/3: numpy's search branch
    assert cfg.q1 >= 1 / 3
    assert sbm_edges_device(cfg, 0) is None
    g, labels = P.sbm_generate(cfg)
    src, dst, _ = sbm_edges(cfg)
    assert g.num_edges == src.size
