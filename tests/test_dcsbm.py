"""DC-SBM generator (BASELINE config 4; SURVEY.md section 8(d) spec): host-only native code, CPU tests.

The reference has no DC-SBM, so the bar is the spec itself: independent
Bernoulli edges with P(i~j) = min(1, theta_i theta_j q_{c_i c_j}), deterministic under a seed
and independent of the thread count.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

from paper_1602_02018_b200 import _lib
from paper_1602_02018_b200.sbm import c4_config, dcsbm_edges


def native_edges(sizes, theta, q1, q2, seed, nthreads=0):
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    n = int(sizes.sum())
    cap = n * n
    src = np.empty(cap, dtype=np.int64)
    dst = np.empty(cap, dtype=np.int64)
    m = C.c_int64(0)
    _lib.call("csc_dcsbm_edges", n, int(sizes.size), _lib.ptr(sizes), _lib.ptr(theta), C.c_double(q1),
              C.c_double(q2), C.c_uint64(seed), nthreads, C.c_int64(cap), _lib.ptr(src), _lib.ptr(dst), C.byref(m))
    return src[: m.value], dst[: m.value]


def test_pair_frequencies_match_bernoulli_probabilities():
    """Empirical P(i~j) over many seeds vs min(1, theta_i theta_j q): every pair within 5 sigma,
    clipped pairs (p = 1) always present, and the chi-square of all pairs near its dof."""
    rng = np.random.default_rng(3)
    sizes = np.array([9, 7, 8])
    n = int(sizes.sum())
    comm = np.repeat(np.arange(3), sizes)
    theta = 1.0 + rng.pareto(2.5, n)
    theta[[0, 9]] = [6.0, 5.0]  # heavy nodes: some pairs clip at probability 1
    q1, q2 = 0.12, 0.03
    qm = np.where(comm[:, None] == comm[None, :], q1, q2)
    P = np.minimum(1.0, theta[:, None] * theta[None, :] * qm)
    iu = np.triu_indices(n, 1)
    p = P[iu]
    reps = 4000
    hits = np.zeros((n, n))
    for seed in range(reps):
        s, d = native_edges(sizes, theta, q1, q2, seed)
        assert np.all(s < d)
        hits[s, d] += 1
    f = hits[iu]
    assert np.all(f[p == 1.0] == reps)
    var = p * (1 - p) / reps
    live = p < 1.0
    z = (f[live] / reps - p[live]) / np.sqrt(var[live])
    assert np.abs(z).max() < 5.0
    chi2 = float(np.sum(z ** 2))
    dof = int(live.sum())
    assert abs(chi2 - dof) < 6 * math.sqrt(2 * dof)


def test_thread_count_and_seed_determinism():
    rng = np.random.default_rng(5)
    sizes = np.array([300, 250, 450])
    theta = 1.0 + rng.pareto(2.5, 1000)
    a = native_edges(sizes, theta, 0.02, 0.004, 77, nthreads=1)
    b = native_edges(sizes, theta, 0.02, 0.004, 77, nthreads=7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = native_edges(sizes, theta, 0.02, 0.004, 78, nthreads=3)
    assert not (c[0].size == a[0].size and np.array_equal(c[0], a[0]))


def test_edge_cases():
    # empty graph, single community, zero probabilities
    s, d = native_edges([0], np.zeros(0), 0.1, 0.1, 1)
    assert s.size == 0
    s, d = native_edges([5], np.ones(5), 1.0, 0.0, 1)  # complete graph K5
    assert s.size == 10
    s, d = native_edges([4, 4], np.ones(8), 0.0, 0.0, 1)
    assert s.size == 0
    s, d = native_edges([3, 3], np.ones(6), 0.0, 1.0, 1)  # complete bipartite K3,3
    assert s.size == 9 and np.all((s < 3) & (d >= 3))
    with pytest.raises(ValueError):
        native_edges([3, -1], np.ones(2), 0.1, 0.1, 1)
    with pytest.raises(ValueError):
        native_edges([2], np.array([1.0, np.nan]), 0.1, 0.1, 1)


def test_c4_graph_shape():
    """BASELINE config 4 stand-in: mean degree 5.5, heavy-tailed rows, deterministic."""
    cfg = c4_config()
    s, d, comm, theta = dcsbm_edges(cfg)
    n = cfg.num_nodes
    deg = np.bincount(s, minlength=n) + np.bincount(d, minlength=n)
    assert abs(deg.mean() - 5.5) < 0.05
    assert deg.max() > 200 and (deg > 100).sum() > 30
    assert np.all(s < d) and np.unique(s * n + d).size == s.size
    # community-level means of theta are 1 (normalised per community)
    means = np.bincount(comm, weights=theta) / np.bincount(comm)
    assert np.allclose(means, 1.0)
    s2, d2, _, _ = dcsbm_edges(cfg)
    assert np.array_equal(s, s2) and np.array_equal(d, d2)
