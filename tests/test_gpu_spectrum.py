"""Eigencount + dichotomy: same probe trace, same rounded decisions, same lambda_k as the reference."""

from __future__ import annotations

import numpy as np
import pytest

from gpu_util import c1_graph, c1_op, options, oracle_csr
from oracle import cpu_ref as O
import paper_1602_02018_b200 as P
from paper_1602_02018_b200._rng import substream

pytestmark = pytest.mark.gpu


def check_trace(est, golden, tol):
    trace = np.asarray(est.trace)
    ref = golden["trace"]
    assert trace.shape == ref.shape
    assert np.array_equal(trace[:, 0], ref[:, 0])
    assert np.max(np.abs(trace[:, 1] - ref[:, 1]) / np.abs(ref[:, 1])) <= tol
    assert [O.round_half_up(c) for c in trace[:, 1]] == [O.round_half_up(c) for c in ref[:, 1]]
    assert est.lambda_k_hat == float(golden["lambda_k_hat"])


@pytest.mark.parametrize("rec", [0, 1])
@pytest.mark.parametrize("private", [False, True])
def test_dichotomy_trace_c1_fp64(c1_golden, rec, private):
    with options(recurrence=rec):
        est = P.estimate_lambda_k(c1_op(), 20, rng=substream(0, "probe"), private_rng=private)
    check_trace(est, c1_golden, 1e-9)


def test_dichotomy_trace_c1_fp32(c1_golden):
    est = P.estimate_lambda_k(c1_op("float32"), 20, rng=substream(0, "probe"))
    check_trace(est, c1_golden, 1e-4)


def test_eigencount_vs_oracle():
    g, _ = c1_graph()
    for lam in (0.3, 1.0, 2.0):
        a = P.eigencount(c1_op(), lam, rng=np.random.default_rng(5), num_signals=9)
        b = O.eigencount(oracle_csr(g), lam, 50, 9, np.random.default_rng(5))
        assert abs(a.count - b) <= 1e-10 * abs(b)
    full = P.eigencount(c1_op(), 2.0, rng=np.random.default_rng(0))
    assert full.num_signals == 14 and abs(full.count - 1000) <= 100


def test_hooks_and_validation():
    k3 = P.laplacian_op(P.build_graph([(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)]))
    w = np.array([0.0, 1.5, 1.5])

    def factory(lam):
        exact = float(np.sum(w <= lam))

        def fn(X):
            out = np.zeros_like(X)
            out.flat[0] = np.sqrt(exact)
            return out

        return fn

    est = P.estimate_lambda_k(k3, 2, rng=np.random.default_rng(0), max_steps=12, apply_factory=factory)
    assert est.warning is True
    assert [round(c) for _, c in est.trace] == [1, 3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        P.eigencount(k3, 0.0, rng=np.random.default_rng(0))
    with pytest.raises(ValueError):
        P.eigencount(k3, 1.0, num_signals=0, rng=np.random.default_rng(0))
    with pytest.raises(ValueError):
        P.estimate_lambda_k(k3, 3, rng=np.random.default_rng(0))
    two = P.laplacian_op(P.build_graph([(0, 1, 1.0), (2, 3, 1.0)]))
    assert P.eigencount(two, 1.0, num_signals=64, rng=np.random.default_rng(3)).rounded == 2
    e2 = P.estimate_lambda_k(two, 2, num_signals=64, rng=np.random.default_rng(0))
    assert e2.trace[0][0] == 1.0 and 0 < e2.lambda_k_hat < 2


def test_deterministic_and_refine(c1_golden):
    a = P.estimate_lambda_k(c1_op(), 20, rng=np.random.default_rng(123))
    b = P.estimate_lambda_k(c1_op(), 20, rng=np.random.default_rng(123))
    assert a.trace == b.trace and a.lambda_k_hat == b.lambda_k_hat
    plain = P.estimate_lambda_k(c1_op(), 20, rng=np.random.default_rng(9))
    ref = P.estimate_lambda_k(c1_op(), 20, rng=np.random.default_rng(9), refine=True)
    assert ref.lambda_k_hat <= plain.lambda_k_hat
