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


def test_fp32_guard_reprobes_in_fp64(c1_golden, monkeypatch):
    """Every probe inside the (widened) guard band is re-run in fp64 on the same block:
    the trace then equals the fp64 trace bit for bit (spectrum.py:49-50, 125-137)."""
    from paper_1602_02018_b200 import spectrum as S

    e64 = P.estimate_lambda_k(c1_op(), 20, rng=substream(0, "probe"))
    monkeypatch.setattr(S, "FP32_GUARD_RTOL", 10.0)
    e32 = P.estimate_lambda_k(c1_op("float32"), 20, rng=substream(0, "probe"))
    assert e32.fp64_reprobes == list(range(len(e32.trace)))
    assert e32.trace == e64.trace and e32.lambda_k_hat == e64.lambda_k_hat
    # fp64 operators never re-probe; the default band leaves C1's probes alone
    assert e64.fp64_reprobes == []
    monkeypatch.setattr(S, "FP32_GUARD_RTOL", 1e-5)
    plain = P.estimate_lambda_k(c1_op("float32"), 20, rng=substream(0, "probe"))
    assert plain.lambda_k_hat == float(c1_golden["lambda_k_hat"])


def test_fp32_guard_boundary_predicate():
    from paper_1602_02018_b200.spectrum import near_decision_boundary

    assert near_decision_boundary(19.5004, 20) and near_decision_boundary(20.4996, 20)
    assert not near_decision_boundary(19.51, 20) and not near_decision_boundary(20.0, 20)
    assert not near_decision_boundary(45_850.5, 20)  # far from k: cannot flip a decision


def test_fp32_guard_in_run_csc_diagnostics(monkeypatch):
    from paper_1602_02018_b200 import spectrum as S

    monkeypatch.setattr(S, "FP32_GUARD_RTOL", 10.0)
    r32 = P.run_csc(c1_op("float32"), P.CscParams(k=20, d=28, seed=0))
    r64 = P.run_csc(c1_op(), P.CscParams(k=20, d=28, seed=0))
    assert r32.diagnostics["probe_fp64_reprobes"] == list(range(r32.diagnostics["probe_iterations"]))
    assert "probe_fp64_reprobes" not in r64.diagnostics
    assert r32.diagnostics["lambda_k_hat"] == r64.diagnostics["lambda_k_hat"]
