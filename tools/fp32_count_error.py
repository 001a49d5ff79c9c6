"""fp32 vs fp64 eigencount on every probe of the fp64 dichotomy (C1-C4): the numbers behind
spectrum.FP32_GUARD_RTOL.  Prints one line per config; run on a GPU box:

    python tools/fp32_count_error.py > gpurun_out/fp32_guard.txt
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._rng import substream  # noqa: E402
from paper_1602_02018_b200._signals import device_normal_block  # noqa: E402
from paper_1602_02018_b200.sbm import c4_config  # noqa: E402
from paper_1602_02018_b200.spectrum import default_num_signals, device_count, near_decision_boundary  # noqa: E402


def sbm(N, k, s=16.0):
    return P.sbm_generate(P.SbmConfig(num_nodes=N, k=k, avg_degree=s, epsilon=P.critical_epsilon(s, k) / 4.0, seed=0))[0]


def main():
    cases = [("C1", lambda: sbm(1000, 20), 20), ("C2", lambda: sbm(100_000, 20), 20),
             ("C3", lambda: sbm(1_000_000, 100), 100), ("C4", lambda: P.dcsbm_generate(c4_config())[0], 250)]
    worst = 0.0
    for name, make, k in cases:
        g = make()
        op64, op32 = P.laplacian_op(g), P.laplacian_op(g, dtype="float32")
        est = P.estimate_lambda_k(op64, k, rng=substream(0, "probe"))
        rng = substream(0, "probe")
        ds = default_num_signals(g.num_nodes)
        rel, margin, flagged = [], [], 0
        for lam, c64_trace in est.trace:
            blk = device_normal_block(rng, g.num_nodes, ds, op64.device)
            filt = P.design_lowpass(min(lam, 2.0 - 1e-12), 50)
            c64 = device_count(op64, filt, blk)
            c32 = device_count(op32, filt, blk)
            assert c64 == c64_trace
            rel.append(abs(c32 - c64) / abs(c64))
            margin.append(min(abs(c64 - (k - 0.5)), abs(c64 - (k + 0.5))))
            flagged += near_decision_boundary(c32, k)
        worst = max(worst, max(rel))
        print(f"{name}: N={g.num_nodes} k={k} probes={len(rel)} lambda_hat={est.lambda_k_hat!r} warning={est.warning} "
              f"max |c32-c64|/c64={max(rel):.3e} median={float(np.median(rel)):.3e} "
              f"min distance of an fp64 count to k+-1/2={min(margin):.4g} guard_reprobes={flagged}", flush=True)
    print(f"worst relative fp32 count error {worst:.3e}; guard rtol {P.spectrum.FP32_GUARD_RTOL:g} "
          f"= {P.spectrum.FP32_GUARD_RTOL / worst:.0f}x")


if __name__ == "__main__":
    main()
