"""A/B for SURVEY.md section 8(f-2), the speculative / batched eigencount dichotomy.

The probe stream is lambda-independent (spectrum.py:84), so probe t+1's block R_{t+1} is known
while probe t runs.  A speculative round would filter [R_t | R_{t+1}] in ONE pass over the CSR
(shared gathers), R_t with its cut-off and R_{t+1} with BOTH candidate cut-offs of the next
bisection step (forward recurrence: T_l shared, one more accumulator), resolving two probes
per round instead of one.

This measures what such a round costs at best, against the two sequential probes it replaces:
  seq       2 x (Clenshaw filter + SUMSQ on an N x ds block)            (the shipped path)
  lb_clen   1 x (Clenshaw filter + SUMSQ on an N x 2ds block)           (lower bound: no extra accumulator)
  lb_fwd    1 x (forward-recurrence filter + SUMSQ on an N x 2ds block) (closer bound: the speculative round
                                                                         needs the forward recurrence and
                                                                         still one accumulator more)
Speculation can only pay if lb_fwd < seq.  Run on a GPU box:

    python tools/speculative_ab.py > gpurun_out/speculative_ab.txt
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200 import _lib  # noqa: E402
from paper_1602_02018_b200.sbm import c4_config  # noqa: E402
from paper_1602_02018_b200.spectrum import default_num_signals, device_count  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cases = [
        ("C3", lambda: P.sbm_generate(P.SbmConfig(num_nodes=1_000_000, k=100, avg_degree=16.0,
                                                  epsilon=P.critical_epsilon(16.0, 100) / 4.0, seed=0))[0], 0.4331),
        ("C4", lambda: P.dcsbm_generate(c4_config())[0], 0.1523),
    ]
    for name, make, lam in cases:
        g = make()
        op = P.laplacian_op(g, dtype="float32")
        ds = default_num_signals(g.num_nodes)
        rng = np.random.default_rng(0)
        R1 = torch.tensor(rng.standard_normal((g.num_nodes, ds)) / np.sqrt(ds), device="cuda")
        R2 = torch.tensor(rng.standard_normal((g.num_nodes, 2 * ds)) / np.sqrt(2 * ds), device="cuda")
        filt = P.design_lowpass(lam, 50)
        seq = 2.0 * timed(lambda: device_count(op, filt, R1))
        lb_clen = timed(lambda: device_count(op, filt, R2))
        _lib.set_option("recurrence", 1)
        try:
            lb_fwd = timed(lambda: device_count(op, filt, R2))
        finally:
            _lib.set_option("recurrence", 0)
        verdict = "speculation can pay" if lb_fwd < seq else "rejected: a speculative round costs more than two probes"
        print(f"{name}: N={g.num_nodes} ds={ds} fp32  seq(2 probes)={seq:.3f} ms  lb_clenshaw(2ds)={lb_clen:.3f} ms "
              f"({lb_clen / seq:.3f}x)  lb_forward(2ds)={lb_fwd:.3f} ms ({lb_fwd / seq:.3f}x)  -> {verdict}",
              flush=True)


if __name__ == "__main__":
    main()
