"""Break the e2e features call into copy-in / compute / copy-out to see where host time goes."""
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._signals import normal_block, pinned_empty  # noqa: E402
from paper_1602_02018_b200.features import RandomSignals, build_features, features_into  # noqa: E402

N, d = 1_000_000, 56
g, _ = P.sbm_generate(P.SbmConfig(num_nodes=N, k=100, avg_degree=16.0, epsilon=P.critical_epsilon(16.0, 100) / 4))
op = P.laplacian_op(g, dtype="float32")
filt = P.design_lowpass(0.43, 50)
host = pinned_empty((N, d))
normal_block(np.random.default_rng(0), N, d, host)
out = pinned_empty((N, d))
dev = torch.empty((N, d), dtype=torch.float64, device="cuda")


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print("h2d pinned 448MB  ms", t(lambda: dev.copy_(torch.from_numpy(host), non_blocking=True)))
print("d2h pinned 448MB  ms", t(lambda: torch.from_numpy(out).copy_(dev, non_blocking=True)))
Xd = dev.float()
Fd = torch.empty_like(Xd)
print("device features   ms", t(lambda: features_into(op, filt, Xd, Fd)))
print("device f64 io     ms", t(lambda: features_into(op, filt, dev, torch.empty_like(dev))))
sig = RandomSignals(matrix=host, distribution="gaussian", seed=None)
print("e2e build_features ms", t(lambda: build_features(op, filt, sig, out=out)))
pageable = np.empty((N, d))
print("e2e pageable out  ms", t(lambda: build_features(op, filt, sig, out=pageable)))
