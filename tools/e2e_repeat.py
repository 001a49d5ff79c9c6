"""Time individual e2e build_features calls (host fp64 in/out) to expose run-to-run variance."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._signals import normal_block  # noqa: E402
from paper_1602_02018_b200.features import RandomSignals, build_features  # noqa: E402

N, d = 1_000_000, 56
g, _ = P.sbm_generate(P.SbmConfig(num_nodes=N, k=100, avg_degree=16.0, epsilon=P.critical_epsilon(16.0, 100) / 4))
op = P.laplacian_op(g, dtype="float32")
filt = P.design_lowpass(0.43, 50)
host_t = torch.empty((N, d), dtype=torch.float64, pin_memory=True)
host = host_t.numpy()
normal_block(np.random.default_rng(0), N, d, host)
out_t = torch.empty((N, d), dtype=torch.float64, pin_memory=True)
out = out_t.numpy()
sig = RandomSignals(matrix=host, distribution="gaussian", seed=None)
times = []
for i in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    build_features(op, filt, sig, out=out)
    torch.cuda.synchronize()
    times.append((time.perf_counter() - t0) * 1e3)
print("e2e ms:", " ".join(f"{t:.1f}" for t in times), flush=True)
