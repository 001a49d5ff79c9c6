"""Time the two parts of one eigencount probe at C3: device parity RNG and the fused filter."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS, make_graph  # noqa: E402
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._signals import device_normal_block  # noqa: E402
from paper_1602_02018_b200.spectrum import device_count  # noqa: E402

g, _ = make_graph(P, CONFIGS["c3"])
op = P.laplacian_op(g, dtype="float32")
rng = np.random.default_rng(0)
buf = torch.empty((1_000_000, 28), dtype=torch.float64, device="cuda")
filt = P.design_lowpass(0.43, 50)
for _ in range(2):
    device_normal_block(rng, 1_000_000, 28, 0, buf)
    device_count(op, filt, buf)
torch.cuda.synchronize()
for name, fn in [("rng", lambda: device_normal_block(rng, 1_000_000, 28, 0, buf)),
                 ("count", lambda: device_count(op, filt, buf)),
                 ("host numpy rng", lambda: rng.standard_normal((1_000_000, 28)))]:
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name:16s} {(time.perf_counter() - t0) / 5 * 1e3:8.2f} ms", flush=True)
