"""Split the probe stage at C3: filter-only probes, RNG-only draws, and the two overlapped."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS, make_graph  # noqa: E402
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._signals import DeviceProbeStream, device_normal_block  # noqa: E402
from paper_1602_02018_b200.spectrum import device_count  # noqa: E402
from paper_1602_02018_b200.filters import design_lowpass  # noqa: E402

from paper_1602_02018_b200 import _lib  # noqa: E402

for kv in sys.argv[1:]:
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
print("options:", sys.argv[1:], flush=True)
g, _ = make_graph(P, CONFIGS["c3"])
op = P.laplacian_op(g, dtype="float32")
N, ds = 1_000_000, 28
rng = np.random.default_rng(0)
buf = torch.empty((N, ds), dtype=torch.float64, device="cuda")
device_normal_block(rng, N, ds, 0, buf)
lams = [1.0, 0.5, 0.25, 0.375, 0.4375, 0.40625, 0.421875, 0.4296875, 0.43359375, 0.431640625, 0.4326171875, 0.43310546875]
filts = [design_lowpass(min(l, 2 - 1e-12), 50, damping="jackson") for l in lams]
for f in filts[:2]:
    device_count(op, f, buf)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    for f in filts:
        device_count(op, f, buf)
    t1 = time.perf_counter()
    for _ in filts:
        device_normal_block(rng, N, ds, 0, buf)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = DeviceProbeStream(rng, N, ds, 0)
    for f in filts:
        device_count(op, f, st.take())
    st.close()
    t3 = time.perf_counter()
    print(f"12 probes: filter only {t1 - t0:.4f} s | rng only {t2 - t1:.4f} s | streamed (rng ahead) {t3 - t2:.4f} s",
          flush=True)
