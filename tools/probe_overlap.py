"""Does the probe RNG (worker thread, side stream) overlap the eigencount filter (main stream)?"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS, make_graph  # noqa: E402
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._signals import DeviceProbeStream  # noqa: E402
from paper_1602_02018_b200.spectrum import device_count  # noqa: E402

g, _ = make_graph(P, CONFIGS["c3"])
op = P.laplacian_op(g, dtype="float32")
filt = P.design_lowpass(0.43, 50)
for rep in range(2):
    st = DeviceProbeStream(np.random.default_rng(rep), 1_000_000, 28, 0)
    tw = tc = 0.0
    t00 = time.perf_counter()
    for _ in range(8):
        t0 = time.perf_counter()
        blk = st.take()
        t1 = time.perf_counter()
        device_count(op, filt, blk)
        t2 = time.perf_counter()
        tw += t1 - t0
        tc += t2 - t1
    st.close()
    print(f"rep {rep}: total {(time.perf_counter() - t00) * 1e3 / 8:.1f} ms/probe, waiting for rng {tw * 1e3 / 8:.1f}, "
          f"count {tc * 1e3 / 8:.1f}", flush=True)
