"""Time the device RNG alone, and concurrently with the filter (threads)."""
import sys
import threading
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
filt = P.design_lowpass(0.43, 50)
side = torch.cuda.Stream()
rng = np.random.default_rng(0)
buf = torch.empty((1_000_000, 28), dtype=torch.float64, device="cuda")
buf2 = torch.empty_like(buf)
device_normal_block(rng, 1_000_000, 28, 0, buf2, side)
device_count(op, filt, buf)
torch.cuda.synchronize()


def rng_job(out):
    t0 = time.perf_counter()
    device_normal_block(rng, 1_000_000, 28, 0, buf2, side)
    out.append(time.perf_counter() - t0)


for mode in ("alone", "with count", "alone"):
    res = []
    t0 = time.perf_counter()
    th = threading.Thread(target=rng_job, args=(res,))
    th.start()
    if mode == "with count":
        tc = time.perf_counter()
        device_count(op, filt, buf)
        tc = time.perf_counter() - tc
    else:
        tc = 0.0
    th.join()
    print(f"{mode:12s} rng {res[0] * 1e3:6.1f} ms  count {tc * 1e3:6.1f} ms  wall {(time.perf_counter() - t0) * 1e3:6.1f} ms",
          flush=True)
