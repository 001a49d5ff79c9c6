"""Time the features filter on a BASELINE config under different libcsc options.

python tools/sweep_filter.py [--config c3] [--reps 5] [--combos "panel_width=16,recurrence=0;panel_width=64"]
Prints one line per combo: ms per filter (CUDA events), kernel-only ms, algorithmic GB/s, workload GB/s.
"""

from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import CONFIGS, P_ORDER, filter_bytes, make_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--combos", default="")
    ap.add_argument("--width", type=int, default=0, help="signal columns (0 = ceil(4 ln N))")
    ap.add_argument("--dtype", default=None)
    args = ap.parse_args()
    import torch

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import _lib
    from paper_1602_02018_b200.features import features_into

    cfg = CONFIGS[args.config]
    dtype = args.dtype or cfg["dtype"]
    N, k, s = cfg["N"], cfg["k"], cfg["s"]
    d = args.width or int(math.ceil(4 * math.log(N)))
    g, _ = make_graph(P, cfg)
    op = P.laplacian_op(g, dtype=dtype)
    tdt = torch.float32 if dtype == "float32" else torch.float64
    X = torch.randn(N, d, dtype=torch.float64, device="cuda").div_(math.sqrt(d)).to(tdt)
    F = torch.empty_like(X)
    filt = P.design_lowpass(0.43, P_ORDER)
    work = filter_bytes(N, int(g.indices.size), d, 4 if dtype == "float32" else 8, P_ORDER)
    props = torch.cuda.get_device_properties(0)
    print(f"device {props.name} L2 {getattr(props, 'L2_cache_size', 0) / 2**20:.0f} MiB, N={N} d={d} {dtype} "
          f"nnz={int(g.indices.size)}", flush=True)
    combos = [c for c in args.combos.split(";") if c.strip()] or [""]
    for combo in combos:
        old = {}
        for kv in filter(None, combo.split(",")):
            key, val = kv.split("=")
            old[key] = _lib.get_option(key)
            _lib.set_option(key, int(val))
        for _ in range(2):
            features_into(op, filt, X, F)
        torch.cuda.synchronize()
        _lib.set_option("profile", 1)
        _lib.profile_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            features_into(op, filt, X, F)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        kms, nl, kb = _lib.profile_read()
        _lib.set_option("profile", 0)
        print(f"{combo or 'default':45s} {ms:8.3f} ms/filter  kernel {kms / args.reps:8.3f} ms  "
              f"{nl // args.reps:4d} launches  alg {kb / (kms / 1e3) / 1e9:7.1f} GB/s  "
              f"workload {work / (ms / 1e3) / 1e9:7.1f} GB/s", flush=True)
        for key, val in old.items():
            _lib.set_option(key, val)


if __name__ == "__main__":
    main()
