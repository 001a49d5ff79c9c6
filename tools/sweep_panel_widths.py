"""Time one order-50 filter on a config's graph for single panels of given widths.

python tools/sweep_panel_widths.py [--config c3] [--widths 4,16,32,36,64] [--reps 10] [--opts tight_panels=1]

Each width w runs with panel_width forced to the next power of two >= w, so the block is one
panel (pow2-padded, or w rounded to 16 B with tight_panels=1).  Prints ms per filter and
ms per step launch: the per-panel cost model behind the block-CG panel plan.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--widths", default="4,8,16,24,28,32,36,40,48,50,56,64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--opts", default="")
    ap.add_argument("--dtype", default="")
    ap.add_argument("--pw", type=int, default=0, help="panel_width option: 0 = next power of two >= w (one panel), "
                    "-1 = the library's automatic plan, >0 = that value")
    args = ap.parse_args()

    import torch

    import paper_1602_02018_b200 as P
    import paper_1602_02018_b200._lib as L
    from bench import CONFIGS, P_ORDER, make_graph
    from paper_1602_02018_b200.features import features_into

    for kv in filter(None, args.opts.split(",")):
        k, v = kv.split("=")
        L.set_option(k, int(v))
    cfg = CONFIGS[args.config]
    dtype = args.dtype or cfg["dtype"]
    g, _ = make_graph(P, cfg)
    op = P.laplacian_op(g, dtype=dtype)
    tdt = torch.float32 if dtype == "float32" else torch.float64
    filt = P.design_lowpass(0.43, P_ORDER)
    for w in [int(x) for x in args.widths.split(",")]:
        pw = 4 if tdt == torch.float32 else 2
        while pw < w:
            pw *= 2
        pw = pw if args.pw == 0 else max(args.pw, 0)
        L.set_option("panel_width", pw)
        X = torch.randn(g.num_nodes, w, dtype=torch.float64, device="cuda").to(tdt)
        F = torch.empty_like(X)
        for _ in range(2):
            features_into(op, filt, X, F)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            features_into(op, filt, X, F)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        print(json.dumps({"config": args.config, "dtype": dtype, "w": w, "panel_width_opt": pw, "opts": args.opts,
                          "ms_per_filter": round(ms, 3), "ms_per_step": round(ms / P_ORDER, 4)}), flush=True)
        del X, F
    L.set_option("panel_width", 0)


if __name__ == "__main__":
    main()
