"""Kernel timeline of the bench's features step (torch.profiler / CUPTI): per-kernel durations and
the GPU idle gaps between consecutive kernels over a few steps.

python tools/step_timeline.py [--config c3] [--steps 3]
"""

from __future__ import annotations

import argparse
import math
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import CONFIGS, P_ORDER, make_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--async-steps", action="store_true", help="features_into(..., zero_rows=False)")
    ap.add_argument("--csc", action="store_true", help="profile one warm run_csc instead of feature steps")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200.features import features_into

    cfg = CONFIGS[args.config]
    N = cfg["N"]
    d = int(math.ceil(4 * math.log(N)))
    g, _ = make_graph(P, cfg)
    op = P.laplacian_op(g, dtype=cfg["dtype"])
    X = torch.randn(N, d, dtype=torch.float64, device="cuda").div_(math.sqrt(d)).float()
    F = torch.empty_like(X)
    filt = P.design_lowpass(0.43, P_ORDER)
    for _ in range(3):
        features_into(op, filt, X, F)
    torch.cuda.synchronize()
    if args.csc:
        prm = P.CscParams(k=cfg["k"], d=d, seed=0)
        P.run_csc(op, prm)
        torch.cuda.synchronize()
        args.steps = 1
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            if args.csc:
                P.run_csc(op, prm)
            else:
                features_into(op, filt, X, F, zero_rows=not args.async_steps)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    gaps = 0.0
    for a, b in zip(evs, evs[1:]):
        gaps += max(0.0, b.time_range.start - a.time_range.end)
    for e in evs:
        key = e.name[:80]
        tot[key] += e.time_range.end - e.time_range.start
        cnt[key] += 1
    span = evs[-1].time_range.end - evs[0].time_range.start
    print(f"{args.steps} steps: span {span / 1e3 / args.steps:.3f} ms/step, busy {sum(tot.values()) / 1e3 / args.steps:.3f}, "
          f"gaps {gaps / 1e3 / args.steps:.3f} ms/step")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {v / 1e3 / args.steps:8.3f} ms/step  {cnt[k] // args.steps:4d}/step  {k}")
    # idle time: the span minus the union of all (possibly concurrent) device intervals, and
    # the largest idle intervals with the work on either side
    idle = []
    end, last = evs[0].time_range.end, evs[0]
    for e in evs[1:]:
        if e.time_range.start > end:
            idle.append((e.time_range.start - end, last.name[:50], e.name[:50], end - evs[0].time_range.start))
        if e.time_range.end > end:
            end, last = e.time_range.end, e
    print(f"idle (span - union of device intervals): {sum(i[0] for i in idle) / 1e3 / args.steps:.3f} ms/step in "
          f"{len(idle)} intervals")
    for us, a, b, at in sorted(idle, reverse=True)[:15]:
        print(f"  {us:9.1f} us at {at / 1e3:9.3f} ms  after {a}  before {b}")


if __name__ == "__main__":
    main()
