"""A/B-time the features filter under two builds of libcsc_b200.so on the same GPU.

python tools/ab_filter.py [--lib-a tools/_ab/libcsc_b200_base.so] [--lib-b paper_1602_02018_b200/libcsc_b200.so]
                          [--opts-a "unroll=2"] [--opts-b ""] [--config c3] [--width 0] [--dtype float32]
                          [--rounds 6] [--reps 20]

Each round runs one subprocess per build (alternating A, B, A, B, ... so clock and thermal drift
hit both); a subprocess builds the graph, warms up, then times --reps filters with CUDA events.
Prints per-round ms/filter and the min / median per build.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import json, math, sys
sys.path.insert(0, {root!r})
import paper_1602_02018_b200._lib as L
from pathlib import Path
L.LIB_PATH = Path({lib!r})
import torch
import paper_1602_02018_b200 as P
from paper_1602_02018_b200.features import features_into
from bench import CONFIGS, P_ORDER, make_graph
for kv in filter(None, {opts!r}.split(",")):
    k, v = kv.split("=")
    L.set_option(k, int(v))
cfg = CONFIGS[{config!r}]
dtype = {dtype!r} or cfg["dtype"]
N = cfg["N"]
d = {width} or int(math.ceil(4 * math.log(N)))
g, _ = make_graph(P, cfg)
if {weighted}:  # same edges, weights drawn from {{0.5, 1, 2.25, 3}} (symmetric: drawn per i < j edge)
    import numpy as np
    rows = np.repeat(np.arange(g.num_nodes), np.diff(g.indptr))
    keep = rows < g.indices
    w = np.random.default_rng(1).choice([0.5, 1.0, 2.25, 3.0], int(keep.sum()))
    g = P.build_graph(np.column_stack([rows[keep], g.indices[keep], w]), num_nodes=g.num_nodes)
op = P.laplacian_op(g, dtype=dtype)
tdt = torch.float32 if dtype == "float32" else torch.float64
X = torch.randn(N, d, dtype=torch.float64, device="cuda").div_(math.sqrt(d)).to(tdt)
F = torch.empty_like(X)
filt = P.design_lowpass(0.43, P_ORDER)
for _ in range(3):
    features_into(op, filt, X, F)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range({reps}):
    features_into(op, filt, X, F)
e1.record()
torch.cuda.synchronize()
print(json.dumps({{"ms": e0.elapsed_time(e1) / {reps}, "lib": L.LIB_PATH.name}}))
"""


def main():
    ap = argparse.ArgumentParser()
    lib = str(ROOT / "paper_1602_02018_b200" / "libcsc_b200.so")
    ap.add_argument("--lib-a", default=lib)
    ap.add_argument("--lib-b", default=lib)
    ap.add_argument("--opts-a", default="")
    ap.add_argument("--opts-b", default="")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--dtype", default="")
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--weighted", action="store_true", help="random edge weights on the config's graph")
    args = ap.parse_args()
    libs = {"A": str(Path(args.lib_a).resolve()), "B": str(Path(args.lib_b).resolve())}
    opts = {"A": args.opts_a, "B": args.opts_b}
    times: dict[str, list[float]] = {"A": [], "B": []}
    for r in range(args.rounds):
        for tag in ("A", "B") if r % 2 == 0 else ("B", "A"):
            code = CHILD.format(root=str(ROOT), lib=libs[tag], opts=opts[tag], config=args.config, dtype=args.dtype,
                                width=args.width, reps=args.reps, weighted=bool(args.weighted))
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=os.environ,
                                 cwd=str(ROOT))
            if out.returncode != 0:
                print(out.stderr[-2000:])
                raise SystemExit(f"{tag} failed")
            ms = json.loads(out.stdout.strip().splitlines()[-1])["ms"]
            times[tag].append(ms)
            print(f"round {r} {tag} {ms:8.3f} ms/filter", flush=True)
    for tag in ("A", "B"):
        t = times[tag]
        print(f"{tag} {Path(libs[tag]).name:24s} {opts[tag] or 'defaults':18s} min {min(t):8.3f}  median {statistics.median(t):8.3f} ms/filter "
              f"(config {args.config} width {args.width or 'default'} {args.dtype or 'config dtype'})")


if __name__ == "__main__":
    main()
