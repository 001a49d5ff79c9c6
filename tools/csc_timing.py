"""Time run_csc at a BASELINE config several times (cold + warm) with stage timings."""
import argparse
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS, make_graph  # noqa: E402
import paper_1602_02018_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dtype", default=None)
ap.add_argument("--option", action="append", default=[], help="libcsc option key=value")
ap.add_argument("--lib", default=None, help="another build of libcsc_b200.so (A/B)")
args = ap.parse_args()
from paper_1602_02018_b200 import _lib  # noqa: E402

if args.lib:
    _lib.LIB_PATH = Path(args.lib).resolve()

for kv in args.option:
    key, val = kv.split("=")
    _lib.set_option(key, int(val))
cfg = CONFIGS[args.config]
g, truth = make_graph(P, cfg)
op = P.laplacian_op(g, dtype=args.dtype or cfg["dtype"])
d = int(math.ceil(4 * math.log(cfg["N"])))
res = None
for r in range(args.reps):
    del res  # the previous result's N x k soft indicators (64 GB at C5) must not outlive the next call
    res = None
    t0 = time.perf_counter()
    res = P.run_csc(op, P.CscParams(k=cfg["k"], d=d, seed=0))
    wall = time.perf_counter() - t0
    print(json.dumps({"rep": r, "wall_s": round(wall, 4), "stages": {k: round(v, 4) for k, v in res.diagnostics["timings"].items()},
                      "lambda": res.diagnostics["lambda_k_hat"], "ari": round(P.adjusted_rand_index(truth, res.labels), 4)}), flush=True)
