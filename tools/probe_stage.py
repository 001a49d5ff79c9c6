"""Time the probe stage (estimate_lambda_k as run_csc calls it) at a config, several times."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS, make_graph  # noqa: E402
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200._rng import substream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
cfg = CONFIGS[args.config]
g, _ = make_graph(P, cfg)
op = P.laplacian_op(g, dtype=cfg["dtype"])
for r in range(args.reps):
    t0 = time.perf_counter()
    est = P.estimate_lambda_k(op, cfg["k"], order=50, rng=substream(0, "probe"), private_rng=True, device_rng=True)
    print(f"rep {r}: {time.perf_counter() - t0:.4f} s, {est.iterations} probes, lambda {est.lambda_k_hat}", flush=True)
