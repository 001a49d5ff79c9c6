"""Time SBM generation at a config: host restatement vs device generator, and the CSR build."""
import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1602_02018_b200 as P  # noqa: E402
from paper_1602_02018_b200.sbm import sbm_edges, sbm_edges_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=1_000_000)
ap.add_argument("--k", type=int, default=100)
ap.add_argument("--host", action="store_true")
args = ap.parse_args()
cfg = P.SbmConfig(num_nodes=args.N, k=args.k, avg_degree=16, epsilon=P.critical_epsilon(16, args.k) / 4, seed=0)
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    src, dst, _ = sbm_edges_device(cfg, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g, _ = P.sbm_generate(cfg)
    t2 = time.perf_counter()
    print(f"device edges {t1 - t0:.3f} s ({src.numel()} edges); sbm_generate (device edges + CSR + export) {t2 - t1:.3f} s",
          flush=True)
if args.host:
    t0 = time.perf_counter()
    sbm_edges(cfg)
    print(f"host edges {time.perf_counter() - t0:.3f} s", flush=True)
