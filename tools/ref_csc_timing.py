"""Time the reference package's own run_csc on this host's CPU (this container only: it
imports the read-only reference tree) at C1/C2 and write profiles/ref_csc_cpu.json."""
import json
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
import cscluster as R  # noqa: E402

out = {}
for name, N, k in (("c1", 1000, 20), ("c2", 100_000, 20)):
    cfg = R.SbmConfig(num_nodes=N, k=k, avg_degree=16, epsilon=R.critical_epsilon(16, k) / 4, seed=0)
    t0 = time.perf_counter()
    g, truth = R.sbm_generate(cfg)
    t_gen = time.perf_counter() - t0
    op = R.laplacian_op(g)
    d = int(math.ceil(4 * math.log(N)))
    t0 = time.perf_counter()
    res = R.run_csc(op, R.CscParams(k=k, d=d, seed=0))
    wall = time.perf_counter() - t0
    out[name] = {"N": N, "k": k, "d": d, "wall_s": wall, "sbm_generate_s": t_gen,
                 "stages_s": res.diagnostics["timings"], "lambda_k_hat": res.diagnostics["lambda_k_hat"],
                 "probe_iterations": res.diagnostics["probe_iterations"],
                 "ari_vs_truth": R.adjusted_rand_index(truth, res.labels), "cores": 1, "host_nproc": os.cpu_count()}
    print(name, json.dumps(out[name]), flush=True)
Path(__file__).resolve().parents[1].joinpath("profiles", "ref_csc_cpu.json").write_text(json.dumps(out, indent=1))
