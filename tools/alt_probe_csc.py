import sys, time, math, gc
sys.path.insert(0, ".")
from bench import CONFIGS, make_graph
import paper_1602_02018_b200 as P
from paper_1602_02018_b200._rng import substream
import torch
cfg = CONFIGS["c3"]
g, truth = make_graph(P, cfg)
op = P.laplacian_op(g, dtype="float32")
def probe():
    t0 = time.perf_counter()
    P.estimate_lambda_k(op, 100, order=50, rng=substream(0, "probe"), private_rng=True, device_rng=True)
    return time.perf_counter() - t0
res = None
for r in range(4):
    print("probe", round(probe(), 4), flush=True)
    res = P.run_csc(op, P.CscParams(k=100, d=56, seed=0))
    t = res.diagnostics["timings"]
    print("csc", round(t["total"], 4), "probe", round(t["probe"], 4), "km", round(t["kmeans"], 4), flush=True)
    print("probe after csc (res alive)", round(probe(), 4), flush=True)
    res = None; gc.collect(); torch.cuda.empty_cache()
    print("probe after free", round(probe(), 4), flush=True)
