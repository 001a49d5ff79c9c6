"""Per-column CG comparison against the reference capture (tests/golden/pipeline_<tag>.npz):
iterations, final residual / target, and the indicator columns' relative difference on the
captured row subsample.  python tools/headline_cg_diag.py [c4|c3] [float64|float32]"""
import json, math, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1602_02018_b200 as P
from conftest import golden, sbm_config

tag = sys.argv[1] if len(sys.argv) > 1 else "c4"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
if len(sys.argv) > 3:  # recurrence option: 0 Clenshaw (default), 1 forward -- another valid operation order
    from paper_1602_02018_b200 import _lib
    _lib.set_option("recurrence", int(sys.argv[3]))
gz = golden(f"pipeline_{tag}")
if tag == "c3":
    g, truth = P.sbm_generate(sbm_config(1_000_000, 100))
else:
    from paper_1602_02018_b200.sbm import c4_config
    g, truth, _ = P.dcsbm_generate(c4_config())
k = int(gz["truth"].max()) + 1
N = g.num_nodes
res = P.run_csc(P.laplacian_op(g, dtype=dtype), P.CscParams(k=k, d=int(math.ceil(4 * math.log(N))), seed=0))
d = res.diagnostics
cnt = np.bincount(gz["kmeans_labels"], minlength=k)
target = 1e-6 * np.sqrt(cnt)
its, rits = np.asarray(d["solver_iterations"]), gz["solver_iterations"]
rr, ours = gz["solver_residuals"], np.asarray(d["solver_residuals"])
S, R = res.soft[gz["rows"]], gz["soft_rows"]
nr = np.linalg.norm(R, axis=0)
colerr = np.where(nr > 0, np.linalg.norm(S - R, axis=0) / np.where(nr > 0, nr, 1.0), np.linalg.norm(S - R, axis=0))
np.savez_compressed(ROOT / "gpurun_out" / f"cgdiag_{tag}_{dtype}_{sys.argv[3] if len(sys.argv) > 3 else 0}.npz",
                    its=its, soft_rows=S, labels=res.labels.astype(np.int32), residuals=ours)
print(f"{tag} {dtype}: columns {k}, iterations equal {int((its == rits).sum())}, max |dX|/|X| over equal-iteration columns "
      f"{colerr[its == rits].max():.3e}, overall soft_rows relerr {np.linalg.norm(S - R) / np.linalg.norm(R):.3e}")
print(f"  final residual / target: reference min {np.min(rr / target):.4f} max {np.max(rr / target):.4f}; ours min "
      f"{np.min(ours / target):.4f} max {np.max(ours / target):.4f}")
for j in np.flatnonzero(its != rits):
    print(f"  column {j}: ours {its[j]} reference {rits[j]}; final residual/target ours {ours[j] / target[j]:.4f} "
          f"reference {rr[j] / target[j]:.4f}; column relerr {colerr[j]:.3e}")
eq = its == rits
srt = np.sort(colerr[eq])[::-1]
print("  equal-iteration columns, largest column relerr:", " ".join(f"{x:.2e}" for x in srt[:8]),
      "| median", f"{np.median(colerr[eq]):.2e}")
worst = np.argsort(-np.where(eq, colerr, 0))[:5]
for j in worst:
    print(f"    column {j}: iterations {its[j]}, reference residual/target {rr[j] / target[j]:.4f}, relerr {colerr[j]:.2e}")
print("  labels ARI vs reference", P.adjusted_rand_index(res.labels, gz["labels"]), "identical labels",
      int((res.labels == gz["labels"]).sum()), "of", N)
