import sys, collections
sys.path.insert(0, "/root/repo")
from bench import CONFIGS, make_graph
import paper_1602_02018_b200 as P
g, truth = make_graph(P, CONFIGS["c3"])
op = P.laplacian_op(g, dtype="float32")
r = P.run_csc(op, P.CscParams(k=100, d=56, seed=0))
its = r.diagnostics["solver_iterations"]
print(sorted(collections.Counter(its).items()))
print("panel maxima (32-wide):", [max(its[i:i + 32]) for i in range(0, 100, 32)], "sum", sum(its), "vs", 100 * max(its))
