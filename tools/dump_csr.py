"""Write a BASELINE config's graph as raw int32 indptr / indices files (for tools/microbench).

python tools/dump_csr.py [--config c3] [--out /tmp/csr_c3]  ->  <out>.indptr.bin, <out>.indices.bin
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from bench import CONFIGS, make_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--out", default="/tmp/csr_c3")
    args = ap.parse_args()
    import paper_1602_02018_b200 as P

    g, _ = make_graph(P, CONFIGS[args.config])
    np.asarray(g.indptr, dtype=np.int32).tofile(args.out + ".indptr.bin")
    np.asarray(g.indices, dtype=np.int32).tofile(args.out + ".indices.bin")
    print(f"{args.config}: N={g.num_nodes} nnz={g.indices.size} -> {args.out}.*.bin")


if __name__ == "__main__":
    main()
