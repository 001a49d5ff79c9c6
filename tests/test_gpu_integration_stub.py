"""The ctypes binding INTEGRATION.md shows for the reference package runs as written."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import relerr
from gpu_util import c1_graph, c1_op
import paper_1602_02018_b200 as P

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_integration_md_ctypes_stub():
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(# cscluster/_b200\.py\n.*?)```", text, re.S).group(1)
    lib = str(ROOT / "paper_1602_02018_b200" / "libcsc_b200.so")
    ns: dict = {}
    exec(compile(block.replace('"libcsc_b200.so"', repr(lib)), "INTEGRATION.md", "exec"), ns)
    g, _ = c1_graph()
    op = ns["B200Laplacian"](g)
    X = np.random.default_rng(4).standard_normal((g.num_nodes, 5))
    filt = P.design_lowpass(0.45, 50)
    assert relerr(ns["apply_filter"](filt, op, X), P.apply_filter(filt, c1_op(), X)) <= 1e-14
    assert ns["apply_filter"](filt, op, X[:, 0]).shape == (g.num_nodes,)
