"""``cscluster`` alias for re-running the reference's own test modules against the drop-in.

TEST INFRASTRUCTURE ONLY (never imported by the product).  ``import cscluster`` resolves
to ``paper_1602_02018_b200``: the package's public names, and its modules under the
reference's module names (``cscluster.graph`` is ``paper_1602_02018_b200.graph``, ...), so
``monkeypatch.setattr("cscluster.pipeline.kmeans", ...)`` patches the drop-in's own binding
(the seam reference test_pipeline.py:101-110 uses).

Names outside the hot path (SURVEY.md section 2 OUT OF SCOPE) that the reference modules
import at module level are supplied here as test doubles or stubs:
  - ``dense_eig`` / ``EigenBasis``: the dense oracle, restated as numpy.linalg.eigh of
    ``op.dense()`` (reference oracle.py:63-80; the reference uses its own Householder/QL);
    it is what the relational tests compare the GPU filter against;
  - ``error_split`` / ``check_resolution_bound`` / ``run_sc_baseline`` and the rest raise
    NotImplementedError; the tests that need them are deselected (tests/ref_suite/run.py).
"""

from __future__ import annotations

import importlib
import sys
from dataclasses import dataclass

import numpy as np

import paper_1602_02018_b200 as _P
from paper_1602_02018_b200 import *  # noqa: F401,F403

DEFAULT_DENSE_CAP = 5000


class DenseCapError(ValueError):
    pass


@dataclass
class EigenBasis:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray

    @property
    def num_nodes(self) -> int:
        return int(self.eigenvalues.size)

    def leading(self, k: int) -> np.ndarray:
        return self.eigenvectors[:, :k]


def dense_eig(op, *, cap: int = DEFAULT_DENSE_CAP, vectors: bool = True) -> EigenBasis:
    n = op.num_nodes
    if n > cap:
        raise DenseCapError(f"dense eigendecomposition refused for N={n} > cap={cap}")
    L = op.dense()
    if vectors:
        w, V = np.linalg.eigh(L)
        return EigenBasis(eigenvalues=w, eigenvectors=V)
    return EigenBasis(eigenvalues=np.linalg.eigvalsh(L), eigenvectors=np.empty((n, 0)))


def _out_of_scope(name):
    def stub(*args, **kwargs):
        raise NotImplementedError(f"{name} is outside the drop-in's hot path (SURVEY.md section 2)")

    stub.__name__ = name
    return stub


for _name in ("error_split", "check_resolution_bound", "run_sc_baseline", "spectral_clustering", "coherence",
              "modularity", "sweep", "expand_sweep_spec", "symmetric_eigh"):
    globals()[_name] = _out_of_scope(_name)

_oracle = type(sys)("cscluster.oracle")
_oracle.EigenBasis, _oracle.dense_eig, _oracle.DenseCapError = EigenBasis, dense_eig, DenseCapError
_oracle.DEFAULT_DENSE_CAP = DEFAULT_DENSE_CAP

# submodules by import path: the package attribute ``kmeans`` is the function, not the module
for _mod in ("graph", "filters", "spectrum", "features", "sampling", "pipeline", "kmeans", "result", "sbm", "_rng"):
    sys.modules[f"cscluster.{_mod}"] = importlib.import_module(f"paper_1602_02018_b200.{_mod}")
    # and as package attributes, where no public name shadows them (monkeypatch resolves
    # "cscluster.pipeline.kmeans" by getattr from the package)
    if _mod not in globals():
        globals()[_mod] = sys.modules[f"cscluster.{_mod}"]
sys.modules["cscluster.oracle"] = _oracle
oracle = _oracle
