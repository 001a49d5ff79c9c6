"""Clustering result container (reference result.py).

``soft`` may be held on the GPU by the pipeline; it is copied to a host fp64
array the first time it is read, so runs that only need labels never pay the
N x k device-to-host copy.
"""

from __future__ import annotations

import csv
import json
from pathlib import Path
from typing import Any

import numpy as np


def _plain(v: Any) -> Any:
    if isinstance(v, np.ndarray):
        return [_plain(x) for x in v.tolist()]
    if isinstance(v, np.bool_):
        return bool(v)
    if isinstance(v, np.integer):
        return int(v)
    if isinstance(v, np.floating):
        return float(v)
    if isinstance(v, dict):
        return {k: _plain(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_plain(x) for x in v]
    return v


class ClusterResult:
    """Hard partition, soft indicators (N x k) and run diagnostics."""

    def __init__(self, labels: np.ndarray, soft: Any, diagnostics: dict[str, Any] | None = None,
                 num_clusters: int | None = None):
        self.labels = labels
        self._soft = soft
        self.diagnostics = {} if diagnostics is None else diagnostics
        self._k = num_clusters  # set when ``soft`` holds only this rank's columns (column-sharded runs)

    @property
    def soft(self) -> np.ndarray:
        s = self._soft
        if not isinstance(s, np.ndarray):
            s = s.detach().to("cpu").double().numpy()
            self._soft = s
        return s

    @soft.setter
    def soft(self, value) -> None:
        self._soft = value

    @property
    def num_nodes(self) -> int:
        return int(self.labels.size)

    @property
    def num_clusters(self) -> int:
        return int(self._k if self._k is not None else self._soft.shape[1])

    def to_dict(self, *, include_timings: bool = False) -> dict[str, Any]:
        diag = {k: _plain(v) for k, v in self.diagnostics.items() if include_timings or k != "timings"}
        return {
            "diagnostics": diag,
            "labels": [int(x) for x in self.labels],
            "num_clusters": self.num_clusters,
            "num_nodes": self.num_nodes,
        }

    def to_json(self, *, include_timings: bool = False, indent: int | None = None) -> str:
        return json.dumps(self.to_dict(include_timings=include_timings), sort_keys=True, indent=indent)

    def save_json(self, path, *, include_timings: bool = False) -> None:
        Path(path).write_text(self.to_json(include_timings=include_timings, indent=2) + "\n", encoding="utf-8")

    def save_labels_csv(self, path) -> None:
        with Path(path).open("w", encoding="utf-8", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["node_id", "label"])
            for i, lab in enumerate(self.labels):
                w.writerow([i, int(lab)])
