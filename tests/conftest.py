from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"

# the reference's own test modules run through tests/ref_suite/run.py (own rootdir and a
# ``cscluster`` alias), driven by tests/test_gpu_ref_suite.py, never collected directly
collect_ignore = ["ref_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libcsc_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def c1_config():
    from paper_1602_02018_b200.sbm import SbmConfig, critical_epsilon

    return SbmConfig(num_nodes=1000, k=20, avg_degree=16.0, epsilon=critical_epsilon(16.0, 20) / 4.0, seed=0)


def sbm_config(N, k, s=16.0, seed=0):
    from paper_1602_02018_b200.sbm import SbmConfig, critical_epsilon

    return SbmConfig(num_nodes=N, k=k, avg_degree=s, epsilon=critical_epsilon(s, k) / 4.0, seed=seed)


def relerr(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="session")
def c1_golden():
    return golden("pipeline_c1")


@pytest.fixture(scope="session")
def graphs_golden():
    return golden("graphs")


@pytest.fixture(scope="session")
def filter_golden():
    return golden("filter_c1")


D_C1 = int(math.ceil(4 * math.log(1000)))
