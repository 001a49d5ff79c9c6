"""Re-run the reference's own hot-path test modules against the drop-in (TEST INFRASTRUCTURE).

    python tests/ref_suite/run.py fetch      # in the build container: copy the modules from
                                            # /root/reference/pkg/tests into oracle/_ref/ref_tests/
                                            # (git-ignored: the place for reference-derived files)
    python tests/ref_suite/run.py [pytest args]   # on a GPU box: run them, ``cscluster`` -> the drop-in

The modules: test_graph, test_filters, test_spectrum, test_features,
test_sampling, test_pipeline, test_kmeans, plus their conftest.py / helpers.py.  They are not
committed (reference sources stay out of the repository); ``oracle/_ref/ref_tests/`` travels to the GPU
box with the working tree.  Deselected, with the reason:
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
VENDORED = HERE.parents[1] / "oracle" / "_ref" / "ref_tests"
SOURCE = Path("/root/reference/pkg/tests")
MODULES = ("conftest.py", "helpers.py", "test_graph.py", "test_filters.py", "test_spectrum.py",
           "test_features.py", "test_sampling.py", "test_pipeline.py", "test_kmeans.py")

DESELECT = {
    # Theorem 4.1 diagnostics (error_split / check_resolution_bound): OUT OF SCOPE, SURVEY.md section 2
    "test_filters.py::TestApply::test_excluded_eigenvector_suppressed": "needs error_split (out of scope)",
    "test_filters.py::TestErrorSplit::test_ideal_filter_zero_errors": "error_split (out of scope)",
    "test_filters.py::TestErrorSplit::test_error_shrinks_with_order": "error_split (out of scope)",
    "test_filters.py::TestErrorSplit::test_requires_sorted_spectrum": "error_split (out of scope)",
    "test_filters.py::TestResolutionBound": "check_resolution_bound (out of scope)",
    # exact-SC baseline: OUT OF SCOPE (dense oracle)
    "test_pipeline.py::TestRunScBaseline": "run_sc_baseline (dense oracle, out of scope)",
    # fail against the reference itself as shipped
    "test_pipeline.py::TestDefaults::test_n_capped_at_graph_size": "fails on the reference (test arithmetic)",
    "test_pipeline.py::TestRunCsc::test_lambda_warning_marks_run": "fails on the reference (count reaches k)",
}


def fetch() -> None:
    VENDORED.mkdir(parents=True, exist_ok=True)
    for name in MODULES:
        shutil.copyfile(SOURCE / name, VENDORED / name)
    print(f"copied {len(MODULES)} files to {VENDORED}")


def run(extra: list[str]) -> int:
    if not VENDORED.exists():
        print(f"{VENDORED} missing: run `python {__file__} fetch` in the build container first")
        return 2
    repo = HERE.parents[1]
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(HERE / "shim"), str(repo), str(VENDORED), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", str(VENDORED), "-p", "no:cacheprovider", "--rootdir", str(VENDORED),
           "--confcutdir", str(VENDORED), "-o", "addopts=", "-rA"]
    for node in DESELECT:
        cmd += ["--deselect", node]
    return subprocess.call(cmd + extra, env=env, cwd=str(VENDORED))


if __name__ == "__main__":
    if sys.argv[1:2] == ["fetch"]:
        fetch()
    else:
        sys.exit(run(sys.argv[1:]))
