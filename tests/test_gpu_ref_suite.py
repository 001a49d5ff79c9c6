"""The reference's own hot-path test modules, re-pointed at the drop-in
through the ``cscluster`` alias of tests/ref_suite (run.py lists what is deselected and why)."""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


@pytest.mark.skipif(not (HERE.parent / "oracle" / "_ref" / "ref_tests").exists(),
                    reason="reference test modules not fetched (tests/ref_suite/run.py fetch)")
def test_reference_suite_passes_on_the_drop_in():
    out = subprocess.run([sys.executable, str(HERE / "ref_suite" / "run.py"), "-q"], capture_output=True, text=True,
                         timeout=1800)
    log = HERE.parent / "gpurun_out"
    if log.is_dir():
        (log / "ref_suite.log").write_text(out.stdout + out.stderr)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
