"""The reference's own pytest suite with its kernel seam (moesim.kernels.replay_policy) served
by the oracle's C replay (oracle/run_reference_suite.py).  Build container only: skipped where
/root/reference is absent (the GPU box)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not Path("/root/reference/pkg/tests").exists(), reason="reference not present")
def test_reference_suite_passes_with_oracle_replay():
    out = subprocess.run([sys.executable, str(ROOT / "oracle" / "run_reference_suite.py"),
                          "--deselect", "test_kernels.py::test_numpy_backend_subprocess_identical"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    tail = out.stdout[-3000:]
    assert out.returncode == 0, tail
    assert "208 passed" in tail and "oracle.replay_policy served" in tail, tail


@pytest.mark.skipif(not Path("/root/reference/pkg/tests").exists(), reason="reference not present")
def test_reference_host_tests_pass_on_this_package():
    """The reference's own test_traces / test_metrics / test_costmodel / test_simulate against
    this package's drop-in modules (`moesim.*` aliased to them; tests/refsuite_on_package.py).
    The single deselected test samples a Zipf trace, which is a GPU kernel here."""
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "refsuite_on_package.py"),
                          "-k", "not test_skew_increases_gini"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    tail = out.stdout[-3000:]
    assert out.returncode == 0, tail
    assert "61 passed" in tail, tail
