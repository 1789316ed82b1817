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
