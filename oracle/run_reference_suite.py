"""ORACLE -- test infrastructure only (see oracle/__init__.py).  Runs in the build container,
never on the GPU box (it reads /root/reference).

Pins the oracle's policy replay (oracle/replay.c) with the reference's OWN test suite: the
reference package is imported read-only from /root/reference/pkg/src, its
`moesim.kernels.replay_policy` (kernels.py:60-147, the seam every simulate / compare / sweep
path goes through, simulate.py:169) is replaced by `oracle.replay_policy`, and the
reference's pytest suite runs unchanged.  Nothing is written under /root/reference (no
bytecode, no pytest cache, numba's cache in /tmp).

python oracle/run_reference_suite.py [pytest args...]   -> exit code of pytest

Result here: 208 passed, 1 failed -- the same single failure the reference has on its own
(test_kernels.py::test_numpy_backend_subprocess_identical spawns `python -c "import moesim"`
with a scrubbed environment, which needs `pip install -e`).
"""
import os
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parents[1]


class _PatchReplay:
    """pytest plugin: swap the reference kernel seam for the oracle before collection."""

    def __init__(self):
        self.calls = 0

    def pytest_configure(self, config):
        import moesim.kernels as k

        import oracle

        def replay(acts, num_experts, capacity, policy, decay_factor, decay_period):
            self.calls += 1
            return oracle.replay_policy(acts, num_experts, capacity, policy, decay_factor,
                                        decay_period)

        k.replay_policy = replay

    def pytest_terminal_summary(self, terminalreporter):
        terminalreporter.write_line(f"oracle.replay_policy served {self.calls} replay calls")


def main(argv):
    if not REF.exists():
        print("reference not present (GPU box): nothing to run")
        return 0
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF / "src"))
    sys.path.insert(0, str(ROOT))
    import pytest

    args = [str(REF / "tests"), "-q", "-p", "no:cacheprovider",
            "--rootdir", tempfile.mkdtemp(prefix="refsuite_")] + list(argv)
    return pytest.main(args, plugins=[_PatchReplay()])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
