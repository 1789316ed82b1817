"""configs[0] tiny decode (graph mode) for launch-list profiling: 64 tokens."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse  # noqa: E402

import bench  # noqa: E402

a = argparse.Namespace(tiny_tokens=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
print(bench.run_tiny(a))
