"""K4 isolated: 8 resident Mixtral-8x7B experts x 128 token rows, grouped SwiGLU up and grouped
down (split 1), as in bench.py's gemm_isolated.  Run under ncu for the full-set capture."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402

print(bench.isolated_gemm(4096, 14336))
