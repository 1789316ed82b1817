import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    return np.random.default_rng(0)


def random_stream(rng, E, K, T):
    return np.stack([np.sort(rng.choice(E, size=K, replace=False)) for _ in range(T)]).astype(np.int64) \
        if T else np.zeros((0, K), np.int64)


def golden_streams():
    """Yield (E, K, C, T, code, df, dp, acts, rb, ev) from the reference-generated fixture."""
    z = np.load(GOLDEN / "policy_streams.npz")
    idx, dfdp = z["index"], z["dfdp"]
    for (E, K, C, T, code, a_off, m_off), (df, dp) in zip(idx, dfdp):
        acts = z["acts"][a_off:a_off + T * K].reshape(T, K)
        rb = z["rb"][m_off:m_off + T * E].reshape(T, E)
        ev = z["ev"][m_off:m_off + T * E].reshape(T, E)
        yield int(E), int(K), int(C), int(T), int(code), float(df), int(dp), acts, rb, ev
