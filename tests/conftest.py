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


def refsuite_calls():
    """Every distinct moesim.kernels.replay_policy call of the reference's own test suite,
    with the reference's outputs (tests/golden/make_refsuite_golden.py):
    yields (acts (T,K) int64, E, C, policy, decay_factor, decay_period, rb (T,E), ev (T,E))."""
    z = np.load(GOLDEN / "refsuite_replay.npz")
    meta, dfs = z["meta"], z["decay_factor"]
    n_out = int((meta[:, 0] * meta[:, 2]).sum())
    rb_all = np.unpackbits(z["rb"])[:n_out]
    ev_all = np.unpackbits(z["ev"])[:n_out]
    acts_all = z["acts"].astype(np.int64)
    ia = io = 0
    for (T, K, E, C, pol, dp), df in zip(meta, dfs):
        T, K, E = int(T), int(K), int(E)
        acts = acts_all[ia: ia + T * K].reshape(T, K)
        rb = rb_all[io: io + T * E].reshape(T, E)
        ev = ev_all[io: io + T * E].reshape(T, E)
        ia += T * K
        io += T * E
        yield acts, E, int(C), int(pol), float(df), int(dp), rb, ev


def refsuite_run_models():
    """Every distinct moesim.toymoe.run_model config of the reference's own test suite with the
    reference's traces (tests/golden/make_refsuite_golden.py): yields
    ((L, E, K, d, alpha, skew, seed, T), acts (T,L,K), guessed (T,L-1,K), actual (T,L-1,K))."""
    z = np.load(GOLDEN / "refsuite_run_model.npz")
    ia = ig = 0
    for row in z["config"]:
        L, E, K, d = (int(v) for v in row[:4])
        alpha, skew = float(row[4]), float(row[5])
        seed, T = int(row[6]), int(row[7])
        Ts = T if L >= 2 else 0   # the reference returns empty speculation grids (toymoe.py:187-189)
        na, ng = T * L * K, Ts * max(L - 1, 0) * K
        acts = z["acts"][ia: ia + na].astype(np.int64).reshape(T, L, K)
        guessed = z["guessed"][ig: ig + ng].astype(np.int64).reshape(Ts, max(L - 1, 0), K)
        actual = z["actual"][ig: ig + ng].astype(np.int64).reshape(Ts, max(L - 1, 0), K)
        ia += na
        ig += ng
        yield (L, E, K, d, alpha, skew, seed, T), acts, guessed, actual


def refsuite_policy_steps():
    """Every distinct moesim.policies.policy_step call of the reference's suite, with the
    reference's result (state + outcome) or the name of the error it raised."""
    import gzip
    import json

    with gzip.open(GOLDEN / "refsuite_policy_step.jsonl.gz", "rt") as f:
        for line in f:
            yield json.loads(line)


def refsuite_tracegen_calls():
    """Every distinct gen_zipf / gen_markov call of the reference's suite with its trace:
    yields (meta dict, acts (T, L, K))."""
    z = np.load(GOLDEN / "refsuite_tracegen.npz")
    i = 0
    for m in z["meta"]:
        kind, L, E, K, T = (int(v) for v in m[:5])
        meta = dict(kind="zipf" if kind == 0 else "markov", L=L, E=E, K=K, T=T, skew=float(m[5]),
                    per_layer_permutation=bool(int(m[6])), seed=int(m[7]), repeat_prob=float(m[8]),
                    base_tokens=int(m[10]), base_seed=int(m[11]))
        n = T * L * K
        yield meta, z["acts"][i: i + n].astype(np.int64).reshape(T, L, K)
        i += n
