"""Record every `moesim.kernels.replay_policy` call the reference's own pytest suite makes
(inputs and the reference's outputs, stock numba backend), deduplicated, as a fixture the GPU
replay is checked against (tests/test_replay_gpu.py::test_reference_suite_replay_calls); and
every distinct `moesim.toymoe.run_model(config)` call with its activation / speculation traces
(tests/test_toymoe_gpu.py::test_reference_suite_run_model_configs).

Runs only where /root/reference exists (the build container); nothing is written there.

python tests/golden/make_refsuite_golden.py   -> tests/golden/refsuite_replay.npz,
                                                 tests/golden/refsuite_run_model.npz
"""
import hashlib
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "refsuite_replay.npz"
OUT_RM = Path(__file__).resolve().parent / "refsuite_run_model.npz"


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF / "src"))
    import pytest

    seen, calls = set(), []
    rm_seen, rm_calls = set(), []

    class Record:
        def pytest_configure(self, config):
            import moesim.kernels as k

            stock = k.replay_policy

            def replay(acts, num_experts, capacity, policy, decay_factor, decay_period):
                rb, ev = stock(acts, num_experts, capacity, policy, decay_factor, decay_period)
                a = np.ascontiguousarray(acts, np.int64)
                key = hashlib.sha1(a.tobytes() + repr((a.shape, num_experts, capacity, policy,
                                                        float(decay_factor), int(decay_period))).encode()).digest()
                if key not in seen:
                    seen.add(key)
                    calls.append((a.copy(), int(num_experts), int(capacity), int(policy),
                                  float(decay_factor), int(decay_period), rb.copy(), ev.copy()))
                return rb, ev

            k.replay_policy = replay
            import moesim.toymoe as tm

            stock_rm = tm.run_model

            def run_model(cfg):
                act, spec = stock_rm(cfg)
                sh = cfg.shape
                key = (sh.num_layers, sh.num_experts, sh.top_k, cfg.hidden_dim,
                       float(cfg.mixing_scale), float(cfg.skew), cfg.seed, cfg.tokens)
                if key not in rm_seen:
                    rm_seen.add(key)
                    rm_calls.append((key, np.asarray(act.activations, np.int64),
                                     np.asarray(spec.guessed, np.int64), np.asarray(spec.actual, np.int64)))
                return act, spec

            tm.run_model = run_model

    rc = pytest.main([str(REF / "tests"), "-q", "-p", "no:cacheprovider",
                      "--rootdir", tempfile.mkdtemp(prefix="refsuite_")], plugins=[Record()])
    meta = np.array([[a.shape[0], a.shape[1], E, C, p, dp] for a, E, C, p, df, dp, _, _ in calls],
                    np.int64)
    dfs = np.array([df for _, _, _, _, df, _, _, _ in calls], np.float64)
    acts = np.concatenate([a.reshape(-1) for a, *_ in calls]).astype(np.int16)
    rb = np.packbits(np.concatenate([r.reshape(-1) for *_, r, _ in calls]).astype(np.uint8))
    ev = np.packbits(np.concatenate([e.reshape(-1) for *_, e in calls]).astype(np.uint8))
    np.savez_compressed(OUT, meta=meta, decay_factor=dfs, acts=acts, rb=rb, ev=ev)
    print(f"pytest rc={rc}; {len(calls)} distinct replay calls -> {OUT} "
          f"({OUT.stat().st_size / 1e6:.2f} MB)")
    keys = np.array([k for k, *_ in rm_calls], np.float64)   # L, E, K, d, alpha, skew, seed, T
    np.savez_compressed(OUT_RM, config=keys,
                        acts=np.concatenate([a.reshape(-1) for _, a, _, _ in rm_calls]).astype(np.int16),
                        guessed=np.concatenate([g.reshape(-1) for _, _, g, _ in rm_calls]).astype(np.int16),
                        actual=np.concatenate([x.reshape(-1) for *_, x in rm_calls]).astype(np.int16))
    print(f"{len(rm_calls)} distinct run_model configs -> {OUT_RM}")


if __name__ == "__main__":
    main()
