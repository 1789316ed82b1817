"""Record every `moesim.kernels.replay_policy` call the reference's own pytest suite makes
(inputs and the reference's outputs, stock numba backend), deduplicated, as a fixture the GPU
replay is checked against (tests/test_replay_gpu.py::test_reference_suite_replay_calls); and
every distinct `moesim.toymoe.run_model(config)` call with its activation / speculation traces
(tests/test_toymoe_gpu.py::test_reference_suite_run_model_configs); every distinct
`moesim.policies.policy_step` call with its result or error (tests/test_replay_gpu.py::
test_reference_suite_policy_steps); every distinct `gen_zipf` / `gen_markov` call with its trace
(tests/test_tracegen.py::test_reference_suite_tracegen_calls); every gate_select /
speculate_next / forward_token call with its result or error
(tests/test_toymoe_gpu.py::test_reference_suite_model_api_calls).

Runs only where /root/reference exists (the build container); nothing is written there.

python tests/golden/make_refsuite_golden.py   -> tests/golden/refsuite_replay.npz,
                                                 tests/golden/refsuite_run_model.npz,
                                                 tests/golden/refsuite_policy_step.jsonl.gz,
                                                 tests/golden/refsuite_tracegen.npz,
                                                 tests/golden/refsuite_toymoe_calls.json.gz
"""
import gzip
import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "refsuite_replay.npz"
OUT_RM = Path(__file__).resolve().parent / "refsuite_run_model.npz"
OUT_PS = Path(__file__).resolve().parent / "refsuite_policy_step.jsonl.gz"
OUT_TG = Path(__file__).resolve().parent / "refsuite_tracegen.npz"
OUT_TM = Path(__file__).resolve().parent / "refsuite_toymoe_calls.json.gz"


def _state(st):
    return {"capacity": st.capacity, "resident": sorted(int(e) for e in st.resident),
            "recency": [int(e) for e in st.recency],
            "freq": sorted([int(e), float(f)] for e, f in st.freq.items()), "step": int(st.step)}


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF / "src"))
    import pytest

    seen, calls = set(), []
    rm_seen, rm_calls = set(), []
    ps_seen, ps_calls = set(), []
    tg_seen, tg_calls = set(), []
    tm_calls = []

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
            import moesim.policies as pm

            stock_ps = pm.policy_step

            def policy_step(state, kind, activated, future=None):
                rec = {"state": _state(state), "kind": str(kind), "activated": [int(e) for e in activated],
                       "future": None if future is None else [sorted(int(e) for e in f) for f in future]}
                try:
                    st2, out = stock_ps(state, kind, activated, future)
                    rec["result"] = {"state": _state(st2), **{
                        k: sorted(int(e) for e in getattr(out, k))
                        for k in ("hits", "misses", "evicted", "loaded", "resident_before", "resident_after")}}
                except Exception as exc:  # the reference's validation errors are part of the contract
                    rec["error"] = type(exc).__name__
                    st2 = out = None
                key = json.dumps(rec, sort_keys=True)
                if key not in ps_seen:
                    ps_seen.add(key)
                    ps_calls.append(rec)
                if st2 is None:
                    raise exc_of(rec["error"])
                return st2, out

            def exc_of(name):
                from moesim import errors

                return getattr(errors, name, ValueError)("recorded")

            pm.policy_step = policy_step
            def record_call(kind, args, fn):
                rec = {"kind": kind, **args}
                try:
                    res = fn()
                except Exception as exc:
                    rec["error"] = type(exc).__name__
                    tm_calls.append(rec)
                    raise
                if kind == "gate_select":
                    rec["result"] = [[int(e), float(p)] for e, p in res]
                elif kind == "speculate_next":
                    rec["result"] = sorted(int(e) for e in res)
                else:
                    rec["result"] = {"values": [float(v) for v in res[0].values], "layer": int(res[0].layer),
                                     "selected": sorted(int(e) for e in res[1])}
                tm_calls.append(rec)
                return res

            def gate_args(h, gate, k):
                return {"h": [float(v) for v in h.values], "h_layer": int(h.layer),
                        "w": np.asarray(gate.weights, np.float64).tolist(),
                        "b": None if gate.bias is None else np.asarray(gate.bias, np.float64).tolist(), "k": int(k)}

            stock_gs, stock_sn, stock_ft = tm.gate_select, tm.speculate_next, tm.forward_token
            tm.gate_select = lambda h, gate, k: record_call("gate_select", gate_args(h, gate, k),
                                                            lambda: stock_gs(h, gate, k))
            tm.speculate_next = lambda h, gate, k: record_call("speculate_next", gate_args(h, gate, k),
                                                               lambda: stock_sn(h, gate, k))

            def forward_token(model, h_in, layer):
                c = model.config
                args = {"config": [c.shape.num_layers, c.shape.num_experts, c.shape.top_k, c.hidden_dim,
                                   float(c.mixing_scale), float(c.skew), c.seed, c.tokens],
                        "h": [float(v) for v in h_in.values], "h_layer": int(h_in.layer), "layer": int(layer),
                        # the model's actual arrays (tests may hand-build or alter them)
                        "weights": {"gate_w": [np.asarray(g.weights, np.float64).tolist() for g in model.gates],
                                    "gate_b": [None if g.bias is None else np.asarray(g.bias, np.float64).tolist()
                                               for g in model.gates],
                                    "mixing": np.asarray(model.mixing, np.float64).tolist(),
                                    "w1": np.asarray(model.expert_w1, np.float64).tolist(),
                                    "w2": np.asarray(model.expert_w2, np.float64).tolist()}}
                return record_call("forward_token", args, lambda: stock_ft(model, h_in, layer))

            tm.forward_token = forward_token
            import moesim.tracegen as tg

            for fname in ("gen_zipf", "gen_markov"):
                stock_g = getattr(tg, fname)

                def gen(params, _stock=stock_g, _name=fname):
                    tr = _stock(params)
                    sh = params.shape
                    if _name == "gen_zipf":
                        meta = (0, sh.num_layers, sh.num_experts, sh.top_k, params.num_tokens,
                                float(params.skew_exponent), int(params.per_layer_permutation),
                                params.seed, 0.0, 0.0, 1, 0)
                    else:
                        b = params.base
                        meta = (1, sh.num_layers, sh.num_experts, sh.top_k, params.num_tokens,
                                float(b.skew_exponent), int(b.per_layer_permutation), params.seed,
                                float(params.repeat_prob), 0.0, b.num_tokens, b.seed)
                    if meta not in tg_seen:
                        tg_seen.add(meta)
                        tg_calls.append((meta, np.asarray(tr.activations, np.int64)))
                    return tr

                setattr(tg, fname, gen)

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
    with open(OUT_PS, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
        for rec in ps_calls:
            f.write((json.dumps(rec, sort_keys=True) + "\n").encode())
    print(f"{len(ps_calls)} distinct policy_step calls -> {OUT_PS} ({OUT_PS.stat().st_size / 1e6:.2f} MB)")
    np.savez_compressed(OUT_TG, meta=np.array([m for m, _ in tg_calls], np.float64),
                        acts=np.concatenate([a.reshape(-1) for _, a in tg_calls]).astype(np.int16))
    print(f"{len(tg_calls)} distinct tracegen calls -> {OUT_TG} ({OUT_TG.stat().st_size / 1e6:.2f} MB)")
    with open(OUT_TM, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as f:
        f.write(json.dumps(tm_calls, sort_keys=True).encode())
    print(f"{len(tm_calls)} gate_select / speculate_next / forward_token calls -> {OUT_TM}")


if __name__ == "__main__":
    main()
