"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the reference is not on the GPU box):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py
It imports moesim from /root/reference/pkg/src (read-only; numba's cache is redirected to
/tmp so nothing is written into the reference tree) and writes small fixtures:

  policy_streams.npz   random activation streams x all policies -> replay_policy masks
  toy_t1/*.jsonl       tiny config (L=4,E=8,K=2,d=256,alpha=0.1,seed=42,T=64): activation
                       and speculation traces, event logs LRU/LFU at C=2 and C=4
  toy_t1_1024.npz      the same config at T=1024: activations, guesses + event-log digests
  toy_small.npz        small run_model configs (incl. the reference's straight-line case)
  forward_cases.npz    forward_token / gate_select outputs on random small models
  tracegen.npz         gen_zipf / gen_markov traces (tracegen.py:78-112) for a set of params
  manifest.json        sha256 of every artefact + versions used
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import moesim  # noqa: E402
from moesim import kernels  # noqa: E402
from moesim.policies import PolicyKind  # noqa: E402
from moesim.simulate import SimConfig, simulate, write_event_log  # noqa: E402
from moesim.toymoe import (  # noqa: E402
    HiddenState, ToyModelConfig, ToyMoeModel, forward_token, gate_select, run_model)
from moesim.traces import ModelShape, write_trace  # noqa: E402
from moesim.metrics import cache_metrics, speculation_metrics  # noqa: E402

OUT = Path(__file__).resolve().parent
POLICIES = [
    ("lru", 0, 1.0, 1), ("lfu", 1, 1.0, 1), ("lfu-aged:0.5:4", 2, 0.5, 4),
    ("lfu-aged:0.3:3", 2, 0.3, 3), ("lfu-aged:0.7:5", 2, 0.7, 5), ("lfu-aged:0.9:1", 2, 0.9, 1),
    ("opt", 3, 1.0, 1),
]


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def trace_bytes(tr) -> bytes:
    buf = io.BytesIO()
    write_trace(tr, buf)
    return buf.getvalue()


def log_bytes(log) -> bytes:
    buf = io.BytesIO()
    write_event_log(log, buf)
    return buf.getvalue()


def policy_streams(manifest):
    rng = np.random.default_rng(2511)
    acts_all, rb_all, ev_all, index = [], [], [], []
    a_off = m_off = 0
    for n in range(400):
        E = int(rng.integers(2, 9)) if n < 300 else int(rng.integers(9, 40))
        K = int(rng.integers(1, min(E, 8) + 1))
        C = int(rng.integers(K, E + 1))
        T = int(rng.integers(1, 80))
        acts = np.stack([np.sort(rng.choice(E, size=K, replace=False)) for _ in range(T)]).astype(np.int64)
        for name, code, df, dp in POLICIES:
            rb, ev = kernels.replay_policy(acts, E, C, code, df, dp)
            index.append([E, K, C, T, code, a_off, m_off])
            rb_all.append(rb.ravel())
            ev_all.append(ev.ravel())
            acts_all.append(acts.ravel())
            a_off += acts.size
            m_off += rb.size
    np.savez_compressed(
        OUT / "policy_streams.npz", index=np.array(index, np.int64),
        dfdp=np.array([[df, dp] for _ in range(400) for (_, _, df, dp) in POLICIES], np.float64),
        acts=np.concatenate(acts_all), rb=np.concatenate(rb_all), ev=np.concatenate(ev_all))
    manifest["policy_streams.npz"] = {"streams": 400, "policies": [p[0] for p in POLICIES]}


def toy_t1(manifest):
    d = OUT / "toy_t1"
    d.mkdir(exist_ok=True)
    cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, skew=1.0,
                         seed=42, tokens=64)
    act, spec = run_model(cfg)
    files = {"activation.jsonl": trace_bytes(act), "speculation.jsonl": trace_bytes(spec)}
    digests = {}
    for pol in ("lru", "lfu"):
        for C in (2, 4):
            log = simulate(act, SimConfig(policy=PolicyKind.parse(pol), cache_size=C))
            files[f"events_{pol}_c{C}.jsonl"] = log_bytes(log)
            m = cache_metrics(log)
            digests[f"{pol}_c{C}"] = {"hits": m.total_hits, "misses": m.total_misses,
                                      "hit_rate": m.hit_rate}
    for name, b in files.items():
        (d / name).write_bytes(b)
    manifest["toy_t1"] = {"config": "L=4,E=8,K=2,d=256,alpha=0.1,skew=1,seed=42,T=64",
                          "sha256": {k: sha(v) for k, v in files.items()}, "metrics": digests,
                          "speculation_precision": speculation_metrics(spec).precision}


def toy_t1_1024(manifest):
    cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, skew=1.0,
                         seed=42, tokens=1024)
    act, spec = run_model(cfg)
    logs = {}
    for pol in ("lru", "lfu", "lfu-aged:0.5:16", "opt"):
        for C in (2, 4, 6):
            log = simulate(act, SimConfig(policy=PolicyKind.parse(pol), cache_size=C))
            m = cache_metrics(log)
            logs[f"{pol}_c{C}"] = {"sha256": sha(log_bytes(log)), "hits": m.total_hits,
                                   "hit_rate": m.hit_rate}
    np.savez_compressed(OUT / "toy_t1_1024.npz", acts=act.activations, guessed=spec.guessed,
                        actual=spec.actual)
    manifest["toy_t1_1024"] = {"activation_sha256": sha(trace_bytes(act)),
                               "speculation_sha256": sha(trace_bytes(spec)), "event_logs": logs,
                               "speculation_precision": speculation_metrics(spec).precision}


SMALL = [  # (L, E, K, d, alpha, skew, seed, T)
    (2, 4, 2, 4, 0.1, 1.0, 7, 6),
    (4, 8, 2, 16, 0.1, 1.0, 42, 64),
    (5, 8, 2, 16, 0.0, 1.0, 1, 24),
    (6, 8, 2, 16, 0.5, 1.0, 3, 32),
    (3, 8, 3, 12, 0.2, 0.0, 9, 20),
    (1, 8, 2, 16, 0.1, 1.0, 5, 5),
    (3, 6, 1, 10, 0.3, 2.0, 11, 17),
]


def toy_small(manifest):
    out = {}
    for i, (L, E, K, d, a, s, seed, T) in enumerate(SMALL):
        act, spec = run_model(ToyModelConfig(ModelShape(L, E, K), hidden_dim=d, mixing_scale=a,
                                             skew=s, seed=seed, tokens=T))
        out[f"acts_{i}"] = act.activations
        out[f"guessed_{i}"] = spec.guessed
        out[f"actual_{i}"] = spec.actual
    np.savez_compressed(OUT / "toy_small.npz", configs=np.array(SMALL, np.float64), **out)
    manifest["toy_small.npz"] = {"configs": SMALL}


def forward_cases(manifest):
    rng = np.random.default_rng(77)
    rows = {}
    for i in range(6):
        L, E, K, d = 3, int(rng.integers(4, 9)), 2, int(rng.integers(4, 24))
        cfg = ToyModelConfig(ModelShape(L, E, K), hidden_dim=d, mixing_scale=float(rng.uniform(0, 0.5)),
                             seed=int(rng.integers(0, 1000)))
        model, _ = ToyMoeModel.build(cfg)
        x = rng.standard_normal(d)
        l = int(rng.integers(0, L))
        h, sel = forward_token(model, HiddenState(x, -1), l)
        picks = gate_select(HiddenState(x, -1), model.gates[l], E)
        rows[f"cfg_{i}"] = np.array([L, E, K, d, cfg.mixing_scale, cfg.seed, l], np.float64)
        rows[f"x_{i}"] = x
        rows[f"h_{i}"] = h.values
        rows[f"sel_{i}"] = np.array(sorted(sel), np.int64)
        rows[f"gate_ids_{i}"] = np.array([e for e, _ in picks], np.int64)
        rows[f"gate_p_{i}"] = np.array([p for _, p in picks], np.float64)
    np.savez_compressed(OUT / "forward_cases.npz", **rows)
    manifest["forward_cases.npz"] = {"cases": 6}


# (kind, L, E, K, T, skew, per_layer_permutation, repeat_prob, seed)
TRACEGEN = [
    ("zipf", 4, 8, 2, 300, 1.0, True, 0.0, 0), ("zipf", 32, 8, 2, 200, 1.2, True, 0.0, 42),
    ("zipf", 3, 8, 2, 100, 0.0, True, 0.0, 1), ("zipf", 2, 16, 4, 150, 2.5, False, 0.0, 7),
    ("zipf", 2, 5, 5, 40, 1.0, True, 0.0, 3), ("zipf", 2, 8, 2, 0, 1.0, True, 0.0, 3),
    ("markov", 4, 8, 2, 300, 1.0, True, 0.3, 0), ("markov", 32, 8, 2, 200, 1.2, True, 0.6, 42),
    ("markov", 3, 8, 2, 100, 1.0, True, 1.0, 5), ("markov", 3, 8, 2, 100, 1.0, True, 0.0, 5),
    ("markov", 2, 16, 4, 120, 0.5, False, 0.45, 9), ("markov", 2, 6, 6, 30, 1.0, True, 0.5, 2),
]


def tracegen_cases(manifest):
    from moesim.tracegen import MarkovParams, ZipfParams, gen_markov, gen_zipf

    rows = {}
    for i, (kind, L, E, K, T, skew, perm, rp, seed) in enumerate(TRACEGEN):
        shape = ModelShape(L, E, K)
        zp = ZipfParams(shape, T, skew_exponent=skew, per_layer_permutation=perm, seed=seed)
        if kind == "zipf":
            tr = gen_zipf(zp)
        else:
            tr = gen_markov(MarkovParams(shape, T, repeat_prob=rp, base=zp, seed=seed))
        rows[f"acts_{i}"] = tr.activations
    np.savez_compressed(OUT / "tracegen.npz", **rows)
    manifest["tracegen.npz"] = {"cases": [list(c) for c in TRACEGEN]}


def main():
    manifest = {"numpy": np.__version__, "moesim": moesim.__version__, "backend": kernels.BACKEND}
    if sys.argv[1:] == ["--only", "tracegen"]:
        manifest = json.loads((OUT / "manifest.json").read_text())
        tracegen_cases(manifest)
        (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
        return
    policy_streams(manifest)
    toy_t1(manifest)
    toy_t1_1024(manifest)
    toy_small(manifest)
    forward_cases(manifest)
    tracegen_cases(manifest)
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    print(json.dumps({k: v for k, v in manifest.items() if k.startswith("toy_t1")}, indent=1))


if __name__ == "__main__":
    main()
