"""Full-depth parity at the benchmarked shapes, against the fp64 oracle.

configs[1]: Mixtral-8x7B shape, all 32 layers, the bench's cache size (4) under LRU and LFU.
configs[4]: Mixtral-8x22B shape (d=6144, f=16384) with the bench's 8x22B engine options
(coded-only store, LFU + early prefetch with one staging buffer per layer), 4 layers.

The oracle is oracle.decode_layerwise: MixtralRef's fp64 arithmetic in the reference's `h @ W`
layout (toymoe.py:138-146 with the SwiGLU body) evaluated layer-major so one layer of fp64
experts is alive at a time.  Bar (north star):
  * expert selections bit-exact wherever the oracle's k-th/(k+1)-th logit gap is >= 1e-3
    (toymoe.py:114 ordering); below that the tie is stated (counted) and teacher-forced;
  * the live cache trace (resident_before / evicted) bit-exact against the C oracle replay
    of the selections (kernels.py:60-147), per policy;
  * layer outputs within 1e-2 relative (bf16 weights, fp32 activations vs fp64);
  * reference-definition guesses equal wherever their gap is >= 1e-3;
  * demand bytes == misses x expert bytes with prefetch off (costmodel.py:90-111).
Set MOEB200_PARITY_OUT=<file> to append each case's tie / error summary as one JSON line.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.model import replay_layers
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine
from paper_2511_05814_b200.policies import PolicyKind

pytestmark = pytest.mark.gpu

TIE_TOL = 1e-3


def _run_engine(cfg, seed, X, modes):
    T = X.shape[0]
    runs = []
    with OffloadEngine(cfg) as eng:
        eng.init_random(seed)
        for pol, pf in modes:
            eng.set_mode(policy=pol, cache_size=cfg.cache_size, prefetch=pf)
            t0 = eng.tokens_done
            s0 = eng.stats()
            out = eng.decode(X)
            s1 = eng.stats()
            runs.append({"mode": (str(pol), pf), "out": out, "rec": eng.records(t0, T),
                         "gaps": eng.record_gaps(t0, T),
                         "early": eng.record_early_guesses(t0, T),
                         "stats": {k: s1[k] - s0[k] for k in s1 if isinstance(s1[k], int)}})
    return runs


def _check(name, cfg, seed, T, modes):
    X = oracle.MixtralRef.inputs(seed, T, cfg.hidden_dim)
    runs = _run_engine(cfg, seed, X, modes)
    first = runs[0]
    # routing does not depend on the cache: every mode decodes identically
    for r in runs[1:]:
        assert np.array_equal(r["out"], first["out"]), r["mode"]
        for k in ("acts", "guessed", "probs"):
            assert np.array_equal(r["rec"][k], first["rec"][k]), (r["mode"], k)
    ref = oracle.MixtralRef(cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden_dim,
                            cfg.ffn_dim, cfg.mixing_scale, seed=seed, layout="ref",
                            renormalize=cfg.renormalize, rms_norm=cfg.rms_norm,
                            rms_eps=cfg.rms_eps, store_layers=cfg.store_layers)
    lw = oracle.decode_layerwise(ref, X, forced=first["rec"]["acts"], tol=TIE_TOL)
    acts = first["rec"]["acts"]
    # selections: equal everywhere once the stated near-ties are forced; each forced step
    # had an oracle gap below the tolerance (decode_layerwise never forces above it)
    assert np.array_equal(lw["acts"], acts), np.argwhere((lw["acts"] != acts).any(-1))[:8]
    assert all(g < TIE_TOL for _, _, g in lw["forced_ties"])
    # the engine's own margins agree with the oracle's (fp32 logits vs fp64)
    fin = np.isfinite(lw["gaps"])
    assert np.abs(first["gaps"][fin] - lw["gaps"][fin]).max() < 1e-3
    near = int((lw["gaps"] < TIE_TOL).sum())
    # reference-definition guesses where the guess is not itself a near-tie
    gsafe = lw["guess_gaps"] >= TIE_TOL
    assert np.array_equal(first["rec"]["guessed"][gsafe], lw["guessed"][gsafe])
    # outputs
    rel = float(np.abs(first["out"] - lw["outs"]).max() / np.abs(lw["outs"]).max())
    assert rel < 1e-2, rel
    # live cache traces == the C oracle's replay of the same selections, per policy
    for r in runs:
        pol = PolicyKind.parse(r["mode"][0])
        rb, ev = replay_layers(acts, cfg.num_experts, cfg.cache_size, *pol.device_params())
        assert np.array_equal(r["rec"]["resident_before"], np.transpose(rb, (1, 0, 2))), r["mode"]
        assert np.array_equal(r["rec"]["evicted"], np.transpose(ev, (1, 0, 2))), r["mode"]
        hits = int(sum(rb[l, t, acts[t, l]].sum() for t in range(T) for l in range(cfg.num_layers)))
        assert r["stats"]["hits"] == hits and r["stats"]["misses"] == T * cfg.num_layers * cfg.top_k - hits
        if r["mode"][1] == "off":
            assert r["stats"]["demand_bytes"] == r["stats"]["misses"] * cfg.expert_bytes
        else:   # the prefetch decisions against the restated rule
            nb = cfg.cache_size + (cfg.prefetch_buffers or cfg.top_k)
            issued, used = oracle.prefetch_oracle(acts, r["early"], r["rec"]["resident_before"], nb)
            assert r["stats"]["prefetch_issued"] == int(issued.sum())
            assert r["stats"]["prefetch_used"] == int(used.sum())
            assert r["stats"]["h2d_bytes"] == r["stats"]["demand_link_bytes"] + r["stats"]["prefetch_bytes"]
    summary = {"case": name, "tokens": T, "layers": cfg.num_layers, "steps": T * cfg.num_layers,
               "modes": [list(r["mode"]) for r in runs],
               "near_ties_lt_1e-3": near, "forced_ties": len(lw["forced_ties"]),
               "min_topk_gap": float(lw["gaps"].min()), "max_rel_err": rel,
               "max_gap_abs_diff": float(np.abs(first["gaps"][fin] - lw["gaps"][fin]).max()),
               "guess_near_ties_lt_1e-3": int((~gsafe).sum())}
    print(json.dumps(summary))
    if os.environ.get("MOEB200_PARITY_OUT"):
        with open(os.environ["MOEB200_PARITY_OUT"], "a") as fh:
            fh.write(json.dumps(summary) + "\n")


def test_configs1_full_depth_vs_fp64_oracle():
    """All 32 layers of the Mixtral-8x7B shape, 12 tokens, C = 4, LRU and LFU, coded transfers."""
    cfg = EngineConfig.mixtral_8x7b(cache_size=4, compress=2, max_tokens=64)
    _check("configs[1] mixtral_8x7b L=32 C=4", cfg, 42, 12,
           [(PolicyKind.lru(), "off"), (PolicyKind.lfu(), "off")])


def test_configs4_shape_vs_fp64_oracle():
    """The 8x22B shape (its own stream-geometry branches: d=6144, f=16384) on 4 layers with the
    bench's 8x22B options: coded-only store, LFU + early prefetch, one staging buffer."""
    cfg = EngineConfig.mixtral_8x22b(num_layers=4, cache_size=4, compress=2, max_tokens=64,
                                     prefetch="early", prefetch_buffers=1,
                                     policy=PolicyKind.lfu())
    _check("configs[4] mixtral_8x22b L=4 C=4", cfg, 43, 16,
           [(PolicyKind.lfu(), "early"), (PolicyKind.lfu(), "off"), (PolicyKind.lru(), "off")])
