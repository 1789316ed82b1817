"""The reference's K7-pinning scenarios at the sizes their scenario files name,
on the GPU paths of this package, against per-instance results recorded from the reference
(tests/golden/make_scenario_golden.py; scenarios.py:201-303):

  05-policy-equivalence  500 traces x {lru, lfu} x C in {1,2,3} = 3000 instances: simulate
                         (the batched GPU replay) agrees with a policy_step replay (the GPU
                         per-step API) step for step; hits and event arrays == the reference's
  06-opt-dominance       100 gen_zipf traces (GPU sampler) x C in {2,3,4}: opt / lru / lfu hit
                         counts == the reference's, opt never below lru / lfu
  09-compulsory-miss     the same traces x 4 policies at C = E: misses == distinct experts
"""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2511_05814_b200.metrics import cache_metrics
from paper_2511_05814_b200.policies import PolicyKind, policy_step, warm_state
from paper_2511_05814_b200.simulate import SimConfig, simulate
from paper_2511_05814_b200.tracegen import ZipfParams, gen_zipf
from paper_2511_05814_b200.traces import ActivationTrace, ModelShape

pytestmark = pytest.mark.gpu

G = np.load(GOLDEN / "scenarios_full.npz")
META = json.loads(str(G["meta"]))


def test_scenario_05_policy_equivalence_full_scale():
    p = META["05"]["params"]
    E = int(p["experts"])
    acts_all = G["pe_acts"]
    assert acts_all.shape[0] == int(p["traces"]) == 500
    instances = mismatches = 0
    hits, digests = [], []
    for acts in acts_all:
        tr = ActivationTrace(ModelShape(1, E, 1), acts[:, None, :])
        for pol in ("lru", "lfu"):
            kind = PolicyKind.parse(pol)
            for c in (1, 2, 3):
                log = simulate(tr, SimConfig(policy=kind, cache_size=c))
                hits.append(cache_metrics(log).total_hits)
                digests.append(hashlib.sha256(log.resident_before[0].tobytes()
                                              + log.evicted[0].tobytes()).hexdigest()[:16])
                state = warm_state(kind, c)
                ok = True
                for step in log.steps():
                    state, outcome = policy_step(state, kind, set(tr.activations[step.token, 0].tolist()))
                    if outcome != step.outcome:
                        ok = False
                        break
                instances += 1
                mismatches += 0 if ok else 1
    assert {"instances": instances, "mismatches": mismatches} == META["05"]["summary"]
    assert np.array_equal(np.array(hits), G["pe_hits"])
    assert list(digests) == list(G["pe_digest"])


def _zipf_traces(p):
    skews = [float(s) for s in p.get("skews", "0,0.5,1.0").split(",")]
    shape = ModelShape(1, int(p["experts"]), int(p["top_k"]))
    return [gen_zipf(ZipfParams(shape=shape, num_tokens=int(p["tokens"]),
                                skew_exponent=skews[i % len(skews)], seed=int(p["seed"]) + i))
            for i in range(int(p["traces"]))]


def test_scenario_06_opt_dominance_full_scale():
    p = META["06"]["params"]
    traces = _zipf_traces(p)
    assert np.array_equal(np.stack([t.activations for t in traces]), G["zipf_acts"])
    sizes = META["cache_sizes_06"]
    hits = np.zeros((len(traces), len(sizes), 3), np.int64)
    violations = 0
    for i, tr in enumerate(traces):
        for j, c in enumerate(sizes):
            for q, pol in enumerate(("opt", "lru", "lfu")):
                hits[i, j, q] = cache_metrics(simulate(tr, SimConfig(PolicyKind.parse(pol), c))).total_hits
            violations += int(hits[i, j, 0] < hits[i, j, 1] or hits[i, j, 0] < hits[i, j, 2])
    assert np.array_equal(hits, G["od_hits"])
    assert {"instances": len(traces) * len(sizes), "violations": violations} == META["06"]["summary"]


def test_scenario_09_compulsory_miss_bound_full_scale():
    p = META["09"]["params"]
    traces = _zipf_traces(p)
    pols = META["policies_09"]
    misses = np.zeros((len(traces), len(pols)), np.int64)
    violations = 0
    for i, tr in enumerate(traces):
        E = tr.shape.num_experts
        for q, pol in enumerate(pols):
            log = simulate(tr, SimConfig(PolicyKind.parse(pol), E))
            misses[i, q] = int(log.miss_counts(0).sum())
            violations += int(misses[i, q] != len(np.unique(tr.activations[:, 0, :])))
    assert np.array_equal(misses, G["cm_misses"])
    assert {"instances": len(traces) * len(pols), "violations": violations} == META["09"]["summary"]
