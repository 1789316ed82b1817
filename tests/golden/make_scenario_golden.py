"""Run the reference's K7-pinning scenarios at the sizes their scenario files name and record
per-instance results, so the GPU replay is pinned at full scale on the B200
(tests/test_scenarios_gpu.py):

  05-policy-equivalence   500 random single-expert traces x {lru, lfu} x C in {1, 2, 3}:
                          simulate (the kernel) == policy_step replay; per instance: hits and a
                          digest of the event arrays
  06-opt-dominance        100 gen_zipf traces (E=8, K=2, T=64) x C in {2, 3, 4}: hits of opt,
                          lru, lfu per instance
  09-compulsory-miss      the same 100 traces x {lru, lfu, lfu-aged:0.5:16, opt} at C = E:
                          misses per instance (== distinct experts)

The recipes' own summary dicts (scenarios.py:201-303) are stored beside.  Runs only where
/root/reference exists (the build container); nothing is written there.

python tests/golden/make_scenario_golden.py  -> tests/golden/scenarios_full.npz
"""
import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "scenarios_full.npz"


def _params(name):
    out = {}
    for line in (REF / "scenarios" / name).read_text().splitlines():
        line = line.strip()
        if not line or line.startswith("#") or "=" not in line:
            continue
        k, v = (x.strip() for x in line.split("=", 1))
        out[k] = v
    return out


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF / "src"))
    from moesim import scenarios
    from moesim.metrics import cache_metrics
    from moesim.policies import PolicyKind
    from moesim.simulate import SimConfig, simulate
    from moesim.traces import ActivationTrace, ModelShape

    out = {}
    # 05: the recipe's trace stream restated (rng.integers, scenarios.py:201-226), per instance
    p5 = _params("05-policy-equivalence.scenario")
    summary5 = scenarios._recipe_policy_equivalence(p5)
    E, T, n = int(p5["experts"]), int(p5["tokens"]), int(p5["traces"])
    rng = np.random.default_rng(int(p5["seed"]))
    acts5, hits5, dig5 = [], [], []
    for _ in range(n):
        acts = rng.integers(0, E, size=(T, 1, 1)).astype(np.int64)
        acts5.append(acts[:, 0, :])
        tr = ActivationTrace(ModelShape(1, E, 1), acts)
        for pol in ("lru", "lfu"):
            for c in (1, 2, 3):
                log = simulate(tr, SimConfig(policy=PolicyKind.parse(pol), cache_size=c))
                hits5.append(cache_metrics(log).total_hits)
                dig5.append(hashlib.sha256(log.resident_before[0].tobytes()
                                           + log.evicted[0].tobytes()).hexdigest()[:16])
    out["pe_acts"] = np.stack(acts5)
    out["pe_hits"] = np.array(hits5, np.int64)
    out["pe_digest"] = np.array(dig5)
    # 06 / 09: gen_zipf traces (scenarios.py:107-124), per-instance counts
    p6 = _params("06-opt-dominance.scenario")
    summary6 = scenarios._recipe_opt_dominance(p6)
    traces = scenarios._random_traces(p6, default_count=100)
    out["zipf_acts"] = np.stack([t.activations for t in traces])        # (100, T, 1, K)
    sizes = [int(c) for c in p6["cache_sizes"].split(",")]
    hits6 = np.zeros((len(traces), len(sizes), 3), np.int64)
    for i, tr in enumerate(traces):
        for j, c in enumerate(sizes):
            for q, pol in enumerate(("opt", "lru", "lfu")):
                hits6[i, j, q] = cache_metrics(simulate(tr, SimConfig(PolicyKind.parse(pol), c))).total_hits
    out["od_hits"] = hits6
    p9 = _params("09-compulsory-miss-bound.scenario")
    summary9 = scenarios._recipe_compulsory_miss(p9)
    traces9 = scenarios._random_traces(p9, default_count=100)
    assert all(np.array_equal(a.activations, b.activations) for a, b in zip(traces, traces9))
    pols9 = p9["policies"].split(",")
    miss9 = np.zeros((len(traces9), len(pols9)), np.int64)
    for i, tr in enumerate(traces9):
        for q, pol in enumerate(pols9):
            log = simulate(tr, SimConfig(PolicyKind.parse(pol), tr.shape.num_experts))
            miss9[i, q] = int(log.miss_counts(0).sum())
    out["cm_misses"] = miss9
    out["meta"] = np.array(json.dumps({
        "05": {"params": p5, "summary": summary5}, "06": {"params": p6, "summary": summary6},
        "09": {"params": p9, "summary": summary9}, "policies_09": pols9, "cache_sizes_06": sizes}))
    np.savez_compressed(OUT, **out)
    print(json.dumps({"05": summary5, "06": summary6, "09": summary9}))


if __name__ == "__main__":
    main()
