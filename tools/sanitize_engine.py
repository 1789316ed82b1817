"""Engine workloads small enough for compute-sanitizer (racecheck / synccheck / memcheck).

Each case builds a small Mixtral-shaped engine, runs a few decode (or prefill) tokens through
every kernel family the live engine launches -- fused mix+gate (`gate_cache_kernel` partials),
`stream_gemv_kernel` up/down, the exponent decoder, the SM-transfer fetch kernel, the prefetch
planner, the PDL token graph, `pf_plan_kernel` + the tcgen05 grouped GEMM for prefill -- and
checks the trace against the oracle replay, so a sanitizer run also proves the kernels still
compute the right thing under instrumentation.

    compute-sanitizer --tool racecheck python tools/sanitize_engine.py [case ...]
"""
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import oracle  # noqa: E402  (test infrastructure: the checker)
from oracle.model import replay_layers  # noqa: E402
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine  # noqa: E402
from paper_2511_05814_b200.policies import PolicyKind  # noqa: E402

SMALL = dict(num_layers=3, num_experts=8, top_k=2, hidden_dim=512, ffn_dim=1792,
             expert_kind="swiglu", mixing_scale=0.1 * math.sqrt(16 / 512), max_tokens=64,
             rms_norm=True)

CASES = {
    "lru_copy": dict(policy=PolicyKind.lru(), transfer="copy_engine"),
    "lfu_sm": dict(policy=PolicyKind.lfu(), transfer="sm"),
    "lfu_prefetch": dict(policy=PolicyKind.lfu(), prefetch="early", transfer="copy_engine"),
    "coded": dict(policy=PolicyKind.lru(), compress=2, transfer="copy_engine"),
    "coded_prefetch": dict(policy=PolicyKind.lfu(), compress=1, prefetch="early"),
    "prefill": dict(policy=PolicyKind.lru(), transfer="copy_engine"),
}


def run(name: str, T: int = 6) -> None:
    kw = dict(SMALL)
    kw.update(CASES[name])
    cfg = EngineConfig(**kw)
    X = oracle.MixtralRef.inputs(5, T, cfg.hidden_dim)
    t0 = time.time()
    with OffloadEngine(cfg) as eng:
        eng.init_random(5)
        if name == "prefill":
            eng.prefill(X)
        else:
            eng.decode(X[: T // 2])
            eng.decode(X[T // 2:])   # second call: the token graph path (warm)
        rec = eng.records(0, T)
    code, df, dp = cfg.policy.device_params()
    rb, ev = replay_layers(rec["acts"], cfg.num_experts, cfg.cache_size, code, df, dp)
    ok = (np.array_equal(rec["resident_before"], rb.transpose(1, 0, 2))
          and np.array_equal(rec["evicted"], ev.transpose(1, 0, 2)))
    print(f"case {name}: {T} tokens, trace == oracle replay: {ok}, {time.time() - t0:.1f} s",
          flush=True)
    assert ok, name


if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        run(c)
    print("sanitize_engine: all cases done")
