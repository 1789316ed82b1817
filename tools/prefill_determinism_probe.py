"""Is the configs[3] prefill deterministic at full scale?  The same 512 tokens prefilled three
times from a cold C=4 LRU cache (reset between), records and outputs compared; the hit counts
and H2D bytes per run, and the first differing (token, layer) if any.

python tools/prefill_determinism_probe.py [--layers 32] [--tokens 512]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id
    from paper_2511_05814_b200.policies import PolicyKind

    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--cache", type=int, default=6)
    a = ap.parse_args()
    cfg = EngineConfig.mixtral_8x7b(num_layers=a.layers, cache_size=a.cache, max_tokens=4096,
                                    prefetch="early", compress=1)
    eng = OffloadEngine(cfg)
    eng.init_random(42)
    X = torch.stack([hash_weights(42, tensor_id(5, 100000 + t), 1.0, cfg.hidden_dim, "f32")
                     for t in range(a.tokens)])
    runs = []
    for r in range(3):
        eng.set_mode(policy=PolicyKind.lru(), cache_size=4, prefetch="off")
        s0 = eng.stats()
        t0 = eng.tokens_done
        out = eng.prefill_device(X)
        torch.cuda.synchronize()
        eng.sync()
        s1 = eng.stats()
        rec = eng.records(t0, a.tokens)
        runs.append((rec, out.cpu().numpy(), s1["hits"] - s0["hits"], s1["h2d_bytes"] - s0["h2d_bytes"]))
        print(json.dumps({"run": r, "hits": runs[-1][2], "h2d_bytes": runs[-1][3]}), flush=True)
        if r == 0:   # a decode in between, as the bench's variants do
            eng.set_mode(policy=PolicyKind.lfu(), cache_size=a.cache, prefetch="early")
            eng.decode_device(X[:8])
            eng.sync()
    base = runs[0]
    for r, (rec, out, hits, nb) in enumerate(runs[1:], 1):
        same_acts = np.array_equal(rec["acts"], base[0]["acts"])
        same_rb = np.array_equal(rec["resident_before"], base[0]["resident_before"])
        diff = None
        if not same_acts:
            idx = np.argwhere((rec["acts"] != base[0]["acts"]).any(-1))
            diff = idx[0].tolist()
        print(json.dumps({"run": r, "acts_equal": same_acts, "rb_equal": same_rb,
                          "out_equal": bool(np.array_equal(out, base[1])),
                          "max_abs_out_diff": float(np.abs(out - base[1]).max()),
                          "first_diff_token_layer": diff}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
