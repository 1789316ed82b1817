"""Do the bench's per-launch CUDA events (engine.profile) slow the copy-engine decode itself?

Same engine, same 16 tokens after a reset (identical cache traces, identical copies), timed with
one event pair around the whole decode; alternately with per-launch kernel events on and off.

python tools/profile_overhead_probe.py [--layers 32] [--policy lru] [--reps 2]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id
    from paper_2511_05814_b200.policies import PolicyKind

    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--policy", default="lru")
    ap.add_argument("--prefetch", action="store_true")
    ap.add_argument("--tokens", type=int, default=16)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    cfg = EngineConfig.mixtral_8x7b(num_layers=a.layers, cache_size=4, max_tokens=256,
                                    prefetch="early" if a.prefetch else "off", compress=1)
    eng = OffloadEngine(cfg)
    eng.init_random(42)
    pol = PolicyKind.lfu() if a.policy == "lfu" else PolicyKind.lru()
    eng.set_mode(policy=pol, cache_size=4, prefetch="early" if a.prefetch else "off")
    D = cfg.hidden_dim
    x = torch.stack([hash_weights(42, tensor_id(5, t), 1.0, D, "f32") for t in range(4 + a.tokens)])
    s = torch.cuda.current_stream()
    out = []
    for rep in range(a.reps):
        for prof in (True, False):
            eng.reset()
            eng.decode_device(x[:4])
            eng.sync()
            eng.profile(prof)
            st0 = eng.stats()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            eng.decode_device(x[4:])
            e1.record(s)
            torch.cuda.synchronize()
            eng.sync()
            eng.profile(False)
            st1 = eng.stats()
            ms = e0.elapsed_time(e1)
            rec = {"rep": rep, "kernel_events": prof, "ms_per_token": ms / a.tokens,
                   "tokens_per_s": a.tokens / (ms / 1e3),
                   "misses": st1["misses"] - st0["misses"],
                   "h2d_GBps": (st1["h2d_bytes"] - st0["h2d_bytes"]) / (ms / 1e3) / 1e9}
            out.append(rec)
            print(json.dumps(rec), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
