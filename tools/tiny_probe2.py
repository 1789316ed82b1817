"""Where does a configs[0] tiny token go?  The same 256 tokens through the engine at cache size 2
(the config), 8 (every expert resident after warm-up: the compute-only floor) and with the
copy-engine transfer instead of SM zero-copy fetches; us/token and H2D bytes/token each.

python tools/tiny_probe2.py
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine
    from paper_2511_05814_b200.policies import PolicyKind
    from paper_2511_05814_b200.toymoe import ToyModelConfig, ToyMoeModel
    from paper_2511_05814_b200.traces import ModelShape

    T = 256
    cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, seed=42, tokens=T)
    model, rng = ToyMoeModel.build(cfg)
    x = torch.from_numpy(rng.standard_normal((T, 256)).astype(np.float32)).cuda()
    s = torch.cuda.current_stream()
    for transfer, C in (("auto", 2), ("auto", 8), ("copy_engine", 2), ("copy_engine", 8)):
        ecfg = EngineConfig(num_layers=4, num_experts=8, top_k=2, hidden_dim=256,
                            expert_kind="toy_tanh", cache_size=C, policy=PolicyKind.lru(),
                            mixing_scale=0.1, max_tokens=T + 64, transfer=transfer)
        with OffloadEngine(ecfg) as eng:
            eng.load_toy_model(model)
            eng.decode_device(x[:64])   # warm-up (C=8: all experts resident from here on)
            eng.sync()
            st0 = eng.stats()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.record(s)
            eng.decode_device(x)
            b.record(s)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            eng.sync()
            st1 = eng.stats()
            ms = a.elapsed_time(b)
            print(json.dumps({"transfer": transfer, "cache_size": C, "us_per_token": ms * 1e3 / T,
                              "wall_us_per_token": wall * 1e6 / T,
                              "misses_per_token": (st1["misses"] - st0["misses"]) / T,
                              "h2d_bytes_per_token": (st1["h2d_bytes"] - st0["h2d_bytes"]) / T,
                              "fetched_bytes_per_token": (st1.get("fetched_bytes", 0)
                                                          - st0.get("fetched_bytes", 0)) / T}),
                  flush=True)


if __name__ == "__main__":
    main()
