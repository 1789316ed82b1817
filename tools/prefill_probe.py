"""Prefill probe (configs[3] shape on a reduced layer count): cold prefill of T tokens, then
per-kernel-class times.  Used under ncu for the launch list / full captures of K4."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layers", type=int, default=2)
p.add_argument("--tokens", type=int, default=512)
p.add_argument("--cache-size", type=int, default=4)
p.add_argument("--repeat", type=int, default=2)
a = p.parse_args()
cfg = EngineConfig.mixtral_8x7b(num_layers=a.layers, cache_size=a.cache_size, max_tokens=4096)
with OffloadEngine(cfg) as eng:
    eng.init_random(42)
    X = torch.stack([hash_weights(42, tensor_id(5, t), 1.0, 4096, "f32") for t in range(a.tokens)])
    for r in range(a.repeat):
        eng.profile(True)
        k0 = eng.kernel_times()
        s0 = eng.stats()
        eng.prefill_device(X)
        eng.sync()
        k1 = eng.kernel_times()
        s1 = eng.stats()
        eng.profile(False)
        k = {n: k1[n] - k0[n] for n in k1}
        gb = (s1["prefill_bytes"] - s0["prefill_bytes"]) / 1e9
        print(f"prefill #{r}: {k['prefill_ms']:.2f} ms total, GEMM {k['gemm_launches']} launches "
              f"{k['gemm_ms']:.3f} ms = {k['gemm_flops'] / k['gemm_ms'] / 1e9:.0f} TFLOP/s, "
              f"{k['gemm_bytes'] / k['gemm_ms'] / 1e6:.0f} GB/s algorithmic; H2D {gb:.2f} GB "
              f"= {gb / (k['prefill_ms'] / 1e3):.1f} GB/s")
