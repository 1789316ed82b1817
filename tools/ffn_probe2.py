"""Live FFN launch spans with no copies in flight: cache 8 of 8 (after warm-up every step hits)."""
import os
import sys
from pathlib import Path

os.environ["MOE_PROF_DUMP"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = EngineConfig.mixtral_8x7b(num_layers=L, cache_size=8, max_tokens=256)
with OffloadEngine(cfg) as eng:
    eng.init_random(42)
    X = torch.stack([hash_weights(42, tensor_id(5, t), 1.0, 4096, "f32") for t in range(48)])
    eng.decode_device(X[:40])
    eng.sync()
    s0 = eng.stats()
    eng.profile(True)
    eng.kernel_times()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.decode_device(X[40:48])
    b.record()
    torch.cuda.synchronize()
    k = eng.kernel_times()
    s1 = eng.stats()
    print(f"ms/token {a.elapsed_time(b) / 8:.3f} misses {s1['misses'] - s0['misses']}", k, file=sys.stderr)
