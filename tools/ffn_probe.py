"""Per-launch decode FFN timings (MOE_PROF_DUMP): live launches vs the isolated microbench."""
import os
import sys
from pathlib import Path

os.environ["MOE_PROF_DUMP"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = EngineConfig.mixtral_8x7b(num_layers=L, cache_size=4, max_tokens=256)
with OffloadEngine(cfg) as eng:
    eng.init_random(42)
    X = torch.stack([hash_weights(42, tensor_id(5, t), 1.0, 4096, "f32") for t in range(12)])
    eng.decode_device(X[:4])
    eng.sync()
    eng.profile(True)
    eng.kernel_times()
    eng.decode_device(X[4:12])
    print(eng.kernel_times(), file=sys.stderr)
