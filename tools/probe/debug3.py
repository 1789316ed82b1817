import sys, time, os, faulthandler
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine
from paper_2511_05814_b200.toymoe import ToyModelConfig, ToyMoeModel
from paper_2511_05814_b200.traces import ModelShape
from paper_2511_05814_b200.policies import PolicyKind
mode = sys.argv[1]
cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, seed=42, tokens=2)
model, rng = ToyMoeModel.build(cfg)
inputs = rng.standard_normal((2, 256))
ecfg = EngineConfig(num_layers=4, num_experts=8, top_k=2, hidden_dim=256, expert_kind="toy_tanh", cache_size=2, policy=PolicyKind.lru(), mixing_scale=0.1, max_tokens=2)
eng=OffloadEngine(ecfg)
eng.load_toy_model(model)
s = torch.cuda.Stream()
x=torch.tensor(inputs.astype(np.float32), device="cuda")
torch.cuda.synchronize()
t=time.time()
with torch.cuda.stream(s):
    y=eng.decode_device(x)
print("enqueued", flush=True)
if mode == "poll":
    while not s.query():
        time.sleep(0.001)
else:
    torch.cuda.synchronize()
print("done %.3fs" % (time.time()-t), flush=True)
eng.sync()
print(eng.records(0,2)["acts"].tolist(), flush=True)
eng.close()
