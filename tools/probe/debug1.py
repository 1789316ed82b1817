import sys, time, math, os
t0=time.time()
import torch
print("import torch %.1fs" % (time.time()-t0), flush=True)
sys.path.insert(0, '.')
import numpy as np
import oracle
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id
std=float(np.float32(1/math.sqrt(1792)))
for tid in [tensor_id(4,0,0,3), tensor_id(4,0,0,1)]:
    n=1792*512
    dev=hash_weights(7,tid,std,n,"bf16").cpu().numpy().view(np.uint16)
    o=oracle.hash_fill(7,tid,std,n)
    bad=np.flatnonzero(dev!=o)
    print("isolated hash tid", tid, "mismatches", bad.size, bad[:10], dev[bad[:5]], o[bad[:5]], flush=True)
cfg=EngineConfig(num_layers=4,num_experts=8,top_k=2,hidden_dim=512,ffn_dim=1792,expert_kind="swiglu",max_tokens=16)
with OffloadEngine(cfg) as eng:
    eng.init_random(7)
    for (l,e) in [(0,0),(1,3)]:
        w1,w3,w2=eng.swiglu_weights(l,e)
        o=oracle.hash_fill(7,tensor_id(4,l,e,3),std,1792*512)
        bad=np.flatnonzero(w2.ravel()!=o)
        print("engine w2", l, e, "mismatches", bad.size, bad[:10], flush=True)
        o1=oracle.hash_fill(7,tensor_id(4,l,e,1),float(np.float32(1/math.sqrt(512))),1792*512)
        print("engine w1 mismatches", (w1.ravel()!=o1).sum(), flush=True)
print("now toy decode", flush=True)
os.environ["MOE_DEBUG"]="1"
from paper_2511_05814_b200.toymoe import ToyModelConfig, ToyMoeModel
from paper_2511_05814_b200.traces import ModelShape
from paper_2511_05814_b200.policies import PolicyKind
cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, seed=42, tokens=2)
model, rng = ToyMoeModel.build(cfg)
inputs = rng.standard_normal((2, 256))
ecfg = EngineConfig(num_layers=4, num_experts=8, top_k=2, hidden_dim=256, expert_kind="toy_tanh", cache_size=2, policy=PolicyKind.lru(), mixing_scale=0.1, max_tokens=2)
t=time.time()
eng=OffloadEngine(ecfg)
print("create %.2fs"%(time.time()-t), flush=True)
eng.load_toy_model(model)
print("loaded", flush=True)
x=torch.tensor(inputs.astype(np.float32), device="cuda")
y=eng.decode_device(x)
print("enqueued", flush=True)
torch.cuda.synchronize()
print("synced", y[:, :4], flush=True)
print(eng.records(0,2)["acts"])
eng.close()
