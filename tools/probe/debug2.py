import sys, time, math, os, faulthandler
faulthandler.dump_traceback_later(80, exit=True)
sys.path.insert(0, '.')
import numpy as np, torch
import oracle
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, tensor_id
part = sys.argv[1]
if part == "weights":
    cfg=EngineConfig(num_layers=4,num_experts=8,top_k=2,hidden_dim=512,ffn_dim=1792,expert_kind="swiglu",max_tokens=16)
    sd=float(np.float32(1/math.sqrt(512))); sf=float(np.float32(1/math.sqrt(1792)))
    for rep in range(3):
        with OffloadEngine(cfg) as eng:
            eng.init_random(7)
            bad=0
            for l in range(4):
                for e in range(8):
                    w1,w3,w2=eng.swiglu_weights(l,e)
                    for w,m,sd_ in ((w1,1,sd),(w3,2,sd),(w2,3,sf)):
                        o=oracle.hash_fill(7,tensor_id(4,l,e,m),sd_,1792*512)
                        nb=int((w.ravel()!=o).sum())
                        if nb: print("mismatch", l, e, m, nb, np.flatnonzero(w.ravel()!=o)[:5], flush=True)
                        bad+=nb
            print(os.environ.get("MOE_PIN_MODE","register"), "rep", rep, "total mismatches", bad, flush=True)
else:
    os.environ["MOE_DEBUG"]="1"
    from paper_2511_05814_b200.toymoe import ToyModelConfig, ToyMoeModel
    from paper_2511_05814_b200.traces import ModelShape
    from paper_2511_05814_b200.policies import PolicyKind
    cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, seed=42, tokens=2)
    model, rng = ToyMoeModel.build(cfg)
    inputs = rng.standard_normal((2, 256))
    ecfg = EngineConfig(num_layers=4, num_experts=8, top_k=2, hidden_dim=256, expert_kind="toy_tanh", cache_size=2, policy=PolicyKind.lru(), mixing_scale=0.1, max_tokens=2)
    eng=OffloadEngine(ecfg)
    eng.load_toy_model(model)
    s = torch.cuda.Stream() if part == "stream" else None
    x=torch.tensor(inputs.astype(np.float32), device="cuda")
    torch.cuda.synchronize()
    if s is not None:
        with torch.cuda.stream(s):
            y=eng.decode_device(x)
    else:
        y=eng.decode_device(x)
    print("enqueued", flush=True)
    torch.cuda.synchronize()
    print("synced", y[:, :4], flush=True)
    print(eng.records(0,2)["acts"])
    eng.close()
