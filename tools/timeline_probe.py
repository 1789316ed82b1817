"""Where does the link idle in the copy-engine decode?  Runs the configs[1] decode (C=4, 16
tokens after 4 warm-up) with MOE_TIMELINE set (per-step copy-stream / compute-stream events,
csrc/engine.cu) and attributes every gap between consecutive demand-copy spans to
  post   last landing of the previous demand step -> that layer's FFN done (decode + down)
  hits   whole layers in between whose experts all hit (no copies)
  route  previous layer done -> this step's gate done (mix + gate)
  issue  gate done -> this step's first copy starts (mailbox, host forwarder, copy launch)

python tools/timeline_probe.py [--compress 0|1] [--policy lru|lfu] [--prefetch]
"""
import argparse
import csv
import json
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def analyse(path, tokens, layers):
    rows = [r for r in csv.DictReader(open(path))]
    rows = [{k: float(v) for k, v in r.items()} for r in rows]
    rows = rows[-tokens * layers:]            # the timed tokens
    t0 = rows[0]["gate_end_ms"]
    busy = sum(r["copy_end_ms"] - r["copy_start_ms"] for r in rows if r["n_demand"] > 0)
    total = rows[-1]["layer_done_ms"] - t0
    acc = {"post": 0.0, "hits": 0.0, "route": 0.0, "issue": 0.0}
    prev = None
    for i, r in enumerate(rows):
        if r["n_demand"] == 0:
            continue
        if prev is not None:
            p = rows[prev]
            acc["post"] += max(0.0, p["layer_done_ms"] - p["copy_end_ms"])
            acc["hits"] += max(0.0, rows[i - 1]["layer_done_ms"] - p["layer_done_ms"])
            acc["route"] += max(0.0, r["gate_end_ms"] - rows[i - 1]["layer_done_ms"])
            acc["issue"] += max(0.0, r["copy_start_ms"] - max(r["gate_end_ms"], p["copy_end_ms"]))
        prev = i
    host = sorted(r["host_issue_us"] for r in rows if r["n_demand"] > 0)
    steps = sum(1 for r in rows if r["n_demand"] > 0)
    return {"ms_total": total, "ms_link_busy": busy, "link_busy_frac": busy / total,
            "gap_ms_per_token": {k: v / tokens for k, v in acc.items()},
            "gap_us_per_demand_step": {k: v * 1e3 / max(1, steps) for k, v in acc.items()},
            "host_handle_mail_us_median": host[len(host) // 2] if host else None,
            "demand_steps": steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--compress", type=int, default=1)
    ap.add_argument("--policy", default="lru")
    ap.add_argument("--prefetch", action="store_true")
    ap.add_argument("--tokens", type=int, default=16)
    a = ap.parse_args()
    path = os.path.join(tempfile.mkdtemp(), "timeline.csv")
    os.environ["MOE_TIMELINE"] = path
    import torch

    from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id
    from paper_2511_05814_b200.policies import PolicyKind

    cfg = EngineConfig.mixtral_8x7b(cache_size=4, max_tokens=256, compress=a.compress,
                                    prefetch="early" if a.prefetch else "off")
    eng = OffloadEngine(cfg)
    eng.init_random(42)
    eng.set_mode(policy=PolicyKind.lfu() if a.policy == "lfu" else PolicyKind.lru(), cache_size=4,
                 prefetch="early" if a.prefetch else "off")
    x = torch.stack([hash_weights(42, tensor_id(5, t), 1.0, cfg.hidden_dim, "f32")
                     for t in range(4 + a.tokens)])
    eng.decode_device(x[:4])
    eng.sync()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.decode_device(x[4:])
    e1.record(s)
    torch.cuda.synchronize()
    eng.sync()
    ms = e0.elapsed_time(e1)
    eng.close()
    out = analyse(path, a.tokens, cfg.num_layers)
    out.update({"compress": a.compress, "policy": a.policy, "prefetch": a.prefetch,
                "tokens_per_s": a.tokens / (ms / 1e3)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
