#!/usr/bin/env python
"""Decode bench for the MoE-offloading engine (BASELINE.json metric).

metric   decode tokens/s per GPU and cache hit rate (LRU vs LFU vs prefetch) at cache size k
workload configs[1]: Mixtral-8x7B-shaped bf16 (L=32, E=8, K=2, d=4096, f=14336) with
         random-init (counter-hash) weights, batch-1 decode, per-layer HBM cache of 4 experts,
         experts streamed from pinned host DRAM.  One step = one decode token through all 32
         layers.  The headline `value` is LRU at C=4; LFU and LFU+prefetch run on the same
         engine (cold caches each) and are reported under "variants".
timing   W untimed warm-up tokens, then K tokens bracketed by barrier + synchronize, CUDA
         events on the compute stream, max over ranks.  Every step streams >= 23.6 GB of
         weights (mixing + 2 experts x 32 layers) through HBM, far above the 126 MB L2.
e2e      the same decode through the public API (OffloadEngine.decode on a host array):
         H2D of the token's input and D2H of its output inside the timed region; the timed
         tokens replayed from the same cold + warm-up cache state (identical misses).
reference arm (--impl reference): the oracle port of the reference path (numpy fp64 in the
         reference's `h @ W` layout, all host threads) on the same config and token stream:
         32 tokens through the first 8 of the 32 layers (every layer does identical work),
         best of 3, per-token time scaled by L / 8 (`layers_sampled`, `scale` say so).

Run: python bench.py [--gpus N --steps K --warmup W]; multi-GPU via torch.distributed.run
(independent request streams, one engine per GPU, no collective on the hot path).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode tokens/s per GPU and cache hit rate (LRU vs LFU vs prefetch) at cache size k"
L, E, K, D, F = 32, 8, 2, 4096, 14336
EXPERT_BYTES = 3 * F * D * 2                       # 352,321,536
HBM_BYTES_PER_TOKEN = L * (2 * D * D + 2 * D * E + K * 3 * D * F * 2)  # 23,624,417,792
# (L, E, K, d, f) of the two benchmarked shapes (BASELINE.json configs[1] / [4])
MODELS = {"mixtral_8x7b": (32, 8, 2, 4096, 14336), "mixtral_8x22b": (56, 8, 2, 6144, 16384)}
TIE_TOL = 1e-3   # top-k logit margin below which a selection is a stated near-tie (north star)


def workload_config(model: str, world: int, cache_size: int, policy: str) -> dict:
    """The workload both arms run, key for key (only the line's impl / dtype differ).  The
    synthetic model's departures from SURVEY 8d's literal recipe are part of the workload."""
    Lm, Em, Km, Dm, Fm = MODELS[model]
    hbm = Lm * (2 * Dm * Dm + 2 * Dm * Em + Km * 3 * Dm * Fm * 2)
    return {
        "workload": f"{'configs[4]' if model == 'mixtral_8x22b' else 'configs[1]'}: {model}-shaped "
                    f"batch-1 decode, {policy} cache {cache_size}/layer, experts in host DRAM",
        "model": f"{model}-shape (L={Lm},E={Em},K={Km},d={Dm},f={Fm}), random-init",
        "global_batch": world, "seq_len": 1, "parallelism": f"replicas x{world}",
        "cache_size": cache_size, "policy": policy,
        "l2": f"inputs larger than L2: each step streams >= {hbm / 1e9:.1f} GB of weights "
              "(mixing + 2 experts per layer) through HBM",
        "tokens": "counter-hash N(0,1)-shaped f32 inputs, one independent token per step",
        "synthetic_model": {
            "weights": "counter-hash Irwin-Hall (sum of 4 uniforms, bell-shaped) bf16, std as SURVEY 8d",
            "gate_bias_std": "0.25 (SURVEY 8d: 1.0 -- bias-dominated routing under RMSNorm, DESIGN 5)",
            "rms_norm": "unit-scale RMSNorm (eps 1e-5) before gate and experts (not in toymoe; "
                        "a 32-layer SwiGLU residual overflows without it, DESIGN 5)",
            "routing": "softmax over E, top-k by logit (ties to the lower id), unrenormalised "
                       "(toymoe.py:93-115)",
            "host_store": ("one node-shared pinned copy per node, page-locked by every replica"
                           if world > 1 else "one pinned host copy for the GPU"),
        },
    }


def fp64_layer_bytes(shape) -> int:
    _, Em, _, Dm, Fm = shape
    return Em * 3 * Dm * Fm * 8 + Dm * Dm * 8 + 2 * Em * Dm * 8


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=16)
    p.add_argument("--warmup", type=int, default=4)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--cache-size", type=int, default=4)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--variants", default=None,
                   help="headline = the first; policy[+prefetch][@cache_size]. Default: configs[1] "
                        "and [2] (LRU, LFU, LFU+prefetch, LRU+prefetch at C=4; LFU, LFU+prefetch "
                        "at C=2; LRU, LFU, LFU+prefetch at C=6) "
                        "for 8x7B, configs[4] (LFU+prefetch at C=4) for 8x22B")
    p.add_argument("--e2e-steps", type=int, default=-1,
                   help="tokens replayed through the public API (-1 = all --steps timed tokens, "
                        "0 = skip; same stream and starting cache state as the timed region)")
    p.add_argument("--cpu-sample-tokens", type=int, default=32)
    p.add_argument("--cpu-sample-layers", type=int, default=8,
                   help="layers the CPU path times (fp64 experts of 8 layers: 90 GB for 8x7B; "
                        "clamped to what fits in 45%% of free host RAM)")
    p.add_argument("--cpu-repeats", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--layers", type=int, default=0,
                   help="fewer layers than the model (invalidates the headline; diagnostics)")
    p.add_argument("--model", choices=["mixtral_8x7b", "mixtral_8x22b"], default="mixtral_8x7b")
    p.add_argument("--compress", choices=["auto", "on", "off"], default="auto",
                   help="exponent-coded (lossless) expert transfers; auto = on with a private store")
    p.add_argument("--store-layers", type=int, default=-1,
                   help="host expert store depth; -1 = all layers if they fit in 85%% of host RAM, "
                        "else as many as fit (deeper layers alias l %% S; SURVEY H5)")
    p.add_argument("--sweep-cache", default="",
                   help="e.g. 2,4,6: LFU and LFU+prefetch at each cache size (configs[2])")
    p.add_argument("--prefill-tokens", type=int, default=512,
                   help="configs[3]: prefill this many tokens (tcgen05 GEMM path), 0 = skip")
    p.add_argument("--prefill-decode", type=int, default=256,
                   help="decode tokens timed after the prefill (configs[3]: 256)")
    p.add_argument("--trace-variants", default="zipf:1.0",
                   help="trace-driven decode (SURVEY 8f.3): comma list of zipf:<skew> / "
                        "markov:<repeat_prob>; LRU and LFU on each; '' = skip")
    p.add_argument("--tiny-tokens", type=int, default=1024,
                   help="configs[0]: tiny toy-MoE decode (L=4,E=8,K=2,d=256), LRU C=2; 0 = skip")
    p.add_argument("--replay-streams", type=int, default=2048,
                   help="SURVEY 8f.1 replay sweep: independent layer streams (0 = skip)")
    p.add_argument("--replay-tokens", type=int, default=8192)
    p.add_argument("--shared-store", action="store_true",
                   help="host experts in a node-shared segment (automatic when WORLD_SIZE > 1)")
    p.add_argument("--peer-tier", action="store_true",
                   help="N>1: NVLink peer-HBM miss tier (SURVEY 8f.4): each replica holds 1/N of "
                        "the raw experts in HBM and serves the others' misses over NVLink")
    p.add_argument("--section-8x22b", type=int, default=1,
                   help="configs[4] section after the configs[1] run: 8x22B engine in a child "
                        "bench (LFU + prefetch, C=4), summarised in the line (0 = skip)")
    return p.parse_args()


# ---- distributed plumbing ----------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def gpu_of(local):
    """The rank's GPU: its local rank, or MOEB200_REPLICA_DEVICE for every rank (several
    replicas sharing one GPU -- a one-GPU check of the replica path; the ranks then talk gloo)."""
    dev = os.environ.get("MOEB200_REPLICA_DEVICE")
    return int(dev) if dev is not None else local


def dist_init(world, local):
    import torch
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available() and "MOEB200_REPLICA_DEVICE" not in os.environ:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")


def replicas_per_gpu(world):
    return int(os.environ.get("LOCAL_WORLD_SIZE", "1")) if "MOEB200_REPLICA_DEVICE" in os.environ else 1


def _coll_device():
    import torch
    import torch.distributed as dist

    return "cuda" if (torch.cuda.is_available() and dist.get_backend() == "nccl") else "cpu"


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def broadcast_ints(values, world):
    """Rank 0's integers on every rank (identical engine configs across replicas)."""
    if world == 1:
        return values
    import torch
    import torch.distributed as dist

    t = torch.tensor(values, dtype=torch.int64, device=_coll_device())
    dist.broadcast(t, src=0)
    return [int(v) for v in t.tolist()]


# ---- clocks ------------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.gpu_idle,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, names = [], None, set()
        keys = ["gpu_idle", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for k, v in zip(keys, parts[3:8]):
                if v.lower() == "active":
                    names.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(names), "samples": len(sm)}


# ---- helpers -----------------------------------------------------------------------------

def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


def host_available_bytes() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 62


def h2d_peak_gbs(dev) -> float:
    """Copy-engine H2D peak: 1 GiB pinned -> device, best of 5 (CUDA events)."""
    import torch

    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device=dev)
    best = float("inf")
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    del src, dst
    return n / (best / 1e3) / 1e9


def committed_ffn_traffic():
    """dram bytes per expert-FFN launch from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "ncu_ffn_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return None
    return None


# ---- CPU path (oracle port of the reference, test-infrastructure only) -------------------

def cpu_reference_sample(seed: int, tokens: int, layers: int, warmup: int, shape=(L, E, K, D, F),
                         layout: str = "ref", repeats: int = 3, cache_size: int = 4,
                         policy: int = 0, t_base: int = 0):
    """Time the oracle port on the stream's timed tokens [warmup, warmup + tokens) through the
    first `layers` layers, token-major like run_model (toymoe.py:175-185) plus the policy
    replay (kernels.py:60-147); best of `repeats`; tokens/s scaled to the full depth by
    L / layers (every layer does identical work).  layout "ref": the reference's arithmetic
    (numpy fp64, `h @ W`, BASELINE.md variant (i)); "dev": the tuned variant (ii), fp32 `W h`
    GEMVs on the weights' row-major (nn.Linear) layout.  All host BLAS threads.  The weights
    are materialised first (untimed).  Returns (baseline dict, acts (tokens, layers, K))."""
    import numpy as np

    import oracle
    from oracle.model import replay_layers

    Ls, Es, Ks, Ds, Fs = shape
    per = fp64_layer_bytes(shape) * (1.0 if layout == "ref" else 0.5)
    layers = max(1, min(layers, Ls, int(0.45 * host_available_bytes() // per)))
    alpha = 0.1 * math.sqrt(16 / Ds)
    ref = oracle.MixtralRef(Ls, Es, Ks, Ds, Fs, alpha, seed=seed, layout=layout,
                            layers=list(range(layers)), rms_norm=True)
    X = oracle.MixtralRef.inputs(seed, tokens, Ds, t0=t_base + warmup)
    t_gen = time.perf_counter()
    ref.materialize()
    t_gen = time.perf_counter() - t_gen
    times, acts = [], None
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        _, acts = ref.decode(X)
        replay_layers(acts, Es, cache_size, policy)
        times.append(time.perf_counter() - t0)
    del ref
    best = min(times)
    per_token = best / tokens * (Ls / layers)
    what = "numpy fp64 `h @ W`" if layout == "ref" else "numpy fp32 `W h`, row-major weights"
    return ({"value": 1.0 / per_token, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
             "sample": f"{tokens} tokens x {layers} of {Ls} layers ({what}, {os.cpu_count()} BLAS "
                       f"threads) + the policy replay, best of {len(times)}, scaled by {Ls}/{layers}",
             "layers_sampled": layers, "scale": Ls / layers, "tokens": tokens,
             "repeats": len(times), "best_s": best, "seconds_timed": sum(times),
             "materialise_s_untimed": t_gen}, acts)


def run_reference(args, world, rank, local):
    """--impl reference: the reference's CPU path (oracle port) on the same config."""
    if rank != 0:
        return
    shape = MODELS[args.model]
    policy = "lfu+prefetch" if args.model == "mixtral_8x22b" else "lru"
    cpu, _ = cpu_reference_sample(args.seed, args.cpu_sample_tokens, args.cpu_sample_layers,
                                  args.warmup, shape=shape, repeats=args.cpu_repeats,
                                  cache_size=args.cache_size, policy=1 if policy.startswith("lfu") else 0)
    value = cpu["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.model, world, args.cache_size, policy),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": f"each step = {cpu['tokens']} timed tokens x {cpu['layers_sampled']} layers on the "
                f"host (the driver's --steps/--warmup size nothing here); value = tokens/s of the "
                f"full {shape[0]}-layer model from the measured per-layer time (x {cpu['scale']:g})",
    }
    print(json.dumps(line), flush=True)


# ---- our engine ------------------------------------------------------------------------

def speculation_precision(rec) -> float:
    """metrics.speculation_metrics precision (metrics.py:217-249) of the engine's
    reference-definition guesses (gate l on the output of l-1) over the timed tokens."""
    g, a = rec["guessed"], rec["acts"][:, 1:, :]
    if g.size == 0:
        return None
    tp = sum(len(set(g[t, l]) & set(a[t, l])) for t in range(g.shape[0]) for l in range(g.shape[1]))
    return tp / g.size


def early_precision(rec, early):
    """Precision of the early guesses the prefetch acted on: |early(t, l) & acts(t, l+1)| / K,
    the reference's speculation precision (metrics.py:217-249) applied to gate_{l+1}(h'_l)."""
    a = rec["acts"][:, 1:, :]
    if early is None or early.size == 0:
        return None
    tp = sum(len(set(early[t, l]) & set(a[t, l])) for t in range(a.shape[0]) for l in range(a.shape[1]))
    return tp / early.size


def variant_parity(rec_all, rec, gaps, early, s0, s1, policy, csize, nb, n_exp):
    """Parity of one timed variant, checked here against the oracle (bench's checker role):
    the live cache trace of every token since the variant's cold start (rec_all: warm-up +
    timed) against the C oracle's replay of the engine's own selections (kernels.py:60-147);
    with prefetch, the timed region's issued / used decisions against oracle.prefetch_oracle;
    the timed selections' near-tie margins as the engine recorded them."""
    import numpy as np

    from oracle.model import prefetch_oracle, replay_layers

    code, df, dp = policy.device_params()
    rb, ev = replay_layers(rec_all["acts"], n_exp, csize, code, df, dp)
    out = {"trace_equals_oracle_replay": bool(
               np.array_equal(rec_all["resident_before"], np.transpose(rb, (1, 0, 2)))
               and np.array_equal(rec_all["evicted"], np.transpose(ev, (1, 0, 2)))),
           "near_ties_lt_1e-3": int((gaps < TIE_TOL).sum()),
           "min_topk_gap": float(np.nanmin(gaps)) if gaps.size else None,
           "steps": int(gaps.size)}
    if early is not None:
        issued, used = prefetch_oracle(rec["acts"], early, rec["resident_before"], nb)
        out["prefetch_issued_used_equal_oracle"] = bool(
            int(issued.sum()) == s1["prefetch_issued"] - s0["prefetch_issued"]
            and int(used.sum()) == s1["prefetch_used"] - s0["prefetch_used"])
    return out


def fp64_selection_check(head_rec, head_gaps, cpu_acts):
    """The headline's expert selections against the fp64 oracle's on the same tokens: the CPU
    baseline decoded the headline's timed tokens through the first layers in the reference's
    arithmetic, so its selections are compared step by step (toymoe.py:114 order)."""
    import numpy as np

    n = min(head_rec["acts"].shape[0], cpu_acts.shape[0])
    ls = cpu_acts.shape[1]
    eng = head_rec["acts"][:n, :ls]
    diff = (eng != cpu_acts[:n]).any(-1)
    near = head_gaps[:n, :ls] < TIE_TOL
    return {"tokens": n, "layers": ls, "steps": int(n * ls), "equal_steps": int((~diff).sum()),
            "mismatches": int(diff.sum()), "mismatches_at_near_ties": int((diff & near).sum()),
            "all_equal": bool(not diff.any())}


def parse_variant(v: str, default_c: int):
    """'lru' | 'lfu' | 'lfu+prefetch' | 'lfu@6' | 'lfu+prefetch@2' -> (policy, C, prefetch)."""
    from paper_2511_05814_b200.policies import PolicyKind

    name, _, c = v.partition("@")
    policy = PolicyKind.lfu() if name.startswith("lfu") else PolicyKind.lru()
    return policy, int(c) if c else default_c, "prefetch" in name


def run_ours(args, world, rank, local):
    gpu = gpu_of(local)
    import torch

    from paper_2511_05814_b200 import _native, replicas
    from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine, hash_weights, tensor_id

    dev = torch.device("cuda", gpu)
    torch.cuda.set_device(dev)
    factory = EngineConfig.mixtral_8x22b if args.model == "mixtral_8x22b" else EngineConfig.mixtral_8x7b
    if args.variants is None:
        args.variants = ("lfu+prefetch" if args.model == "mixtral_8x22b" else
                         "lru,lfu,lfu+prefetch,lru+prefetch,lfu@2,lfu+prefetch@2,lru@6,lfu@6,lfu+prefetch@6")
    variants = [v for v in args.variants.split(",") if v]
    if args.sweep_cache:
        variants = [f"{p}@{c}" for c in args.sweep_cache.split(",") for p in ("lfu", "lfu+prefetch")]
    parsed = [parse_variant(v, args.cache_size) for v in variants]
    cap_c = max(c for _, c, _ in parsed)
    want_prefetch = any(pf for _, _, pf in parsed)
    base_cfg = factory()
    nl = args.layers or base_cfg.num_layers
    # host memory: raw store + coded store when both fit; else the coded store alone
    # (compress = 2, private stores); else raw with layer aliasing
    shared = world > 1 or args.shared_store
    per_layer = base_cfg.num_experts * base_cfg.expert_bytes
    budget = 0.85 * host_available_bytes()
    store_layers, compress = args.store_layers, 0
    want_comp = args.compress != "off"
    if want_comp and nl * per_layer * 1.75 <= budget:
        compress = 1
    elif want_comp and not shared:
        compress = 2
        if store_layers < 0 and nl * per_layer * 0.67 > budget:
            store_layers = max(1, int(budget // (0.67 * per_layer)))
    elif want_comp and args.compress == "on":
        compress = 1
    if store_layers < 0:
        store_layers = 0 if (compress == 2 or nl * per_layer * (1.75 if compress else 1.0) <= budget) \
            else max(1, int(budget // (per_layer * (1.75 if compress else 1.0))))
    # HBM: per-layer pool of C policy + S staging buffers; deeper models stage 1 guess per layer
    import torch as _t
    hbm = _t.cuda.get_device_properties(gpu).total_memory // max(1, replicas_per_gpu(world))
    dense = nl * (2 * base_cfg.hidden_dim ** 2 + 4 * base_cfg.num_experts * base_cfg.hidden_dim)
    pf_bufs = 0
    if want_prefetch and nl * (cap_c + base_cfg.top_k) * base_cfg.expert_bytes + dense > 0.9 * hbm:
        pf_bufs = 1
    # every replica must build the same engine (shared stores): rank 0's host view decides
    store_layers, pf_bufs, compress = broadcast_ints([store_layers, pf_bufs, int(compress)], world)
    cfg = factory(num_layers=nl, cache_size=cap_c, prefetch="early" if want_prefetch else "off",
                  max_tokens=4096, device=gpu, store_layers=store_layers,
                  prefetch_buffers=pf_bufs, compress=compress)
    D, F, EB = cfg.hidden_dim, cfg.ffn_dim, cfg.expert_bytes
    cpu = cpu32 = cpu_acts = None
    head_policy, _, _ = parsed[0]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        shape = MODELS[args.model]
        # (i) the reference's arithmetic (the baseline); (ii) a tuned fp32 port beside it
        # (report both).  Same token stream as the engine's timed tokens: the
        # fp64 selections double as a full-scale parity check of the headline's first layers
        code = head_policy.device_params()[0]
        cpu, cpu_acts = cpu_reference_sample(args.seed, args.cpu_sample_tokens, args.cpu_sample_layers,
                                             args.warmup, shape=shape, repeats=args.cpu_repeats,
                                             cache_size=parsed[0][1], policy=code)
        cpu32, _ = cpu_reference_sample(args.seed, args.cpu_sample_tokens, args.cpu_sample_layers,
                                        args.warmup, shape=shape, layout="dev",
                                        repeats=args.cpu_repeats, cache_size=parsed[0][1], policy=code)
    pcie_peak = h2d_peak_gbs(dev)

    t_setup = time.perf_counter()
    store = None
    coded = None
    local_rank, local_world = replicas.local_world()
    if world > 1 or args.shared_store:
        # one host copy of the experts per node, page-locked by every local replica
        nbytes = cfg.host_store_layers * cfg.num_experts * EB
        name = replicas.store_name(cfg, args.seed, os.environ.get("TORCHELASTIC_RUN_ID", ""))
        holder = {}

        def fill(st):
            holder["eng"] = OffloadEngine(cfg, store=st)
            holder["eng"].init_random(args.seed)

        store = replicas.open_shared_store(name, nbytes, local_rank, lambda: barrier(world), fill)
        eng = holder.get("eng")
        if eng is None:
            eng = OffloadEngine(cfg, store=store)
            eng.init_random(args.seed, init_experts=False)
        if cfg.compress == 1:
            coded = replicas.open_shared_coded(name + "x", eng, local_rank, lambda: barrier(world))
    else:
        eng = OffloadEngine(cfg)
        eng.init_random(args.seed)
    peer = None
    if args.peer_tier and world > 1:
        import torch.distributed as dist

        def gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        peer = replicas.open_peer_tier(eng, rank, world, gather)
        barrier(world)
    t_setup = time.perf_counter() - t_setup
    st0 = eng.stats()
    compressed_ratio = (st0["compressed_store_bytes"] / (cfg.host_store_layers * cfg.num_experts * EB)
                        if cfg.compress else 1.0)
    # independent request stream per rank: token inputs from the counter hash (f32, std 1)
    base = replicas.rank_token_base(rank)
    n_tok = args.warmup + args.steps
    inputs = torch.stack([hash_weights(args.seed, tensor_id(5, base + t), 1.0, D, "f32")
                          for t in range(n_tok)])
    stream = torch.cuda.current_stream()
    results = {}
    launches_timed = None
    ktimes = None
    profiled_tps = None
    clocks = None
    e2e = None
    for v, (policy, csize, prefetch) in zip(variants, parsed):
        eng.set_mode(policy=policy, cache_size=csize, prefetch="early" if prefetch else "off")
        t0_tok = eng.tokens_done
        eng.decode_device(inputs[: args.warmup])
        eng.sync()
        headline = v == variants[0]
        s0 = eng.stats()
        n0 = _native.kernel_launches()
        barrier(world)
        torch.cuda.synchronize()
        sampler = ClockSampler(gpu) if headline else None
        if sampler:
            sampler.__enter__()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.decode_device(inputs[args.warmup: args.warmup + args.steps])
        b.record(stream)
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__()
            clocks = sampler.summary()
        barrier(world)
        tps, ms, total_tok = replicas.reduce_timing(a.elapsed_time(b), args.steps, world)
        eng.sync()
        n1 = _native.kernel_launches()
        s1 = eng.stats()
        if headline:
            launches_timed = n1 - n0
            # kernel timings: the same tokens replayed from the same (cold + warm-up) state with
            # per-launch CUDA events and in-kernel spans; the events slow a DMA-bound decode by a
            # few percent, so the headline value above is taken without them
            eng.reset()
            eng.decode_device(inputs[: args.warmup])
            eng.sync()
            eng.profile(True)
            k0 = eng.kernel_times()
            torch.cuda.synchronize()
            pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            pa.record(stream)
            eng.decode_device(inputs[args.warmup: args.warmup + args.steps])
            pb.record(stream)
            torch.cuda.synchronize()
            eng.sync()
            k1 = eng.kernel_times()
            eng.profile(False)
            ktimes = {k: k1[k] - k0[k] for k in k1}
            profiled_tps = args.steps / (pa.elapsed_time(pb) / 1e3)
        hits, misses = s1["hits"] - s0["hits"], s1["misses"] - s0["misses"]
        demand = s1["demand_bytes"] - s0["demand_bytes"]
        h2d = s1["h2d_bytes"] - s0["h2d_bytes"]
        demand_link = s1["demand_link_bytes"] - s0["demand_link_bytes"]
        busy = s1["copy_busy_ms"] - s0["copy_busy_ms"]
        rec = eng.records(t0_tok + args.warmup, args.steps)
        gaps = eng.record_gaps(t0_tok + args.warmup, args.steps)
        early = eng.record_early_guesses(t0_tok + args.warmup, args.steps) if prefetch else None
        nb = csize + ((cfg.prefetch_buffers or cfg.top_k) if prefetch else 0)
        # the trace is replayed from the cold cache set_mode left, warm-up tokens included
        rec_all = eng.records(t0_tok, args.warmup + args.steps)
        par = variant_parity(rec_all, rec, gaps, early, s0, s1, policy, csize, nb, cfg.num_experts)
        if headline:
            head_rec, head_gaps = rec, gaps
        results[v] = {
            "policy": str(policy), "cache_size": csize, "prefetch": prefetch,
            "tokens_per_s": tps,
            "ms_per_step": ms / args.steps,
            "hit_rate": hits / max(1, hits + misses),
            "misses_per_token": misses / args.steps,
            "h2d_GBps": h2d / (ms / 1e3) / 1e9,
            "demand_copy_GBps": demand_link / (busy / 1e3) / 1e9 if busy > 0 else None,
            "pcie_frac_of_measured_h2d_peak": (h2d / (ms / 1e3) / 1e9) / pcie_peak,
            "pcie_bound_tokens_per_s": pcie_peak * 1e9 / max(1.0, misses / args.steps * EB * compressed_ratio),
            "expert_GBps_delivered": (demand + s1["prefetch_bytes"] - s0["prefetch_bytes"]
                                      + s1["prefill_bytes"] - s0["prefill_bytes"]) / (ms / 1e3) / 1e9,
            "peer_tier_GBps": (s1["peer_bytes"] - s0["peer_bytes"]) / (ms / 1e3) / 1e9,
            "prefetch_issued": s1["prefetch_issued"] - s0["prefetch_issued"],
            "prefetch_used": s1["prefetch_used"] - s0["prefetch_used"],
            "prefetch_wasted_bytes": s1["prefetch_wasted_bytes"] - s0["prefetch_wasted_bytes"],
            "speculation_precision": speculation_precision(rec),
            "early_guess_precision": early_precision(rec, early) if prefetch else None,
            "check_hits_from_records": int(sum(
                int(rec["resident_before"][t, l, rec["acts"][t, l]].sum())
                for t in range(args.steps) for l in range(nl))) == hits,
            "parity": par,
        }
        ne = args.steps if args.e2e_steps < 0 else min(args.e2e_steps, args.steps)
        if headline and ne > 0:
            # public API, host buffers: H2D of the input and D2H of the output every step, on the
            # same token stream from the same (cold + warm-up) cache state as the timed region:
            # exactly the timed tokens, so its misses and copies are the headline's
            xs = inputs[args.warmup: args.warmup + ne].cpu().numpy()
            eng.reset()
            eng.decode_device(inputs[: args.warmup])
            eng.sync()
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            for i in range(ne):
                eng.decode(xs[i: i + 1])
            e_tps, _, _ = replicas.reduce_timing((time.perf_counter() - t0) * 1e3, ne, world)
            e2e = {"value": e_tps, "unit": "tokens/s",
                   "h2d_bytes_per_step": D * 4, "d2h_bytes_per_step": D * 4,
                   "tokens": ne, "same_tokens_as_timed_region": ne == args.steps}
    trace_driven = run_trace_driven(args, eng, inputs, stream, world) if args.trace_variants else None
    prefill = None
    if args.prefill_tokens > 0:
        prefill = run_prefill(args, eng, inputs, base, stream, world, pcie_peak)
    eng.close()
    peer = None   # the peer tier's HBM (and mapped peers) after the engine that used it
    if coded is not None:
        barrier(world)
        coded.close()
    gemm_iso = isolated_gemm(D, F) if rank == 0 and args.prefill_tokens > 0 else None
    gemm_iso_t = isolated_gemm(D, F, 1024) if rank == 0 and args.prefill_tokens > 0 else None
    tiny = run_tiny(args) if rank == 0 and world == 1 and args.tiny_tokens > 0 else None
    replay = run_replay(args) if rank == 0 and world == 1 and args.replay_streams > 0 else None
    # last of the GPU sections: its allocations and frees cannot disturb the timed ones above
    ffn_iso = isolated_ffn(D, F) if rank == 0 and world == 1 else None
    if store is not None:
        barrier(world)
        store.close()
    # every replica checked its own live traces against the oracle replay: count them
    ranks_ok = sum_over_ranks(float(all(r["parity"]["trace_equals_oracle_replay"]
                                        and r["parity"].get("prefetch_issued_used_equal_oracle", True)
                                        for r in results.values())), world)
    if rank != 0:
        return
    head = results[variants[0]]
    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # dominant kernel = the expert FFN launches that stream weights (device-counted bytes);
    # the all-launch figure (incl. phase launches that found no expert) is reported beside
    ffn_gbs = (ktimes["ffn_active_bytes"] / (ktimes["ffn_active_ms"] / 1e3) / 1e9
               if ktimes["ffn_active_ms"] > 0 else None)
    ffn_all_gbs = (ktimes["ffn_expert_runs"] * EB / (ktimes["ffn_ms"] / 1e3) / 1e9
                   if ktimes["ffn_ms"] > 0 else None)
    traffic = committed_ffn_traffic() if args.model == "mixtral_8x7b" else None
    xb, xms, xkms = ktimes.get("xdec_bytes", 0), ktimes.get("xdec_ms", 0.0), ktimes.get("xdec_kernel_ms", 0.0)
    roofline_decode = None
    if xb and xms > 0:
        roofline_decode = {
            "kernel": "xc::decode23p_kernel: exponent-coded expert parts -> bf16 in the cache buffer",
            "bound": "hbm", "achieved": xb / (xms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": xb / (xms / 1e3) / 1e9 / hbm_peak,
            "achieved_in_kernel": xb / (xkms / 1e3) / 1e9 if xkms > 0 else None,
            "frac_in_kernel": xb / (xkms / 1e3) / 1e9 / hbm_peak if xkms > 0 else None,
            "launches": ktimes["xdec_launches"], "bytes_per_launch": xb / max(1, ktimes["xdec_launches"]),
            "algorithmic_bytes": "coded part read + bf16 weights written (~3.35 B / weight)",
            "traffic": 339.4e6, "traffic_unit": "DRAM bytes of one w1|w3-part launch (ncu --set full: "
                                                "160.6 MB read + 178.9 MB written; algorithmic 393.0 MB; "
                                                "profiles/ncu_xc_decode_r2.md)",
            "note": "persistent, bulk-copy fed; issue-bound in practice (ncu: issue slots 59 %, "
                    "DRAM 42 %, 98.3 us per 117 M-weight part); overlapped with the H2D copies except "
                    "for the step's last w2 piece",
            "peak_source": peaks.get("source", "MEASURED_PEAKS.json hbm_gbs"),
        }
    line = {
        "metric": METRIC,
        "value": head["tokens_per_s"],
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (counter-hash random-init weights and token inputs)",
        "config": workload_config(args.model, world, head["cache_size"], variants[0]),
        "engine": {
            "layers_run": nl, "setup_s": round(t_setup, 1), "shared_store": store is not None,
            "host_store_layers": cfg.host_store_layers,
            "expert_transfer": ("exponent-coded bf16, lossless (csrc/expcodec.cuh), "
                                f"{compressed_ratio:.3f} of the raw bytes"
                                + (", coded store only" if cfg.compress == 2 else "")
                                if cfg.compress else "raw bf16"),
            "prefetch_buffers_per_layer": (cfg.prefetch_buffers or cfg.top_k) if want_prefetch else 0,
            "peer_tier": (f"NVLink peer-HBM tier: 1/{world} of the raw experts per replica's HBM, "
                          "misses of peer-homed experts copied device to device"
                          if args.peer_tier and world > 1 else "off"),
        },
        "hit_rate": head["hit_rate"],
        "variants": results,
        "pcie": {"bound": "pcie", "achieved": head["h2d_GBps"], "peak": pcie_peak,
                 "unit": "GB/s", "frac": head["h2d_GBps"] / pcie_peak,
                 "copy_engine_GBps_while_busy": head["demand_copy_GBps"],
                 "peak_source": "measured here: 1 GiB pinned cudaMemcpyAsync, best of 5"},
        "roofline_ffn": {
            "kernel": "expert FFN: stream_gemv_kernel up (w1|w3) + down (w2), bulk-copy pipelines",
            "bound": "hbm", "achieved": ffn_gbs, "peak": hbm_peak, "unit": "GB/s",
            "frac": ffn_gbs / hbm_peak if ffn_gbs else None,
            "launches": ktimes["ffn_active_launches"],
            "bytes_per_launch": (ktimes["ffn_active_bytes"] / ktimes["ffn_active_launches"]
                                 if ktimes["ffn_active_launches"] else None),
            "achieved_incl_empty_phase_launches": ffn_all_gbs,
            "achieved_in_kernel": (ktimes["ffn_active_bytes"] / (ktimes["ffn_kernel_ms"] / 1e3) / 1e9
                                   if ktimes.get("ffn_kernel_ms") else None),
            "frac_in_kernel": (ktimes["ffn_active_bytes"] / (ktimes["ffn_kernel_ms"] / 1e3) / 1e9 / hbm_peak
                               if ktimes.get("ffn_kernel_ms") else None),
            "in_kernel_note": "globaltimer span first CTA start -> last CTA end per launch. The "
                              "CUDA-event span of a single launch is inflated while the copy "
                              "engine runs: tools/event_chunk_probe.py times a 235 MB elementwise "
                              "SM kernel at 78 us alone and at ~103 us with an event pair per "
                              "launch while >= 16 MB host->device copies are in flight "
                              "(profiles/box_probe_r2.md). The events are recorded on an "
                              "identical replay of the timed tokens, not in the headline run "
                              "(they slow it by 1-3 %: tools/profile_overhead_probe.py)",
            "traffic": traffic.get("dram_bytes_per_expert") if traffic else None,
            "traffic_unit": "DRAM bytes per expert (ncu, profiles/ncu_ffn_traffic.json)",
            "algorithmic_bytes_per_expert": EB,
            "peak_source": peaks.get("source", "MEASURED_PEAKS.json hbm_gbs"),
        },
        "roofline_decode": roofline_decode,
        "ffn_isolated_events": ffn_iso,
        "kernel_timing": ("per-launch CUDA events + in-kernel spans on an identical replay of the "
                          "timed tokens (same starting cache state); that replay ran at "
                          f"{profiled_tps:.3f} tokens/s, the headline without the events"),
        "kernel_ms_per_step": {k: ktimes[k] / args.steps for k in ("mix_ms", "gate_ms", "ffn_ms",
                                                                 "finalize_ms", "xdec_ms",
                                                                 "ffn_kernel_ms", "xdec_kernel_ms")},
    }
    # the dominant kernel = the larger in-kernel device time over the timed region
    ffn_k, dec_k = ktimes.get("ffn_kernel_ms", 0.0), ktimes.get("xdec_kernel_ms", 0.0)
    dom = "decode" if roofline_decode and dec_k > ffn_k else "ffn"
    line["roofline"] = dict(roofline_decode if dom == "decode" else line["roofline_ffn"])
    line["roofline"]["dominant_by"] = (f"in-kernel device time in the timed region: expert FFN "
                                       f"{ffn_k / args.steps:.2f} ms/step, exponent decode "
                                       f"{dec_k / args.steps:.2f} ms/step; the other kernel's object "
                                       f"is roofline_{'ffn' if dom == 'decode' else 'decode'}")
    if cpu32:
        line["cpu_baseline_fp32"] = cpu32
        line["speedup_vs_cpu_port_fp32"] = head["tokens_per_s"] / cpu32["value"]
    if trace_driven:
        line["trace_driven"] = trace_driven
    if tiny:
        line["tiny"] = tiny
    if replay:
        line["replay"] = replay
    if prefill:
        tf_peak = float(peaks.get("bf16_tflops", 1590.0))
        for rec in [prefill["gemm"]] + [r for r in (gemm_iso, gemm_iso_t) if r]:
            rec["tensor_frac"] = rec["tflops"] / tf_peak
            rec["hbm_frac"] = rec["algorithmic_GBps"] / hbm_peak
            rec["bound"] = "tensor" if rec["tensor_frac"] >= rec["hbm_frac"] else "hbm"
            if rec.get("in_kernel_GBps"):
                rec["in_kernel_hbm_frac"] = rec["in_kernel_GBps"] / hbm_peak
                rec["in_kernel_tensor_frac"] = rec["in_kernel_tflops"] / tf_peak
            rec["peaks"] = {"bf16_tflops": tf_peak, "hbm_gbs": hbm_peak,
                            "source": peaks.get("source", "MEASURED_PEAKS.json")}
        prefill["gemm_isolated"] = gemm_iso
        prefill["gemm_isolated_tensor_bound"] = gemm_iso_t
        line["prefill"] = prefill
    # ---- the line's tail: the driver keeps the end of stdout, so the contract keys and the
    # metric's comparison table come last, compact
    roof = line.pop("roofline")
    line["roofline"] = {k: roof[k] for k in ("kernel", "bound", "achieved", "peak", "unit", "frac",
                                             "traffic", "achieved_in_kernel", "frac_in_kernel")
                        if k in roof}
    line["roofline"]["detail"] = "roofline_decode / roofline_ffn above"
    line["cpu_baseline"] = cpu
    line["e2e"] = e2e
    line["clocks"] = clocks
    line["gpu_launches"] = launches_timed
    if cpu:
        line["speedup_vs_cpu_port"] = head["tokens_per_s"] / cpu["value"]
    pars = [r["parity"] for r in results.values()]
    parity = {
        "traces_equal_oracle_replay_all_variants": all(p["trace_equals_oracle_replay"] for p in pars),
        "prefetch_issued_used_equal_oracle": all(p.get("prefetch_issued_used_equal_oracle", True)
                                                 for p in pars),
        "near_ties_lt_1e-3": sum(p["near_ties_lt_1e-3"] for p in pars),
        "steps_checked": sum(p["steps"] for p in pars),
        "min_topk_gap": min(p["min_topk_gap"] for p in pars),
    }
    if cpu_acts is not None:
        parity["fp64_selections_headline"] = fp64_selection_check(head_rec, head_gaps, cpu_acts)
    parity["replicas_with_oracle_equal_traces"] = f"{int(ranks_ok)}/{world}"
    parity["full_depth_tests"] = ("tests/test_fullscale_gpu.py: configs[1] 32 layers and the "
                                  "configs[4] shape vs the fp64 oracle")
    line["variants_summary"] = {
        v: {"tok_s": round(r["tokens_per_s"], 3), "hit": round(r["hit_rate"], 4),
            "pcie_frac": round(r["pcie_frac_of_measured_h2d_peak"], 3),
            "pcie_bound_tok_s": round(r["pcie_bound_tokens_per_s"], 2),
            "spec_prec": None if r["speculation_precision"] is None else round(r["speculation_precision"], 3),
            **({"early_prec": round(r["early_guess_precision"], 3),
                "pf_issued": r["prefetch_issued"], "pf_used": r["prefetch_used"],
                "pf_wasted_GB": round(r["prefetch_wasted_bytes"] / 1e9, 2)} if r["prefetch"] else {})}
        for v, r in results.items()}
    line["parity"] = parity
    if args.model == "mixtral_8x7b" and args.section_8x22b and world == 1:
        line["mixtral_8x22b"] = run_8x22b_section(args)
    print(json.dumps(line), flush=True)


def run_8x22b_section(args):
    """configs[4] in a child bench process (its own engine, host store and fp64 sample; the
    parent's 8x7B engine and stores are already released): LFU + prefetch at C = 4, the child's
    full line kept in its `detail`, the comparison numbers summarised here."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--model", "mixtral_8x22b",
           "--steps", str(args.steps), "--warmup", str(args.warmup), "--seed", str(args.seed),
           "--cpu-sample-layers", str(min(2, args.cpu_sample_layers)), "--cpu-sample-tokens", "16",
           "--cpu-repeats", "1",
           "--prefill-tokens", "0", "--tiny-tokens", "0", "--replay-streams", "0",
           "--trace-variants", "", "--section-8x22b", "0"]
    if args.layers:
        cmd += ["--layers", str(args.layers)]
    if args.no_cpu_baseline:
        cmd += ["--no-cpu-baseline"]
    t0 = time.perf_counter()
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    wall = time.perf_counter() - t0
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode != 0 or not lines:
        return {"error": f"rc={out.returncode}: {out.stderr[-400:]}"}
    d = json.loads(lines[-1])
    v = d["variants"][next(iter(d["variants"]))]
    return {"workload": d["config"]["workload"], "tok_s": d["value"],
            "e2e_tok_s": (d.get("e2e") or {}).get("value"), "hit": round(d["hit_rate"], 4),
            "pcie_frac": round(d["pcie"]["frac"], 3),
            "cpu_tok_s": (d.get("cpu_baseline") or {}).get("value"),
            "speedup_vs_cpu_port": d.get("speedup_vs_cpu_port"),
            "host_store_layers": d["engine"]["host_store_layers"], "setup_s": d["engine"]["setup_s"],
            "pf_issued": v["prefetch_issued"], "pf_used": v["prefetch_used"],
            "parity": d["parity"], "child_wall_s": round(wall, 1)}


def run_tiny(args):
    """configs[0]: the reference's own tiny config (ToyModelConfig(ModelShape(4, 8, 2), d=256,
    alpha=0.1, seed=42), T tokens, LRU cache 2/layer) through the engine (toy tanh experts, f32),
    beside the reference algorithm on the host (oracle port of toymoe.run_model + the policy
    replay, numpy fp64).  Latency-bound: reported as tokens/s, us/token and launches/token,
    with the engine's activation trace checked against the oracle's."""
    import numpy as np
    import torch

    import oracle
    from oracle.model import replay_layers
    from paper_2511_05814_b200 import _native
    from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine
    from paper_2511_05814_b200.policies import PolicyKind
    from paper_2511_05814_b200.toymoe import ToyModelConfig, ToyMoeModel
    from paper_2511_05814_b200.traces import ModelShape

    Lt, Et, Kt, dt, T = 4, 8, 2, 256, args.tiny_tokens
    cfg = ToyModelConfig(ModelShape(Lt, Et, Kt), hidden_dim=dt, mixing_scale=0.1, seed=42, tokens=T)
    model, rng = ToyMoeModel.build(cfg)
    inputs = rng.standard_normal((T, dt))
    reps = 3
    ecfg = EngineConfig(num_layers=Lt, num_experts=Et, top_k=Kt, hidden_dim=dt, expert_kind="toy_tanh",
                        cache_size=2, policy=PolicyKind.lru(), mixing_scale=0.1,
                        max_tokens=(reps + 1) * T + 64)
    stream = torch.cuda.current_stream()
    with OffloadEngine(ecfg) as eng:
        eng.load_toy_model(model)
        x = torch.from_numpy(inputs.astype(np.float32)).cuda()
        # warm-up: the whole stream once (a ~0.1 s latency-bound section follows CPU-only work,
        # so the GPU must be back at full clock), then the best of `reps` cold-cache passes
        eng.decode_device(x)
        eng.sync()
        ms, launches = float("inf"), 0
        for r in range(reps):
            eng.reset()
            n0 = _native.kernel_launches()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            eng.decode_device(x)
            b.record(stream)
            torch.cuda.synchronize()
            eng.sync()
            ms = min(ms, a.elapsed_time(b))
            launches = _native.kernel_launches() - n0
        rec = eng.records(reps * T, T)
        eng.reset()
        t0 = time.perf_counter()
        eng.decode(inputs[:64].astype(np.float32))   # public API, host arrays, synced
        e2e_tps = 64 / (time.perf_counter() - t0)
    w = oracle.toy_weights(Lt, Et, dt, 1.0, 42, T)
    t0 = time.perf_counter()
    acts, _, _ = oracle.toy_run_model(Lt, Et, Kt, dt, 0.1, 1.0, 42, T, weights=w)
    replay_layers(acts, Et, 2, 0)
    cpu_s = time.perf_counter() - t0
    return {"workload": "configs[0]: tiny MoE (4 layers, 8 experts top-2, d=256) decode, LRU cache "
                        "2/layer (toy tanh experts, f32 on the GPU)",
            "tokens": T, "timing": f"best of {reps} cold-cache passes after a full warm-up pass",
            "tokens_per_s": T / (ms / 1e3), "us_per_token": ms * 1e3 / T,
            "launches_per_token": launches / T, "e2e_tokens_per_s": e2e_tps,
            "trace_equals_oracle": bool(np.array_equal(rec["acts"], acts)),
            "cpu_baseline": {"value": T / cpu_s, "unit": "tokens/s", "cores": os.cpu_count(),
                             "kind": "port",
                             "sample": f"oracle toy_run_model (numpy fp64, toymoe.py:159-190) + "
                                       f"policy replay, {T} tokens"}}


def run_replay(args):
    """the offline policy replay (K7, kernels.replay_policy / simulate's layer
    loop) as a sweep workload -- `replay_streams` independent Zipf layer streams of T steps,
    each replayed under LRU / LFU / LFU-aged at C = 2, 4, 6 (one warp per stream, inputs resident
    in HBM) -- beside the oracle's C replay (the reference algorithm, kernels.py:60-147) on all
    host threads.  Decisions are checked equal on a sample."""
    import concurrent.futures as cf
    import ctypes

    import numpy as np
    import torch

    import oracle
    from paper_2511_05814_b200 import _native
    from paper_2511_05814_b200.tracegen import ZipfParams, gen_zipf
    from paper_2511_05814_b200.traces import ModelShape

    S, T, Er, Kr = args.replay_streams, args.replay_tokens, 8, 2
    tr = gen_zipf(ZipfParams(ModelShape(S, Er, Kr), T, skew_exponent=1.0, seed=args.seed))
    acts = np.ascontiguousarray(np.transpose(tr.activations, (1, 0, 2)))          # (S, T, K)
    lib = _native.lib()
    d_acts = torch.from_numpy(acts).cuda()
    rb = torch.empty((S, T, Er), dtype=torch.uint8, device="cuda")
    ev = torch.empty_like(rb)
    configs = [(0, 1.0, 1), (1, 1.0, 1), (2, 0.5, 16)]
    caps = (2, 4, 6)
    stream = torch.cuda.current_stream()
    sp = _native.stream_ptr()

    def one(code, df, dp, C):
        _native.check(lib.moe_replay_policy_layers(d_acts.data_ptr(), S, T, Kr, Er, C, code, df, dp,
                                                   rb.data_ptr(), ev.data_ptr(), sp))

    for code, df, dp in configs:       # warm-up
        one(code, df, dp, 4)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for code, df, dp in configs:
        for C in caps:
            one(code, df, dp, C)
    b.record(stream)
    torch.cuda.synchronize()
    gpu_s = a.elapsed_time(b) / 1e3
    steps = S * T * len(configs) * len(caps)
    # the last launch (LFU-aged, C = 6) against the oracle on a sample of streams
    grb = rb.cpu().numpy()
    ok = all(np.array_equal(grb[i], oracle.replay_policy(acts[i], Er, 6, 2, 0.5, 16)[0])
             for i in range(0, S, max(1, S // 16)))
    # CPU: the oracle's C replay, one stream per task, all host threads (ctypes drops the GIL)
    ncpu = os.cpu_count() or 1
    cpu_streams = S
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(ncpu) as ex:
        for code, df, dp in configs:
            for C in caps:
                list(ex.map(lambda i: oracle.replay_policy(acts[i], Er, C, code, df, dp), range(cpu_streams)))
    cpu_s = time.perf_counter() - t0
    cpu_steps = cpu_streams * T * len(configs) * len(caps)
    return {"workload": f"SURVEY 8f.1 offline replay sweep: {S} Zipf(1.0) layer streams x {T} steps "
                        f"(E=8, K=2) x {{lru, lfu, lfu-aged:0.5:16}} x C in {{2,4,6}}",
            "steps": steps, "gpu_ms": gpu_s * 1e3, "steps_per_s": steps / gpu_s,
            "decisions_equal_oracle_sample": bool(ok),
            "cpu_baseline": {"value": cpu_steps / cpu_s, "unit": "steps/s", "cores": ncpu,
                             "kind": "port", "sample": f"oracle C replay (kernels.py:60-147), "
                                                       f"{cpu_streams} streams x 9 configs, {ncpu} threads"},
            "reference_published": "numba kernel ~25 M steps/s, one stream, 'typical machine' (pkg/README.md:144-145)"}


def run_trace_driven(args, eng, inputs, stream, world):
    """Decode with routing taken from a synthetic activation trace (gen_zipf / gen_markov, the
    reference's workload generators) instead of the gate: LRU vs LFU at the bench's cache size
    with real transfers (the paper's expert-imbalance study at Mixtral scale)."""
    import torch

    from paper_2511_05814_b200.policies import PolicyKind
    from paper_2511_05814_b200.traces import ModelShape
    from paper_2511_05814_b200.tracegen import MarkovParams, ZipfParams, gen_markov, gen_zipf

    cfg = eng.config
    shape = ModelShape(cfg.num_layers, cfg.num_experts, cfg.top_k)
    n = args.warmup + args.steps
    out = {}
    for spec in args.trace_variants.split(","):
        kind, _, val = spec.partition(":")
        v = float(val) if val else (1.0 if kind == "zipf" else 0.3)
        zp = ZipfParams(shape, n, skew_exponent=v if kind == "zipf" else 1.0, seed=args.seed)
        tr = gen_zipf(zp) if kind == "zipf" else gen_markov(MarkovParams(shape, n, v, zp, seed=args.seed))
        for pol in ("lru", "lfu"):
            eng.set_mode(policy=PolicyKind.parse(pol), cache_size=args.cache_size, prefetch="off")
            eng.decode_device(inputs[: args.warmup], routing=tr.activations[: args.warmup])
            eng.sync()
            s0 = eng.stats()
            barrier(world)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            eng.decode_device(inputs[args.warmup: n], routing=tr.activations[args.warmup: n])
            b.record(stream)
            torch.cuda.synchronize()
            eng.sync()
            ms = max_over_ranks(a.elapsed_time(b), world)
            s1 = eng.stats()
            hits, misses = s1["hits"] - s0["hits"], s1["misses"] - s0["misses"]
            out[f"{spec}/{pol}"] = {"tokens_per_s": args.steps / (ms / 1e3),
                                    "hit_rate": hits / max(1, hits + misses),
                                    "misses_per_token": misses / args.steps}
    return out


def run_prefill(args, eng, inputs, base, stream, world, pcie_peak):
    """configs[3]: cold LRU C=4 cache, prefill P tokens as one batch (mixing map and SwiGLU
    experts as tcgen05 grouped GEMMs, one H2D load per needed expert per layer), then decode."""
    import torch

    from paper_2511_05814_b200.engine import hash_weights, tensor_id
    from paper_2511_05814_b200.policies import PolicyKind

    P, Dd = args.prefill_tokens, inputs.shape[1]
    X = torch.stack([hash_weights(args.seed, tensor_id(5, base + 100000 + t), 1.0, Dd, "f32")
                     for t in range(P)])
    # warm-up: the first prefill on an engine allocates its batch buffers (~3 GB) and builds
    # the GEMM tile tables -- ~0.1 s that is not part of a prefill's steady-state cost
    eng.set_mode(policy=PolicyKind.lru(), cache_size=args.cache_size, prefetch="off")
    eng.prefill_device(X)
    torch.cuda.synchronize()
    eng.sync()
    # timed: cold cache, no per-launch events
    eng.set_mode(policy=PolicyKind.lru(), cache_size=args.cache_size, prefetch="off")
    s0 = eng.stats()
    barrier(world)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    eng.prefill_device(X)
    b.record(stream)
    torch.cuda.synchronize()
    ms_p = max_over_ranks(a.elapsed_time(b), world)
    eng.sync()
    s1 = eng.stats()
    # GEMM timings: the same prefill replayed from the same cold state with per-launch events
    eng.set_mode(policy=PolicyKind.lru(), cache_size=args.cache_size, prefetch="off")
    eng.profile(True)
    k0 = eng.kernel_times()
    eng.prefill_device(X)
    torch.cuda.synchronize()
    eng.sync()
    k1 = eng.kernel_times()
    eng.profile(False)
    k = {n: k1[n] - k0[n] for n in k1}
    nbytes = s1["prefill_bytes"] - s0["prefill_bytes"]
    hits, misses = s1["hits"] - s0["hits"], s1["misses"] - s0["misses"]
    out = {
        "workload": f"configs[3]: prefill {P} tokens (one batch) + decode, LRU cache "
                    f"{args.cache_size}/layer, cold start (after one untimed warm-up prefill; "
                    "GEMM timings from a profiled replay)",
        "prefill_tokens": P, "prefill_ms": ms_p,
        "prefill_tokens_per_s": sum_over_ranks(P / (ms_p / 1e3), world),
        "prefill_hit_rate": hits / max(1, hits + misses),
        "h2d_GB": nbytes / 1e9, "h2d_GBps": nbytes / (ms_p / 1e3) / 1e9,
        "pcie_frac_of_measured_h2d_peak": nbytes / (ms_p / 1e3) / 1e9 / pcie_peak,
        "gemm": {"kernel": "tc::grouped_gemm_kernel (tcgen05.mma 128x256x16, TMA, TMEM; mix + "
                           "SwiGLU up + split-K down), live in the prefill",
                 "launches": k["gemm_launches"], "ms": k["gemm_ms"],
                 "tflops": k["gemm_flops"] / (k["gemm_ms"] / 1e3) / 1e12 if k["gemm_ms"] else None,
                 "algorithmic_GBps": k["gemm_bytes"] / (k["gemm_ms"] / 1e3) / 1e9 if k["gemm_ms"] else None,
                 "in_kernel_ms": k["gemm_kernel_ms"],
                 "in_kernel_GBps": (k["gemm_bytes"] / (k["gemm_kernel_ms"] / 1e3) / 1e9
                                    if k["gemm_kernel_ms"] else None),
                 "in_kernel_tflops": (k["gemm_flops"] / (k["gemm_kernel_ms"] / 1e3) / 1e12
                                      if k["gemm_kernel_ms"] else None),
                 "share_of_prefill": k["gemm_ms"] / ms_p},
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_prefill_sample(args.seed, P, X)
        out["cpu_baseline_fp32"] = cpu_prefill_sample(args.seed, P, X, layout="dev")
    if args.prefill_decode > 0:
        xs = torch.stack([hash_weights(args.seed, tensor_id(5, base + 200000 + t), 1.0, Dd, "f32")
                          for t in range(args.prefill_decode)])
        h0 = eng.stats()
        a.record(stream)
        eng.decode_device(xs)
        b.record(stream)
        torch.cuda.synchronize()
        ms_d = max_over_ranks(a.elapsed_time(b), world)
        h1 = eng.stats()
        dh, dm = h1["hits"] - h0["hits"], h1["misses"] - h0["misses"]
        out["decode_after_prefill"] = {"tokens": args.prefill_decode,
                                       "tokens_per_s": args.prefill_decode / (ms_d / 1e3),
                                       "hit_rate": dh / max(1, dh + dm)}
        out["request_ms"] = ms_p + ms_d  # the whole configs[3] request: prefill + decode
    return out


def cpu_prefill_sample(seed, P, X, layers=1, layout="ref"):
    """configs[3] CPU side: the oracle's batched prefill restatement over the same P tokens on
    `layers` of the 32 layers, scaled by 32 / layers, all host threads; layout "ref": numpy
    fp64 in the reference's `h @ W` layout (variant (i)), "dev": the tuned fp32 port (ii).
    The experts are materialised untimed first."""
    import oracle
    from oracle.model import mixtral_prefill_fp32

    alpha = 0.1 * math.sqrt(16 / D)
    ref = oracle.MixtralRef(L, E, K, D, F, alpha, seed=seed, layout=layout,
                            layers=list(range(layers)), rms_norm=True)
    t_gen = time.perf_counter()
    ref.materialize()
    t_gen = time.perf_counter() - t_gen
    x = X.cpu().numpy()
    t0 = time.perf_counter()
    if layout == "ref":
        oracle.mixtral_prefill(ref, x)
    else:
        mixtral_prefill_fp32(ref, x)
    dt = time.perf_counter() - t0
    per_batch = dt * (L / layers)
    what = ("oracle.mixtral_prefill, numpy fp64 batched GEMMs" if layout == "ref" else
            "oracle.model.mixtral_prefill_fp32, numpy fp32 sgemm on row-major weights")
    return {"value": P / per_batch, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{P} tokens x {layers} of {L} layers ({what}), scaled by {L}/{layers}; "
                      f"{dt:.1f} s timed, {t_gen:.1f} s untimed weight materialisation"}


def isolated_ffn(Dd, Ff):
    """The decode FFN GEMVs alone (moe_microbench_gemv): resident experts, no copies in flight,
    20 back-to-back launches under one CUDA-event pair (launch gaps included) over rotating
    weight sets larger than L2 -- the event-timed counterpart of `roofline_ffn`'s in-kernel
    figure without the per-launch inflation concurrent DMA adds (profiles/box_probe_r2.md)."""
    import ctypes

    import torch

    from paper_2511_05814_b200 import _native

    lib = _native.lib()
    peak = float(measured_peaks().get("hbm_gbs", 6650.0))
    out = {}
    for name, kernel, experts in (("up_1_expert", 1, 1), ("up_2_experts", 1, 2),
                                  ("down_1_expert", 2, 1), ("down_2_experts", 2, 2)):
        ms, nb = ctypes.c_float(), ctypes.c_int64()
        _native.check(lib.moe_microbench_gemv(kernel, Dd, Ff, experts, 0, 6, 0, 0, 20,
                                              ctypes.byref(ms), ctypes.byref(nb)))
        gbs = nb.value / (ms.value / 1e3) / 1e9
        out[name] = {"us": round(ms.value * 1e3, 1), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3)}
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def isolated_gemm(Dd, Ff, m=128):
    """K4 alone: the 8 experts of one layer resident in HBM, m token rows each (m = 128: 512
    tokens x top-2, HBM-bound; m = 1024: 4096 tokens, tensor-bound): grouped SwiGLU up (w1|w3)
    then grouped down, CUDA events per launch."""
    import ctypes

    import torch

    from paper_2511_05814_b200 import _native

    lib = _native.lib()
    G = 8
    gm = (ctypes.c_int32 * G)(*([m] * G))
    X = torch.randn(G * m, Dd, device="cuda").bfloat16()
    W13 = (torch.randn(G, 2 * Ff, Dd, device="cuda") / Dd ** 0.5).bfloat16()
    act = torch.empty(G * m, Ff, device="cuda", dtype=torch.bfloat16)
    W2 = (torch.randn(G * Dd, Ff, device="cuda") / Ff ** 0.5).bfloat16()
    out = torch.empty(G * m, Dd, device="cuda", dtype=torch.float32)
    ms_u, ms_d = ctypes.c_float(0), ctypes.c_float(0)
    _native.check(lib.moe_tc_grouped_swiglu_bf16(X.data_ptr(), W13.data_ptr(), act.data_ptr(), G, gm,
                                                 Ff, Dd, 6, ctypes.byref(ms_u), _native.stream_ptr()))
    _native.check(lib.moe_tc_grouped_gemm_bf16(act.data_ptr(), W2.data_ptr(), out.data_ptr(), G, gm,
                                               Dd, Ff, 1, 6, ctypes.byref(ms_d), _native.stream_ptr()))
    torch.cuda.synchronize()
    rows = G * m
    flops = 2.0 * rows * 2 * Ff * Dd + 2.0 * rows * Ff * Dd
    nbytes = G * 3 * Ff * Dd * 2 + rows * Dd * 2 + 2 * rows * Ff * 2 + rows * Dd * 4
    ms = ms_u.value + ms_d.value
    del X, W13, act, W2, out
    torch.cuda.empty_cache()
    return {"kernel": f"tc::grouped_gemm_kernel isolated: 8 resident experts x {m} rows, SwiGLU up + "
                      "down (2 launches, weights 2.82 GB > L2)", "rows_per_expert": m,
            "up_ms": ms_u.value, "down_ms": ms_d.value, "ms": ms,
            "tflops": flops / (ms / 1e3) / 1e12, "algorithmic_GBps": nbytes / (ms / 1e3) / 1e9}


def main():
    args = parse_args()
    world, rank, local = dist_env()
    dist_init(world, local)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank, local)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    main()
